import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2210_01465_b200 as tk
for radix, kind in (([8, 8, 6, 6, 4, 4, 2, 2], tk.ADJACENT), ([8, 4, 4, 4, 2, 2, 4], tk.HAMMING)):
    fit, ok = O.gen_iid(O.space_size(radix), 0.2, 3)
    with tk.Landscape(radix) as land:
        land.load_dense(fit, ok)
        s = land.analyze(kind, emit_csr=True, node_limit=1 << 32)
        print(radix, kind, s.n_edges, s.iterations)
