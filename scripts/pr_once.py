"""One C5 (or --workload) FFG build + PageRank on cuda:0, for ncu captures of a
single PageRank launch:

    ncu --set full -k regex:pagerank -c 1 python scripts/pr_once.py [c5|c3|c2] [reps] [hamming]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2210_01465_b200 as tk  # noqa: E402

SHAPES = {"c5": ([8, 8, 8, 6, 6, 6, 4, 4, 4, 4, 2, 2], 0, 0.10, 5),
          "c3": ([8, 8, 8, 8, 6, 6, 4, 4, 2, 2], 1, 0.0, 3),
          "c2": ([16, 12, 8, 8, 8, 4, 2, 2], 0, 0.30, 2)}


def main():
    radix, gen, q, seed = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "c5"]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    kind = tk.HAMMING if len(sys.argv) > 3 and sys.argv[3] == "hamming" else tk.ADJACENT
    with tk.Landscape(radix) as land:
        land.generate(gen, q, seed)
        land.build_ffg(kind, node_limit=1 << 32, emit_csr=False)
        for _ in range(reps):
            t0 = time.perf_counter()
            it, res, s = land.pagerank()
            info = land.kernel_info()
            print(f"iterations={it} res={res:.3e} sum={s:.15f} kernel={info['pagerank_kernel']} "
                  f"ms={info['ms_pagerank']:.3f} wall={1e3 * (time.perf_counter() - t0):.1f}")


if __name__ == "__main__":
    main()
