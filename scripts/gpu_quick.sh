mkdir -p gpurun_out/r02b
timeout 900 python -m pytest tests/test_descents.py tests/test_cpp_dropin.py tests/test_sharded.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r02b/pytest.log 2>&1; echo "exit=$?" >> gpurun_out/r02b/pytest.log
python - > gpurun_out/r02b/descent_time.txt 2>&1 <<'PY'
import time, numpy as np, oracle as O, paper_2210_01465_b200 as tk, torch
radix=[8, 8, 8, 6, 6, 6, 4, 4, 4, 4, 2, 2]
with tk.Landscape(radix, device=0) as land:
    land.generate(0, 0.10, 5)
    for kind in (1, 0):
        land.build_ffg(kind, node_limit=1<<32, emit_csr=False)
        for W in (10**6, 10**7, 10**8):
            land.descents(W, 1); torch.cuda.synchronize()
            t=time.time(); a,f,e=land.descents(W, 2); dt=time.time()-t
            print(f"kind={kind} walkers={W} {dt*1e3:.1f} ms evals={e} ({e/dt/1e9:.2f} G evals/s) at_minima={int(a.sum())} fail={f}")
PY
