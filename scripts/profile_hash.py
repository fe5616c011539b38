"""Sparse ingestion at C5 scale: the valid-set hash table build + densify
(tk_land_load_sparse), timed with CUDA events, for the ncu hash-probe L2 hit
rate capture:

    python scripts/profile_hash.py                       # timing line (JSON)
    ncu --metrics lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,\
gpu__time_duration.sum -k regex:hash python scripts/profile_hash.py --once
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    import torch

    import paper_2210_01465_b200 as tk

    radix = [8, 8, 8, 6, 6, 6, 4, 4, 4, 4, 2, 2]
    with tk.Landscape(radix) as src:
        src.generate(0, 0.10, 5)
        fit, ok = src.fitness()
    keys = np.flatnonzero(ok).astype(np.uint64)
    vals = fit[keys]
    rng = np.random.default_rng(0)
    perm = rng.permutation(keys.shape[0])  # cache files list configurations unordered
    keys, vals = keys[perm], vals[perm]
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    dv = torch.from_numpy(vals).cuda()
    land = tk.Landscape(radix)
    L = land.L
    import ctypes as C

    def load():
        st = L.tk_land_load_sparse(land.h, C.c_void_p(dk.data_ptr()), C.c_void_p(dv.data_ptr()),
                                   keys.shape[0], tk._abi.TK_MEM_DEVICE)
        assert st == 0, tk._abi.last_error()

    reps = 1 if "--once" in sys.argv else 5
    load()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        load()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    f2, o2 = land.fitness()
    assert np.array_equal(o2, ok) and np.array_equal(f2.view(np.uint64), fit.view(np.uint64))
    print(json.dumps({"workload": "c5 valid set, unordered keys", "valid_keys": int(keys.shape[0]),
                      "nodes": int(fit.shape[0]), "ms_per_load": round(ms, 3),
                      "keys_per_s": round(keys.shape[0] / (ms / 1e3), 1)}))
    land.close()


if __name__ == "__main__":
    main()
