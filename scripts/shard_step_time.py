"""Per-shard PageRank step time on one GPU (virtual shards, one process).

    python scripts/shard_step_time.py [--shards 1 2 8] [--steps 29]

Every shard of a G-way key-range split of the C5 space is built on device 0
and its step kernel (tk_shard_pagerank_step: staged pull over the shard's
tiles, c' stored locally and pushed into the peers' replicas, partial
reduction) is timed with CUDA events on the library stream.  The numbers are
the kernel time one GPU of a G-GPU box would spend per iteration, without the
NVLink latency of the remote stores (the peers are on the same device here)
and without the all-reduce.  TK_LIB=<path> selects a library build, so two
formulations can be compared on the same box.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

C5 = (8, 8, 8, 6, 6, 6, 4, 4, 4, 4, 2, 2)


def main() -> int:
    import torch

    from paper_2210_01465_b200 import sharded as S

    ap = argparse.ArgumentParser()
    ap.add_argument("--shards", type=int, nargs="+", default=[1, 2, 8])
    ap.add_argument("--steps", type=int, default=29)
    args = ap.parse_args()
    out = {"lib": os.environ.get("TK_LIB", "product"), "workload": "c5", "per_shard_step_ms": {}}
    for g in args.shards:
        shards = [S.GpuShard(C5, r, g, device=0) for r in range(g)]
        for s in shards:
            s.land.generate(0, 0.10, 5)
        S.connect_peers_local(shards)
        for s in shards:
            s.build(1)
        ms = []
        for s in shards:
            stream = torch.cuda.ExternalStream(s.land.stream, device=torch.device("cuda", 0))
            dang = s.pagerank_init(0.85)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            times = []
            for _ in range(args.steps):
                e0.record(stream)
                res = s.pagerank_step(dang, 0.85)  # synchronises the stream
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
                dang = res[1] if isinstance(res, (tuple, list)) else dang
            ms.append(float(np.median(times[2:])))
        # the same steps enqueued back to back (tk_shard_pagerank_step_dev, no
        # host synchronisation between them): GPU time per step without the
        # host round trip of the synchronous call above
        ms_dev = []
        for s in shards:
            stream = torch.cuda.ExternalStream(s.land.stream, device=torch.device("cuda", 0))
            tot = torch.zeros(3, dtype=torch.float64, device="cuda:0")
            part = torch.zeros(3, dtype=torch.float64, device="cuda:0")
            s.land.shard_pagerank_init_dev(0.85, tot.data_ptr())
            for _ in range(3):
                s.land.shard_pagerank_step_dev(tot.data_ptr(), 0.85, part.data_ptr())
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                s.land.shard_pagerank_step_dev(tot.data_ptr(), 0.85, part.data_ptr())
            e1.record(stream)
            e1.synchronize()
            ms_dev.append(e0.elapsed_time(e1) / args.steps)
        n = shards[0].land.n
        out.setdefault("per_shard_step_ms_async", {})[g] = round(max(ms_dev), 4)
        out["per_shard_step_ms"][g] = {
            "max_over_shards": round(max(ms), 4), "mean": round(float(np.mean(ms)), 4),
            "ranks_per_shard": int(-(-n // g)),
            "gb_s_at_20B": round(20 * n / g / (max(ms) / 1e3) / 1e9, 1),
            "gb_s_at_36B": round(36 * n / g / (max(ms) / 1e3) / 1e9, 1)}
        for s in shards:
            s.land.close()
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    sys.exit(main())
