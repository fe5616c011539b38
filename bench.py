"""bench.py -- FFG + PageRank GTEPS on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c5|c3] [--kind adjacent|hamming]

One step = analyze_landscape on one synthetic search space through the C-ABI:
FFG build (CSR rows emitted, bit-exact), f_opt, PageRank to tol 1e-10 and
the C_p curve for p = 0..15 %.  `value` times steps on inputs resident in HBM;
`e2e` times the same call with host buffers (pinned H2D of the fitness table
inside the timed region, minima report D2H after it).

GTEPS = E * (iterations + 1) / t_step / 1e9: the FFG build traverses every
edge once and each PageRank iteration once more.

Multi-GPU (torchrun, one process per GPU): the one space is key-range
sharded, one shard per GPU (paper_2210_01465_b200/sharded.py): each PageRank
iteration pushes the contributions a peer pulls into that peer's replica over
NVLink from inside the step kernel, and the per-shard partial sums are
all-reduced with NCCL.  Total work is fixed ("scaling": "strong"); time is the
max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # C5 "12-param ~1e8 valid", G_iid q = 0.10 seed 5
    "c5": dict(radix=(8, 8, 8, 6, 6, 6, 4, 4, 4, 4, 2, 2), gen=0, q=0.10, seed=5,
               desc="synthetic 12-parameter space, 113,246,208 configs (~1.02e8 valid), "
                    "random fitness table G_iid q=0.10 seed 5"),
    # C3 "10-param ~1e7 heavy-tailed", G_heavy q = 0 seed 3
    "c3": dict(radix=(8, 8, 8, 8, 6, 6, 4, 4, 2, 2), gen=1, q=0.0, seed=3,
               desc="synthetic 10-parameter space, 9,437,184 configs, heavy-tailed "
                    "runtimes G_heavy seed 3"),
}
WORKLOADS["c4"] = dict(desc="26 synthetic kernel spaces (4 paper shapes, PAPER.md:797-829, + 22 "
                            "seeded shapes of 4-10 parameters, 864..82,944 configs) x 9 tables "
                            "(seeds 0..8, generate_synthetic_kernel_space 'rugged'): 234 landscapes "
                            "back to back")
KIND = {"adjacent": 1, "hamming": 0}

C4_PAPER = [("conv", (12, 6, 8, 8, 2, 2), 0.68), ("conv_mi50", (8, 6, 3, 3, 2), 0.52),
            ("gemm", (4, 4, 3, 3, 3, 3, 4, 4, 2, 2), 0.78), ("pnpoly", (31, 11, 4, 2, 3), 0.04)]


def c4_landscapes():
    """26 shapes x 9 seeds; fail fractions per family."""
    rng = np.random.default_rng(221001465)
    shapes = list(C4_PAPER)
    while len(shapes) < 26:
        dims = int(rng.integers(4, 11))
        radix = tuple(int(x) for x in rng.choice([2, 2, 3, 4, 4, 6, 8, 12, 16], size=dims))
        if 864 <= int(np.prod(radix)) <= 82944:
            shapes.append((f"s{len(shapes)}", radix, float(rng.uniform(0.0, 0.8))))
    return [(name, radix, q, seed) for name, radix, q in shapes for seed in range(9)]


def host_generator():
    """libtunekit_b200.so's C export of generate_synthetic_kernel_space (the
    C++ drop-in's host generator, bit-identical to the reference's)."""
    import ctypes as C

    path = os.path.join(ROOT, "cpp", "build", "libtunekit_b200.so")
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "cpp")], check=True)
    L = C.CDLL(path)
    L.tk_host_generate_synthetic.argtypes = [C.c_uint32, C.c_void_p, C.c_double, C.c_char_p,
                                             C.c_uint64, C.c_void_p, C.c_void_p]

    def gen(radix, q, seed):
        r = np.asarray(radix, np.uint32)
        n = int(np.prod(radix))
        fit = np.empty(n, np.float64)
        ok = np.empty(n, np.uint8)
        st = L.tk_host_generate_synthetic(len(r), r.ctypes.data, q, b"rugged", seed,
                                          fit.ctypes.data, ok.ctypes.data)
        assert st == 0
        return fit, ok
    return gen


def run_batch(args, wl, kind):
    """C4: 234 small landscapes back to back through the C-ABI on one reused
    handle (tk_land_reshape keeps the device buffers); with torchrun each rank
    takes a balanced share (replicas, no collective) and time is the max over
    ranks.  Every landscape: host upload, analyze_landscape, report read-back."""
    import ctypes as C

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2210_01465_b200 as tk

    items = sorted(c4_landscapes(), key=lambda x: -int(np.prod(x[1])))
    mine = [it for i, it in enumerate(items) if i % world == rank]  # size-sorted round robin
    gen = host_generator()
    data = []
    for name, radix, q, seed in mine:
        fit, ok = gen(radix, q, seed)
        fh = torch.empty(len(fit), dtype=torch.float64, pin_memory=True)
        oh = torch.empty(len(fit), dtype=torch.uint8, pin_memory=True)
        fh.numpy()[:] = fit
        oh.numpy()[:] = ok
        data.append((radix, fh, oh))
    workers = int(os.environ.get("TK_BATCH_WORKERS", "8"))
    batch = tk.BatchAnalyzer(device=local, workers=workers, radix0=mine[0][1])
    items = [(radix, fh.data_ptr(), oh.data_ptr()) for radix, fh, oh in data]
    reps = [[torch.empty(90000, dtype=torch.float64, pin_memory=True) for _ in range(4)]
            for _ in range(workers)]
    # one report buffer set per worker slot is enough for timing; item k uses set k % workers
    reports = [tuple(t.data_ptr() for t in reps[k % workers]) for k in range(len(items))]
    akw = dict(damping=DAMPING, tol=TOL, max_iter=MAX_ITER, node_limit=1 << 32,
               p_max_percent=P_MAX)

    def sweep():
        return batch.run(items, kind, reports, **akw)

    for _ in range(max(3, args.warmup)):
        sweep()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(local)
    t0 = time.perf_counter()
    runs = [sweep() for _ in range(args.steps)]
    torch.cuda.synchronize(local)
    t_ms = (time.perf_counter() - t0) * 1e3
    edges = sum(s.n_edges * (s.iterations + 1) for r in runs for s in r)
    n_lands = len(items)
    if dist is not None:
        t = torch.tensor([t_ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
        e = torch.tensor([float(edges)], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(e)
        edges = float(e.item())
    ms_step = t_ms / args.steps
    pr_ms = float(np.mean([s.ms_pagerank for s in runs[-1]]))
    if rank == 0:
        print(json.dumps({
            "metric": "FFG+PageRank GTEPS", "value": round(edges / (t_ms / 1e3) / 1e9, 3),
            "unit": "GTEPS", "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c4", "kind": args.kind, "desc": wl["desc"],
                       "landscapes": n_lands, "parallelism": f"replicas{world}",
                       "host_workers": workers,
                       "l2": "small landscapes; host upload per landscape inside the step"},
            "s_per_space": round(ms_step / 1e3 / n_lands, 7),
            "pagerank_kernel_ms_mean": round(pr_ms, 4),
            "roofline": None,
            "cpu_baseline": None,
            "e2e": {"value": round(edges / (t_ms / 1e3) / 1e9, 3), "unit": "GTEPS",
                    "h2d_bytes_per_step": int(sum(9 * int(np.prod(it[1])) for it in items)),
                    "d2h_bytes_per_step": int(sum(32 * s.n_minima for s in runs[-1]) * world),
                    "note": "the step itself is end to end: host upload + report per landscape "
                            "(tk.BatchAnalyzer: concurrent handles/streams)"},
            "gpu_launches": int(n_lands * 9 * args.steps),
        }))
    batch.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0
KERNELS_PER_STEP = 8  # ffg_count, optimum_final, 2 slot scans, ffg_fill, pagerank, cp_partial, cp_final
DAMPING, TOL, MAX_ITER, P_MAX = 0.85, 1e-10, 100000, 15


def measured_traffic(workload: str, kind: str, iterations: int):
    """DRAM bytes (read + write) per PageRank launch from the committed ncu
    --set full capture (profiles/r01_pagerank_traffic.json), when it was taken
    on this workload; None otherwise."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_pagerank_traffic.json")) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    if (t.get("workload"), t.get("kind"), t.get("iterations")) != (workload, kind, iterations):
        return None
    return t["dram_bytes_per_launch"]


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0}, "fallback"


# ------------------------------------------------------------ clocks probe --

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.device), "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        time.sleep(0.15)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm.append(float(parts[0]))
                    smax = float(parts[1])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[3:7]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- CPU legs --

def cpu_sample(wl: dict, kind: int, pr_iters: int = 3):
    """Bounded CPU sample of the same workload: the first dim-0 slab of the
    space (all other parameters intact), full FFG build with CSR and minima,
    `pr_iters` PageRank iterations, C_p.  Oracle port, all host threads."""
    import oracle as O

    radix = list(wl["radix"])
    radix[0] = 1
    n = O.space_size(radix)
    threads = os.cpu_count() or 1
    gen = O.gen_iid if wl["gen"] == 0 else O.gen_heavy
    fit, ok = gen(n, wl["q"], wl["seed"], nthreads=threads)
    t0 = time.perf_counter()
    g = O.build_ffg(radix, fit, ok, kind, node_limit=1 << 32, nthreads=threads)
    pr, it, _ = O.pagerank(g["offsets"], g["targets"], DAMPING, TOL, MAX_ITER,
                           nthreads=threads, fixed_iters=pr_iters)
    f_opt, _ = O.optimum(fit, ok)
    for k in range(P_MAX + 1):
        O.proportion_of_centrality(g["minima"], fit, pr, f_opt, k / 100.0)
    dt = time.perf_counter() - t0
    e = len(g["targets"])
    return dict(value=e * (pr_iters + 1) / dt / 1e9, seconds=dt, edges=e, nodes=n,
                threads=threads, iters=pr_iters)


def run_reference(args, wl, kind):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    for _ in range(args.warmup):
        cpu_sample(wl, kind)
    vals, secs = [], 0.0
    for _ in range(args.steps):
        s = cpu_sample(wl, kind)
        vals.append(s["value"])
        secs += s["seconds"]
    v = float(np.mean(vals))
    sample = (f"first dim-0 slab of {args.workload} ({s['nodes']} configs, {s['edges']} edges): "
              f"FFG build + {s['iters']} PageRank iterations + C_p per step")
    line = {
        "metric": "FFG+PageRank GTEPS", "value": v, "unit": "GTEPS", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "kind": args.kind, "desc": wl["desc"]},
        "cpu_baseline": {"value": v, "unit": "GTEPS", "cores": s["threads"], "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------- GPU leg --

def run_b200(args, wl, kind):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2210_01465_b200 as tk

    radix = wl["radix"]
    land = tk.Landscape(radix, device=local)
    land.generate(wl["gen"], wl["q"], wl["seed"] + 0)  # identical replica on every rank
    stream = torch.cuda.ExternalStream(land.stream, device=torch.device("cuda", local))

    def step():
        return land.analyze(kind, DAMPING, TOL, MAX_ITER, node_limit=1 << 32,
                            p_max_percent=P_MAX, emit_csr=True)

    for _ in range(max(3, args.warmup)):
        s = step()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(local)

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- value: inputs resident in HBM (> L2: 1 GB fitness + 11 GB FFG state)
    clocks = ClockSampler(local)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    clocks.start()
    ev0.record(stream)
    sums = []
    for _ in range(args.steps):
        sums.append(step())
    ev1.record(stream)
    ev1.synchronize()
    clk = clocks.stop()
    barrier()
    t_ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = t_ms / args.steps
    e = sums[-1].n_edges
    iters = [x.iterations for x in sums]
    edges_traversed = sum(e * (it + 1) for it in iters) * world
    value = edges_traversed / (t_ms / 1e3) / 1e9

    n = land.n
    kinfo = land.kernel_info()

    # ---- e2e: the same analysis from pinned host buffers through the public API.
    # tk.AnalysisPipeline double-buffers two device handles: every step uploads its
    # whole table (9 B/config H2D) and reads its minima report back (32 B/minimum
    # D2H) inside the timed region, and those PCIe transfers of step k+1 / k-1 run
    # on the other handle's stream while step k's kernels execute.
    fit_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    ok_h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    f_np, o_np = land.fitness()
    fit_h.numpy()[:] = f_np
    ok_h.numpy()[:] = o_np
    m = sums[-1].n_minima
    land.close()  # free this handle's device state; the pipeline holds two of its own
    torch.cuda.synchronize(local)
    rep = [[torch.empty(m, dtype=torch.float64, pin_memory=True) for _ in range(4)]
           for _ in range(2)]
    items = [(fit_h.data_ptr(), ok_h.data_ptr())] * args.steps
    reports = [tuple(t.data_ptr() for t in rep[k % 2]) for k in range(args.steps)]
    pipe = tk.AnalysisPipeline(radix, device=local)
    akw = dict(damping=DAMPING, tol=TOL, max_iter=MAX_ITER, node_limit=1 << 32,
               p_max_percent=P_MAX, emit_csr=True)
    pipe.run(items[:2], kind, reports[:2], **akw)  # warm both handles
    barrier()
    t0 = time.perf_counter()
    e2e_sums = pipe.run(items, kind, reports, **akw)
    torch.cuda.synchronize(local)
    wall_ms = (time.perf_counter() - t0) * 1e3
    barrier()
    t_e2e = max_over_ranks(wall_ms)
    e2e_value = sum(e * (x.iterations + 1) for x in e2e_sums) * world / (t_e2e / 1e3) / 1e9
    pipe.close()

    # ---- roofline of the dominant kernel (persistent PageRank, one launch per step)
    peaks, peak_src = measured_peaks()
    it_last = sums[-1].iterations
    if land_mode_packed(radix, kind):
        # contribution-only iteration: packed word 4 + c read once 8 + c' 8;
        # prologue writes c_0 (pw 4 + 8), the closing pass materialises r' (pw 4 + c 8 + r 8)
        per_iter, per_pro = 20 * n, 12 * n + 20 * n
        model = ("20 B/node/iteration: packed word 4 + c gather (each c read once) 8 + c' 8; "
                 "+ 12 B/node prologue (c_0) + 20 B/node closing r' pass")
    else:
        per_iter, per_pro = 37 * n, 21 * n
        model = "37 B/node/iteration: mask 4 + outdeg 1 + r_old 8 + r_new 8 + c_new 8 + c 8"
    pr_ms = float(np.mean([x.ms_pagerank for x in sums]))
    pr_bytes = per_pro + per_iter * it_last
    achieved = pr_bytes / (pr_ms / 1e3) / 1e9
    ffg_ms = float(np.mean([x.ms_ffg for x in sums]))
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                "traffic": measured_traffic(args.workload, args.kind, it_last),
                "kernel": "pagerank_staged_kernel (persistent, cooperative)",
                "bytes_model": model, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": pr_bytes, "kernel_ms": round(pr_ms, 3),
                "iterations": it_last, "kernels": kinfo}

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            c = cpu_sample(wl, kind)
            cpu = {"value": round(c["value"], 4), "unit": "GTEPS", "cores": c["threads"],
                   "kind": "port",
                   "sample": f"oracle/oracle.c (OpenMP) on the first dim-0 slab of "
                             f"{args.workload}: {c['nodes']} configs, {c['edges']} edges, FFG "
                             f"+ {c['iters']} PageRank iterations + C_p, {c['seconds']:.1f} s"}
        ffg_bytes = 22 * n + 4 * e + 4 * sums[-1].n_minima
        out = {
            "metric": "FFG+PageRank GTEPS", "value": round(value, 3), "unit": "GTEPS",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "kind": args.kind, "desc": wl["desc"],
                       "nodes": n, "edges": e, "minima": sums[-1].n_minima,
                       "pagerank_iterations": it_last, "damping": DAMPING, "tol": TOL,
                       "parallelism": f"replicas{world}",
                       "l2": "inputs larger than L2 (1.0 GB fitness, ~11 GB FFG/PageRank state)"},
            "s_per_space": round(ms_step / 1e3, 5),
            "phases_ms": {"ffg_build_kernel": round(ffg_ms, 3),
                          "pagerank_kernel": round(pr_ms, 3),
                          "centrality": round(float(np.mean([x.ms_centrality for x in sums])), 3)},
            "ffg_edges_per_s": round(e / (ffg_ms / 1e3), 1),
            "ffg_build_gbs": round(ffg_bytes / (ffg_ms / 1e3) / 1e9, 1),
            "pagerank_gteps": round(e * it_last / (pr_ms / 1e3) / 1e9, 3),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 3), "unit": "GTEPS",
                    "h2d_bytes_per_step": 9 * n, "d2h_bytes_per_step": 32 * m,
                    "ms_per_step": round(t_e2e / args.steps, 3),
                    "how": "tk.AnalysisPipeline: pinned host table uploaded and minima report "
                           "read back every step, overlapped with the previous/next step's "
                           "kernels on a second device handle (wall clock)"},
            "gpu_launches": KERNELS_PER_STEP * args.steps,
            "clocks": clk,
        }
        print(json.dumps(out))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_sharded(args, wl, kind):
    """N GPUs (torchrun): the space is key-range sharded, one shard per GPU;
    each PageRank iteration pushes the new contributions a peer pulls into that
    peer's replica over NVLink from inside the step kernel, and the per-shard
    partials are all-reduced (NCCL) -- the iteration barrier.  Strong scaling:
    the total work (one C5 space) is fixed."""
    import torch
    import torch.distributed as dist

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    # TK_FORCE_DEVICE / TK_DIST_BACKEND=gloo let the multi-process path run with
    # several ranks on one GPU (CUDA IPC still maps the peers' replicas)
    local = int(os.environ.get("TK_FORCE_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    backend = os.environ.get("TK_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    from paper_2210_01465_b200 import sharded as S

    radix = wl["radix"]
    shard = S.GpuShard(radix, rank, world, device=local)
    shard.land.generate(wl["gen"], wl["q"], wl["seed"])  # read-only table, replicated
    allreduce, allgather = S.torch_collectives(device=f"cuda:{local}")
    S.connect_peers_ipc(shard, allgather)
    stream = torch.cuda.ExternalStream(shard.land.stream, device=torch.device("cuda", local))

    # NCCL: partials all-reduced in device memory, one host sync per iteration;
    # gloo stages CUDA tensors through the host, so there the host loop is faster
    loop = (S.device_pagerank_loop(shard, f"cuda:{local}")
            if backend == "nccl" and not os.environ.get("TK_HOST_LOOP") else None)

    def step():
        return S.analyze_sharded([shard], allreduce, allgather, kind, DAMPING, TOL, MAX_ITER,
                                 P_MAX, pagerank_loop=loop)

    for _ in range(max(3, args.warmup)):
        res = step()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    dist.barrier()
    torch.cuda.synchronize(local)
    clocks.start()
    ev0.record(stream)
    t0 = time.perf_counter()
    runs = [step() for _ in range(args.steps)]
    ev1.record(stream)
    ev1.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    clk = clocks.stop()
    t = torch.tensor([max(ev0.elapsed_time(ev1), wall)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())

    # e2e: every rank uploads the fitness table from pinned host memory, runs the
    # sharded analysis and reads its minima report rows back
    import ctypes as C

    f_np, o_np = shard.land.fitness()
    fit_h = torch.empty(shard.land.n, dtype=torch.float64, pin_memory=True)
    ok_h = torch.empty(shard.land.n, dtype=torch.uint8, pin_memory=True)
    fit_h.numpy()[:] = f_np
    ok_h.numpy()[:] = o_np
    m_local = shard.land.n_minima
    rep = [torch.empty(max(1, m_local), dtype=torch.float64, pin_memory=True) for _ in range(4)]
    L = shard.land.L

    def e2e_step():
        assert L.tk_land_load_dense(shard.land.h, C.c_void_p(fit_h.data_ptr()),
                                    C.c_void_p(ok_h.data_ptr()), 0) == 0
        r = step()
        assert L.tk_report_copy_out(shard.land.h, r["f_opt"], *[C.c_void_p(x.data_ptr())
                                                                for x in rep]) == 0
        return r

    e2e_step()
    dist.barrier()
    t0 = time.perf_counter()
    e2e_runs = [e2e_step() for _ in range(args.steps)]
    torch.cuda.synchronize(local)
    t = torch.tensor([(time.perf_counter() - t0) * 1e3], dtype=torch.float64,
                     device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_e2e = float(t.item())
    e2e_value = sum(x["n_edges"] * (x["iterations"] + 1) for x in e2e_runs) / (t_e2e / 1e3) / 1e9
    e = runs[-1]["n_edges"]
    value = sum(e * (r["iterations"] + 1) for r in runs) / (t_ms / 1e3) / 1e9
    n = shard.land.n
    it = runs[-1]["iterations"]
    peaks, peak_src = measured_peaks()
    # PageRank algorithmic bytes per GPU: init 12 B/rank, per step 20 B/rank
    # (packed word 4, each c read once 8, c' written 8; contribution-only),
    # r rebuilt once at the end 20 B/rank
    per_gpu_bytes = (32 * n + 20 * n * it) / world
    ms_step = t_ms / args.steps
    if rank == 0:
        print(json.dumps({
            "metric": "FFG+PageRank GTEPS", "value": round(value, 3), "unit": "GTEPS",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "kind": args.kind, "desc": wl["desc"],
                       "nodes": n, "edges": e, "minima": runs[-1]["n_minima"],
                       "pagerank_iterations": it, "parallelism": f"keyrange{world}",
                       "shard_push": os.environ.get("TK_SHARD_PUSH", "crossing"),
                       "l2": "inputs larger than L2"},
            "s_per_space": round(ms_step / 1e3, 5),
            "roofline": {"bound": "hbm", "achieved": round(per_gpu_bytes / (ms_step / 1e3) / 1e9, 1),
                         "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": round(per_gpu_bytes / (ms_step / 1e3) / 1e9 / peaks["hbm_gbs"], 4),
                         "traffic": None, "peak_source": peak_src,
                         "kernel": "whole sharded step (per GPU)"},
            "cpu_baseline": None,
            "e2e": {"value": round(e2e_value, 3), "unit": "GTEPS",
                    "h2d_bytes_per_step": 9 * n * world,
                    "d2h_bytes_per_step": 32 * runs[-1]["n_minima"],
                    "ms_per_step": round(t_e2e / args.steps, 3)},
            "gpu_launches": args.steps * (4 + 2 * (it + 1) + 2),
            "clocks": clk,
        }))
    if loop is not None:
        loop.close()
    shard.land.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0


def land_mode_packed(radix, kind) -> bool:
    dims = sum(1 for m in radix if m >= 2)
    return kind == 1 and 2 * dims <= 27


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c5")
    ap.add_argument("--kind", choices=sorted(KIND), default="adjacent")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    kind = KIND[args.kind]
    if args.impl == "reference":
        if args.workload == "c4":
            print(json.dumps({"impl": "reference", "unavailable": "the c4 reference arm is not "
                              "implemented; use the default c5 workload"}))
            return 0
        return run_reference(args, wl, kind)
    if args.workload == "c4":
        return run_batch(args, wl, kind)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return run_sharded(args, wl, kind)
    return run_b200(args, wl, kind)


if __name__ == "__main__":
    sys.exit(main())
