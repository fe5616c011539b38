"""bench.py -- FFG + PageRank GTEPS on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c5|c3|c4] [--kind adjacent|hamming]

One step = analyze_landscape on one synthetic search space through the C-ABI:
FFG build (CSR rows emitted, bit-exact), f_opt, PageRank to tol 1e-10 and
the C_p curve for p = 0..15 %.  `value` times steps on inputs resident in HBM;
`e2e` times the same call with host buffers (pinned H2D of the fitness table
inside the timed region, minima report D2H after it).

GTEPS = E * (iterations + 1) / t_step / 1e9: the FFG build traverses every
edge once and each PageRank iteration once more.

Multi-GPU: `--gpus N` (N > 1) relaunches itself under torch.distributed.run
(one process per GPU) unless it already runs under it.  The one space is
key-range sharded, one shard per GPU (paper_2210_01465_b200/sharded.py): each
PageRank iteration pushes the contributions a peer pulls into that peer's
replica over NVLink from inside the step kernel, and the per-shard partial
sums are all-reduced with NCCL.  Total work is one fixed space at every N
("scaling": "strong"); time is the max over ranks.

--impl reference: the CPU path (oracle/oracle.c, the C restatement of the
reference's FFG / PageRank / C_p contract -- the reference declares the path
but has no implementation) on the SAME workload: full space,
PageRank to convergence, all host threads; plus a 1-thread column.
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
    # BASELINE.json configs[0]: 4-parameter GEMM-like, random table
    "c1": dict(radix=(12, 12, 12, 12), gen=0, q=0.0, seed=1,
               desc="synthetic 4-parameter GEMM-like space, 20,736 configs, random fitness "
                    "table G_iid seed 1"),
    # configs[1] (C2): 8-parameter conv-like, ~30 % invalid, the reference's own
    # generate_synthetic_kernel_space "rugged" (host-generated: it uses libm sin)
    "c2": dict(radix=(16, 12, 8, 8, 8, 4, 2, 2), gen=2, q=0.30, seed=2,
               desc="synthetic 8-parameter convolution-like space, 1,572,864 configs (~1.1e6 "
                    "valid, ~30 % failed), generate_synthetic_kernel_space 'rugged' seed 2"),
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
    threaded = bool(os.environ.get("TK_BATCH_THREADS"))
    if rank == 0:
        print(json.dumps({
            "metric": "FFG+PageRank GTEPS", "value": round(edges / (t_ms / 1e3) / 1e9, 3),
            "unit": "GTEPS", "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "parallelism": f"replicas{world}",
            "config": {"workload": "c4", "kind": args.kind, "desc": wl["desc"],
                       "landscapes": n_lands,
                       "host_workers": workers,
                       "l2": "small landscapes; host upload per landscape inside the step"},
            "s_per_space": round(ms_step / 1e3 / n_lands, 7),
            "pagerank_kernel_ms_mean": round(pr_ms, 4) if threaded else None,
            "roofline": None,
            "cpu_baseline": None,
            "e2e": {"value": round(edges / (t_ms / 1e3) / 1e9, 3), "unit": "GTEPS",
                    "h2d_bytes_per_step": int(sum(9 * int(np.prod(it[0])) for it in items)),
                    "d2h_bytes_per_step": int(sum(32 * s.n_minima for s in runs[-1]) * world),
                    "note": "the step itself is end to end: host upload + report per landscape "
                            + ("(tk.BatchAnalyzer: concurrent handles/streams)" if threaded else
                               "(tk.BatchAnalyzer -> tk_batch_analyze: one upload, one launch "
                               "with one CTA per landscape, one read-back)")},
            "batch_path": "threads" if threaded else "batched",
            # threads: ~9 kernels per landscape; batched: one batch_analyze_kernel per step
            "gpu_launches": int(n_lands * 9 * args.steps) if threaded else int(args.steps),
        }))
    batch.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0
FFG_BYTES_PER_NODE = 22
FFG_BYTES_MODEL = ("22 B/node + 4 B/edge + 4 B/minimum: fitness 8 + ok 1 + packed word 4 + flags 1 "
                   "+ CSR offset 8, targets, minima")
KERNELS_PER_STEP = 8  # ffg_count, optimum_final, 2 slot scans, ffg_fill, pagerank, cp_partial, cp_final
DAMPING, TOL, MAX_ITER, P_MAX = 0.85, 1e-10, 100000, 15


def kernel_source_sha() -> str:
    import hashlib

    h = hashlib.sha256()
    for f in ("tk_staged.cu", "tk_internal.cuh"):
        with open(os.path.join(ROOT, "paper_2210_01465_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def hamming_traffic(workload: str, iterations: int, kernel: str):
    """DRAM bytes (read + write) of one Hamming PageRank (all dimension-group
    passes) from the committed ncu launch list (profiles/hamming_traffic.json),
    used only for the same workload, iteration count and tk_hamsplit.cu source;
    (None, why) otherwise."""
    import hashlib

    if kernel != "ham_split":
        return None, f"capture taken on the ham_split kernel, not {kernel}"
    try:
        with open(os.path.join(ROOT, "profiles", "hamming_traffic.json")) as f:
            t = json.load(f)
        with open(os.path.join(ROOT, "paper_2210_01465_b200", "csrc", "tk_hamsplit.cu"), "rb") as f:
            sha = hashlib.sha256(f.read()).hexdigest()[:16]
    except (OSError, ValueError):
        return None, "no committed capture"
    if (t.get("workload"), t.get("iterations")) != (workload, iterations):
        return None, "capture taken on another workload"
    if t.get("kernel_source_sha") != sha:
        return None, f"capture taken on kernel source {t.get('kernel_source_sha')}, not this one"
    return t["dram_bytes_per_pagerank"], t.get("source", "")


def measured_traffic(workload: str, kind: str, iterations: int):
    """DRAM bytes (read + write) per PageRank launch from the committed ncu
    --set full capture (profiles/pagerank_traffic.json, scripts/
    capture_traffic.sh), used only when it was taken on this workload AND on
    this kernel source (sha of csrc/tk_staged.cu + tk_internal.cuh);
    (None, why) otherwise."""
    try:
        with open(os.path.join(ROOT, "profiles", "pagerank_traffic.json")) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None, "no committed capture"
    if (t.get("workload"), t.get("kind"), t.get("iterations")) != (workload, kind, iterations):
        return None, "capture taken on another workload"
    if t.get("kernel_source_sha") != kernel_source_sha():
        return None, f"capture taken on kernel source {t.get('kernel_source_sha')}, not this one"
    return t["dram_bytes_per_launch"], t.get("source", "")


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

def host_cpu():
    """nproc and the lscpu model name of this host."""
    model = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.SubprocessError):
        pass
    return {"nproc": os.cpu_count() or 1, "model": model}


def cpu_inputs(wl, radix=None, threads=None):
    import oracle as O

    radix = list(radix or wl["radix"])
    nt = threads or os.cpu_count() or 1
    if wl["gen"] == 2:
        return radix, *O.gen_synthetic(radix, wl["q"], "rugged", wl["seed"], nthreads=nt)
    gen = O.gen_iid if wl["gen"] == 0 else O.gen_heavy
    return radix, *gen(O.space_size(radix), wl["q"], wl["seed"], nthreads=nt)


def cpu_analyze(radix, fit, ok, kind, threads):
    """One analyze_landscape on the CPU path (oracle/oracle.c): FFG build with
    CSR and minima, f_opt, PageRank to convergence (tol 1e-10; the out-CSR is
    transposed inside, as pagerank(const FitnessFlowGraph&) must), C_p for
    p = 0..15 %.  Per-phase wall times."""
    import oracle as O

    t0 = time.perf_counter()
    g = O.build_ffg(radix, fit, ok, kind, node_limit=1 << 32, nthreads=threads)
    t1 = time.perf_counter()
    f_opt, _ = O.optimum(fit, ok)
    pr, it, _ = O.pagerank(g["offsets"], g["targets"], DAMPING, TOL, MAX_ITER, nthreads=threads)
    t2 = time.perf_counter()
    curve = [O.proportion_of_centrality(g["minima"], fit, pr, f_opt, k / 100.0)
             for k in range(P_MAX + 1)]
    t3 = time.perf_counter()
    e = len(g["targets"])
    return dict(value=e * (it + 1) / (t3 - t0) / 1e9, seconds=t3 - t0, edges=e,
                nodes=len(fit), minima=g["minima"], iterations=it, pagerank=pr, c_p=curve,
                threads=threads,
                phases_s={"ffg": round(t1 - t0, 3), "pagerank": round(t2 - t1, 3),
                          "centrality": round(t3 - t2, 3)})


def cpu_one_thread(wl, kind):
    """The 1-thread column (the reference code has no threads) on
    a bounded sample: the first dim-0 slab of the workload (every other
    parameter intact), full analysis to convergence."""
    radix = list(wl["radix"])
    radix[0] = 1
    radix, fit, ok = cpu_inputs(wl, radix)
    c = cpu_analyze(radix, fit, ok, kind, 1)
    return {"value": round(c["value"], 5), "unit": "GTEPS", "cores": 1,
            "sample": f"first dim-0 slab ({c['nodes']} configs, {c['edges']} edges, "
                      f"{c['iterations']} PageRank iterations to convergence), {c['seconds']:.1f} s",
            "phases_s": c["phases_s"]}


def config_block(args, wl, n, e, m, iters):
    """The `config` object, identical in both arms for one workload."""
    return {"workload": args.workload, "kind": args.kind, "desc": wl["desc"], "nodes": n,
            "edges": e, "minima": m, "pagerank_iterations": iters, "damping": DAMPING,
            "tol": TOL, "l2": l2_note(n, e)}


def l2_note(n, e):
    state = 9 * n + 4 * e + 8 * n + 32 * n  # table, CSR targets + offsets, PageRank vectors
    if state > 126e6:
        return (f"inputs larger than L2 ({9 * n / 1e9:.2f} GB fitness table, "
                f"~{state / 1e9:.1f} GB FFG/PageRank state vs 126 MB L2)")
    return (f"inputs smaller than L2 (~{state / 1e6:.1f} MB state): steps run back to back "
            "without an L2 flush (a parity/latency workload, not the headline line)")


def run_reference(args, wl, kind):
    """The reference arm: the CPU path on the same workload as the GPU arm
    (whole space, PageRank to convergence, C_p curve), all host threads.  The
    input table is generated once, outside the timed steps (as the GPU arm's
    `value` has it resident)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    radix, fit, ok = cpu_inputs(wl)
    for _ in range(args.warmup):
        cpu_analyze(radix, fit, ok, kind, threads)
    runs = [cpu_analyze(radix, fit, ok, kind, threads) for _ in range(args.steps)]
    secs = sum(r["seconds"] for r in runs)
    last = runs[-1]
    edges = sum(r["edges"] * (r["iterations"] + 1) for r in runs)
    v = edges / secs / 1e9
    one = cpu_one_thread(wl, kind)
    host = host_cpu()
    line = {
        "metric": "FFG+PageRank GTEPS", "value": round(v, 5), "unit": "GTEPS",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(args, wl, last["nodes"], last["edges"], len(last["minima"]),
                               last["iterations"]),
        "phases_s": last["phases_s"],
        "cpu_baseline": {"value": round(v, 5), "unit": "GTEPS", "cores": threads,
                         "kind": "port", "host": host, "same_config": True,
                         "sample": f"the whole {args.workload} workload per step ({last['nodes']} "
                                   f"configs, {last['edges']} edges, {last['iterations']} "
                                   f"PageRank iterations): oracle/oracle.c, OpenMP, {threads} "
                                   "threads",
                         "one_thread": one},
        "e2e": {"value": round(v, 5), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reproduce": f"python bench.py --impl reference --workload {args.workload} "
                     f"--kind {args.kind} --steps {args.steps} --warmup {args.warmup}",
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
    if wl["gen"] == 2:  # the reference's generator, host-side (libm sin), then uploaded
        hfit, hok = host_generator()(radix, wl["q"], wl["seed"])
        land.load_dense(hfit, hok)
        del hfit, hok
    else:
        land.generate(wl["gen"], wl["q"], wl["seed"])  # device generator, bit-identical
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
    e_last, m_last, it_last = sums[-1].n_edges, sums[-1].n_minima, sums[-1].iterations

    # ---- the GPU results of this workload, kept for the parity check below
    gpu_minima = gpu_pr = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gpu_minima = land.minima().astype(np.int64)
        gpu_pr = land.pagerank_vector()
    gpu_curve = list(sums[-1].c_p[: sums[-1].n_cp])

    # ---- second column: the same space under the Hamming neighbourhood
    ham = None
    if args.kind == "adjacent" and not args.no_hamming:
        hs = [land.analyze(0, DAMPING, TOL, MAX_ITER, node_limit=1 << 32,
                           p_max_percent=P_MAX, emit_csr=True)]  # warm
        h0 = torch.cuda.Event(enable_timing=True)
        h1 = torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        hs = [land.analyze(0, DAMPING, TOL, MAX_ITER, node_limit=1 << 32, p_max_percent=P_MAX,
                           emit_csr=True) for _ in range(3)]
        h1.record(stream)
        h1.synchronize()
        h_ms = h0.elapsed_time(h1) / 3
        he, hit = hs[-1].n_edges, hs[-1].iterations
        hpr = float(np.mean([x.ms_pagerank for x in hs]))
        hkern = {"ham_split": "ham_split_kernel (one pass per dimension group and iteration)",
                 "ham_tiled": "pagerank_ham_tiled_kernel"}.get(
                     land.kernel_info()["pagerank_kernel"], land.kernel_info()["pagerank_kernel"])
        # contribution-only Hamming iteration: u64 in-mask 8 + outdeg 1 + c read once 8 + c' 8
        hbytes = 25 * n * hit + 33 * n
        peaks, _ = measured_peaks()
        ham = {"value": round(he * (hit + 1) * 3 / (h_ms * 3 / 1e3) / 1e9, 3), "unit": "GTEPS",
               "ms_per_step": round(h_ms, 3), "edges": he, "pagerank_iterations": hit,
               "phases_ms": {"ffg_build_kernel": round(float(np.mean([x.ms_ffg for x in hs])), 3),
                             "pagerank_kernel": round(hpr, 3)},
               "roofline": {"bound": "hbm", "kernel": hkern,
                            "achieved": round(hbytes / (hpr / 1e3) / 1e9, 1),
                            "peak": peaks["hbm_gbs"], "unit": "GB/s",
                            "frac": round(hbytes / (hpr / 1e3) / 1e9 / peaks["hbm_gbs"], 4),
                            "bytes_model": "25 B/node/iteration: u64 in-mask 8 + outdeg 1 + c "
                                           "read once 8 + c' 8; + 33 B/node prologue and "
                                           "closing pass",
                            "algorithmic_bytes_per_launch": hbytes,
                            "traffic": None}}
        ht, hsrc = hamming_traffic(args.workload, hit, land.kernel_info()["pagerank_kernel"])
        ham["roofline"]["traffic"] = ht
        ham["roofline"]["traffic_source"] = hsrc

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
    m = m_last
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
    traffic, traffic_src = measured_traffic(args.workload, args.kind, it_last)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                "traffic": traffic, "traffic_source": traffic_src,
                "kernel": "pagerank_staged_kernel (persistent, cooperative)",
                "bytes_model": model, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": pr_bytes, "kernel_ms": round(pr_ms, 3),
                "iterations": it_last, "kernels": kinfo}
    ffg_bytes = FFG_BYTES_PER_NODE * n + 4 * e_last + 4 * m_last
    roofline_ffg = {"bound": "hbm", "kernel": "ffg_count_staged_kernel + ffg_fill_kernel",
                    "achieved": round(ffg_bytes / (ffg_ms / 1e3) / 1e9, 1),
                    "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": round(ffg_bytes / (ffg_ms / 1e3) / 1e9 / peaks["hbm_gbs"], 4),
                    "bytes_model": FFG_BYTES_MODEL, "algorithmic_bytes_per_build": ffg_bytes,
                    "phase_ms": round(ffg_ms, 3)}

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            threads = os.cpu_count() or 1
            _, cfit, cok = cpu_inputs(wl)
            c = cpu_analyze(list(radix), cfit, cok, kind, threads)
            # parity of this very run: the GPU results above against the CPU path
            parity = {
                "edges_equal": c["edges"] == e_last,
                "minima_equal": bool(np.array_equal(c["minima"].astype(np.int64), gpu_minima)),
                "iterations_equal": c["iterations"] == it_last,
                "pagerank_rel_l1": float(np.abs(gpu_pr - c["pagerank"]).sum()
                                         / np.abs(c["pagerank"]).sum()),
                "c_p_max_abs_diff": float(max(abs(a - b) for a, b in zip(gpu_curve, c["c_p"]))),
            }
            parity["ok"] = bool(parity["edges_equal"] and parity["minima_equal"]
                                and parity["iterations_equal"]
                                and parity["pagerank_rel_l1"] <= 1e-12
                                and parity["c_p_max_abs_diff"] <= 1e-9)
            cpu = {"value": round(c["value"], 5), "unit": "GTEPS", "cores": threads,
                   "kind": "port", "host": host_cpu(), "same_config": True,
                   "sample": f"the whole {args.workload} workload once ({c['nodes']} configs, "
                             f"{c['edges']} edges, {c['iterations']} PageRank iterations): "
                             f"oracle/oracle.c, OpenMP, {threads} threads, {c['seconds']:.1f} s",
                   "phases_s": c["phases_s"],
                   "one_thread": cpu_one_thread(wl, kind),
                   "parity_vs_gpu": parity}
            del c
        out = {
            "metric": "FFG+PageRank GTEPS", "value": round(value, 3), "unit": "GTEPS",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": round(ms_step, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "parallelism": f"replicas{world}",
            "config": config_block(args, wl, n, e_last, m_last, it_last),
            "s_per_space": round(ms_step / 1e3, 5),
            "phases_ms": {"ffg_build_kernel": round(ffg_ms, 3),
                          "pagerank_kernel": round(pr_ms, 3),
                          "centrality": round(float(np.mean([x.ms_centrality for x in sums])), 3)},
            "ffg_edges_per_s": round(e_last / (ffg_ms / 1e3), 1),
            "pagerank_gteps": round(e_last * it_last / (pr_ms / 1e3) / 1e9, 3),
            "roofline": roofline,
            "roofline_ffg": roofline_ffg,
            "hamming": ham,
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
    if wl["gen"] == 2:
        hfit, hok = host_generator()(radix, wl["q"], wl["seed"])
        shard.land.load_dense(hfit, hok)
        del hfit, hok
    else:
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
            "parallelism": f"keyrange{world}", "dist_backend": backend,
            "shard_push": os.environ.get("TK_SHARD_PUSH", "crossing"),
            "nvlink_bytes_per_gpu_per_iteration": nvlink_push_bytes(radix, world),
            "config": config_block(args, wl, n, e, runs[-1]["n_minima"], it),
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


def nvlink_push_bytes(radix, world: int) -> int:
    """Expected NVLink bytes one GPU stores into its peers per PageRank
    iteration under TK_SHARD_PUSH=crossing: c'[v] (8 B) along
    every direction (dim i, +/-) whose neighbour exists and lies in another
    shard, counted over the largest shard."""
    from paper_2210_01465_b200.sharded import shard_range

    radix = [m for m in radix if m >= 2]
    n = int(np.prod(radix))
    strides = [int(np.prod(radix[i + 1:])) for i in range(len(radix))]
    worst = 0
    for g in range(world):
        lo, hi = shard_range(n, g, world)
        tot = 0
        for s_i, m_i in zip(strides, radix):
            # + direction: v in [max(lo, hi - s_i), hi) with digit_i(v) < m_i - 1
            v = np.arange(max(lo, hi - s_i), hi, dtype=np.int64)
            tot += int(((v // s_i) % m_i < m_i - 1).sum()) if hi < n else 0
            v = np.arange(lo, min(hi, lo + s_i), dtype=np.int64)
            tot += int(((v // s_i) % m_i > 0).sum()) if lo > 0 else 0
        worst = max(worst, 8 * tot)
    return worst


def relaunch(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: run this same command
    under torch.distributed.run, one process per GPU (rendezvous on
    127.0.0.1).  Rank 0 prints the line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator size visible in the log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


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
    ap.add_argument("--no-hamming", action="store_true", help="skip the Hamming column")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
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
