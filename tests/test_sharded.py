"""The key-range sharding protocol of paper_2210_01465_b200/sharded.py.

CPU: world_size-2 gloo run (and virtual shards in one process) with CPU
stand-in shards built on the oracle, checked against the unsharded oracle --
this covers the shard ranges, the per-iteration reduction and stop rule, the
f_opt and C_p combination.  GPU: virtual shards of the real kernels on one
device (peer replicas as plain device pointers) against the oracle.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_2210_01465_b200 import sharded as S

RADIX = [6, 5, 4, 4, 3]
Q, SEED = 0.2, 4


class CpuShard:
    """Test stand-in: the oracle's FFG restricted to [lo, hi), a numpy pull step,
    and the c replica exchanged with the supplied allgather of slices."""

    def __init__(self, radix, fit, ok, rank, nranks, gather_slices):
        self.radix, self.fit, self.ok = radix, fit, ok
        self.n = len(fit)
        self.lo, self.hi = S.shard_range(self.n, rank, nranks)
        self.gather_slices = gather_slices

    def build(self, kind):
        g = O.build_ffg(self.radix, self.fit, self.ok, kind, node_limit=1 << 32)
        off, tg = g["offsets"], g["targets"]
        self.deg = np.diff(off).astype(np.int64)
        src = np.repeat(np.arange(self.n), self.deg)
        order = np.lexsort((src, tg))  # in-CSR, sources ascending per target
        self.in_src, self.in_tgt = src[order], tg[order]
        self.in_off = np.searchsorted(self.in_tgt, np.arange(self.n + 1))
        self.minima = g["minima"][(g["minima"] >= self.lo) & (g["minima"] < self.hi)]
        own = slice(self.lo, self.hi)
        return int(self.deg[own].sum()), len(self.minima)

    def optimum(self):
        sl = slice(self.lo, self.hi)
        okr = np.flatnonzero(self.ok[sl])
        if okr.size == 0:
            return (0.0, 0, False)
        f = self.fit[sl][okr]
        i = int(np.argmin(f))  # first minimum = lowest rank
        return (float(f[i]), int(self.lo + okr[i]), True)

    def _c(self, r):
        c = np.where(self.deg[self.lo:self.hi] > 0, r / np.maximum(self.deg[self.lo:self.hi], 1), 0)
        return c

    def pagerank_init(self, d):
        self.r = np.full(self.hi - self.lo, 1.0 / self.n)
        self.c_full = self.gather_slices(self._c(self.r))
        sinks = self.deg[self.lo:self.hi] == 0
        return float(self.r[sinks].sum())

    def pagerank_step(self, D, d):
        n = self.n
        rn = np.empty_like(self.r)
        for v in range(self.lo, self.hi):
            acc = 0.0
            for u in self.in_src[self.in_off[v]:self.in_off[v + 1]]:
                acc += self.c_full[u]
            rn[v - self.lo] = (1.0 - d) / n + d * (acc + D / n)
        res = float(np.abs(rn - self.r).sum())
        sinks = self.deg[self.lo:self.hi] == 0
        self.r = rn
        self.c_full = self.gather_slices(self._c(rn))
        return res, float(rn[sinks].sum()), float(rn.sum())

    def centrality(self, f_opt, ps):
        r = self.r[self.minima - self.lo]
        f = self.fit[self.minima]
        nums = [float(r[(f <= f_opt) if p == 0 else (f < (1.0 + p) * f_opt)].sum()) for p in ps]
        return np.array(nums), float(r.sum())


def reference(kind):
    fit, ok = O.gen_synthetic(RADIX, Q, "rugged", SEED)
    return fit, ok, O.analyze(RADIX, fit, ok, kind)


def check(res, ref, fit, ok, kind):
    g = ref["ffg"]
    assert res["n_edges"] == len(g["targets"]) and res["n_minima"] == len(g["minima"])
    assert (res["f_opt"], res["opt_rank"]) == (ref["f_opt"], ref["opt_rank"])
    assert res["iterations"] == ref["iterations"]
    assert abs(res["pagerank_sum"] - 1.0) < 1e-9
    for (k, c), (k2, c2) in zip(res["c_p_curve"], ref["c_p_curve"]):
        assert k == k2 and abs(c - c2) <= 1e-9


def test_shard_ranges_cover_space():
    for n in (1, 511, 512, 513, 20736, 113246208):
        for g in (1, 2, 3, 4, 8):
            rs = [S.shard_range(n, r, g) for r in range(g)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(lo % S.TILE == 0 or lo == n for lo, _ in rs)  # empty tail shards


@pytest.mark.parametrize("nshards", [1, 3])
def test_virtual_shards_cpu(nshards):
    kind = O.ADJACENT
    fit, ok, ref = reference(kind)
    n = len(fit)
    box = {}

    def gather_for(rank):
        def g(slice_):
            box[rank] = slice_
            if len(box) == nshards:  # every shard has contributed: publish
                full = np.concatenate([box[r] for r in range(nshards)])
                box.clear()
                box["full"] = full
            return None
        return g

    shards = [CpuShard(RADIX, fit, ok, r, nshards, gather_for(r)) for r in range(nshards)]
    # single-process lockstep: wrap init/step so the replica is published after all shards ran

    class Lock:
        def __init__(self, s):
            self.s = s

        def build(self, kind):
            return self.s.build(kind)

        def optimum(self):
            return self.s.optimum()

        def centrality(self, f_opt, ps):
            return self.s.centrality(f_opt, ps)

    def wrap(method):
        def run(*a):
            out = [getattr(s, method)(*a) for s in shards]
            full = box.pop("full")
            for s in shards:
                s.c_full = full
            return out
        return run

    init, step = wrap("pagerank_init"), wrap("pagerank_step")

    class Group:
        def build(self, kind):
            es = [s.build(kind) for s in shards]
            return sum(e for e, _ in es), sum(m for _, m in es)

        def optimum(self):
            return min((o for o in (s.optimum() for s in shards) if o[2]), default=(0, 0, False))

        def pagerank_init(self, d):
            return sum(init(d))

        def pagerank_step(self, D, d):
            return np.sum(step(D, d), axis=0)

        def centrality(self, f_opt, ps):
            parts = [s.centrality(f_opt, ps) for s in shards]
            return sum(p[0] for p in parts), sum(p[1] for p in parts)

    res = S.analyze_sharded([Group()], lambda x: np.asarray(x, np.float64), lambda xs: xs, kind)
    check(res, ref, fit, ok, kind)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        fit, ok = O.gen_synthetic(RADIX, Q, "rugged", SEED)

        def gather_slices(sl):
            parts = [None] * world
            dist.all_gather_object(parts, sl)
            return np.concatenate(parts)

        shard = CpuShard(RADIX, fit, ok, rank, world, gather_slices)
        allreduce, allgather = S.torch_collectives()
        res = S.analyze_sharded([shard], allreduce, allgather, kind)
        out.put((rank, res))
        del torch
    finally:
        dist.destroy_process_group()


class LocalGroup:
    """Several shards of one process stepped in lockstep; their partials are
    summed locally (the cross-process reduction is then the identity)."""

    def __init__(self, shards):
        self.shards = shards

    def build(self, kind):
        es = [s.build(kind) for s in self.shards]
        return sum(e for e, _ in es), sum(m for _, m in es)

    def optimum(self):
        feas = [o for o in (s.optimum() for s in self.shards) if o[2]]
        return min(feas) if feas else (0.0, 0, False)

    def pagerank_init(self, d):
        return sum(s.pagerank_init(d) for s in self.shards)

    def pagerank_step(self, D, d):
        return np.sum([s.pagerank_step(D, d) for s in self.shards], axis=0)

    def centrality(self, f_opt, ps):
        parts = [s.centrality(f_opt, ps) for s in self.shards]
        return sum(p[0] for p in parts), sum(p[1] for p in parts)


@pytest.mark.gpu
@pytest.mark.parametrize("push", ["crossing", "edges"])  # TK_SHARD_PUSH
@pytest.mark.parametrize("nshards", [1, 2, 3, 8])
@pytest.mark.parametrize("radix", [[8, 8, 6, 6, 4, 4, 2], [6, 5, 4, 4, 3], [2, 9, 7, 5, 3]])
def test_virtual_gpu_shards_match_oracle(radix, nshards, push, monkeypatch):
    import torch

    monkeypatch.setenv("TK_SHARD_PUSH", push)

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n = O.space_size(radix)
    fit, ok = O.gen_iid(n, 0.2, 31)
    ref = O.analyze(radix, fit, ok, O.ADJACENT, node_limit=1 << 32)
    shards = [S.GpuShard(radix, g, nshards, device=0) for g in range(nshards)]
    for s in shards:
        s.land.load_dense(fit, ok)
    S.connect_peers_local(shards)
    res = S.analyze_sharded([LocalGroup(shards)], lambda x: np.asarray(x, np.float64),
                            lambda xs: xs, O.ADJACENT)
    check(res, ref, fit, ok, O.ADJACENT)
    r = np.concatenate([s.land.shard_pagerank_vector(s.lo, s.hi) for s in shards])
    assert np.abs(r - ref["pagerank"]).sum() <= 1e-12
    for s in shards:
        s.land.close()


def _gpu_ipc_worker(rank, world, port, out, dev_loop=False, backend="gloo"):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank if backend == "nccl" else 0  # nccl: one GPU per rank, peers over NVLink
    if backend == "nccl":
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        radix = [8, 8, 6, 6, 4, 4, 2]
        n = O.space_size(radix)
        fit, ok = O.gen_iid(n, 0.2, 31)
        shard = S.GpuShard(radix, rank, world, device=dev)
        shard.land.load_dense(fit, ok)
        allreduce, allgather = S.torch_collectives(device=f"cuda:{dev}" if backend == "nccl"
                                                   else None)
        S.connect_peers_ipc(shard, allgather)
        loop = S.device_pagerank_loop(shard, f"cuda:{dev}") if dev_loop else None
        res = S.analyze_sharded([shard], allreduce, allgather, O.ADJACENT, pagerank_loop=loop)
        r = shard.land.shard_pagerank_vector(shard.lo, shard.hi)
        if loop is not None:
            loop.close()
        out.put((rank, res, shard.lo, r))
        dist.barrier()  # peers stay mapped until everyone is done
        shard.land.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("dev_loop", [False, True])
def test_two_processes_one_gpu_cuda_ipc(dev_loop):
    """The multi-process path end to end on one device: two ranks, replicas
    mapped with CUDA IPC, remote pushes through the mapped pointers; with the
    host-driven iteration and with device-side iteration control (partials
    all-reduced in device memory)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_ipc_worker, args=(r, 2, port, q, dev_loop)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rk, res, lo, r = q.get(timeout=300)
        got[rk] = (res, lo, r)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    radix = [8, 8, 6, 6, 4, 4, 2]
    n = O.space_size(radix)
    fit, ok = O.gen_iid(n, 0.2, 31)
    ref = O.analyze(radix, fit, ok, O.ADJACENT, node_limit=1 << 32)
    check(got[0][0], ref, fit, ok, O.ADJACENT)
    r = np.concatenate([got[k][2] for k in (0, 1)])
    assert np.abs(r - ref["pagerank"]).sum() <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_device_loop_multi_gpu(world):
    """DevicePagerankLoop under NCCL, one process per GPU, peers' replicas
    mapped over NVLink with CUDA IPC.  Needs `world` visible GPUs."""
    import torch

    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_ipc_worker, args=(r, world, port, q, True, "nccl"))
             for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rk, res, lo, r = q.get(timeout=300)
        got[rk] = (res, lo, r)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    radix = [8, 8, 6, 6, 4, 4, 2]
    n = O.space_size(radix)
    fit, ok = O.gen_iid(n, 0.2, 31)
    ref = O.analyze(radix, fit, ok, O.ADJACENT, node_limit=1 << 32)
    check(got[0][0], ref, fit, ok, O.ADJACENT)
    r = np.concatenate([got[k][2] for k in range(world)])
    assert np.abs(r - ref["pagerank"]).sum() <= 1e-12


@pytest.mark.gpu
def test_bench_self_launch_two_ranks_one_gpu():
    """`python bench.py --gpus 2` with no launcher re-executes itself under
    torch.distributed.run; on a one-GPU box both ranks share the device over
    gloo (TK_FORCE_DEVICE=0).  Rank 0 prints one N=2 line."""
    import json
    import subprocess
    import sys

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TK_FORCE_DEVICE="0", TK_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                        "--workload", "c3", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["parallelism"] == "keyrange2"
    assert line["scaling"] == "strong" and line["value"] > 0
    assert line["nvlink_bytes_per_gpu_per_iteration"] > 0


@pytest.mark.parametrize("kind", [O.ADJACENT, O.HAMMING])
def test_two_process_gloo(kind):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    fit, ok, ref = reference(kind)
    for r in (0, 1):
        check(results[r], ref, fit, ok, kind)
    assert results[0] == results[1]


@pytest.mark.gpu
def test_whole_space_calls_refuse_a_sharded_handle():
    """A sharded handle holds only its key range: the whole-space entry points
    return TK_ESTATE instead of shard-local or uninitialised data (tk_landscape.h
    key-range sharding section)."""
    import torch

    import paper_2210_01465_b200 as tk

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    radix = [8, 8, 6, 6, 4]
    n = O.space_size(radix)
    fit, ok = O.gen_iid(n, 0.2, 7)
    s = S.GpuShard(radix, 0, 2, device=0)
    s.land.load_dense(fit, ok)
    s.build(O.ADJACENT)
    for call in (lambda: s.land.optimum(), lambda: s.land.ffg_arrays(), lambda: s.land.census(),
                 lambda: s.land.pagerank(), lambda: s.land.centrality(1.0, [0.0]),
                 lambda: s.land.analyze(O.ADJACENT)):
        with pytest.raises(tk.Error, match="sharded handle"):
            call()
    s.land.close()
