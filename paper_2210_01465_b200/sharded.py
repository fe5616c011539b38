"""Key-range sharded analyze_landscape across GPUs.

Rank g of G owns the configuration ranks [lo_g, hi_g): chunk = ceil(N / G)
rounded up to one 512-rank tile, lo_g = g * chunk.  Every rank holds the full
fitness table (8N bytes, read-only) and a full-length replica of the PageRank
contribution vector c; it computes the FFG rows, PageRank values and C_p
partials of its own ranks only.

Per iteration (SURVEY.md A7 with the sums split by shard):
  1. each shard runs one pull step over its ranks, reading c from its replica;
     the kernel writes the new c'[v] into its own replica and -- over NVLink,
     from the same kernel -- into the replica of every peer that owns an
     out-neighbour of v (the only ranks that will pull c'[v]);
  2. the three partial sums (L1 change, dangling mass, sum of r') are summed
     across ranks; that reduction doubles as the barrier that makes every
     peer's remote stores visible before the next step reads them.
The stop rule is evaluated on the summed residual, so all ranks stop on the
same iteration.  f_opt is the minimum of the per-shard (fitness, rank) minima,
C_p the ratio of the summed per-shard numerators and denominators.

The protocol is written against two small interfaces so the same code drives
GPU shards over NCCL (`torch.distributed`, one process per GPU), several
virtual shards on one GPU (tests), and CPU stand-ins over gloo (tests).
"""
from __future__ import annotations

import numpy as np

TILE = 512


def shard_range(n: int, rank: int, nranks: int):
    """[lo, hi) of `rank` (landscape-wide rank ids)."""
    chunk = -(-n // nranks)
    chunk = -(-chunk // TILE) * TILE
    lo = min(n, rank * chunk)
    hi = min(n, lo + chunk)
    return lo, hi


class NonConvergenceError(RuntimeError):
    def __init__(self, iterations, residual):
        super().__init__(f"PageRank did not converge: iterations={iterations} "
                         f"residual={residual:.6e}")
        self.iterations = iterations
        self.residual = residual


def analyze_sharded(shards, allreduce_sum, allgather, kind, damping=0.85, tol=1e-10,
                    max_iter=100000, p_max_percent=15, pagerank_loop=None):
    """Drive `shards` (the shards of this process) through one sharded
    analyze_landscape.

    shards         objects with build(kind), optimum() -> (f, rank, has),
                   pagerank_init(d) -> dangling partial, pagerank_step(D, d)
                   -> (res, dang, sum), centrality(f_opt, ps) -> (nums, den)
    allreduce_sum  f(np.ndarray) -> elementwise sum over all processes
    allgather      f(list) -> concatenation of every process's list
    pagerank_loop  optional f(damping, tol, max_iter) -> (iterations, residual,
                   sum, converged) replacing the host-driven iteration below
                   (device_pagerank_loop: partials all-reduced in device memory)
    """
    edges = minima = 0
    for s in shards:
        e, m = s.build(kind)
        edges += e
        minima += m
    edges, minima = (int(x) for x in allreduce_sum(np.array([edges, minima], np.float64)))

    cands = allgather([s.optimum() for s in shards])
    feas = [(f, r) for f, r, has in cands if has]
    if not feas:
        raise RuntimeError("NoFeasiblePoint: search space has no ok entry")
    f_opt, opt_rank = min(feas)  # lexicographic: lowest rank among equal fitness

    if pagerank_loop is not None:
        it, res, total, converged = pagerank_loop(damping, tol, max_iter)
    else:
        dang = allreduce_sum(np.array([sum(s.pagerank_init(damping) for s in shards)]))[0]
        it, res, total = 0, 0.0, 0.0
        converged = False
        while it < max_iter:
            part = np.zeros(3)
            for s in shards:
                part += np.asarray(s.pagerank_step(dang, damping), np.float64)
            res, dang, total = allreduce_sum(part)
            it += 1
            if res < tol:
                converged = True
                break
    if not converged:
        raise NonConvergenceError(it, res)

    ps = [k / 100.0 for k in range(p_max_percent + 1)]
    acc = np.zeros(len(ps) + 1)
    for s in shards:
        nums, den = s.centrality(f_opt, ps)
        acc[:-1] += nums
        acc[-1] += den
    acc = allreduce_sum(acc)
    if not acc[-1] > 0:
        raise RuntimeError("proportion_of_centrality: minima hold zero PageRank mass")
    return dict(n_edges=edges, n_minima=minima, f_opt=f_opt, opt_rank=opt_rank,
                iterations=it, residual=float(res), pagerank_sum=float(total),
                c_p_curve=[(k, float(acc[k] / acc[-1])) for k in range(len(ps))])


# ------------------------------------------------------------ GPU shards --

class GpuShard:
    """One shard resident on one GPU: a tk_land restricted to [lo, hi)."""

    def __init__(self, radix, rank, nranks, device=0):
        from .landscape import Landscape

        self.land = Landscape(radix, device=device)
        self.rank, self.nranks = rank, nranks
        self.lo, self.hi = self.land.set_shard(rank, nranks)

    def build(self, kind):
        return self.land.build_ffg(kind, node_limit=1 << 32, emit_csr=False)

    def optimum(self):
        return self.land.shard_optimum()

    def pagerank_init(self, damping):
        return self.land.shard_pagerank_init(damping)

    def pagerank_step(self, dangling, damping):
        return self.land.shard_pagerank_step(dangling, damping)

    def centrality(self, f_opt, ps):
        return self.land.shard_centrality(f_opt, ps)


def connect_peers_local(shards):
    """Virtual shards of one process: hand every shard the others' replicas."""
    ptrs = [s.land.replica_ptrs() for s in shards]
    for s in shards:
        s.land.set_peer_ptrs(ptrs)


def connect_peers_ipc(shard, allgather):
    """One shard per process: exchange CUDA IPC handles of the replicas."""
    handles = allgather([shard.land.ipc_handles()])
    shard.land.open_peers(handles)


class DevicePagerankLoop:
    """PageRank iteration control with the partial sums kept in device memory
    (one shard per process, torch.distributed initialised).  Step i's kernel
    and partial reduction are enqueued on the shard's stream and its three
    partials all-reduced in place on that stream (NCCL under torchrun); the
    reduced totals are copied to pinned host memory behind an event, and step
    i+1 -- which reads the reduced dangling mass from device memory -- is
    enqueued before the host waits for that event.  So the stop test of step
    i overlaps step i+1.  When step i converges, step i+1 was speculative: it
    wrote its contributions into the other parity buffer, and tk_shard_pagerank_rewind drops
    it (every rank speculates identically, so the collectives stay matched).
    An instance is the pagerank_loop callable of analyze_sharded; close() it
    before the process group and the CUDA context go away."""

    def __init__(self, shard, device):
        import torch

        self.shard = shard
        self.stream = torch.cuda.ExternalStream(shard.land.stream, device=torch.device(device))
        self.bufs = [torch.zeros(3, dtype=torch.float64, device=device) for _ in range(3)]
        self.host = [torch.zeros(3, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        self.evs = [torch.cuda.Event() for _ in range(2)]

    def _launch(self, i, damping):
        """step i: totals in bufs[i % 3] -> partials in bufs[(i + 1) % 3]"""
        import torch.distributed as dist

        dst = self.bufs[(i + 1) % 3]
        self.shard.land.shard_pagerank_step_dev(self.bufs[i % 3].data_ptr(), damping,
                                                dst.data_ptr())
        dist.all_reduce(dst)
        self.host[i % 2].copy_(dst, non_blocking=True)
        self.evs[i % 2].record(self.stream)

    def __call__(self, damping, tol, max_iter):
        import torch
        import torch.distributed as dist

        with torch.cuda.stream(self.stream):
            self.shard.land.shard_pagerank_init_dev(damping, self.bufs[0].data_ptr())
            dist.all_reduce(self.bufs[0])
            self._launch(0, damping)
            i = 0
            while True:
                if i + 1 < max_iter:
                    self._launch(i + 1, damping)  # speculative until step i's test is read
                self.evs[i % 2].synchronize()
                res, _, total = (float(x) for x in self.host[i % 2])
                if res < tol or i + 1 >= max_iter:
                    if i + 1 < max_iter:
                        self.stream.synchronize()
                        self.shard.land.shard_pagerank_rewind()
                    return i + 1, res, total, res < tol
                i += 1

    def close(self):
        import torch

        self.stream.synchronize()
        self.bufs = self.host = self.evs = None
        torch.cuda.synchronize()


def device_pagerank_loop(shard, device):
    """DevicePagerankLoop(shard, device) -- see there."""
    return DevicePagerankLoop(shard, device)


def torch_collectives(device=None):
    """allreduce_sum / allgather over the default torch.distributed group."""
    import torch
    import torch.distributed as dist

    dev = device if dist.get_backend() == "nccl" else "cpu"

    def allreduce_sum(x):
        t = torch.as_tensor(np.asarray(x, np.float64), device=dev)
        dist.all_reduce(t)
        return t.cpu().numpy()

    def allgather(items):
        out = [None] * dist.get_world_size()
        dist.all_gather_object(out, items)
        return [x for part in out for x in part]

    return allreduce_sum, allgather
