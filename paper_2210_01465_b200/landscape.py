"""Host-side mirror of the reference's landscape interface over the C-ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/tunekit/landscape.hpp (declarations only in the
reference) so tests read like the reference's own would:

  classify_points        landscape.hpp:15-24     -> PointCensus
  build_ffg              landscape.hpp:30-45     -> FitnessFlowGraph
  pagerank               landscape.hpp:47-52     -> numpy f64[N]
  proportion_of_centrality  landscape.hpp:54-58  -> float
  analyze_landscape      landscape.hpp:60-79     -> CentralityReport
  minima_fraction_report landscape.hpp:87-94     -> MinimaFractionReport

Errors map onto the reference's classes (errors.hpp:10-44).  Every call runs
on the GPU through libtk_landscape.so; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import TK_ADJACENT, TK_HAMMING  # noqa: F401  (re-export)

HAMMING, ADJACENT = TK_HAMMING, TK_ADJACENT
K_FAIL_FITNESS = 1.0e10  # cache.hpp:15


# ------------------------------------------------------------------ errors --

class Error(RuntimeError):
    """errors.hpp:10-13"""


class InvalidArgument(Error):
    """errors.hpp:15-19"""


class NoFeasiblePoint(Error):
    """errors.hpp:32-35"""


class NonConvergence(Error):
    """errors.hpp:37-42"""

    def __init__(self, what: str, iterations: int, residual: float):
        super().__init__(what)
        self.iterations = iterations
        self.residual = residual


def _check(st: int, iterations: int = 0, residual: float = 0.0) -> None:
    if st == _abi.TK_OK:
        return
    msg = _abi.last_error()
    if st in (_abi.TK_EINVAL, _abi.TK_ELIMIT):
        raise InvalidArgument(msg)
    if st == _abi.TK_ENOFEAS:
        raise NoFeasiblePoint(msg)
    if st == _abi.TK_ENOCONV:
        raise NonConvergence(msg, iterations, residual)
    raise Error(f"{_abi.load().tk_status_name(st).decode()}: {msg}")


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def neighbourhood_from_string(s: str) -> int:
    """space.cpp:12-17"""
    if s in ("hamming", "Hamming"):
        return HAMMING
    if s in ("adjacent", "Adjacent"):
        return ADJACENT
    raise InvalidArgument(f"unknown neighbourhood: {s} (expected hamming or adjacent)")


# ------------------------------------------------------------ data types --

class SearchSpaceCache:
    """The slice of cache.hpp:23-82 the landscape path reads: the space shape
    (list sizes, dim 0 most significant) and the rank-indexed mean/ok tables."""

    def __init__(self, radix, mean, ok, kernel: str = "", device: str = ""):
        self.radix = [int(m) for m in radix]
        self.mean_ = np.ascontiguousarray(mean, np.float64)
        self.ok_ = np.ascontiguousarray(ok, np.uint8)
        n = int(np.prod(self.radix, dtype=np.uint64)) if self.radix else 1
        if self.mean_.shape != (n,) or self.ok_.shape != (n,):
            raise InvalidArgument("cache tables must hold one entry per configuration")
        self.kernel, self.device = kernel, device

    def size(self) -> int:
        return self.mean_.shape[0]

    def mean(self, rank: int) -> float:
        return float(self.mean_[rank])

    def ok(self, rank: int) -> bool:
        return bool(self.ok_[rank])

    def ok_count(self) -> int:
        return int(self.ok_.sum())

    def _opt(self):
        # the cache is immutable (cache.hpp:23-25): one device pass, memoised
        if getattr(self, "_opt_memo", None) is None:
            with Landscape(self.radix) as land:
                land.load_dense(self.mean_, self.ok_)
                self._opt_memo = land.optimum()
        return self._opt_memo

    def optimum(self) -> float:
        """cache.cpp:89-93 (computed on the device)."""
        return self._opt()[0]

    def optimum_rank(self) -> int:
        return self._opt()[1]


@dataclass
class PointCensus:  # landscape.hpp:15-22
    kind: int = ADJACENT
    total: int = 0
    fail_points: int = 0
    local_minima: int = 0
    interior: int = 0
    minima_ranks: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))


@dataclass
class FitnessFlowGraph:  # landscape.hpp:30-42
    kind: int
    node_count: int
    offsets: np.ndarray
    targets: np.ndarray
    fitness: np.ndarray
    is_sink: np.ndarray
    minima: np.ndarray

    def out_degree(self, u: int) -> int:
        return int(self.offsets[u + 1] - self.offsets[u])


@dataclass
class MinimumInfo:  # landscape.hpp:60-65
    rank: int
    fitness: float
    fraction_of_optimum: float
    pagerank: float


@dataclass
class CentralityReport:  # landscape.hpp:67-75 (minima as columns, not row objects)
    kind: int
    damping: float
    f_opt: float
    minima_ranks: np.ndarray
    minima_fitness: np.ndarray
    minima_fraction: np.ndarray
    minima_pagerank: np.ndarray
    c_p_curve: list
    pagerank_iterations: int
    pagerank_sum: float
    n_edges: int = 0
    timings_ms: dict = field(default_factory=dict)

    @property
    def minima(self) -> list[MinimumInfo]:
        return [MinimumInfo(int(r), float(f), float(q), float(p)) for r, f, q, p in
                zip(self.minima_ranks, self.minima_fitness, self.minima_fraction,
                    self.minima_pagerank)]


@dataclass
class MinimaFractionReport:  # landscape.hpp:88-92
    fractions: np.ndarray
    median: float = 0.0
    mean: float = 0.0


# -------------------------------------------------------- device handle --

class Landscape:
    """One search space resident on one GPU (a tk_land handle)."""

    def __init__(self, radix, device: int = 0):
        self.L = _abi.load()
        r = np.ascontiguousarray(radix, np.uint32)
        self.radix = [int(x) for x in r]
        h = C.c_void_p()
        _check(self.L.tk_land_create(device, len(r), _ptr(r), C.byref(h)))
        self.h = h
        n = C.c_uint64()
        _check(self.L.tk_land_info(self.h, C.byref(n), None))
        self.n = n.value
        self.n_edges = 0
        self.n_minima = 0

    def reshape(self, radix):
        """Re-target this handle at another space, keeping its device buffers."""
        r = np.ascontiguousarray(radix, np.uint32)
        _check(self.L.tk_land_reshape(self.h, len(r), _ptr(r)))
        self.radix = [int(x) for x in r]
        n = C.c_uint64()
        _check(self.L.tk_land_info(self.h, C.byref(n), None))
        self.n = n.value
        self.n_edges = self.n_minima = 0

    def close(self):
        if getattr(self, "h", None):
            self.L.tk_land_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(self.L.tk_land_stream(self.h) or 0)

    def kernel_info(self) -> dict:
        sb, sp, g = C.c_int(), C.c_int(), C.c_int()
        mb, mp = C.c_float(), C.c_float()
        _check(self.L.tk_land_kernel_info(self.h, C.byref(sb), C.byref(sp), C.byref(g),
                                          C.byref(mb), C.byref(mp)))
        return dict(staged_build=bool(sb.value), staged_pagerank=sp.value > 0,
                    pagerank_kernel={1: "staged", 2: "rows", 3: "ham_staged",
                                     4: "ham_tiled", 5: "ring", 6: "ham_split"}.get(sp.value, "per-lane"),
                    pagerank_grid=g.value, ms_build=mb.value, ms_pagerank=mp.value)

    # ---- ingestion
    def load_dense(self, fitness, ok, device_ptrs: bool = False):
        if device_ptrs:  # (fitness_ptr, ok_ptr) as ints
            _check(self.L.tk_land_load_dense(self.h, C.c_void_p(fitness), C.c_void_p(ok),
                                             _abi.TK_MEM_DEVICE))
            return
        f = np.ascontiguousarray(fitness, np.float64)
        o = np.ascontiguousarray(ok, np.uint8)
        if f.shape != (self.n,) or o.shape != (self.n,):
            raise InvalidArgument("fitness/ok must have one entry per configuration")
        _check(self.L.tk_land_load_dense(self.h, _ptr(f), _ptr(o), _abi.TK_MEM_HOST))

    def load_sparse(self, keys, fitness):
        k = np.ascontiguousarray(keys, np.uint64)
        f = np.ascontiguousarray(fitness, np.float64)
        _check(self.L.tk_land_load_sparse(self.h, _ptr(k), _ptr(f), k.shape[0],
                                          _abi.TK_MEM_HOST))

    def load_configs(self, configs, fitness):
        c = np.ascontiguousarray(configs, np.int32)
        f = np.ascontiguousarray(fitness, np.float64)
        if c.ndim != 2 or c.shape[1] != len(self.radix):
            raise InvalidArgument("configs must be int32[n_valid][dims]")
        _check(self.L.tk_land_load_configs(self.h, _ptr(c), _ptr(f), c.shape[0],
                                           _abi.TK_MEM_HOST))

    def generate(self, gen: int, fail_fraction: float, seed: int):
        _check(self.L.tk_land_generate(self.h, gen, fail_fraction, seed))

    def fitness(self):
        f = np.empty(self.n, np.float64)
        o = np.empty(self.n, np.uint8)
        _check(self.L.tk_land_copy_fitness(self.h, _ptr(f), _ptr(o)))
        return f, o

    def lookup(self, keys):
        k = np.ascontiguousarray(keys, np.uint64)
        f = np.empty(k.shape[0], np.float64)
        hit = np.empty(k.shape[0], np.uint8)
        _check(self.L.tk_land_lookup(self.h, _ptr(k), k.shape[0], _ptr(f), _ptr(hit)))
        return f, hit

    def optimum(self):
        f, r = C.c_double(), C.c_uint64()
        _check(self.L.tk_optimum(self.h, C.byref(f), C.byref(r)))
        return f.value, r.value

    # ---- FFG
    def build_ffg(self, kind: int, node_limit: int = 1_000_000, emit_csr: bool = True):
        e, m = C.c_uint64(), C.c_uint64()
        _check(self.L.tk_ffg_build(self.h, kind, node_limit, int(emit_csr), C.byref(e),
                                   C.byref(m)))
        self.kind = kind
        self.n_edges, self.n_minima = e.value, m.value
        return self.n_edges, self.n_minima

    def ffg_arrays(self):
        off = np.empty(self.n + 1, np.uint64)
        tg = np.empty(max(1, self.n_edges), np.uint32)
        sk = np.empty(self.n, np.uint8)
        mn = np.empty(max(1, self.n_minima), np.uint32)
        _check(self.L.tk_ffg_copy_out(self.h, _ptr(off), _ptr(tg), _ptr(sk), _ptr(mn)))
        return off, tg[: self.n_edges], sk, mn[: self.n_minima]

    def minima(self) -> np.ndarray:
        """FitnessFlowGraph::minima (landscape.hpp:37) alone, without the CSR."""
        mn = np.empty(max(1, self.n_minima), np.uint32)
        _check(self.L.tk_ffg_copy_out(self.h, None, None, None, _ptr(mn)))
        return mn[: self.n_minima]

    def census(self, with_ranks: bool = True) -> PointCensus:
        fp, lm, it = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(self.L.tk_census(self.h, C.byref(fp), C.byref(lm), C.byref(it), None))
        ranks = np.zeros(lm.value, np.uint64)
        if with_ranks and lm.value:
            _check(self.L.tk_census(self.h, C.byref(fp), C.byref(lm), C.byref(it), _ptr(ranks)))
        return PointCensus(self.kind, self.n, fp.value, lm.value, it.value, ranks)

    # ---- random-walk validator
    def descents(self, walkers: int, seed: int = 0, restart_scan: bool = True):
        """hillclimb.cpp:48-87 climb_random_first from `walkers` uniform starts,
        on the device (tk_descents), in the neighbourhood of the last build.
        Returns (arrivals per FFG minimum in ffg minima order, arrivals at
        failed sinks, fitness evaluations)."""
        arr = np.zeros(self.n_minima, np.uint64)
        fail, ev = C.c_uint64(), C.c_uint64()
        _check(self.L.tk_descents(self.h, walkers, seed, int(restart_scan),
                                  _ptr(arr) if arr.size else None, C.byref(fail), C.byref(ev)))
        return arr, fail.value, ev.value

    # ---- PageRank / C_p
    def pagerank(self, damping=0.85, tol=1e-10, max_iter=100000):
        it, res, s = C.c_int64(), C.c_double(), C.c_double()
        st = self.L.tk_pagerank(self.h, damping, tol, max_iter, C.byref(it), C.byref(res),
                                C.byref(s))
        _check(st, it.value, res.value)
        self.iterations, self.residual, self.pagerank_sum = it.value, res.value, s.value
        return it.value, res.value, s.value

    def pagerank_vector(self):
        r = np.empty(self.n, np.float64)
        _check(self.L.tk_pagerank_copy_out(self.h, _ptr(r)))
        return r

    def centrality(self, f_opt: float, ps):
        p = np.ascontiguousarray(ps, np.float64)
        out = np.empty(p.shape[0], np.float64)
        _check(self.L.tk_centrality(self.h, f_opt, _ptr(p), p.shape[0], _ptr(out)))
        return out

    def report_rows(self, f_opt: float):
        m = self.n_minima
        ranks = np.empty(m, np.uint64)
        fit = np.empty(m, np.float64)
        frac = np.empty(m, np.float64)
        pr = np.empty(m, np.float64)
        _check(self.L.tk_report_copy_out(self.h, f_opt, _ptr(ranks), _ptr(fit), _ptr(frac),
                                         _ptr(pr)))
        return ranks, fit, frac, pr

    # ---- key-range sharding (sharded.py drives these)
    def set_shard(self, rank: int, nranks: int):
        lo, hi = C.c_uint64(), C.c_uint64()
        _check(self.L.tk_land_set_shard(self.h, rank, nranks, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def replica_ptrs(self):
        c0, c1 = C.c_void_p(), C.c_void_p()
        _check(self.L.tk_land_replica_ptrs(self.h, C.byref(c0), C.byref(c1)))
        return c0.value, c1.value

    def set_peer_ptrs(self, ptrs):
        arr0 = (C.c_void_p * len(ptrs))(*[p[0] for p in ptrs])
        arr1 = (C.c_void_p * len(ptrs))(*[p[1] for p in ptrs])
        _check(self.L.tk_land_set_peer_ptrs(self.h, arr0, arr1))

    def ipc_handles(self) -> bytes:
        buf = C.create_string_buffer(128)
        _check(self.L.tk_land_ipc_handles(self.h, buf))
        return buf.raw

    def open_peers(self, handles):
        blob = b"".join(handles)
        _check(self.L.tk_land_open_peers(self.h, C.create_string_buffer(blob, len(blob))))

    def shard_optimum(self):
        f, r, has = C.c_double(), C.c_uint64(), C.c_int()
        _check(self.L.tk_shard_optimum(self.h, C.byref(f), C.byref(r), C.byref(has)))
        return f.value, r.value, bool(has.value)

    def shard_pagerank_init(self, damping):
        d = C.c_double()
        _check(self.L.tk_shard_pagerank_init(self.h, damping, C.byref(d)))
        return d.value

    def shard_pagerank_step(self, dangling, damping):
        r, d, s = C.c_double(), C.c_double(), C.c_double()
        _check(self.L.tk_shard_pagerank_step(self.h, dangling, damping, C.byref(r), C.byref(d),
                                             C.byref(s)))
        return r.value, d.value, s.value

    def shard_pagerank_init_dev(self, damping, partials_ptr: int):
        """Asynchronous on this handle's stream; partials to device memory."""
        _check(self.L.tk_shard_pagerank_init_dev(self.h, damping, C.c_void_p(partials_ptr)))

    def shard_pagerank_step_dev(self, totals_ptr: int, damping, partials_ptr: int):
        """Asynchronous on this handle's stream: reads the previous step's
        all-reduced totals from device memory, writes this shard's partials."""
        _check(self.L.tk_shard_pagerank_step_dev(self.h, C.c_void_p(totals_ptr), damping,
                                                 C.c_void_p(partials_ptr)))

    def shard_pagerank_rewind(self):
        _check(self.L.tk_shard_pagerank_rewind(self.h))

    def shard_centrality(self, f_opt, ps):
        p = np.ascontiguousarray(ps, np.float64)
        nums = np.zeros(p.shape[0], np.float64)
        den = C.c_double()
        _check(self.L.tk_shard_centrality(self.h, f_opt, _ptr(p), p.shape[0], _ptr(nums),
                                          C.byref(den)))
        return nums, den.value

    def shard_pagerank_vector(self, lo, hi):
        r = np.empty(hi - lo, np.float64)
        _check(self.L.tk_shard_pagerank_copy_out(self.h, _ptr(r)))
        return r

    def load_dense_host_ptrs(self, fitness_ptr: int, ok_ptr: int):
        """Upload from host buffers given as raw pointers (pinned memory for
        asynchronous DMA); one entry per configuration."""
        _check(self.L.tk_land_load_dense(self.h, C.c_void_p(fitness_ptr), C.c_void_p(ok_ptr),
                                         _abi.TK_MEM_HOST))

    def report_copy_out_ptrs(self, f_opt: float, rank_ptr: int, fit_ptr: int, ratio_ptr: int,
                             pr_ptr: int):
        """Minima report rows (rank u32 as u64 slot, fitness, f_opt/f, PageRank) into
        caller buffers of n_minima entries each (host or pinned)."""
        _check(self.L.tk_report_copy_out(self.h, f_opt, C.c_void_p(rank_ptr),
                                         C.c_void_p(fit_ptr), C.c_void_p(ratio_ptr),
                                         C.c_void_p(pr_ptr)))

    def analyze(self, kind: int, damping=0.85, tol=1e-10, max_iter=100000,
                node_limit=1_000_000, p_max_percent=15, emit_csr=False):
        s = _abi.ReportSummary()
        st = self.L.tk_analyze(self.h, kind, damping, tol, max_iter, node_limit,
                               p_max_percent, int(emit_csr), C.byref(s))
        _check(st, s.iterations, s.residual)
        self.kind = kind
        self.n_edges, self.n_minima = s.n_edges, s.n_minima
        return s


class AnalysisPipeline:
    """End-to-end analysis of a stream of search spaces of one shape, double
    buffered over two device handles: while one handle runs analyze_landscape,
    a worker thread reads the previous space's minima report back from the
    other handle and uploads the next space's table into it (its own CUDA
    stream, DMA from pinned host memory), so the PCIe transfers of step k+1
    overlap the kernels of step k.  Every step still moves its whole input
    table host->device and its report device->host.

    items: sequence of (fitness_ptr, ok_ptr) pinned host buffers (ints);
    reports: per step a tuple of four pointers (rank, fitness, ratio, pagerank)
    with room for n_minima entries, or None to skip the read-back.
    """

    def __init__(self, radix, device: int = 0):
        from concurrent.futures import ThreadPoolExecutor

        self.lands = [Landscape(radix, device), Landscape(radix, device)]
        self.pool = ThreadPoolExecutor(1)

    def close(self):
        self.pool.shutdown(wait=True)
        for land in self.lands:
            land.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def run(self, items, kind: int, reports=None, **analyze_kw):
        """Analyse every item; returns the list of report summaries.  The
        worker queue is FIFO: upload(k), read_back(k - 1), upload(k + 1), ...
        so a handle's read-back always precedes its next upload, and the main
        thread waits for upload(k) before analysing on handle k % 2."""
        n = len(items)
        out = [None] * n
        if n == 0:
            return out

        def upload(k):
            self.lands[k % 2].load_dense_host_ptrs(*items[k])

        def read_back(k, s):
            if reports is not None and reports[k] is not None:
                self.lands[k % 2].report_copy_out_ptrs(s.f_opt, *reports[k])

        fut_up = self.pool.submit(upload, 0)
        pending = []
        for k in range(n):
            fut_up.result()  # table k resident on handle k % 2
            if k + 1 < n:
                fut_up = self.pool.submit(upload, k + 1)  # overlaps analyze(k)
            out[k] = self.lands[k % 2].analyze(kind, **analyze_kw)
            pending.append(self.pool.submit(read_back, k, out[k]))  # overlaps analyze(k + 1)
        for f in pending:
            f.result()
        return out


class BatchAnalyzer:
    """End-to-end analysis of a batch of independent search spaces of any
    shapes on one GPU (the C4 workload: many small landscapes back to back).
    `workers` host threads each own a device handle (own CUDA stream) and pull
    spaces from a shared queue -- upload, analyze_landscape, report read-back
    -- so host-side launch and synchronisation latency of one space overlaps
    the kernels of the others.  Results come back in input order.

    items: sequence of (radix, fitness_ptr, ok_ptr) host buffers (ints, pinned
    for asynchronous DMA); reports: None or per item a tuple of four pointers
    (rank, fitness, ratio, pagerank) with room for n_minima entries."""

    def __init__(self, device: int = 0, workers: int = 8, radix0=(2,)):
        from concurrent.futures import ThreadPoolExecutor

        self.workers = max(1, int(workers))
        self.device = device
        self.lands = [Landscape(list(radix0), device) for _ in range(self.workers)]
        self.pool = ThreadPoolExecutor(self.workers)

    def close(self):
        self.pool.shutdown(wait=True)
        for land in self.lands:
            land.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def run(self, items, kind: int, reports=None, **analyze_kw):
        """Analyse every item.  Spaces of <= 2^20 configurations (and <= 64
        neighbour slots) go through one tk_batch_analyze call -- one upload, one
        launch with one CTA per space, one read-back; others (or
        TK_BATCH_THREADS=1, or emit_csr) through the worker threads."""
        if not analyze_kw.get("emit_csr") and not os.environ.get("TK_BATCH_THREADS"):
            got = self._run_batched(items, kind, reports, **analyze_kw)
            if got is not None:
                return got
        return self._run_threads(items, kind, reports, **analyze_kw)

    def _run_batched(self, items, kind, reports, damping=0.85, tol=1e-10, max_iter=100000,
                     node_limit=1_000_000, p_max_percent=15, emit_csr=False):
        n = len(items)
        arr = (_abi.BatchItem * max(1, n))()
        for k, (radix, fp, op) in enumerate(items):
            radix = [int(m) for m in radix]
            size = int(np.prod(radix, dtype=np.int64))
            slots = sum((2 if kind == ADJACENT else m - 1) for m in radix if m >= 2)
            if size > (1 << 20) or slots > 64 or len(radix) > 32:
                return None
            if size > node_limit:
                raise InvalidArgument(f"node_limit {node_limit} below the space size {size}")
            it = arr[k]
            it.dims = len(radix)
            for i, m in enumerate(radix):
                it.radix[i] = m
            it.fitness, it.ok = fp, op
            if reports is not None and reports[k] is not None:
                (it.minima_ranks, it.minima_fitness, it.minima_fraction,
                 it.minima_pagerank) = reports[k]
                it.minima_capacity = (1 << 62)
        L = _abi.load()
        _check(L.tk_batch_analyze(self.device, arr, n, kind, damping, tol, max_iter,
                                  p_max_percent, _abi.TK_MEM_HOST))
        out = []
        for k in range(n):
            it = arr[k]
            st = it.status
            if st != _abi.TK_OK:
                s = it.summary
                msgs = {_abi.TK_ENOFEAS: "no feasible point (every configuration failed)",
                        _abi.TK_ENOCONV: f"pagerank did not converge in {s.iterations} iterations",
                        _abi.TK_EDEGEN: "proportion_of_centrality: minima hold zero PageRank mass",
                        _abi.TK_EINVAL: "space not supported by the batch path"}
                if st == _abi.TK_ENOFEAS:
                    raise NoFeasiblePoint(msgs[st])
                if st == _abi.TK_ENOCONV:
                    raise NonConvergence(msgs[st], s.iterations, s.residual)
                if st == _abi.TK_EINVAL:
                    raise InvalidArgument(msgs[st])
                raise Error(msgs.get(st, f"status {st}"))
            s = _abi.ReportSummary()
            C.pointer(s)[0] = it.summary
            out.append(s)
        return out

    def _run_threads(self, items, kind: int, reports=None, **analyze_kw):
        import threading

        out = [None] * len(items)
        nxt = [0]
        lock = threading.Lock()

        def worker(w):
            land = self.lands[w]
            while True:
                with lock:
                    k = nxt[0]
                    nxt[0] += 1
                if k >= len(items):
                    return
                radix, fp, op = items[k]
                if list(radix) != land.radix:
                    land.reshape(radix)
                land.load_dense_host_ptrs(fp, op)
                s = land.analyze(kind, **analyze_kw)
                if reports is not None and reports[k] is not None:
                    land.report_copy_out_ptrs(s.f_opt, *reports[k])
                out[k] = s

        futs = [self.pool.submit(worker, w) for w in range(self.workers)]
        for f in futs:
            f.result()
        return out


# ------------------------------------------------- reference-shaped calls --

def classify_points(cache: SearchSpaceCache, kind: int) -> PointCensus:
    """landscape.hpp:24 -- strict census."""
    with Landscape(cache.radix) as land:
        land.load_dense(cache.mean_, cache.ok_)
        land.build_ffg(kind, node_limit=1 << 32, emit_csr=False)
        return land.census()


def build_ffg(cache: SearchSpaceCache, kind: int, node_limit: int = 1_000_000
              ) -> FitnessFlowGraph:
    """landscape.hpp:44-45"""
    with Landscape(cache.radix) as land:
        land.load_dense(cache.mean_, cache.ok_)
        land.build_ffg(kind, node_limit, emit_csr=True)
        off, tg, sk, mn = land.ffg_arrays()
        return FitnessFlowGraph(kind, land.n, off, tg, cache.mean_.copy(), sk, mn)


def pagerank(g: FitnessFlowGraph, damping: float = 0.85, tol: float = 1e-10,
             max_iter: int = 100000, device: int = 0) -> np.ndarray:
    """landscape.hpp:51-52 -- arbitrary out-CSR, transposed and iterated on the GPU."""
    L = _abi.load()
    off = np.ascontiguousarray(g.offsets, np.uint64)
    tg = np.ascontiguousarray(g.targets, np.uint32)
    n = off.shape[0] - 1
    r = np.empty(max(1, n), np.float64)
    it, res = C.c_int64(), C.c_double()
    st = L.tk_pagerank_csr(device, n, _ptr(off), _ptr(tg) if tg.size else None, damping, tol,
                           max_iter, _ptr(r), C.byref(it), C.byref(res))
    _check(st, it.value, res.value)
    pagerank.last_iterations = it.value
    return r[:n]


def proportion_of_centrality(g: FitnessFlowGraph, pr, f_opt: float, p: float,
                             device: int = 0) -> float:
    """landscape.hpp:56-58 (SURVEY.md A8 threshold)."""
    L = _abi.load()
    mins = np.ascontiguousarray(g.minima, np.int64)
    mf = np.ascontiguousarray(np.asarray(g.fitness)[mins], np.float64)
    mp = np.ascontiguousarray(np.asarray(pr)[mins], np.float64)
    out = C.c_double()
    _check(L.tk_proportion_of_centrality(device, mins.shape[0], _ptr(mf), _ptr(mp), f_opt, p,
                                         C.byref(out)))
    return out.value


def analyze_landscape(cache: SearchSpaceCache, kind: int, damping: float = 0.85,
                      p_max_percent: int = 15, node_limit: int = 1_000_000,
                      tol: float = 1e-10, max_iter: int = 100000) -> CentralityReport:
    """landscape.hpp:77-79, plus the node_limit overload."""
    with Landscape(cache.radix) as land:
        land.load_dense(cache.mean_, cache.ok_)
        s = land.analyze(kind, damping, tol, max_iter, node_limit, p_max_percent)
        ranks, fit, frac, prv = land.report_rows(s.f_opt)
        return CentralityReport(kind, damping, s.f_opt, ranks, fit, frac, prv,
                                [(k, s.c_p[k]) for k in range(s.n_cp)], s.iterations,
                                s.pagerank_sum, s.n_edges,
                                dict(ffg=s.ms_ffg, pagerank=s.ms_pagerank,
                                     centrality=s.ms_centrality))


def minima_fraction_report(cache: SearchSpaceCache, kind: int) -> MinimaFractionReport:
    """landscape.hpp:87-94: f_opt / f over the FFG minima, ascending."""
    with Landscape(cache.radix) as land:
        land.load_dense(cache.mean_, cache.ok_)
        land.build_ffg(kind, node_limit=1 << 32, emit_csr=False)
        f_opt, _ = land.optimum()
        mins = land.minima()
    fr = np.sort(f_opt / cache.mean_[mins])
    k = fr.size
    if k == 0:
        return MinimaFractionReport(fr)
    med = fr[k // 2] if k % 2 else 0.5 * (fr[k // 2 - 1] + fr[k // 2])
    # sequential sum (cumsum), the order of the C++ drop-in's loop
    return MinimaFractionReport(fr, float(med), float(np.cumsum(fr)[-1] / k))
