"""ctypes bindings of the CPU oracle (oracle.c) and the reference probes (_ref).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` leg, always as the checker or
the CPU baseline -- never as the product path.  See oracle.h for the parity
pinning story.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libtkref.so")

HAMMING, ADJACENT = 0, 1
OK, EINVAL, ELIMIT, ENOFEAS, ENOCONV, EDEGEN = 0, 1, 2, 3, 4, 5

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")


def build() -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.or_space_strides.restype = C.c_uint64
        L.or_space_strides.argtypes = [C.c_uint32, _u32p, _u64p]
        L.or_max_neighbours.restype = C.c_uint32
        L.or_max_neighbours.argtypes = [C.c_uint32, _u32p, C.c_int]
        L.or_neighbour_ranks.restype = C.c_uint32
        L.or_neighbour_ranks.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_int, _u64p]
        L.or_ffg_count.argtypes = [C.c_uint32, _u32p, _f64p, _u8p, C.c_int, C.c_uint64,
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_int]
        L.or_ffg_fill.argtypes = [C.c_uint32, _u32p, _f64p, _u8p, C.c_int, _u64p, _u32p,
                                  _u8p, _u32p, C.c_int]
        L.or_pagerank.argtypes = [C.c_uint64, _u64p, _u32p, C.c_double, C.c_double,
                                  C.c_int64, _f64p, C.POINTER(C.c_int64),
                                  C.POINTER(C.c_double), C.c_int, C.c_int64]
        L.or_proportion_of_centrality.argtypes = [C.c_uint64, _u32p, _f64p, _f64p,
                                                  C.c_double, C.c_double,
                                                  C.POINTER(C.c_double)]
        L.or_optimum.argtypes = [C.c_uint64, _f64p, _u8p, C.POINTER(C.c_double),
                                 C.POINTER(C.c_uint64)]
        L.or_census.argtypes = [C.c_uint32, _u32p, _f64p, _u8p, C.c_int,
                                C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                C.POINTER(C.c_uint64), C.c_void_p]
        L.or_hash_uniform.restype = C.c_double
        L.or_hash_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        for fn in (L.or_gen_iid, L.or_gen_heavy):
            fn.argtypes = [C.c_uint64, C.c_double, C.c_uint64, _f64p, _u8p, C.c_int]
        L.or_gen_synthetic.argtypes = [C.c_uint32, _u32p, C.c_double, C.c_double,
                                       C.c_double, C.c_double, C.c_uint64, _f64p, _u8p,
                                       C.c_int]
        L.or_descents.argtypes = [C.c_uint32, _u32p, _f64p, C.c_int, C.c_uint64, C.c_uint64,
                                  C.c_int, _u32p, C.POINTER(C.c_uint64), C.c_int]
        _lib = L
    return _lib


def ref():
    """The reference's own compiled space/cache/generators (oracle/_ref)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            build()
        if not os.path.exists(REF_PATH):
            raise FileNotFoundError("oracle/_ref/libtkref.so not built (reference absent)")
        R = C.CDLL(REF_PATH)
        R.ref_space_size.restype = C.c_uint64
        R.ref_space_size.argtypes = [C.c_uint32, _u32p, _u64p]
        R.ref_neighbour_ranks.restype = C.c_uint32
        R.ref_neighbour_ranks.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_int, _u64p]
        R.ref_all_neighbours.restype = C.c_uint64
        R.ref_all_neighbours.argtypes = [C.c_uint32, _u32p, C.c_int, _u64p, _u32p]
        R.ref_generate_synthetic.argtypes = [C.c_uint32, _u32p, C.c_double, C.c_char_p,
                                             C.c_uint64, _f64p, _u8p,
                                             C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        R.ref_generate_nk.argtypes = [C.c_int, C.c_int, C.c_uint64, _f64p]
        R.ref_optimum.argtypes = [C.c_uint32, _u32p, _f64p, _u8p, C.POINTER(C.c_double),
                                  C.POINTER(C.c_uint64)]
        R.ref_load_cache.restype = C.c_longlong
        R.ref_load_cache.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p]
        R.ref_save_synthetic.argtypes = [C.c_uint32, _u32p, C.c_double, C.c_char_p, C.c_uint64,
                                         C.c_char_p]
        R.ref_ffg.argtypes = [C.c_uint32, _u32p, _f64p, _u8p, C.c_int, _u64p, _u32p,
                              C.c_uint64, _u8p, _u32p, C.POINTER(C.c_uint64),
                              C.POINTER(C.c_uint64)]
        _ref = R
    return _ref


def ref_available() -> bool:
    try:
        ref()
        return True
    except (FileNotFoundError, OSError, subprocess.CalledProcessError):
        return False


# ------------------------------------------------------------------ helpers --

def _radix(radix) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(radix, dtype=np.uint32))


def space_size(radix) -> int:
    r = _radix(radix)
    s = np.zeros(len(r), np.uint64)
    return int(lib().or_space_strides(len(r), r, s))


def strides(radix) -> np.ndarray:
    r = _radix(radix)
    s = np.zeros(len(r), np.uint64)
    lib().or_space_strides(len(r), r, s)
    return s


def max_neighbours(radix, kind) -> int:
    r = _radix(radix)
    return int(lib().or_max_neighbours(len(r), r, kind))


def neighbour_ranks(radix, rank, kind) -> np.ndarray:
    r = _radix(radix)
    out = np.zeros(max(1, max_neighbours(r, kind)), np.uint64)
    k = lib().or_neighbour_ranks(len(r), r, rank, kind, out)
    return out[:k].copy()


class OracleError(RuntimeError):
    def __init__(self, status, what=""):
        super().__init__(f"oracle status {status}: {what}")
        self.status = status


def build_ffg(radix, fit, ok, kind, node_limit=1_000_000, nthreads=1):
    """landscape.hpp:44-45 -> dict(offsets, targets, is_sink, minima)."""
    r = _radix(radix)
    fit = np.ascontiguousarray(fit, np.float64)
    ok = np.ascontiguousarray(ok, np.uint8)
    e, m = C.c_uint64(), C.c_uint64()
    st = lib().or_ffg_count(len(r), r, fit, ok, kind, node_limit, C.byref(e), C.byref(m),
                            nthreads)
    if st:
        raise OracleError(st, "build_ffg")
    n = fit.shape[0]
    offsets = np.zeros(n + 1, np.uint64)
    targets = np.zeros(max(1, e.value), np.uint32)
    is_sink = np.zeros(n, np.uint8)
    minima = np.zeros(max(1, m.value), np.uint32)
    st = lib().or_ffg_fill(len(r), r, fit, ok, kind, offsets, targets, is_sink, minima,
                           nthreads)
    if st:
        raise OracleError(st, "build_ffg fill")
    return dict(offsets=offsets, targets=targets[: e.value], is_sink=is_sink,
                minima=minima[: m.value])


def pagerank(offsets, targets, damping=0.85, tol=1e-10, max_iter=100000, nthreads=1,
             fixed_iters=0):
    """landscape.hpp:47-52 -> (r, iterations, residual)."""
    offsets = np.ascontiguousarray(offsets, np.uint64)
    targets = np.ascontiguousarray(targets, np.uint32)
    if targets.size == 0:
        targets = np.zeros(1, np.uint32)
    n = offsets.shape[0] - 1
    r = np.zeros(max(1, n), np.float64)
    it, res = C.c_int64(), C.c_double()
    st = lib().or_pagerank(n, offsets, targets, damping, tol, max_iter, r, C.byref(it),
                           C.byref(res), nthreads, fixed_iters)
    if st:
        raise OracleError(st, f"pagerank iterations={it.value} residual={res.value}")
    return r[:n], it.value, res.value


def proportion_of_centrality(minima, fit, pr, f_opt, p):
    minima = np.ascontiguousarray(minima, np.uint32)
    if minima.size == 0:
        raise OracleError(EDEGEN, "no minima")
    out = C.c_double()
    st = lib().or_proportion_of_centrality(minima.shape[0], minima,
                                           np.ascontiguousarray(fit, np.float64),
                                           np.ascontiguousarray(pr, np.float64),
                                           f_opt, p, C.byref(out))
    if st:
        raise OracleError(st, "proportion_of_centrality")
    return out.value


def optimum(fit, ok):
    f, r = C.c_double(), C.c_uint64()
    st = lib().or_optimum(len(fit), np.ascontiguousarray(fit, np.float64),
                          np.ascontiguousarray(ok, np.uint8), C.byref(f), C.byref(r))
    if st:
        raise OracleError(st, "optimum")
    return f.value, r.value


def descents(radix, fit, kind, walkers, seed, restart_scan=True, nthreads=0):
    """hillclimb.cpp:48-87 climb_random_first from `walkers` uniform starts
    (oracle.c or_descents; same draws as the device validator).  Returns the
    per-rank arrival counts (u32[N]) and the number of fitness evaluations."""
    r = np.ascontiguousarray(radix, np.uint32)
    fit = np.ascontiguousarray(fit, np.float64)
    counts = np.zeros(fit.shape[0], np.uint32)
    ev = C.c_uint64()
    st = lib().or_descents(len(r), r, fit, kind, walkers, seed, int(restart_scan), counts,
                           C.byref(ev), nthreads)
    if st:
        raise OracleError(st, "descents")
    return counts, ev.value


def census(radix, fit, ok, kind):
    r = _radix(radix)
    fit = np.ascontiguousarray(fit, np.float64)
    ok = np.ascontiguousarray(ok, np.uint8)
    fp, lm, it = C.c_uint64(), C.c_uint64(), C.c_uint64()
    mins = np.zeros(fit.shape[0], np.uint64)
    st = lib().or_census(len(r), r, fit, ok, kind, C.byref(fp), C.byref(lm), C.byref(it),
                         mins.ctypes.data)
    if st:
        raise OracleError(st, "census")
    return dict(total=fit.shape[0], fail_points=fp.value, local_minima=lm.value,
                interior=it.value, minima_ranks=mins[: lm.value].copy())


def analyze(radix, fit, ok, kind, damping=0.85, p_max_percent=15, tol=1e-10,
            max_iter=100000, nthreads=1, node_limit=1 << 32):
    """landscape.hpp:77-79 analyze_landscape restated on the oracle."""
    g = build_ffg(radix, fit, ok, kind, node_limit=node_limit, nthreads=nthreads)
    f_opt, opt_rank = optimum(fit, ok)
    pr, iters, res = pagerank(g["offsets"], g["targets"], damping, tol, max_iter,
                              nthreads=nthreads)
    curve = [(k, proportion_of_centrality(g["minima"], fit, pr, f_opt, k / 100.0))
             for k in range(p_max_percent + 1)]
    return dict(ffg=g, f_opt=f_opt, opt_rank=opt_rank, pagerank=pr, iterations=iters,
                residual=res, c_p_curve=curve, pagerank_sum=float(np.sum(pr)))


def gen_iid(n, q, seed, nthreads=1):
    fit = np.empty(n, np.float64)
    ok = np.empty(n, np.uint8)
    lib().or_gen_iid(n, q, seed, fit, ok, nthreads)
    return fit, ok


def gen_heavy(n, q, seed, nthreads=1):
    fit = np.empty(n, np.float64)
    ok = np.empty(n, np.uint8)
    lib().or_gen_heavy(n, q, seed, fit, ok, nthreads)
    return fit, ok


PROFILES = {"smooth": (0.0, 0.01, 0.02), "ridged": (0.6, 0.02, 0.02),
            "rugged": (0.3, 0.08, 0.02)}  # generators.cpp:81-87


def gen_synthetic(radix, q, profile, seed, nthreads=1):
    r = _radix(radix)
    n = space_size(r)
    fit = np.empty(n, np.float64)
    ok = np.empty(n, np.uint8)
    rs, noise, jit = PROFILES[profile]
    st = lib().or_gen_synthetic(len(r), r, q, rs, noise, jit, seed, fit, ok, nthreads)
    if st:
        raise OracleError(st, "gen_synthetic")
    return fit, ok
