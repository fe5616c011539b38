"""GPU parity: the CUDA path through the C-ABI against the CPU oracle and the
golden fixtures of the reference's own code.

Bars (BASELINE.json north_star): FFG CSR, is_sink and minima bit-exact;
PageRank within 1e-12 relative L1 with the same iteration count; C_p within
1e-9 absolute.
"""
import hashlib

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

PR_RTOL = 1e-12  # relative L1 on the rank vector
CP_ATOL = 1e-9   # absolute on C_p


@pytest.fixture(scope="module")
def tk():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2210_01465_b200 as tk

    tk._abi.load()
    return tk


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rel_l1(a, b):
    return float(np.abs(a - b).sum() / np.abs(b).sum())


def gpu_ffg(tk, radix, fit, ok, kind):
    with tk.Landscape(radix) as land:
        land.load_dense(fit, ok)
        land.build_ffg(kind, node_limit=1 << 32, emit_csr=True)
        return land.ffg_arrays()


# ------------------------------------------------------------------ inputs --

@pytest.mark.parametrize("gen", [0, 1])
def test_device_generators_bit_identical(tk, gen):
    n = 1 << 20
    with tk.Landscape([1 << 10, 1 << 10]) as land:
        land.generate(gen, 0.3, 17)
        f, o = land.fitness()
    rf, ro = (O.gen_iid if gen == 0 else O.gen_heavy)(n, 0.3, 17, nthreads=8)
    assert np.array_equal(f.view(np.uint64), rf.view(np.uint64))
    assert np.array_equal(o, ro)


def test_sparse_hash_ingest_matches_dense(tk):
    radix = [12, 6, 8, 8, 2, 2]
    fit, ok = O.gen_synthetic(radix, 0.68, "rugged", 3)
    keys = np.flatnonzero(ok).astype(np.uint64)
    rng = np.random.default_rng(0)
    perm = rng.permutation(keys.shape[0])
    with tk.Landscape(radix) as land:
        land.load_sparse(keys[perm], fit[keys][perm])
        f, o = land.fitness()
        assert np.array_equal(f.view(np.uint64), fit.view(np.uint64))
        assert np.array_equal(o, ok)
        q = np.array([keys[0], keys[-1], 0, len(fit) - 1], np.uint64)
        lf, hit = land.lookup(q)
        assert list(hit) == [1, 1, ok[0], ok[-1]]
        assert lf[0] == fit[keys[0]]
        # configurations as index vectors -> mixed-radix keys on the device
        strides = O.strides(radix).astype(np.int64)
        cfg = np.stack([(keys.astype(np.int64) // s) % m for s, m in zip(strides, radix)], 1)
        land.load_configs(cfg.astype(np.int32), fit[keys])
        f2, o2 = land.fitness()
        assert np.array_equal(f2.view(np.uint64), fit.view(np.uint64))
        assert np.array_equal(o2, ok)
        with pytest.raises(tk.InvalidArgument):
            land.load_sparse(np.array([1, 2, 1], np.uint64), np.ones(3))
        with pytest.raises(tk.InvalidArgument):
            land.load_sparse(np.array([len(fit)], np.uint64), np.ones(1))
        bad = cfg[:2].copy()
        bad[1, 0] = radix[0]
        with pytest.raises(tk.InvalidArgument):
            land.load_configs(bad.astype(np.int32), np.ones(2))


# --------------------------------------------------------------------- FFG --

@pytest.mark.parametrize("kind", [O.HAMMING, O.ADJACENT])
def test_ffg_matches_reference_golden(tk, golden, kind):
    meta, arrays = golden
    for rec in meta["synthetic"]:
        fit, ok = O.gen_synthetic(rec["radix"], rec["q"], rec["profile"], rec["seed"])
        off, tg, sk, mn = gpu_ffg(tk, rec["radix"], fit, ok, kind)
        ref = rec["ffg"][str(kind)]
        assert len(tg) == ref["edges"], rec["key"]
        assert sha(off) == ref["sha_offsets"], rec["key"]
        assert sha(tg) == ref["sha_targets"], rec["key"]
        assert sha(sk) == ref["sha_is_sink"], rec["key"]
        assert sha(mn) == ref["sha_minima"], rec["key"]


@pytest.mark.parametrize("radix,kind,gen", [
    ([12, 12, 12, 12], O.ADJACENT, "iid"),               # C1, packed masks
    ([16, 12, 8, 8, 8, 4, 2, 2], O.ADJACENT, "syn"),     # C2 shape
    ([2] * 16, O.ADJACENT, "iid"),                       # 32 ordered slots (u32, unpacked)
    ([2] * 20, O.ADJACENT, "iid"),                       # 40 ordered slots (u64)
    ([3] * 14, O.HAMMING, "heavy"),                      # 28 Hamming slots
    ([8, 8, 6, 6, 4, 4, 2], O.HAMMING, "iid"),           # 33 Hamming slots (u64)
    ([5, 1, 7, 1, 3], O.ADJACENT, "syn"),                # singleton dims are dropped
    ([1], O.ADJACENT, "iid"),                            # single node
])
def test_ffg_and_census_bit_exact(tk, radix, kind, gen):
    n = O.space_size(radix)
    if gen == "iid":
        fit, ok = O.gen_iid(n, 0.2, 5)
    elif gen == "heavy":
        fit, ok = O.gen_heavy(n, 0.1, 6)
    else:
        fit, ok = O.gen_synthetic(radix, 0.3, "rugged", 7)
    ref = O.build_ffg(radix, fit, ok, kind, node_limit=1 << 32, nthreads=8)
    with tk.Landscape(radix) as land:
        land.load_dense(fit, ok)
        land.build_ffg(kind, node_limit=1 << 32, emit_csr=True)
        off, tg, sk, mn = land.ffg_arrays()
        cen = land.census()
    assert np.array_equal(off, ref["offsets"])
    assert np.array_equal(tg, ref["targets"])
    assert np.array_equal(sk, ref["is_sink"])
    assert np.array_equal(mn, ref["minima"])
    rc = O.census(radix, fit, ok, kind)
    assert cen.fail_points == rc["fail_points"]
    assert cen.local_minima == rc["local_minima"]
    assert cen.interior == rc["interior"]
    assert np.array_equal(cen.minima_ranks, rc["minima_ranks"])


@pytest.mark.parametrize("path", ["staged", "v1"])
def test_ffg_with_nan_fitness_bit_exact(tk, monkeypatch, path):
    """NaN fitness values (all fp64 comparisons with them are false): the FFG
    edges (f(v) < f(u)), sinks and minima stay bit-exact, and the strict census
    keeps its definition -- every neighbour strictly greater -- so a NaN node or
    a NaN neighbour is never a census minimum."""
    if path == "v1":
        monkeypatch.setenv("TK_KERNELS", "v1")
    radix = [8, 6, 6, 4, 4]
    fit, ok = O.gen_iid(O.space_size(radix), 0.2, 7)
    fit = fit.copy()
    fit[[5, 777, 2048]] = np.nan
    ref = O.build_ffg(radix, fit, ok, O.ADJACENT, node_limit=1 << 32, nthreads=8)
    off, tg, sk, mn = gpu_ffg(tk, radix, fit, ok, O.ADJACENT)
    assert np.array_equal(off, ref["offsets"]) and np.array_equal(tg, ref["targets"])
    assert np.array_equal(sk, ref["is_sink"]) and np.array_equal(mn, ref["minima"])
    with tk.Landscape(radix) as land:
        land.load_dense(fit, ok)
        land.build_ffg(O.ADJACENT, node_limit=1 << 32, emit_csr=False)
        cen = land.census()
    rc = O.census(radix, fit, ok, O.ADJACENT)
    assert np.array_equal(cen.minima_ranks, rc["minima_ranks"])


def test_census_with_ties(tk):
    # SPEC.md:387 constant space: no strict minima, every ok node an FFG minimum
    radix = [4, 3, 5]
    fit = np.full(60, 2.5)
    ok = np.ones(60, np.uint8)
    ok[7] = 0
    fit[7] = 1e10
    for kind in (O.HAMMING, O.ADJACENT):
        with tk.Landscape(radix) as land:
            land.load_dense(fit, ok)
            _, m = land.build_ffg(kind)
            c = land.census()
        assert c.local_minima == 0 and c.fail_points == 1 and c.interior == 59
        assert m == 59


def test_node_limit_and_errors(tk):
    with tk.Landscape([64, 64]) as land:
        fit, ok = O.gen_iid(4096, 0.0, 1)
        land.load_dense(fit, ok)
        with pytest.raises(tk.InvalidArgument, match="node limit"):
            land.build_ffg(O.ADJACENT, node_limit=4095)
        with pytest.raises(tk.Error):
            land.pagerank()  # build first
    with tk.Landscape([3, 3]) as land:
        land.load_dense(np.full(9, 1e10), np.zeros(9, np.uint8))
        with pytest.raises(tk.NoFeasiblePoint):
            land.analyze(O.ADJACENT)


# ---------------------------------------------------------------- PageRank --

@pytest.mark.parametrize("radix,kind", [
    ([12, 12, 12, 12], O.ADJACENT),
    ([2] * 16, O.ADJACENT),
    ([2] * 20, O.ADJACENT),
    ([3] * 10, O.HAMMING),
    ([8, 8, 6, 6, 4, 4, 2], O.HAMMING),
    ([16, 12, 8, 8, 8, 4, 2, 2], O.ADJACENT),
])
def test_pagerank_structured_matches_oracle(tk, radix, kind):
    n = O.space_size(radix)
    fit, ok = O.gen_iid(n, 0.25, 11)
    ref = O.analyze(radix, fit, ok, kind, nthreads=1, node_limit=1 << 32)
    with tk.Landscape(radix) as land:
        land.load_dense(fit, ok)
        land.build_ffg(kind, node_limit=1 << 32, emit_csr=False)
        it, res, s = land.pagerank()
        r = land.pagerank_vector()
        f_opt, orank = land.optimum()
        cps = land.centrality(f_opt, [k / 100.0 for k in range(16)])
    assert it == ref["iterations"]
    assert rel_l1(r, ref["pagerank"]) <= PR_RTOL
    assert abs(s - 1.0) < 1e-9
    assert (f_opt, orank) == (ref["f_opt"], ref["opt_rank"])
    assert np.max(np.abs(cps - [c for _, c in ref["c_p_curve"]])) <= CP_ATOL


@pytest.mark.parametrize("path", ["staged", "v1"])
@pytest.mark.parametrize("radix,q", [
    ([8, 8, 8, 6, 6, 6, 4, 4, 4, 4, 2, 1], 0.1),   # C5 shape minus its last dim
    ([12, 12, 12, 12], 0.0),
    ([7, 5, 3, 2, 9], 0.3),                         # odd strides: unaligned ranges
    ([1000, 3], 0.2),                               # near window only / far only
    ([3, 1000], 0.2),
    ([2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2], 0.5),  # 26 slots, packed limit
    ([5], 0.0),
])
def test_staged_and_v1_paths_match_oracle(tk, monkeypatch, path, radix, q):
    if path == "v1":
        monkeypatch.setenv("TK_KERNELS", "v1")
    n = O.space_size(radix)
    fit, ok = O.gen_iid(n, q, 23)
    if q == 0.0 and n < 100:
        ok[:] = 1
    ref = O.build_ffg(radix, fit, ok, O.ADJACENT, node_limit=1 << 32, nthreads=8)
    with tk.Landscape(radix) as land:
        land.load_dense(fit, ok)
        land.build_ffg(O.ADJACENT, node_limit=1 << 32, emit_csr=True)
        off, tg, sk, mn = land.ffg_arrays()
        cen = land.census()
        it, res, s = land.pagerank()
        r = land.pagerank_vector()
        info = land.kernel_info()
    assert info["staged_build"] == (path == "staged")
    assert info["staged_pagerank"] == (path == "staged")
    assert np.array_equal(off, ref["offsets"]) and np.array_equal(tg, ref["targets"])
    assert np.array_equal(sk, ref["is_sink"]) and np.array_equal(mn, ref["minima"])
    rc = O.census(radix, fit, ok, O.ADJACENT)
    assert np.array_equal(cen.minima_ranks, rc["minima_ranks"])
    rr, rit, _ = O.pagerank(ref["offsets"], ref["targets"], nthreads=1)
    assert it == rit and rel_l1(r, rr) <= PR_RTOL


# Row-tiled PageRank (tk_rows.cu): shapes whose trailing dims span 16 ranks,
# one per in-row structure, plus odd column lengths (tiles straddling columns)
# and the C2 shape; the staged kernel (TK_PR_ROWS=0) on the same shapes.
@pytest.mark.parametrize("rows", ["rows", "rows_win", "staged"])
@pytest.mark.parametrize("radix,q", [
    ([8, 6, 6, 4, 4, 4, 2, 2], 0.1),      # C5's trailing dims (4,2,2)
    ([6, 8, 8, 4, 4], 0.2),               # (4,4)
    ([3] + [2] * 10, 0.3),                # (2,2,2,2)
    ([12, 12, 16, 16], 0.0),              # (16)
    ([8, 8, 8, 8, 2], 0.1),               # (8,2)
    ([16, 12, 2, 8], 0.1),                # (2,8)
    ([8, 12, 10, 2, 4, 2], 0.2),          # (2,4,2), column of 5*... rows
    ([5, 16, 8, 2, 2, 4], 0.2),           # (2,2,4)
    ([7, 8, 4, 3, 4, 2, 2], 0.25),        # odd radices: super-columns, straddling tiles
    ([16, 12, 8, 8, 8, 4, 2, 2], 0.3),    # C2 shape
])
def test_row_tiled_pagerank_matches_oracle(tk, monkeypatch, rows, radix, q):
    monkeypatch.setenv("TK_PR_ROWS", "0" if rows == "staged" else "1")
    if rows == "staged":
        monkeypatch.setenv("TK_PR_STAGED", "1")
    if rows == "rows_win":  # the largest window the ring allows, however few columns
        monkeypatch.setenv("TK_ROW_MINCOLS", "1")
    n = O.space_size(radix)
    fit, ok = O.gen_iid(n, q, 29)
    if q == 0.0:
        ok[:] = 1
    ref = O.analyze(radix, fit, ok, O.ADJACENT, nthreads=8, node_limit=1 << 32)
    with tk.Landscape(radix) as land:
        land.load_dense(fit, ok)
        s = land.analyze(tk.ADJACENT, node_limit=1 << 32)
        r = land.pagerank_vector()
        info = land.kernel_info()
    assert info["pagerank_kernel"] == rows.split("_")[0]
    assert s.iterations == ref["iterations"]
    assert rel_l1(r, ref["pagerank"]) <= PR_RTOL
    for k, c in ref["c_p_curve"]:
        assert abs(s.c_p[k] - c) <= CP_ATOL


@pytest.mark.parametrize("path", ["split", "staged", "tiled", "v1"])
@pytest.mark.parametrize("radix,q", [
    ([6, 6, 4, 4, 4, 4, 2, 2], 0.2),       # uniform / tile-aligned / per-thread digits
    ([4, 4, 4, 4, 4, 4, 4, 4, 4, 4], 0.1),  # split: three dimension groups (LO / LOHI / HI / OUTER)
    ([8, 8, 8, 6, 6, 6, 4, 4, 2], 0.1),    # split: C5's outer dims, three groups
    ([8, 4, 4, 4, 2, 2, 4], 0.0),          # N = 8192, one uniform dim
    ([8, 8, 8, 4, 4, 4, 4, 2, 2], 0.1),    # 35 Hamming slots: u64 in-masks
    ([4, 4, 4, 4, 2], 0.3),                # N = 512: one tile, all digits per thread
    ([7, 5, 3, 4, 4, 4, 2, 2, 2], 0.15),   # odd outer radices, block of 512 (one tile)
    ([3, 5, 8, 4, 4, 4, 2, 2], 0.05),      # block of 2048 ranks (4 tiles per block)
    ([5, 3, 16, 4, 4, 4, 2, 2], 0.4),      # block of 4096 (8 tiles), 40 % failed
    ([2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2], 0.1),  # 5 outer binary dims
])
def test_hamming_tiled_pagerank_matches_oracle(tk, monkeypatch, path, radix, q):
    """The Hamming kernels (tk_hamsplit.cu: in-edge sum split by dimension
    groups; tk_hamming.cu: staged -- outer lines through a TMA ring, inner lines
    from a block copy -- and tiled) and the per-lane one agree with the oracle:
    same iteration count, rank vector within 1e-12, C_p within 1e-9."""
    monkeypatch.setenv("TK_HAM_SPLIT", "1" if path == "split" else "0")
    if path == "v1":
        monkeypatch.setenv("TK_KERNELS", "v1")
    if path == "staged":
        monkeypatch.setenv("TK_HAM_STAGED", "1")
    n = O.space_size(radix)
    fit, ok = O.gen_iid(n, q, 31)
    ref = O.analyze(radix, fit, ok, O.HAMMING, nthreads=8, node_limit=1 << 32)
    with tk.Landscape(radix) as land:
        land.load_dense(fit, ok)
        land.build_ffg(O.HAMMING, node_limit=1 << 32, emit_csr=False)
        it, res, s = land.pagerank()
        r = land.pagerank_vector()
        f_opt, _ = land.optimum()
        cps = land.centrality(f_opt, [k / 100.0 for k in range(16)])
        used = land.kernel_info()["pagerank_kernel"]
    if path == "staged" and n > 512 and radix != [8, 8, 8, 6, 6, 6, 4, 4, 2]:  # strides off 512
        assert used == "ham_staged", used
    if path == "split" and max(radix) <= 8:
        assert used == "ham_split", used
    assert it == ref["iterations"]
    assert rel_l1(r, ref["pagerank"]) <= PR_RTOL
    assert abs(s - 1.0) < 1e-9
    assert np.max(np.abs(cps - [c for _, c in ref["c_p_curve"]])) <= CP_ATOL


def test_pagerank_csr_dropin_matches_oracle(tk):
    radix = [8, 6, 3, 3, 2]
    fit, ok = O.gen_synthetic(radix, 0.52, "rugged", 2)
    cache = tk.SearchSpaceCache(radix, fit, ok)
    for kind in (O.HAMMING, O.ADJACENT):
        g = tk.build_ffg(cache, kind)
        r = tk.pagerank(g)
        ref, it, _ = O.pagerank(g.offsets, g.targets)
        assert tk.pagerank.last_iterations == it
        assert rel_l1(r, ref) <= PR_RTOL
        f_opt = cache.optimum()
        for p in (0.0, 0.01, 0.05, 0.15, 3.0):
            got = tk.proportion_of_centrality(g, r, f_opt, p)
            exp = O.proportion_of_centrality(g.minima, fit, ref, f_opt, p)
            assert abs(got - exp) <= CP_ATOL


def test_pagerank_spec_examples(tk):
    FFG = tk.FitnessFlowGraph
    one = FFG(O.ADJACENT, 1, np.array([0, 0], np.uint64), np.zeros(0, np.uint32),
              np.ones(1), np.ones(1, np.uint8), np.zeros(1, np.uint32))
    assert tk.pagerank(one)[0] == 1.0
    ab = FFG(O.ADJACENT, 2, np.array([0, 1, 1], np.uint64), np.array([1], np.uint32),
             np.array([2.0, 1.0]), np.array([0, 1], np.uint8), np.array([1], np.uint32))
    r = tk.pagerank(ab, damping=1.0, tol=1e-15)
    assert abs(r[0] - 1 / 3) < 1e-14 and abs(r[1] - 2 / 3) < 1e-14
    with pytest.raises(tk.NonConvergence) as e:
        tk.pagerank(ab, max_iter=3)
    assert e.value.iterations == 3 and e.value.residual > 0
    for bad in (dict(damping=1.5), dict(tol=0.0), dict(max_iter=0)):
        with pytest.raises(tk.InvalidArgument):
            tk.pagerank(ab, **bad)


def test_analyze_landscape_matches_oracle(tk, golden):
    meta, _ = golden
    for rec in meta["synthetic"]:
        if rec["status"] != 0:
            continue
        fit, ok = O.gen_synthetic(rec["radix"], rec["q"], rec["profile"], rec["seed"])
        cache = tk.SearchSpaceCache(rec["radix"], fit, ok)
        for kind in (O.HAMMING, O.ADJACENT):
            rep = tk.analyze_landscape(cache, kind)
            ref = O.analyze(rec["radix"], fit, ok, kind)
            assert rep.f_opt == rec["f_opt"]
            assert rep.pagerank_iterations == ref["iterations"]
            mins = ref["ffg"]["minima"]
            assert np.array_equal(rep.minima_ranks, mins.astype(np.uint64))
            assert np.array_equal(rep.minima_fitness, fit[mins])
            assert np.array_equal(rep.minima_fraction, rec["f_opt"] / fit[mins])
            assert rel_l1(rep.minima_pagerank, ref["pagerank"][mins]) <= 1e-11
            assert abs(rep.pagerank_sum - 1.0) < 1e-9
            for (k, c), (k2, c2) in zip(rep.c_p_curve, ref["c_p_curve"]):
                assert k == k2 and abs(c - c2) <= CP_ATOL


# ------------------------------------------- full-size, size-independent checks --

@pytest.mark.parametrize("kind", [O.ADJACENT, O.HAMMING])
@pytest.mark.parametrize("config", ["c1", "c2"])
def test_baseline_c1_c2_instances_match_oracle(tk, config, kind):
    """BASELINE.json configs[0] and configs[1] exactly as the bench runs them:
    C1 = (12,12,12,12) G_iid q = 0 seed 1 generated on the device; C2 =
    (16,12,8,8,8,4,2,2) generate_synthetic_kernel_space 'rugged' q = 0.3 seed 2
    (the reference's generator, restated bit-for-bit by the oracle).  FFG CSR
    and minima bit-exact, PageRank within 1e-12 with the same iteration count,
    C_p within 1e-9, the report rows exact."""
    if config == "c1":
        radix = [12, 12, 12, 12]
        with tk.Landscape(radix) as src:
            src.generate(0, 0.0, 1)
            fit, ok = src.fitness()
        assert np.array_equal(fit.view(np.uint64), O.gen_iid(O.space_size(radix), 0.0, 1)[0].view(np.uint64))
    else:
        radix = [16, 12, 8, 8, 8, 4, 2, 2]
        fit, ok = O.gen_synthetic(radix, 0.30, "rugged", 2)
    ref = O.analyze(radix, fit, ok, kind, nthreads=8, node_limit=1 << 32)
    with tk.Landscape(radix) as land:
        land.load_dense(fit, ok)
        s = land.analyze(kind, node_limit=1 << 32, emit_csr=True)
        off, tg, sk, mn = land.ffg_arrays()
        r = land.pagerank_vector()
        rows = land.report_rows(s.f_opt)
    g = ref["ffg"]
    assert np.array_equal(off, g["offsets"]) and np.array_equal(tg, g["targets"])
    assert np.array_equal(sk, g["is_sink"]) and np.array_equal(mn, g["minima"])
    assert s.iterations == ref["iterations"]
    assert rel_l1(r, ref["pagerank"]) <= PR_RTOL
    for k, c in ref["c_p_curve"]:
        assert abs(s.c_p[k] - c) <= CP_ATOL
    ranks, fmin, frac, prm = rows
    assert np.array_equal(ranks, g["minima"].astype(np.uint64))
    assert np.array_equal(fmin.view(np.uint64), fit[g["minima"]].view(np.uint64))
    assert np.array_equal(frac, ref["f_opt"] / fit[g["minima"]])


@pytest.mark.parametrize("radix,kind,gen,q", [
    ([8, 8, 8, 8, 6, 6, 4, 4, 2, 2], O.ADJACENT, 1, 0.0),   # C3 shape, heavy tails
    ([8, 8, 8, 8, 6, 6, 4, 4, 2, 2], O.HAMMING, 1, 0.0),
])
def test_c3_scale_properties_and_parity(tk, radix, kind, gen, q):
    n = O.space_size(radix)
    with tk.Landscape(radix) as land:
        land.generate(gen, q, 3)
        e, m = land.build_ffg(kind, node_limit=1 << 32, emit_csr=True)
        # tie-free, no failures: E is structural
        if kind == O.ADJACENT:
            assert e == sum(n * (mm - 1) // mm for mm in radix)
        else:
            assert e == sum(n * (mm - 1) // 2 for mm in radix)
        off, tg, sk, mn = land.ffg_arrays()
        fit, ok = land.fitness()
        it, res, s = land.pagerank()
        r = land.pagerank_vector()
        f_opt, _ = land.optimum()
        cps = land.centrality(f_opt, [k / 100.0 for k in range(16)])
    ref = O.build_ffg(radix, fit, ok, kind, node_limit=1 << 32, nthreads=8)
    assert np.array_equal(off, ref["offsets"]) and np.array_equal(tg, ref["targets"])
    assert np.array_equal(mn, ref["minima"])
    assert abs(s - 1.0) < 1e-9 and res < 1e-10
    assert np.all(np.diff(cps) >= -1e-15) and 0 <= cps[0] and cps[-1] <= 1 + 1e-15
    rr, rit, _ = O.pagerank(off, tg, nthreads=8)
    assert it == rit and rel_l1(r, rr) <= PR_RTOL


def test_analysis_pipeline_matches_single_handle(tk):
    """tk.AnalysisPipeline (double-buffered uploads / report read-backs over two
    handles) returns, per space, exactly what one handle's analyze + report
    rows return, on a stream of different spaces of one shape."""
    radix = [8, 6, 6, 4, 4, 2]
    tables = [O.gen_synthetic(radix, q, "rugged", seed) for seed, q in
              ((0, 0.3), (1, 0.1), (2, 0.5), (3, 0.0), (4, 0.2))]
    want = []
    for fit, ok in tables:
        with tk.Landscape(radix) as land:
            land.load_dense(fit, ok)
            s = land.analyze(tk.ADJACENT, emit_csr=True)
            want.append((s.iterations, s.n_edges, s.n_minima, list(s.c_p[:16]),
                         land.report_rows(s.f_opt)))
    hosts = [(np.ascontiguousarray(f, np.float64), np.ascontiguousarray(o, np.uint8))
             for f, o in tables]
    items = [(f.ctypes.data, o.ctypes.data) for f, o in hosts]
    bufs = [[np.empty(max(1, w[2]), dt) for dt in (np.uint64, np.float64, np.float64,
                                                   np.float64)] for w in want]
    reports = [tuple(b.ctypes.data for b in bb) for bb in bufs]
    with tk.AnalysisPipeline(radix) as pipe:
        got = pipe.run(items, tk.ADJACENT, reports, emit_csr=True)
    for s, w, bb in zip(got, want, bufs):
        assert (s.iterations, s.n_edges, s.n_minima) == w[:3]
        assert list(s.c_p[:16]) == w[3]
        for a, b in zip(bb, w[4]):
            assert np.array_equal(a[: w[2]], b)


@pytest.mark.parametrize("path", ["batched", "batched_one_cta", "threads"])
@pytest.mark.parametrize("kind", [O.ADJACENT, O.HAMMING])
def test_batch_analyzer_matches_oracle(tk, monkeypatch, path, kind):
    """tk.BatchAnalyzer on both of its paths -- one tk_batch_analyze launch with
    one CTA per space, and worker threads driving several handles / streams --
    against the oracle: iterations, edges and minima exact, C_p within 1e-9,
    report rows (ranks, fitness, fraction of optimum) exact and the minima's
    PageRank within 1e-12."""
    if path == "threads":
        monkeypatch.setenv("TK_BATCH_THREADS", "1")
    if path == "batched_one_cta":  # one CTA per space (no CTA groups)
        monkeypatch.setenv("TK_BATCH_NOGROUP", "1")
    shapes = [[8, 6, 3, 3, 2], [12, 6, 8, 8, 2, 2], [4, 4, 3, 3, 3, 3, 4, 4, 2, 2],
              [31, 11, 4, 2, 3], [6, 5, 4, 3, 2, 2, 2], [7, 1, 5], [2, 2]]
    tables = []
    for k, radix in enumerate(shapes * 2):
        fit, ok = O.gen_synthetic(radix, 0.1 * (k % 5), "rugged", k)
        tables.append((radix, np.ascontiguousarray(fit, np.float64),
                       np.ascontiguousarray(ok, np.uint8)))
    refs = [O.analyze(radix, fit, ok, kind, node_limit=1 << 32) for radix, fit, ok in tables]
    bufs = [[np.empty(max(1, len(r["ffg"]["minima"])), dt) for dt in (np.uint64, np.float64,
                                                                    np.float64, np.float64)]
            for r in refs]
    items = [(radix, f.ctypes.data, o.ctypes.data) for radix, f, o in tables]
    with tk.BatchAnalyzer(workers=4) as batch:
        got = batch.run(items, kind, [tuple(b.ctypes.data for b in bb) for bb in bufs],
                        node_limit=1 << 32)
    for (radix, fit, ok), s, ref, bb in zip(tables, got, refs, bufs):
        g = ref["ffg"]
        mins = g["minima"]
        assert s.iterations == ref["iterations"], radix
        assert s.n_edges == len(g["targets"]) and s.n_minima == len(mins)
        assert s.f_opt == fit[ok.astype(bool)].min()
        for k, c in ref["c_p_curve"]:
            assert abs(s.c_p[k] - c) <= CP_ATOL
        ranks, fmin, frac, prm = (b[: len(mins)] for b in bb)
        assert np.array_equal(ranks, mins.astype(np.uint64))
        assert np.array_equal(fmin.view(np.uint64), fit[mins].view(np.uint64))
        assert np.array_equal(frac, fit[ok.astype(bool)].min() / fit[mins])
        assert np.max(np.abs(prm - ref["pagerank"][mins]), initial=0.0) <= 1e-12


def test_batch_analyze_statuses(tk):
    """Per-item statuses of the batched path: a space whose configurations all
    failed raises NoFeasiblePoint (errors.hpp:32-35), like analyze_landscape."""
    radix = [4, 3]
    fit = np.full(12, 1e10)
    ok = np.zeros(12, np.uint8)
    with tk.BatchAnalyzer() as batch:
        with pytest.raises(tk.NoFeasiblePoint):
            batch.run([(radix, fit.ctypes.data, ok.ctypes.data)], O.ADJACENT)


@pytest.mark.slow
def test_c5_full_size_parity(tk):
    """BASELINE C5 at its full size (113,246,208 configurations, 1.02e9 edges):
    the device-generated table, the FFG CSR and minima bit-exact against the
    oracle, PageRank with the same iteration count and within 1e-12 relative
    L1, and the C_p curve within 1e-9 -- the bench workload itself."""
    import os

    radix = [8, 8, 8, 6, 6, 6, 4, 4, 4, 4, 2, 2]
    threads = os.cpu_count() or 8
    with tk.Landscape(radix) as land:
        land.generate(0, 0.10, 5)
        s = land.analyze(tk.ADJACENT, node_limit=1 << 32, emit_csr=True)
        off, tg, sk, mn = land.ffg_arrays()
        r = land.pagerank_vector()
        fit, ok = land.fitness()
    assert (s.n_edges, s.n_minima, s.iterations) == (1023020492, 5917841, 29)
    rf, ro = O.gen_iid(O.space_size(radix), 0.10, 5, nthreads=threads)
    assert np.array_equal(fit.view(np.uint64), rf.view(np.uint64)) and np.array_equal(ok, ro)
    del rf, ro
    ref = O.analyze(radix, fit, ok, O.ADJACENT, nthreads=threads, node_limit=1 << 32)
    g = ref["ffg"]
    assert np.array_equal(off, g["offsets"]) and np.array_equal(tg, g["targets"])
    assert np.array_equal(sk, g["is_sink"]) and np.array_equal(mn, g["minima"])
    assert s.iterations == ref["iterations"]
    assert rel_l1(r, ref["pagerank"]) <= PR_RTOL
    for k, c in ref["c_p_curve"]:
        assert abs(s.c_p[k] - c) <= CP_ATOL


def test_c4_bench_workload_matches_oracle(tk):
    """The C4 bench workload itself (bench.c4_landscapes: 4 paper shapes + 22
    seeded shapes x 9 seeds, 234 landscapes) through tk.BatchAnalyzer, against
    the oracle: iterations, edge and minima counts exact, C_p curve within 1e-9,
    report rows (minima ranks and fitness bit-exact, fraction of optimum exact,
    PageRank of each minimum within 1e-12 of the oracle's)."""
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    tables = []
    for _name, radix, q, seed in bench.c4_landscapes():
        fit, ok = O.gen_synthetic(list(radix), q, "rugged", seed)
        tables.append((list(radix), np.ascontiguousarray(fit, np.float64),
                       np.ascontiguousarray(ok, np.uint8)))
    refs = [O.analyze(radix, fit, ok, O.ADJACENT, node_limit=1 << 32) for radix, fit, ok in tables]
    bufs = [[np.empty(max(1, len(r["ffg"]["minima"])), dt)
             for dt in (np.uint64, np.float64, np.float64, np.float64)] for r in refs]
    items = [(radix, f.ctypes.data, o.ctypes.data) for radix, f, o in tables]
    with tk.BatchAnalyzer(workers=8) as batch:
        got = batch.run(items, tk.ADJACENT, [tuple(b.ctypes.data for b in bb) for bb in bufs],
                        node_limit=1 << 32)
    assert len(got) == 234
    for (radix, fit, ok), s, ref, bb in zip(tables, got, refs, bufs):
        g = ref["ffg"]
        mins = g["minima"]
        assert s.iterations == ref["iterations"], radix
        assert s.n_edges == len(g["targets"]) and s.n_minima == len(mins)
        for k, c in ref["c_p_curve"]:
            assert abs(s.c_p[k] - c) <= CP_ATOL
        ranks, fmin, frac, prm = (b[: len(mins)] for b in bb)
        f_opt = fit[ok.astype(bool)].min()
        assert np.array_equal(ranks, mins.astype(np.uint64))
        assert np.array_equal(fmin.view(np.uint64), fit[mins].view(np.uint64))
        assert np.array_equal(frac, f_opt / fit[mins])
        assert np.max(np.abs(prm - ref["pagerank"][mins]), initial=0.0) <= 1e-12


# Ring PageRank (tk_ring.cu): chunks of consecutive tiles per CTA, a shared-
# memory ring of c for the dims within the ring's reach, far ranges staged.
# Small chunks (TK_RING_CHUNK) make the kernel eligible at test sizes and put
# many chunk boundaries (drain + warm-up) into every sweep.
@pytest.mark.parametrize("chunk", ["2", "3", "4", "16"])
@pytest.mark.parametrize("radix,q", [
    ([8, 8, 6, 6, 4, 4, 4, 2, 2], 0.1),    # C5's lower dims: ring dims 2.., far dims 0-1
    ([16, 12, 8, 8, 8, 4, 2, 2], 0.3),     # C2 shape
    ([6, 10, 8, 6, 4, 4, 4, 2], 0.2),      # ring reach not a power of two
    ([3, 5, 7, 9, 16, 16, 2], 0.15),       # odd radices, far stride 4608 (even)
    ([40, 32, 24, 16], 0.05),              # 4 dims
    ([7, 3, 5, 6, 4, 4, 4, 2, 2, 3], 0.1), # N = 1935360, odd tile count
])
def test_ring_pagerank_matches_oracle(tk, monkeypatch, chunk, radix, q):
    monkeypatch.setenv("TK_RING_CHUNK", chunk)
    monkeypatch.setenv("TK_PR_RING", "1")
    n = O.space_size(radix)
    if (n + 511) // 512 < 148 * int(chunk):
        pytest.skip("fewer tiles than one chunk per SM")
    fit, ok = O.gen_iid(n, q, 41)
    ref = O.analyze(radix, fit, ok, O.ADJACENT, nthreads=8, node_limit=1 << 32)
    with tk.Landscape(radix) as land:
        land.load_dense(fit, ok)
        s = land.analyze(tk.ADJACENT, node_limit=1 << 32)
        r = land.pagerank_vector()
        info = land.kernel_info()
    assert info["pagerank_kernel"] == "ring", info
    assert s.iterations == ref["iterations"]
    assert rel_l1(r, ref["pagerank"]) <= PR_RTOL
    for k, c in ref["c_p_curve"]:
        assert abs(s.c_p[k] - c) <= CP_ATOL


@pytest.mark.parametrize("radix,q", [
    ([8, 6, 3, 3, 2], 0.52),
    ([16, 12, 8, 8, 8, 4, 2, 2], 0.3),     # C2 shape: 49,152 warp slots of look-back
    ([7, 3, 5, 6, 4, 4, 4, 2, 2, 3], 0.1), # N not a multiple of the tile
])
def test_fused_ffg_build_matches_oracle(tk, monkeypatch, radix, q):
    """The one-pass FFG build (TK_FFG_FUSED=1: count, warp-slot decoupled
    look-back and CSR emission in one kernel) is bit-exact against the oracle."""
    monkeypatch.setenv("TK_FFG_FUSED", "1")
    fit, ok = O.gen_synthetic(radix, q, "rugged", 4)
    ref = O.build_ffg(radix, fit, ok, O.ADJACENT, node_limit=1 << 32, nthreads=8)
    with tk.Landscape(radix) as land:
        land.load_dense(fit, ok)
        land.build_ffg(O.ADJACENT, node_limit=1 << 32, emit_csr=True)
        off, tg, sk, mn = land.ffg_arrays()
    assert np.array_equal(off, ref["offsets"]) and np.array_equal(tg, ref["targets"])
    assert np.array_equal(sk, ref["is_sink"]) and np.array_equal(mn, ref["minima"])


def test_batch_analyze_device_inputs_and_long_cp_curve(tk):
    """tk_batch_analyze with device-resident tables (TK_MEM_DEVICE) and a C_p
    curve of 31 points (past the CTA-group kernel's partial width: the one-CTA
    kernel runs), against the oracle."""
    import ctypes as C

    import torch

    from paper_2210_01465_b200 import _abi

    shapes = [[12, 6, 8, 8, 2, 2], [8, 6, 3, 3, 2], [4, 4, 3, 3, 3, 3, 4, 4, 2, 2]]
    tables = [O.gen_synthetic(r, 0.3, "rugged", 11 + k) for k, r in enumerate(shapes)]
    dev = [(torch.from_numpy(np.ascontiguousarray(f)).cuda(), torch.from_numpy(o.astype(np.uint8)).cuda())
           for f, o in tables]
    for p_max in (15, 30):
        arr = (_abi.BatchItem * len(shapes))()
        for k, r in enumerate(shapes):
            arr[k].dims = len(r)
            for i, m in enumerate(r):
                arr[k].radix[i] = m
            arr[k].fitness, arr[k].ok = dev[k][0].data_ptr(), dev[k][1].data_ptr()
        L = _abi.load()
        assert L.tk_batch_analyze(0, arr, len(shapes), O.ADJACENT, 0.85, 1e-10, 100000, p_max,
                                  _abi.TK_MEM_DEVICE) == 0
        for k, r in enumerate(shapes):
            fit, ok = tables[k]
            ref = O.analyze(r, fit, ok, O.ADJACENT, p_max_percent=p_max, node_limit=1 << 32)
            s = arr[k].summary
            assert arr[k].status == 0
            assert s.iterations == ref["iterations"] and s.n_cp == p_max + 1
            assert s.n_minima == len(ref["ffg"]["minima"])
            for kk, c in ref["c_p_curve"]:
                assert abs(s.c_p[kk] - c) <= CP_ATOL
