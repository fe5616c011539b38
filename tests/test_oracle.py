"""Pin the CPU oracle (oracle/oracle.c) before trusting it as the checker.

* against the golden fixtures generated from the reference's own compiled code
  (tests/golden/make_golden.py, oracle/_ref): neighbour order, strides,
  synthetic caches, f_opt, FFG CSR + minima;
* against the SPEC.md known answers for the landscape module;
* PageRank against networkx (independent implementation, same semantics);
* property suites from SPEC.md:428-432 and acceptance criteria 1 and 5
  (SPEC.md:580,584).
"""
import hashlib

import numpy as np
import pytest

import oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------ golden: space --

def test_neighbour_lists_match_reference(golden):
    meta, arrays = golden
    for rec in meta["neighbours"]:
        radix = rec["radix"]
        assert O.space_size(radix) == rec["size"]
        assert [int(x) for x in O.strides(radix)] == rec["strides"]
        cnt = np.zeros(rec["size"], np.uint32)
        parts = []
        for u in range(rec["size"]):
            nb = O.neighbour_ranks(radix, u, rec["kind"])
            cnt[u] = len(nb)
            parts.append(nb)
        ranks = np.concatenate(parts) if parts else np.zeros(0, np.uint64)
        assert sha(cnt) == rec["sha_counts"], rec["key"]
        assert sha(ranks) == rec["sha_ranks"], rec["key"]
        if rec["key"] + "_ranks" in arrays:
            assert np.array_equal(arrays[rec["key"] + "_ranks"], ranks)


def test_synthetic_generator_matches_reference(golden):
    meta, arrays = golden
    for rec in meta["synthetic"]:
        fit, ok = O.gen_synthetic(rec["radix"], rec["q"], rec["profile"], rec["seed"])
        assert sha(fit) == rec["sha_fit"], rec["key"]
        assert sha(ok) == rec["sha_ok"], rec["key"]
        if rec["status"] == 0:
            f_opt, r = O.optimum(fit, ok)
            assert f_opt == rec["f_opt"] and r == rec["opt_rank"]
        else:
            with pytest.raises(O.OracleError):
                O.optimum(fit, ok)


@pytest.mark.parametrize("kind", [O.HAMMING, O.ADJACENT])
def test_ffg_matches_reference_loop(golden, kind):
    meta, arrays = golden
    for rec in meta["synthetic"]:
        fit, ok = O.gen_synthetic(rec["radix"], rec["q"], rec["profile"], rec["seed"])
        g = O.build_ffg(rec["radix"], fit, ok, kind, nthreads=2)
        ref = rec["ffg"][str(kind)]
        assert len(g["targets"]) == ref["edges"], rec["key"]
        assert len(g["minima"]) == ref["minima"], rec["key"]
        assert sha(g["offsets"]) == ref["sha_offsets"], rec["key"]
        assert sha(g["targets"]) == ref["sha_targets"], rec["key"]
        assert sha(g["is_sink"]) == ref["sha_is_sink"], rec["key"]
        assert sha(g["minima"]) == ref["sha_minima"], rec["key"]


# ------------------------------------------------ SPEC known answers (PR/C_p) --

def test_spec_two_point_edge():
    # 2-point space, f = (1, 2) -> single edge 2nd -> 1st
    g = O.build_ffg([2], np.array([1.0, 2.0]), np.array([1, 1], np.uint8), O.ADJACENT)
    assert list(g["offsets"]) == [0, 0, 1] and list(g["targets"]) == [0]
    assert list(g["minima"]) == [0]


@pytest.mark.parametrize("m", [1, 2, 7, 64])
def test_spec_monotone_path(m):
    # monotone 1-D space: m-1 downhill edges, one minimum
    fit = np.arange(m, dtype=np.float64) + 1.0
    ok = np.ones(m, np.uint8)
    g = O.build_ffg([m], fit, ok, O.ADJACENT)
    assert len(g["targets"]) == m - 1
    assert all(g["targets"][u - 1] == u - 1 for u in range(1, m))
    assert list(g["minima"]) == [0]
    c = O.census([m], fit, ok, O.ADJACENT)
    assert c["local_minima"] == 1


def test_spec_constant_space_census():
    # constant fitness: 0 census minima (strict), every node is an
    # FFG sink (no edges on ties) so the FFG minima are all ok nodes
    fit = np.full(24, 3.0)
    ok = np.ones(24, np.uint8)
    c = O.census([2, 3, 4], fit, ok, O.HAMMING)
    assert c["local_minima"] == 0 and c["interior"] == 24
    g = O.build_ffg([2, 3, 4], fit, ok, O.HAMMING)
    assert len(g["targets"]) == 0 and len(g["minima"]) == 24


def test_spec_single_node_pagerank():
    # SPEC.md:403
    r, it, res = O.pagerank(np.array([0, 0], np.uint64), np.zeros(0, np.uint32))
    assert r[0] == 1.0


def test_spec_two_node_d1():
    # a -> b, d = 1.0: (1/3, 2/3)
    r, it, res = O.pagerank(np.array([0, 1, 1], np.uint64), np.array([1], np.uint32),
                            damping=1.0, tol=1e-15)
    assert abs(r[0] - 1 / 3) < 1e-14 and abs(r[1] - 2 / 3) < 1e-14


def test_spec_symmetric_nodes_equal_rank():
    # star: centre -> 4 leaves; leaves symmetric
    off = np.array([0, 4, 4, 4, 4, 4], np.uint64)
    r, _, _ = O.pagerank(off, np.array([1, 2, 3, 4], np.uint32))
    assert np.ptp(r[1:]) == 0.0


def test_spec_cp_examples():
    # C_0 covers exactly the global minima; large p -> 1
    fit, ok = O.gen_synthetic([8, 6, 3, 3, 2], 0.3, "rugged", 4)
    res = O.analyze([8, 6, 3, 3, 2], fit, ok, O.ADJACENT, p_max_percent=15)
    g, pr, f_opt = res["ffg"], res["pagerank"], res["f_opt"]
    glob = [m for m in g["minima"] if fit[m] == f_opt]
    assert res["c_p_curve"][0][1] == pytest.approx(pr[glob].sum() / pr[g["minima"]].sum(),
                                                   abs=1e-15)
    assert O.proportion_of_centrality(g["minima"], fit, pr, f_opt, 10.0) == 1.0


def test_pagerank_nonconvergence_and_args():
    off = np.array([0, 1, 1], np.uint64)
    tg = np.array([1], np.uint32)
    with pytest.raises(O.OracleError) as e:
        O.pagerank(off, tg, max_iter=3)
    assert e.value.status == O.ENOCONV
    for bad in (dict(damping=1.5), dict(damping=-0.1), dict(tol=0.0), dict(max_iter=0)):
        with pytest.raises(O.OracleError) as e:
            O.pagerank(off, tg, **bad)
        assert e.value.status == O.EINVAL


def test_node_limit():
    fit, ok = O.gen_iid(4096, 0.0, 1)
    with pytest.raises(O.OracleError) as e:
        O.build_ffg([64, 64], fit, ok, O.ADJACENT, node_limit=4095)
    assert e.value.status == O.ELIMIT


# ------------------------------------------------------ networkx cross-check --

@pytest.mark.parametrize("kind", [O.HAMMING, O.ADJACENT])
def test_pagerank_matches_networkx(kind):
    nx = pytest.importorskip("networkx")
    radix = [6, 5, 4, 3]
    fit, ok = O.gen_synthetic(radix, 0.25, "rugged", 9)
    g = O.build_ffg(radix, fit, ok, kind)
    n = len(fit)
    r, it, res = O.pagerank(g["offsets"], g["targets"], tol=1e-14)
    G = nx.DiGraph()
    G.add_nodes_from(range(n))
    for u in range(n):
        for v in g["targets"][g["offsets"][u]:g["offsets"][u + 1]]:
            G.add_edge(u, int(v))
    ref = nx.pagerank(G, alpha=0.85, tol=1e-15, max_iter=10000)
    ref = np.array([ref[i] for i in range(n)])
    assert np.abs(r - ref).sum() / np.abs(ref).sum() < 1e-12


# ----------------------------------------------------------------- properties --

def _topo_ok(n, off, tg):
    indeg = np.bincount(tg.astype(np.int64), minlength=n)
    stack = [u for u in range(n) if indeg[u] == 0]
    seen = 0
    while stack:
        u = stack.pop()
        seen += 1
        for v in tg[off[u]:off[u + 1]]:
            indeg[v] -= 1
            if indeg[v] == 0:
                stack.append(int(v))
    return seen == n


@pytest.mark.parametrize("seed", range(4))
def test_properties(seed):
    # SPEC.md:428-432, acceptance 5
    radix = [5, 4, 3, 3]
    fit, ok = O.gen_synthetic(radix, 0.3, "rugged", seed)
    for kind in (O.HAMMING, O.ADJACENT):
        res = O.analyze(radix, fit, ok, kind)
        g = res["ffg"]
        assert _topo_ok(len(fit), g["offsets"], g["targets"])
        assert abs(res["pagerank_sum"] - 1.0) < 1e-9
        cps = [c for _, c in res["c_p_curve"]]
        assert all(0.0 <= c <= 1.0 for c in cps)
        assert all(a <= b for a, b in zip(cps, cps[1:]))
        # positive rescaling preserves edges, minima and C_p
        res2 = O.analyze(radix, np.where(ok == 1, fit * 3.5, fit), ok, kind)
        if np.all(fit[ok == 1] * 3.5 < 1e10):
            assert np.array_equal(res2["ffg"]["targets"], g["targets"])
            assert np.allclose([c for _, c in res2["c_p_curve"]], cps, atol=1e-12)


def test_pagerank_relabel_invariance():
    radix = [4, 4, 3]
    fit, ok = O.gen_synthetic(radix, 0.2, "rugged", 3)
    g = O.build_ffg(radix, fit, ok, O.HAMMING)
    n = len(fit)
    r, _, _ = O.pagerank(g["offsets"], g["targets"], tol=1e-14)
    perm = np.random.default_rng(0).permutation(n)  # new label of old node u
    inv = np.argsort(perm)
    off, tg = [0], []
    for new in range(n):
        u = inv[new]
        row = perm[g["targets"][g["offsets"][u]:g["offsets"][u + 1]]]
        tg.extend(row)
        off.append(len(tg))
    r2, _, _ = O.pagerank(np.array(off, np.uint64), np.array(tg, np.uint32), tol=1e-14)
    assert np.abs(r2[perm] - r).sum() < 1e-12


def test_edge_count_formula():
    # E = (1 - q^2) * sum_i N (m_i - 1) / m_i   (Adjacent, tie-free)
    radix = [8, 6, 4, 4, 2]
    n = O.space_size(radix)
    fit, ok = O.gen_iid(n, 0.0, 5)
    g = O.build_ffg(radix, fit, ok, O.ADJACENT)
    assert len(g["targets"]) == sum(n * (m - 1) // m for m in radix)
    g = O.build_ffg(radix, fit, ok, O.HAMMING)
    assert len(g["targets"]) == sum(n * (m - 1) // 2 for m in radix)


def _census_bruteforce(radix, fit, ok, kind):
    shape = tuple(radix)
    F = fit.reshape(shape)
    okr = ok.reshape(shape).astype(bool)
    strict = okr.copy()
    for i, m in enumerate(shape):
        for delta in range(1, m):
            if kind == O.ADJACENT and delta > 1:
                break
            for sgn in (1, -1):
                sh = np.roll(F, -sgn * delta, axis=i)
                idx = np.arange(m)
                valid = (idx + sgn * delta >= 0) & (idx + sgn * delta < m)
                vshape = [1] * len(shape)
                vshape[i] = m
                valid = valid.reshape(vshape)
                strict &= ~(valid & ~(sh > F))
    return np.flatnonzero(strict.ravel())


def test_census_matches_bruteforce_50_caches():
    # SPEC.md:580 acceptance 1: 50 seeded caches <= 4096 points, 0 mismatches
    rng = np.random.default_rng(7)
    for s in range(50):
        dims = int(rng.integers(1, 6))
        radix = [int(x) for x in rng.integers(1, 8, size=dims)]
        while O.space_size(radix) > 4096:
            radix[int(np.argmax(radix))] -= 1
        prof = ["smooth", "ridged", "rugged"][s % 3]
        fit, ok = O.gen_synthetic(radix, float(rng.uniform(0, 0.6)), prof, s)
        if s % 5 == 0:  # inject ties
            fit = np.where(ok == 1, np.round(fit, 1), fit)
        for kind in (O.HAMMING, O.ADJACENT):
            c = O.census(radix, fit, ok, kind)
            bf = _census_bruteforce(radix, fit, ok, kind)
            assert np.array_equal(c["minima_ranks"], bf), (s, radix, kind)
            assert c["fail_points"] == int((ok == 0).sum())
