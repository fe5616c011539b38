"""The GPU random-walk validator (tk_descents).

Batched randomized first-improvement descents -- the reference's
climb_random_first (/root/reference/proj/src/hillclimb.cpp:48-87) -- one
walker per device thread.  Parity: the oracle restates the same descent with
the same per-walker draws (oracle.c or_descents), so the arrival counts are
bit-identical.  Property (acceptance 4 at scale): the arrival
frequencies at the minima track PageRank restricted to the minima (Spearman
rho >= 0.9), checked here on C2- and C3-sized spaces instead of <= 4096 points.
"""
import numpy as np
import pytest

import oracle as O

CASES = [  # radix, generator, fail fraction, seed
    ([8, 6, 3, 3, 2], "rugged", 0.52, 0),
    ([12, 6, 8, 8, 2, 2], "ridged", 0.68, 1),
    ([5, 1, 4, 3, 1, 7], "smooth", 0.2, 2),  # radix-1 dimensions carry no slots
    ([31, 11, 4, 2, 3], "rugged", 0.04, 3),
    ([2, 2, 2, 2, 2, 2, 2, 2, 2, 2], "rugged", 0.3, 4),
]


def test_oracle_descents_end_in_sinks():
    """Every descent ends at an FFG sink (no strictly better neighbour); the
    draws are a function of (seed, walker) only."""
    for radix, prof, q, seed in CASES:
        fit, ok = O.gen_synthetic(radix, q, prof, seed)
        for kind in (O.ADJACENT, O.HAMMING):
            g = O.build_ffg(radix, fit, ok, kind)
            deg = np.diff(g["offsets"])
            for restart in (True, False):
                c, ev = O.descents(radix, fit, kind, 5000, 11, restart)
                assert c.sum() == 5000 and ev > 0
                assert np.all(deg[c > 0] == 0)
                c2, ev2 = O.descents(radix, fit, kind, 5000, 11, restart, nthreads=1)
                assert np.array_equal(c, c2) and ev == ev2


def test_oracle_descents_no_slots():
    c, ev = O.descents([1, 1], np.array([3.0]), O.ADJACENT, 10, 0)
    assert c.tolist() == [10] and ev == 0


def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2210_01465_b200 as tk

    return tk


@pytest.mark.gpu
@pytest.mark.parametrize("restart", [True, False])
@pytest.mark.parametrize("kind", [O.ADJACENT, O.HAMMING])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_descents_match_oracle(case, kind, restart):
    tk = _gpu()
    radix, prof, q, seed = CASES[case]
    fit, ok = O.gen_synthetic(radix, q, prof, seed)
    g = O.build_ffg(radix, fit, ok, kind)
    walkers = 200_003
    counts, ev = O.descents(radix, fit, kind, walkers, 97 + case, restart)
    with tk.Landscape(radix, device=0) as land:
        land.load_dense(fit, ok)
        land.build_ffg(kind, emit_csr=False)
        arr, fail, gev = land.descents(walkers, 97 + case, restart)
    mins = g["minima"]
    assert np.array_equal(arr, counts[mins].astype(np.uint64))
    assert fail == walkers - int(counts[mins].sum())
    assert gev == ev


@pytest.mark.gpu
def test_descents_need_a_build():
    tk = _gpu()
    radix = [4, 4]
    fit, ok = O.gen_synthetic(radix, 0.0, "rugged", 0)
    with tk.Landscape(radix, device=0) as land:
        land.load_dense(fit, ok)
        with pytest.raises(tk.Error):
            land.descents(10)


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["c2", "c3"])
@pytest.mark.parametrize("kind", [O.ADJACENT, O.HAMMING])
def test_descents_track_pagerank_at_scale(workload, kind):
    """SPEC.md:430 at C2 size (1.57M configs, generate_synthetic_kernel_space
    'rugged', 30 % failed) and C3 size (9.4M configs, heavy-tailed G_heavy):
    Spearman rho between device descent arrivals and device PageRank over the
    minima >= 0.9."""
    tk = _gpu()
    scipy_stats = pytest.importorskip("scipy.stats")
    if workload == "c2":
        radix = [16, 12, 8, 8, 8, 4, 2, 2]
        fit, ok = O.gen_synthetic(radix, 0.30, "rugged", 2)
    else:
        radix = [8, 8, 8, 8, 6, 6, 4, 4, 2, 2]
        fit, ok = O.gen_heavy(O.space_size(radix), 0.0, 3)
    n = len(fit)
    with tk.Landscape(radix, device=0) as land:
        land.load_dense(fit, ok)
        land.build_ffg(kind, node_limit=1 << 32, emit_csr=False)
        land.pagerank()
        r = land.pagerank_vector()
        mins = land.minima()
        arr, fail, ev = land.descents(8 * n, 5)
    assert int(arr.sum()) + fail == 8 * n
    rho = scipy_stats.spearmanr(arr, r[mins]).correlation
    assert rho >= 0.9, (workload, kind, len(mins), rho)
