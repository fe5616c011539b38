"""SPEC.md:583 acceptance 4 / SPEC.md:430 property: on 20 synthetic spaces of
<= 4096 points, the arrival frequencies of 10^4 randomized first-improvement
descents correlate with PageRank over the minima (Spearman rho >= 0.9).

A randomized first-improvement step (the reference's climb_random_first,
src/hillclimb.cpp:48-87, scanning the neighbour slots in a fresh uniform
permutation) lands on a uniformly random strictly-better neighbour, i.e. one
step of a random walk on the FFG; the descent ends in a sink.  The walks are
vectorised over the 10^4 walkers.  The CPU variant checks the oracle's
PageRank; the GPU variant the CUDA path.
"""
import numpy as np
import pytest

import oracle as O

scipy_stats = pytest.importorskip("scipy.stats")


def spaces():
    rng = np.random.default_rng(2022)
    out = []
    while len(out) < 20:
        dims = int(rng.integers(2, 6))
        radix = [int(x) for x in rng.integers(2, 9, size=dims)]
        n = O.space_size(radix)
        if 256 <= n <= 4096:
            out.append((radix, float(rng.uniform(0.0, 0.4)), ["smooth", "ridged", "rugged"][len(out) % 3],
                        len(out)))
    return out


def descent_frequencies(offsets, targets, n, walkers=10_000, seed=0):
    rng = np.random.default_rng(seed)
    pos = rng.integers(0, n, size=walkers)  # uniform starts
    deg = np.diff(offsets).astype(np.int64)
    while True:
        moving = deg[pos] > 0
        if not moving.any():
            break
        p = pos[moving]
        pick = offsets[p].astype(np.int64) + (rng.random(p.size) * deg[p]).astype(np.int64)
        pos[moving] = targets[pick]
    return np.bincount(pos, minlength=n)


def rho(radix, q, prof, seed, kind, pagerank_fn):
    fit, ok = O.gen_synthetic(radix, q, prof, seed)
    g = O.build_ffg(radix, fit, ok, kind)
    pr = pagerank_fn(g)
    freq = descent_frequencies(g["offsets"], g["targets"], len(fit), seed=seed)
    mins = g["minima"]
    if len(mins) < 5:
        return None  # rank correlation needs a handful of minima
    return scipy_stats.spearmanr(freq[mins], pr[mins]).correlation


@pytest.mark.parametrize("kind", [O.ADJACENT, O.HAMMING])
def test_descents_track_pagerank_oracle(kind):
    rs = [rho(*s, kind, lambda g: O.pagerank(g["offsets"], g["targets"])[0]) for s in spaces()]
    rs = [r for r in rs if r is not None]
    assert len(rs) >= 10
    assert min(rs) >= 0.9 - 1e-12, rs  # rho is discrete; 0.9 exactly with 5 minima


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [O.ADJACENT, O.HAMMING])
def test_descents_track_pagerank_gpu(kind):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2210_01465_b200 as tk

    def gpu_pr(g):
        fg = tk.FitnessFlowGraph(kind, len(g["is_sink"]), g["offsets"], g["targets"], None,
                                 g["is_sink"], g["minima"])
        return tk.pagerank(fg)

    rs = [rho(*s, kind, gpu_pr) for s in spaces()]
    rs = [r for r in rs if r is not None]
    assert len(rs) >= 10 and min(rs) >= 0.9 - 1e-12, rs
