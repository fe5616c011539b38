"""Valid-set ingestion with constraint-shaped key sets.

Constraints show up in a cache as absent or failed configurations
(/root/reference/proj/src/cache_io.cpp:79-112), so
the valid set is usually skewed: trailing parameters fixed, whole key ranges
missing.  Round 1's hash table probed only inside a key's residue class mod
32 and spun forever on such sets.  Here:

* CPU: a restatement of the device probe sequence (csrc/tk_kernels.cu hprobe)
  inserts skewed key sets into a table of the production capacity and shows
  that every insert and every absent-key lookup terminates;
* GPU: load_sparse / load_configs / lookup / analyze on constraint-shaped
  valid sets against the oracle, and the same through the C++
  analyze_cache_file (tk_analyze --device-ingest).
"""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle as O

M64 = (1 << 64) - 1
EMPTY = M64


def mix64(x):
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def hprobe(key, j, mask):
    """csrc/tk_kernels.cu hprobe, restated."""
    if j < 4:
        return ((((mix64(key >> 5) + j) & M64) << 5) | (key & 31)) & mask
    h1 = mix64(key ^ 0x6A09E667F3BCC909)
    h2 = mix64((key + 0xBB67AE8584CAA73B) & M64) | 1
    return (h1 + (j - 4) * h2) & mask


def capacity(nv):
    cap = 64
    while cap < 2 * nv:
        cap <<= 1
    return cap


def simulate(keys, queries):
    cap = capacity(len(keys))
    mask = cap - 1
    table = [EMPTY] * cap
    worst = 0
    for k in keys:
        for j in range(4 + cap):
            s = hprobe(k, j, mask)
            if table[s] == EMPTY:
                table[s] = k
                worst = max(worst, j + 1)
                break
        else:
            raise AssertionError("insert did not terminate")
    for q in queries:
        for j in range(4 + cap):
            s = hprobe(q, j, mask)
            if table[s] in (q, EMPTY):
                worst = max(worst, j + 1)
                break
        else:
            raise AssertionError("lookup did not terminate")
    return worst


def skewed_sets():
    n = 1 << 14
    r = np.arange(n, dtype=np.uint64)
    return {
        "mod32": r[r % 32 == 0],                       # last five binary params fixed
        "mod4": r[r % 4 == 0],                         # keys = 0 mod 4 (round-1 spin at 2,048)
        "cluster": r[(r >= 3000) & (r < 7000)],        # one contiguous key range
        "radix_1000x32": np.arange(1000, dtype=np.uint64) * 32,  # ADVICE repro
    }


@pytest.mark.parametrize("name", list(skewed_sets()))
def test_probe_sequence_terminates_on_skewed_sets(name):
    keys = [int(k) for k in skewed_sets()[name]]
    absent = [k + 1 for k in keys[:500]] + [k + 32 * 4096 for k in keys[:200]]
    absent = [q for q in absent if q not in set(keys)]
    worst = simulate(keys, absent)
    # double hashing over the whole table at load <= 1/2 keeps chains short
    assert worst < 64, worst


# ------------------------------------------------------------------ GPU --

CASES = {
    # radix, valid predicate over the digit matrix
    "trail5_fixed": ([8, 6, 4, 2, 2, 2, 2, 2], lambda d: (d[:, 3:] == 0).all(1)),
    "mod4": ([16, 12, 8, 4, 2, 2], lambda d: (d[:, 4] == 0) & (d[:, 5] == 0)),
    "one_last_value": ([1000, 32], lambda d: d[:, 1] == 0),
    "clustered": ([16, 16, 16], lambda d: (d[:, 0] >= 3) & (d[:, 0] < 9) & (d[:, 2] % 3 != 1)),
}


def digits(radix):
    n = O.space_size(radix)
    st = O.strides(radix).astype(np.int64)
    r = np.arange(n, dtype=np.int64)
    return np.stack([(r // s) % m for s, m in zip(st, radix)], 1)


def case_table(name, seed=11):
    radix, pred = CASES[name]
    d = digits(radix)
    valid = pred(d)
    n = d.shape[0]
    rng = np.random.default_rng(seed)
    fit = np.full(n, 1e10)
    fit[valid] = 1.0 + rng.random(int(valid.sum()))
    return radix, d, fit, valid.astype(np.uint8)


@pytest.fixture(scope="module")
def tk():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2210_01465_b200 as tk

    tk._abi.load()
    return tk


@pytest.mark.gpu
@pytest.mark.parametrize("ingest", ["direct", "partition"])
@pytest.mark.parametrize("name", list(CASES))
def test_constraint_shaped_load_sparse_configs_lookup(tk, monkeypatch, name, ingest):
    """Both ingest paths: the direct scatter and the slice-partitioned one
    (TK_INGEST_PARTITION=1)."""
    if ingest == "partition":
        monkeypatch.setenv("TK_INGEST_PARTITION", "1")
    radix, d, fit, ok = case_table(name)
    keys = np.flatnonzero(ok).astype(np.uint64)
    perm = np.random.default_rng(1).permutation(keys.size)
    with tk.Landscape(radix) as land:
        land.load_sparse(keys[perm], fit[keys][perm])
        f, o = land.fitness()
        assert np.array_equal(f.view(np.uint64), fit.view(np.uint64))
        assert np.array_equal(o, ok)
        # absent keys inside a crowded residue class, present keys, keys >= N
        absent = np.flatnonzero(ok == 0)[:4096].astype(np.uint64)
        q = np.concatenate([keys[:4096], absent, np.array([len(fit), 2**40], np.uint64)])
        lf, hit = land.lookup(q)
        assert np.array_equal(hit, (q < len(fit)) & (ok[np.minimum(q, len(fit) - 1)] == 1))
        assert np.array_equal(lf[: min(4096, keys.size)], fit[keys[:4096]])
        assert (lf[hit == 0] == 1e10).all()
        land.load_configs(d[keys[perm]].astype(np.int32), fit[keys][perm])
        f2, o2 = land.fitness()
        assert np.array_equal(f2.view(np.uint64), fit.view(np.uint64))
        assert np.array_equal(o2, ok)
        kind = O.ADJACENT
        s = land.analyze(kind, node_limit=1 << 32, p_max_percent=15)
    ref = O.analyze(radix, fit, ok, kind, node_limit=1 << 32)
    assert s.iterations == ref["iterations"]
    assert s.n_minima == len(ref["ffg"]["minima"])
    for k, c in ref["c_p_curve"]:
        assert abs(s.c_p[k] - c) <= 1e-9


@pytest.mark.gpu
def test_load_rejects_failed_range_means(tk):
    """A11: an ok mean >= 1e10 is rejected at upload; failed entries are
    normalised to 1e10 on a dense load (cache.cpp:49-53)."""
    radix = [4, 4]
    with tk.Landscape(radix) as land:
        with pytest.raises(tk.InvalidArgument):
            land.load_sparse(np.array([1, 2], np.uint64), np.array([1.0, 1e10]))
        fit = np.linspace(1, 2, 16)
        ok = np.ones(16, np.uint8)
        ok[3] = 0
        land.load_dense(fit, ok)
        f, _ = land.fitness()
        assert f[3] == 1e10 and f[4] == fit[4]
        fit[5] = 2e10
        with pytest.raises(tk.InvalidArgument):
            land.load_dense(fit, ok)


def write_kt_cache(path, radix, fit, ok):
    """A Kernel Tuner style cache: numeric tune_params ascending, only the
    valid configurations present (constraints -> absent entries)."""
    values = [[(i + 1) * 8 for i in range(m)] for m in radix]
    keys = [f"p{i}" for i in range(len(radix))]
    d = digits(radix)
    cache = {}
    for r in np.flatnonzero(ok):
        cache[",".join(str(values[i][d[r, i]]) for i in range(len(radix)))] = {"time": float(fit[r])}
    json.dump({"kernel_name": "constrained", "device_name": "B200", "tune_params_keys": keys,
               "tune_params": dict(zip(keys, values)), "cache": cache}, open(path, "w"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["trail5_fixed", "mod4"])
def test_analyze_cache_file_constraint_shaped(tk, tmp_path, name):
    from paper_2210_01465_b200 import build

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    build.build()
    subprocess.run(["make", "-s", "-C", os.path.join(root, "cpp")], check=True)
    radix, _, fit, ok = case_table(name)
    path = str(tmp_path / "cache.json")
    write_kt_cache(path, radix, fit, ok)
    rep_path = str(tmp_path / "rep.json")
    r = subprocess.run([os.path.join(root, "cpp", "build", "tk_analyze"), path, "--json", rep_path,
                        "--device-ingest", "--node-limit", str(1 << 32)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rep = json.load(open(rep_path))
    ref = O.analyze(radix, fit, ok, O.ADJACENT, node_limit=1 << 32)
    assert rep["pagerank_iterations"] == ref["iterations"]
    assert [m["rank"] for m in rep["minima"]] == [int(x) for x in ref["ffg"]["minima"]]
    for e, (k, c) in zip(rep["c_p_curve"], ref["c_p_curve"]):
        assert e["p_percent"] == k and abs(e["c_p"] - c) <= 1e-9
