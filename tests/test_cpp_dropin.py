"""The C++ drop-in (cpp/src/landscape*.cpp over the C-ABI, built against the
reference's own headers and host classes -- cpp/Makefile).

CPU: the drop-in library defines the landscape.hpp surface and links the
reference's host classes instead of carrying copies of them; the reference's
cache writer round-trips through the oracle's generator.
GPU: cpp/build/test_dropin drives every landscape.hpp entry point; its dumps --
FFG, PageRank, C_p, census, report JSON, minima / C_p-curve CSVs,
minima_fraction_report and the three export_graph formats -- are compared with
the CPU oracle.
"""
import hashlib
import os
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "cpp")
BUILD = os.path.join(CPP, "build")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def built():
    from paper_2210_01465_b200 import build

    build.build()
    subprocess.run(["make", "-s", "-C", CPP], check=True)
    return BUILD


def dump(built, *args):
    return subprocess.run([os.path.join(built, "tk_gen_dump"), *map(str, args)],
                          capture_output=True, check=True).stdout


def test_dropin_links_the_reference_host_classes(built):
    """The drop-in ships only the landscape implementation: the host classes it
    takes as arguments come from the reference's own sources (cpp/Makefile
    compiles proj/src/*.cpp where they lie into libtunekit_ref.so)."""
    lib = os.path.join(built, "libtunekit_b200.so")
    ref = os.path.join(built, "libtunekit_ref.so")
    if not (os.path.exists(lib) and os.path.exists(ref)):
        pytest.skip("C++ drop-in not built on this host (needs /root/reference)")
    defined = lambda p: subprocess.run(["nm", "-DC", "--defined-only", p], capture_output=True,  # noqa: E731
                                       text=True).stdout
    mine, theirs = defined(lib), defined(ref)
    for sym in ("tunekit::build_ffg", "tunekit::pagerank", "tunekit::analyze_landscape",
                "tunekit::proportion_of_centrality", "tunekit::classify_points",
                "tunekit::minima_fraction_report", "tunekit::export_graph",
                "tunekit::write_minima_csv", "tunekit::write_cp_curve_csv",
                "tunekit::random_descents", "tunekit::analyze_landscapes"):
        assert sym in mine, sym
    for sym in ("tunekit::ParameterSpace::rank_of", "tunekit::SearchSpaceCache::finalize",
                "tunekit::generate_synthetic_kernel_space", "tunekit::load_cache"):
        assert sym in theirs and sym not in mine, sym
    needed = subprocess.run(["readelf", "-d", lib], capture_output=True, text=True).stdout
    assert "libtunekit_ref.so" in needed and "libtk_landscape.so" in needed


def _num(v):
    """landscape_io.cpp num(): shortest round-trip decimal (std::to_chars)."""
    return float(v)


def _colour(fraction, global_min):
    """Fig. 6 colouring (landscape.hpp:98-100): green global
    minimum, one flood colour below 0.75, red -> blue over [0.75, 1)."""
    if global_min:
        return "#00a000"
    if not fraction >= 0.75:
        return "#c8c8c8"
    t = (fraction - 0.75) / 0.25
    rnd = lambda x: int(np.floor(x + 0.5))  # noqa: E731  (std::lround, x >= 0)
    return "#%02x30%02x" % (rnd(220.0 * (1.0 - t)), rnd(220.0 * t))


def _check_graph_exports(tmp_path, fit, ok, g):
    """DOT / GraphML / EdgeCsv of export_graph (landscape.hpp:96-102) against
    the oracle's CSR, minima and fractions of optimum."""
    import xml.etree.ElementTree as ET

    off, tg, mins = g["offsets"], g["targets"], g["minima"]
    n = len(off) - 1
    f_opt = fit[ok.astype(bool)].min()
    is_min = np.zeros(n, bool)
    is_min[mins] = True
    frac = f_opt / fit
    edges = [(u, int(t)) for u in range(n) for t in tg[off[u]:off[u + 1]]]
    # EdgeCsv: header + one line per edge, CSR order
    lines = open(os.path.join(tmp_path, "graph.csv")).read().splitlines()
    assert lines[0] == "source,target"
    assert [tuple(map(int, ln.split(","))) for ln in lines[1:]] == edges
    # GraphML: node data and edge list
    root = ET.parse(os.path.join(tmp_path, "graph.graphml")).getroot()
    ns = {"g": "http://graphml.graphdrawing.org/xmlns"}
    nodes = root.findall("g:graph/g:node", ns)
    assert [nd.get("id") for nd in nodes] == [f"n{u}" for u in range(n)]
    for u, nd in enumerate(nodes):
        d = {e.get("key"): e.text for e in nd.findall("g:data", ns)}
        assert _num(d["fitness"]) == fit[u]
        assert _num(d["fraction"]) == frac[u]
        assert d["minimum"] == ("true" if is_min[u] else "false")
        assert d["colour"] == _colour(frac[u], is_min[u] and fit[u] == f_opt)
        assert d["size"] == ("3" if is_min[u] else "1")
    got = [(int(e.get("source")[1:]), int(e.get("target")[1:]))
           for e in root.findall("g:graph/g:edge", ns)]
    assert got == edges
    # DOT: node attributes and edges
    dot = open(os.path.join(tmp_path, "graph.dot")).read().splitlines()
    assert dot[0] == "digraph ffg {" and dot[-1] == "}"
    node_lines = [ln for ln in dot if "[fillcolor=" in ln]
    assert len(node_lines) == n
    for u, ln in enumerate(node_lines):
        assert ln.strip().startswith(f"{u} [")
        assert f'fillcolor="{_colour(frac[u], is_min[u] and fit[u] == f_opt)}"' in ln
        assert f"width={'0.5' if is_min[u] else '0.2'}" in ln
        assert _num(ln.split('tooltip="f=')[1].split('"')[0]) == fit[u]
    got = [tuple(map(int, ln.strip().rstrip(";").split(" -> "))) for ln in dot if " -> " in ln]
    assert got == edges


@pytest.mark.gpu
def test_dropin_on_gpu_matches_oracle(built, tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    path = os.path.join(built, "test_dropin")
    if not os.path.exists(path):
        pytest.skip("test_dropin not built on this host")
    radix, q, prof, seed = [8, 6, 3, 3, 2], 0.52, "rugged", 5
    r = subprocess.run([path, str(tmp_path), str(q), prof, str(seed), *map(str, radix)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
    fit, ok = O.gen_synthetic(radix, q, prof, seed)
    for kind, name in ((O.HAMMING, "hamming"), (O.ADJACENT, "adjacent")):
        ref = O.analyze(radix, fit, ok, kind)
        g = ref["ffg"]
        rd = lambda f, dt: np.fromfile(os.path.join(tmp_path, f), dt)  # noqa: E731
        assert np.array_equal(rd(f"ffg_{name}_offsets.bin", np.uint64), g["offsets"])
        assert np.array_equal(rd(f"ffg_{name}_targets.bin", np.uint32), g["targets"])
        assert np.array_equal(rd(f"ffg_{name}_is_sink.bin", np.uint8), g["is_sink"])
        assert np.array_equal(rd(f"ffg_{name}_minima.bin", np.uint32), g["minima"])
        pr = rd(f"pr_{name}.bin", np.float64)
        assert np.abs(pr - ref["pagerank"]).sum() <= 1e-12
        for line, (k, c) in zip(open(os.path.join(tmp_path, f"cp_{name}.txt")),
                                ref["c_p_curve"]):
            kk, v = line.split()
            assert int(kk) == k and abs(float.fromhex(v) - c) <= 1e-9
        import json

        rep = json.load(open(os.path.join(tmp_path, f"report_{name}.json")))
        assert rep["pagerank_iterations"] == ref["iterations"]
        assert [m["rank"] for m in rep["minima"]] == [int(x) for x in g["minima"]]
        cen = O.census(radix, fit, ok, kind)
        t, fp, lm, it = map(int, open(os.path.join(tmp_path, f"census_{name}.txt")).read().split())
        assert (fp, lm, it) == (cen["fail_points"], cen["local_minima"], cen["interior"])
        assert np.array_equal(rd(f"census_{name}_ranks.bin", np.uint64), cen["minima_ranks"])
        # write_minima_csv (landscape.hpp:83-84): one row per FFG minimum, rank order
        f_opt = fit[ok.astype(bool)].min()
        pr_ref = ref["pagerank"]
        lines = open(os.path.join(tmp_path, f"minima_{name}.csv")).read().splitlines()
        assert lines[0] == "rank,configuration,fitness,fraction_of_optimum,pagerank"
        assert len(lines) == len(g["minima"]) + 1
        for ln, m in zip(lines[1:], g["minima"]):
            rk, key, f, fr, p = ln.rsplit(",", 3)[0].split(",", 1) + ln.rsplit(",", 3)[1:]
            digits = np.unravel_index(int(m), radix)
            assert int(rk) == m and key == ",".join(str(16 * int(x)) for x in digits).join('""')
            assert _num(f) == fit[m] and _num(fr) == f_opt / fit[m]
            assert abs(_num(p) - pr_ref[m]) <= 1e-12
        # write_cp_curve_csv (landscape.hpp:85)
        lines = open(os.path.join(tmp_path, f"cpcurve_{name}.csv")).read().splitlines()
        assert lines[0] == "p_percent,c_p" and len(lines) == len(ref["c_p_curve"]) + 1
        for ln, (k, c) in zip(lines[1:], ref["c_p_curve"]):
            kk, v = ln.split(",")
            assert int(kk) == k and abs(_num(v) - c) <= 1e-9
        # minima_fraction_report (landscape.hpp:87-94): f_opt / f over the minima,
        # ascending, median and mean
        fr = np.sort(f_opt / fit[g["minima"]])
        got = rd(f"fraction_{name}.bin", np.float64)
        assert np.array_equal(got, fr)
        med, mean, cnt = open(os.path.join(tmp_path, f"fraction_{name}.txt")).read().split()
        k = len(fr)
        want_med = fr[k // 2] if k % 2 else 0.5 * (fr[k // 2 - 1] + fr[k // 2])
        acc = 0.0
        for x in fr:
            acc += float(x)
        assert int(cnt) == k and float.fromhex(med) == want_med
        assert float.fromhex(mean) == acc / k
        # random_descents (extensions.hpp): the device validator through C++,
        # bit-identical to the oracle's restatement of climb_random_first
        counts, ev = O.descents(radix, fit, kind, 100000, 7)
        arr = rd(f"descents_{name}_arrivals.bin", np.uint64)
        assert np.array_equal(arr, counts[g["minima"]].astype(np.uint64))
        fa, dev = map(int, open(os.path.join(tmp_path, f"descents_{name}.txt")).read().split())
        assert fa == 100000 - int(counts[g["minima"]].sum()) and dev == ev
        if kind == O.ADJACENT:
            _check_graph_exports(tmp_path, fit, ok, g)


# ----------------------------------------------------------- cache files --

def test_save_load_round_trip(built, tmp_path):
    path = str(tmp_path / "c.json")
    dump(built, "savecache", path, 0.3, "rugged", 9, 5, 4, 3)
    out = dump(built, "loadcache", path)
    n = 60
    fit = np.frombuffer(out[: 8 * n], np.float64)
    ok = np.frombuffer(out[8 * n: 9 * n], np.uint8)
    ref_fit, ref_ok = O.gen_synthetic([5, 4, 3], 0.3, "rugged", 9)
    assert np.array_equal(fit.view(np.uint64), ref_fit.view(np.uint64))
    assert np.array_equal(ok, ref_ok)


@pytest.mark.gpu
@pytest.mark.parametrize("ingest", [[], ["--device-ingest"]])
def test_analyze_cli_matches_oracle(built, tmp_path, ingest):
    import json

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    radix, q, seed = [8, 6, 3, 3, 2], 0.52, 3
    path = str(tmp_path / "cache.json")
    dump(built, "savecache", path, q, "rugged", seed, *radix)
    rep_path = str(tmp_path / "rep.json")
    r = subprocess.run([os.path.join(built, "tk_analyze"), path, "--json", rep_path,
                        "--minima-csv", str(tmp_path / "m.csv"), *ingest],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rep = json.load(open(rep_path))
    fit, ok = O.gen_synthetic(radix, q, "rugged", seed)
    ref = O.analyze(radix, fit, ok, O.ADJACENT)
    assert rep["pagerank_iterations"] == ref["iterations"]
    assert [m["rank"] for m in rep["minima"]] == [int(x) for x in ref["ffg"]["minima"]]
    for e, (k, c) in zip(rep["c_p_curve"], ref["c_p_curve"]):
        assert e["p_percent"] == k and abs(e["c_p"] - c) <= 1e-9
    # exit codes of errors.hpp:8-9
    bad = subprocess.run([os.path.join(built, "tk_analyze"), path, "--neighbourhood", "diagonal"],
                         capture_output=True, text=True)
    assert bad.returncode == 2
    missing = subprocess.run([os.path.join(built, "tk_analyze"), str(tmp_path / "none.json")],
                             capture_output=True, text=True)
    assert missing.returncode == 1
