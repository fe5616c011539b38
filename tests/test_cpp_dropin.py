"""The C++ drop-in (include/tunekit/*.hpp + cpp/src, over the C-ABI).

CPU: the host classes (ParameterSpace, SearchSpaceCache, generators) are pinned
against the golden fixtures made from the reference's own build, and
landscape.cpp is shown to compile and link against the REFERENCE's own headers
and sources (source-level drop-in).
GPU: cpp/build/test_dropin drives every landscape.hpp entry point; its dumps
are compared with the CPU oracle.
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


def test_generators_match_reference(built, golden):
    meta, _ = golden
    for rec in meta["synthetic"]:
        n = rec["size"]
        r = subprocess.run([os.path.join(built, "tk_gen_dump"), "synthetic", str(rec["q"]),
                            rec["profile"], str(rec["seed"]), *map(str, rec["radix"])],
                           capture_output=True)
        assert r.returncode == 0, r.stderr
        fit = np.frombuffer(r.stdout[: 8 * n], np.float64)
        ok = np.frombuffer(r.stdout[8 * n:], np.uint8)
        assert sha(fit) == rec["sha_fit"], rec["key"]
        assert sha(ok) == rec["sha_ok"], rec["key"]
        r = subprocess.run([os.path.join(built, "tk_gen_dump"), "optimum", str(rec["q"]),
                            rec["profile"], str(rec["seed"]), *map(str, rec["radix"])],
                           capture_output=True, text=True)
        if rec["status"] == 0:
            f_hex, rank = r.stdout.split()
            assert float.fromhex(f_hex) == rec["f_opt"] and int(rank) == rec["opt_rank"]
        else:
            assert r.returncode == 4  # NoFeasiblePoint
    for rec in meta["nk"]:
        fit = np.frombuffer(dump(built, "nk", rec["n"], rec["k"], rec["seed"]), np.float64)
        assert sha(fit) == rec["sha_fit"], rec["key"]


def test_neighbour_ranks_match_reference(built, golden):
    meta, _ = golden
    for rec in meta["neighbours"]:
        out = dump(built, "neighbours", rec["kind"], *rec["radix"])
        n = rec["size"]
        assert sha(np.frombuffer(out[: 4 * n], np.uint32)) == rec["sha_counts"]
        assert sha(np.frombuffer(out[4 * n:], np.uint64)) == rec["sha_ranks"]


def test_conformance_build_against_reference_headers(built):
    """landscape.cpp + landscape_io.cpp + the driver, compiled with the
    reference's include/tunekit first on the include path and linked with the
    reference's own src/{value,space,cache,generators}.cpp."""
    if not os.path.exists("/root/reference/proj/src/space.cpp"):
        pytest.skip("reference sources not present on this host")
    exe = os.path.join(built, "conformance_ref")
    assert os.path.exists(exe)
    nm = subprocess.run(["nm", "-C", "--defined-only", exe], capture_output=True, text=True).stdout
    for sym in ("tunekit::build_ffg", "tunekit::pagerank", "tunekit::analyze_landscape",
                "tunekit::proportion_of_centrality", "tunekit::classify_points",
                "tunekit::export_graph", "tunekit::write_minima_csv"):
        assert sym in nm, sym


@pytest.mark.gpu
@pytest.mark.parametrize("exe", ["test_dropin", "conformance_ref"])
def test_dropin_on_gpu_matches_oracle(built, tmp_path, exe):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    path = os.path.join(built, exe)
    if not os.path.exists(path):
        pytest.skip(f"{exe} not built on this host")
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
        lines = open(os.path.join(tmp_path, f"minima_{name}.csv")).read().splitlines()
        assert lines[0].startswith("rank,") and len(lines) == len(g["minima"]) + 1
    assert open(os.path.join(tmp_path, "graph.dot")).read().startswith("digraph")


# ----------------------------------------------------------- cache files --

def test_load_cache_matches_reference(built, golden):
    """cache_io.cpp against the reference's own load_cache of the same files
    (a reference-written native cache and a Kernel Tuner style file)."""
    meta, arrays = golden
    gd = os.path.join(ROOT, "tests", "golden")
    for rec in meta["cache_files"]:
        out = dump(built, "loadcache", os.path.join(gd, rec["file"]))
        n = rec["size"]
        fit = np.frombuffer(out[: 8 * n], np.float64)
        ok = np.frombuffer(out[8 * n: 9 * n], np.uint8)
        pres = np.frombuffer(out[9 * n:], np.uint8)
        assert np.array_equal(fit.view(np.uint64), arrays[rec["name"] + "_fit"].view(np.uint64))
        assert np.array_equal(ok, arrays[rec["name"] + "_ok"])
        assert np.array_equal(pres, arrays[rec["name"] + "_present"])


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
