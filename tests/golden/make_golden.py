"""Generate the golden fixtures from the reference's OWN compiled code.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It loads oracle/_ref/libtkref.so -- the reference's src/{value,space,cache,
generators}.cpp compiled where they lie plus the extern "C" probes in
oracle/ref_shim.cpp -- and records:

  * neighbour lists       ParameterSpace::neighbour_ranks   (space.cpp:167-187)
  * strides / size        ParameterSpace ctor                (space.cpp:48-53)
  * synthetic caches      generate_synthetic_kernel_space    (generators.cpp:89-145)
  * NK landscapes         generate_nk_landscape              (generators.cpp:25-79)
  * f_opt / optimum rank  SearchSpaceCache::finalize/optimum (cache.cpp:55-98)
  * FFG CSR + minima      the intended build_ffg loop over neighbour_ranks and
                          SearchSpaceCache::mean/ok (SURVEY.md s3 HOT LOOP 1)

Small cases are stored as arrays (golden.npz), larger ones as sha256 digests
(golden.json).  The fixtures travel to the GPU box; the reference does not.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

PAPER_SHAPES = {  # PAPER.md:797-829 / SPEC.md:88 (Appendix A value-list sizes)
    "conv": (12, 6, 8, 8, 2, 2),
    "conv_mi50": (8, 6, 3, 3, 2),
    "gemm": (4, 4, 3, 3, 3, 3, 4, 4, 2, 2),
    "pnpoly": (31, 11, 4, 2, 3),
}
PAPER_FAIL = {"conv": 0.68, "conv_mi50": 0.52, "gemm": 0.78, "pnpoly": 0.04}  # Table II ratios

NEIGHBOUR_SPACES = [(3, 1, 4), (8, 6, 3, 3, 2), (2, 2, 2, 2, 2, 2, 2, 2), (5, 7), (16,),
                    (12, 12, 12, 12), (31, 11, 4, 2, 3)]
FULL_LIMIT = 9000  # store arrays (not only digests) up to this many nodes


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    R = oracle.ref()
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"neighbours": [], "synthetic": [], "nk": []}

    for radix in NEIGHBOUR_SPACES:
        r = np.array(radix, np.uint32)
        st = np.zeros(len(r), np.uint64)
        n = int(R.ref_space_size(len(r), r, st))
        for kind in (oracle.HAMMING, oracle.ADJACENT):
            mx = max(1, oracle.max_neighbours(r, kind))
            out = np.zeros(n * mx, np.uint64)
            cnt = np.zeros(n, np.uint32)
            k = int(R.ref_all_neighbours(len(r), r, kind, out, cnt))
            key = f"nb_{'x'.join(map(str, radix))}_{kind}"
            rec = dict(key=key, radix=list(radix), kind=kind, size=n,
                       strides=[int(x) for x in st], total=k,
                       sha_counts=sha(cnt), sha_ranks=sha(out[:k]))
            if n <= 2000:
                arrays[key + "_counts"] = cnt
                arrays[key + "_ranks"] = out[:k]
            meta["neighbours"].append(rec)

    cases = []
    for name, radix in PAPER_SHAPES.items():
        seeds = range(9) if name in ("conv_mi50", "pnpoly") else range(2)
        for s in seeds:
            cases.append((name, radix, PAPER_FAIL[name], "rugged", s))
    cases += [("c1_shape", (12, 12, 12, 12), 0.0, "smooth", 1),
              ("ridged", (6, 5, 4, 3, 2), 0.2, "ridged", 3),
              ("allfail_edge", (4, 4), 0.999999, "rugged", 11)]
    for name, radix, q, prof, seed in cases:
        r = np.array(radix, np.uint32)
        n = oracle.space_size(r)
        fit = np.empty(n, np.float64)
        ok = np.empty(n, np.uint8)
        fo, orr = C.c_double(), C.c_uint64()
        st = R.ref_generate_synthetic(len(r), r, q, prof.encode(), seed, fit, ok,
                                      C.byref(fo), C.byref(orr))
        key = f"syn_{name}_{seed}"
        rec = dict(key=key, name=name, radix=list(radix), q=q, profile=prof, seed=seed,
                   size=n, status=int(st), sha_fit=sha(fit), sha_ok=sha(ok),
                   ok_count=int(ok.sum()))
        if st == 0:
            rec.update(f_opt=fo.value, f_opt_hex=fo.value.hex(), opt_rank=int(orr.value))
        full = n <= 2000 or (n <= FULL_LIMIT and seed == 0)
        rec["full"] = full
        if full:
            arrays[key + "_fit"] = fit
            arrays[key + "_ok"] = ok
        rec["ffg"] = {}
        for kind in (oracle.HAMMING, oracle.ADJACENT):
            cap = n * max(1, oracle.max_neighbours(r, kind))
            off = np.zeros(n + 1, np.uint64)
            tg = np.zeros(max(1, cap), np.uint32)
            sk = np.zeros(n, np.uint8)
            mn = np.zeros(n, np.uint32)
            e, m = C.c_uint64(), C.c_uint64()
            rc = R.ref_ffg(len(r), r, fit, ok, kind, off, tg, cap, sk, mn, C.byref(e),
                           C.byref(m))
            assert rc == 0
            E, M = int(e.value), int(m.value)
            rec["ffg"][str(kind)] = dict(edges=E, minima=M, sha_offsets=sha(off),
                                         sha_targets=sha(tg[:E]), sha_is_sink=sha(sk),
                                         sha_minima=sha(mn[:M]))
            if full and E <= 200_000:
                arrays[f"{key}_k{kind}_offsets"] = off
                arrays[f"{key}_k{kind}_targets"] = tg[:E]
                arrays[f"{key}_k{kind}_minima"] = mn[:M]
        meta["synthetic"].append(rec)

    # k = 0 is left out: the reference's link loop (generators.cpp:38-44) never
    # stops at k = 0 and indexes past its 2-entry tables (undefined behaviour).
    for nn, kk, seed in [(10, 3, 5), (16, 4, 1), (12, 1, 2)]:
        fit = np.empty(1 << nn, np.float64)
        assert R.ref_generate_nk(nn, kk, seed, fit) == 0
        key = f"nk_{nn}_{kk}_{seed}"
        meta["nk"].append(dict(key=key, n=nn, k=kk, seed=seed, sha_fit=sha(fit)))
        if nn <= 12:
            arrays[key + "_fit"] = fit

    # cache files: one written by the reference's save_cache, one Kernel Tuner
    # style file (tune_params, error strings, null, times arrays, booleans);
    # the expected tables are the reference's own load_cache of each
    native = os.path.join(HERE, "cache_native.json")
    assert R.ref_save_synthetic(3, np.array([3, 4, 2], np.uint32), 0.25, b"rugged", 5,
                                native.encode()) == 0
    kt = {"kernel_name": "kt_demo", "device_name": "B200",
          "tune_params_keys": ["block", "tile", "unroll"],
          "tune_params": {"block": [128, 32, 64], "tile": [1, 2], "unroll": [True, False]},
          "cache": {}}
    rng = np.random.default_rng(11)
    for b in (32, 64, 128):
        for t in (1, 2):
            for u in (0, 1):
                key = f"{b},{t},{u}"
                r = rng.random()
                if r < 0.2:
                    kt["cache"][key] = {"time": "CompilationFailedConfig"}
                elif r < 0.3:
                    kt["cache"][key] = None
                elif r < 0.6:
                    kt["cache"][key] = {"times": [float(x) for x in rng.random(4) + 1.0]}
                else:
                    kt["cache"][key] = {"time": float(rng.random() + 1.0)}
    ktp = os.path.join(HERE, "cache_kt.json")
    with open(ktp, "w") as f:
        json.dump(kt, f, indent=1)
    meta["cache_files"] = []
    for name, path in (("cache_native", native), ("cache_kt", ktp)):
        n = R.ref_load_cache(path.encode(), None, None, None)
        assert n > 0
        fit = np.empty(n, np.float64)
        ok = np.empty(n, np.uint8)
        pres = np.empty(n, np.uint8)
        assert R.ref_load_cache(path.encode(), fit.ctypes.data, ok.ctypes.data, pres.ctypes.data) == n
        arrays[name + "_fit"], arrays[name + "_ok"], arrays[name + "_present"] = fit, ok, pres
        meta["cache_files"].append(dict(name=name, file=os.path.basename(path), size=int(n)))

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"wrote {len(arrays)} arrays, {len(meta['synthetic'])} synthetic cases")


if __name__ == "__main__":
    main()
