"""Build the sm_100a shared library in-tree (it travels to the GPU box with the repo).

    python -m paper_2210_01465_b200.build        # or __graft_entry__.build()

Produces paper_2210_01465_b200/libtk_landscape.so exporting the C-ABI of
include/tk_landscape.h.  nvcc cross-compiles without a GPU.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtk_landscape.so")
SOURCES = ["tk_kernels.cu", "tk_staged.cu", "tk_hamming.cu", "tk_hamsplit.cu", "tk_rows.cu", "tk_ring.cu",
           "tk_descent.cu", "tk_batch.cu", "tk_abi.cu"]
HEADERS = ["tk_internal.cuh", "tk_kernels.cuh", "tk_pipe.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise FileNotFoundError("nvcc not found")


def host_cxx() -> str:
    # the image exports CC/CXX pointing at a wrapper without the full runtime;
    # nvcc needs a plain g++ as its host compiler
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def flags(extra=()) -> list[str]:
    return [*ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false",
            "-ccbin", host_cxx(), "-Xcompiler", "-fPIC,-ffp-contract=off",
            "-I", os.path.join(ROOT, "include"), "-I", CSRC, *extra]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


# experiment variants (A/B on the GPU via TK_LIB=<path>); "" is the product build
VARIANTS = {
    "": [],
    "t256": ["-DTK_TILE=256", "-DTK_CTAS_PER_SM=2"],  # 256-rank tiles, two CTAs per SM
    "p1": ["-DTK_PROD_WARPS=1"],                      # one producer warp (round-1 layout)
    "p2": ["-DTK_PROD_WARPS=2"],
    "ne": ["-DTK_NO_EVICT=1"],                        # no L2 evict-first hints
    "trace": ["-DTK_TRACE=1"],                        # per-tile timeline of block 0 (stderr)
    "p6": ["-DTK_PROD_WARPS=6"],
    "pw3": ["-DTK_PW_AHEAD=3"],
    "hm1": ["-DTK_HAM_MINB=1"],
    "sp3": ["-DTK_SP_MINB=3"],  # Hamming dimension-group passes: 3 CTAs per SM (42 registers)
    "sp1": ["-DTK_SP_MINB=1"],
    "hu4": ["-DTK_HAM_UNROLL=4"],
    "pw4": ["-DTK_PW_AHEAD=4"],
    "s3": ["-DTK_MAX_STAGES=3"],  # at most 3 pipeline stages (more L1 left)
    # timing experiments (wrong results, fixed 29 iterations)
    "xnodim0": ["-DTK_X_ITERS=29", "-DTK_X_NODIM0=1"],
    "xnocomp": ["-DTK_X_ITERS=29", "-DTK_X_NOCOMP=1"],
    "xnocomp0": ["-DTK_X_ITERS=29", "-DTK_X_NOCOMP=1", "-DTK_X_NODIM0=1"],
    "xhalf": ["-DTK_X_ITERS=29", "-DTK_X_HALFLDS=1"],
    "spw": ["-DTK_STAGE_PW=1"],  # packed words staged by the producers
    "xnopw": ["-DTK_X_ITERS=29", "-DTK_X_NOPW=1"],  # no packed-word loads
    "xnofillnopw": ["-DTK_X_ITERS=29", "-DTK_X_NOPW=1", "-DTK_X_NOFILL=1"],
    "xnodadd": ["-DTK_X_ITERS=29", "-DTK_X_NODADD=1"],  # loads kept, fp64 chain replaced by XOR
    "xnofill": ["-DTK_X_ITERS=29", "-DTK_X_NOFILL=1"],  # no bulk copies into the stages
    "xnofilldadd": ["-DTK_X_ITERS=29", "-DTK_X_NOFILL=1", "-DTK_X_NODADD=1"],
    # staged Hamming timing experiments (wrong results)
    "hxnw": ["-DTK_X_ITERS=37", "-DTK_HX_NOWAIT=1"],  # consumers do not wait for the ring data
    "hxnc": ["-DTK_X_ITERS=37", "-DTK_HX_NOCOPY=1"],  # producers arrive without copying
}


def lib_path(variant: str = "") -> str:
    return LIB if not variant else LIB.replace(".so", f"_{variant}.so")


def build(force: bool = False, verbose: bool = False, variant: str = "") -> str:
    out = lib_path(variant)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "tk_landscape.h"))
    if not force and not _stale(out, deps):
        return out
    from concurrent.futures import ThreadPoolExecutor

    objs, cmds = [], []
    common = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "tk_landscape.h")]
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", f"{'_' + variant if variant else ''}.o"))
        objs.append(obj)
        if not force and not _stale(obj, [os.path.join(CSRC, src), *common]):
            continue  # translation unit unchanged since its object was built
        cmds.append([nvcc(), *flags((["-Xptxas", "-v"] if verbose else []) + VARIANTS[variant]),
                     "-c", os.path.join(CSRC, src), "-o", obj])
    with ThreadPoolExecutor(max(1, len(cmds))) as ex:  # translation units compile independently
        for f in [ex.submit(subprocess.run, c, check=True) for c in cmds]:
            f.result()
    cmd = [nvcc(), *ARCH, "-ccbin", host_cxx(), "-shared", "-o", out, *objs]
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant=var))
