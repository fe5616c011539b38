"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/tk_landscape.h declares (no compute calls here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tk_landscape.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tk_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2210_01465_b200 import build

    return build.build()


def test_header_matches_binding_list():
    from paper_2210_01465_b200 import _abi

    assert declared_symbols() == sorted(_abi.EXPORTS)


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (tk_[a-z_]+)\b", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_reports_version(lib_path):
    from paper_2210_01465_b200 import _abi

    L = _abi.load(lib_path)
    assert L.tk_abi_version() == 1
    assert L.tk_status_name(4) == b"TK_ENOCONV"


def test_kernels_are_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_null_handle_is_einval(lib_path):
    from paper_2210_01465_b200 import _abi

    L = _abi.load(lib_path)
    n = C.c_uint64()
    assert L.tk_land_info(None, C.byref(n), None) == _abi.TK_EINVAL
    assert b"null" in L.tk_last_error()
