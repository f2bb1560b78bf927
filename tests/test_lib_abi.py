"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/adaptsolve.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "adaptsolve.h")
LIB = os.path.join(ROOT, "paper_2007_11208_b200", "libadaptsolve.so")


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+\**(as_\w+)\s*\(", src, re.M)))


def test_header_declares_boundary():
    names = declared()
    for must in ("as_solve", "as_solve_f64", "as_solve_f32", "as_solve_ex", "as_detect"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    lib = ctypes.CDLL(LIB)
    for name in declared():
        assert hasattr(lib, name), name
    lib.as_version.restype = ctypes.c_int
    assert lib.as_version() == 1
    lib.as_strerror.restype = ctypes.c_char_p
    assert b"singular" in lib.as_strerror(1)


def test_binding_names_match_header():
    import paper_2007_11208_b200 as AS
    for name in declared():
        assert name in AS.EXPORTS


def test_sm100a_sass_present():
    """The library carries sm_100a SASS with fp64 tensor-core MMA (DMMA)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("no cuobjdump")
    out = subprocess.run(["cuobjdump", "-lelf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "DMMA" in sass


def test_workspace_bytes_cpu():
    import paper_2007_11208_b200 as AS
    b = AS.workspace_bytes(0, 1024, 1)
    assert b > 8 * 1024 * 1024
