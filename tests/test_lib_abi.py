"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/adaptsolve.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "adaptsolve.h")
LIB = os.path.join(ROOT, "paper_2007_11208_b200", "libadaptsolve.so")
DEBUG_LIB = os.path.join(ROOT, "paper_2007_11208_b200", "libadaptsolve_debug.so")
_DECL = r"^\s*(?:int|int64_t|void|double|const char\*)\s+\**(as_\w+)\s*\("


def _split_header():
    src = open(HDR).read()
    a = src.index("#ifdef AS_DEBUG")
    b = src.index("#endif /* AS_DEBUG */")
    return src[:a] + src[b:], src[a:b]


def declared():
    """Symbols of the release boundary (outside the AS_DEBUG block)."""
    return sorted(set(re.findall(_DECL, _split_header()[0], re.M)))


def declared_debug():
    """Test-only symbols declared inside #ifdef AS_DEBUG."""
    return sorted(set(re.findall(_DECL, _split_header()[1], re.M)))


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
    assert sorted(AS.DEBUG_EXPORTS) == declared_debug()


def test_debug_exports_only_in_debug_build():
    """the test-only exports exist only in the -DAS_DEBUG build."""
    if not os.path.exists(DEBUG_LIB):
        import __graft_entry__
        __graft_entry__.build()
    rel, dbg = ctypes.CDLL(LIB), ctypes.CDLL(DEBUG_LIB)
    assert declared_debug(), "no AS_DEBUG block in the header"
    for name in declared_debug():
        assert not hasattr(rel, name), name
        assert hasattr(dbg, name), name
    for name in declared():
        assert hasattr(dbg, name), name


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
    # FORCE_METHOD reserves a band factor of any width (3n rows of W)
    assert AS.workspace_bytes(0, 1024, 1, AS.OPT_FORCE_METHOD) > b
    assert AS.workspace_bytes(0, -1, 1) == -1 and AS.workspace_bytes(7, 8, 1) == -1
