"""CPU oracle for the adaptive solver of arXiv 2007.11208 -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  The product path
(``paper_2007_11208_b200``) never imports it: the two share no code.

Thin ctypes wrapper over ``liboracle.so`` (plain unblocked C, see
``oracle_impl.h``; every function there cites the PAPER.md passage it follows).
Matrices are numpy arrays in column-major (Fortran) order; float64 selects the
``_d`` routines, float32 the ``_f`` routines.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

# flag bits (mirror oracle.h)
BANDED, LOWER, UPPER, SPD = 0x1, 0x2, 0x4, 0x8
F_CHOL_FAILED, F_SINGULAR, F_RCOND_LOW, F_FALLBACK = 1 << 8, 1 << 9, 1 << 10, 1 << 11
F_POORLY_COND, F_NONFINITE, F_SVD_NOCONV, F_RANK_DEF = 1 << 12, 1 << 13, 1 << 14, 1 << 15
M_BAND, M_TRI_LOWER, M_TRI_UPPER, M_CHOL, M_LU, M_SVD = 1, 2, 3, 4, 5, 6
OPT_NO_FALLBACK, OPT_FORCE_METHOD, OPT_FULLSCAN = 0x1, 0x2, 0x8
OPT_CHECK_FINITE = 0x4
OPT_SYM_INDEF = 0x20
M_LDLT = 7
F_SYMMETRIC = 1 << 16
ERR_NONFINITE = 3
F_NONFINITE = 1 << 13
ERR_SINGULAR_NO_FALLBACK, ERR_SVD_NOT_CONVERGED = 1, 2


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2 -ffp-contract=off, no fast-math)."""
    src = [os.path.join(_HERE, f) for f in ("oracle.c", "oracle_impl.h", "oracle.h")]
    if not force and os.path.exists(_SO) and all(os.path.getmtime(_SO) >= os.path.getmtime(s) for s in src):
        return _SO
    cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
           "-Wall", "-Wno-unused-function", "-o", _SO + ".tmp", os.path.join(_HERE, "oracle.c"), "-lm"]
    subprocess.check_call(cmd)
    os.replace(_SO + ".tmp", _SO)    # a running process keeps its mapped copy
    return _SO


class Structure(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("pad", C.c_int32), ("kl", C.c_int64), ("ku", C.c_int64),
                ("max_diag", C.c_double)]


class Options(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("force_method", C.c_int32), ("rcond_threshold", C.c_double),
                ("lsq_cutoff", C.c_double), ("max_sweeps", C.c_int32), ("pad", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("method", C.c_int32), ("primary_method", C.c_int32),
                ("sweeps", C.c_int32), ("kl", C.c_int64), ("ku", C.c_int64), ("rcond", C.c_double),
                ("anorm", C.c_double), ("rank", C.c_int64), ("info", C.c_int64), ("chol_fail_col", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_SO)
        P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
        for s in ("d", "f"):
            g = lambda name: getattr(_lib, f"{name}_{s}")
            g("or_detect").argtypes = [P, I64, I64, P]
            g("or_getrf").argtypes = [P, I64, I64, P]; g("or_getrf").restype = I64
            g("or_getrs").argtypes = [P, I64, I64, P, P, I64, I64]
            g("or_potrf").argtypes = [P, I64, I64]; g("or_potrf").restype = I64
            g("or_sytrf").argtypes = [P, I64, I64, P]; g("or_sytrf").restype = I64
            g("or_sytrs").argtypes = [P, I64, I64, P, P, I64, I64]
            g("or_trsv").argtypes = [P, I64, I64, I, I, I, P]
            g("or_band_pack").argtypes = [P, I64, I64, I64, I64, P, I64]; g("or_band_pack").restype = D
            g("or_gbtrf").argtypes = [I64, I64, I64, P, I64, P]; g("or_gbtrf").restype = I64
            g("or_gbtrs").argtypes = [I64, I64, I64, P, I64, P, P, I64, I64, I]
            g("or_norm1").argtypes = [P, I64, I64]; g("or_norm1").restype = D
            g("or_rcond").argtypes = [I, P, I64, I64, I64, I64, P, I, D, P]; g("or_rcond").restype = D
            g("or_geqr").argtypes = [P, I64, I64, P, I64, I64]
            g("or_jacobi").argtypes = [P, I64, I64, P, I, P]; g("or_jacobi").restype = I
            g("or_lsq_svd").argtypes = [P, I64, I64, P, I64, I64, P, I64, D, I, P, P, P]; g("or_lsq_svd").restype = I64
            g("or_solve").argtypes = [P, I64, I64, P, I64, I64, P, I64, P, P, P]; g("or_solve").restype = I
        _lib.or_set_threads.argtypes = [C.c_int]
        _lib.or_get_threads.restype = C.c_int
    return _lib


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def get_threads() -> int:
    return int(lib().or_get_threads())


def _sfx(a: np.ndarray) -> str:
    if a.dtype == np.float64:
        return "d"
    if a.dtype == np.float32:
        return "f"
    raise TypeError(f"oracle supports float64/float32, got {a.dtype}")


def _fortran(a: np.ndarray) -> np.ndarray:
    a = np.asarray(a)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return np.asfortranarray(a)


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _fn(name: str, a: np.ndarray):
    return getattr(lib(), f"{name}_{_sfx(a)}")


# ---------------------------------------------------------------- detection
@dataclass
class Detect:
    flags: int
    kl: int
    ku: int
    max_diag: float

    @property
    def banded(self):
        return bool(self.flags & BANDED)

    @property
    def lower(self):
        return bool(self.flags & LOWER)

    @property
    def upper(self):
        return bool(self.flags & UPPER)

    @property
    def spd(self):
        return bool(self.flags & SPD)

    @property
    def method(self) -> int:
        """First-match dispatch order of P:164-169."""
        if self.flags & BANDED:
            return M_BAND
        if self.flags & LOWER:
            return M_TRI_LOWER
        if self.flags & UPPER:
            return M_TRI_UPPER
        if self.flags & SPD:
            return M_CHOL
        return M_LU


def detect(A: np.ndarray) -> Detect:
    A = _fortran(A)
    n = A.shape[0]
    st = Structure()
    _fn("or_detect", A)(_ptr(A), max(1, A.shape[0]), n, C.byref(st))
    return Detect(st.flags, st.kl, st.ku, st.max_diag)


# ---------------------------------------------------------------- pieces
def getrf(A: np.ndarray):
    W = _fortran(A).copy(order="F")
    n = W.shape[0]
    ipiv = np.zeros(n, dtype=np.int64)
    info = _fn("or_getrf", W)(_ptr(W), max(1, n), n, _ptr(ipiv))
    return W, ipiv, int(info)


def getrs(W, ipiv, B):
    X = _fortran(B).astype(W.dtype, copy=True, order="F")
    n = W.shape[0]
    _fn("or_getrs", W)(_ptr(W), max(1, n), n, _ptr(np.ascontiguousarray(ipiv, dtype=np.int64)), _ptr(X), max(1, n), X.shape[1])
    return X


def potrf(A):
    L = _fortran(A).copy(order="F")
    n = L.shape[0]
    info = _fn("or_potrf", L)(_ptr(L), max(1, n), n)
    return np.tril(L), int(info)


def sytrf(A):
    """Bunch-Kaufman L D L^T (lower) of the oracle: (W, ipiv 0-based with -(kp+1) for 2x2 blocks, info)."""
    W = _fortran(A).copy(order="F")
    n = W.shape[0]
    ipiv = np.zeros(n, dtype=np.int64)
    info = _fn("or_sytrf", W)(_ptr(W), max(1, n), n, _ptr(ipiv))
    return W, ipiv, int(info)


def sytrs(W, ipiv, B):
    W = _fortran(W)
    X = _fortran(B).astype(W.dtype, copy=True).reshape(W.shape[0], -1, order="F")
    n = W.shape[0]
    _fn("or_sytrs", W)(_ptr(W), max(1, n), n, _ptr(np.ascontiguousarray(ipiv, dtype=np.int64)), _ptr(X), max(1, n),
                       X.shape[1])
    return X


def trsv(A, b, upper: bool, trans: bool = False, unit: bool = False):
    A = _fortran(A)
    x = np.array(b, dtype=A.dtype, copy=True).reshape(-1)
    n = A.shape[0]
    _fn("or_trsv", A)(_ptr(A), max(1, n), n, int(upper), int(trans), int(unit), _ptr(x))
    return x


def band_pack(A, kl, ku):
    A = _fortran(A)
    n = A.shape[0]
    ldab = 2 * kl + ku + 1
    ab = np.zeros((ldab, n), dtype=A.dtype, order="F")
    anorm = _fn("or_band_pack", A)(_ptr(A), max(1, n), n, kl, ku, _ptr(ab), ldab)
    return ab, anorm


def gbtrf(ab, kl, ku):
    ab = np.asfortranarray(ab).copy(order="F")
    n = ab.shape[1]
    ipiv = np.zeros(n, dtype=np.int64)
    info = _fn("or_gbtrf", ab)(n, kl, ku, _ptr(ab), ab.shape[0], _ptr(ipiv))
    return ab, ipiv, int(info)


def gbtrs(ab, kl, ku, ipiv, B, trans=False):
    X = _fortran(B).astype(ab.dtype, copy=True, order="F")
    n = ab.shape[1]
    _fn("or_gbtrs", ab)(n, kl, ku, _ptr(ab), ab.shape[0], _ptr(np.ascontiguousarray(ipiv, dtype=np.int64)),
                        _ptr(X), max(1, n), X.shape[1], int(trans))
    return X


def norm1(A):
    A = _fortran(A)
    return _fn("or_norm1", A)(_ptr(A), max(1, A.shape[0]), A.shape[0])


KIND_LU, KIND_BAND, KIND_TRI, KIND_CHOL = 0, 1, 2, 3


def rcond(kind, F, anorm, n=None, kl=0, ku=0, ipiv=None, upper=False):
    """rcond estimate from factors F (LU W / band ab / triangle A / Cholesky L)."""
    F = np.asfortranarray(F)
    n = F.shape[1] if n is None else n
    ns = C.c_int(0)
    ip = np.ascontiguousarray(ipiv, dtype=np.int64) if ipiv is not None else np.zeros(1, dtype=np.int64)
    r = _fn("or_rcond", F)(kind, _ptr(F), F.shape[0], n, kl, ku, _ptr(ip), int(upper), float(anorm), C.byref(ns))
    return r, ns.value


def geqr(A, B):
    W = _fortran(A).copy(order="F")
    Cm = _fortran(B).astype(W.dtype, copy=True, order="F")
    n = W.shape[0]
    _fn("or_geqr", W)(_ptr(W), max(1, n), n, _ptr(Cm), max(1, n), Cm.shape[1])
    return W, Cm


def jacobi(M, max_sweeps=30):
    M = _fortran(M).copy(order="F")
    n = M.shape[0]
    V = np.zeros((n, n), dtype=M.dtype, order="F")
    conv = C.c_int(0)
    sweeps = _fn("or_jacobi", M)(_ptr(M), max(1, n), n, _ptr(V), max_sweeps, C.byref(conv))
    return M, V, int(sweeps), bool(conv.value)


def lsq_svd(A, B, cut=None, max_sweeps=30):
    A = _fortran(A)
    B = _fortran(B).astype(A.dtype, copy=False)
    n, nrhs = A.shape[0], B.shape[1]
    X = np.zeros((n, nrhs), dtype=A.dtype, order="F")
    sig = np.zeros(n, dtype=A.dtype)
    sw, cv = C.c_int(0), C.c_int(0)
    eps = float(np.finfo(A.dtype).eps)
    cut = n * eps if cut is None else cut
    rank = _fn("or_lsq_svd", A)(_ptr(A), max(1, n), n, _ptr(B), max(1, n), nrhs, _ptr(X), max(1, n), float(cut),
                                max_sweeps, _ptr(sig), C.byref(sw), C.byref(cv))
    return X, int(rank), sig, int(sw.value), bool(cv.value)


# ---------------------------------------------------------------- solve
def solve(A, B, *, no_fallback=False, force_method=None, fullscan=False, rcond_threshold=-1.0,
          lsq_cutoff=-1.0, max_sweeps=30, check_finite=False, sym_indef=False):
    """The adaptive solve (oracle_impl.h: or_solve).  Returns (ret, X, report dict, sigma)."""
    A = _fortran(A)
    B = _fortran(B).astype(A.dtype, copy=False)
    n, nrhs = A.shape[0], B.shape[1]
    X = np.zeros((n, nrhs), dtype=A.dtype, order="F")
    sig = np.zeros(max(n, 1), dtype=A.dtype)
    o = Options()
    o.flags = (OPT_NO_FALLBACK if no_fallback else 0) | (OPT_FORCE_METHOD if force_method else 0) | \
        (OPT_FULLSCAN if fullscan else 0) | (OPT_CHECK_FINITE if check_finite else 0) | \
        (OPT_SYM_INDEF if sym_indef else 0)
    o.force_method = int(force_method or 0)
    o.rcond_threshold = rcond_threshold
    o.lsq_cutoff = lsq_cutoff
    o.max_sweeps = max_sweeps
    rep = Report()
    ret = _fn("or_solve", A)(_ptr(A), max(1, n), n, _ptr(B), max(1, n), nrhs, _ptr(X), max(1, n),
                             C.byref(o), C.byref(rep), _ptr(sig))
    return int(ret), X, rep.as_dict(), sig[:n]
