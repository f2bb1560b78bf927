"""paper_2007_11208_b200 -- B200-native adaptive solver for A X = B.

Thin Python binding over ``libadaptsolve.so`` (C ABI in ``include/adaptsolve.h``):
argument marshalling only.  Every step of the solve (structure detection,
banded / triangular / Cholesky / LU factorizations, the rcond estimate, the SVD
fallback) runs in the library's CUDA kernels for sm_100a.  There is no CPU or
PyTorch fallback: if the library is missing this module refuses to import.

Matrices are torch CUDA tensors in column-major layout (``stride(0) == 1``), as
produced by :func:`to_device` from Fortran-ordered numpy arrays.  PyTorch is
used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libadaptsolve.so")
# the same sources built with -DAS_DEBUG: adds the test-only as_debug_* exports (loaded on demand by
# the reconstruction tests and the diagnostic tools, never by the solve, the bench or smoke())
DEBUG_LIB_PATH = os.path.join(_HERE, "libadaptsolve_debug.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libadaptsolve.so not found at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'`"
                      " (there is deliberately no CPU fallback)")

# AS_USE_DEBUG_LIB=1 (diagnostic tools only): every call goes through the -DAS_DEBUG build, so the
# as_debug_* diagnostics see the plans of the solves made through this module
_USE_DEBUG = os.environ.get("AS_USE_DEBUG_LIB", "") not in ("", "0")
_lib = C.CDLL(DEBUG_LIB_PATH if _USE_DEBUG else LIB_PATH)

AS_F64, AS_F32 = 0, 1
FLAG_BANDED, FLAG_LOWER, FLAG_UPPER, FLAG_SPD = 0x1, 0x2, 0x4, 0x8
FLAG_CHOL_FAILED, FLAG_SINGULAR, FLAG_RCOND_LOW, FLAG_FALLBACK = 1 << 8, 1 << 9, 1 << 10, 1 << 11
FLAG_POORLY_COND, FLAG_SVD_NOCONV, FLAG_RANK_DEF = 1 << 12, 1 << 14, 1 << 15
FLAG_NONFINITE = 1 << 13
METHOD_BAND, METHOD_TRI_LOWER, METHOD_TRI_UPPER, METHOD_CHOL, METHOD_LU, METHOD_SVD = 1, 2, 3, 4, 5, 6
OPT_NO_FALLBACK, OPT_FORCE_METHOD, OPT_FULLSCAN = 0x1, 0x2, 0x8
OPT_SKIP_DETECT, OPT_CHECK_FINITE, OPT_SYM_INDEF = 0x10, 0x4, 0x20
METHOD_LDLT, FLAG_SYMMETRIC = 7, 1 << 16
ERR_SINGULAR_NO_FALLBACK, ERR_SVD_NOT_CONVERGED, ERR_NONFINITE = 1, 2, 3

EXPORTS = ("as_solve", "as_solve_f64", "as_solve_f32", "as_solve_ex", "as_solve_async", "as_solve_host",
           "as_solve_batched", "as_detect", "as_workspace_bytes", "as_last_kernel_nodes", "as_release_all",
           "as_strerror", "as_version", "as_set_instrumentation", "as_last_stage_ms", "as_measure_fp64_peak",
           "as_set_exec_mode", "as_bench_gemm")
DEBUG_EXPORTS = ("as_debug_factor", "as_debug_timestamps", "as_debug_lu_trace", "as_debug_panel_time")


class Options(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("force_method", C.c_int32), ("rcond_threshold", C.c_double),
                ("lsq_cutoff", C.c_double), ("max_sweeps", C.c_int32), ("reserved", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("method", C.c_int32), ("primary_method", C.c_int32), ("sweeps", C.c_int32),
                ("kl", C.c_int64), ("ku", C.c_int64), ("rcond", C.c_double), ("anorm", C.c_double),
                ("rank", C.c_int64), ("info", C.c_int64), ("chol_fail_col", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Structure(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("method", C.c_int32), ("kl", C.c_int64), ("ku", C.c_int64),
                ("max_diag", C.c_double), ("nonfinite_seen", C.c_int32), ("reserved", C.c_int32)]


P, I64, D, U32, I32 = C.c_void_p, C.c_int64, C.c_double, C.c_uint32, C.c_int32
_lib.as_solve.argtypes = [I32, P, I64, I64, P, I64, I64, P, P, P, P]
_lib.as_solve.restype = C.c_int
_lib.as_solve_ex.argtypes = [I32, P, I64, I64, P, I64, I64, P, P, P, P, P]
_lib.as_solve_ex.restype = C.c_int
_lib.as_solve_async.argtypes = [I32, P, I64, I64, P, I64, I64, P, P, P, P, P]
_lib.as_solve_async.restype = C.c_int
_lib.as_solve_host.argtypes = [I32, P, I64, I64, P, I64, I64, P, P, P, P]
_lib.as_solve_batched.argtypes = [I32, I64, I64, I64, P, I64, I64, P, I64, I64, P, I64, I64, P, P, P, P, P]
_lib.as_solve_batched.restype = C.c_int
_lib.as_solve_host.restype = C.c_int
_lib.as_detect.argtypes = [I32, P, I64, I64, U32, P, P]
_lib.as_detect.restype = C.c_int
_lib.as_workspace_bytes.argtypes = [I32, I64, I64, U32]
_lib.as_workspace_bytes.restype = I64
_lib.as_strerror.argtypes = [C.c_int]
_lib.as_strerror.restype = C.c_char_p
_lib.as_version.restype = C.c_int
_lib.as_last_kernel_nodes.restype = I64


def lib():
    return _lib


def version() -> int:
    return _lib.as_version()


def strerror(code: int) -> str:
    return _lib.as_strerror(code).decode()


def _dt(t) -> int:
    import torch
    if t.dtype == torch.float64:
        return AS_F64
    if t.dtype == torch.float32:
        return AS_F32
    raise TypeError(f"adaptsolve supports float64/float32, got {t.dtype}")


def _ld(t) -> int:
    """Column-major leading dimension of a 2-D (or 1-D) CUDA tensor."""
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor (use to_device)")
    rows = t.shape[0]
    if rows > 1 and t.stride(0) != 1:
        raise ValueError("expected a column-major tensor (stride(0) == 1); use to_device()")
    if t.dim() == 1 or t.shape[1] <= 1:
        return max(1, rows)
    return max(1, t.stride(1))


def _stream_ptr(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def empty_colmajor(rows: int, cols: int, dtype, device="cuda"):
    """rows x cols CUDA tensor in column-major layout (stride(0) == 1, ld = rows)."""
    import torch
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


def to_device(a: np.ndarray, device="cuda"):
    """Fortran-ordered numpy (n x m) -> column-major CUDA tensor (stride(0) == 1)."""
    import torch
    a = np.asarray(a)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    t = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(a).T)).to(device)
    return t.t()


def to_host(t) -> np.ndarray:
    return np.asfortranarray(t.t().contiguous().cpu().numpy().T)


def make_options(no_fallback=False, force_method=None, fullscan=False, rcond_threshold=-1.0, lsq_cutoff=-1.0,
                 max_sweeps=30, skip_detect=False, check_finite=False, sym_indef=False) -> Options:
    o = Options()
    o.flags = (OPT_NO_FALLBACK if no_fallback else 0) | (OPT_FORCE_METHOD if force_method else 0) | \
        (OPT_FULLSCAN if fullscan else 0) | (OPT_SKIP_DETECT if skip_detect else 0) | \
        (OPT_CHECK_FINITE if check_finite else 0) | (OPT_SYM_INDEF if sym_indef else 0)
    o.force_method = int(force_method or 0)
    o.rcond_threshold = float(rcond_threshold)
    o.lsq_cutoff = float(lsq_cutoff)
    o.max_sweeps = int(max_sweeps)
    return o


def as_solve(A, B, X=None, stream=None):
    """as_solve(A, lda, n, B, ldb, nrhs, X, &flags, &rcond, stream).  Returns (ret, X, flags, rcond)."""
    n, nrhs = A.shape[0], (B.shape[1] if B.dim() == 2 else 1)
    if X is None:
        X = empty_colmajor(n, nrhs, B.dtype) if B.dim() == 2 else B.new_empty(n)
    flags, rc = C.c_uint32(0), C.c_double(0)
    ret = _lib.as_solve(_dt(A), A.data_ptr(), _ld(A), n, B.data_ptr(), _ld(B), nrhs, X.data_ptr(), C.byref(flags),
                        C.byref(rc), _stream_ptr(stream))
    return ret, X, flags.value, rc.value


def as_solve_ex(A, B, X=None, options: Options | None = None, sigma_out=None, stream=None):
    """Returns (ret, X, report dict)."""
    n, nrhs = A.shape[0], (B.shape[1] if B.dim() == 2 else 1)
    if X is None:
        X = empty_colmajor(n, nrhs, B.dtype) if B.dim() == 2 else B.new_empty(n)
    rep = Report()
    ret = _lib.as_solve_ex(_dt(A), A.data_ptr(), _ld(A), n, B.data_ptr(), _ld(B), nrhs, X.data_ptr(),
                           C.byref(options) if options is not None else None, C.byref(rep),
                           sigma_out.data_ptr() if sigma_out is not None else None, _stream_ptr(stream))
    return ret, X, rep.as_dict()


def as_solve_async(A, B, X, options: Options | None = None, rep_dev=None, stream=None) -> int:
    n, nrhs = A.shape[0], (B.shape[1] if B.dim() == 2 else 1)
    return _lib.as_solve_async(_dt(A), A.data_ptr(), _ld(A), n, B.data_ptr(), _ld(B), nrhs, X.data_ptr(),
                               C.byref(options) if options is not None else None,
                               rep_dev.data_ptr() if rep_dev is not None else None, None, _stream_ptr(stream))


def as_solve_host(A: np.ndarray, B: np.ndarray, options: Options | None = None, stream=None, X: np.ndarray | None = None):
    """Host (numpy, Fortran-order) buffers in and out; copies inside the call."""
    A = np.asfortranarray(A)
    B = np.asfortranarray(B.reshape(B.shape[0], -1))
    n, nrhs = A.shape[0], B.shape[1]
    if X is None:
        X = np.empty((n, nrhs), dtype=A.dtype, order="F")
    dt = AS_F64 if A.dtype == np.float64 else AS_F32
    rep = Report()
    ret = _lib.as_solve_host(dt, A.ctypes.data, max(1, n), n, B.ctypes.data, max(1, n), nrhs, X.ctypes.data,
                             C.byref(options) if options is not None else None, C.byref(rep), _stream_ptr(stream))
    return ret, X, rep.as_dict()


def as_solve_batched(A, B, X=None, options: Options | None = None, sigma_out=None, stream=None):
    """Batched solve of A[b] X[b] = B[b].  A: (batch, n, n) CUDA tensor whose matrices are column-major
    (A.stride(1) == 1, i.e. created as to_device_batched); B: (batch, n, nrhs) likewise.  Returns
    (ret, X, reports) with reports a (batch, 11) view of the device as_report array and the
    per-system return codes as an int32 CUDA tensor (no host sync happens here)."""
    import torch
    batch, n = A.shape[0], A.shape[1]
    nrhs = B.shape[2]
    if X is None:
        X = empty_colmajor_batched(batch, n, nrhs, B.dtype, device=B.device)
    for t in (A, B, X):
        if t.shape[1] > 1 and t.stride(1) != 1:
            raise ValueError("expected column-major matrices (stride(1) == 1); use to_device_batched()")
    rep = torch.zeros((batch, C.sizeof(Report)), dtype=torch.uint8, device=A.device)
    rets = torch.zeros(batch, dtype=torch.int32, device=A.device)
    ret = _lib.as_solve_batched(_dt(A), n, nrhs, batch, A.data_ptr(), max(1, A.stride(2)), A.stride(0),
                                B.data_ptr(), max(1, B.stride(2) if nrhs > 1 else n), B.stride(0),
                                X.data_ptr(), max(1, X.stride(2) if nrhs > 1 else n), X.stride(0),
                                C.byref(options) if options is not None else None, rep.data_ptr(), rets.data_ptr(),
                                sigma_out.data_ptr() if sigma_out is not None else None, _stream_ptr(stream))
    return ret, X, rep, rets


def reports_to_host(rep) -> list:
    """Device report array (from as_solve_batched) -> list of dicts."""
    raw = rep.cpu().numpy().tobytes()
    sz = C.sizeof(Report)
    out = []
    for b in range(rep.shape[0]):
        r = Report.from_buffer_copy(raw[b * sz:(b + 1) * sz])
        out.append(r.as_dict())
    return out


def empty_colmajor_batched(batch: int, rows: int, cols: int, dtype, device="cuda"):
    import torch
    return torch.empty((batch, cols, rows), dtype=dtype, device=device).transpose(1, 2)


def to_device_batched(a: np.ndarray, device="cuda"):
    """(batch, n, m) numpy -> CUDA tensor whose matrices are column-major (stride(1) == 1)."""
    import torch
    a = np.asarray(a)
    t = torch.from_numpy(np.ascontiguousarray(np.transpose(a, (0, 2, 1)))).to(device)
    return t.transpose(1, 2)


def as_detect(A, fullscan=False, stream=None, check_finite=False):
    st = Structure()
    fl = (OPT_FULLSCAN if fullscan else 0) | (OPT_CHECK_FINITE if check_finite else 0)
    ret = _lib.as_detect(_dt(A), A.data_ptr(), _ld(A), A.shape[0], fl, C.byref(st), _stream_ptr(stream))
    return ret, {k: getattr(st, k) for k, _ in st._fields_}


_dbg = None


def debug_lib():
    """libadaptsolve_debug.so (the -DAS_DEBUG build with the as_debug_* exports), loaded on demand."""
    global _dbg
    if _dbg is None:
        if not os.path.exists(DEBUG_LIB_PATH):
            raise ImportError(f"{DEBUG_LIB_PATH} not found (built with libadaptsolve.so by build())")
        d = _lib if _USE_DEBUG else C.CDLL(DEBUG_LIB_PATH)
        d.as_debug_factor.argtypes = [I32, I32, P, I64, I64, I64, I64, P, P, P]
        d.as_debug_factor.restype = I64
        d.as_debug_timestamps.argtypes = [P]
        d.as_debug_timestamps.restype = C.c_int
        d.as_debug_panel_time.argtypes = [C.c_int, C.c_int, P, C.c_int64, C.c_int64, C.c_int64, C.c_int, P, C.c_int,
                                          C.c_int]
        d.as_debug_panel_time.restype = C.c_double
        d.as_debug_lu_trace.argtypes = [P, P, C.c_int]
        d.as_debug_lu_trace.restype = C.c_int
        d.as_solve_ex.argtypes = _lib.as_solve_ex.argtypes
        d.as_solve_ex.restype = C.c_int
        d.as_set_instrumentation.argtypes = [C.c_int]
        d.as_set_exec_mode.argtypes = [C.c_int]
        _dbg = d
    return _dbg



def as_debug_factor(A, method: int, stream=None):
    """Test-only: the primary factorization alone (LU: W = L\\U and 0-based ipiv; Cholesky: L in the
    lower triangle).  Returns (info, W, ipiv) with W column-major n x n on A's device."""
    import torch
    n = A.shape[0]
    Wt = empty_colmajor(n, n, A.dtype, device=A.device)
    ipiv = torch.empty(n, dtype=torch.int64, device=A.device)
    info = debug_lib().as_debug_factor(_dt(A), method, A.data_ptr(), _ld(A), n, 0, 0, Wt.data_ptr(), ipiv.data_ptr(),
                                _stream_ptr(stream))
    return int(info), Wt, ipiv


_lib.as_set_instrumentation.argtypes = [C.c_int]
_lib.as_last_stage_ms.argtypes = [P]
_lib.as_last_stage_ms.restype = C.c_int


_lib.as_measure_fp64_peak.argtypes = [C.c_int, P]
_lib.as_measure_fp64_peak.restype = C.c_double


def measure_fp64_peak(iters: int = 20000, stream=None) -> float:
    """fp64 DMMA TFLOP/s of a register-resident loop (roofline denominator)."""
    return float(_lib.as_measure_fp64_peak(int(iters), _stream_ptr(stream)))


_lib.as_set_exec_mode.argtypes = [C.c_int]
_lib.as_bench_gemm.argtypes = [C.c_int, I64, I64, I64, C.c_int, C.c_int]
_lib.as_bench_gemm.restype = C.c_double


def bench_gemm(M, N, K, dtype_code=AS_F64, trans_b=False, iters=5) -> float:
    """TFLOP/s of the library's trailing-update GEMM kernel."""
    return float(_lib.as_bench_gemm(dtype_code, M, N, K, int(trans_b), iters))


def debug_panel_time(W, k0, nbp, kind=0, iters=5, dbg=0):
    """Average device time (us) of one panel factorization of the column-major device matrix W
    (kind 0/1: LU register / cooperative panel, 2/3: Cholesky cluster panel / POTF2 + L21)."""
    n = W.shape[0]
    Wc = W.clone()
    src = W.clone()
    return debug_lib().as_debug_panel_time(_dt(W), kind, Wc.data_ptr(), W.stride(1), n, k0, nbp, src.data_ptr(),
                                    iters, dbg)




def debug_lu_trace():
    """[(kind, block, start_us, end_us)] of the last LU factorization (AS_LU_TRACE=1), or None."""
    cap = 2048
    lo, hi = (C.c_ulonglong * cap)(), (C.c_ulonglong * cap)()
    cnt = debug_lib().as_debug_lu_trace(lo, hi, cap)
    if cnt <= 0:
        return None
    starts = [lo[i] for i in range(cnt) if lo[i] != 0xFFFFFFFFFFFFFFFF]
    if not starts:
        return None
    t0 = min(starts)
    kinds = ["gemm", "panel1", "panel2", "gemm_la"]
    out = []
    for i in range(cnt):
        if lo[i] != 0xFFFFFFFFFFFFFFFF and hi[i]:
            out.append((kinds[i % 4], i // 4, (lo[i] - t0) / 1e3, (hi[i] - t0) / 1e3))
    return out


def debug_timestamps(raw: bool = False):
    """Phase stamps (ns, %globaltimer) of the last call, relative to the first stamp."""
    out = (C.c_ulonglong * 16)()
    if debug_lib().as_debug_timestamps(out) != 0:
        return None
    v = list(out)
    if raw:
        return v
    t0 = v[0]
    return [(x - t0) / 1e3 if x else None for x in v]   # microseconds


def set_exec_mode(eager: bool) -> None:
    """eager=True: plans built afterwards launch kernels directly (profiling mode)."""
    _lib.as_set_exec_mode(1 if eager else 0)


def set_instrumentation(enable: bool) -> None:
    """Plans built afterwards record CUDA events around the solve's top-level stages."""
    _lib.as_set_instrumentation(1 if enable else 0)


def last_stage_ms():
    """Device-timed [detect, factor+estimate, gate+solve/fallback, total] ms of the last call (or None)."""
    out = (C.c_double * 4)()
    if _lib.as_last_stage_ms(out) != 0:
        return None
    return list(out)


def last_kernel_nodes() -> int:
    """Kernel launches (graph kernel nodes) the last synchronous call executed."""
    return int(_lib.as_last_kernel_nodes())


def workspace_bytes(dtype_code: int, n: int, nrhs: int, opts: int = 0) -> int:
    return int(_lib.as_workspace_bytes(dtype_code, n, nrhs, opts))


def release_all() -> None:
    _lib.as_release_all()
