"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (north star, readings Z18-Z21 in DESIGN.md):
  detection flags, kl/ku, method, CHOL_FAILED, SINGULAR, FALLBACK, gate bit: bit-exact;
  fp64: eta <= 1e-13 and phi <= 1e-15 cond_1 (cond_1 = anorm / rcond_oracle);
  fp32: eta <= 1e-5 and phi <= 1e-6 cond_1 against the fp64 oracle on the promoted data.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
from helpers import backward_error, forward_diff, load_fig1

pytestmark = pytest.mark.gpu

AS = pytest.importorskip("paper_2007_11208_b200") if torch.cuda.is_available() else None


def gpu_solve(A, B, **opt):
    o = AS.make_options(**opt) if opt else None
    ret, X, rep = AS.as_solve_ex(AS.to_device(A), AS.to_device(B), options=o)
    torch.cuda.synchronize()
    return ret, AS.to_host(X), rep


def oracle_opts(opt):
    return {k: v for k, v in opt.items()}


def check_parity(A, B, fp32=False, **opt):
    ret, X, rep = gpu_solve(A, B, **opt)
    oret, Xo, orep, _ = oracle.solve(A, B, **oracle_opts(opt))
    assert ret == oret, (ret, oret, rep, orep)
    # exact bits: detection verdicts, method, chol-failed, singular, gate, fallback
    mask = 0xFF | oracle.F_CHOL_FAILED | oracle.F_SINGULAR | oracle.F_RCOND_LOW | oracle.F_FALLBACK | oracle.F_POORLY_COND
    assert (rep["flags"] & mask) == (orep["flags"] & mask), (hex(rep["flags"]), hex(orep["flags"]), rep, orep)
    assert rep["method"] == orep["method"] and rep["primary_method"] == orep["primary_method"]
    if orep["kl"] >= 0:
        assert (rep["kl"], rep["ku"]) == (orep["kl"], orep["ku"])
    if ret != 0:
        return rep, orep
    # soft rcond check where the estimate is numerically meaningful (rcond >> eps)
    if orep["rcond"] > 1e-10 and rep["rcond"] > 0:
        assert abs(np.log2(rep["rcond"] / orep["rcond"])) <= 1.0, (rep["rcond"], orep["rcond"])
    if not (rep["flags"] & oracle.F_FALLBACK):
        if fp32:
            A64, B64 = A.astype(np.float64), B.astype(np.float64)
            _, Xr, rr, _ = oracle.solve(A64, B64, no_fallback=True)
            cond = rr["anorm"] / rr["rcond"]
            assert backward_error(A64, X, B64) <= 1e-5
            assert forward_diff(X, Xr) <= 1e-6 * cond
        else:
            cond = orep["anorm"] / orep["rcond"] if orep["rcond"] > 0 else np.inf
            assert backward_error(A, X, B) <= 1e-13, backward_error(A, X, B)
            assert forward_diff(X, Xo) <= 1e-15 * cond, (forward_diff(X, Xo), cond)
    return rep, orep


# ------------------------------------------------------------------ detection
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("seed", range(24))
def test_detect_random_patterns(seed, dtype):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    i, j = np.indices((n, n))
    kind = seed % 6
    if kind == 0:
        kl, ku = int(rng.integers(0, n)), int(rng.integers(0, n))
        A = np.where((i - j <= kl) & (j - i <= ku), rng.standard_normal((n, n)), 0.0)
    elif kind == 1:
        A = np.tril(rng.standard_normal((n, n)))
    elif kind == 2:
        A = np.triu(rng.standard_normal((n, n)))
    elif kind == 3:
        A = W.random_spd_fig3(n, seed)
    elif kind == 4:
        A = np.eye(n) * 3.0
        A[rng.integers(0, n), rng.integers(0, n)] = 1e-300 if dtype == np.float64 else 1e-30
    else:
        A = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.01)
        A[np.arange(n), np.arange(n)] = 5.0
    A = np.asfortranarray(A.astype(dtype))
    d = oracle.detect(A)
    for fullscan in (False, True):
        ret, st = AS.as_detect(AS.to_device(A), fullscan=fullscan)
        assert ret == 0
        assert st["flags"] == d.flags, (st, d)
        assert st["method"] == d.method
        if fullscan or d.banded:
            assert (st["kl"], st["ku"]) == (d.kl, d.ku)


def test_detect_fig1_and_edges():
    for name, M in load_fig1().items():
        d = oracle.detect(M)
        ret, st = AS.as_detect(AS.to_device(M), fullscan=True)
        assert st["flags"] == d.flags and (st["kl"], st["ku"]) == (d.kl, d.ku), name
    # -0.0 and NaN corners, lda padding
    n = 130
    A = np.eye(n)
    A[0, n - 1] = -0.0
    A[n - 1, 0] = np.nan
    big = np.full((n + 3, n), 9.0, order="F")
    big[:n] = A
    import torch as T
    tA = AS.to_device(big)[:n]
    ret, st = AS.as_detect(tA, fullscan=True)
    d = oracle.detect(np.asfortranarray(A))
    assert st["flags"] == d.flags and (st["kl"], st["ku"]) == (d.kl, d.ku)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", ["asym", "asym_small_rel", "asym_tiny_abs", "maxdiag", "diag_sum", "none"])
def test_detect_fig4_interior_pair(case, dtype):
    # Fig. 4 lines 12-16 decided on one element pair inside an interior below-diagonal tile pair
    # (rows 192..255, cols 64..127 of n = 300): the kernel's index-check-free path must agree
    # with the oracle on each condition, including the two halves of lines 13-14.
    n, i, j = 300, 200, 70
    A = np.diag(np.full(n, 10.0))
    a = b = 0.5
    if case == "asym":
        b = 0.5 * (1 + 1e-3)                           # delta > tol and > tol m: dies
    elif case == "asym_small_rel":
        a = 1e3                                        # one ulp apart: delta > tol, < tol m: alive
        b = float(np.nextafter(dtype(a), dtype(np.inf)))
        A[i, i] = A[j, j] = 1e4
    elif case == "asym_tiny_abs":
        a, b = 1e-20, 2e-20                            # delta < tol: alive
    elif case == "maxdiag":
        a = b = 10.0                                   # |a| >= max diag: dies
    elif case == "diag_sum":
        A[i, i] = A[j, j] = 1.0
        a = b = 1.0                                    # |a| + |b| >= d_i + d_j: dies
    A[i, j], A[j, i] = a, b
    A = np.asfortranarray(A.astype(dtype))
    d = oracle.detect(A)
    for fullscan in (False, True):
        ret, st = AS.as_detect(AS.to_device(A), fullscan=fullscan)
        assert ret == 0
        assert st["flags"] == d.flags, (case, st, d)
    if case in ("none", "asym_tiny_abs", "asym_small_rel"):
        assert d.flags & oracle.SPD
    else:
        assert not d.flags & oracle.SPD


@pytest.mark.parametrize("tag", ["C1", "C2", "C3a", "C3b", "C4"])
def test_detect_configs_full_size(tag):
    A, _ = W.make(tag)
    d = oracle.detect(A)
    ret, st = AS.as_detect(AS.to_device(A))
    assert st["flags"] == d.flags and st["method"] == d.method
    if d.banded:
        assert (st["kl"], st["ku"]) == (d.kl, d.ku)


# ------------------------------------------------------------------ solves, small sizes spanning tiles
@pytest.mark.parametrize("n", [1, 2, 3, 17, 64, 65, 200, 333, 700, 1100])
def test_lu_dense(n):
    A = W.random_dense(n, seed=n, shift=2.0)
    B = np.asfortranarray(np.random.default_rng(n).standard_normal((n, 3)))
    check_parity(A, B)


@pytest.mark.parametrize("n", [63, 128, 129, 191, 192, 255, 256])
@pytest.mark.parametrize("fp32", [False, True])
def test_lu_small_cluster(n, fp32):
    """n <= 256 takes the one-cluster LU (64 columns per CTA, rows in registers): every CTA-count
    boundary and ragged last block, no diagonal shift (real pivoting), fp64 and fp32."""
    A = W.random_dense(n, seed=100 + n)
    B = np.asfortranarray(np.random.default_rng(n).standard_normal((n, 2)))
    if fp32:
        check_parity(A.astype(np.float32, order="F"), B.astype(np.float32, order="F"), fp32=True)
    else:
        rep, _ = check_parity(A, B)
        assert rep["primary_method"] == oracle.M_LU


@pytest.mark.parametrize("n,zcol", [(200, 70), (256, 255), (130, 0)])
def test_lu_small_zero_pivot(n, zcol):
    """An exactly zero column gives an exact zero pivot (singular): SINGULAR and the
    SVD fallback bit-exact against the oracle; with NO_FALLBACK the singular error code."""
    A = W.random_dense(n, seed=7 + n)
    A[:, zcol] = 0.0
    B = np.asfortranarray(np.random.default_rng(n).standard_normal((n, 1)))
    rep, orep = check_parity(A, B)
    assert rep["flags"] & oracle.F_SINGULAR
    check_parity(A, B, no_fallback=True)


def test_lu_small_ties():
    """Entries in {-1, 0, 1}: many exactly tied pivot candidates (first-max rule, Z15)."""
    n = 250
    A = np.asfortranarray(np.random.default_rng(11).integers(-1, 2, (n, n)).astype(np.float64))
    A[np.arange(n), np.arange(n)] += 0.5
    B = np.asfortranarray(np.random.default_rng(12).standard_normal((n, 3)))
    check_parity(A, B)


@pytest.mark.parametrize("n,kl,ku", [(40, 1, 1), (300, 3, 2), (257, 8, 8), (500, 0, 5), (500, 6, 0), (1000, 20, 3), (300, 30, 25), (3000, 2, 2)])
def test_banded(n, kl, ku):
    A = W.random_banded(n, kl, ku, seed=n + kl, dominant=(kl + ku) % 2 == 0)
    B = np.asfortranarray(np.random.default_rng(1).standard_normal((n, 2)))
    rep, orep = check_parity(A, B)
    assert rep["primary_method"] == oracle.M_BAND


@pytest.mark.parametrize("n,kl,ku,nrhs", [(256, 1, 1, 1), (777, 8, 8, 4), (1000, 16, 1, 3), (1500, 2, 7, 2),
                                          (3001, 4, 4, 33), (8192, 8, 8, 4)])
def test_banded_partitioned(n, kl, ku, nrhs):
    """Strictly diagonally dominant bands take the partitioned (SPIKE) path: C2 recipe."""
    A, B = W.make("C2", n=n, kl=kl, ku=ku, nrhs=nrhs)
    rep, orep = check_parity(A, B)
    assert rep["primary_method"] == oracle.M_BAND and (rep["kl"], rep["ku"]) == (kl, ku)
    A32, B32 = A.astype(np.float32, order="F"), B.astype(np.float32, order="F")
    if n <= 3001:
        check_parity(A32, B32, fp32=True)


@pytest.mark.parametrize("n", [5, 64, 129, 300])
@pytest.mark.parametrize("upper", [False, True])
def test_triangular(n, upper):
    A = W.random_triangular(n, upper, seed=n)
    B = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 5)))
    rep, _ = check_parity(A, B)
    assert rep["primary_method"] == (oracle.M_TRI_UPPER if upper else oracle.M_TRI_LOWER)


@pytest.mark.parametrize("n", [4, 63, 64, 150, 257, 1000, 2100])
def test_spd(n):
    A = W.random_spd_fig3(n, seed=n)
    B = np.asfortranarray(np.random.default_rng(3).standard_normal((n, 4)))
    rep, _ = check_parity(A, B)
    assert rep["primary_method"] == oracle.M_CHOL


def test_chol_fail_to_lu():
    A = np.asfortranarray(np.array([[1, .9, .9], [.9, 1, -.9], [.9, -.9, 1]]))
    rep, _ = check_parity(A, np.asfortranarray(np.array([[1.0], [2.0], [3.0]])))
    assert rep["flags"] & oracle.F_CHOL_FAILED and rep["chol_fail_col"] == 2
    # larger: symmetric indefinite that passes Fig. 4
    n = 100
    rng = np.random.default_rng(5)
    S = rng.uniform(-0.5, 0.5, (n, n))
    S = (S + S.T) / 2
    S[np.arange(n), np.arange(n)] = 1.0
    S[np.abs(S) >= 1] = 0.4
    A = np.asfortranarray(S)
    if oracle.detect(A).spd:
        check_parity(A, np.asfortranarray(rng.standard_normal((n, 2))))


def test_singular_fallback_and_no_fallback():
    A = np.asfortranarray(np.array([[1.0, 2.0], [2.0, 4.0]]))
    B = np.asfortranarray(np.array([[3.0], [6.0]]))
    ret, X, rep = gpu_solve(A, B)
    assert ret == 0 and rep["method"] == oracle.M_SVD and rep["rank"] == 1
    assert np.allclose(X.ravel(), [0.6, 1.2], atol=1e-14)
    ret, X, rep = gpu_solve(A, B, no_fallback=True)
    assert ret == oracle.ERR_SINGULAR_NO_FALLBACK


def test_diag_gate_pin():
    A = np.asfortranarray(np.diag([1.0, 1e-17]))
    B = np.asfortranarray(np.ones((2, 1)))
    ret, X, rep = gpu_solve(A, B)
    assert rep["flags"] & oracle.F_FALLBACK and rep["rank"] == 1 and np.allclose(X.ravel(), [1, 0])
    ret, X, rep = gpu_solve(A, B, no_fallback=True)
    assert ret == 0 and rep["flags"] & oracle.F_POORLY_COND and np.array_equal(X.ravel(), [1.0, 1e17])


@pytest.mark.parametrize("n", [64, 200])
def test_illcond_fallback_small(n):
    A, B, U, sigma, V = W.illcond_c4(n=n)
    ret, X, rep = gpu_solve(A, B)
    oret, Xo, orep, sig_o = oracle.solve(A, B)
    assert rep["flags"] & oracle.F_FALLBACK and orep["flags"] & oracle.F_FALLBACK
    assert abs(rep["rank"] - orep["rank"]) <= 1
    rho = np.linalg.norm(B - A @ X) / np.linalg.norm(B)
    rho_o = np.linalg.norm(B - A @ Xo) / np.linalg.norm(B)
    assert abs(rho - rho_o) <= 1e-2 * rho_o


@pytest.mark.parametrize("method", [oracle.M_LU, oracle.M_CHOL, oracle.M_BAND])
def test_force_method(method):
    A = W.random_banded(120, 2, 2, seed=4, dominant=True)
    A = np.asfortranarray((A + A.T) / 2)
    B = np.asfortranarray(np.ones((120, 1)))
    rep, _ = check_parity(A, B, force_method=method)
    assert rep["primary_method"] == method


@pytest.mark.parametrize("method", [oracle.M_LU, oracle.M_CHOL, oracle.M_TRI_LOWER])
def test_skip_detect_standard_solver(method):
    """AS_OPT_SKIP_DETECT (the paper's "standard solver"): no detection verdicts, the forced
    method's X matches the oracle's forced solve; illegal without FORCE_METHOD or with BAND."""
    A = W.random_triangular(150, False, seed=3) if method == oracle.M_TRI_LOWER else W.random_spd_fig3(150, seed=3)
    B = np.asfortranarray(np.random.default_rng(3).standard_normal((150, 2)))
    o = AS.make_options(force_method=method, skip_detect=True)
    ret, X, rep = AS.as_solve_ex(AS.to_device(A), AS.to_device(B), options=o)
    torch.cuda.synchronize()
    assert ret == 0 and rep["primary_method"] == method and (rep["flags"] & 0xF) == 0
    oret, Xo, orep, _ = oracle.solve(A, B, force_method=method)
    assert oret == 0
    Xg = AS.to_host(X)
    assert backward_error(A, Xg, B) <= 1e-13
    assert forward_diff(Xg, Xo) <= 1e-15 * orep["anorm"] / orep["rcond"]
    bad = AS.make_options(skip_detect=True)
    assert AS.as_solve_ex(AS.to_device(A), AS.to_device(B), options=bad)[0] == -9
    bad = AS.make_options(force_method=oracle.M_BAND, skip_detect=True)
    assert AS.as_solve_ex(AS.to_device(A), AS.to_device(B), options=bad)[0] == -9


def test_fp32_paths():
    for A, B in [W.make("C1", n=200), W.make("C2", n=300, nrhs=2), W.make("C3a", n=130, nrhs=3),
                 W.make("C3b", n=150, nrhs=3)]:
        check_parity(A.astype(np.float32, order="F"), B.astype(np.float32, order="F"), fp32=True)


def test_inplace_alias():
    A, B = W.make("C1", n=100)
    tA, tB = AS.to_device(A), AS.to_device(B)
    ret, X, rep = AS.as_solve_ex(tA, tB, X=tB)
    torch.cuda.synchronize()
    _, Xo, _, _ = oracle.solve(A, B)
    assert forward_diff(AS.to_host(tB), Xo) < 1e-12


def test_host_entry_point():
    A, B = W.make("C1", n=150)
    ret, X, rep = AS.as_solve_host(A, B)
    _, Xo, orep, _ = oracle.solve(A, B)
    assert ret == 0 and rep["method"] == orep["method"]
    assert forward_diff(X, Xo) <= 1e-15 * orep["anorm"] / orep["rcond"]


def test_empty_and_illegal():
    e = torch.empty((0, 0), dtype=torch.float64, device="cuda")
    ret, X, rep = AS.as_solve_ex(e, e, X=e)
    assert ret == 0 and rep["rcond"] == 1.0
    A = AS.to_device(np.eye(3))
    import ctypes as C
    ret = AS.lib().as_solve(0, A.data_ptr(), 2, 3, A.data_ptr(), 3, 1, A.data_ptr(), None, None, None)
    assert ret == -3
    hostA = np.eye(3)
    ret = AS.lib().as_solve(0, hostA.ctypes.data, 3, 3, A.data_ptr(), 3, 1, A.data_ptr(), None, None, None)
    assert ret == -2


# ------------------------------------------------------------------ BASELINE configs at full size
@pytest.mark.parametrize("tag", ["C1", "C2", "C3a", "C3b"])
def test_config_full_size_parity(tag):
    """Full-size configs the oracle finishes in seconds: element-wise parity with the oracle."""
    A, B = W.make(tag)
    rep, orep = check_parity(A, B)
    expect = {"C1": oracle.M_LU, "C2": oracle.M_BAND, "C3a": oracle.M_CHOL, "C3b": oracle.M_TRI_UPPER}[tag]
    assert rep["method"] == expect


# C4 / C5 / C5f at full size: tests/test_gpu_r02.py (graded against committed oracle references)


# ------------------------------------------------------------------ T3: factor reconstruction (as_debug_factor)
def _perm_from_ipiv(ipiv):
    perm = np.arange(len(ipiv))
    for j, p in enumerate(ipiv):
        perm[[j, p]] = perm[[p, j]]
    return perm


@pytest.mark.parametrize("n", [1, 5, 64, 200, 256, 257, 700])
@pytest.mark.parametrize("fp32", [False, True])
def test_debug_factor_lu_reconstruction(n, fp32):
    """P A = L U from the GPU factors (xGETRF): both LU paths (one-cluster n <= 256, blocked
    above), |L| <= 1 (partial pivoting), first pivot equal to the oracle's (exact first-max rule, Z15),
    and the oracle's factors reconstruct to the same bound."""
    A = W.random_dense(n, seed=300 + n)
    if fp32:
        A = A.astype(np.float32, order="F")
    eps = np.finfo(A.dtype).eps
    info, Wd, ipiv = AS.as_debug_factor(AS.to_device(A), oracle.M_LU)
    torch.cuda.synchronize()
    assert info == 0
    F = AS.to_host(Wd).astype(np.float64)
    piv = ipiv.cpu().numpy()
    assert np.all((piv >= np.arange(n)) & (piv < n))
    L = np.tril(F, -1) + np.eye(n)
    U = np.triu(F)
    A64 = A.astype(np.float64)
    R = A64[_perm_from_ipiv(piv)] - L @ U
    bound = 4 * n * eps * np.abs(A64).max() * max(1.0, np.abs(U).max() / np.abs(A64).max())
    assert np.abs(R).max() <= 10 * bound, (np.abs(R).max(), bound)
    assert np.abs(L).max() <= 1.0
    Wo, ipo, oinfo = oracle.getrf(A)
    assert oinfo == 0 and piv[0] == ipo[0]
    assert (piv == ipo).mean() >= 0.95


def test_debug_factor_lu_zero_column():
    """An exactly zero column j: info = j + 1 (first zero pivot), as the oracle's getrf."""
    n = 150
    A = W.random_dense(n, seed=9)
    A[:, 40] = 0.0
    info, _, _ = AS.as_debug_factor(AS.to_device(A), oracle.M_LU)
    _, _, oinfo = oracle.getrf(A)
    assert info == oinfo == 41


@pytest.mark.parametrize("n", [3, 64, 300, 1000])
def test_debug_factor_cholesky_reconstruction(n):
    """L L^T = A from the GPU Cholesky factor (xPOTRF) and the non-positive-pivot column of an
    indefinite matrix equal to the oracle's."""
    A = W.random_spd_fig3(n, seed=n)
    info, Wd, _ = AS.as_debug_factor(AS.to_device(A), oracle.M_CHOL)
    torch.cuda.synchronize()
    assert info == 0
    L = np.tril(AS.to_host(Wd))
    eps = np.finfo(np.float64).eps
    assert np.abs(L @ L.T - A).max() <= 8 * n * eps * np.abs(A).max()
    Lo, oinfo = oracle.potrf(A)
    assert oinfo == 0 and np.abs(L - Lo).max() <= 1e3 * n * eps * np.abs(Lo).max()
    B = A.copy(order="F")
    B[n // 2, n // 2] = -1.0
    info, _, _ = AS.as_debug_factor(AS.to_device(B), oracle.M_CHOL)
    _, oinfo = oracle.potrf(B)
    assert info == oinfo and info > 0


@pytest.mark.parametrize("n", [200, 300])
def test_lu_padded_lda(n):
    """lda > n (a row-padded view): both LU paths read A through lda and W through its own ld."""
    A = W.random_dense(n, seed=40 + n)
    B = np.asfortranarray(np.random.default_rng(n).standard_normal((n, 2)))
    big = np.full((n + 5, n), 7.0, order="F")
    big[:n] = A
    dA = AS.to_device(big)[:n]
    assert dA.stride(1) == n + 5
    ret, X, rep = AS.as_solve_ex(dA, AS.to_device(B))
    torch.cuda.synchronize()
    assert ret == 0 and rep["primary_method"] == oracle.M_LU
    _, Xo, orep, _ = oracle.solve(A, B)
    Xg = AS.to_host(X)
    assert backward_error(A, Xg, B) <= 1e-13
    assert forward_diff(Xg, Xo) <= 1e-15 * orep["anorm"] / orep["rcond"]
