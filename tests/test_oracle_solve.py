"""Pins for the oracle's factorizations, rcond estimator, SVD fallback and dispatch.

Sources of truth (never the oracle itself): the paper's/SPEC's worked values
(tests/golden/pins.json, each cited), closed forms (Hilbert inverse, diagonal
and permutation systems, C4's generated spectrum), invariants (PA = LU,
L L^T = A, orthogonality), brute force in exact rationals (n <= 8), and
independent library routines (scipy's LAPACK) for special cases.
"""
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg as sla
from scipy.linalg import lapack

import oracle
import workloads as W
from helpers import (F, backward_error, exact_cond1, exact_inverse, exact_solve, forward_diff, hilbert,
                     hilbert_inverse_exact, load_pins)

PINS = load_pins()
EPS = np.finfo(np.float64).eps


# ---------------------------------------------------------------- worked values
@pytest.mark.parametrize("case", PINS["lu_cases"])
def test_lu_pins(case):
    W_, ipiv, info = oracle.getrf(F(case["A"]))
    assert info == 0
    x = oracle.getrs(W_, ipiv, F(case["b"]).reshape(-1, 1)).ravel()
    if case.get("exact"):
        assert np.array_equal(x, np.array(case["x"], float)), case["cite"]
    else:
        assert np.allclose(x, case["x"], rtol=0, atol=4 * EPS * 10), case["cite"]


def test_lu_singular_and_minnorm():
    c = PINS["lu_singular"]
    _, _, info = oracle.getrf(F(c["A"]))
    assert info == c["singular_col"] + 1
    ret, X, rep, _ = oracle.solve(F(c["A"]), F(c["b"]))
    assert ret == 0 and rep["flags"] & oracle.F_SINGULAR and rep["flags"] & oracle.F_FALLBACK
    assert rep["method"] == oracle.M_SVD and rep["rank"] == c["rank"] and rep["rcond"] == 0.0
    assert np.allclose(X.ravel(), c["x_minnorm"], atol=1e-14)
    ret, X, rep, _ = oracle.solve(F(c["A"]), F(c["b"]), no_fallback=True)
    assert ret == oracle.ERR_SINGULAR_NO_FALLBACK


def test_cholesky_pins():
    c = PINS["chol_case"]
    L, info = oracle.potrf(F(c["A"]))
    assert info == 0 and np.array_equal(L, F(c["L"]))
    ret, X, rep, _ = oracle.solve(F(c["A"]), F(c["b"]))
    assert rep["primary_method"] == oracle.M_CHOL
    assert np.array_equal(X.ravel(), np.array(c["x"])), c["cite"]
    f = PINS["chol_fail"]
    _, info = oracle.potrf(F(f["A"]))
    assert info == f["fail_col"] + 1


def test_cholesky_failure_goes_to_lu():
    c = PINS["chol_to_lu"]
    A = F(c["A"])
    assert oracle.detect(A).flags == oracle.SPD          # passes Fig. 4
    assert np.linalg.eigvalsh(A).min() < 0               # but indefinite
    _, info = oracle.potrf(A)
    assert info == 3                                     # fails at column 2 (0-based)
    ret, X, rep, _ = oracle.solve(A, F(c["b"]))
    assert ret == 0 and rep["flags"] & oracle.F_CHOL_FAILED and rep["method"] == oracle.M_LU
    assert rep["chol_fail_col"] == 2
    xe = np.array(c["x_num"], float) / c["x_den"]
    assert np.allclose(X.ravel(), xe, rtol=0, atol=1e-14)


def test_triangular_pins():
    c = PINS["tri_case"]
    x = oracle.trsv(F(c["L"]), np.array(c["b"], float), upper=False)
    assert np.array_equal(x, np.array(c["x"], float))
    # diagonal: x_i = b_i / d_i, one IEEE division each -> bit exact
    rng = np.random.default_rng(0)
    d = rng.uniform(0.5, 2, 50)
    b = rng.standard_normal(50)
    ret, X, rep, _ = oracle.solve(np.asfortranarray(np.diag(d)), b)
    assert np.array_equal(X.ravel(), b / d)


def test_band_pins():
    c = PINS["band_case"]
    A = F(c["A"])
    ab, anorm = oracle.band_pack(A, 0, 0)
    abf, ipiv, info = oracle.gbtrf(ab, 0, 0)
    x = oracle.gbtrs(abf, 0, 0, ipiv, F(c["b"]).reshape(-1, 1)).ravel()
    assert info == 0 and np.array_equal(x, np.array(c["x"], float))
    # Fig. 1(a) packed with kl=ku=1: main-diagonal row is [1,2,3,4,5]
    from helpers import load_fig1
    ab, _ = oracle.band_pack(load_fig1()["a"], 1, 1)
    assert np.array_equal(ab[1 + 1, :], [1, 2, 3, 4, 5])      # row kl+ku
    assert np.array_equal(ab[1 + 1 - 1, 1:], [9, 8, 7, 6])    # super-diagonal row
    assert np.array_equal(ab[1 + 1 + 1, :-1], [6, 7, 8, 9])   # sub-diagonal row
    assert np.all(ab[0, :] == 0)                              # kl fill row


def test_band_tridiag_toeplitz():
    n = 100
    A = np.asfortranarray(4 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1))
    b = A @ np.ones(n)
    ret, X, rep, _ = oracle.solve(A, b)
    assert rep["method"] == oracle.M_BAND and (rep["kl"], rep["ku"]) == (1, 1)
    assert np.abs(X.ravel() - 1).max() < 1e-12


@pytest.mark.parametrize("seed", range(6))
def test_band_lu_matches_lapack_dgbtrf(seed):
    """Independent library pin: LAPACK dgbtrf on the same band (pivoting case)."""
    rng = np.random.default_rng(seed)
    n, kl, ku = 60, int(rng.integers(1, 5)), int(rng.integers(0, 4))
    A = W.random_banded(n, kl, ku, seed=seed)
    ab, _ = oracle.band_pack(A, kl, ku)
    abf, ipiv, info = oracle.gbtrf(ab, kl, ku)
    lab, lpiv, linfo = lapack.dgbtrf(ab.copy(order="F"), kl, ku)
    assert info == linfo == 0
    assert np.array_equal(ipiv, lpiv)                # identical pivot sequence
    assert np.abs(abf - lab).max() <= 1e-13 * max(1, np.abs(lab).max())
    B = np.asfortranarray(rng.standard_normal((n, 3)))
    X = oracle.gbtrs(abf, kl, ku, ipiv, B)
    XL, _ = lapack.dgbtrs(lab, kl, ku, B, lpiv)
    assert forward_diff(X, XL) <= 10 * n * EPS * np.linalg.cond(A, 1)
    XT = oracle.gbtrs(abf, kl, ku, ipiv, B, trans=True)
    assert backward_error(A.T, XT, B) < 1e-15


@pytest.mark.parametrize("seed", range(6))
def test_getrf_invariants_and_lapack(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 80))
    A = np.asfortranarray(rng.standard_normal((n, n)))
    Wf, ipiv, info = oracle.getrf(A)
    assert info == 0
    L = np.tril(Wf, -1) + np.eye(n)
    U = np.triu(Wf)
    PA = A.copy()
    for j in range(n):                           # apply the interchanges in order
        PA[[j, ipiv[j]]] = PA[[ipiv[j], j]]
    assert np.abs(PA - L @ U).max() <= n * EPS * np.abs(A).sum(axis=0).max()
    assert np.all(np.abs(L) <= 1.0)              # partial pivoting bound
    lu, piv, linfo = lapack.dgetrf(A.copy(order="F"))
    assert np.array_equal(ipiv, piv)             # same pivots as LAPACK
    assert np.abs(lu - Wf).max() <= 1e-10 * np.abs(lu).max()


@pytest.mark.parametrize("seed", range(4))
def test_potrf_invariant(seed):
    A = W.random_spd_fig3(40 + 10 * seed, seed)
    L, info = oracle.potrf(A)
    assert info == 0
    assert np.abs(L @ L.T - A).max() <= 40 * A.shape[0] * EPS * np.abs(A).max()
    Lref = np.linalg.cholesky(A)
    assert np.abs(L - Lref).max() < 1e-12


# ---------------------------------------------------------------- rcond estimator
@pytest.mark.parametrize("case", PINS["rcond_cases"])
def test_rcond_pins(case):
    ret, X, rep, _ = oracle.solve(F(case["A"]), np.ones(2))
    assert rep["rcond"] == pytest.approx(case["rcond"], rel=1e-15), case["cite"]


def test_rcond_matches_lapack_con():
    """The estimator follows xLACN2 step by step: LAPACK's xxCON must agree."""
    rng = np.random.default_rng(7)
    A = np.asfortranarray(rng.standard_normal((120, 120)))
    Wf, ipiv, _ = oracle.getrf(A)
    an = np.abs(A).sum(axis=0).max()
    r, ns = oracle.rcond(oracle.KIND_LU, Wf, an, ipiv=ipiv)
    lu, piv, _ = lapack.dgetrf(A.copy(order="F"))
    rl, _ = lapack.dgecon(lu, an, norm="1")
    assert r == pytest.approx(rl, rel=1e-12)
    U = np.asfortranarray(np.triu(A) + 10 * np.eye(120))
    an = np.abs(np.triu(U)).sum(axis=0).max()
    r, _ = oracle.rcond(oracle.KIND_TRI, U, an, upper=True)
    rl, _ = lapack.dtrcon(U, norm="1", uplo="U")
    assert r == pytest.approx(rl, rel=1e-12)
    S = W.random_spd_fig3(90, 1)
    L, _ = oracle.potrf(S)
    an = np.abs(S).sum(axis=0).max()
    r, _ = oracle.rcond(oracle.KIND_CHOL, np.asfortranarray(L), an)
    c, _ = lapack.dpotrf(S.copy(order="F"), lower=1)
    rl, _ = lapack.dpocon(c, an, uplo="L")
    assert r == pytest.approx(rl, rel=1e-12)
    Bm = W.random_banded(150, 3, 2, seed=4)
    ab, anb = oracle.band_pack(Bm, 3, 2)
    abf, bpiv, _ = oracle.gbtrf(ab, 3, 2)
    r, _ = oracle.rcond(oracle.KIND_BAND, abf, anb, kl=3, ku=2, ipiv=bpiv)
    lab, lpiv, _ = lapack.dgbtrf(ab.copy(order="F"), 3, 2)
    rl, _ = lapack.dgbcon(3, 2, lab, lpiv, anb, norm="1")
    assert r == pytest.approx(rl, rel=1e-12)


@pytest.mark.parametrize("seed", range(30))
def test_rcond_brackets_exact(seed):
    """Brute force (exact rationals): the estimate is a lower bound of ||A^-1||_1,
    so rcond_est >= rcond_exact, and within 10x of it."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 9))
    A = np.asfortranarray(rng.integers(-9, 10, (n, n)).astype(float) + np.diag(rng.integers(0, 3, n)))
    try:
        cond = exact_cond1(A.tolist())
    except ZeroDivisionError:
        pytest.skip("singular draw")
    ret, X, rep, _ = oracle.solve(A, np.ones(n), force_method=oracle.M_LU, no_fallback=True)
    if rep["flags"] & oracle.F_SINGULAR:
        pytest.skip("singular pivot")
    r_exact = float(1 / cond)
    assert rep["rcond"] >= r_exact * (1 - 1e-10)
    assert rep["rcond"] <= 10 * r_exact
    # solution vs exact rational solution within c * n * eps * cond_1
    xe = np.array([float(v) for v in exact_solve(A.tolist(), np.ones(n))])
    assert forward_diff(X, xe.reshape(-1, 1)) <= 10 * n * EPS * float(cond)


@pytest.mark.parametrize("n", [2, 5, 8, 10])
def test_hilbert_closed_form(n):
    H = hilbert(n)
    Hinv = hilbert_inverse_exact(n)
    assert all(abs(sum(Fraction(1, i + k + 1) * Hinv[k][j] for k in range(n)) - (i == j)) == 0
               for i in range(n) for j in range(n))
    b = np.ones(n)
    xe = np.array([float(sum(Hinv[i][k] for k in range(n))) for i in range(n)])
    ret, X, rep, _ = oracle.solve(H, b)
    assert rep["primary_method"] == oracle.M_CHOL and not rep["flags"] & oracle.F_FALLBACK
    cond = max(sum(abs(Hinv[i][j]) for i in range(n)) for j in range(n)) * H.sum(axis=0).max()
    assert forward_diff(X, xe.reshape(-1, 1)) <= 10 * n * EPS * cond
    assert rep["rcond"] >= 1 / cond * (1 - 1e-8)


def test_hilbert_12_falls_back():
    ret, X, rep, _ = oracle.solve(hilbert(12), np.ones(12))
    assert rep["flags"] & oracle.F_RCOND_LOW and rep["flags"] & oracle.F_FALLBACK


@pytest.mark.parametrize("seed", range(12))
def test_bruteforce_paths_exact(seed):
    """Every structured path vs exact rational solutions, n <= 8."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(4, 9))
    kind = seed % 4
    if kind == 0:
        A = np.triu(rng.integers(-5, 6, (n, n)).astype(float), 1) + np.diag(rng.integers(1, 6, n))
        want = oracle.M_TRI_UPPER
    elif kind == 1:
        A = np.tril(rng.integers(-5, 6, (n, n)).astype(float), -1) + np.diag(rng.integers(1, 6, n))
        want = oracle.M_TRI_LOWER
    elif kind == 2:
        R = rng.integers(-3, 4, (n, n)).astype(float)
        A = R.T @ R + n * 9 * np.eye(n)
        want = oracle.M_CHOL
    else:
        A = rng.integers(-5, 6, (n, n)).astype(float) + 20 * np.eye(n)
        A[0, n - 1] = A[n - 1, 0] + 1       # asymmetric, full band
        want = oracle.M_LU
    A = np.asfortranarray(A)
    b = rng.integers(-9, 10, n).astype(float)
    ret, X, rep, _ = oracle.solve(A, b)
    assert rep["primary_method"] == want
    xe = np.array([float(v) for v in exact_solve(A.tolist(), b)])
    cond = float(exact_cond1(A.tolist()))
    assert forward_diff(X, xe.reshape(-1, 1)) <= 10 * n * EPS * cond


def test_permutation_bit_exact():
    for n in (3, 8, 64):
        P = np.zeros((n, n))
        P[(np.arange(n) + 1) % n, np.arange(n)] = 1.0        # cyclic shift
        P = np.asfortranarray(P)
        d = oracle.detect(P)
        assert d.method == oracle.M_LU and (d.kl, d.ku) == (1, n - 1)
        b = np.random.default_rng(n).standard_normal(n)
        ret, X, rep, _ = oracle.solve(P, b)
        assert np.array_equal(X.ravel(), P.T @ b) and rep["rcond"] == 1.0


# ---------------------------------------------------------------- fallback / SVD
def test_fallback_gate_pin():
    c = PINS["fallback_case"]
    A = F(c["A"])
    ret, X, rep, _ = oracle.solve(A, F(c["b"]))
    assert rep["flags"] & oracle.F_RCOND_LOW and rep["flags"] & oracle.F_FALLBACK and rep["method"] == oracle.M_SVD
    assert rep["rank"] == c["rank"] and np.allclose(X.ravel(), c["x_fallback"], atol=1e-15)
    assert rep["rcond"] == pytest.approx(1e-17, rel=1e-12)     # primary (TRCON) estimate, never the SVD's
    ret, X, rep, _ = oracle.solve(A, F(c["b"]), no_fallback=True)
    assert ret == 0 and rep["flags"] & oracle.F_POORLY_COND and not rep["flags"] & oracle.F_FALLBACK
    assert np.array_equal(X.ravel(), [1.0, 1e17])              # primary solution returned


@pytest.mark.parametrize("case", PINS["svd_cases"])
def test_svd_pins(case):
    A = F(case["A"])
    n = A.shape[0]
    b = np.array(case.get("b", [1.0] * n))
    X, rank, sig, sweeps, conv = oracle.lsq_svd(A, b)
    assert conv
    assert np.allclose(sig, case["sigma"] if "sigma" in case else np.linalg.svd(A, compute_uv=False), atol=1e-15)
    if "x" in case:
        assert np.allclose(X.ravel(), case["x"], atol=1e-15) and rank == case["rank"]


@pytest.mark.parametrize("seed", range(5))
def test_svd_vs_numpy(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 60))
    A = np.asfortranarray(rng.standard_normal((n, n)))
    if seed % 2:
        U, s, Vt = np.linalg.svd(A)
        s[n // 2:] = 0.0                       # rank deficient
        A = np.asfortranarray((U * s) @ Vt)
    b = rng.standard_normal((n, 2))
    X, rank, sig, sweeps, conv = oracle.lsq_svd(A, b)
    assert conv
    s_np = np.linalg.svd(A, compute_uv=False)
    assert np.abs(sig - s_np).max() <= 1e-13 * s_np[0]
    Xp = np.linalg.pinv(A, rcond=n * EPS) @ b
    assert np.abs(X - Xp).max() <= 1e-10 * max(1, np.abs(Xp).max())
    assert rank == int((s_np > n * EPS * s_np[0]).sum())


def test_qr_and_jacobi_invariants():
    rng = np.random.default_rng(3)
    n = 40
    A = np.asfortranarray(rng.standard_normal((n, n)))
    R, Cm = oracle.geqr(A, A)                   # with B = A, Q^T A = R
    R = np.triu(R)
    assert np.abs(Cm - R).max() < 1e-13 * np.abs(A).max() * n
    assert np.abs(R.T @ R - A.T @ A).max() < 1e-12 * np.abs(A.T @ A).max()
    M, V, sweeps, conv = oracle.jacobi(np.asfortranarray(R.T))
    assert conv and sweeps < 30
    G = M.T @ M
    off = G - np.diag(np.diag(G))
    assert np.abs(off).max() <= 1e-13 * np.abs(G).max()
    assert np.abs(V.T @ V - np.eye(n)).max() < 1e-13
    assert np.abs(R.T @ V - M).max() < 1e-12 * np.abs(R).max()


def test_c4_closed_form_small():
    """C4's recipe at n=128: sigma known in closed form, rank at cut n*eps, and
    rho*(r) = ||(I - U_r U_r^T) b|| / ||b|| from the generator's U."""
    n = 128
    A, B, U, sigma, V = W.illcond_c4(n=n)
    ret, X, rep, sig = oracle.solve(A, B)
    assert rep["flags"] & oracle.F_FALLBACK and rep["method"] == oracle.M_SVD
    assert np.abs(sig - sigma).max() <= 1e-13
    rank_cf = int((sigma > n * EPS * sigma[0]).sum())
    assert abs(rep["rank"] - rank_cf) <= 1
    r = rep["rank"]
    b = B[:, 0]
    rho_star = np.linalg.norm(b - U[:, :r] @ (U[:, :r].T @ b)) / np.linalg.norm(b)
    rho = np.linalg.norm(b - A @ X[:, 0]) / np.linalg.norm(b)
    assert abs(rho - rho_star) <= 1e-2 * rho_star


def test_thread_invariance():
    A = W.random_dense(150, seed=5)
    B = np.asfortranarray(np.random.default_rng(0).standard_normal((150, 3)))
    oracle.set_threads(1)
    r1 = oracle.solve(A, B)
    oracle.set_threads(4)
    r4 = oracle.solve(A, B)
    S = W.random_spd_fig3(120, 2)
    oracle.set_threads(1)
    s1 = oracle.solve(S, B[:120])
    oracle.set_threads(4)
    s4 = oracle.solve(S, B[:120])
    assert np.array_equal(r1[1], r4[1]) and r1[2] == r4[2]
    assert np.array_equal(s1[1], s4[1])


def test_force_method_and_baselines():
    """FORCE_METHOD=LU ('standard' solver) agrees with adaptive on structured inputs."""
    for A in (W.random_banded(100, 2, 2, seed=1, dominant=True), W.random_triangular(100, False, seed=2),
              W.random_spd_fig3(100, 3)):
        b = np.ones(100)
        _, Xa, ra, _ = oracle.solve(A, b)
        _, Xg, rg, _ = oracle.solve(A, b, force_method=oracle.M_LU)
        assert rg["method"] == oracle.M_LU and ra["method"] != oracle.M_LU
        assert forward_diff(Xa, Xg) < 1e-10


def test_float32_solve():
    A, B = W.make("C1", n=64)
    A32, B32 = A.astype(np.float32, order="F"), B.astype(np.float32, order="F")
    ret, X, rep, _ = oracle.solve(A32, B32)
    assert X.dtype == np.float32 and rep["method"] == oracle.M_LU
    assert backward_error(A32, X, B32) < 1e-6
    _, X64, _, _ = oracle.solve(A32.astype(np.float64), B32.astype(np.float64))
    assert forward_diff(X, X64) < 1e-6 / rep["rcond"]


# ------------------------------------------------------------------ non-finite input (Z28/Z29)
@pytest.mark.parametrize("seed", range(8))
def test_check_finite_matches_isfinite(seed):
    """CHECK_FINITE rejects exactly the inputs numpy's isfinite() rejects (NaN, +Inf, -Inf anywhere in A
    or B); finite inputs solve bit-identically to the default path."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 40))
    A = np.asfortranarray(rng.standard_normal((n, n)) + 4 * np.eye(n))
    B = np.asfortranarray(rng.standard_normal((n, 2)))
    r0, X0, rep0, _ = oracle.solve(A, B)
    r1, X1, rep1, _ = oracle.solve(A, B, check_finite=True)
    assert r0 == r1 == 0 and np.array_equal(X0, X1) and rep0["flags"] == rep1["flags"]
    bad = [np.nan, np.inf, -np.inf][seed % 3]
    tgt = A if seed % 2 == 0 else B
    i, j = int(rng.integers(0, n)), int(rng.integers(0, tgt.shape[1]))
    A2, B2 = A.copy(order="F"), B.copy(order="F")
    (A2 if tgt is A else B2)[i, j] = bad
    assert not (np.isfinite(A2).all() and np.isfinite(B2).all())
    r, _, rep, _ = oracle.solve(A2, B2, check_finite=True)
    assert r == oracle.ERR_NONFINITE
    assert rep["flags"] & oracle.F_NONFINITE
    assert (rep["flags"] >> 4) & 0xF == 0 and rep["rcond"] == 0.0      # no method ran
    # detection verdicts are still the literal ones
    assert (rep["flags"] & 0xF) == oracle.detect(A2).flags


def test_nonfinite_reaching_svd_is_an_error():
    """Without CHECK_FINITE a NaN/Inf in A makes the rcond estimate non-finite or 0, the gate sends the
    call to the SVD, whose singular values are then non-finite: the min-norm solution is undefined
    (Z29) -> AS_ERR_NONFINITE, never a silent 'rank 0' answer."""
    for bad in (np.nan, np.inf):
        A = F([[4.0, 1.0, 0.5], [1.0, bad, 2.0], [0.5, 1.0, 3.0]])
        B = F([[1.0], [2.0], [3.0]])
        r, _, rep, _ = oracle.solve(A, B)
        assert r == oracle.ERR_NONFINITE, (bad, r, rep)
        assert rep["flags"] & oracle.F_NONFINITE and rep["flags"] & oracle.F_FALLBACK
        assert rep["rank"] == -1 and not rep["flags"] & oracle.F_RANK_DEF


@pytest.mark.parametrize("seed", range(4))
def test_band_pack_anorm_is_the_1norm(seed):
    """band_pack's band 1-norm: every non-zero of a banded matrix lies in the band, so it equals the
    plain max column sum of |A| (numpy), independent of the packing code."""
    rng = np.random.default_rng(100 + seed)
    n, kl, ku = 60 + seed, 1 + seed, 3 - seed % 3
    A = W.random_banded(n, kl, ku, seed=seed)
    A[int(rng.integers(0, n)), :] *= 7.0    # a heavy row (stays inside the band) so no column sum is typical
    _, anorm = oracle.band_pack(A, kl, ku)
    assert anorm == pytest.approx(np.abs(A).sum(axis=0).max(), rel=4 * n * 2.2e-16)


# ------------------------------------------------------------------ LDL^T, Bunch-Kaufman (Z30)
def _sym_indef(n, seed):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n))
    return np.asfortranarray((M + M.T) / 2)


@pytest.mark.parametrize("n,seed", [(1, 0), (2, 1), (5, 2), (17, 3), (40, 4), (60, 5), (60, 6)])
def test_sytrf_matches_lapack_dsytf2(n, seed):
    """For n below LAPACK's block size dsytrf is the unblocked dsytf2: the oracle's pivots must be
    LAPACK's exactly (1-based kp, negative for 2x2 blocks) and its factors equal up to rounding."""
    A = _sym_indef(n, seed)
    if n >= 5:
        A[2, 2] = 0.0                       # forces interchanges / 2x2 blocks early
    W, ipiv, info = oracle.sytrf(A)
    lu, piv, linfo = lapack.dsytrf(A, lower=1)
    assert info == linfo == 0
    lp = np.where(ipiv >= 0, ipiv + 1, ipiv)
    assert np.array_equal(lp, piv), (lp, piv)
    L = np.tril(W)
    assert np.allclose(L, np.tril(lu), rtol=1e-12, atol=1e-12 * np.abs(A).max())


@pytest.mark.parametrize("seed", range(5))
def test_sytrs_solves(seed):
    """x = A^{-1} b through the LDL^T factors equals the exact rational solution (n <= 8)."""
    rng = np.random.default_rng(40 + seed)
    n = 3 + seed
    A = rng.integers(-4, 5, (n, n)).astype(np.float64)
    A = np.asfortranarray(A + A.T)
    b = rng.integers(-5, 6, n).astype(np.float64)
    if abs(np.linalg.det(A)) < 1e-6:
        A[np.arange(n), np.arange(n)] += 7.0
    W, ipiv, info = oracle.sytrf(A)
    assert info == 0
    x = oracle.sytrs(W, ipiv, b)[:, 0]
    xe = np.array([float(v) for v in exact_solve(A, b)])
    assert np.abs(x - xe).max() <= 1e-12 * max(1.0, np.abs(xe).max())


def test_sym_indef_dispatch_and_rcond():
    """SYM_INDEF: an exactly symmetric indefinite matrix takes LDL^T (method 7, SYMMETRIC bit), its
    rcond equals LAPACK's dsycon on the same factors, the solution is the linear solve; without the
    option the paper's flowchart is unchanged (general LU); a likely-sympd matrix whose Cholesky fails
    takes LDL^T when exactly symmetric."""
    A = _sym_indef(50, 9)
    B = np.asfortranarray(np.random.default_rng(9).standard_normal((50, 2)))
    r, X, rep, _ = oracle.solve(A, B, sym_indef=True)
    assert r == 0 and rep["method"] == oracle.M_LDLT and rep["flags"] & oracle.F_SYMMETRIC
    assert np.abs(X - np.linalg.solve(A, B)).max() <= 1e-10 * np.abs(X).max()
    lu, piv, _ = lapack.dsytrf(A, lower=1)
    anorm = np.abs(A).sum(axis=0).max()
    rc, _ = lapack.dsycon(lu, piv, anorm, lower=1)
    assert rep["rcond"] == pytest.approx(rc, rel=1e-12)
    r2, _, rep2, _ = oracle.solve(A, B)
    assert rep2["method"] == oracle.M_LU and not rep2["flags"] & oracle.F_SYMMETRIC
    M = np.full((20, 20), -0.45)
    np.fill_diagonal(M, 1.0)
    r3, X3, rep3, _ = oracle.solve(np.asfortranarray(M), B[:20].copy(order="F"), sym_indef=True)
    assert rep3["flags"] & oracle.F_CHOL_FAILED and rep3["method"] == oracle.M_LDLT
    assert np.abs(M @ X3 - B[:20]).max() <= 1e-12 * np.abs(B).max() * 20
    # asymmetric by one ulp: not exactly symmetric -> LU
    A4 = A.copy(order="F")
    A4[3, 7] = np.nextafter(A4[3, 7], 10.0)
    assert oracle.solve(A4, B, sym_indef=True)[2]["method"] == oracle.M_LU
