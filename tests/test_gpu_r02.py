"""GPU parity, round 2: the LU paths the large configs really take, full-size references for
C4 / C5 / C5f (committed oracle results, tools/oracle_refs.py), non-finite input, the 25% rule on
two far extents, and the Jacobi sweep cap.

Bars as in test_gpu_parity.py (north star, Z18-Z21, Z28-Z29)."""
import os

import numpy as np
import pytest
import torch

import oracle
import workloads as W
from helpers import backward_error, forward_diff
from test_gpu_parity import check_parity, gpu_solve

pytestmark = pytest.mark.gpu

AS = pytest.importorskip("paper_2007_11208_b200") if torch.cuda.is_available() else None
REFS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "refs")
MASK = 0xFF | oracle.F_CHOL_FAILED | oracle.F_SINGULAR | oracle.F_RCOND_LOW | oracle.F_FALLBACK | \
    oracle.F_POORLY_COND | oracle.F_NONFINITE | oracle.F_SVD_NOCONV


def _ref(tag):
    p = os.path.join(REFS, f"{tag}.npz")
    if not os.path.exists(p):
        pytest.fail(f"missing {p}: run tools/oracle_refs.py {tag}")
    return np.load(p)


# ------------------------------------------------------------------ LU: cooperative panel + look-ahead sizes
@pytest.mark.parametrize("n,nrhs", [(1600, 8), (2048, 17), (3000, 33), (4096, 32)])
@pytest.mark.parametrize("fp32", [False, True])
def test_lu_mid_sizes_vs_oracle(n, nrhs, fp32):
    """n > 1536 runs the cooperative panel (lu.cu) and n >= 2048 the look-ahead stream: graded
    element-wise against the oracle (phi <= 1e-15 cond_1, fp32: 1e-6 cond_1 vs the fp64 oracle on
    the promoted data), plus the gate bit."""
    A, B = W.make("C5", n=n, nrhs=nrhs, seed=n)
    if fp32:
        A, B = np.asfortranarray(A.astype(np.float32)), np.asfortranarray(B.astype(np.float32))
    rep, orep = check_parity(A, B, fp32=fp32, no_fallback=True)
    assert rep["primary_method"] == oracle.M_LU


# ------------------------------------------------------------------ full-size configs against committed references
def test_config_c5_full_size_vs_oracle():
    """C5 (n=16384, 32 RHS): X against the oracle's X (computed once per input hash by
    tools/oracle_refs.py, which calls only oracle/): eta <= 1e-13, phi <= 1e-15 cond_1, flags."""
    ref = _ref("C5")
    A, B = W.make("C5")
    assert W.sha256(A, B) == str(ref["sha256"])
    ret, X, rep = gpu_solve(A, B)
    assert ret == int(ref["ret"]) == 0
    assert (rep["flags"] & MASK) == (int(ref["flags"]) & MASK), (hex(rep["flags"]), hex(int(ref["flags"])))
    assert rep["method"] == int(ref["method"]) == oracle.M_LU
    cond = float(ref["anorm"]) / float(ref["rcond"])
    assert abs(np.log2(rep["rcond"] / float(ref["rcond"]))) <= 1.0
    assert backward_error(A, X, B) <= 1e-13
    assert forward_diff(X, ref["X"]) <= 1e-15 * cond, (forward_diff(X, ref["X"]), cond)


def test_config_c5f_full_size_vs_oracle():
    """C5f (C5 rounded to fp32, NO_FALLBACK, Z21): gate-bit parity with the fp32 oracle unless either
    rcond is within 10% of the threshold; X against the fp64 oracle on the promoted data:
    eta <= 1e-5, phi <= 1e-6 cond_1."""
    ref = _ref("C5f")
    A, B = W.make("C5f")
    assert W.sha256(A, B) == str(ref["sha256"])
    ret, X, rep = gpu_solve(A, B, no_fallback=True)
    assert ret == 0 == int(ref["ret32"])
    assert (rep["flags"] & 0xFF) == (int(ref["flags32"]) & 0xFF)
    thr = 2.0 ** -24
    knife = any(abs(r / thr - 1.0) <= 0.1 for r in (rep["rcond"], float(ref["rcond32"])))
    if not knife:
        assert (rep["flags"] & oracle.F_RCOND_LOW) == (int(ref["flags32"]) & oracle.F_RCOND_LOW)
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    cond = float(ref["anorm"]) / float(ref["rcond"])
    assert backward_error(A64, X, B64) <= 1e-5
    assert forward_diff(X, ref["X"]) <= 1e-6 * cond


def test_config_c4_full_size_vs_oracle():
    """C4 (n=1024): gate + fallback bits, singular values against the oracle's (same A, so the
    rounding of A's formation cancels) and against the closed form (both <= 1e-13), rank = oracle's
    +-1, residual rho within 1% of the oracle's.  The oracle runs here
    (seconds): C4's Haar factors come from a LAPACK QR whose rounding differs between machines, so the
    input bytes (and a stored reference) are not portable."""
    n = 1024
    A, B, U, sigma, V = W.illcond_c4(n=n)
    oret, Xo, orep, osig = oracle.solve(A, B)
    ref = {"ret": oret, "flags": orep["flags"], "sigma": osig, "rank": orep["rank"], "X": Xo}
    sig = torch.zeros(n, dtype=torch.float64, device="cuda")
    ret, Xd, rep = AS.as_solve_ex(AS.to_device(A), AS.to_device(B), sigma_out=sig)
    torch.cuda.synchronize()
    X = AS.to_host(Xd)
    assert ret == int(ref["ret"]) == 0
    assert (rep["flags"] & MASK) == (int(ref["flags"]) & MASK)
    assert rep["method"] == oracle.M_SVD and rep["primary_method"] == oracle.M_LU
    s = sig.cpu().numpy()
    assert np.abs(s - ref["sigma"]).max() <= 1e-13, np.abs(s - ref["sigma"]).max()
    assert np.abs(s - sigma).max() <= 1e-13, np.abs(s - sigma).max()
    assert abs(rep["rank"] - int(ref["rank"])) <= 1
    b = B[:, 0]
    rho = np.linalg.norm(b - A @ X[:, 0]) / np.linalg.norm(b)
    rho_or = np.linalg.norm(b - A @ ref["X"][:, 0]) / np.linalg.norm(b)
    assert abs(rho - rho_or) <= 1e-2 * rho_or, (rho, rho_or)


def test_svd_sweep_cap_not_converged():
    """max_sweeps = 1 on an ill-conditioned system: both sides report SVD_NOT_CONVERGED (+2) after
    exactly one sweep (the cap of Z16)."""
    A, B, *_ = W.illcond_c4(n=96)
    ret, X, rep = gpu_solve(A, B, max_sweeps=1)
    oret, Xo, orep, _ = oracle.solve(A, B, max_sweeps=1)
    assert ret == oret == oracle.ERR_SVD_NOT_CONVERGED
    assert (rep["flags"] & MASK) == (orep["flags"] & MASK)
    assert rep["flags"] & oracle.F_SVD_NOCONV and rep["sweeps"] == orep["sweeps"] == 1


# ------------------------------------------------------------------ non-finite input (Z28, Z29)
@pytest.mark.parametrize("where", ["A", "B"])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
@pytest.mark.parametrize("fp32", [False, True])
def test_check_finite(where, bad, fp32):
    for n, i, j in ((40, 7, 31), (300, 299, 0), (300, 150, 151)):
        A, B = W.make("C1", n=n, nrhs=2, seed=n)
        if fp32:
            A, B = np.asfortranarray(A.astype(np.float32)), np.asfortranarray(B.astype(np.float32))
        (A if where == "A" else B)[i, j % B.shape[1] if where == "B" else j] = bad
        ret, _, rep = gpu_solve(A, B, check_finite=True)
        oret, _, orep, _ = oracle.solve(A, B, check_finite=True)
        assert ret == oret == AS.ERR_NONFINITE
        assert (rep["flags"] & MASK) == (orep["flags"] & MASK), (hex(rep["flags"]), hex(orep["flags"]))
        assert rep["method"] == 0
        if where == "A":
            _, st = AS.as_detect(AS.to_device(A), check_finite=True)
            assert st["nonfinite_seen"] == 1


def test_check_finite_clean_input_unchanged():
    """A finite input solves identically with and without CHECK_FINITE (same flags, same X bits)."""
    for tag, kw in (("C1", {}), ("C2", dict(n=2000, nrhs=2)), ("C3a", dict(n=300, nrhs=3))):
        A, B = W.make(tag, **kw)
        r0, X0, rep0 = gpu_solve(A, B)
        r1, X1, rep1 = gpu_solve(A, B, check_finite=True)
        assert r0 == r1 == 0 and rep0["flags"] == rep1["flags"]
        assert np.array_equal(X0, X1)
        _, st = AS.as_detect(AS.to_device(A), check_finite=True)
        assert st["nonfinite_seen"] == 0


@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_nonfinite_reaching_svd(bad):
    A = np.asfortranarray(np.array([[4.0, 1.0, 0.5], [1.0, bad, 2.0], [0.5, 1.0, 3.0]]))
    B = np.asfortranarray(np.array([[1.0], [2.0], [3.0]]))
    ret, _, rep = gpu_solve(A, B)
    oret, _, orep, _ = oracle.solve(A, B)
    assert ret == oret == AS.ERR_NONFINITE
    assert (rep["flags"] & MASK) == (orep["flags"] & MASK)
    assert rep["rank"] == orep["rank"] == -1


# ------------------------------------------------------------------ 25% rule on extents raised by different tile pairs
@pytest.mark.parametrize("n,far", [(1024, (300, 20, 10, 210)), (2000, (1500, 1000, 0, 400)), (700, (600, 450, 5, 105))])
def test_density_two_far_extents(n, far):
    """A lone far sub-diagonal and a lone far super-diagonal element in different tile pairs: each
    extent alone passes the 25% rule, together they do not (Z2/Z3) -> not banded."""
    i1, j1, i2, j2 = far
    A = np.asfortranarray(np.eye(n) * 3.0)
    A[i1, j1] = 0.5
    A[i2, j2] = 0.25
    d = oracle.detect(A)
    assert not d.banded and d.kl == max(i1 - j1, 0) and d.ku == max(j2 - i2, 0)
    for fullscan in (False, True):
        _, st = AS.as_detect(AS.to_device(A), fullscan=fullscan)
        assert st["flags"] == d.flags, (st, d.flags)
    B = np.asfortranarray(np.ones((n, 1)))
    check_parity(A, B)


# ------------------------------------------------------------------ the leaf panel (m > 1536 rows, lu.cu)
@pytest.mark.parametrize("n,zcol", [(2000, 50), (2000, 1000), (1700, 0)])
def test_lu_leaf_panel_zero_pivot(n, zcol):
    """An exactly zero column inside a tall (leaf-panel) block: SINGULAR at the same column as the
    oracle, fallback bits exact; NO_FALLBACK gives the singular error code."""
    A = W.random_dense(n, seed=17 + n + zcol)
    A[:, zcol] = 0.0
    B = np.asfortranarray(np.random.default_rng(n).standard_normal((n, 1)))
    rep, orep = check_parity(A, B)
    assert rep["flags"] & oracle.F_SINGULAR and rep["info"] == orep["info"] == zcol + 1
    check_parity(A, B, no_fallback=True)


def test_lu_leaf_panel_ties():
    """Entries in {-1, 0, 1} at n = 1800: exactly tied pivot candidates across CTAs and leaves; the
    first-max rule on positions (Z15) must give the oracle's pivots, hence its solution."""
    n = 1800
    A = np.asfortranarray(np.random.default_rng(21).integers(-1, 2, (n, n)).astype(np.float64))
    A[np.arange(n), np.arange(n)] += 0.5
    B = np.asfortranarray(np.random.default_rng(22).standard_normal((n, 2)))
    check_parity(A, B)
    info, Wd, ipiv = AS.as_debug_factor(AS.to_device(A), oracle.M_LU)
    torch.cuda.synchronize()
    Wo, ipo, oinfo = oracle.getrf(A)
    piv = ipiv.cpu().numpy()
    # ties are decided exactly; the first divergence (if any) can only come from rounding later on
    assert (piv[:64] == ipo[:64]).all()


@pytest.mark.parametrize("n", [1600, 3000])
@pytest.mark.parametrize("fp32", [False, True])
def test_lu_leaf_panel_reconstruction(n, fp32):
    """P A = L U from the GPU factors at sizes whose first blocks take the leaf panel: |L| <= 1,
    backward error of the factorization, pivots equal to the oracle's (random data: no near ties)."""
    A = W.random_dense(n, seed=500 + n)
    if fp32:
        A = A.astype(np.float32, order="F")
    eps = np.finfo(A.dtype).eps
    info, Wd, ipiv = AS.as_debug_factor(AS.to_device(A), oracle.M_LU)
    torch.cuda.synchronize()
    assert info == 0
    F = AS.to_host(Wd).astype(np.float64)
    piv = ipiv.cpu().numpy()
    L = np.tril(F, -1) + np.eye(n)
    U = np.triu(F)
    A64 = A.astype(np.float64)
    perm = np.arange(n)
    for j, p in enumerate(piv):
        perm[[j, p]] = perm[[p, j]]
    R = A64[perm] - L @ U
    bound = 4 * n * eps * np.abs(A64).max() * max(1.0, np.abs(U).max() / np.abs(A64).max())
    assert np.abs(R).max() <= 10 * bound, (np.abs(R).max(), bound)
    assert np.abs(L).max() <= 1.0
    Wo, ipo, oinfo = oracle.getrf(A)
    # fp32 at n = 3000: near-ties of rounding-different candidates diverge early (both valid partial
    # pivoting); fp64 random data has none
    assert oinfo == 0 and piv[0] == ipo[0] and (fp32 or (piv == ipo).mean() >= 0.95)


# ------------------------------------------------------------------ narrow bands: the register chain (band_chain.cu)
@pytest.mark.parametrize("n,kl,ku", [(100, 2, 2), (250, 2, 2), (500, 2, 2), (1000, 2, 2), (3000, 2, 2), (40, 1, 1),
                                     (2000, 1, 1), (777, 3, 1), (1500, 0, 3), (1500, 3, 0), (600, 1, 2), (5000, 3, 3),
                                     (64, 0, 0)])
@pytest.mark.parametrize("fp32", [False, True])
def test_narrow_band_chain(n, kl, ku, fp32):
    """Non-dominant bands with kl, ku <= 3 (the paper's random 5-diagonal Table 1 class, tridiagonals):
    partial pivoting happens (N(0,1) entries), graded against the oracle's xGBTRF/xGBCON/xGBTRS."""
    A = W.random_banded(n, kl, ku, seed=n + 10 * kl + ku)
    # N(0,1) bands plus a diagonal shift of 1.5: rows are not all dominant (partial pivoting happens),
    # yet the condition stays moderate (a bare random triangular band is exponentially ill-conditioned:
    # its LU underflows and the gate decides on rounding)
    A[np.arange(n), np.arange(n)] += 1.5 * np.sign(A[np.arange(n), np.arange(n)] + 1e-300)
    if kl == ku == 0:
        A = np.asfortranarray(np.diag(np.random.default_rng(n).standard_normal(n) + 3.0))
    B = np.asfortranarray(np.random.default_rng(n).standard_normal((n, 3)))
    if fp32:
        A, B = np.asfortranarray(A.astype(np.float32)), np.asfortranarray(B.astype(np.float32))
    rep, orep = check_parity(A, B, fp32=fp32)
    if n >= 64:
        assert rep["primary_method"] == oracle.M_BAND


def test_narrow_band_chain_pivots_and_singular():
    """A tridiagonal that needs an interchange at every step (|sub| > |diag|), one with an exact zero
    pivot (singular -> fallback bits), 40 right-hand sides (more than one per lane)."""
    n = 1200
    rng = np.random.default_rng(5)
    A = np.zeros((n, n))
    i = np.arange(n)
    A[i, i] = 0.1 * rng.standard_normal(n)
    A[i[1:], i[:-1]] = 1.0 + rng.random(n - 1)
    A[i[:-1], i[1:]] = rng.standard_normal(n - 1)
    A = np.asfortranarray(A)
    B = np.asfortranarray(rng.standard_normal((n, 40)))
    check_parity(A, B)
    A2 = A.copy(order="F")
    A2[:, 600] = 0.0
    A2[600, :] = 0.0
    rep, orep = check_parity(A2, B[:, :2].copy(order="F"))
    assert rep["flags"] & oracle.F_SINGULAR


# ------------------------------------------------------------------ race evidence (compute-sanitizer is closed on this pool)
@pytest.mark.parametrize("case", ["lu_leaf", "lu_coop", "lu_cluster", "upper", "spd", "band_spike", "band_chain", "svd"])
def test_repeat_bitwise_deterministic(case):
    """Every path with cross-CTA exchanges (sync-free epoch-tagged TRSM words, sequence-numbered and
    self-validating panel slots, spin grid barriers) solves the same input 25 times: X, flags and
    rcond must be bitwise identical every time (no floating-point atomics on numeric paths, so any
    difference is a race), and equal the oracle's within the parity bars."""
    mats = {
        "lu_leaf": lambda: W.make("C5", n=11000, nrhs=2, seed=3),      # first blocks: leaf panel (m > 10240)
        "lu_coop": lambda: W.make("C5", n=3000, nrhs=2, seed=4),
        "lu_cluster": lambda: W.make("C5", n=1000, nrhs=2, seed=5),
        "upper": lambda: (W.random_triangular(2500, upper=True, seed=6), np.ones((2500, 3))),
        "spd": lambda: (W.random_spd_fig3(1500, seed=7), np.ones((1500, 3))),
        "band_spike": lambda: W.make("C2", n=5000, nrhs=3),
        "band_chain": lambda: (W.random_banded(3000, 2, 2, seed=8), np.ones((3000, 2))),
        "svd": lambda: W.illcond_c4(n=160, seed=9)[:2],
    }
    A, B = mats[case]()
    A, B = np.asfortranarray(A), np.asfortranarray(B)
    dA, dB = AS.to_device(A), AS.to_device(B)
    X = AS.empty_colmajor(B.shape[0], B.shape[1], dB.dtype)
    ref = None
    for _ in range(25 if A.shape[0] < 8000 else 6):
        ret, _, rep = AS.as_solve_ex(dA, dB, X=X)
        torch.cuda.synchronize()
        cur = (ret, rep["flags"], rep["rcond"], X.cpu().numpy().tobytes())
        if ref is None:
            ref = cur
        else:
            assert cur == ref, case
    if A.shape[0] <= 3000:
        check_parity(A, B)


# ------------------------------------------------------------------ estimator: same steps as the oracle
@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 200, 384, 512])
@pytest.mark.parametrize("kind", ["lu", "spd", "lower", "upper"])
def test_estimator_rcond_tight(kind, n):
    """The device xLACN2 state machine (rcond.cu) runs the oracle's estimator steps (Z13b)
    through the same factors: same iteration, same vectors, so the estimate agrees to rounding
    (1e-8 relative), not only within the soft factor-of-two bar."""
    rng = np.random.default_rng(1000 * n + len(kind))
    if kind == "lu":
        A = rng.standard_normal((n, n)) + 4.0 * np.eye(n)
    elif kind == "spd":
        A = W.random_spd_fig3(n, seed=n) if n > 1 else np.array([[2.5]])
    else:
        T = np.tril(rng.standard_normal((n, n)) / 8.0, -1) + np.diag(1.0 + rng.random(n))
        A = T if kind == "lower" else T.T
    A = np.asfortranarray(A)
    B = np.asfortranarray(rng.standard_normal((n, 3)))
    ret, X, rep = gpu_solve(A, B)
    oret, Xo, orep, _ = oracle.solve(A, B)
    assert ret == oret == 0
    assert rep["primary_method"] == orep["primary_method"]
    assert (rep["flags"] & MASK) == (orep["flags"] & MASK)
    assert orep["rcond"] > 0
    assert abs(rep["rcond"] / orep["rcond"] - 1.0) <= 1e-8, (rep["rcond"], orep["rcond"])


# ------------------------------------------------------------------ detection: TMA tile pipeline (single candidate left)
def _padded(A, lda):
    """A (n x n) as a column-major device view with leading dimension lda (poison beyond row n)."""
    n = A.shape[0]
    big = np.full((lda, n), 7.0, dtype=A.dtype, order="F")
    big[:n] = A
    return AS.to_device(big)[:n]


def _tma_cases(n, dtype, rng):
    i, j = np.indices((n, n))
    dense = rng.standard_normal((n, n))
    up = np.triu(dense) + np.diag(np.full(n, 3.0))
    lo = np.tril(dense) + np.diag(np.full(n, 3.0))
    sym = (dense + dense.T) / (8.0 * n) + np.diag(1.0 + rng.random(n))
    yield "upper", up
    yield "lower", lo
    yield "sympd", sym
    # one non-zero in the other triangle: next to the diagonal inside a diagonal tile, in an interior
    # tile, in the last (ragged) tile row, and a -0.0 (a zero) / NaN (a non-zero)
    spots = [(65, 64), (n // 2 + 3, 70), (n - 1, n // 2), (n - 2, n - 3), (200, 3)]
    for k, (r, c) in enumerate(spots):
        M = up.copy(); M[r, c] = 1e-300 if dtype == np.float64 else 1e-30
        yield f"upper_nz{k}", M
        M = lo.copy(); M[c, r] = -2.0
        yield f"lower_nz{k}", M
    M = up.copy(); M[300, 5] = -0.0
    yield "upper_negzero", M
    M = up.copy(); M[301, 5] = np.nan
    yield "upper_nan", M
    # Fig. 4 lines 12-16 violated on one element pair (interior pair, diagonal tile, ragged edge tile)
    for k, (r, c) in enumerate([(n // 2 + 3, 70), (130, 129), (n - 1, n - 66), (n - 1, 64)]):
        M = sym.copy(); M[r, c] *= 1.0 + 1e-3                      # lines 13-14
        yield f"sympd_asym{k}", M
        M = sym.copy(); M[r, c] = M[c, r] = 5.0                     # line 15: |a| >= max diag
        yield f"sympd_maxdiag{k}", M
        M = sym.copy(); M[r, c] = M[c, r] = 0.5 * (M[r, r] + M[c, c])   # line 16 (equality kills)
        yield f"sympd_diagsum{k}", M
    M = sym.copy(); M[400, 100] = M[100, 400] = np.nan             # NaN compares false: survives Fig. 4
    yield "sympd_nan", M
    M = sym.copy(); M[7, 7] = np.nan                               # NaN on the diagonal (line 8: no kill)
    yield "sympd_nan_diag", M


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("n,pad", [(1024, 0), (1100, 0), (1537, 3), (2049, 7)])
def test_detect_tma_single_candidate(n, pad, dtype):
    """n >= 1024 with 16-byte aligned columns and one candidate left after the diagonal pass runs the
    TMA tile pipeline (detect_pairs_tma): every verdict bit-exact against the oracle, on clean
    triangular / sympd inputs and with a single deciding element in each kind of tile."""
    rng = np.random.default_rng(n)
    lda = n + pad                     # (1537 + 3) and (2049 + 7) are multiples of 4: aligned in fp32 too
    assert (lda * np.dtype(dtype).itemsize) % 16 == 0
    for name, M in _tma_cases(n, dtype, rng):
        A = np.asfortranarray(M.astype(dtype))
        d = oracle.detect(A)
        ret, st = AS.as_detect(_padded(A, lda))
        assert ret == 0
        assert st["flags"] == d.flags and st["method"] == d.method, (name, n, st, d)


def test_detect_tma_matches_direct_path_in_solve():
    """The same solve with the TMA pass and (lda odd: columns not 16-byte aligned) without it."""
    n = 1100
    A, B = W.make("C3b", n=n, nrhs=3)
    ret, X1, rep1 = gpu_solve(A, B)
    big = np.full((n + 1, n), 3.0, order="F"); big[:n] = A
    o = AS.make_options()
    ret2, X2, rep2 = AS.as_solve_ex(AS.to_device(big)[:n], AS.to_device(B), options=o)
    torch.cuda.synchronize()
    assert ret == ret2 == 0 and rep1["flags"] == rep2["flags"] and rep1["method"] == rep2["method"] == oracle.M_TRI_UPPER
    assert np.array_equal(X1, AS.to_host(X2))


def _tma_generic_cases(n, rng):
    i, j = np.indices((n, n))
    dense = rng.standard_normal((n, n))

    def band(kl, ku, dom=False):
        M = np.where((i - j <= kl) & (j - i <= ku), dense, 0.0)
        if dom:
            M[np.arange(n), np.arange(n)] = 1.0 + np.abs(M).sum(axis=1)
        return M

    yield "diagonal", band(0, 0)
    yield "lower_band", band(5, 0)
    yield "upper_band", band(0, 7)
    yield "band_8_8", band(8, 8, dom=True)
    yield "band_200_3", band(200, 3)
    yield "band_63_64", band(63, 64)
    # around the 25% capacity boundary: n (kl + ku + 1) - ... against n^2 / 4
    for kl, ku in [(n // 8, n // 8 - 8), (n // 8 + 4, n // 8 + 4), (n // 4 - 40, 0), (0, n // 4 + 40), (n // 7, n // 9)]:
        yield f"band_{kl}_{ku}", band(kl, ku)
    sb = band(4, 4)
    sb = (sb + sb.T) / 20.0
    sb[np.arange(n), np.arange(n)] = 2.0 + rng.random(n)
    yield "sympd_band", sb
    M = sb.copy(); M[n - 3, n - 6] *= 1.0 + 1e-3
    yield "sympd_band_asym_edge", M
    M = sb.copy(); M[700, 697] = M[697, 700] = 3.5
    yield "sympd_band_maxdiag", M
    # two lone far elements in different tile pairs: each extent passes the 25% rule alone, not together
    M = np.eye(n); M[n // 3 + 20, 20] = 1.0; M[10, n // 5 + 10] = 1.0
    yield "two_far_elements", M
    M = band(1, 1); M[n - 100, 50] = 1e-200
    yield "tridiag_plus_far", M
    M = np.tril(band(3, 3)); M[5, 900] = -0.0
    yield "lower_band_negzero", M
    M = dense * (rng.random((n, n)) < 0.002); M[np.arange(n), np.arange(n)] = 5.0
    yield "sparse_random", M
    yield "dense", dense


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("n,pad", [(1024, 0), (1100, 0), (2049, 7)])
def test_detect_tma_several_candidates(n, pad, dtype):
    """Banded / sparse / dense inputs at n >= 1024 through the TMA pair pass with several candidates alive:
    flags, method and (when banded) the exact extents against the oracle."""
    rng = np.random.default_rng(n + 1)
    for name, M in _tma_generic_cases(n, rng):
        A = np.asfortranarray(M.astype(dtype))
        d = oracle.detect(A)
        ret, st = AS.as_detect(_padded(A, n + pad))
        assert ret == 0
        assert st["flags"] == d.flags and st["method"] == d.method, (name, n, st, d)
        if d.banded:
            assert (st["kl"], st["ku"]) == (d.kl, d.ku), (name, st, d)


# ------------------------------------------------------------------ Cholesky: two panels per step (K = 128 bulk update)
_PAIRS_SNIPPET = r"""
import sys
import numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import oracle, workloads as W
import paper_2007_11208_b200 as AS
from helpers import backward_error, forward_diff
for n, nrhs in [(640, 3), (1100, 5), (2112, 9)]:
    A, B = W.make("C3a", n=n, nrhs=nrhs, seed=n)
    ret, X, rep = AS.as_solve_ex(AS.to_device(A), AS.to_device(B))
    torch.cuda.synchronize()
    oret, Xo, orep, _ = oracle.solve(A, B)
    X = AS.to_host(X)
    assert ret == oret == 0 and rep["method"] == orep["method"] == oracle.M_CHOL, (ret, rep, orep)
    assert (rep["flags"] & 0xFFFF) == (orep["flags"] & 0xFFFF)
    assert backward_error(A, X, B) <= 1e-13
    assert forward_diff(X, Xo) <= 1e-15 * orep["anorm"] / orep["rcond"]
    assert abs(np.log2(rep["rcond"] / orep["rcond"])) <= 1.0
# fp32 through the same schedule, graded against the fp64 oracle on the promoted data
A, B = W.make("C3a", n=1100, nrhs=4, seed=9)
A32, B32 = np.asfortranarray(A.astype(np.float32)), np.asfortranarray(B.astype(np.float32))
ret, X, rep = AS.as_solve_ex(AS.to_device(A32), AS.to_device(B32))
torch.cuda.synchronize()
A64, B64 = A32.astype(np.float64), B32.astype(np.float64)
_, Xr, rr, _ = oracle.solve(A64, B64, no_fallback=True)
X = AS.to_host(X)
assert ret == 0 and rep["method"] == oracle.M_CHOL
assert backward_error(A64, X, B64) <= 1e-5 and forward_diff(X, Xr) <= 1e-6 * rr["anorm"] / rr["rcond"]
# not positive definite in the second panel of a pair: falls back to LU exactly like the oracle
A, B = W.make("C3a", n=700, nrhs=2, seed=5)
A[100, 100] = 0.01
A = np.asfortranarray(A)
ret, X, rep = AS.as_solve_ex(AS.to_device(A), AS.to_device(B))
torch.cuda.synchronize()
oret, Xo, orep, _ = oracle.solve(A, B)
assert ret == oret and (rep["flags"] & 0xFFFF) == (orep["flags"] & 0xFFFF) and rep["method"] == orep["method"], (rep, orep)
print("pairs ok")
"""


def test_chol_paired_panels_small_n():
    """The paired-panel Cholesky schedule (default for n >= 6144) forced down to n >= 512 in a child
    process (the threshold is read once per process): oracle parity incl. the failure -> LU branch."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, AS_CHOL_PAIRS_MIN_N="512")
    r = subprocess.run([sys.executable, "-c", _PAIRS_SNIPPET.format(root=root, tests=os.path.join(root, "tests"))],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "pairs ok" in r.stdout, r.stdout + r.stderr


def test_detect_tma_alignment_is_part_of_the_plan():
    """Same n and lda, A 16-byte aligned (TMA pair pass) and offset by one element (register-direct pass),
    alternating on one stream: two plans, identical verdicts and solutions."""
    n, nrhs = 1100, 2
    A, B = W.make("C3a", n=n, nrhs=nrhs, seed=3)
    flat = torch.empty(n * n + 1, dtype=torch.float64, device="cuda")
    views = []
    for off in (0, 1):
        v = flat[off:off + n * n].view(n, n).t()
        assert (v.data_ptr() % 16 == 0) == (off == 0)
        views.append(v)
    dB = AS.to_device(B)
    outs = []
    for rep_i in range(2):
        for v in views:
            v.copy_(torch.from_numpy(A).to("cuda"))
            ret, st = AS.as_detect(v)
            assert ret == 0
            ret2, X, rep = AS.as_solve_ex(v, dB)
            torch.cuda.synchronize()
            assert ret2 == 0
            outs.append((st["flags"], st["method"], rep["flags"], AS.to_host(X)))
    d = oracle.detect(A)
    for fl, m, rf, X in outs:
        assert fl == d.flags and m == d.method and rf == outs[0][2]
        assert np.array_equal(X, outs[0][3])
