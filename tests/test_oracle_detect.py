"""Pins for the oracle's structure detection (Fig. 4).

Everything here is checked against the paper's printed examples, the
definitions written independently (brute force over all non-zeros), or
mathematical facts (SPD matrices satisfy Fig. 4's necessary conditions) --
never against the oracle itself.
"""
import numpy as np
import pytest

import oracle
import workloads as W
from helpers import F, load_fig1, load_pins

PINS = load_pins()


def test_constants_exact():
    # P:441-443 footnote, P:473 (tol), P:625 (threshold)
    assert np.finfo(np.float64).eps == PINS["eps64"]["value"]
    assert 100 * np.finfo(np.float64).eps == PINS["tol64"]["value"]
    assert 0.5 * np.finfo(np.float64).eps == PINS["thr64"]["value"]
    assert float(np.finfo(np.float32).eps) == PINS["eps32"]["value"]
    assert 0.5 * float(np.finfo(np.float32).eps) == PINS["thr32"]["value"]
    assert 1.0 + PINS["eps64"]["value"] > 1.0 and 1.0 + PINS["eps64"]["value"] / 2 == 1.0


def test_fig1_verdicts():
    m = load_fig1()
    a = oracle.detect(m["a"])   # kl=ku=1, 13/25 = 52% > 25% -> not banded
    assert (a.kl, a.ku) == (1, 1) and a.flags == 0 and a.method == oracle.M_LU
    b = oracle.detect(m["b"])   # lower, 60% -> not banded
    assert (b.kl, b.ku) == (4, 0) and b.flags == oracle.LOWER and b.method == oracle.M_TRI_LOWER
    c = oracle.detect(m["c"])   # sympd example
    assert c.flags == oracle.SPD and c.method == oracle.M_CHOL and c.max_diag == 9.0
    assert np.linalg.eigvalsh(m["c"]).min() > 1.0   # truly SPD (min eigenvalue ~1.392)


@pytest.mark.parametrize("case", PINS["fig4_cases"])
def test_fig4_pins(case):
    d = oracle.detect(F(case["A"]))
    assert d.spd == case["likely_sympd"], case["cite"]


def band_count(n, kl, ku):
    """Brute-force count of positions inside the band (not the closed form)."""
    i, j = np.indices((n, n))
    return int(((i - j <= kl) & (j - i <= ku)).sum())


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 11, 12, 13, 18, 19, 20, 100])
def test_diag_tridiag_pentadiag_thresholds(n):
    # P:352-355 diagonal matrices are banded -- subject to the 25% rule (Z5)
    d = oracle.detect(np.asfortranarray(np.eye(n)))
    assert d.banded == (4 * band_count(n, 0, 0) <= n * n) == (n >= 4)
    assert d.lower and d.upper and d.spd and (d.kl, d.ku) == (0, 0)
    T = np.asfortranarray(np.eye(n) * 4 + np.eye(n, k=1) + np.eye(n, k=-1))
    t = oracle.detect(T)
    assert (t.kl, t.ku) == ((1, 1) if n > 1 else (0, 0))
    if n > 1:
        assert t.banded == (n >= 12) == (4 * band_count(n, 1, 1) <= n * n)
    P5 = np.asfortranarray(sum(np.eye(n, k=k) for k in range(-2, 3)) + 5 * np.eye(n))
    p = oracle.detect(P5)
    if n > 2:
        assert p.banded == (n >= 19) == (4 * band_count(n, 2, 2) <= n * n)


def test_density_equality_is_banded():
    # Z3: 4*count == n^2 counts as banded (I_4: count 4, 16 <= 16)
    assert oracle.detect(np.asfortranarray(np.eye(4))).banded
    assert not oracle.detect(np.asfortranarray(np.eye(3))).banded


@pytest.mark.parametrize("seed", range(40))
def test_bruteforce_random_patterns(seed):
    """kl/ku and triangularity from the plain definitions (max |i-j| over non-zeros)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 24))
    A = np.zeros((n, n))
    kind = seed % 4
    i, j = np.indices((n, n))
    if kind == 0:
        kl, ku = int(rng.integers(0, n)), int(rng.integers(0, n))
        mask = (i - j <= kl) & (j - i <= ku) & (rng.random((n, n)) < 0.7)
    elif kind == 1:
        mask = (i >= j) & (rng.random((n, n)) < 0.5)
    elif kind == 2:
        mask = (i <= j) & (rng.random((n, n)) < 0.5)
    else:
        mask = rng.random((n, n)) < 0.1
    A[mask] = rng.standard_normal(mask.sum())
    A = np.asfortranarray(A)
    d = oracle.detect(A)
    nz = np.argwhere(A != 0)
    kl_true = max([r - c for r, c in nz if r > c], default=0)
    ku_true = max([c - r for r, c in nz if c > r], default=0)
    assert (d.kl, d.ku) == (kl_true, ku_true)
    assert d.banded == (4 * band_count(n, kl_true, ku_true) <= n * n)
    assert d.lower == (not np.any(np.triu(A, 1) != 0))
    assert d.upper == (not np.any(np.tril(A, -1) != 0))


def test_ieee_zero_semantics():
    # Z1: -0.0 is zero; subnormals and NaN are non-zero
    n = 64
    A = np.eye(n)
    A[0, n - 1] = -0.0
    A[n - 1, 0] = -0.0
    d = oracle.detect(np.asfortranarray(A))
    assert (d.kl, d.ku) == (0, 0) and d.banded and d.lower and d.upper
    A[0, n - 1] = 1e-310
    d = oracle.detect(np.asfortranarray(A))
    assert d.ku == n - 1 and d.upper and not d.lower and not d.banded
    A[0, n - 1] = 0.0
    A[n - 1, 0] = np.nan
    d = oracle.detect(np.asfortranarray(A))
    assert d.kl == n - 1 and d.lower and not d.upper


@pytest.mark.parametrize("seed", range(10))
def test_spd_matrices_pass_fig4(seed):
    """Exactly symmetric positive definite matrices satisfy every Fig. 4 condition
    (|a_ij| < sqrt(a_ii a_jj) <= max_diag, 2|a_ij| < a_ii + a_jj by AM-GM)."""
    n = 5 + seed * 7
    A = W.random_spd_fig3(n, seed)                 # Fig. 3 generator
    assert np.array_equal(A, A.T)
    assert oracle.detect(A).spd
    G = np.random.default_rng(seed).standard_normal((n, n))
    B = np.asfortranarray(G @ G.T + 1e-3 * np.eye(n))
    B = np.asfortranarray((B + B.T) / 2)
    assert oracle.detect(B).spd


def test_fig4_each_condition_fails():
    A = W.random_spd_fig3(20, 3)
    base = oracle.detect(A)
    assert base.spd
    B = A.copy(order="F"); B[7, 7] = -B[7, 7]            # (i) diagonal > 0
    assert not oracle.detect(B).spd
    B = A.copy(order="F"); B[5, 2] = B[2, 5] = 1.5 * A.diagonal().max()   # (ii) max modulus on diag
    assert not oracle.detect(B).spd
    B = A.copy(order="F"); B[5, 2] += 1e-6                # (iv) asymmetry beyond 100 eps
    assert not oracle.detect(B).spd
    B = A.copy(order="F"); B[5, 2] = B[5, 2] * (1 + 40 * np.finfo(float).eps)   # within tol (relative)
    assert oracle.detect(B).spd
    # (iii) pairwise dominance: |a_ij|+|a_ji| >= a_ii + a_jj while |a_ij| < max_diag
    C = np.asfortranarray(np.diag([1.0, 1.0, 10.0]))
    C[0, 1] = C[1, 0] = 1.0
    assert not oracle.detect(C).spd


def test_fig4_nan_inf_literal():
    # Z7: NaN passes lines 13/15/16 (comparisons false) -> still "likely"
    A = np.asfortranarray(np.eye(3) * 2)
    A[1, 0] = A[0, 1] = np.nan
    assert oracle.detect(A).spd
    A[1, 0] = A[0, 1] = np.inf
    assert not oracle.detect(A).spd      # line 15: inf >= max_diag


@pytest.mark.parametrize("lda_pad", [0, 3])
def test_lda_padding(lda_pad):
    """Detection reads only the leading n x n block of a padded buffer."""
    n = 30
    A = W.random_banded(n, 2, 1, seed=1)
    big = np.full((n + lda_pad, n), 7.0, order="F")
    big[:n, :] = A
    # oracle wrapper takes the leading block via a Fortran view; check verdict equality
    d1 = oracle.detect(A)
    d2 = oracle.detect(np.asfortranarray(big[:n, :]))
    assert d1 == d2 and (d1.kl, d1.ku) == (2, 1)


def test_config_verdicts_small():
    """Scaled-down config recipes dispatch as BASELINE.json expects."""
    A, _ = W.make("C1", n=64)
    assert oracle.detect(A).method == oracle.M_LU
    A, _ = W.make("C2", n=512)
    d = oracle.detect(A)
    assert d.method == oracle.M_BAND and (d.kl, d.ku) == (8, 8)
    A, _ = W.make("C3a", n=256, nrhs=4)
    assert oracle.detect(A).method == oracle.M_CHOL
    A, _ = W.make("C3b", n=256, nrhs=4)
    d = oracle.detect(A)
    assert d.method == oracle.M_TRI_UPPER and d.flags == oracle.UPPER
    A, _ = W.make("C4", n=128)
    assert oracle.detect(A).method == oracle.M_LU


def test_float32_detection():
    A = W.random_spd_fig3(16, 0).astype(np.float32, order="F")
    assert oracle.detect(A).spd
    B = A.copy(order="F"); B[3, 1] += np.float32(1e-3)
    assert not oracle.detect(B).spd
