"""Seeded synthetic inputs for the adaptive solver (BASELINE.json configs).

This module holds ONLY input generation: no arithmetic of the method lives
here.  It is the one module shared by the oracle side (tests, cpu_baseline)
and the CUDA side (tests, bench, smoke): both consume the same bytes.

Recipe contract: torch CPU ``Generator().manual_seed(seed)``,
float64, draws in the order listed; "flat col-major" means draw k fills
A[k mod n, k div n].  The paper's own workloads are unspecified random systems
 except the Fig. 3 sympd generator, so these configs are
the BASELINE.json recipes, no public dataset is involved.

Every generator returns column-major (Fortran-order) numpy arrays.
"""
from __future__ import annotations

import hashlib

import numpy as np
import torch

CONFIGS = {
    # tag: (description, default kwargs)
    "C1": ("dense general fp64 n=256, N(0,1)+4I, 1 RHS; expect LU", dict(n=256, nrhs=1)),
    "C2": ("banded fp64 n=8192 kl=ku=8, U(-1,1) + dominant diag, 4 RHS; expect band LU", dict(n=8192, nrhs=4, kl=8, ku=8)),
    "C3a": ("SPD fp64 n=4096, G G^T/n + I, 64 RHS; expect Cholesky", dict(n=4096, nrhs=64)),
    "C3b": ("upper-triangular fp64 n=4096, diag U(1,2), N(0,1)/sqrt(n) above, 64 RHS; expect TRTRS", dict(n=4096, nrhs=64)),
    "C4": ("ill-conditioned fp64 n=1024, U diag(logspace(0,-18)) V^T, 1 RHS; expect SVD fallback", dict(n=1024, nrhs=1)),
    "C5": ("dense general fp64 n=16384, N(0,1), 32 RHS; expect blocked LU", dict(n=16384, nrhs=32)),
    "C5f": ("C5's matrix rounded to fp32", dict(n=16384, nrhs=32)),
}


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator()
    g.manual_seed(seed)
    return g


def _colmajor(flat: torch.Tensor, m: int, n: int) -> np.ndarray:
    """Flat draw k -> A[k mod m, k div m] (column-major)."""
    return np.asfortranarray(flat.numpy().reshape(n, m).T)


def rhs(n: int, nrhs: int, seed: int) -> np.ndarray:
    g = _gen(seed)
    return _colmajor(torch.randn(n * nrhs, generator=g, dtype=torch.float64), n, nrhs)


def dense_c1(n=256, nrhs=1, seed=0, shift=4.0):
    """C1: A = randn(n^2) flat col-major; A += shift*I; B = randn(n*nrhs)."""
    g = _gen(seed)
    A = _colmajor(torch.randn(n * n, generator=g, dtype=torch.float64), n, n)
    A[np.arange(n), np.arange(n)] += shift
    B = _colmajor(torch.randn(n * nrhs, generator=g, dtype=torch.float64), n, nrhs)
    return A, B


def banded_c2(n=8192, nrhs=4, kl=8, ku=8, seed=0):
    """C2: zero outside the band; for each column j, rows max(0,j-ku)..min(n-1,j+kl)
    except j, ascending: U[-1,1); then A[j,j] = 1 + sum_{i!=j} |A[j,i]| (row sum);
    B = randn(n*nrhs) flat col-major."""
    g = _gen(seed)
    # enumerate (i, j) in column-major order: j outer, i ascending
    j = np.repeat(np.arange(n), kl + ku + 1)
    i = j + np.tile(np.arange(-ku, kl + 1), n)
    keep = (i >= 0) & (i < n) & (i != j)
    i, j = i[keep], j[keep]
    vals = (2.0 * torch.rand(i.size, generator=g, dtype=torch.float64) - 1.0).numpy()
    A = np.zeros((n, n), dtype=np.float64, order="F")
    A[i, j] = vals
    rowsum = np.zeros(n, dtype=np.float64)
    np.add.at(rowsum, i, np.abs(vals))
    A[np.arange(n), np.arange(n)] = 1.0 + rowsum
    B = _colmajor(torch.randn(n * nrhs, generator=g, dtype=torch.float64), n, nrhs)
    return A, B


def spd_c3a(n=4096, nrhs=64, seed=0):
    """C3a: G = randn(n^2) flat col-major; A = G G^T / n; A = (A + A^T)/2; A += I.
    B = rhs(n, nrhs, seed + 1000) (shared with C3b)."""
    g = _gen(seed)
    G = torch.randn(n * n, generator=g, dtype=torch.float64).reshape(n, n).T  # column-major view
    A = (G @ G.T) / n
    A = (A + A.T) / 2
    A = A + torch.eye(n, dtype=torch.float64)
    A = np.asfortranarray(A.numpy())
    return A, rhs(n, nrhs, seed + 1000)


def upper_c3b(n=4096, nrhs=64, seed=0):
    """C3b: U = 0; U[j,j] = 1 + rand (U[1,2)); strict upper (i<j) flat col-major
    over (j outer, i ascending): randn/sqrt(n).  B = rhs(n, nrhs, seed + 1000)."""
    g = _gen(seed)
    d = 1.0 + torch.rand(n, generator=g, dtype=torch.float64).numpy()
    iu = np.triu_indices(n, 1)           # row-major order of (i, j), i < j
    order = np.lexsort((iu[0], iu[1]))   # -> column-major order: j outer, i ascending
    ii, jj = iu[0][order], iu[1][order]
    vals = (torch.randn(ii.size, generator=g, dtype=torch.float64) / np.sqrt(n)).numpy()
    A = np.zeros((n, n), dtype=np.float64, order="F")
    A[ii, jj] = vals
    A[np.arange(n), np.arange(n)] = d
    return A, rhs(n, nrhs, seed + 1000)


def haar(n: int, g: torch.Generator) -> np.ndarray:
    """Haar-random orthogonal: Q diag(sign(diag R)) of the QR of a Gaussian."""
    Z = torch.randn(n * n, generator=g, dtype=torch.float64).reshape(n, n).T
    Q, R = torch.linalg.qr(Z)
    s = torch.sign(torch.diagonal(R))
    s[s == 0] = 1.0
    return (Q * s).numpy()


def illcond_c4(n=1024, nrhs=1, seed=0, smin_exp=-18.0):
    """C4: A = U diag(sigma) V^T, U, V Haar; sigma_k = 10^(smin_exp*k/(n-1)).
    Returns (A, B, U, sigma, V) -- U/sigma/V for the closed-form pins."""
    g = _gen(seed)
    U = haar(n, g)
    V = haar(n, g)
    k = np.arange(n, dtype=np.float64)
    sigma = 10.0 ** (smin_exp * k / (n - 1)) if n > 1 else np.ones(1)
    A = np.asfortranarray((U * sigma) @ V.T)
    B = _colmajor(torch.randn(n * nrhs, generator=g, dtype=torch.float64), n, nrhs)
    return A, B, U, sigma, V


def dense_c5(n=16384, nrhs=32, seed=0):
    """C5: A = randn(n^2) flat col-major; B = randn(n*nrhs)."""
    g = _gen(seed)
    A = _colmajor(torch.randn(n * n, generator=g, dtype=torch.float64), n, n)
    B = _colmajor(torch.randn(n * nrhs, generator=g, dtype=torch.float64), n, nrhs)
    return A, B


def make(tag: str, **kw):
    """(A, B) for a BASELINE config tag at its default (or overridden) size."""
    kwargs = dict(CONFIGS[tag][1])
    kwargs.update(kw)
    if tag == "C1":
        return dense_c1(**kwargs)
    if tag == "C2":
        return banded_c2(**kwargs)
    if tag == "C3a":
        return spd_c3a(**kwargs)
    if tag == "C3b":
        return upper_c3b(**kwargs)
    if tag == "C4":
        A, B, *_ = illcond_c4(**kwargs)
        return A, B
    if tag == "C5":
        return dense_c5(**kwargs)
    if tag == "C5f":
        A, B = dense_c5(**kwargs)
        return np.asfortranarray(A.astype(np.float32)), np.asfortranarray(B.astype(np.float32))
    raise KeyError(tag)


def sha256(*arrays: np.ndarray) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.asfortranarray(a).tobytes(order="F"))
    return h.hexdigest()


# ------------------------------------------------------------------ small structured inputs
def random_banded(n, kl, ku, seed=0, dominant=False, dtype=np.float64):
    """Random band matrix, N(0,1) entries inside the band (exact zeros outside)."""
    g = _gen(seed)
    A = torch.randn(n, n, generator=g, dtype=torch.float64).numpy()
    i, j = np.indices((n, n))
    A[(i - j > kl) | (j - i > ku)] = 0.0
    if dominant:
        A[np.arange(n), np.arange(n)] = 1.0 + np.abs(A).sum(axis=1)
    return np.asfortranarray(A.astype(dtype))


def random_triangular(n, upper, seed=0, dtype=np.float64):
    g = _gen(seed)
    A = (torch.randn(n, n, generator=g, dtype=torch.float64) / np.sqrt(max(n, 1))).numpy()
    A = np.triu(A, 1) if upper else np.tril(A, -1)
    A[np.arange(n), np.arange(n)] = 1.0 + torch.rand(n, generator=g, dtype=torch.float64).numpy()
    return np.asfortranarray(A.astype(dtype))


def random_spd_fig3(n, seed=0, dtype=np.float64):
    """Fig. 3: R = U[-0.5,0.5]; A = R^T R; diag += 1."""
    g = _gen(seed)
    R = torch.rand(n, n, generator=g, dtype=torch.float64).numpy() - 0.5
    A = R.T @ R
    A[np.arange(n), np.arange(n)] += 1.0
    return np.asfortranarray(A.astype(dtype))


def random_dense(n, seed=0, dtype=np.float64, shift=0.0):
    g = _gen(seed)
    A = torch.randn(n, n, generator=g, dtype=torch.float64).numpy()
    A[np.arange(n), np.arange(n)] += shift
    return np.asfortranarray(A.astype(dtype))
