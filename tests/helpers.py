"""Test helpers: golden loaders, exact rational arithmetic, error metrics.

Nothing here implements the method; these are the independent yardsticks the
oracle (and then the CUDA path) is pinned to.
"""
from __future__ import annotations

import json
import os
from fractions import Fraction
from math import comb

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_pins():
    with open(os.path.join(GOLDEN, "pins.json")) as f:
        return json.load(f)


def load_fig1():
    mats, cur = {}, None
    with open(os.path.join(GOLDEN, "fig1.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line.startswith("["):
                cur = line.strip("[]")
                mats[cur] = []
                continue
            mats[cur].append([float(v) for v in line.split()])
    return {k: np.asfortranarray(np.array(v)) for k, v in mats.items()}


def F(a):
    return np.asfortranarray(np.array(a, dtype=np.float64))


# ---------------------------------------------------------------- exact arithmetic
def exact_inverse(A) -> list[list[Fraction]]:
    """Gauss-Jordan in rationals (brute force, n <= 8)."""
    n = len(A)
    M = [[Fraction(float(A[i][j])) for j in range(n)] + [Fraction(int(i == j)) for j in range(n)] for i in range(n)]
    for c in range(n):
        p = next((r for r in range(c, n) if M[r][c] != 0), None)
        if p is None:
            raise ZeroDivisionError("singular")
        M[c], M[p] = M[p], M[c]
        piv = M[c][c]
        M[c] = [v / piv for v in M[c]]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c]
                M[r] = [a - f * b for a, b in zip(M[r], M[c])]
    return [row[n:] for row in M]


def exact_solve(A, b):
    Ainv = exact_inverse(A)
    n = len(A)
    bb = [Fraction(float(v)) for v in np.asarray(b).reshape(-1)]
    return [sum(Ainv[i][k] * bb[k] for k in range(n)) for i in range(n)]


def exact_cond1(A):
    n = len(A)
    Ainv = exact_inverse(A)
    a1 = max(sum(abs(Fraction(float(A[i][j]))) for i in range(n)) for j in range(n))
    i1 = max(sum(abs(Ainv[i][j]) for i in range(n)) for j in range(n))
    return a1 * i1


def hilbert(n):
    return np.asfortranarray(np.array([[1.0 / (i + j + 1) for j in range(n)] for i in range(n)]))


def hilbert_inverse_exact(n):
    """Closed form (0-based): (H^-1)_ij = (-1)^(i+j) (i+j+1) C(n+i, n-j-1) C(n+j, n-i-1) C(i+j, i)^2."""
    return [[(-1) ** (i + j) * (i + j + 1) * comb(n + i, n - j - 1) * comb(n + j, n - i - 1) * comb(i + j, i) ** 2
             for j in range(n)] for i in range(n)]


# ---------------------------------------------------------------- metrics (north star, Z18)
def backward_error(A, X, B) -> float:
    """eta = max over columns ||A x - b||_inf / (||A||_inf ||x||_inf), evaluated in fp64."""
    A = np.asarray(A, dtype=np.float64)
    X = np.asarray(X, dtype=np.float64).reshape(A.shape[0], -1)
    B = np.asarray(B, dtype=np.float64).reshape(A.shape[0], -1)
    R = A @ X - B
    an = np.abs(A).sum(axis=1).max()
    eta = 0.0
    for c in range(X.shape[1]):
        den = an * np.abs(X[:, c]).max()
        eta = max(eta, np.abs(R[:, c]).max() / den if den > 0 else (0.0 if np.abs(R[:, c]).max() == 0 else np.inf))
    return eta


def forward_diff(X, Xref) -> float:
    """phi = max over columns ||x - x_ref||_1 / ||x_ref||_1."""
    X = np.asarray(X, dtype=np.float64).reshape(Xref.shape[0], -1)
    Xref = np.asarray(Xref, dtype=np.float64).reshape(Xref.shape[0], -1)
    out = 0.0
    for c in range(Xref.shape[1]):
        den = np.abs(Xref[:, c]).sum()
        num = np.abs(X[:, c] - Xref[:, c]).sum()
        out = max(out, num / den if den > 0 else num)
    return out
