"""Oracle dense Cholesky of the SCM (TEST INFRASTRUCTURE ONLY).

PAPER.md P:711-713 / P:735-736 (§3.1 type (i)): "dense Cholesky factorization
for the SCM B" via LAPACK.  B = R R^T, R lower with positive diagonal (unique).
LAPACK potrf through numpy is the library primitive used as this step.
"""
from __future__ import annotations

import numpy as np


def potrf_lower(B):
    """R lower with B = R R^T; uses only the lower triangle of B (LAPACK 'L')."""
    Bl = np.tril(B)
    Bs = Bl + np.tril(Bl, -1).T
    return np.linalg.cholesky(Bs)


def backward_error(B, R):
    Bl = np.tril(B)
    Bs = Bl + np.tril(Bl, -1).T
    return np.linalg.norm(Bs - R @ R.T) / np.linalg.norm(Bs)


def sce_solve(B, G):
    """Solution X of the Schur complement equation B X = G (B dz = g of the HKM
    search direction), B symmetric positive definite given by its lower triangle.  Plain definition
    through LAPACK: X = potrs(potrf(B), G).  (SURVEY §8(f) NEXT row 2.)"""
    import scipy.linalg as sl
    Bl = np.tril(B)
    Bs = Bl + np.tril(Bl, -1).T
    c = sl.cho_factor(Bs, lower=True)
    return sl.cho_solve(c, np.asarray(G, dtype=np.float64))
