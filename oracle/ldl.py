"""Oracle sparse LDL^T of the dual matrix Y on E (TEST INFRASTRUCTURE ONLY).

PAPER.md P:221-225 (§2.1): Y = A_0 - sum A_k z_k is factored Y = N N^T, whose
nonzeros are covered by E.  Type (v).  Unit-lower form used by the
north star: Y = L_Y D_Y L_Y^T (N = L_Y D_Y^{1/2}).

Plain left-looking column algorithm (textbook): for j = 0..n-1,
    w[j:] = Y[j:, j] - sum_{k<j, L_jk != 0} L[j:, k] D_k L_jk,
    D_j = w_j, L[I_j, j] = w[I_j] / D_j.
Raises NotPositiveDefinite(j) when a pivot is <= 0 or NaN (LAPACK rule,
SURVEY.md §8(c) reading #19).
"""
from __future__ import annotations

import numpy as np


class NotPositiveDefinite(Exception):
    def __init__(self, index):
        super().__init__(f"pivot {index} not positive")
        self.index = index


def ldl_on_E(S, yvals):
    n = S.n
    colptr, rowind = S.colptr, S.rowind
    L = np.zeros(S.nnzE)
    D = np.zeros(n)
    rowstruct = [[] for _ in range(n)]
    nextpos = colptr[:-1].copy()          # first stored row of column k that is >= current j
    w = np.zeros(n)
    for j in range(n):
        lo, hi = colptr[j], colptr[j + 1]
        rows = rowind[lo:hi]
        w[rows] = yvals[lo:hi]
        for k in rowstruct[j]:
            p = nextpos[k]                 # rowind[p] == j
            krow = rowind[p:colptr[k + 1]]
            kval = L[p:colptr[k + 1]]
            w[krow] -= kval * (D[k] * kval[0])
            nextpos[k] = p + 1
        d = w[j]
        if not (d > 0.0):
            raise NotPositiveDefinite(j)
        D[j] = d
        L[lo] = 1.0
        L[lo + 1:hi] = w[rows[1:]] / d
        w[rows] = 0.0
        nextpos[j] = lo + 1                # next use of column j is at its first off-diagonal row
        for i in rows[1:].tolist():
            rowstruct[i].append(j)
    return L, D
