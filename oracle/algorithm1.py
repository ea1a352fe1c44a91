"""Oracle Algorithm 1 (TEST INFRASTRUCTURE ONLY).

PAPER.md P:493-530 (§3.1, Algorithm 1), followed step by step:

  Step 1   allocate L-hat on E = union C_r x C_r.
  Step 2   for r = 1..l:
    2-1    P_r = reversal permutation ([P_r]_ij = 1 iff i+j = |C_r|+1);
    2-2    Cholesky  P_r X-bar_{C_r C_r} P_r^T = M_r M_r^T;
    2-3    L_r = P_r M_r^{-T} P_r^T   (so X-bar_{C_rC_r}^{-1} = L_r L_r^T);
  Step 3   put the first |S_r| columns of L_r into L-hat_{C_r S_r}.

Result: X-hat^{-1} = L-hat L-hat^T with X-hat the max-determinant completion
(validity proof P:541-679).  The north star's unit-lower form
X-hat^{-1} = L D L^T follows from L-hat = L D^{1/2} (SURVEY.md §8(c) reading #1):
D_j = L-hat_jj^2, L_ij = L-hat_ij / L-hat_jj.

Cliques C_r must list S_r first (reading #4) so that "the first |S_r| columns"
are the S_r columns.  Library primitives used as steps: numpy.linalg.cholesky
(LAPACK potrf, type (iii) P:717-719) and a triangular inverse.
"""
from __future__ import annotations

import numpy as np


class NotPositiveDefinite(Exception):
    def __init__(self, index):
        super().__init__(f"clique {index} not positive definite")
        self.index = index


def gather_dense(n, keys, vals, C):
    """X-bar_{C C} as a dense symmetric matrix from values on E (lower CSC keys)."""
    C = np.asarray(C, dtype=np.int64)
    r = np.maximum.outer(C, C)
    c = np.minimum.outer(C, C)
    k = c * n + r
    p = np.searchsorted(keys, k.ravel())
    if np.any(p >= keys.size) or np.any(keys[np.minimum(p, keys.size - 1)] != k.ravel()):
        raise ValueError("clique entry outside E")
    return vals[p].reshape(k.shape)


def algorithm1(S, xbar, cliques=None):
    """L-hat on E (CSC order of structure S) from X-bar on E.  Paper's Algorithm 1."""
    n = S.n
    keys = S.key()
    if cliques is None:
        cliques = S.cliques()
    Lhat = np.zeros(S.nnzE)                                   # Step 1
    for r, (C, s) in enumerate(cliques):                      # Step 2
        c = C.size
        X = gather_dense(n, keys, xbar, C)
        P = np.eye(c)[::-1]                                   # 2-1: [P]_ij = 1 iff i+j = c+1
        try:
            M = np.linalg.cholesky(P @ X @ P.T)               # 2-2
        except np.linalg.LinAlgError:
            raise NotPositiveDefinite(r)
        Lr = P @ np.linalg.inv(M).T @ P.T                     # 2-3
        for t in range(s):                                    # Step 3: first |S_r| columns
            j = int(C[t])
            rows = C[t:]
            pos = np.searchsorted(keys, j * n + rows)
            Lhat[pos] = Lr[t:, t]
    return Lhat


def unit_form(S, Lhat):
    """(L, D) with L unit lower on E and D diagonal: L-hat = L D^{1/2} (reading #1)."""
    diag = Lhat[S.colptr[:-1]]
    D = diag ** 2
    cols = np.repeat(np.arange(S.n), np.diff(S.colptr))
    L = Lhat / diag[cols]
    return L, D


def factor_xinv(S, xbar, cliques=None):
    """Oracle (a1): X-bar on E -> (L, D) with X-hat^{-1} = L D L^T."""
    return unit_form(S, algorithm1(S, xbar, cliques))


def columnwise_formula(S, xbar):
    """Algorithm 1 with C_j = {j} u struct(j), S_j = {j}, in closed form.

    L[I, j] = -X-bar[I, I]^{-1} X-bar[I, j];  D_j = 1 / (X-bar_jj + X-bar[j, I] L[I, j]).
    A second route (different partition) used to pin partition independence.
    """
    n = S.n
    keys = S.key()
    L = np.zeros(S.nnzE)
    D = np.zeros(n)
    for j in range(n):
        I = S.struct[j]
        p0 = S.colptr[j]
        L[p0] = 1.0
        xjj = xbar[p0]
        if I.size == 0:
            D[j] = 1.0 / xjj
            continue
        XII = gather_dense(n, keys, xbar, I)
        xIj = xbar[p0 + 1:S.colptr[j + 1]]
        l = -np.linalg.solve(XII, xIj)
        L[p0 + 1:S.colptr[j + 1]] = l
        D[j] = 1.0 / (xjj + xIj @ l)
    return L, D
