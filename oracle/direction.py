"""Oracle search direction and step lengths (TEST INFRASTRUCTURE ONLY).

SURVEY.md §8(f) NEXT rows 1-3.  Plain definitions, dense, in ORIGINAL index order, written out from
PAPER.md §2.2 (HKM direction) exactly as printed:

  g_k  = A_k . (beta mu Y^{-1} - X-hat - X-hat G Y^{-1})
  B dz = g                                                         P:374 (Eq. SCE)
  dY   = G - sum_k A_k dz_k
  dX-hat = beta mu Y^{-1} - X-hat - X-hat dY Y^{-1},
  dX   = (dX-hat + dX-hat^T) / 2                                   P:376 (Eq. dX)

with X . Y replaced by X-hat (completion invariance: every A_k and G lies on E, where
X-hat = X-bar).  dX is kept on E only (the columns of dX-hat are evaluated and kept on
the pattern; DESIGN.md reading).  G is an input (the paper prints G = A_0 - sum A_k z_k; the caller
passes whatever residual matrix it uses).

Column-wise route of P-MATRIX (Eq. newdX; Eq. newdX2):
  [dX-hat]_{*k} = beta mu Y^{-1} e_k - X-hat e_k - X-hat (dY (Y^{-1} e_k)),
with X-hat v and Y^{-1} v by the oracle's own sparse solves (scm.ColumnSolver).

Step lengths (Step 3; Eq. primal_length2):
  alpha_p = min_r max{alpha in (0,1] : X-bar_{C_rC_r} + alpha dX_{C_rC_r} >= 0}
  alpha_d = max{alpha in (0,1] : Y + alpha dY >= 0}
evaluated as 1 if lambda_min >= -1 else -1/lambda_min, lambda_min the smallest generalized eigenvalue
of (dM, M) (LAPACK sygv through scipy.linalg.eigh as the library step).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sl


def dense_on_E(S, vals, perm):
    """Dense symmetric matrix (ORIGINAL order) from lower values on E (elimination-order CSC)."""
    n = S.n
    p = np.asarray(perm, dtype=np.int64)
    M = np.zeros((n, n))
    cols = np.repeat(np.arange(n), np.diff(S.colptr))
    r, c = p[S.rowind], p[cols]
    M[r, c] = vals
    M[c, r] = vals
    return M


def values_on_E(S, M, perm):
    """Lower values on E (elimination-order CSC) of a dense matrix in ORIGINAL order."""
    n = S.n
    p = np.asarray(perm, dtype=np.int64)
    cols = np.repeat(np.arange(n), np.diff(S.colptr))
    return M[p[S.rowind], p[cols]].copy()


def constraint_dense(inst, k):
    """Dense A_k (k = 1..m), ORIGINAL order, from its lower triplets (duplicates summed)."""
    n = inst.n
    lo, hi = inst.a_ptr[k], inst.a_ptr[k + 1]
    A = np.zeros((n, n))
    for r, c, v in zip(inst.a_row[lo:hi], inst.a_col[lo:hi], inst.a_val[lo:hi]):
        A[r, c] += v
        if r != c:
            A[c, r] += v
    return A


def inner(A, M):
    """A . M = trace(A^T M) = sum_ij A_ij M_ij."""
    return float(np.sum(A * M))


def _entries(inst, k):
    """Stored lower triplets of A_k (k = 1..m), symmetric-expanded: (i, j, a) with both orientations."""
    lo, hi = inst.a_ptr[k], inst.a_ptr[k + 1]
    r = inst.a_row[lo:hi].astype(np.int64)
    c = inst.a_col[lo:hi].astype(np.int64)
    v = inst.a_val[lo:hi]
    off = r != c
    return np.concatenate([r, c[off]]), np.concatenate([c, r[off]]), np.concatenate([v, v[off]])


def g_vector(inst, Xh, Yi, G, bmu):
    """g_k = A_k . (beta mu Y^{-1} - X-hat - X-hat G Y^{-1}), k = 1..m, with
    A_k . M = sum_ij [A_k]_ij M_ij summed over the stored entries of A_k."""
    M = bmu * Yi - Xh - Xh @ G @ Yi
    g = np.empty(inst.m)
    for k in range(1, inst.m + 1):
        i, j, a = _entries(inst, k)
        g[k - 1] = float(np.sum(a * M[i, j]))
    return g


def sce(B, g):
    """dz with B dz = g (Eq. SCE), LAPACK potrf/potrs on the lower triangle of B."""
    Bl = np.tril(B)
    Bs = Bl + np.tril(Bl, -1).T
    return sl.cho_solve(sl.cho_factor(Bs, lower=True), g)


def dY_dense(inst, G, dz):
    """dY = G - sum_k A_k dz_k, subtracting dz_k [A_k]_ij at the stored entries of A_k."""
    dY = G.copy()
    for k in range(1, inst.m + 1):
        i, j, a = _entries(inst, k)
        np.subtract.at(dY, (i, j), dz[k - 1] * a)
    return dY


def dX_dense(Xh, Yi, dY, bmu):
    """dX = (dX-hat + dX-hat^T)/2, dX-hat = beta mu Y^{-1} - X-hat - X-hat dY Y^{-1}."""
    dXh = bmu * Yi - Xh - Xh @ dY @ Yi
    return 0.5 * (dXh + dXh.T)


def dX_columns(solver, dY, bmu, cols):
    """Column-wise P-MATRIX route (Eq. newdX2): [dX-hat]_{*k} for k in cols (ORIGINAL ids),
    each column from sparse solves: beta mu y_k - x_k - X-hat (dY y_k)."""
    cols = np.asarray(cols, dtype=np.int64)
    Yk = solver.y(cols)
    Xk = solver.x(cols)
    out = np.empty((solver.n, cols.size))
    for a in range(cols.size):
        u = dY @ Yk[:, a]
        # X-hat u by the factor solves: forward with L, D^{-1}, backward with L^T
        out[:, a] = bmu * Yk[:, a] - Xk[:, a] - _xhat_apply(solver, u)
    return out


def _xhat_apply(solver, u):
    import scipy.sparse.linalg as spl
    z = np.zeros(solver.n)
    z[solver.iperm] = u                 # original -> elimination order
    z = spl.spsolve_triangular(solver.Lcsr, z, lower=True, unit_diagonal=True)
    z = z / solver.D
    z = spl.spsolve_triangular(solver.LTcsr, z, lower=False, unit_diagonal=True)
    return z[solver.iperm]


def _step(M, dM):
    """max{alpha in (0,1] : M + alpha dM >= 0} for M > 0 (generalized eigenvalues of (dM, M))."""
    lam = sl.eigh(dM, M, eigvals_only=True)
    lmin = float(lam.min())
    return 1.0 if lmin >= -1.0 else -1.0 / lmin


def primal_step(S, xbar_E, dX_E):
    """alpha_p = min over cliques C_r of the clique step (Eq. primal_length2)."""
    from .algorithm1 import gather_dense
    keys = S.key()
    a = 1.0
    for C, _ in S.cliques():
        X = gather_dense(S.n, keys, xbar_E, C)
        dX = gather_dense(S.n, keys, dX_E, C)
        a = min(a, _step(X, dX))
    return a


def dual_step(S, y_E, dY_E, perm):
    """alpha_d = max{alpha in (0,1] : Y + alpha dY >= 0} (Step 3), dense."""
    return _step(dense_on_E(S, y_E, perm), dense_on_E(S, dY_E, perm))


def mu(S, xbar_E, y_E):
    """mu = X . Y / n with X . Y = X-bar . Y on E (Y lies on E)."""
    off = np.ones(S.nnzE)
    off[S.colptr[:-1]] = 0.0            # the diagonal is the first entry of each column
    return float(np.sum(xbar_E * y_E * (1.0 + off))) / S.n
