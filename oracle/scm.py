"""Oracle Schur complement matrix (TEST INFRASTRUCTURE ONLY).

Plain definition (PAPER.md, Eq. SCM; completion invariance P:396-401):

    B_kl = (X-hat A_k Y^{-1}) . A_l = trace(A_k X-hat A_l Y^{-1}),  k, l = 1..m,

with X-hat = (L D L^T)^{-1} the max-determinant completion built from the oracle's
own Algorithm 1 factor and Y^{-1} the inverse of the dual matrix.  Written out
over stored entries with the symmetric expansion:

    B_kl = sum_{(i,j,v) in A_k} sum_{(p,q,w) in A_l} v w X-hat_{jp} (Y^{-1})_{qi}.

Dense mode forms X-hat and Y^{-1} densely (LAPACK inverse as a library step).
Sampled-column mode evaluates full columns l through per-RHS solves
x_p = X-hat e_p, y_q = Y^{-1} e_q (Eq. newSCM2; Algorithm 2 Step 3-3,
P:903-912), summing only over the nonzero columns p of A_l (reading #8).
Indices here are ORIGINAL ids; constraint k <-> A_k (k = 1..m, 0-based k-1).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spl

LARGE = 16   # A_k with more stored (symmetric-expanded) entries use the matmul route


def sym_entries(inst):
    """Per constraint k = 1..m: arrays (i, j, v) with off-diagonals in both orientations."""
    out = []
    for k in range(1, inst.m + 1):
        lo, hi = inst.a_ptr[k], inst.a_ptr[k + 1]
        r = inst.a_row[lo:hi].astype(np.int64)
        c = inst.a_col[lo:hi].astype(np.int64)
        v = inst.a_val[lo:hi]
        off = r != c
        out.append((np.concatenate([r, c[off]]), np.concatenate([c, r[off]]), np.concatenate([v, v[off]])))
    return out


def _padded(ents, idx):
    e = max((ents[k][0].size for k in idx), default=0)
    I = np.zeros((len(idx), e), dtype=np.int64)
    J = np.zeros((len(idx), e), dtype=np.int64)
    V = np.zeros((len(idx), e))
    for a, k in enumerate(idx):
        i, j, v = ents[k]
        I[a, :i.size] = i
        J[a, :i.size] = j
        V[a, :i.size] = v
    return I, J, V


def dense_completion(S, L, D, perm):
    """X-hat = (L D L^T)^{-1} densely, returned in ORIGINAL index order."""
    n = S.n
    Ls = sp.csc_matrix((L, S.rowind, S.colptr), shape=(n, n)).toarray()
    Xinv = (Ls * D) @ Ls.T
    Xh_new = np.linalg.inv(Xinv)
    Xh_new = 0.5 * (Xh_new + Xh_new.T)
    return _unpermute(Xh_new, perm)


def dense_y_inverse(S, yvals, perm):
    """Y^{-1} densely from Y on E, in ORIGINAL index order."""
    n = S.n
    Yl = sp.csc_matrix((yvals, S.rowind, S.colptr), shape=(n, n)).toarray()
    Y = Yl + np.tril(Yl, -1).T
    Yi = np.linalg.inv(Y)
    Yi = 0.5 * (Yi + Yi.T)
    return _unpermute(Yi, perm)


def _unpermute(Mnew, perm):
    n = Mnew.shape[0]
    M = np.empty_like(Mnew)
    p = np.asarray(perm, dtype=np.int64)
    M[np.ix_(p, p)] = Mnew          # M[perm[a], perm[b]] = Mnew[a, b]
    return M


def scm_dense(inst, Xh, Yi):
    """Full symmetric B (m x m) from dense X-hat, Y^{-1} (original order)."""
    m = inst.m
    ents = sym_entries(inst)
    sizes = np.array([e[0].size for e in ents])
    small = np.flatnonzero(sizes <= LARGE)
    large = np.flatnonzero(sizes > LARGE)
    B = np.zeros((m, m))
    if small.size:
        I, J, V = _padded(ents, small)
        Bs = np.zeros((small.size, small.size))
        for s in range(I.shape[1]):
            for t in range(I.shape[1]):
                # v_s(k) w_t(l) X-hat[j_s(k), p_t(l)] Y^{-1}[q_t(l), i_s(k)]; (p,q) of A_l = (I,J)[l]
                Bs += (V[:, s][:, None] * V[:, t][None, :]
                       * Xh[np.ix_(J[:, s], I[:, t])] * Yi[np.ix_(I[:, s], J[:, t])])
        B[np.ix_(small, small)] = Bs
    if small.size:
        P, Q, W = _padded(ents, small)
    for k in large:
        i, j, v = ents[k]
        Ak = np.zeros(Xh.shape)
        np.add.at(Ak, (i, j), v)
        G = Xh @ Ak @ Yi            # (X-hat A_k Y^{-1});  B_kl = G . A_l
        if small.size:
            row = np.sum(W * G[P, Q], axis=1)
            B[k, small] = row
            B[small, k] = row
        for l in large:
            p, q, w = ents[l]
            B[k, l] = np.sum(w * G[p, q])
    return B


def scm_bruteforce(inst, Xh, Yi):
    """B_kl = trace(A_k X-hat A_l Y^{-1}) with full dense A_k (tiny n only)."""
    n, m = inst.n, inst.m
    A = []
    for k in range(1, m + 1):
        lo, hi = inst.a_ptr[k], inst.a_ptr[k + 1]
        M = np.zeros((n, n))
        for r, c, v in zip(inst.a_row[lo:hi], inst.a_col[lo:hi], inst.a_val[lo:hi]):
            M[r, c] = v
            M[c, r] = v
        A.append(M)
    B = np.zeros((m, m))
    for k in range(m):
        T = A[k] @ Xh
        for l in range(m):
            B[k, l] = np.trace(T @ A[l] @ Yi)
    return B


class ColumnSolver:
    """x_p = X-hat e_p and y_q = Y^{-1} e_q, original ids, via sparse solves.

    X side: forward with L, scale by D^{-1}, backward with L^T (the oracle's own
    Algorithm 1 factor).  Y side: SuperLU factorization of Y
    (library primitive for Y^{-1} e_q; "N^{-T}N^{-1}[A_j]_{*k}").
    """

    def __init__(self, S, L, D, yvals, perm):
        n = S.n
        self.n = n
        self.perm = np.asarray(perm, dtype=np.int64)
        self.iperm = np.empty(n, dtype=np.int64)
        self.iperm[self.perm] = np.arange(n)
        self.Lcsr = sp.csc_matrix((L, S.rowind, S.colptr), shape=(n, n)).tocsr()
        self.LTcsr = self.Lcsr.T.tocsr()
        self.D = D
        Yl = sp.csc_matrix((yvals, S.rowind, S.colptr), shape=(n, n))
        Y = (Yl + sp.tril(Yl, -1).T).tocsc()
        self.ylu = spl.splu(Y)

    def x(self, p):
        p = np.atleast_1d(np.asarray(p, dtype=np.int64))
        Bm = np.zeros((self.n, p.size))
        Bm[self.iperm[p], np.arange(p.size)] = 1.0
        z = spl.spsolve_triangular(self.Lcsr, Bm, lower=True, unit_diagonal=True)
        z = z / self.D[:, None]
        x = spl.spsolve_triangular(self.LTcsr, z, lower=False, unit_diagonal=True)
        return x[self.iperm, :]                      # back to original row order

    def y(self, q):
        q = np.atleast_1d(np.asarray(q, dtype=np.int64))
        Bm = np.zeros((self.n, q.size))
        Bm[self.iperm[q], np.arange(q.size)] = 1.0     # Y is held in elimination order
        ynew = self.ylu.solve(Bm)
        return ynew[self.iperm, :]


def column_prep(inst):
    """Per-instance tables of scm_columns (constraint entries, small/large split), computed once."""
    ents = sym_entries(inst)
    sizes = np.array([e[0].size for e in ents])
    small = np.flatnonzero(sizes <= LARGE)
    large = np.flatnonzero(sizes > LARGE)
    I, J, V = _padded(ents, small)
    return ents, small, large, I, J, V


def scm_columns(inst, cols, solver: ColumnSolver, chunk=128, prep=None):
    """Full columns B[:, l] (all k) for the constraint indices l in `cols` (0-based).

    The solves x_p, y_q for all nonzero columns of the sampled A_l are done first, in
    multi-RHS chunks (same arithmetic as one solve per RHS, Algorithm 2 Step 3-3).
    `prep` = column_prep(inst) (recomputed when omitted).
    """
    m = inst.m
    ents, small, large, I, J, V = prep if prep is not None else column_prep(inst)
    ps = np.unique(np.concatenate([ents[l][0] for l in cols]))
    qs = np.unique(np.concatenate([ents[l][1] for l in cols]))
    X = np.concatenate([solver.x(ps[a:a + chunk]) for a in range(0, ps.size, chunk)], axis=1)
    Yc = np.concatenate([solver.y(qs[a:a + chunk]) for a in range(0, qs.size, chunk)], axis=1)
    out = np.zeros((m, len(cols)))
    for a, l in enumerate(cols):
        p, q, w = ents[l]
        ip = np.searchsorted(ps, p)
        iq = np.searchsorted(qs, q)
        col = np.zeros(m)
        for t in range(p.size):
            xp = X[:, ip[t]]
            yq = Yc[:, iq[t]]
            # small k: sum_s v_s x_p[j_s] y_q[i_s]
            if small.size:
                col[small] += w[t] * np.sum(V * xp[J] * yq[I], axis=1)
            for k in large:
                i, j, v = ents[k]
                col[k] += w[t] * np.sum(v * xp[j] * yq[i])
        out[:, a] = col
    return out
