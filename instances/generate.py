"""Seeded synthetic SDP instances for the SCM hot path (shared input recipe).

This module is the ONLY code shared by the CUDA path's callers (bench.py, tests)
and the CPU oracle.  It builds the problem data the paper's method consumes
(the primal-dual pair (P)/(D): A_0..A_m, b) and the iterate
pieces the hot path is called on: the partial matrix X-bar given on the extended
sparsity pattern E and the dual matrix Y on E.

It contains none of the method's arithmetic (no Algorithm 1, no solves, no SCM,
no Cholesky).  To honour BASELINE.json's recipe ("X^-1 = L D L^T with L random
on E; Y = L_Y D_Y L_Y^T drawn the same way on E") it must know E, so it carries
its OWN symbolic elimination (merge-of-children rule) and the selected-inversion
recurrence Z[I,j] = -Z[I,I] L[I,j], Z[j,j] = 1/D_j - L[I,j]^T Z[I,j]
("Factors, values and seeds") that turns (L, D) into
X-bar = (L D L^T)^{-1} restricted to E.  The library and the oracle compute E
independently; tests require all three structures to agree bit-exactly.

Recipe: one seed per config; SeedSequence(seed).spawn(6) gives
the streams [weights, L, D, L_Y, D_Y, A_k].  Strictly-lower entries of L and L_Y
are N(0, 0.05^2) drawn in E's CSC order; D, D_Y ~ U[0.5, 2] in index order.
"""
from __future__ import annotations

import dataclasses
import hashlib
import os
from typing import Optional

import numpy as np
import scipy.sparse as sp

from . import graphs, orderings


@dataclasses.dataclass
class Instance:
    name: str
    n: int
    m: int
    # SDP data, ORIGINAL ids, lower triplets (row >= col); entries of A_k are
    # [a_ptr[k], a_ptr[k+1]) for k = 0..m (A_0 is the objective).
    a_ptr: np.ndarray
    a_row: np.ndarray
    a_col: np.ndarray
    a_val: np.ndarray
    b: np.ndarray
    perm: np.ndarray          # perm[new] = old
    # generator-side E (elimination order, lower CSC, rows ascending, diag first)
    colptr: np.ndarray
    rowind: np.ndarray
    L: np.ndarray             # unit lower factor values on E (diag stored as 1)
    D: np.ndarray
    Ly: np.ndarray
    Dy: np.ndarray
    xbar: np.ndarray          # X-bar on E (CSC order)
    y: np.ndarray             # Y on E (CSC order)
    kind: str = "general"     # "maxcut" | "theta" | "blockarrow" | "general"

    @property
    def nnzE(self) -> int:
        return int(self.colptr[-1])

    def sha256(self) -> str:
        h = hashlib.sha256()
        for f in ("a_ptr", "a_row", "a_col", "a_val", "b", "perm", "colptr", "rowind", "xbar", "y"):
            h.update(np.ascontiguousarray(getattr(self, f)).tobytes())
        return h.hexdigest()


# --------------------------------------------------------------------------
# problem data
# --------------------------------------------------------------------------

def _pack(mats, n):
    """mats: list of (rows, cols, vals) in original ids with row >= col."""
    ptr = np.zeros(len(mats) + 1, dtype=np.int64)
    for k, (r, _, _) in enumerate(mats):
        ptr[k + 1] = ptr[k] + len(r)
    rows = np.concatenate([np.asarray(r, dtype=np.int32) for r, _, _ in mats])
    cols = np.concatenate([np.asarray(c, dtype=np.int32) for _, c, _ in mats])
    vals = np.concatenate([np.asarray(v, dtype=np.float64) for _, _, v in mats])
    assert np.all(rows >= cols) and rows.min() >= 0 and rows.max() < n
    return ptr, rows, cols, vals


def _maxcut_data(k: int, rng_w, edges=None):
    """Max-cut SDP on the k x k torus (configs 0, 1, 4), or on the given edge
    list (the 3D torus of configs 5, 6; n = max id + 1).

    A_0 = -(1/4) * Laplacian(W) with W_e Rademacher +-1;
    A_k = e_k e_k^T, b_k = 1.
    """
    e = graphs.torus_edges(k) if edges is None else edges
    n = k * k if edges is None else int(edges.max()) + 1
    w = rng_w.choice(np.array([-1.0, 1.0]), size=len(e))
    deg = np.zeros(n)
    np.add.at(deg, e[:, 0], w)
    np.add.at(deg, e[:, 1], w)
    r0 = np.concatenate([np.arange(n), e[:, 1]])
    c0 = np.concatenate([np.arange(n), e[:, 0]])
    v0 = np.concatenate([-0.25 * deg, 0.25 * w])
    mats = [(r0, c0, v0)] + [([i], [i], [1.0]) for i in range(n)]
    return n, n, mats, np.ones(n), e


def _theta_data(k: int, rng_w):
    """Theta-type max-clique SDP on the k x k torus (config 2).

    A_1 = I (b_1 = 1); one A_k = e_i e_j^T + e_j e_i^T per edge (b_k = 0), so
    m = 1 + #edges (Table 3's m); A_0 = -(I + adjacency).
    """
    n = k * k
    e = graphs.torus_edges(k)
    r0 = np.concatenate([np.arange(n), e[:, 1]])
    c0 = np.concatenate([np.arange(n), e[:, 0]])
    v0 = -np.ones(n + len(e))
    mats = [(r0, c0, v0), (np.arange(n), np.arange(n), np.ones(n))]
    mats += [([b], [a], [1.0]) for a, b in e]
    m = 1 + len(e)
    bb = np.zeros(m)
    bb[0] = 1.0
    return n, m, mats, bb, e


def _blockarrow_data(nblk: int, bsz: int, border: int, m: int, rng_w, rng_a):
    """Block-arrow SDP (config 3).

    A_0: diagonal = n, off-diagonal N(0,1) on the whole pattern.  A_k: c ~ U{1..4}
    distinct positions drawn uniformly from the lower pattern (diag included),
    values N(0,1); a single-entry A_k whose position is already the support of
    another single-entry A_k is redrawn (two such matrices would make B singular).
    """
    pr, pc, n = graphs.block_arrow_lower_pattern(nblk, bsz, border)
    v0 = rng_w.standard_normal(len(pr))
    v0[pr == pc] = float(n)
    mats = [(pr, pc, v0)]
    single = set()
    npos = len(pr)
    for _ in range(m):
        while True:
            c = int(rng_a.integers(1, 5))
            pos = rng_a.choice(npos, size=c, replace=False)
            vals = rng_a.standard_normal(c)
            if c == 1:
                p = int(pos[0])
                if p in single:
                    continue
                single.add(p)
            break
        pos = np.sort(pos)
        mats.append((pr[pos], pc[pos], vals))
    return n, m, mats, np.zeros(m)


def aggregate_edges(n, a_row, a_col):
    """Off-diagonal positions of the aggregate sparsity pattern."""
    off = a_row != a_col
    e = np.stack([a_col[off], a_row[off]], axis=1).astype(np.int64)
    e = np.unique(e, axis=0)
    return e


# --------------------------------------------------------------------------
# generator-side symbolic elimination and factor values
# --------------------------------------------------------------------------

def _symbolic(n, perm, edges):
    """Filled pattern E of the permuted aggregate pattern (merge-of-children rule)."""
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    a = iperm[edges[:, 0]]
    b = iperm[edges[:, 1]]
    lo = np.minimum(a, b)
    hi = np.maximum(a, b)
    order = np.lexsort((hi, lo))
    lo = lo[order]
    hi = hi[order]
    start = np.searchsorted(lo, np.arange(n + 1))
    struct = [None] * n
    children = [[] for _ in range(n)]
    for j in range(n):
        parts = [hi[start[j]:start[j + 1]]]
        for c in children[j]:
            parts.append(struct[c][1:])
        s = np.unique(np.concatenate(parts)) if len(parts) > 1 else np.unique(parts[0])
        struct[j] = s
        if s.size:
            children[int(s[0])].append(j)
    cc = np.array([s.size for s in struct], dtype=np.int64)
    colptr = np.zeros(n + 1, dtype=np.int64)
    colptr[1:] = np.cumsum(cc + 1)
    rowind = np.empty(colptr[-1], dtype=np.int32)
    for j in range(n):
        rowind[colptr[j]] = j
        rowind[colptr[j] + 1:colptr[j + 1]] = struct[j]
    return colptr, rowind


def _blocks(n, colptr, rowind):
    """Group consecutive columns j, j+1 with struct(j) = {j+1} u struct(j+1)."""
    cc = np.diff(colptr) - 1
    blocks = []
    f = 0
    for j in range(n - 1):
        par = rowind[colptr[j] + 1] if cc[j] > 0 else -1
        if not (par == j + 1 and cc[j] == cc[j + 1] + 1):
            blocks.append((f, j))
            f = j + 1
    blocks.append((f, n - 1))
    return blocks


def _random_factor(n, colptr, rng_l, rng_d):
    nnz = int(colptr[-1])
    L = np.empty(nnz)
    diagpos = colptr[:-1]
    mask = np.ones(nnz, dtype=bool)
    mask[diagpos] = False
    L[diagpos] = 1.0
    L[mask] = rng_l.normal(0.0, 0.05, size=nnz - n)
    D = rng_d.uniform(0.5, 2.0, size=n)
    return L, D


def selected_inverse(n, colptr, rowind, L, D, blocks=None):
    """Z = (L D L^T)^{-1} restricted to E, by the selected-inversion recurrence.

    For j = n-1 down to 0 with I = struct(L_{*j}):
        Z[I, j] = -Z[I, I] L[I, j];   Z[j, j] = 1/D_j - L[I, j]^T Z[I, j].
    Columns are grouped in blocks sharing structure so the gathers of Z[U, U]
    happen once per block.
    """
    if blocks is None:
        blocks = _blocks(n, colptr, rowind)
    Z = np.zeros(int(colptr[-1]))
    for (f, l) in reversed(blocks):
        C = rowind[colptr[f]:colptr[f + 1]].astype(np.int64)
        c = C.size
        s = l - f + 1
        U = C[s:]
        u = U.size
        Zc = np.zeros((c, c))
        for q in range(u):
            col = int(U[q])
            seg = rowind[colptr[col]:colptr[col + 1]]
            pos = np.searchsorted(seg, U[q:])
            vals = Z[colptr[col] + pos]
            Zc[s + q:, s + q] = vals
            Zc[s + q, s + q:] = vals
        Lc = np.zeros((c, c))
        for t in range(s):
            Lc[t:, t] = L[colptr[f + t]:colptr[f + t + 1]]
        for t in range(s - 1, -1, -1):
            R = slice(t + 1, c)
            z = -Zc[R, R] @ Lc[R, t]
            Zc[R, t] = z
            Zc[t, R] = z
            Zc[t, t] = 1.0 / D[f + t] - Lc[R, t] @ z
        for t in range(s):
            Z[colptr[f + t]:colptr[f + t + 1]] = Zc[t:, t]
    return Z


def product_on_E(n, colptr, rowind, L, D):
    """Y = L D L^T (its pattern lies inside chordal E), returned on E's lower CSC."""
    cols = np.repeat(np.arange(n), np.diff(colptr))
    Ls = sp.csc_matrix((L, rowind, colptr), shape=(n, n))
    Y = (Ls @ sp.diags(D) @ Ls.T).tocoo()
    keep = Y.row >= Y.col
    yr = Y.row[keep].astype(np.int64)
    yc = Y.col[keep].astype(np.int64)
    keysE = cols.astype(np.int64) * n + rowind.astype(np.int64)
    keysY = yc * n + yr
    pos = np.searchsorted(keysE, keysY)
    assert np.all(keysE[pos] == keysY), "L D L^T has an entry outside E"
    out = np.zeros(int(colptr[-1]))
    np.add.at(out, pos, Y.data[keep])
    return out


# --------------------------------------------------------------------------
# configs
# --------------------------------------------------------------------------

CONFIGS = {
    0: dict(kind="maxcut", k=10, order="md"),
    1: dict(kind="maxcut", k=100, order="nd"),
    2: dict(kind="theta", k=60, order="md"),
    3: dict(kind="blockarrow", nblk=200, bsz=100, border=200, m=5000),
    4: dict(kind="maxcut", k=200, order="nd"),
    # 3D spin-glass torus (Table 3 SpinGlass18 / SpinGlass25),
    # not BASELINE configs
    5: dict(kind="maxcut3d", p=18, order="nd3"),
    6: dict(kind="maxcut3d", p=25, order="nd3"),
}


def build(kind: str, seed: int = 0, name: Optional[str] = None, **kw) -> Instance:
    ss = np.random.SeedSequence(seed).spawn(6)
    rng_w, rng_l, rng_d, rng_ly, rng_dy, rng_a = [np.random.default_rng(s) for s in ss]
    if kind == "maxcut":
        k = kw["k"]
        n, m, mats, b, e = _maxcut_data(k, rng_w)
    elif kind == "maxcut3d":
        n, m, mats, b, e = _maxcut_data(kw["p"], rng_w, graphs.torus3d_edges(kw["p"]))
    elif kind == "theta":
        k = kw["k"]
        n, m, mats, b, e = _theta_data(k, rng_w)
    elif kind == "blockarrow":
        n, m, mats, b = _blockarrow_data(kw["nblk"], kw["bsz"], kw["border"], kw["m"], rng_w, rng_a)
    else:
        raise ValueError(kind)
    a_ptr, a_row, a_col, a_val = _pack(mats, n)
    edges = aggregate_edges(n, a_row, a_col)
    order = kw.get("order", "identity")
    if order == "md":
        perm = orderings.minimum_degree(n, edges)
    elif order == "nd":
        perm = orderings.torus_nested_dissection(kw["k"])
    elif order == "nd3":
        perm = orderings.torus3d_nested_dissection(kw["p"])
    else:
        perm = np.arange(n, dtype=np.int32)
    colptr, rowind = _symbolic(n, perm, edges)
    blocks = _blocks(n, colptr, rowind)
    L, D = _random_factor(n, colptr, rng_l, rng_d)
    Ly, Dy = _random_factor(n, colptr, rng_ly, rng_dy)
    xbar = selected_inverse(n, colptr, rowind, L, D, blocks)
    y = product_on_E(n, colptr, rowind, Ly, Dy)
    return Instance(name=name or kind, n=n, m=m, a_ptr=a_ptr, a_row=a_row, a_col=a_col,
                    a_val=a_val, b=b, perm=perm.astype(np.int32), colptr=colptr, rowind=rowind,
                    L=L, D=D, Ly=Ly, Dy=Dy, xbar=xbar, y=y, kind="maxcut" if kind == "maxcut3d" else kind)


def _source_tag() -> str:
    """Hash of the generator's own sources: a change to the recipe never reuses a stale cached instance."""
    here = os.path.dirname(os.path.abspath(__file__))
    h = hashlib.sha256()
    for f in ("generate.py", "graphs.py", "orderings.py"):
        with open(os.path.join(here, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _cache_dir():
    d = os.environ.get("SDPC_INSTANCE_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "sdpc_instances"))
    return d


def gen_config(i: int, seed: int = 0, cache: bool = True) -> Instance:
    """Instance for BASELINE.json configs[i]."""
    kw = dict(CONFIGS[i])
    kind = kw.pop("kind")
    path = os.path.join(_cache_dir(), f"config{i}_seed{seed}_{_source_tag()}.npz")
    if cache and os.path.exists(path):
        try:
            z = np.load(path, allow_pickle=False)
            fields = {f.name: z[f.name] for f in dataclasses.fields(Instance)
                      if f.name not in ("name", "n", "m", "kind")}
            inst = Instance(name=str(z["name"]), n=int(z["n"]), m=int(z["m"]), kind=str(z["kind"]), **fields)
            return inst
        except Exception:
            pass
    inst = build(kind, seed=seed, name=f"config{i}", **kw)
    if cache:
        try:
            os.makedirs(_cache_dir(), exist_ok=True)
            tmp = path + f".tmp{os.getpid()}.npz"
            np.savez(tmp, **{f.name: getattr(inst, f.name) for f in dataclasses.fields(Instance)})
            os.replace(tmp, path)
        except OSError:
            pass
    return inst


def direction_G(inst: Instance, seed: int = 0, scale: float = 0.1) -> np.ndarray:
    """Synthetic input G of the search direction (the matrix G in g_k and dY;
    DESIGN.md reading: a residual matrix supplied by the caller) as lower values on E (E's CSC order):
    N(0, scale^2) entries, seeded (SeedSequence([seed, 7])).  No method arithmetic."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 7]))
    return scale * rng.standard_normal(int(inst.colptr[-1]))
