"""Oracle symbolic analysis: E, etree, cliques (TEST INFRASTRUCTURE ONLY).

PAPER.md P:228-242 (§2.1): permute with an ordering, generate a chordal graph
from the aggregate sparsity pattern, extract cliques; E = union of
C_r x C_r.  P:747-766 (§3.1): the supernodes of the symbolic Cholesky give the
row sets C_r and column sets S_r, which have the running intersection property.

Route used here (independent of the generator's merge-of-children rule and of the
library's C++ etree/column-count code): the textbook ELIMINATION GAME.  In
elimination order, eliminating vertex v connects all its not-yet-eliminated
neighbours pairwise; struct(v) = those neighbours (the column pattern of the
Cholesky factor).  Adjacency is held as Python-int bitsets.

Supernodes (SURVEY.md §8(c) reading #3): fundamental supernodes of E, i.e.
j and j+1 share a supernode iff struct(j) = {j+1} u struct(j+1) and j+1 has
exactly one child in the elimination tree.  Clique r: S_r = its columns,
C_r = S_r followed by U_r = struct(last column of S_r), ascending (reading #4).
"""
from __future__ import annotations

import numpy as np


def aggregate_pattern(n, a_row, a_col):
    """Off-diagonal lower positions (orig ids) of the aggregate pattern."""
    pos = set()
    for i, j in zip(a_row.tolist(), a_col.tolist()):
        if i != j:
            pos.add((max(i, j), min(i, j)))
    return pos


def _bits(x: int) -> np.ndarray:
    if x == 0:
        return np.zeros(0, dtype=np.int64)
    nb = (x.bit_length() + 7) // 8
    arr = np.frombuffer(x.to_bytes(nb, "little"), dtype=np.uint8)
    return np.flatnonzero(np.unpackbits(arr, bitorder="little")).astype(np.int64)


def elimination_game(n, perm, a_row, a_col):
    """struct(v) for every v (new ids) by playing the elimination game."""
    iperm = np.empty(n, dtype=np.int64)
    iperm[np.asarray(perm, dtype=np.int64)] = np.arange(n)
    high = [0] * n
    for (i, j) in aggregate_pattern(n, a_row, a_col):
        a, b = int(iperm[i]), int(iperm[j])
        lo, hi = min(a, b), max(a, b)
        high[lo] |= 1 << hi
    struct = []
    for v in range(n):
        N = high[v]
        s = _bits(N)
        struct.append(s)
        for u in s.tolist():
            # eliminating v makes its neighbourhood a clique: u gains N's members above u
            high[u] |= (N >> (u + 1)) << (u + 1)
        high[v] = 0
    return struct


class Structure:
    """E (lower CSC, elimination order), etree parent, fundamental supernodes."""

    def __init__(self, n, struct):
        self.n = n
        self.struct = struct
        cc = np.array([s.size for s in struct], dtype=np.int64)
        self.cc = cc
        self.colptr = np.zeros(n + 1, dtype=np.int64)
        self.colptr[1:] = np.cumsum(cc + 1)
        self.rowind = np.empty(int(self.colptr[-1]), dtype=np.int32)
        for j in range(n):
            self.rowind[self.colptr[j]] = j
            self.rowind[self.colptr[j] + 1:self.colptr[j + 1]] = struct[j]
        self.parent = np.array([int(s[0]) if s.size else -1 for s in struct], dtype=np.int32)
        nchild = np.zeros(n, dtype=np.int64)
        for p in self.parent:
            if p >= 0:
                nchild[p] += 1
        sup = [0]
        for j in range(n - 1):
            same = (self.parent[j] == j + 1 and nchild[j + 1] == 1
                    and cc[j] == cc[j + 1] + 1
                    and np.array_equal(struct[j][1:], struct[j + 1]))
            if not same:
                sup.append(j + 1)
        sup.append(n)
        self.super_ptr = np.asarray(sup, dtype=np.int32)

    @property
    def nnzE(self):
        return int(self.colptr[-1])

    def cliques(self):
        """[(C_r, |S_r|)] over fundamental supernodes, C_r = S_r then U_r ascending."""
        out = []
        for r in range(len(self.super_ptr) - 1):
            f, l = int(self.super_ptr[r]), int(self.super_ptr[r + 1])
            C = np.concatenate([np.arange(f, l), self.struct[l - 1]]).astype(np.int64)
            out.append((C, l - f))
        return out

    def column_cliques(self):
        """[(C_j, 1)] with C_j = {j} u struct(j): Algorithm 1's clique sequence with S_j = {j}."""
        return [(np.concatenate([[j], self.struct[j]]).astype(np.int64), 1) for j in range(self.n)]

    def key(self):
        """Sorted int64 keys col*n+row of E's lower positions (CSC order)."""
        cols = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.colptr))
        return cols * self.n + self.rowind.astype(np.int64)


def analyse(n, perm, a_row, a_col) -> Structure:
    return Structure(n, elimination_game(n, perm, a_row, a_col))


def check_invariants(S: Structure, perm, a_row, a_col, full=True):
    """Chordality, pattern cover, supernode partition and running intersection.

    P:228-252 / S:192-195: every {j} u struct(j) is a clique of E (perfect
    elimination ordering); aggregate pattern subset of E; {S_r} partitions
    0..n-1; each U_r lies inside the clique of a later supernode (RIP).
    Returns a list of violation strings (empty = ok).
    """
    bad = []
    n = S.n
    iperm = np.empty(n, dtype=np.int64)
    iperm[np.asarray(perm, dtype=np.int64)] = np.arange(n)
    keys = S.key()
    keyset = keys  # sorted

    def inE(r, c):
        k = np.asarray(c, dtype=np.int64) * n + np.asarray(r, dtype=np.int64)
        p = np.searchsorted(keyset, k)
        p = np.minimum(p, keyset.size - 1)
        return keyset[p] == k

    ar = iperm[np.asarray(a_row, dtype=np.int64)]
    ac = iperm[np.asarray(a_col, dtype=np.int64)]
    if not np.all(inE(np.maximum(ar, ac), np.minimum(ar, ac))):
        bad.append("aggregate pattern not inside E")
    cols = range(n) if full else range(0, n, max(1, n // 2000))
    for j in cols:
        s = S.struct[j]
        if s.size > 1:
            r, c = np.meshgrid(s, s, indexing="ij")
            m = r > c
            if not np.all(inE(r[m], c[m])):
                bad.append(f"struct({j}) not a clique")
                break
    sp = S.super_ptr
    if sp[0] != 0 or sp[-1] != n or np.any(np.diff(sp) <= 0):
        bad.append("supernodes do not partition 0..n-1")
    cl = S.cliques()
    first_col = np.repeat(np.arange(len(cl)), np.diff(sp))
    for r, (C, s) in enumerate(cl):
        U = C[s:]
        if U.size == 0:
            continue
        # U_r must lie in the clique C of the supernode containing min(U_r)
        r2 = int(first_col[U[0]])
        if r2 <= r or not np.all(np.isin(U, cl[r2][0])):
            bad.append(f"running intersection fails at clique {r}")
            break
    return bad
