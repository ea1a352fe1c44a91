"""Graphs and patterns of the five synthetic workloads (input recipe only).

The paper's workloads are lattice graphs (§4 "Max-clique
problems over lattice graphs") used by the max-clique and max-cut
 relaxations.  BASELINE.json's configs use the *toroidal* 2D lattice
(SURVEY.md §8(c) reading #6), plus a synthetic block-arrow pattern (config 3).

Nothing here computes any step of the method; it only lists vertices and edges.
"""
from __future__ import annotations

import numpy as np


def torus_edges(k: int) -> np.ndarray:
    """Edges of the k x k toroidal lattice, vertex id v = r*k + c.

    Each vertex connects to its right and down neighbour (wrapping).  Edges are
    returned as (min id, max id) rows sorted lexicographically (SURVEY §8(d),
    "Edges are listed sorted by (min id, max id)").  k >= 3 gives 2*k*k edges.
    """
    if k < 3:
        raise ValueError("torus needs k >= 3")
    r, c = np.divmod(np.arange(k * k, dtype=np.int64), k)
    right = r * k + (c + 1) % k
    down = ((r + 1) % k) * k + c
    v = np.arange(k * k, dtype=np.int64)
    a = np.concatenate([v, v])
    b = np.concatenate([right, down])
    e = np.stack([np.minimum(a, b), np.maximum(a, b)], axis=1)
    e = np.unique(e, axis=0)  # sorted, and guards k where wraps would coincide
    return e


def block_arrow_lower_pattern(nblk: int, bsz: int, border: int):
    """Lower-triangle (incl. diagonal) pattern of the block-arrow matrix of config 3.

    nblk dense bsz x bsz diagonal blocks followed by a dense `border`-wide border
    (rows/columns n-border..n-1 couple to everything).  Returned as (rows, cols)
    int64 arrays in column-major order (columns ascending, rows ascending).
    """
    n = nblk * bsz + border
    rows, cols = [], []
    b0 = nblk * bsz
    for b in range(nblk):
        lo = b * bsz
        for j in range(lo, lo + bsz):
            rr = np.concatenate([np.arange(j, lo + bsz), np.arange(b0, n)])
            rows.append(rr)
            cols.append(np.full(rr.shape, j))
    for j in range(b0, n):
        rr = np.arange(j, n)
        rows.append(rr)
        cols.append(np.full(rr.shape, j))
    return np.concatenate(rows).astype(np.int64), np.concatenate(cols).astype(np.int64), n


def torus3d_edges(p: int) -> np.ndarray:
    """Edges of the p x p x p toroidal lattice (6 neighbours), vertex id v = (x*p + y)*p + z: the shape of
    the paper's 3D spin-glass set (Table 3 SpinGlass18-25).
    Edges as (min id, max id) rows sorted lexicographically; p >= 3 gives 3 p^3 edges."""
    if p < 3:
        raise ValueError("torus needs p >= 3")
    v = np.arange(p ** 3, dtype=np.int64)
    x, rem = np.divmod(v, p * p)
    y, z = np.divmod(rem, p)
    nb = [((x + 1) % p * p + y) * p + z, (x * p + (y + 1) % p) * p + z, (x * p + y) * p + (z + 1) % p]
    a = np.concatenate([v, v, v])
    b = np.concatenate(nb)
    e = np.stack([np.minimum(a, b), np.maximum(a, b)], axis=1)
    return np.unique(e, axis=0)
