"""Elimination orderings (inputs to the method, SURVEY.md §8(c) reading #5).

The paper permutes Y "with an appropriate order like approximation minimum
ordering" (§2.1) and uses CHOLMOD's AMD, whose
ties are unspecified.  Here the ordering is an INPUT written by the generator:

* exact minimum degree on the elimination graph, ties -> smallest original id
  (configs 0 and 2);
* a geometric nested dissection of the k x k torus (configs 1 and 4), exactly
  the rule stated in SURVEY.md §8(d) "Geometric ND";
* identity (config 3, the block-arrow pattern is already chordal in that order).

All return perm with perm[new] = old.
"""
from __future__ import annotations

import heapq

import numpy as np


def minimum_degree(n: int, edges: np.ndarray) -> np.ndarray:
    """Exact minimum degree via the elimination game; ties -> smallest original id."""
    adj = [set() for _ in range(n)]
    for a, b in edges:
        a = int(a); b = int(b)
        if a != b:
            adj[a].add(b)
            adj[b].add(a)
    heap = [(len(adj[v]), v) for v in range(n)]
    heapq.heapify(heap)
    done = np.zeros(n, dtype=bool)
    order = []
    while heap:
        d, v = heapq.heappop(heap)
        if done[v] or d != len(adj[v]):
            continue  # stale entry
        done[v] = True
        order.append(v)
        nb = adj[v]
        for u in nb:
            au = adj[u]
            au.discard(v)
            au |= nb
            au.discard(u)
            heapq.heappush(heap, (len(au), u))
        adj[v] = set()
    return np.asarray(order, dtype=np.int32)


def _rect(r0, r1, c0, c1, k, out):
    h = r1 - r0
    w = c1 - c0
    if h <= 0 or w <= 0:
        return
    if h * w <= 4:
        for r in range(r0, r1):
            for c in range(c0, c1):
                out.append(r * k + c)
        return
    if w >= h:
        mid = (c0 + c1) // 2
        _rect(r0, r1, c0, mid, k, out)
        _rect(r0, r1, mid + 1, c1, k, out)
        for r in range(r0, r1):
            out.append(r * k + mid)
    else:
        mid = (r0 + r1) // 2
        _rect(r0, mid, c0, c1, k, out)
        _rect(mid + 1, r1, c0, c1, k, out)
        for c in range(c0, c1):
            out.append(mid * k + c)


def torus_nested_dissection(k: int) -> np.ndarray:
    """Geometric nested dissection of the k x k torus (k even), SURVEY.md §8(d)."""
    if k % 2:
        raise ValueError("geometric ND needs even k")
    h = k // 2
    out: list[int] = []
    _rect(1, h, 1, h, k, out)
    _rect(1, h, h + 1, k, k, out)
    _rect(h + 1, k, 1, h, k, out)
    _rect(h + 1, k, h + 1, k, k, out)
    for c in range(k):
        out.append(0 * k + c)
    for c in range(k):
        out.append(h * k + c)
    for r in range(k):
        if r not in (0, h):
            out.append(r * k + 0)
    for r in range(k):
        if r not in (0, h):
            out.append(r * k + h)
    perm = np.asarray(out, dtype=np.int32)
    assert perm.size == k * k and np.unique(perm).size == k * k
    return perm


def _box(lo, hi, p, out):
    """Geometric ND of the open box [lo, hi) (3 dims): split the longest side at its middle plane,
    order both halves, then the plane (lexicographic x, y, z)."""
    ext = [hi[d] - lo[d] for d in range(3)]
    if min(ext) <= 0:
        return
    if ext[0] * ext[1] * ext[2] <= 8:
        for x in range(lo[0], hi[0]):
            for y in range(lo[1], hi[1]):
                for z in range(lo[2], hi[2]):
                    out.append((x * p + y) * p + z)
        return
    d = int(np.argmax(ext))
    mid = (lo[d] + hi[d]) // 2
    h1, l2 = list(hi), list(lo)
    h1[d] = mid
    l2[d] = mid + 1
    _box(lo, h1, p, out)
    _box(l2, hi, p, out)
    pl, ph = list(lo), list(hi)
    pl[d], ph[d] = mid, mid + 1
    for x in range(pl[0], ph[0]):
        for y in range(pl[1], ph[1]):
            for z in range(pl[2], ph[2]):
                out.append((x * p + y) * p + z)


def torus3d_nested_dissection(p: int) -> np.ndarray:
    """Geometric ND of the p x p x p torus (the 3D analogue of the 2D rule of SURVEY §8(d)):
    the top separator is the six planes x, y, z in {0, p/2}, ordered last (x-planes, then y-planes minus
    what is already taken, then z-planes); before it the eight open octants [1, h) or [h+1, p) per axis,
    each ordered by recursive bisection of its longest side."""
    h = p // 2
    out: list[int] = []
    for ox in ((1, h), (h + 1, p)):
        for oy in ((1, h), (h + 1, p)):
            for oz in ((1, h), (h + 1, p)):
                _box([ox[0], oy[0], oz[0]], [ox[1], oy[1], oz[1]], p, out)
    seen = np.zeros(p ** 3, dtype=bool)
    seen[out] = True
    for d in range(3):
        for c in (0, h):
            for a in range(p):
                for b in range(p):
                    xyz = [a, b]
                    xyz.insert(d, c)
                    v = (xyz[0] * p + xyz[1]) * p + xyz[2]
                    if not seen[v]:
                        seen[v] = True
                        out.append(v)
    perm = np.asarray(out, dtype=np.int32)
    assert perm.size == p ** 3 and np.unique(perm).size == p ** 3
    return perm
