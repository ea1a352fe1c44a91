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
