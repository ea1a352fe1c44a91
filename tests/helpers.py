"""Test helpers: golden-file parsing and hand-built tiny instances."""
from __future__ import annotations

import math
import os
from fractions import Fraction

import numpy as np

from instances.generate import Instance

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _val(tok: str) -> float:
    if "sqrt" in tok:
        return float(eval(tok, {"__builtins__": {}}, {"sqrt": lambda x: math.sqrt(float(Fraction(x)) if isinstance(x, str) else x)}))
    return float(Fraction(tok))


def load_golden(name: str) -> dict:
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line or "=" not in line:
                continue
            k, v = line.split("=", 1)
            out[k.strip()] = np.array([_val(t) for t in v.split()])
    return out


def manual_instance(n, mats, perm=None, xbar=None, y=None, colptr=None, rowind=None, L=None, D=None,
                    Ly=None, Dy=None, b=None, kind="general", name="manual"):
    """Instance from explicit lower-triplet matrices [(rows, cols, vals)] for k = 0..m."""
    ptr = np.zeros(len(mats) + 1, dtype=np.int64)
    for k, (r, _, _) in enumerate(mats):
        ptr[k + 1] = ptr[k] + len(r)
    rows = np.concatenate([np.asarray(r, dtype=np.int32) for r, _, _ in mats])
    cols = np.concatenate([np.asarray(c, dtype=np.int32) for _, c, _ in mats])
    vals = np.concatenate([np.asarray(v, dtype=np.float64) for _, _, v in mats])
    m = len(mats) - 1
    z = lambda k: np.zeros(k)
    nnz = int(colptr[-1]) if colptr is not None else 0
    return Instance(name=name, n=n, m=m, a_ptr=ptr, a_row=rows, a_col=cols, a_val=vals,
                    b=np.zeros(m) if b is None else b,
                    perm=np.arange(n, dtype=np.int32) if perm is None else np.asarray(perm, dtype=np.int32),
                    colptr=colptr if colptr is not None else np.zeros(n + 1, dtype=np.int64),
                    rowind=rowind if rowind is not None else np.zeros(0, dtype=np.int32),
                    L=L if L is not None else z(nnz), D=D if D is not None else z(n),
                    Ly=Ly if Ly is not None else z(nnz), Dy=Dy if Dy is not None else z(n),
                    xbar=xbar if xbar is not None else z(nnz), y=y if y is not None else z(nnz), kind=kind)


def three_by_three(kind="maxcut"):
    g = load_golden("three_by_three.txt")
    colptr = np.array([0, 2, 4, 5], dtype=np.int64)
    rowind = np.array([0, 1, 1, 2, 2], dtype=np.int32)
    A0 = ([0, 1, 1, 2, 2], [0, 0, 1, 1, 2], [1.0, 1.0, 1.0, 1.0, 1.0])   # pattern = tridiagonal
    if kind == "maxcut":
        mats = [A0] + [([i], [i], [1.0]) for i in range(3)]
    else:  # theta on the path 1-2-3
        mats = [A0, ([0, 1, 2], [0, 1, 2], [1.0, 1.0, 1.0]), ([1], [0], [1.0]), ([2], [1], [1.0])]
    return manual_instance(3, mats, colptr=colptr, rowind=rowind, xbar=g["xbar_E"], y=g["y_E"],
                           L=g["L_E"], D=g["D"], Ly=g["L_E"], Dy=g["D"], kind=kind, name="3x3" + kind), g


def small(kind, seed=0):
    """Small seeded instances that span several tiles/supernodes (not BASELINE configs)."""
    from instances import build
    if kind == "maxcut_md":
        return build("maxcut", seed=seed, k=6, order="md", name="maxcut6md")
    if kind == "maxcut_nd":
        return build("maxcut", seed=seed, k=8, order="nd", name="maxcut8nd")
    if kind == "theta":
        return build("theta", seed=seed, k=5, order="md", name="theta5")
    if kind == "blockarrow":
        return build("blockarrow", seed=seed, nblk=4, bsz=6, border=3, m=40, name="blockarrow4x6")
    if kind == "maxcut3d":
        return build("maxcut3d", seed=seed, p=6, order="nd3", name="maxcut3d6")
    raise ValueError(kind)


def scm_handle(m, nranks=1, rank=0):
    """A handle whose SCM has order m (max-cut on m isolated vertices, A_k = e_k e_k^T), for tests
    that drive the SCM Cholesky entries on a B of their own."""
    from paper_1310_6919_b200 import Handle
    a_ptr = np.arange(m + 2, dtype=np.int64) - 1
    a_ptr[0] = 0
    idx = np.arange(m, dtype=np.int32)
    return Handle(m, m, a_ptr, idx, idx, np.ones(m), np.ones(m), None, 0, nranks, rank)
