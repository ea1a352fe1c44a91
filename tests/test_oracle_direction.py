"""Pins of the oracle search direction and step lengths (oracle/direction.py), SURVEY §8(f) NEXT rows 1-3.

Each pin is fixed by the paper or by mathematics, not by re-typing the oracle's formula:
closed forms where the identities cancel, the
central-path fixed point, the HKM linearised complementarity the direction solves, the column-wise
route of Eq. newdX2 against the dense route, and boundary properties of the step lengths.
"""
from __future__ import annotations

import numpy as np
import pytest

from instances import direction_G, product_on_E
from oracle import algorithm1 as A1
from oracle import direction as DIR
from oracle import scm as SCM
from oracle import symbolic as SYM
from tests.helpers import small, three_by_three


def _S(inst):
    return SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)


def _identity_E(S):
    v = np.zeros(S.nnzE)
    v[S.colptr[:-1]] = 1.0          # diagonal = first entry of each column
    return v


def test_g_identity_iterate_closed_forms():
    """X-hat = Y = I: beta mu = 1 gives g_k = -A_k . G; G = 0, beta mu = 2 gives g_k = trace(A_k)
    (S:375).  Max-cut on the 3x3 pattern: A_k = e_k e_k^T; theta: A_1 = I, A_2 = E_12, A_3 = E_23."""
    for kind in ("maxcut", "theta"):
        inst, _ = three_by_three(kind)
        I = np.eye(3)
        G = np.array([[0.5, -0.25, 0.0], [-0.25, 2.0, 0.75], [0.0, 0.75, -1.0]])
        g = DIR.g_vector(inst, I, I, G, 1.0)
        if kind == "maxcut":
            np.testing.assert_allclose(g, [-0.5, -2.0, 1.0], atol=1e-15)
        else:
            np.testing.assert_allclose(g, [-(0.5 + 2.0 - 1.0), -2 * -0.25, -2 * 0.75], atol=1e-15)
        g2 = DIR.g_vector(inst, I, I, np.zeros((3, 3)), 2.0)
        np.testing.assert_allclose(g2, [1, 1, 1] if kind == "maxcut" else [3, 0, 0], atol=1e-15)


def test_dY_maxcut_structure():
    """Max-cut (A_k = e_k e_k^T): dY = G - diag(dz) exactly."""
    inst, _ = three_by_three("maxcut")
    G = np.arange(9.0).reshape(3, 3)
    G = G + G.T
    dz = np.array([0.5, -1.0, 2.0])
    np.testing.assert_array_equal(DIR.dY_dense(inst, G, dz), G - np.diag(dz))


@pytest.mark.parametrize("kind", ["maxcut_md", "theta"])
def test_central_path_fixed_point(kind):
    """X-hat = beta mu Y^{-1} and dY = 0 give dX = 0 (the fixed point of Eq. dX)."""
    inst = small(kind)
    S = _S(inst)
    L, D = A1.factor_xinv(S, inst.xbar)
    Xh = SCM.dense_completion(S, L, D, inst.perm)
    bmu = 0.7
    Yi = Xh / bmu                          # Y = bmu X-hat^{-1} = bmu L D L^T lies on E
    dX = DIR.dX_dense(Xh, Yi, np.zeros_like(Xh), bmu)
    assert np.abs(dX).max() < 1e-12 * np.abs(Xh).max()


@pytest.mark.parametrize("kind", ["maxcut_md", "theta", "blockarrow"])
def test_direction_solves_hkm_system(kind):
    """The direction satisfies the HKM linearised complementarity it is defined from,
    dX-hat Y + X-hat dY = beta mu I - X-hat Y (P:376 rearranged), and dY + sum A_k dz_k = G with
    B dz = g; checked densely with independent products."""
    inst = small(kind)
    S = _S(inst)
    L, D = A1.factor_xinv(S, inst.xbar)
    Xh = SCM.dense_completion(S, L, D, inst.perm)
    Yi = SCM.dense_y_inverse(S, inst.y, inst.perm)
    Y = DIR.dense_on_E(S, inst.y, inst.perm)
    G = DIR.dense_on_E(S, direction_G(inst), inst.perm)
    bmu = 0.3 * DIR.mu(S, inst.xbar, inst.y)
    B = SCM.scm_dense(inst, Xh, Yi)
    g = DIR.g_vector(inst, Xh, Yi, G, bmu)
    dz = DIR.sce(B, g)
    np.testing.assert_allclose(B @ dz, g, rtol=1e-10, atol=1e-12 * np.abs(g).max())
    dY = DIR.dY_dense(inst, G, dz)
    S_A = sum(dz[k - 1] * DIR.constraint_dense(inst, k) for k in range(1, inst.m + 1))
    np.testing.assert_allclose(dY + S_A, G, atol=1e-12 * max(1.0, np.abs(G).max()))
    dXh = bmu * Yi - Xh - Xh @ dY @ Yi
    lhs = dXh @ Y + Xh @ dY
    rhs = bmu * np.eye(inst.n) - Xh @ Y
    assert np.abs(lhs - rhs).max() < 1e-9 * max(1.0, np.abs(rhs).max())
    np.testing.assert_allclose(DIR.dX_dense(Xh, Yi, dY, bmu), 0.5 * (dXh + dXh.T), atol=1e-14)


@pytest.mark.parametrize("kind", ["maxcut_nd", "theta"])
def test_pmatrix_columnwise_route_matches_dense(kind):
    """Eq. newdX2 column by column through the factor solves equals the dense dX-hat."""
    inst = small(kind)
    S = _S(inst)
    L, D = A1.factor_xinv(S, inst.xbar)
    Xh = SCM.dense_completion(S, L, D, inst.perm)
    Yi = SCM.dense_y_inverse(S, inst.y, inst.perm)
    solver = SCM.ColumnSolver(S, L, D, inst.y, inst.perm)
    dY = DIR.dense_on_E(S, direction_G(inst, seed=3), inst.perm)
    bmu = 0.25
    cols = list(range(0, inst.n, 3))
    col = DIR.dX_columns(solver, dY, bmu, cols)
    dXh = bmu * Yi - Xh - Xh @ dY @ Yi
    np.testing.assert_allclose(col, dXh[:, cols], atol=1e-12 * np.abs(dXh).max())


def test_mu_scaled_identity():
    """mu = X . Y / n: X-bar = Y = lambda I gives mu = lambda^2."""
    inst = small("maxcut_md")
    S = _S(inst)
    lam = 100.0
    I_E = _identity_E(S)
    assert DIR.mu(S, lam * I_E, lam * I_E) == pytest.approx(lam * lam, rel=1e-15)


def test_step_length_closed_forms():
    """alpha_p with X-bar = I on every clique: dX = -I gives 1, dX = -2I gives 1/2,
    dX >= 0 gives 1; alpha_d with Y = I: dY = -2I gives 1/2, dY = 0 gives 1."""
    inst = small("maxcut_md")
    S = _S(inst)
    I_E = _identity_E(S)
    assert DIR.primal_step(S, I_E, -I_E) == 1.0
    assert DIR.primal_step(S, I_E, -2.0 * I_E) == pytest.approx(0.5, rel=1e-14)
    assert DIR.primal_step(S, I_E, np.abs(direction_G(inst)) * 0 + I_E) == 1.0
    assert DIR.dual_step(S, I_E, -2.0 * I_E, inst.perm) == pytest.approx(0.5, rel=1e-14)
    assert DIR.dual_step(S, I_E, 0.0 * I_E, inst.perm) == 1.0


@pytest.mark.parametrize("kind", ["maxcut_md", "theta"])
def test_step_lengths_are_boundary_points(kind):
    """At alpha_p the binding clique block is singular and every block is PD slightly before it
    (Eq. primal_length2); the same for alpha_d and Y + alpha dY."""
    inst = small(kind)
    S = _S(inst)
    dX_E = -3.0 * inst.xbar + direction_G(inst, seed=1)
    ap = DIR.primal_step(S, inst.xbar, dX_E)
    assert 0.0 < ap < 1.0
    keys = S.key()
    mins = []
    for C, _ in S.cliques():
        X = A1.gather_dense(S.n, keys, inst.xbar, C)
        dX = A1.gather_dense(S.n, keys, dX_E, C)
        assert np.linalg.eigvalsh(X + ap * (1 - 1e-9) * dX).min() > 0
        mins.append(np.linalg.eigvalsh(X + ap * dX).min() / np.linalg.eigvalsh(X).max())
    assert abs(min(mins)) < 1e-10
    Y = DIR.dense_on_E(S, inst.y, inst.perm)
    dY_E = -3.0 * inst.y + direction_G(inst, seed=2)
    dY = DIR.dense_on_E(S, dY_E, inst.perm)
    ad = DIR.dual_step(S, inst.y, dY_E, inst.perm)
    assert 0.0 < ad < 1.0
    assert np.linalg.eigvalsh(Y + ad * (1 - 1e-9) * dY).min() > 0
    assert abs(np.linalg.eigvalsh(Y + ad * dY).min()) < 1e-10 * np.linalg.eigvalsh(Y).max()


def test_values_on_E_roundtrip():
    inst = small("theta")
    S = _S(inst)
    v = direction_G(inst)
    np.testing.assert_array_equal(DIR.values_on_E(S, DIR.dense_on_E(S, v, inst.perm), inst.perm), v)
