"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the fact it checks.  None of these compares the oracle with a
retyped copy of its own formula: the references are worked examples
(tests/golden/, cited), closed forms, textbook/LAPACK special cases,
invariants (max-det optimality, chordality, symmetry/SPD), brute force on tiny
inputs, and an independent implementation (the generator's selected inversion).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import algorithm1 as A1
from oracle import cholesky as CH
from oracle import ldl as LDL
from oracle import scm as SCM
from oracle import symbolic as SYM
from tests.helpers import load_golden, small, three_by_three


def _S(inst):
    return SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


# ----------------------------------------------------------------- worked examples

def test_3x3_structure_and_cliques():
    inst, g = three_by_three()
    S = _S(inst)
    assert S.colptr.tolist() == [0, 2, 4, 5] and S.rowind.tolist() == [0, 1, 1, 2, 2]
    # cliques C_1 = {1,2} (S_1={1}), C_2 = {2,3} (S_2 = {2,3}) in 0-based ids
    assert [(c.tolist(), s) for c, s in S.cliques()] == [([0, 1], 1), ([1, 2], 2)]


def test_3x3_algorithm1_literal_and_unit_form():
    inst, g = three_by_three()
    S = _S(inst)
    Lhat = A1.algorithm1(S, inst.xbar)
    np.testing.assert_allclose(Lhat, g["Lhat_E"], rtol=0, atol=1e-15)
    L, D = A1.unit_form(S, Lhat)
    np.testing.assert_allclose(L, g["L_E"], atol=1e-15)
    np.testing.assert_allclose(D, g["D"], atol=1e-15)
    L2, D2 = A1.columnwise_formula(S, inst.xbar)
    np.testing.assert_allclose(L2, g["L_E"], atol=1e-15)
    np.testing.assert_allclose(D2, g["D"], atol=1e-15)


def test_3x3_completion_and_scm_maxcut():
    inst, g = three_by_three("maxcut")
    S = _S(inst)
    L, D = A1.factor_xinv(S, inst.xbar)
    Xh = SCM.dense_completion(S, L, D, inst.perm)
    np.testing.assert_allclose(Xh.ravel(), g["Xhat"], atol=1e-14)
    spec = load_golden("spec_examples.txt")
    np.testing.assert_allclose(Xh[:, 2], spec["xhat_e3"], atol=1e-14)
    Yi = SCM.dense_y_inverse(S, inst.y, inst.perm)
    B = SCM.scm_dense(inst, Xh, Yi)
    np.testing.assert_allclose(B.ravel(), g["B_maxcut"], atol=1e-13)
    R = CH.potrf_lower(B)
    np.testing.assert_allclose(R.ravel(), g["R_maxcut"], atol=1e-14)


def test_3x3_scm_theta():
    inst, g = three_by_three("theta")
    S = _S(inst)
    L, D = A1.factor_xinv(S, inst.xbar)
    Xh = SCM.dense_completion(S, L, D, inst.perm)
    Yi = SCM.dense_y_inverse(S, inst.y, inst.perm)
    B = SCM.scm_dense(inst, Xh, Yi)
    np.testing.assert_allclose(B.ravel(), g["B_theta"], atol=1e-13)
    Bb = SCM.scm_bruteforce(inst, Xh, Yi)
    np.testing.assert_allclose(Bb.ravel(), g["B_theta"], atol=1e-13)


def test_spec_dense_examples():
    s = load_golden("spec_examples.txt")
    R = CH.potrf_lower(s["chol_in"].reshape(2, 2))
    np.testing.assert_allclose(R.ravel(), s["chol_out"], atol=1e-15)
    with pytest.raises(np.linalg.LinAlgError):
        CH.potrf_lower(s["notpd_in"].reshape(2, 2))


def test_diag_single_clique_S265():
    """X-bar = diag(4, 9) with one clique -> L-hat = diag(1/2, 1/3)."""
    from tests.helpers import manual_instance
    s = load_golden("spec_examples.txt")
    colptr = np.array([0, 2, 3], dtype=np.int64)
    rowind = np.array([0, 1, 1], dtype=np.int32)
    inst = manual_instance(2, [([1], [0], [1.0]), ([0], [0], [1.0]), ([1], [1], [1.0])],
                           colptr=colptr, rowind=rowind, xbar=np.array([4.0, 0.0, 9.0]))
    S = _S(inst)
    Lhat = A1.algorithm1(S, inst.xbar)
    np.testing.assert_allclose(Lhat[S.colptr[:-1]], s["diag_Lhat"], atol=1e-15)
    assert Lhat[1] == 0.0


# ----------------------------------------------------------------- closed forms

def _two_clique_instance(rng):
    """E = C1 x C1 u C2 x C2 with C1 = {0..3}, C2 = {2..6}; S = {0,1}, U = {2,3}, T = {4,5,6}."""
    from tests.helpers import manual_instance
    n = 7
    C1, C2 = range(0, 4), range(2, 7)
    pos = sorted({(max(a, b), min(a, b)) for C in (C1, C2) for a in C for b in C})
    r = [p[0] for p in pos]
    c = [p[1] for p in pos]
    mats = [(r, c, np.ones(len(r)))] + [([i], [i], [1.0]) for i in range(n)]
    G = rng.standard_normal((n, n))
    M = G @ G.T + n * np.eye(n)
    inst = manual_instance(n, mats)
    S = _S(inst)
    cols = np.repeat(np.arange(n), np.diff(S.colptr))
    inst.xbar = M[S.rowind, cols]
    return inst, S, M


def test_two_clique_closed_form_lemma26():
    """X-hat_ST = X-bar_SU X-bar_UU^{-1} X-bar_UT."""
    inst, S, M = _two_clique_instance(np.random.default_rng(3))
    L, D = A1.factor_xinv(S, inst.xbar)
    Xh = SCM.dense_completion(S, L, D, inst.perm)
    Sx, U, T = [0, 1], [2, 3], [4, 5, 6]
    ref = M[np.ix_(Sx, U)] @ np.linalg.solve(M[np.ix_(U, U)], M[np.ix_(U, T)])
    np.testing.assert_allclose(Xh[np.ix_(Sx, T)], ref, rtol=1e-12, atol=1e-13)
    # on E the completion reproduces X-bar (Grone et al.)
    for C in (range(0, 4), range(2, 7)):
        np.testing.assert_allclose(Xh[np.ix_(C, C)], M[np.ix_(C, C)], rtol=1e-13)


def test_single_clique_is_lapack_inverse():
    """E dense: one clique, X-hat = X-bar and L-hat L-hat^T = X-bar^{-1} (LAPACK special case)."""
    from tests.helpers import manual_instance
    n = 9
    rng = np.random.default_rng(5)
    G = rng.standard_normal((n, n))
    M = G @ G.T + np.eye(n)
    r, c = np.tril_indices(n)
    order = np.lexsort((r, c))
    inst = manual_instance(n, [(r[order], c[order], np.ones(r.size)), (np.arange(n), np.arange(n), np.ones(n))])
    S = _S(inst)
    assert len(S.cliques()) == 1
    cols = np.repeat(np.arange(n), np.diff(S.colptr))
    xbar = M[S.rowind, cols]
    Lhat = A1.algorithm1(S, xbar)
    import scipy.sparse as sp
    Lh = sp.csc_matrix((Lhat, S.rowind, S.colptr), shape=(n, n)).toarray()
    np.testing.assert_allclose(Lh @ Lh.T, np.linalg.inv(M), rtol=1e-12, atol=1e-13)


# ----------------------------------------------------------------- invariants

@pytest.mark.parametrize("kind", ["maxcut_md", "maxcut_nd", "theta", "blockarrow"])
def test_roundtrip_generator_factor(kind):
    """Generator (L, D) -> selected inversion -> X-bar -> Algorithm 1 recovers (L, D) (A.2/A.5)."""
    inst = small(kind)
    S = _S(inst)
    L, D = A1.factor_xinv(S, inst.xbar)
    assert np.max(np.abs(L - inst.L)) < 1e-13
    assert np.max(np.abs(D - inst.D) / inst.D) < 1e-13
    Lc, Dc = A1.columnwise_formula(S, inst.xbar)         # partition independence (A.2)
    assert np.max(np.abs(Lc - L)) < 1e-13 and np.max(np.abs(Dc - D) / D) < 1e-13
    Lcc, Dcc = A1.factor_xinv(S, inst.xbar, S.column_cliques())
    assert np.max(np.abs(Lcc - L)) < 1e-13 and np.max(np.abs(Dcc - D) / D) < 1e-13


def test_roundtrip_config0():
    from instances import gen_config
    inst = gen_config(0)
    S = _S(inst)
    L, D = A1.factor_xinv(S, inst.xbar)
    assert np.max(np.abs(L - inst.L)) < 1e-14
    assert np.max(np.abs(D - inst.D) / inst.D) < 1e-14


@pytest.mark.parametrize("kind", ["maxcut_md", "theta", "blockarrow"])
def test_maxdet_optimality(kind):
    """X-hat|_E = X-bar; (X-hat^{-1})_ij = 0 off E exactly; off-E perturbation lowers log det."""
    inst = small(kind)
    S = _S(inst)
    n = inst.n
    L, D = A1.factor_xinv(S, inst.xbar)
    import scipy.sparse as sp
    Ls = sp.csc_matrix((L, S.rowind, S.colptr), shape=(n, n)).toarray()
    Xinv = (Ls * D) @ Ls.T
    Xh_new = np.linalg.inv(Xinv)
    cols = np.repeat(np.arange(n), np.diff(S.colptr))
    np.testing.assert_allclose(Xh_new[S.rowind, cols], inst.xbar, rtol=1e-12, atol=1e-14)
    inE = np.zeros((n, n), dtype=bool)
    inE[S.rowind, cols] = True
    inE |= inE.T
    assert np.all(Xinv[~inE] == 0.0)
    base = np.linalg.slogdet(Xh_new)[1]
    rng = np.random.default_rng(1)
    off = np.argwhere(~inE & (np.arange(n)[:, None] > np.arange(n)[None, :]))
    for (i, j) in off[rng.choice(len(off), size=min(10, len(off)), replace=False)]:
        for eps in (1e-3, -1e-3):
            P = Xh_new.copy()
            P[i, j] += eps
            P[j, i] += eps
            assert np.linalg.slogdet(P)[1] < base


@pytest.mark.parametrize("kind", ["maxcut_md", "maxcut_nd", "theta", "blockarrow", "maxcut3d"])
def test_symbolic_matches_generator_and_invariants(kind):
    inst = small(kind)
    S = _S(inst)
    assert np.array_equal(S.colptr, inst.colptr) and np.array_equal(S.rowind, inst.rowind)
    assert SYM.check_invariants(S, inst.perm, inst.a_row, inst.a_col) == []


def test_blockarrow_nnz_closed_form():
    inst = small("blockarrow")
    nb, bs, bd = 4, 6, 3
    S = _S(inst)
    assert S.nnzE == nb * (bs * (bs + 1) // 2 + bs * bd) + bd * (bd + 1) // 2
    assert len(S.cliques()) == nb + 1


@pytest.mark.parametrize("cfg,nnz,nsuper", [(0, 886, 74), (2, 101289, 2699)])
def test_symbolic_counts_survey(cfg, nnz, nsuper):
    """nnz(E) and supernode counts from SURVEY.md A.1 (independent scratch computation)."""
    from instances import gen_config
    inst = gen_config(cfg)
    S = _S(inst)
    assert S.nnzE == nnz and len(S.super_ptr) - 1 == nsuper
    assert np.array_equal(S.rowind, inst.rowind)
    assert SYM.check_invariants(S, inst.perm, inst.a_row, inst.a_col, full=(cfg == 0)) == []


def test_symbolic_counts_config1():
    from instances import gen_config
    inst = gen_config(1)
    S = _S(inst)
    assert S.nnzE == 359561 and len(S.super_ptr) - 1 == 6656
    assert np.array_equal(S.rowind, inst.rowind)


@pytest.mark.parametrize("kind", ["maxcut_md", "theta", "blockarrow"])
def test_ldl_of_Y(kind):
    """Left-looking LDL^T of Y recovers the generator's (L_Y, D_Y); dense LAPACK special case."""
    inst = small(kind)
    S = _S(inst)
    Ly, Dy = LDL.ldl_on_E(S, inst.y)
    assert np.max(np.abs(Ly - inst.Ly)) < 1e-13 and np.max(np.abs(Dy - inst.Dy) / inst.Dy) < 1e-13
    n = inst.n
    import scipy.sparse as sp
    Yl = sp.csc_matrix((inst.y, S.rowind, S.colptr), shape=(n, n)).toarray()
    C = np.linalg.cholesky(Yl + np.tril(Yl, -1).T)
    np.testing.assert_allclose(Dy, np.diag(C) ** 2, rtol=1e-12)


def test_ldl_not_pd_index():
    inst, g = three_by_three()
    S = _S(inst)
    y = inst.y.copy()
    y[2] = -1.0                                   # Y_11 (0-based) made negative
    with pytest.raises(LDL.NotPositiveDefinite) as e:
        LDL.ldl_on_E(S, y)
    assert e.value.index == 1


@pytest.mark.parametrize("kind", ["maxcut_md", "theta", "blockarrow"])
def test_scm_dense_vs_bruteforce_and_properties(kind):
    inst = small(kind)
    S = _S(inst)
    L, D = A1.factor_xinv(S, inst.xbar)
    Xh = SCM.dense_completion(S, L, D, inst.perm)
    Yi = SCM.dense_y_inverse(S, inst.y, inst.perm)
    B = SCM.scm_dense(inst, Xh, Yi)
    Bb = SCM.scm_bruteforce(inst, Xh, Yi)
    assert _rel(B, Bb) < 1e-13
    assert _rel(B, B.T) < 1e-14                           # symmetric
    assert np.linalg.eigvalsh(B).min() > 0                # SPD: vec(A_k) independent
    if inst.kind == "maxcut":                             # B = X-hat o Y^{-1}
        assert _rel(B, Xh * Yi) < 1e-14
    if inst.kind == "theta":                              # B_11 = trace(X-hat Y^{-1})
        assert abs(B[0, 0] - np.trace(Xh @ Yi)) < 1e-12 * abs(B[0, 0])


def test_scm_theta_identity_iterate():
    """X-hat = Y = I gives B_kl = A_k . A_l: B_11 = n, B_ee = 2, B_1e = 0 (A.3)."""
    inst = small("theta")
    n = inst.n
    Xh = np.eye(n)
    B = SCM.scm_dense(inst, Xh, np.eye(n))
    assert B[0, 0] == n
    assert np.all(np.diag(B)[1:] == 2.0)
    assert np.all(B[0, 1:] == 0.0) and np.all(B[1:, 0] == 0.0)


@pytest.mark.parametrize("kind", ["maxcut_md", "maxcut_nd", "theta", "blockarrow"])
def test_sampled_columns_match_dense(kind):
    """Sampled route (per-RHS solves, Eq. newSCM2) vs dense route: the oracle noise floor."""
    inst = small(kind)
    S = _S(inst)
    L, D = A1.factor_xinv(S, inst.xbar)
    Xh = SCM.dense_completion(S, L, D, inst.perm)
    Yi = SCM.dense_y_inverse(S, inst.y, inst.perm)
    B = SCM.scm_dense(inst, Xh, Yi)
    solver = SCM.ColumnSolver(S, L, D, inst.y, inst.perm)
    cols = list(range(inst.m))
    Bc = SCM.scm_columns(inst, cols, solver)
    assert _rel(Bc, B) < 1e-12
    # free check: x_p restricted to E equals X-bar
    x = solver.x(np.arange(inst.n))
    iperm = np.empty(inst.n, dtype=np.int64)
    iperm[inst.perm] = np.arange(inst.n)
    cols_new = np.repeat(np.arange(inst.n), np.diff(S.colptr))
    xv = x[inst.perm[S.rowind], inst.perm[cols_new]]
    np.testing.assert_allclose(xv, inst.xbar, rtol=1e-12, atol=1e-14)


def test_cholesky_backward_error():
    inst = small("theta")
    S = _S(inst)
    L, D = A1.factor_xinv(S, inst.xbar)
    Xh = SCM.dense_completion(S, L, D, inst.perm)
    Yi = SCM.dense_y_inverse(S, inst.y, inst.perm)
    B = SCM.scm_dense(inst, Xh, Yi)
    R = CH.potrf_lower(B)
    assert CH.backward_error(B, R) < 1e-15
    assert np.all(np.diag(R) > 0) and np.all(np.triu(R, 1) == 0)


def test_algorithm1_not_pd_reports_clique():
    inst, g = three_by_three()
    S = _S(inst)
    x = inst.xbar.copy()
    x[4] = 0.1                 # X-bar_33 = 0.1 makes clique C_2 = {2,3} indefinite (det = 0.2 - 1 < 0)
    with pytest.raises(A1.NotPositiveDefinite) as e:
        A1.algorithm1(S, x)
    assert e.value.index == 1


def test_sce_solve_worked_example_and_residual():
    """SCE B dz = g: SPEC's 2x2 B = [[4,2],[2,5]] with g = (2, 1) gives
    dz = B^{-1} g = (1/16)[[5,-2],[-2,4]] (2, 1) = (1/2, 0) exactly; random SPD: residual and
    multi-RHS = columnwise."""
    from oracle import cholesky as CHO
    x = CHO.sce_solve(np.array([[4.0, 2.0], [2.0, 5.0]]), np.array([2.0, 1.0]))
    np.testing.assert_allclose(x, [0.5, 0.0], atol=1e-15)
    rng = np.random.default_rng(5)
    G = rng.standard_normal((60, 70))
    B = G @ G.T / 70 + np.eye(60)
    Rhs = rng.standard_normal((60, 3))
    X = CHO.sce_solve(np.tril(B), Rhs)
    assert np.linalg.norm(B @ X - Rhs) / np.linalg.norm(Rhs) < 1e-13
    for q in range(3):
        np.testing.assert_allclose(CHO.sce_solve(B, Rhs[:, q]), X[:, q], rtol=1e-12, atol=1e-14)


def test_torus3d_workload_shape():
    """NEXT 4: the 3D torus has n = p^3 vertices of degree 6 (3 p^3 edges); the 3D geometric
    ND is a permutation whose E is chordal with the oracle's elimination game."""
    from instances import graphs, orderings
    for p in (4, 5, 6):
        e = graphs.torus3d_edges(p)
        assert e.shape == (3 * p ** 3, 2)
        deg = np.bincount(e.ravel(), minlength=p ** 3)
        assert np.all(deg == 6)
        perm = orderings.torus3d_nested_dissection(p)
        assert np.array_equal(np.sort(perm), np.arange(p ** 3))
    inst = small("maxcut3d")
    S = _S(inst)
    assert np.array_equal(S.colptr, inst.colptr) and np.array_equal(S.rowind, inst.rowind)
