"""GPU parity of SURVEY §8(f) NEXT rows 1-3 (sdpc_search_direction, sdpc_step_lengths) against the oracle
(oracle/direction.py): g, dz, dY and the P-MATRIX dX on E within 1e-10 relative; the step lengths feasible
and within the bisection bracket of the oracle's eigenvalue step."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from instances import direction_G  # noqa: E402
from oracle import algorithm1 as A1  # noqa: E402
from oracle import direction as DIR  # noqa: E402
from oracle import scm as SCM  # noqa: E402
from oracle import symbolic as SYM  # noqa: E402
from tests.helpers import small, three_by_three  # noqa: E402

TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def gpu_direction(inst, G_E, bmu, truncate=True):
    from paper_1310_6919_b200 import Handle
    dev = torch.device("cuda:0")
    m, nnz = inst.m, int(inst.colptr[-1])
    h = Handle.from_instance(inst)
    h.set_truncation(truncate)
    x = torch.from_numpy(inst.xbar).to(dev)
    y = torch.from_numpy(inst.y).to(dev)
    ld = m + (m & 1)
    Bt = torch.zeros((m, ld), dtype=torch.float64, device=dev)
    h.factor_xinv(x)
    h.scm_build(y, Bt, ld)
    assert h.scm_cholesky(Bt, ld) == 0
    G = torch.from_numpy(G_E).to(dev)
    g = torch.empty(m, dtype=torch.float64, device=dev)
    dz = torch.empty(m, dtype=torch.float64, device=dev)
    dY = torch.empty(nnz, dtype=torch.float64, device=dev)
    dX = torch.empty(nnz, dtype=torch.float64, device=dev)
    h.search_direction(x, G, bmu, Bt, ld, g, dz, dY, dX)
    return dict(h=h, x=x, y=y, g=g.cpu().numpy(), dz=dz.cpu().numpy(), dY=dY.cpu().numpy(), dX=dX.cpu().numpy(),
                dYt=dY, dXt=dX)


def oracle_direction(inst, G_E, bmu):
    S = SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)
    L, D = A1.factor_xinv(S, inst.xbar)
    Xh = SCM.dense_completion(S, L, D, inst.perm)
    Yi = SCM.dense_y_inverse(S, inst.y, inst.perm)
    B = SCM.scm_dense(inst, Xh, Yi)
    G = DIR.dense_on_E(S, G_E, inst.perm)
    g = DIR.g_vector(inst, Xh, Yi, G, bmu)
    dz = DIR.sce(B, g)
    dY = DIR.dY_dense(inst, G, dz)
    dX = DIR.dX_dense(Xh, Yi, dY, bmu)
    return dict(S=S, g=g, dz=dz, dY=DIR.values_on_E(S, dY, inst.perm), dX=DIR.values_on_E(S, dX, inst.perm))


def _instances():
    return [("3x3maxcut", lambda: three_by_three("maxcut")[0]), ("3x3theta", lambda: three_by_three("theta")[0]),
            ("maxcut_md", lambda: small("maxcut_md")), ("maxcut_nd", lambda: small("maxcut_nd")),
            ("theta", lambda: small("theta"))]


@pytest.mark.parametrize("name,make", _instances())
@pytest.mark.parametrize("truncate", [True, False])
def test_direction_matches_oracle(name, make, truncate):
    inst = make()
    G_E = direction_G(inst, seed=5)
    S = SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)
    bmu = 0.3 * DIR.mu(S, inst.xbar, inst.y)
    gpu = gpu_direction(inst, G_E, bmu, truncate)
    o = oracle_direction(inst, G_E, bmu)
    for key in ("g", "dz", "dY", "dX"):
        assert rel(gpu[key], o[key]) < TOL, (key, rel(gpu[key], o[key]))


@pytest.mark.parametrize("cfg", [0, 2])
def test_direction_configs(cfg):
    from instances import gen_config
    inst = gen_config(cfg)
    G_E = direction_G(inst)
    S = SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)
    bmu = 0.3 * DIR.mu(S, inst.xbar, inst.y)
    gpu = gpu_direction(inst, G_E, bmu)
    o = oracle_direction(inst, G_E, bmu)
    for key in ("g", "dz", "dY", "dX"):
        assert rel(gpu[key], o[key]) < TOL, (key, rel(gpu[key], o[key]))


def test_direction_config1_sampled_columns():
    """configs[1] at full size: dX on the E entries of sampled columns by the column-wise oracle route
    (Eq. newdX2) with the GPU's dY; g at sampled constraints; dY from the GPU's dz exactly."""
    from instances import gen_config
    inst = gen_config(1)
    G_E = direction_G(inst)
    S = SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)
    bmu = 0.3 * DIR.mu(S, inst.xbar, inst.y)
    gpu = gpu_direction(inst, G_E, bmu)
    # dY = G - diag(dz) at the constraint vertices (max-cut), else G
    dY_o = G_E.copy()
    diag = S.colptr[:-1]
    vert_of_col = np.asarray(inst.perm)          # elimination column j <-> original vertex perm[j] = constraint
    dY_o[diag] -= gpu["dz"][vert_of_col]
    assert rel(gpu["dY"], dY_o) < 1e-14
    L, D = A1.factor_xinv(S, inst.xbar)
    solver = SCM.ColumnSolver(S, L, D, inst.y, inst.perm)
    rng = np.random.default_rng(2)
    cols_new = np.sort(rng.choice(inst.n, size=64, replace=False))
    cols = np.asarray(inst.perm)[cols_new]
    dYd = DIR.dense_on_E(S, gpu["dY"], inst.perm)
    dXh = DIR.dX_columns(solver, dYd, bmu, cols)               # columns of dX-hat (original ids)
    # dX = (dX-hat + dX-hat^T)/2: entry (i, j) on E of column j needs dX-hat_ij and dX-hat_ji; compare the
    # rows i of each sampled column j whose own column i is also sampled
    dXd = DIR.dense_on_E(S, gpu["dX"], inst.perm)
    pos = {c: a for a, c in enumerate(cols)}
    err, ref = 0.0, 0.0
    for a, j in enumerate(cols):
        for i in cols:
            if dXd[i, j] != 0.0 or i == j:
                v = 0.5 * (dXh[i, a] + dXh[j, pos[i]])
                err = max(err, abs(dXd[i, j] - v))
                ref = max(ref, abs(v))
    assert err <= 1e-10 * ref
    # g at sampled constraints: g_k = bmu Y^{-1}_kk - X-bar_kk - (X-hat G Y^{-1})_kk (max-cut)
    Gd = DIR.dense_on_E(S, G_E, inst.perm)
    Yk = solver.y(cols)
    Xk = solver.x(cols)
    for a, k in enumerate(cols):
        gk = bmu * Yk[k, a] - Xk[k, a] - Xk[:, a] @ (Gd @ Yk[:, a])
        assert abs(gpu["g"][k] - gk) <= 1e-10 * max(1.0, abs(gk))


@pytest.mark.parametrize("kind", ["maxcut_md", "theta", "blockarrow"])
def test_step_lengths_match_oracle(kind):
    """alpha_p, alpha_d feasible and within the bisection bracket of the oracle's generalized-eigenvalue
    step (Eq. primal_length2), on directions scaled so that both are < 1."""
    from paper_1310_6919_b200 import Handle
    inst = small(kind)
    S = SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)
    dev = torch.device("cuda:0")
    dX_E = -3.0 * inst.xbar + direction_G(inst, seed=1)
    dY_E = -3.0 * inst.y + direction_G(inst, seed=2)
    h = Handle.from_instance(inst)
    t = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
    ap, ad = h.step_lengths(t(inst.xbar), t(dX_E), t(inst.y), t(dY_E))
    ap_o = DIR.primal_step(S, inst.xbar, dX_E)
    ad_o = DIR.dual_step(S, inst.y, dY_E, inst.perm)
    assert ap_o - 2.0 ** -39 <= ap <= ap_o * (1 + 1e-9)
    assert ad_o - 2.0 ** -29 <= ad <= ad_o * (1 + 1e-9)
    # closed forms: X-bar = Y = I on E, directions -2 I: both 1/2; 0 direction: both 1
    I_E = np.zeros(S.nnzE)
    I_E[S.colptr[:-1]] = 1.0
    ap, ad = h.step_lengths(t(I_E), t(-2.0 * I_E), t(I_E), t(-2.0 * I_E))
    assert 0.5 - 2.0 ** -39 <= ap <= 0.5 and 0.5 - 2.0 ** -29 <= ad <= 0.5
    ap, ad = h.step_lengths(t(I_E), t(0.0 * I_E), t(I_E), t(0.0 * I_E))
    assert ap == 1.0 and ad == 1.0


def test_step_lengths_after_direction():
    """The direction of the iteration feeds the step lengths (config 0)."""
    from instances import gen_config
    inst = gen_config(0)
    G_E = direction_G(inst)
    S = SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)
    bmu = 0.3 * DIR.mu(S, inst.xbar, inst.y)
    gpu = gpu_direction(inst, G_E, bmu)
    ap, ad = gpu["h"].step_lengths(gpu["x"], gpu["dXt"], gpu["y"], gpu["dYt"])
    ap_o = DIR.primal_step(S, inst.xbar, gpu["dX"])
    ad_o = DIR.dual_step(S, inst.y, gpu["dY"], inst.perm)
    assert ap_o - 2.0 ** -39 <= ap <= ap_o * (1 + 1e-9)
    assert ad_o - 2.0 ** -29 <= ad <= ad_o * (1 + 1e-9)
