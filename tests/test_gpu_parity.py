"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bars (BASELINE.json north_star): structure/ordering/supernode indexing bit-exact; B within
1e-10 relative Frobenius (lower triangle, or full sampled columns on the big configs);
Cholesky factor within 1e-10 of LAPACK potrf applied to the GPU's own B.
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import algorithm1 as A1  # noqa: E402
from oracle import cholesky as CH  # noqa: E402
from oracle import ldl as LDL  # noqa: E402
from oracle import scm as SCM  # noqa: E402
from oracle import symbolic as SYM  # noqa: E402
from tests.helpers import small, three_by_three  # noqa: E402

TOL_B = 1e-10
TOL_R = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def run_gpu(inst, ld=None, chol=True):
    from paper_1310_6919_b200 import Handle
    dev = torch.device("cuda:0")
    m = inst.m
    ld = m if ld is None else ld
    h = Handle.from_instance(inst)
    st = h.get_structure()
    out = dict(h=h, st=st)
    x = torch.from_numpy(inst.xbar).to(dev)
    y = torch.from_numpy(inst.y).to(dev)
    h.factor_xinv(x)
    L = torch.empty(st["nnzE"], dtype=torch.float64, device=dev)
    D = torch.empty(inst.n, dtype=torch.float64, device=dev)
    h.get_xinv_factor(L, D)
    out["L"], out["D"] = L.cpu().numpy(), D.cpu().numpy()
    Bt = torch.full((m, ld), float("nan"), dtype=torch.float64, device=dev)  # B(i,j) = Bt[j, i]
    h.scm_build(y, Bt, ld)
    h.get_y_factor(L, D)
    out["Ly"], out["Dy"] = L.cpu().numpy(), D.cpu().numpy()
    out["Bt"] = Bt
    if m <= 12000:
        out["B"] = Bt[:, :m].T.cpu().numpy().copy()
    if chol:
        out["info"] = h.scm_cholesky(Bt, ld)
        if m <= 12000:
            out["R"] = np.tril(Bt[:, :m].T.cpu().numpy())
    return out


def oracle_dense(inst):
    S = SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)
    L, D = A1.factor_xinv(S, inst.xbar)
    Ly, Dy = LDL.ldl_on_E(S, inst.y)
    Xh = SCM.dense_completion(S, L, D, inst.perm)
    Yi = SCM.dense_y_inverse(S, inst.y, inst.perm)
    B = SCM.scm_dense(inst, Xh, Yi)
    return dict(S=S, L=L, D=D, Ly=Ly, Dy=Dy, B=B, Xh=Xh, Yi=Yi)


def check_all(inst, g, o):
    S = o["S"]
    st = g["st"]
    # (a0) structure, bit-exact
    assert np.array_equal(st["perm"], inst.perm)
    assert np.array_equal(st["colptr"], S.colptr) and np.array_equal(st["rowind"], S.rowind)
    assert np.array_equal(st["parent"], S.parent)
    assert np.array_equal(st["super_ptr"], S.super_ptr)
    # (a1), (a2)
    assert rel(g["L"], o["L"]) < 1e-11 and rel(g["D"], o["D"]) < 1e-11
    assert rel(g["Ly"], o["Ly"]) < 1e-11 and rel(g["Dy"], o["Dy"]) < 1e-11
    # (b)+(c): lower triangle of B
    lo = np.tril_indices(inst.m)
    eb = rel(g["B"][lo], o["B"][lo])
    assert eb < TOL_B, eb
    # (d): against LAPACK potrf of the GPU's own B
    assert g["info"] == 0
    Ro = CH.potrf_lower(g["B"])
    er = rel(g["R"], Ro)
    assert er < TOL_R, er
    assert CH.backward_error(g["B"], g["R"]) < 1e-14
    return eb, er


def test_3x3_worked_example():
    for kind in ("maxcut", "theta"):
        inst, gold = three_by_three(kind)
        g = run_gpu(inst)
        np.testing.assert_allclose(g["L"], gold["L_E"], atol=1e-15)
        np.testing.assert_allclose(g["D"], gold["D"], atol=1e-15)
        key = "B_maxcut" if kind == "maxcut" else "B_theta"
        Bg = np.tril(g["B"])
        np.testing.assert_allclose(Bg, np.tril(gold[key].reshape(3, 3)), atol=1e-13)
        if kind == "maxcut":
            np.testing.assert_allclose(g["R"], gold["R_maxcut"].reshape(3, 3), atol=1e-14)


@pytest.mark.parametrize("kind", ["maxcut_md", "maxcut_nd", "theta", "blockarrow", "maxcut3d"])
def test_small_instances(kind):
    inst = small(kind)
    check_all(inst, run_gpu(inst), oracle_dense(inst))


@pytest.mark.parametrize("seed", [1, 2])
def test_small_seeds_and_padded_ld(seed):
    inst = small("theta", seed=seed)
    o = oracle_dense(inst)
    check_all(inst, run_gpu(inst, ld=inst.m + 3), o)      # odd padded leading dimension
    check_all(inst, run_gpu(inst, ld=inst.m + 8), o)


def test_config0():
    from instances import gen_config
    inst = gen_config(0)
    check_all(inst, run_gpu(inst), oracle_dense(inst))


def test_config2_theta_full():
    """configs[2]: n = 3600, m = 7201 (odd: ragged tiles, 8-byte staging path), dense oracle."""
    from instances import gen_config
    inst = gen_config(2)
    check_all(inst, run_gpu(inst), oracle_dense(inst))


def test_upper_triangle_untouched():
    inst = small("maxcut_nd")
    g = run_gpu(inst)
    up = np.triu_indices(inst.m, 1)
    Bu = g["Bt"][:, :inst.m].T.cpu().numpy()
    assert np.all(np.isnan(Bu[up]))


def test_degenerate_single_vertex():
    from tests.helpers import manual_instance
    inst = manual_instance(1, [([0], [0], [1.0]), ([0], [0], [2.0])],
                           colptr=np.array([0, 1]), rowind=np.array([0], dtype=np.int32),
                           xbar=np.array([4.0]), y=np.array([0.5]))
    g = run_gpu(inst)
    # X-hat = 4, Y^{-1} = 2, A_1 = 2 e e^T: B = trace(A X A Y^{-1}) = 2*4*2*2 = 32, R = sqrt(32)
    assert abs(g["B"][0, 0] - 32.0) < 1e-13 and abs(g["R"][0, 0] - np.sqrt(32.0)) < 1e-13
    assert abs(g["D"][0] - 0.25) < 1e-16


def test_not_pd_clique_reports_index():
    from paper_1310_6919_b200 import SdpcError
    from paper_1310_6919_b200.sdpc import SDPC_ERR_NOT_PD
    inst, _ = three_by_three()
    inst.xbar = inst.xbar.copy()
    inst.xbar[4] = 0.1          # clique C_2 = {2,3} indefinite (oracle test_algorithm1_not_pd_reports_clique)
    with pytest.raises(SdpcError) as e:
        run_gpu(inst)
    assert e.value.status == SDPC_ERR_NOT_PD and e.value.info == 1


def test_not_pd_y_reports_column():
    from paper_1310_6919_b200 import SdpcError
    inst, _ = three_by_three()
    inst.y = inst.y.copy()
    inst.y[2] = -1.0
    with pytest.raises(SdpcError) as e:
        run_gpu(inst)
    assert e.value.info == 1


def test_cholesky_not_pd_reports_leading_minor():
    """LAPACK potrf rule: info = order of the first non-PD leading minor (exact cases)."""
    inst, _ = three_by_three()
    from paper_1310_6919_b200 import Handle
    h = Handle.from_instance(inst)
    dev = torch.device("cuda:0")
    Bt = torch.tensor([[4.0, 2.0, 0.0], [2.0, 1.0, 0.0], [0.0, 0.0, 1.0]], dtype=torch.float64, device=dev)
    assert h.scm_cholesky(Bt, 3, raise_not_pd=False) == 2          # exactly singular 2x2 minor
    Bt = torch.diag(torch.tensor([1.0, 2.0, -1.0], dtype=torch.float64, device=dev))
    assert h.scm_cholesky(Bt, 3, raise_not_pd=False) == 3


@pytest.mark.parametrize("sched", [1, 0])
def test_cholesky_not_pd_deep_index(sched):
    """Failing pivot beyond the first panels (m = 7201): info = 5001 (both schedules)."""
    from instances import gen_config
    from paper_1310_6919_b200 import Handle
    inst = gen_config(2)
    h = Handle.from_instance(inst)
    h.set_cholesky_schedule(sched)
    m = inst.m
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(3)
    G = torch.randn(m, 64, dtype=torch.float64, device=dev, generator=g)
    Bt = G @ G.T / 64 + torch.eye(m, dtype=torch.float64, device=dev)
    Bt[5000, 5000] = -1.0
    assert h.scm_cholesky(Bt, m, raise_not_pd=False) == 5001


def test_iteration_host_matches_device_path():
    from instances import gen_config
    from paper_1310_6919_b200 import Handle
    inst = gen_config(0)
    g = run_gpu(inst)
    h = Handle.from_instance(inst)
    rd = np.zeros(inst.m)
    info = h.iteration_host(inst.xbar, inst.y, rd)
    assert info == 0
    np.testing.assert_allclose(rd, np.diag(g["R"]), rtol=1e-14)


def _full_columns(Bt, cols, m):
    out = []
    for l in cols:
        out.append(torch.cat([Bt[:l, l], Bt[l, l:m]]).cpu().numpy())
    return np.stack(out, axis=1)


def _sampled(inst, seed=1, nsample=1000):
    rng = np.random.default_rng(seed + 1)
    cols = set(rng.choice(inst.m, size=min(nsample, inst.m), replace=False).tolist())
    cols |= {0, inst.m - 1}
    sizes = np.diff(inst.a_ptr)[1:]
    cols.add(int(np.argmax(sizes)))
    return sorted(cols)


@pytest.mark.parametrize("cfg", [1, 3, 4, 5])
def test_full_config_sampled_columns(cfg):
    """configs[1], [3], [4], [5] at full size: both factors, >= 1000 sampled columns of B, plus free checks."""
    from instances import gen_config
    inst = gen_config(cfg)
    S = SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)
    g = run_gpu(inst, chol=False)
    st = g["st"]
    assert np.array_equal(st["colptr"], S.colptr) and np.array_equal(st["rowind"], S.rowind)
    assert np.array_equal(st["super_ptr"], S.super_ptr)
    L, D = A1.factor_xinv(S, inst.xbar)
    assert rel(g["L"], L) < 1e-11 and rel(g["D"], D) < 1e-11
    # (a2) at full size: the multifrontal factor of Y against the oracle's up-looking LDL^T on E
    Ly, Dy = LDL.ldl_on_E(S, inst.y)
    assert rel(g["Ly"], Ly) < 1e-11 and rel(g["Dy"], Dy) < 1e-11
    cols = _sampled(inst)
    solver = SCM.ColumnSolver(S, L, D, inst.y, inst.perm)
    Bo = SCM.scm_columns(inst, cols, solver)
    Bg = _full_columns(g["Bt"], cols, inst.m)
    e = rel(Bg, Bo)
    assert e < TOL_B, e
    # Cholesky at full size: probes ||B v - R (R^T v)|| / ||B v||
    Bt = g["Bt"]
    m = inst.m
    Bl = torch.tril(Bt[:, :m].T)
    V = torch.randn(m, 16, dtype=torch.float64, device=Bt.device, generator=torch.Generator(device=Bt.device).manual_seed(0))
    BV = Bl @ V + torch.tril(Bl, -1).T @ V
    del Bl
    info = g["h"].scm_cholesky(Bt, m)
    assert info == 0
    R = torch.tril(Bt[:, :m].T)
    res = torch.linalg.norm(BV - R @ (R.T @ V)) / torch.linalg.norm(BV)
    assert float(res) < 1e-13


@pytest.mark.parametrize("m", [1, 31, 128, 129, 255, 256, 257, 383, 513, 1000, 1311, 2100])
@pytest.mark.parametrize("pad,sched", [(0, 1), (0, 0), (1, 1)])
def test_cholesky_random_spd_ragged(m, pad, sched):
    """(d) alone: random SPD B of sizes around the 128/256 block edges; the task-graph kernel (even ld,
    sched 1), the multi-launch schedule (sched 0) and odd ld (8-byte staging, falls back to the
    multi-launch schedule); R against LAPACK potrf; strict upper triangle untouched."""
    from tests.helpers import scm_handle
    h = scm_handle(m)
    h.set_cholesky_schedule(sched)
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(m * 7 + pad)
    G = rng.standard_normal((m, m + 8))
    Bh = G @ G.T / (m + 8) + 0.5 * np.eye(m)
    ld = m + pad
    Bt = torch.full((m, ld), float("nan"), dtype=torch.float64, device=dev)   # B(i, j) = Bt[j, i]
    Bt[:, :m] = torch.from_numpy(np.tril(Bh).T.copy()).to(dev)
    Bt[:, :m] = torch.where(torch.from_numpy(np.tril(np.ones((m, m))).T.copy()).to(dev) > 0, Bt[:, :m],
                            torch.tensor(float("nan"), dtype=torch.float64, device=dev))
    assert h.scm_cholesky(Bt, ld) == 0
    Rg = Bt[:, :m].T.cpu().numpy()
    up = np.triu_indices(m, 1)
    assert np.all(np.isnan(Rg[up]))
    Ro = CH.potrf_lower(Bh)
    assert rel(np.tril(Rg), Ro) < TOL_R
    assert CH.backward_error(Bh, np.tril(Rg)) < 1e-14


@pytest.mark.parametrize("kind", ["maxcut_nd", "theta"])
def test_inverse_columns_free_check(kind):
    """(a1)+(b) at once: x_p = X-hat e_p restricted to the pattern equals X-bar (max-det completion,
    SURVEY §8(c) free check), and Y y_q = e_q; full (untruncated) columns via sdpc_get_inverse_columns."""
    from paper_1310_6919_b200 import Handle
    inst = small(kind)
    dev = torch.device("cuda:0")
    h = Handle.from_instance(inst)
    h.set_truncation(False)
    x = torch.from_numpy(inst.xbar).to(dev)
    y = torch.from_numpy(inst.y).to(dev)
    h.factor_xinv(x)
    Bt = torch.zeros((inst.m, inst.m), dtype=torch.float64, device=dev)
    h.scm_build(y, Bt)
    n = inst.n
    cols = np.arange(0, n, max(1, n // 17), dtype=np.int32)
    Xo = torch.zeros((len(cols), n), dtype=torch.float64, device=dev)   # column c at Xo[c]
    Yo = torch.zeros_like(Xo)
    h.get_inverse_columns(cols, Xo, Yo)
    Xo, Yo = Xo.cpu().numpy(), Yo.cpu().numpy()
    perm = np.asarray(inst.perm)
    iperm = np.argsort(perm)
    Ydense = np.zeros((n, n))
    for j in range(n):
        for e in range(inst.colptr[j], inst.colptr[j + 1]):
            i = inst.rowind[e]
            a, b = perm[i], perm[j]
            Ydense[a, b] = Ydense[b, a] = inst.y[e]
    for ci, p in enumerate(cols):
        jp = iperm[p]                               # elimination index of column p
        # pattern entries of column p (both triangles): X-hat_ip = X-bar_ip
        for j in range(n):
            for e in range(inst.colptr[j], inst.colptr[j + 1]):
                i = inst.rowind[e]
                if j == jp:
                    assert abs(Xo[ci][perm[i]] - inst.xbar[e]) < 1e-11 * (1 + abs(inst.xbar[e]))
                elif i == jp:
                    assert abs(Xo[ci][perm[j]] - inst.xbar[e]) < 1e-11 * (1 + abs(inst.xbar[e]))
        r = Ydense @ Yo[ci]
        r[p] -= 1.0
        assert np.max(np.abs(r)) < 1e-11


def test_truncated_and_full_sweeps_agree():
    """max-cut: the truncated backward sweep (default) and the full one give the same B."""
    from paper_1310_6919_b200 import Handle
    inst = small("maxcut_nd")
    dev = torch.device("cuda:0")
    out = []
    for tr in (True, False):
        h = Handle.from_instance(inst)
        h.set_truncation(tr)
        h.factor_xinv(torch.from_numpy(inst.xbar).to(dev))
        Bt = torch.full((inst.m, inst.m), float("nan"), dtype=torch.float64, device=dev)
        h.scm_build(torch.from_numpy(inst.y).to(dev), Bt)
        out.append(np.tril(Bt.T.cpu().numpy()))
    assert rel(out[0], out[1]) < 1e-14


@pytest.mark.parametrize("kind", ["maxcut_nd", "theta", "blockarrow"])
def test_fused_iteration_matches_separate_calls(kind):
    """sdpc_iteration ((a1) || (a2), then (b), (c), (d), one sync) = the three separate calls."""
    from paper_1310_6919_b200 import Handle
    inst = small(kind)
    g = run_gpu(inst)
    dev = torch.device("cuda:0")
    h = Handle.from_instance(inst)
    Bt = torch.full((inst.m, inst.m), float("nan"), dtype=torch.float64, device=dev)
    info = h.iteration(torch.from_numpy(inst.xbar).to(dev), torch.from_numpy(inst.y).to(dev), Bt)
    assert info == 0
    R = np.tril(Bt.T.cpu().numpy())
    assert rel(R, g["R"]) < 1e-13
    assert np.all(np.isnan(Bt.T.cpu().numpy()[np.triu_indices(inst.m, 1)]))


def test_fused_iteration_not_pd_phases():
    from paper_1310_6919_b200 import Handle, SdpcError
    inst, _ = three_by_three()
    dev = torch.device("cuda:0")
    x = torch.from_numpy(inst.xbar).to(dev)
    y = torch.from_numpy(inst.y).to(dev)
    B = torch.zeros((3, 3), dtype=torch.float64, device=dev)
    xb = x.clone()
    xb[4] = 0.1                      # clique 1 indefinite -> (a1) fails first
    with pytest.raises(SdpcError) as e:
        Handle.from_instance(inst).iteration(xb, y, B)
    assert e.value.info == 1
    yb = y.clone()
    yb[2] = -1.0                     # Y not PD at column 1 -> (a2)
    with pytest.raises(SdpcError) as e:
        Handle.from_instance(inst).iteration(x, yb, B)
    assert e.value.info == 1


@pytest.mark.parametrize("m,nrhs", [(1, 1), (129, 2), (1000, 1), (1311, 3), (2048, 1), (3000, 4)])
def test_sce_solve_with_scm_factor(m, nrhs):
    """NEXT row 2 (SCE): sdpc_scm_solve with the factor of sdpc_scm_cholesky against the
    oracle's LAPACK solve, ragged sizes and several right-hand sides."""
    from tests.helpers import scm_handle
    h = scm_handle(m)
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(m + nrhs)
    G = rng.standard_normal((m, m + 4))
    Bh = G @ G.T / (m + 4) + 0.5 * np.eye(m)
    # even ld: the sweeps use the diagonal-tile inverses (16-byte staging); odd m: the serial triangles
    ld = m + (m & 1) if m % 3 else m
    Bt = torch.zeros((m, ld), dtype=torch.float64, device=dev)
    Bt[:, :m] = torch.from_numpy(np.tril(Bh).T.copy()).to(dev)    # column-major lower
    assert h.scm_cholesky(Bt, ld) == 0
    Rhs = rng.standard_normal((m, nrhs))
    Gt = torch.from_numpy(Rhs.T.copy()).to(dev)                    # column-major m x nrhs
    h.scm_solve(Bt, Gt, ld, m, nrhs)
    X = Gt.cpu().numpy().T
    Xo = CH.sce_solve(Bh, Rhs)
    assert rel(X, Xo) < 1e-10
    assert np.linalg.norm(Bh @ X - Rhs) / np.linalg.norm(Rhs) < 1e-12


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_iteration_bitwise_reproducible(cfg):
    """Two sdpc_iteration calls on the same inputs give bitwise identical factors B = R R^T (no atomic
    accumulation anywhere on the path: fixed-order extend-add in (a2), one update order per Cholesky
    tile), and identical L_Y."""
    from instances import gen_config
    from paper_1310_6919_b200 import Handle
    inst = gen_config(cfg)
    h = Handle.from_instance(inst)
    dev = torch.device("cuda:0")
    x = torch.from_numpy(inst.xbar).to(dev)
    y = torch.from_numpy(inst.y).to(dev)
    m = inst.m
    ld = m + (m & 1)
    outs = []
    for _ in range(2):
        Bt = torch.zeros((m, ld), dtype=torch.float64, device=dev)
        assert h.iteration(x, y, Bt, ld) == 0
        Ly = torch.empty(int(inst.colptr[-1]), dtype=torch.float64, device=dev)
        Dy = torch.empty(inst.n, dtype=torch.float64, device=dev)
        h.get_y_factor(Ly, Dy)
        outs.append((Bt.cpu().numpy(), Ly.cpu().numpy(), Dy.cpu().numpy()))
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ["maxcut_md", "theta"])
def test_builtin_minimum_degree_ordering(kind):
    """perm == NULL: the library's exact minimum degree (ties -> smallest original id, SURVEY §8(c)
    reading #5) equals the generator's elimination-game MD bit for bit, and E follows."""
    from instances import orderings
    from instances.generate import aggregate_edges
    from paper_1310_6919_b200 import Handle
    inst = small(kind)
    h = Handle.from_instance(inst, with_perm=False)
    st = h.get_structure()
    edges = aggregate_edges(inst.n, inst.a_row, inst.a_col)
    perm = orderings.minimum_degree(inst.n, edges)
    assert np.array_equal(st["perm"], perm)
    S = SYM.analyse(inst.n, perm, inst.a_row, inst.a_col)
    assert np.array_equal(st["colptr"], S.colptr) and np.array_equal(st["rowind"], S.rowind)
    h2 = Handle.from_instance(gen_config_md0(), with_perm=False)
    assert np.array_equal(h2.get_structure()["perm"], gen_config_md0().perm)


def gen_config_md0():
    from instances import gen_config
    return gen_config(0)


@pytest.mark.parametrize("cfg", [1, 3])
def test_cholesky_full_size_elementwise(cfg):
    """(d) at full size, element-wise against LAPACK potrf of the GPU's own B:
    ||R_gpu - R_lapack||_F / ||R_lapack||_F <= 1e-10, and the backward error ||B - R R^T||_F / ||B||_F <= 1e-14
    (LAPACK's own is ~2e-16 here, the GPU factor's ~5e-16)."""
    from instances import gen_config
    inst = gen_config(cfg)
    g = run_gpu(inst, ld=inst.m + (inst.m & 1), chol=False)
    m = inst.m
    B = np.tril(g["Bt"][:, :m].T.cpu().numpy())
    assert g["h"].scm_cholesky(g["Bt"], m + (m & 1)) == 0
    R = np.tril(g["Bt"][:, :m].T.cpu().numpy())
    Ro = CH.potrf_lower(B)
    assert rel(R, Ro) < TOL_R
    assert CH.backward_error(B, R) <= 1e-14
