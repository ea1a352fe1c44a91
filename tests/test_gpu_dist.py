"""GPU tests of the multi-GPU path on ONE GPU.

* Build: handles created with nranks = P, rank = r write exactly their 2D block-cyclic tiles of B
  (local addresses), equal to the single-rank B; the other local entries stay untouched.
* Cholesky: the P-rank schedule of dist.py with the CUDA tile kernels (sdpc_potrf_tile,
  sdpc_trsm_panel, sdpc_update_tiles), ranks emulated by host threads (ThreadComm) that only
  exchange tiles between complete kernels (no kernel waits on another rank), against LAPACK.
"""
from __future__ import annotations

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import cholesky as CH  # noqa: E402
from paper_1310_6919_b200 import dist as D  # noqa: E402
from tests.helpers import scm_handle, small  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()


def _single_B(inst):
    from paper_1310_6919_b200 import Handle
    dev = torch.device("cuda:0")
    h = Handle.from_instance(inst)
    x = torch.from_numpy(inst.xbar).to(dev)
    y = torch.from_numpy(inst.y).to(dev)
    h.factor_xinv(x)
    Bt = torch.full((inst.m, inst.m), float("nan"), dtype=torch.float64, device=dev)
    h.scm_build(y, Bt, inst.m)
    return np.tril(Bt.T.cpu().numpy())


@pytest.mark.parametrize("kind", ["maxcut_nd", "theta", "blockarrow"])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_dist_build_writes_own_tiles(kind, P):
    from paper_1310_6919_b200 import Handle
    from instances import gen_config
    inst = gen_config(2) if kind == "theta" else small(kind)
    Bref = _single_B(inst)
    dev = torch.device("cuda:0")
    x = torch.from_numpy(inst.xbar).to(dev)
    y = torch.from_numpy(inst.y).to(dev)
    for r in range(P):
        L = D.Layout(inst.m, P, r)
        h = Handle.from_instance(inst, nranks=P, rank=r)
        lay = h.get_scm_layout()
        assert (lay["Pr"], lay["Pc"], lay["myrow"], lay["mycol"], lay["mloc"], lay["nloc"]) == \
            (L.Pr, L.Pc, L.myrow, L.mycol, L.mloc, L.nloc)
        h.factor_xinv(x)
        Bt = torch.full((max(1, L.nloc), L.lld), float("nan"), dtype=torch.float64, device=dev)
        h.scm_build(y, Bt, L.lld)
        got = Bt[:L.nloc, :L.mloc].T.cpu().numpy()
        want = D.local_tiles_of(Bref, L)
        # owned lower entries equal the single-rank B; strict-upper parts of diagonal tiles and
        # tiles above the diagonal are never written
        mask = np.zeros_like(want, dtype=bool)
        for I in range(L.myrow, L.nt, L.Pr):
            for J in range(L.mycol, L.nt, L.Pc):
                if I < J:
                    continue
                r0, c0 = L.local_row_of_tile(I), L.local_col_of_tile(J)
                hgt, wid = L.tile_rows(I), L.tile_rows(J)
                blk = np.ones((hgt, wid), dtype=bool)
                if I == J:
                    blk = np.tril(blk)
                mask[r0:r0 + hgt, c0:c0 + wid] = blk
        assert np.all(np.isnan(got[~mask]))
        err = np.linalg.norm(got[mask] - want[mask]) / max(np.linalg.norm(want[mask]), 1e-300)
        assert err < 1e-13, (r, err)
        h.destroy()


def _run_threads(m, P, bad=None, seed=0):
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((m, m + 3))
    B = G @ G.T / (m + 3) + 0.5 * np.eye(m)
    if bad is not None:
        B[bad, bad] = -1.0
    layouts = [D.Layout(m, P, r) for r in range(P)]
    shared = D.ThreadComm.make_shared(layouts[0])
    results = [None] * P
    errors = []

    # the tile kernels only need the SCM order m and the process grid: each rank's handle is made
    # for a max-cut problem with m constraints and nranks = P, rank = r
    def worker(r):
        try:
            L = layouts[r]
            torch.cuda.set_device(0)
            h = scm_handle(L.m, L.P, L.rank)
            ops = h
            Bt = torch.zeros((max(1, L.nloc), L.lld), dtype=torch.float64, device=dev)
            Bt[:L.nloc, :L.mloc] = torch.from_numpy(D.local_tiles_of(np.tril(B), L).T.copy()).to(dev)
            comm = D.ThreadComm(L, shared, sync=torch.cuda.synchronize)
            info = D.dist_cholesky(ops, Bt, L, comm, dev)
            torch.cuda.synchronize()
            results[r] = (info, Bt[:L.nloc, :L.mloc].T.cpu().numpy())
            h.destroy()
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)
            for bar in [shared.world, *shared.col, *shared.row]:
                bar.abort()

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errors, errors
    return B, layouts, results


@pytest.mark.parametrize("m,P", [(700, 2), (1300, 4), (1100, 3), (2100, 8)])
def test_dist_cholesky_tile_kernels_threads(m, P):
    B, layouts, results = _run_threads(m, P, seed=m + P)
    R = CH.potrf_lower(B)
    for L, (info, got) in zip(layouts, results):
        assert info == 0
        want = D.local_tiles_of(R, L)
        # below-diagonal tiles and lower parts of diagonal tiles: R; strict upper of diagonal tiles:
        # untouched (zero, from tril(B))
        err = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)
        assert err < 1e-12, (L.rank, err)


def test_dist_cholesky_not_pd_threads():
    _, _, results = _run_threads(900, 4, bad=600, seed=5)
    assert all(info == 601 for info, _ in results)


# ---------------------------------------------------------------------------------------------- C-ABI
# sdpc_scm_cholesky for nranks > 1 lives in the library (dist_chol.cu): NCCL communicators created by
# sdpc_create from an sdpc_get_unique_id id, or the virtual-rank transport on one device.

def _virtual_factor(B_lower, P, seed_handles=None):
    """Distribute lower(B) over P virtual ranks, factor through sdpc_scm_cholesky_virtual, gather R."""
    from paper_1310_6919_b200.sdpc import scm_cholesky_virtual
    m = B_lower.shape[0]
    dev = torch.device("cuda:0")
    layouts = [D.Layout(m, P, r) for r in range(P)]
    hs = seed_handles or [scm_handle(m, P, r) for r in range(P)]
    lld = max(L.lld for L in layouts)
    Bts = []
    for L in layouts:
        Bt = torch.zeros((max(1, L.nloc), lld), dtype=torch.float64, device=dev)
        Bt[:L.nloc, :L.mloc] = torch.from_numpy(D.local_tiles_of(B_lower, L).T.copy()).to(dev)
        Bts.append(Bt)
    info = scm_cholesky_virtual(hs, Bts, lld)
    torch.cuda.synchronize()
    R = np.zeros((m, m))
    for L, Bt in zip(layouts, Bts):
        loc = Bt[:L.nloc, :L.mloc].T.cpu().numpy()
        for I in range(L.myrow, L.nt, L.Pr):
            for J in range(L.mycol, I + 1, L.Pc):
                r0, c0 = L.local_row_of_tile(I), L.local_col_of_tile(J)
                h, w = L.tile_rows(I), L.tile_rows(J)
                R[I * D.NB:I * D.NB + h, J * D.NB:J * D.NB + w] = loc[r0:r0 + h, c0:c0 + w]
    return info, np.tril(R)


@pytest.mark.parametrize("m,P", [(700, 2), (1300, 4), (1100, 3), (2100, 8), (1500, 6), (300, 4)])
def test_abi_virtual_ranks_cholesky(m, P):
    """The library's distributed schedule on P virtual ranks (one GPU) against LAPACK potrf."""
    rng = np.random.default_rng(m * 3 + P)
    G = rng.standard_normal((m, m + 5))
    B = G @ G.T / (m + 5) + 0.5 * np.eye(m)
    info, R = _virtual_factor(np.tril(B), P)
    assert info == 0
    Ro = CH.potrf_lower(B)
    assert np.linalg.norm(R - Ro) / np.linalg.norm(Ro) < 1e-12


def test_abi_virtual_ranks_not_pd():
    rng = np.random.default_rng(9)
    m = 900
    G = rng.standard_normal((m, m + 5))
    B = G @ G.T / (m + 5) + 0.5 * np.eye(m)
    B[600, 600] = -1.0
    info, _ = _virtual_factor(np.tril(B), 4)
    assert info == 601


@pytest.mark.parametrize("kind", ["maxcut_nd", "theta"])
@pytest.mark.parametrize("P", [2, 4])
def test_abi_distributed_build_and_cholesky_vs_oracle(kind, P):
    """Row (e) end to end through the C ABI: every virtual rank builds its 2D block-cyclic tiles of B
    (sdpc_scm_build, nranks = P), the ranks factor B collectively (sdpc_scm_cholesky_virtual); the
    gathered B is compared with the ORACLE's dense B and R with LAPACK potrf of the oracle's B."""
    from oracle import algorithm1 as A1, scm as SCM, symbolic as SYM
    from instances import gen_config
    from paper_1310_6919_b200 import Handle
    from paper_1310_6919_b200.sdpc import scm_cholesky_virtual
    inst = gen_config(2) if kind == "theta" else small(kind)
    m = inst.m
    S = SYM.analyse(inst.n, inst.perm, inst.a_row, inst.a_col)
    L0, D0 = A1.factor_xinv(S, inst.xbar)
    Bo = SCM.scm_dense(inst, SCM.dense_completion(S, L0, D0, inst.perm),
                       SCM.dense_y_inverse(S, inst.y, inst.perm))
    dev = torch.device("cuda:0")
    x = torch.from_numpy(inst.xbar).to(dev)
    y = torch.from_numpy(inst.y).to(dev)
    layouts = [D.Layout(m, P, r) for r in range(P)]
    lld = max(L.lld for L in layouts)
    hs, Bts = [], []
    for L in layouts:
        h = Handle.from_instance(inst, nranks=P, rank=L.rank)
        h.factor_xinv(x)
        Bt = torch.zeros((max(1, L.nloc), lld), dtype=torch.float64, device=dev)
        h.scm_build(y, Bt, lld)
        hs.append(h)
        Bts.append(Bt)
    Bg = np.zeros((m, m))
    for L, Bt in zip(layouts, Bts):
        loc = Bt[:L.nloc, :L.mloc].T.cpu().numpy()
        for I in range(L.myrow, L.nt, L.Pr):
            for J in range(L.mycol, I + 1, L.Pc):
                r0, c0 = L.local_row_of_tile(I), L.local_col_of_tile(J)
                h_, w_ = L.tile_rows(I), L.tile_rows(J)
                Bg[I * D.NB:I * D.NB + h_, J * D.NB:J * D.NB + w_] = loc[r0:r0 + h_, c0:c0 + w_]
    Bg = np.tril(Bg)
    lo = np.tril_indices(m)
    assert np.linalg.norm(Bg[lo] - Bo[lo]) / np.linalg.norm(Bo[lo]) < 1e-10
    assert scm_cholesky_virtual(hs, Bts, lld) == 0
    R = np.zeros((m, m))
    for L, Bt in zip(layouts, Bts):
        loc = Bt[:L.nloc, :L.mloc].T.cpu().numpy()
        for I in range(L.myrow, L.nt, L.Pr):
            for J in range(L.mycol, I + 1, L.Pc):
                r0, c0 = L.local_row_of_tile(I), L.local_col_of_tile(J)
                h_, w_ = L.tile_rows(I), L.tile_rows(J)
                R[I * D.NB:I * D.NB + h_, J * D.NB:J * D.NB + w_] = loc[r0:r0 + h_, c0:c0 + w_]
    Ro = CH.potrf_lower(Bo)
    assert np.linalg.norm(np.tril(R) - Ro) / np.linalg.norm(Ro) < 1e-10


def test_abi_nccl_communicator_one_rank():
    """sdpc_get_unique_id + sdpc_create with the id (an NCCL world of one rank and its row / column
    communicators): sdpc_scm_cholesky takes the collective path (NCCL broadcasts / all-gather / all-reduce
    on one rank) and matches LAPACK."""
    from paper_1310_6919_b200.sdpc import get_unique_id, Handle
    m = 1300
    uid = get_unique_id()
    assert len(uid) == 128
    a_ptr = np.arange(m + 2, dtype=np.int64) - 1
    a_ptr[0] = 0
    idx = np.arange(m, dtype=np.int32)
    h = Handle(m, m, a_ptr, idx, idx, np.ones(m), np.ones(m), None, 0, 1, 0, nccl_id=uid)
    rng = np.random.default_rng(4)
    G = rng.standard_normal((m, m + 5))
    B = G @ G.T / (m + 5) + 0.5 * np.eye(m)
    dev = torch.device("cuda:0")
    ld = m + (m & 1)
    Bt = torch.zeros((m, ld), dtype=torch.float64, device=dev)
    Bt[:, :m] = torch.from_numpy(np.tril(B).T.copy()).to(dev)
    assert h.scm_cholesky(Bt, ld) == 0
    R = np.tril(Bt[:, :m].T.cpu().numpy())
    Ro = CH.potrf_lower(B)
    assert np.linalg.norm(R - Ro) / np.linalg.norm(Ro) < 1e-12
    h.destroy()
