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
