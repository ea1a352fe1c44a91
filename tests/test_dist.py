"""Multi-process (gloo, CPU) tests of the distributed SCM Cholesky schedule.

The schedule in paper_1310_6919_b200/dist.py (2D block-cyclic tiles, diagonal broadcast down the
process column, panel broadcast along process rows + all-gather within process columns, local
trailing updates) runs on world_size 2, 3 and 4 with the gloo backend.  The local tile operations
are CPU test doubles with the semantics sdpc.h states for sdpc_potrf_tile / sdpc_trsm_panel /
sdpc_update_tiles, so these tests pin the host logic (ownership, packing, collectives, info); the
CUDA tile kernels themselves are pinned by the -m gpu tests.  Reference: LAPACK potrf of the full B.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cholesky as CH
from paper_1310_6919_b200 import dist as D


class CpuTileOps:
    """CPU doubles of the three tile entries (semantics of include/sdpc.h)."""

    def __init__(self, L: D.Layout):
        self.L = L

    @staticmethod
    def _mat(t, rows, cols):        # column-major view: element (r, c) at t[c, r]
        return t[:cols, :rows].T

    def potrf_tile(self, A, n, lda, inv, info_dev, stream=None):
        M = self._mat(A, n, n)
        Lo = torch.tril(M)
        S = Lo + torch.tril(Lo, -1).T
        Lc, info = torch.linalg.cholesky_ex(S)
        mask = torch.tril(torch.ones(n, n, dtype=torch.bool))
        if int(info) != 0:
            info_dev[0] = int(info)
            return
        M[mask] = Lc[mask]
        for b in range((n + 127) // 128):
            o, w = 128 * b, min(128, n - 128 * b)
            Li = torch.linalg.inv(Lc[o:o + w, o:o + w])
            blk = torch.zeros(128, 128, dtype=M.dtype)
            blk[:w, :w] = Li
            inv[b * 16384:(b + 1) * 16384].view(128, 128).copy_(blk.T)   # column-major

    def trsm_panel(self, A, rows, lda, Lt, ldl, inv, kb, stream=None):
        Am = self._mat(A, rows, kb)
        Lm = torch.tril(self._mat(Lt, kb, kb))
        Am.copy_(torch.linalg.solve_triangular(Lm, Am.T, upper=False).T)

    def update_tiles(self, C, ldc, P, ldp, k1, K, stream=None, jlo=0, jhi=0):
        L = self.L
        Pm = self._mat(P, ldp, K)                    # row r = global row k1 + r
        for I in range(L.myrow, L.nt, L.Pr):
            for J in range(L.mycol, L.nt, L.Pc):
                if J * D.NB < k1 or I < J or J < jlo or (jhi > 0 and J >= jhi):
                    continue
                h, w = L.tile_rows(I), L.tile_rows(J)
                r, c = L.local_row_of_tile(I), L.local_col_of_tile(J)
                upd = Pm[I * D.NB - k1:I * D.NB - k1 + h] @ Pm[J * D.NB - k1:J * D.NB - k1 + w].T
                if I == J:
                    upd = torch.tril(upd)
                Cm = self._mat(C[c:, r:], h, w)
                Cm -= upd


def _spd(m, seed, bad=None):
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((m, m + 5))
    B = G @ G.T / (m + 5) + 0.5 * np.eye(m)
    if bad is not None:
        B[bad, bad] = -1.0
    return B


def _worker(rank, world, port, m, seed, bad, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = D.Layout(m, world, rank)
        B = _spd(m, seed, bad)
        loc = D.local_tiles_of(np.tril(B), L)
        Bt = torch.zeros((max(1, L.nloc), L.lld), dtype=torch.float64)
        Bt[:L.nloc, :L.mloc] = torch.from_numpy(loc.T.copy())
        info = D.dist_cholesky(CpuTileOps(L), Bt, L, D.TorchComm(L), torch.device("cpu"))
        res = dict(rank=rank, info=info)
        if bad is None:
            R = CH.potrf_lower(B)
            want = D.local_tiles_of(R, L)
            # upper parts of diagonal tiles must be untouched (zero here, from tril(B))
            got = Bt[:L.nloc, :L.mloc].T.numpy()
            res["err"] = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))
        q.put(res)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, m, seed=0, bad=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, m, seed, bad, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda r: r["rank"])


@pytest.mark.parametrize("world,m", [(2, 700), (3, 1100), (4, 1300), (4, 200)])
def test_dist_cholesky_matches_lapack(world, m):
    out = _run(world, m, seed=world * 100 + m)
    for r in out:
        assert r["info"] == 0
        assert r["err"] < 1e-12, r


def test_dist_cholesky_not_pd_info():
    # pivot 601 (tile 2 of a 2x2 grid) fails; LAPACK rule: info = 601 on every rank
    out = _run(4, 900, seed=7, bad=600)
    assert all(r["info"] == 601 for r in out), out


def test_layout_matches_scalapack_conventions():
    assert [D.grid_shape(p) for p in (1, 2, 3, 4, 6, 8)] == [(1, 1), (1, 2), (1, 3), (2, 2), (2, 3), (2, 4)]
    m = 1300
    for P in (1, 2, 4, 8):
        Ls = [D.Layout(m, P, r) for r in range(P)]
        # every global entry of the lower triangle has exactly one owner; local sizes = numroc
        assert sum(L.mloc for L in Ls if L.mycol == 0) == m
        assert sum(L.nloc for L in Ls if L.myrow == 0) == m
        for (i, j) in [(0, 0), (255, 0), (256, 255), (1299, 1299), (1000, 513)]:
            owner, lr, lc = Ls[0].global_to_local(i, j)
            L = Ls[owner]
            assert 0 <= lr < L.mloc and 0 <= lc < L.nloc
            assert (i // 256) % L.Pr == L.myrow and (j // 256) % L.Pc == L.mycol
        for k in range(Ls[0].nt):
            got = sorted(t for pr in range(Ls[0].Pr) for t in Ls[0].tiles_after(k, pr))
            assert got == list(range(k + 1, Ls[0].nt))
