"""Multi-GPU SCM build + Cholesky: one process per GPU, B 2D block-cyclic.

Plumbing only: every arithmetic step runs in libsdpc kernels (sdpc_scm_build for this rank's tiles,
sdpc_potrf_tile / sdpc_trsm_panel / sdpc_update_tiles for the factorization); this module moves tiles
between ranks with collectives (torch.distributed over NCCL on GPUs, gloo in the CPU tests).

Layout (ScaLAPACK convention, ``include/sdpc.h``): kScmNB = 256 tiles; Pr x Pc grid with Pr the
largest divisor of P <= sqrt(P); rank = myrow * Pc + mycol; tile (I, J) on (I mod Pr, J mod Pc).
The local array is column-major mloc x nloc with leading dimension lld, held as a torch tensor
``Bt`` of shape (nloc, lld) with local element (r, c) at ``Bt[c, r]``.

Build (the columns of B are independent).  Rank (pr, pc) evaluates exactly its tiles: the
columns l with (l / 256) mod Pc == pc need x_p, y_q only for the columns p, q of A_l (Eq. newSCM2,
P:686-688), so its solves cover 1/Pc of the RHS (replicated over the Pr ranks of a process column,
SURVEY §8(e) "each GPU keeps 1/Pr of its blocks"); (a1), (a2) are replicated.  No exchange step.

Cholesky: right-looking blocked, per step k (tile column k):
  1. owner of (k, k) factors the tile (sdpc_potrf_tile);
  2. the factored tile + its 128-block inverses are broadcast down process column k mod Pc;
  3. process column k mod Pc solves its panel tiles (sdpc_trsm_panel);
  4. the panel reaches every rank: broadcast along each process row from column k mod Pc, then
     all-gather within each process column (the transposed operand of the update);
  5. every rank updates its trailing tiles (sdpc_update_tiles): tile column k+1 first, the rest on a
     side stream while panel k+1 is factored and communicated (depth-1 lookahead).
"""
from __future__ import annotations

import threading

NB = 256            # kScmNB (tile of the 2D block-cyclic distribution; sdpc.h)
INV_ELEMS = 2 * 128 * 128
NO_ERROR = 0x7F7F7F7F


def grid_shape(P: int):
    """Pr x Pc with Pr the largest divisor of P not above sqrt(P) (1x1, 1x2, 2x2, 2x4, ...)."""
    pr = 1
    d = 1
    while d * d <= P:
        if P % d == 0:
            pr = d
        d += 1
    return pr, P // pr


def numroc(m: int, p: int, P: int, nb: int = NB) -> int:
    """Rows (or columns) of an m-long dimension held by process coordinate p of P (tile nb)."""
    nt = (m + nb - 1) // nb
    return sum(min(nb, m - t * nb) for t in range(p, nt, P))


class Layout:
    """2D block-cyclic layout of the m x m SCM on rank `rank` of `P` (mirrors sdpc_get_scm_layout)."""

    def __init__(self, m: int, P: int, rank: int):
        self.m, self.P, self.rank = m, P, rank
        self.Pr, self.Pc = grid_shape(P)
        self.myrow, self.mycol = divmod(rank, self.Pc)
        self.mloc = numroc(m, self.myrow, self.Pr)
        self.nloc = numroc(m, self.mycol, self.Pc)
        self.lld = max(1, self.mloc + (self.mloc & 1))     # even: 16-byte aligned columns
        self.nt = (m + NB - 1) // NB

    def rank_of(self, pr: int, pc: int) -> int:
        return pr * self.Pc + pc

    def col_ranks(self, pc: int):
        return [self.rank_of(pr, pc) for pr in range(self.Pr)]

    def row_ranks(self, pr: int):
        return [self.rank_of(pr, pc) for pc in range(self.Pc)]

    def tiles_after(self, k: int, pr: int):
        """Global tile rows I > k held by process row pr, ascending."""
        first = k + 1 + ((pr - (k + 1)) % self.Pr)
        return list(range(first, self.nt, self.Pr))

    def local_row_of_tile(self, I: int) -> int:
        return (I // self.Pr) * NB

    def local_col_of_tile(self, J: int) -> int:
        return (J // self.Pc) * NB

    def tile_rows(self, I: int) -> int:
        return min(NB, self.m - I * NB)

    def global_to_local(self, i: int, j: int):
        """(owner rank, local row, local col) of global entry (i, j)."""
        I, J = i // NB, j // NB
        return (self.rank_of(I % self.Pr, J % self.Pc), (I // self.Pr) * NB + i % NB, (J // self.Pc) * NB + j % NB)


# ----------------------------------------------------------------------------- communicators

class TorchComm:
    """torch.distributed collectives on the process-row / process-column subgroups (NCCL on GPU)."""

    def __init__(self, layout: Layout):
        import torch.distributed as dist
        self.dist = dist
        self.L = layout
        # every rank must create every subgroup, in the same order
        self.col_groups = [dist.new_group(layout.col_ranks(pc)) for pc in range(layout.Pc)]
        self.row_groups = [dist.new_group(layout.row_ranks(pr)) for pr in range(layout.Pr)]

    def bcast_col(self, t, src_row: int):
        L = self.L
        if L.Pr > 1:
            self.dist.broadcast(t, src=L.rank_of(src_row, L.mycol), group=self.col_groups[L.mycol])

    def bcast_row(self, t, src_col: int):
        L = self.L
        if L.Pc > 1:
            self.dist.broadcast(t, src=L.rank_of(L.myrow, src_col), group=self.row_groups[L.myrow])

    def allgather_col(self, outs, t):
        L = self.L
        if L.Pr > 1:
            self.dist.all_gather(outs, t, group=self.col_groups[L.mycol])
        else:
            outs[0].copy_(t)

    def allreduce_min(self, t):
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MIN)


class ThreadComm:
    """The same collectives between threads of one process (each thread = one rank), for the
    single-GPU emulation of the P-rank schedule: only host threads wait on one another (barriers
    after a device synchronize); every kernel runs to completion on its own, no device-side waits
    between ranks."""

    class _Shared:
        def __init__(self, layout0: Layout):
            L = layout0
            self.world = threading.Barrier(L.P)
            self.col = [threading.Barrier(L.Pr) for _ in range(L.Pc)]
            self.row = [threading.Barrier(L.Pc) for _ in range(L.Pr)]
            self.slots = [None] * L.P

    def __init__(self, layout: Layout, shared: "ThreadComm._Shared", sync=None):
        self.L = layout
        self.S = shared
        self.sync = sync or (lambda: None)

    @classmethod
    def make_shared(cls, layout0: Layout):
        return cls._Shared(layout0)

    def _exchange(self, t, bar):
        self.sync()
        self.S.slots[self.L.rank] = t
        bar.wait()
        return list(self.S.slots)

    def _done(self, bar):
        self.sync()
        bar.wait()

    def bcast_col(self, t, src_row: int):
        L = self.L
        bar = self.S.col[L.mycol]
        src = self._exchange(t, bar)[L.rank_of(src_row, L.mycol)]
        if src is not t:
            t.copy_(src)
        self._done(bar)

    def bcast_row(self, t, src_col: int):
        L = self.L
        bar = self.S.row[L.myrow]
        src = self._exchange(t, bar)[L.rank_of(L.myrow, src_col)]
        if src is not t:
            t.copy_(src)
        self._done(bar)

    def allgather_col(self, outs, t):
        L = self.L
        bar = self.S.col[L.mycol]
        vals = self._exchange(t, bar)
        for pr in range(L.Pr):
            outs[pr].copy_(vals[L.rank_of(pr, L.mycol)])
        self._done(bar)

    def allreduce_min(self, t):
        bar = self.S.world
        vals = self._exchange(t.clone(), bar)
        m = vals[0]
        for v in vals[1:]:
            m = m.minimum(v)
        self._done(bar)
        t.copy_(m)


# ----------------------------------------------------------------------------- distributed Cholesky

def update_flops(L: Layout, k: int, jlo: int = 0, jhi: int = 0) -> float:
    """Algorithmic flops of this rank's trailing update at step k (2 * kb per updated entry),
    restricted to the global tile columns [jlo, jhi) (jhi <= 0: no bound)."""
    kb = min(NB, L.m - k * NB)
    fl = 0.0
    for I in range(L.myrow, L.nt, L.Pr):
        if I <= k:
            continue
        h = L.tile_rows(I)
        for J in range(L.mycol, I + 1, L.Pc):
            if J <= k or J < jlo or (jhi > 0 and J >= jhi):
                continue
            w = L.tile_rows(J)
            fl += 2.0 * kb * (h * (h + 1) / 2 if I == J else h * w)
    return fl


def dist_cholesky(ops, Bt, L: Layout, comm, dev, stream=None, timer=None):
    """Factor the distributed SCM in place (lower(B) <- R).  Returns the LAPACK-style info (0 or the
    1-based order of the first non-PD leading minor), identical on every rank.

    Depth-1 lookahead: after panel k is on every rank, the tile column k+1 is updated first (on the
    main stream), panel k+1 is factored, solved and communicated, while the rest of the trailing
    update of step k runs on a side stream (GPU); panel buffers are double-buffered.

    ops: sdpc Handle (GPU) or a test double with the same potrf_tile / trsm_panel / update_tiles.
    Bt:  local array, torch tensor (nloc, lld), local element (r, c) at Bt[c, r].
    timer: optional list; gets (start event, end event, algorithmic flops) per local update launch.
    """
    import torch
    m, lld = L.m, L.lld
    f64 = torch.float64
    cuda = dev.type == "cuda"
    main = torch.cuda.current_stream(dev) if cuda else None
    side = torch.cuda.Stream(device=dev) if cuda else None
    diagbuf = torch.zeros(NB * NB + INV_ELEMS, dtype=f64, device=dev)
    dtile = diagbuf[:NB * NB].view(NB, NB)        # tile (r, c) at dtile[c, r], ld NB
    dinv = diagbuf[NB * NB:]
    infos = torch.full((L.nt,), NO_ERROR, dtype=torch.int32, device=dev)
    max_tiles = (L.nt + L.Pr - 1) // L.Pr
    piece = [torch.zeros(NB * max_tiles * NB, dtype=f64, device=dev) for _ in range(2)]
    gathered = [[torch.zeros_like(piece[0]) for _ in range(L.Pr)] for _ in range(2)] if L.Pr > 1 else None
    pfull = [torch.zeros(NB * L.nt * NB, dtype=f64, device=dev) for _ in range(2)] if L.Pr > 1 else None

    def panel(k):
        """Steps 1-4 for tile column k: returns (P, ldp, k1, kb) with P the panel on every rank,
        or None when k is the last tile column."""
        buf = k & 1
        k0 = k * NB
        kb = min(NB, m - k0)
        prk, pck = k % L.Pr, k % L.Pc
        k1 = k0 + kb
        mine = L.tiles_after(k, L.myrow)
        r0 = L.local_row_of_tile(mine[0]) if mine else L.mloc
        rows = L.mloc - r0
        if L.mycol == pck:
            lc = L.local_col_of_tile(k)
            if L.myrow == prk:
                lr = L.local_row_of_tile(k)
                ops.potrf_tile(Bt[lc:, lr:], kb, lld, dinv, infos[k:], stream)
                dtile[:kb, :kb].copy_(Bt[lc:lc + kb, lr:lr + kb])
            comm.bcast_col(diagbuf, prk)
            if rows > 0:
                ops.trsm_panel(Bt[lc:, r0:], rows, lld, dtile, NB, dinv, kb, stream)
        if k1 >= m:
            return None
        npr = len(mine)
        ldpc = max(1, npr) * NB
        pv = piece[buf][:kb * ldpc].view(kb, ldpc)
        if L.mycol == pck and rows > 0:
            pv[:, :rows].copy_(Bt[L.local_col_of_tile(k):L.local_col_of_tile(k) + kb, r0:L.mloc])
        comm.bcast_row(piece[buf], pck)
        if L.Pr == 1:
            return pv, ldpc, k1, kb
        comm.allgather_col(gathered[buf], piece[buf])
        ntr = L.nt - (k + 1)                     # panel tile rows k+1 .. nt-1
        ldp = ntr * NB
        P = pfull[buf][:kb * ldp].view(kb, ldp)
        Pt = P.view(kb, ntr, NB)
        for pr in range(L.Pr):
            tl = L.tiles_after(k, pr)
            if not tl:
                continue
            t0 = tl[0] - (k + 1)
            src = gathered[buf][pr][:kb * len(tl) * NB].view(kb, len(tl), NB)
            Pt[:, t0::L.Pr, :].copy_(src)
        return P, ldp, k1, kb

    def update(P, ldp, k1, kb, k, jlo, jhi, strm):
        if timer is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(strm)
        ops.update_tiles(Bt, lld, P, ldp, k1, kb, strm, jlo, jhi)
        if timer is not None:
            e1.record(strm)
            timer.append((e0, e1, update_flops(L, k, jlo, jhi)))

    cur = panel(0)
    prev_done = None
    for k in range(L.nt):
        if cur is None:
            break
        P, ldp, k1, kb = cur
        # 5a. tile column k+1 first (it holds panel k+1); it needs the bulk update of step k-1
        if cuda and prev_done is not None:
            main.wait_event(prev_done)
        update(P, ldp, k1, kb, k, k + 1, k + 2, main)
        # 5b. the rest of the trailing update on the side stream, overlapping panel k+1
        if cuda:
            side.wait_stream(main)
            with torch.cuda.stream(side):
                update(P, ldp, k1, kb, k, k + 2, 0, side)
            prev_done = torch.cuda.Event()
            prev_done.record(side)
        else:
            update(P, ldp, k1, kb, k, k + 2, 0, None)
        cur = panel(k + 1)
    if cuda:
        main.wait_stream(side)
    # info: smallest failing global column over all ranks (LAPACK rule)
    loc = torch.full((1,), NO_ERROR, dtype=torch.int64, device=dev)
    bad = (infos != NO_ERROR).nonzero().flatten()
    if bad.numel() > 0:
        k = int(bad[0])
        loc[0] = k * NB + int(infos[k])
    comm.allreduce_min(loc)
    v = int(loc[0])
    return 0 if v == NO_ERROR else v


def local_tiles_of(Bfull_lower, L: Layout):
    """Test helper: this rank's local array (numpy, shape (mloc, nloc)) cut from a global matrix."""
    import numpy as np
    out = np.zeros((L.mloc, L.nloc))
    for I in range(L.myrow, L.nt, L.Pr):
        for J in range(L.mycol, L.nt, L.Pc):
            r, c = L.local_row_of_tile(I), L.local_col_of_tile(J)
            h, w = L.tile_rows(I), L.tile_rows(J)
            out[r:r + h, c:c + w] = Bfull_lower[I * NB:I * NB + h, J * NB:J * NB + w]
    return out
