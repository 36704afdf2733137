"""Row-strip sharding of one scene across the GPUs of a node (north_star:
"Large scenes are partitioned into row strips across the GPUs ... with an NCCL
halo exchange of boundary rows over NVLink").

Host logic only: strip planning and the neighbour halo exchange, written
against ``torch.distributed`` so the same code runs over NCCL on GPUs and over
gloo on CPU (tests).  The compute on each strip is ``lfe_extract_rows``.

Each rank keeps ONE contiguous buffer ``[halo_above | owned rows | halo_below]``
so a strip is a single pitched image for liblfe.  The exchange is the only
data-path collective: rank k sends its first ``halo`` owned rows to k-1 and its
last ``halo`` owned rows to k+1.
"""
from __future__ import annotations

from dataclasses import dataclass


def _bytes(t):
    """Rows travel as bytes: NCCL has no uint16 type, and a byte view of whole
    contiguous rows is the same memory."""
    import torch
    return t if t.dtype == torch.uint8 else t.view(torch.uint8)


def exchange_rows(pairs, group=None, staged=None):
    """Post one neighbour exchange: for each (send_rows, recv_rows, peer) an
    isend of send_rows and an irecv into recv_rows (NCCL P2P on GPUs); returns
    the works to wait on.  For a gloo group over device buffers (several ranks
    sharing one GPU in tests; NCCL refuses that) the rows go through host
    memory and the returned work copies the received rows into place on wait()
    (``staged=True`` forces that path, e.g. to test it on CPU buffers)."""
    import torch
    import torch.distributed as dist
    if not pairs:
        return []
    if staged is None:
        staged = pairs[0][0].is_cuda and dist.get_backend(group) == "gloo"
    ops, recv = [], []
    for snd, rcv, peer in pairs:
        if staged:
            r = torch.empty_like(rcv, device="cpu")
            ops.append(dist.P2POp(dist.isend, snd.cpu(), peer, group))
            ops.append(dist.P2POp(dist.irecv, r, peer, group))
            recv.append((rcv, r))
        else:
            ops.append(dist.P2POp(dist.isend, snd, peer, group))
            ops.append(dist.P2POp(dist.irecv, rcv, peer, group))
    works = dist.batch_isend_irecv(ops)
    if not staged:
        return works

    class _Staged:
        def wait(self):
            for w in works:
                w.wait()
            for dst, src in recv:
                dst.copy_(src)
            return True

    return [_Staged()]


def plan_strips(H: int, world: int, halo: int):
    """Contiguous, balanced row ranges [a, b) covering [0, H).  Every strip must
    hold at least ``halo`` rows so one neighbour exchange suffices."""
    if world < 1 or H < 1:
        raise ValueError("bad H/world")
    base, extra = divmod(H, world)
    out, a = [], 0
    for k in range(world):
        b = a + base + (1 if k < extra else 0)
        out.append((a, b))
        a = b
    if world > 1 and min(b - a for a, b in out) < halo:
        raise ValueError(f"strip of {min(b - a for a, b in out)} rows < halo {halo}: use fewer ranks")
    return out


@dataclass
class StripShard:
    H: int
    W: int
    rank: int
    world: int
    halo: int

    def __post_init__(self):
        self.plan = plan_strips(self.H, self.world, self.halo)
        self.a, self.b = self.plan[self.rank]
        self.rows = self.b - self.a
        self.ha = self.halo if self.rank > 0 else 0
        self.hb = self.halo if self.rank < self.world - 1 else 0

    @property
    def buf_rows(self) -> int:
        return self.ha + self.rows + self.hb

    def alloc(self, dtype, device):
        import torch
        self.buf = torch.zeros((self.buf_rows, self.W), dtype=dtype, device=device)
        return self.buf

    def load_owned(self, full_image_rows):
        """Copy this rank's owned rows (from a full-image tensor/array)."""
        import torch
        src = full_image_rows[self.a:self.b]
        if not isinstance(src, torch.Tensor):
            src = torch.from_numpy(src)
        self.buf[self.ha:self.ha + self.rows].copy_(src)

    def exchange(self, group=None, staged=None):
        """Post the halo exchange (isend/irecv with both neighbours); returns the
        works to wait on.  Owned rows are not modified."""
        h, pairs = self.halo, []
        B = _bytes(self.buf)
        if self.rank > 0:
            pairs.append((B[self.ha:self.ha + h], B[0:self.ha], self.rank - 1))
        if self.rank < self.world - 1:
            e = self.ha + self.rows
            pairs.append((B[e - h:e], B[e:e + self.hb], self.rank + 1))
        return exchange_rows(pairs, group, staged)

    def allreduce_stats(self, t_stats, group=None):
        """Adaptive thresholds (NEXT-2): the 9 exact int64 sums of lfe_stats are
        additive over disjoint row ranges, so one SUM all-reduce of every rank's
        owned-row partial gives the whole-image statistics (bit-exact)."""
        import torch.distributed as dist
        if self.world > 1:
            if t_stats.is_cuda and dist.get_backend(group) == "gloo":
                h = t_stats.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
                t_stats.copy_(h)
            else:
                dist.all_reduce(t_stats, op=dist.ReduceOp.SUM, group=group)
        return t_stats

    def edge_flags(self) -> int:
        from .lfe import LFE_BOTTOM_IS_EDGE, LFE_TOP_IS_EDGE
        return (LFE_TOP_IS_EDGE if self.rank == 0 else 0) | (LFE_BOTTOM_IS_EDGE if self.rank == self.world - 1 else 0)

    def band(self, s: int, n: int):
        """Arguments of lfe_extract_rows for owned rows [s, s+n) of this strip:
        (s, n, halo_above, halo_below, flags, needs_exchange)."""
        from .lfe import LFE_BOTTOM_IS_EDGE, LFE_TOP_IS_EDGE
        h, R = self.halo, self.rows
        flags, need = 0, False
        if self.rank == 0:                    # buffer row 0 is the image top
            ha = s
            flags |= LFE_TOP_IS_EDGE
        else:
            ha = h
            need |= s < h                     # reads received rows above
        if self.rank == self.world - 1:       # last buffer row is the image bottom
            hb = R - s - n
            flags |= LFE_BOTTOM_IS_EDGE
        else:
            hb = h
            need |= s + n > R - h             # reads received rows below
        return (s, n, ha, hb, flags, need)

    def bands(self):
        """The interior band (local rows only: computable while the exchange is
        in flight) followed by the boundary bands that wait for it."""
        h, R = self.halo, self.rows
        lo = 0 if self.rank == 0 else h
        hi = R if self.rank == self.world - 1 else R - h
        if hi - lo <= 0:
            return [self.band(0, R)]
        out = [self.band(lo, hi - lo)]
        if lo > 0:
            out.append(self.band(0, lo))
        if hi < R:
            out.append(self.band(hi, R - hi))
        return out


def plan_bands(bands: int, H: int, world: int, halo: int):
    """Work of each rank for a multispectral scene (c4).  Bands
    are independent images; the band-major row line (bands x H rows) is cut
    into `world` contiguous, equal pieces, each cut snapped to a band boundary
    when it would leave fewer than `halo` rows of a band on one side (so one
    neighbour exchange still suffices).  When world divides bands this deals
    out whole bands and needs no collective at all.  Returns, per rank, a list
    of (band, a, b) owned row ranges.  Raises ValueError when a piece of a band
    that is cut on either side would still hold fewer than `halo` rows (as
    plan_strips does)."""
    if bands < 1 or world < 1 or H < 1:
        raise ValueError("bad bands/H/world")
    T = bands * H
    cuts = [0]
    for k in range(1, world):
        c = round(k * T / world)
        b0 = (c // H) * H
        if c == b0:
            pass  # already on a band boundary
        elif c - b0 < halo:
            c = b0
        elif b0 + H - c < halo:
            c = b0 + H
        cuts.append(max(c, cuts[-1]))
    cuts.append(T)
    work = []
    for k in range(world):
        lo, hi, items = cuts[k], cuts[k + 1], []
        u = lo
        while u < hi:
            b = u // H
            e = min(hi, (b + 1) * H)
            items.append((b, u - b * H, e - b * H))
            u = e
        work.append(items)
    # a piece of a band cut on either side must itself hold a halo of rows, or its
    # neighbour's exchange would need rows from beyond the adjacent rank
    short = [(k, it) for k, items in enumerate(work) for it in items
             if (it[1] > 0 or it[2] < H) and it[2] - it[1] < halo]
    if short:
        k, (b, a, e) = short[0]
        raise ValueError(f"rank {k} would own rows [{a}, {e}) of band {b}: {e - a} rows < halo {halo}; use fewer ranks")
    return work


class BandShard:
    """One rank's share of a multispectral scene (c4): the row ranges
    ``plan_bands`` gives it.  Whole bands are computed in ONE lfe_extract_bands
    launch with no collective; a band cut between two ranks is a strip of that
    band, with the same one-hop halo exchange as a scene (only between the two
    ranks sharing the band).

    ``whole``: the bands owned entirely (consecutive); ``parts``: (band, a, b,
    peer_above, peer_below) for pieces of cut bands, each with its own buffer
    [halo above | rows | halo below] (peers are ranks, or None at a band edge)."""

    def __init__(self, bands: int, H: int, W: int, rank: int, world: int, halo: int):
        self.nbands, self.H, self.W, self.rank, self.world, self.halo = bands, H, W, rank, world, halo
        items = plan_bands(bands, H, world, halo)[rank]
        self.whole = [b for b, a, e in items if a == 0 and e == H]
        if self.whole and self.whole != list(range(self.whole[0], self.whole[-1] + 1)):
            raise AssertionError("whole bands of one rank are consecutive")
        self.parts = []
        for k, (b, a, e) in enumerate(items):
            if a == 0 and e == H:
                continue
            # a cut piece is the first item (continues the previous rank's band) and/or
            # the last (continued by the next rank)
            above = rank - 1 if a > 0 else None
            below = rank + 1 if e < H else None
            self.parts.append((b, a, e, above, below))

    def alloc(self, dtype, device):
        import torch
        self.whole_buf = (torch.zeros((len(self.whole), self.H, self.W), dtype=dtype, device=device)
                          if self.whole else None)
        self.part_bufs = []
        for b, a, e, above, below in self.parts:
            ha = self.halo if above is not None else 0
            hb = self.halo if below is not None else 0
            self.part_bufs.append(torch.zeros((ha + e - a + hb, self.W), dtype=dtype, device=device))
        return self

    def load_owned(self, scene):
        """Copy the owned rows from a [bands, H, W] host array."""
        import torch
        if self.whole:
            self.whole_buf.copy_(torch.from_numpy(scene[self.whole[0]:self.whole[-1] + 1]))
        for (b, a, e, above, _), buf in zip(self.parts, self.part_bufs):
            ha = self.halo if above is not None else 0
            buf[ha:ha + e - a].copy_(torch.from_numpy(scene[b, a:e]))

    def exchange(self, group=None, staged=None):
        """Post the halo exchange of the cut pieces (isend/irecv with the rank
        sharing the band); returns the works to wait on."""
        h, pairs = self.halo, []
        for (b, a, e, above, below), buf in zip(self.parts, self.part_bufs):
            B = _bytes(buf)
            ha = h if above is not None else 0
            if above is not None:
                pairs.append((B[ha:ha + h], B[0:ha], above))
            if below is not None:
                end = ha + e - a
                pairs.append((B[end - h:end], B[end:end + h], below))
        return exchange_rows(pairs, group, staged)

    def part_calls(self):
        """lfe_extract_rows arguments per cut piece: (piece index, s, n, halo_above,
        halo_below, flags, needs_exchange) -- the rows computable before the
        exchange completes first, the boundary rows after."""
        from .lfe import LFE_BOTTOM_IS_EDGE, LFE_TOP_IS_EDGE
        h, out_first, out_after = self.halo, [], []
        for k, (b, a, e, above, below) in enumerate(self.parts):
            R = e - a
            lo = h if above is not None else 0
            hi = R - h if below is not None else R

            def call(s, n):
                flags, need = 0, False
                if above is None:
                    ha, flags = s, flags | LFE_TOP_IS_EDGE
                else:
                    ha, need = h, need or s < h
                if below is None:
                    hb, flags = R - s - n, flags | LFE_BOTTOM_IS_EDGE
                else:
                    hb, need = h, need or s + n > R - h
                return (k, s, n, ha, hb, flags, need)

            if hi - lo <= 0:
                out_after.append(call(0, R))
                continue
            out_first.append(call(lo, hi - lo))
            if lo > 0:
                out_after.append(call(0, lo))
            if hi < R:
                out_after.append(call(hi, R - hi))
        return out_first + out_after

    def owned_pixels(self) -> int:
        return (len(self.whole) * self.H + sum(e - a for _, a, e, _, _ in self.parts)) * self.W


class PeerStripShard:
    """Row strips whose halo rows stay in the neighbours' HBM (north_star's
    multi-GPU row strips on one NVLink/NVSwitch node, with no exchange step):
    each rank holds ONLY its owned rows; at setup the ranks swap CUDA IPC
    handles of those buffers (one all_gather_object) and map their neighbours'
    (lfe_ipc_open enables peer access), and every step is ONE
    lfe_extract_rows_peer launch that TMA-loads the halo rows from the
    neighbours' memory.  Each rank also exposes a uint64 "input ready" flag
    (lfe_signal) that its neighbours' kernels wait on before reading its rows.

    Host logic only (gloo-testable: the plan and the peer geometry); the device
    calls go through lfe.py."""

    def __init__(self, H: int, W: int, rank: int, world: int, halo: int):
        from .lfe import LFE_PEER_ROWS
        self.H, self.W, self.rank, self.world, self.halo = H, W, rank, world, halo
        self.peer_rows = max(halo, LFE_PEER_ROWS)  # rows read from each neighbour (lfe.h)
        self.plan = plan_strips(H, world, self.peer_rows)
        self.a, self.b = self.plan[rank]
        self.rows = self.b - self.a
        self.ha = halo if rank > 0 else 0          # halo rows a neighbour supplies above / below
        self.hb = halo if rank < world - 1 else 0
        self.peer = {}  # rank -> (base pointer of its buffer, pitch, rows, flag pointer)
        self._opened = []

    def edge_flags(self) -> int:
        from .lfe import LFE_BOTTOM_IS_EDGE, LFE_TOP_IS_EDGE
        return (LFE_TOP_IS_EDGE if self.rank == 0 else 0) | (LFE_BOTTOM_IS_EDGE if self.rank == self.world - 1 else 0)

    def alloc(self, dtype, device):
        import torch
        self.buf = torch.zeros((self.rows, self.W), dtype=dtype, device=device)
        self.flag = torch.zeros(1, dtype=torch.int64, device=device)
        return self.buf

    def load_owned(self, full_image_rows):
        import torch
        src = full_image_rows[self.a:self.b]
        if not isinstance(src, torch.Tensor):
            src = torch.from_numpy(src)
        self.buf.copy_(src)

    def neighbours(self):
        return [k for k in (self.rank - 1, self.rank + 1) if 0 <= k < self.world]

    def connect(self, group=None):
        """Swap IPC handles of every rank's buffer and flag; map the neighbours'."""
        import torch.distributed as dist

        from . import lfe
        mine = (lfe.lfe_ipc_export(self.buf.data_ptr()), lfe.lfe_ipc_export(self.flag.data_ptr()),
                self.buf.stride(0) * self.buf.element_size(), self.rows)
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        for k in self.neighbours():
            (hb, ob), (hf, of), pitch, rows = allh[k]
            pb = lfe.lfe_ipc_open(hb, ob)
            self._opened.append((pb, ob))
            pf = lfe.lfe_ipc_open(hf, of)
            self._opened.append((pf, of))
            self.peer[k] = (pb, pitch, rows, pf)

    def call_args(self):
        """(d_above, above_pitch, d_below, below_pitch, wait_above, wait_below) for
        lfe_extract_rows_peer: the neighbour above's last LFE_PEER_ROWS rows, the
        neighbour below's first rows, and their flags."""
        h = self.peer_rows
        da = pa = db = pb = fa = fb = 0
        if self.rank > 0:
            base, pitch, rows, flag = self.peer[self.rank - 1]
            da, pa, fa = base + (rows - h) * pitch, pitch, flag
        if self.rank < self.world - 1:
            base, pitch, rows, flag = self.peer[self.rank + 1]
            db, pb, fb = base, pitch, flag
        return da, pa, db, pb, fa, fb

    def close(self):
        from . import lfe
        for p, off in self._opened:
            lfe.lfe_ipc_close(p, off)
        self._opened = []
        self.peer = {}
