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

    def exchange(self, group=None):
        """Post the halo exchange (isend/irecv with both neighbours); returns the
        works to wait on.  Owned rows are not modified."""
        import torch
        import torch.distributed as dist
        if self.buf.is_cuda and dist.get_backend(group) == "gloo":
            return self._exchange_host_staged(group)
        h, ops = self.halo, []
        # rows travel as bytes: NCCL has no uint16 type, and a byte view of whole
        # contiguous rows is the same memory
        B = self.buf if self.buf.dtype == torch.uint8 else self.buf.view(torch.uint8)
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, B[self.ha:self.ha + h], self.rank - 1, group))
            ops.append(dist.P2POp(dist.irecv, B[0:self.ha], self.rank - 1, group))
        if self.rank < self.world - 1:
            e = self.ha + self.rows
            ops.append(dist.P2POp(dist.isend, B[e - h:e], self.rank + 1, group))
            ops.append(dist.P2POp(dist.irecv, B[e:e + self.hb], self.rank + 1, group))
        return dist.batch_isend_irecv(ops) if ops else []

    def _exchange_host_staged(self, group):
        """The same exchange for a gloo group over device buffers (no NCCL, e.g.
        several ranks sharing one GPU in tests): rows go through host memory; the
        returned works copy the received rows into the device buffer on wait()."""
        import torch
        import torch.distributed as dist
        h, ops, recv = self.halo, [], []
        B = self.buf if self.buf.dtype == torch.uint8 else self.buf.view(torch.uint8)
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, B[self.ha:self.ha + h].cpu(), self.rank - 1, group))
            r = torch.empty_like(B[0:self.ha], device="cpu")
            ops.append(dist.P2POp(dist.irecv, r, self.rank - 1, group))
            recv.append((B[0:self.ha], r))
        if self.rank < self.world - 1:
            e = self.ha + self.rows
            ops.append(dist.P2POp(dist.isend, B[e - h:e].cpu(), self.rank + 1, group))
            r = torch.empty_like(B[e:e + self.hb], device="cpu")
            ops.append(dist.P2POp(dist.irecv, r, self.rank + 1, group))
            recv.append((B[e:e + self.hb], r))
        works = dist.batch_isend_irecv(ops) if ops else []

        class _Staged:
            def wait(self_inner):
                for w in works:
                    w.wait()
                for dst, src in recv:
                    dst.copy_(src)
                return True

        return [_Staged()] if works else []

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
