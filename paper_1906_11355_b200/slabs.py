"""Multi-GPU slab decomposition of the MCLAHE path (one process per GPU).

The volume is cut along dim 0 at interpolation-cell boundaries into
balanced slabs, one per rank.  Every rank runs the four
passes on its own rows; the only cross-rank traffic is

* global range mode: one 8-byte-per-value MAX all-reduce of
  (~key(lo), key(hi), nonfinite)  -- exact (integer keys of doubles);
* adaptive mode: the per-tile (min, max) keys of the tile rows two slabs
  share, MAX-combined with the neighbour (tiles straddle the cut);
* the partial integer counts of those shared tile rows, SUM-combined.

Integer combines are order-independent, so every rank ends with exactly the
counts (hence bit-identical LUTs and output) a single GPU computes.  No LUT
exchange is needed: both neighbours build the shared rows' mappings from the
same combined counts.  The exchange only ever involves ranks whose tile-row
windows overlap (neighbours), via batched NCCL send/recv.

``run_local`` emulates G slabs in one process on one device (the "fake
slab" mode used by the parity tests); ``run_rank`` is the torch.distributed
path used by bench.py under torchrun.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import _native as N
from .api import Plan


def cell_ranges(extent: int, kernel: int) -> list[tuple[int, int]]:
    """Original-row ranges of the interpolation cells along one dimension
    (lower neighbour of neighbor_kernels, src/interpolation.cpp:24-29)."""
    before = (2 * kernel - 1 - ((extent - 1) % kernel)) // 2
    g = (extent + 2 * kernel - 1 - ((extent - 1) % kernel)) // kernel
    out = []
    for c in range(g - 1):
        lo = 0 if c == 0 else (2 * kernel * c + kernel) // 2 - before
        hi = extent if c == g - 2 else (2 * kernel * (c + 1) + kernel) // 2 - before
        lo, hi = max(lo, 0), min(hi, extent)
        if hi > lo:
            out.append((lo, hi))
    return out


def slab_cuts(extent: int, kernel: int, world: int) -> list[tuple[int, int]]:
    """Cell-aligned [begin, end) rows per rank, balanced by row count."""
    cells = cell_ranges(extent, kernel)
    if world > len(cells):
        raise N.ValidationError(
            f"cannot split {len(cells)} interpolation cells along dim 0 over {world} slabs")
    cuts, start, ci = [], 0, 0
    for r in range(world):
        target = extent * (r + 1) / world
        lo_e, hi_e = ci + 1, len(cells) - (world - r - 1)  # keep >= 1 cell per later rank
        e = len(cells) if r == world - 1 else min(
            range(lo_e, hi_e + 1), key=lambda k: abs(cells[k - 1][1] - target))
        cuts.append((start, cells[e - 1][1]))
        start, ci = cells[e - 1][1], e
    return cuts


@dataclass
class Window:
    begin: int  # first tile row held
    end: int    # one past the last


def overlaps(windows: list[Window], me: int) -> list[tuple[int, int, int]]:
    """(peer, first, last) tile rows my window shares with each peer."""
    out = []
    w = windows[me]
    for r, o in enumerate(windows):
        if r == me:
            continue
        a, b = max(w.begin, o.begin), min(w.end, o.end)
        if b > a:
            out.append((r, a, b))
    return out


def combine_rows(mine, received: list, first_row: int, windows_me: Window, op: str):
    """In-place combine of received partial rows into my window buffer.
    ``mine`` is [window rows, ...]; each received item is (first, last, rows)."""
    import torch
    for a, b, rows in received:
        dst = mine[a - windows_me.begin:b - windows_me.begin]
        if op == "sum":
            dst += rows
        elif op == "max":
            torch.maximum(dst, rows, out=dst)
        else:
            raise ValueError(op)


def _rows(t, plan: Plan):
    """View a per-tile workspace array as [tile rows, tiles_per_row, ...]."""
    return t.view(plan.info.tile_row_end - plan.info.tile_row_begin, plan.info.tiles_per_row,
                  *t.shape[1:])


def _window(plan: Plan) -> Window:
    return Window(int(plan.info.tile_row_begin), int(plan.info.tile_row_end))


def run_local(x, kernel, n_bins=256, clip_limit=1.0, adaptive=False, slabs: int = 2,
              cuts=None):
    """Emulates ``slabs`` ranks on one device (same code path as run_rank,
    with the collectives done in-process).  Returns the assembled output."""
    import torch
    shape = tuple(x.shape)
    cuts = cuts or slab_cuts(shape[0], int(kernel[0]), slabs)
    code = N.F64 if x.dtype == torch.float64 else N.F32
    plans = [Plan(shape, kernel, n_bins, clip_limit, adaptive, code, a, b) for a, b in cuts]
    xs = [x[a:b].contiguous() for a, b in cuts]
    ws = [p.new_workspace(x.device) for p in plans]
    wins = [_window(p) for p in plans]
    for p, xi, w in zip(plans, xs, ws):
        p.reset(w)
        p.range(xi, w)
    if adaptive:
        _local_exchange(plans, wins, [_rows(p.tile_range_view(w), p) for p, w in zip(plans, ws)],
                        "max")
    flags = torch.stack([p.range_view(w) for p, w in zip(plans, ws)]).amax(0)
    for p, w in zip(plans, ws):
        p.range_view(w).copy_(flags)  # the all-reduce
        p.make_params(w)
    for p, xi, w in zip(plans, xs, ws):
        p.histograms(xi, w)
    _local_exchange(plans, wins, [_rows(p.counts_view(w), p) for p, w in zip(plans, ws)], "sum")
    outs = []
    for p, xi, w in zip(plans, xs, ws):
        p.mappings(w)
        o = torch.empty_like(xi)
        p.interpolate(xi, o, w)
        p.check(w)
        outs.append(o)
    return torch.cat(outs, 0)


def _local_exchange(plans, wins, bufs, op):
    snaps = [b.clone() for b in bufs]
    for me in range(len(plans)):
        recv = [(a, b, snaps[r][a - wins[r].begin:b - wins[r].begin])
                for r, a, b in overlaps(wins, me)]
        combine_rows(bufs[me], recv, 0, wins[me], op)


class DistExchange:
    """Neighbour exchange over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, windows: list[Window], rank: int, group=None):
        self.windows, self.rank, self.group = windows, rank, group

    def _host_staged(self) -> bool:
        import torch.distributed as dist
        return dist.get_backend(self.group) == "gloo"

    def allreduce_max(self, t):
        import torch.distributed as dist
        if t.is_cuda and self._host_staged():  # gloo: exchange through host memory
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX, group=self.group)
            t.copy_(h)
            return
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)

    def rows(self, buf, op: str):
        """Combine the shared tile rows of ``buf`` ([window rows, ...]) with
        every rank whose window overlaps mine."""
        import torch
        import torch.distributed as dist
        me = self.windows[self.rank]
        peers = overlaps(self.windows, self.rank)
        if not peers:
            return
        ops, recv = [], []
        staged = buf.is_cuda and self._host_staged()
        for r, a, b in peers:
            # rows are the outer dim: the shared rows are a contiguous view,
            # sent as is (every send completes before the in-place combine
            # below); gloo has no CUDA P2P, so it is staged through the host
            send = buf[a - me.begin:b - me.begin]
            if staged:
                send = send.cpu()
            rbuf = torch.empty_like(send)
            ops.append(dist.P2POp(dist.isend, send, r, group=self.group))
            ops.append(dist.P2POp(dist.irecv, rbuf, r, group=self.group))
            recv.append((a, b, rbuf))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if staged:
            recv = [(a, b, t.to(buf.device)) for a, b, t in recv]
        combine_rows(buf, recv, 0, me, op)


def all_windows(shape, kernel, n_bins, clip_limit, adaptive, cuts, dtype=N.F32) -> list[Window]:
    """Tile-row windows of every rank's plan (host arithmetic only)."""
    out = []
    for a, b in cuts:
        p = Plan(shape, kernel, n_bins, clip_limit, adaptive, dtype, a, b)
        out.append(_window(p))
    return out


def run_rank(x_local, shape, kernel, n_bins, clip_limit, adaptive, rank: int, world: int,
             out=None, group=None, plan: Plan | None = None, ws=None, windows=None):
    """One rank's share of a slab-decomposed MCLAHE (x_local = its rows)."""
    import torch
    cuts = slab_cuts(shape[0], int(kernel[0]), world)
    code = N.F64 if x_local.dtype == torch.float64 else N.F32
    if plan is None:
        a, b = cuts[rank]
        plan = Plan(shape, kernel, n_bins, clip_limit, adaptive, code, a, b)
    if windows is None:
        windows = all_windows(shape, kernel, n_bins, clip_limit, adaptive, cuts, code)
    ex = DistExchange(windows, rank, group)
    ws = ws if ws is not None else plan.new_workspace(x_local.device)
    plan.reset(ws)
    plan.range(x_local, ws)
    if adaptive:
        ex.rows(_rows(plan.tile_range_view(ws), plan), "max")
    ex.allreduce_max(plan.range_view(ws))
    plan.make_params(ws)
    plan.histograms(x_local, ws)
    ex.rows(_rows(plan.counts_view(ws), plan), "sum")
    plan.mappings(ws)
    out = out if out is not None else torch.empty_like(x_local)
    plan.interpolate(x_local, out, ws)
    return out, plan, ws
