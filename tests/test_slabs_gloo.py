"""Multi-process (gloo, world_size 2 and 3) test of the slab exchange layer
(paper_1906_11355_b200/slabs.py) on CPU: every rank holds the partial
counts / range keys of ITS rows for the tile rows of its window; after
DistExchange the shared rows must equal the full-volume values the oracle
computes, bit for bit.  The GPU kernels are exercised by the fake-slab GPU
tests; this covers the distributed plumbing (windows, neighbour send/recv,
all-reduce) that bench.py uses under torchrun."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

SHAPE, KERNEL, NB = (37, 12, 10), (8, 4, 5), 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    rng = np.random.default_rng(7)
    return (np.round(rng.random(SHAPE) * 12) / 12).astype(np.float32)


def _partial_tile_rows(x, rows, window, adaptive):
    """Per-slab partial counts (global range) / min-max keys over the tile
    rows of `window`, counting only padded positions whose mirror source row
    lies in `rows` -- what the rank's histogram / range pass produces."""
    before, after, grid = O.geometry(x.shape, KERNEL)
    D = x.ndim
    lo_g, hi_g = float(x.min()), float(x.max())
    tpr = int(np.prod(grid[1:]))
    counts = np.zeros((window[1] - window[0], tpr, NB), np.int32)
    kmin = np.full((window[1] - window[0], tpr), np.iinfo(np.int64).min, np.int64)
    kmax = kmin.copy()
    for t0 in range(window[0], window[1]):
        for rest in range(tpr):
            tc = (t0,) + np.unravel_index(rest, grid[1:])
            idx = []
            for d in range(D):
                o = np.arange(tc[d] * KERNEL[d], (tc[d] + 1) * KERNEL[d]) - before[d]
                s = x.shape[d]
                m = np.mod(o, 2 * s)
                idx.append(np.where(m >= s, 2 * s - 1 - m, m))
            sel0 = idx[0][(idx[0] >= rows[0]) & (idx[0] < rows[1])]
            if sel0.size == 0:
                continue
            blk = x[np.ix_(sel0, *idx[1:])].astype(np.float64).ravel()
            b = O.bin_index_array(blk, lo_g, hi_g, NB)
            counts[t0 - window[0], rest] = np.bincount(b, minlength=NB)
            kmin[t0 - window[0], rest] = ~_okey(blk.min())
            kmax[t0 - window[0], rest] = _okey(blk.max())
    return counts, kmin, kmax


def _okey(v):
    i = np.array([v], np.float64).view(np.int64)[0]
    return int(i) if i >= 0 else int(i ^ np.int64(0x7FFFFFFFFFFFFFFF))


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1906_11355_b200 import Plan, slabs as S
        x = _data()
        cuts = S.slab_cuts(SHAPE[0], KERNEL[0], world)
        windows = S.all_windows(SHAPE, KERNEL, NB, 0.1, False, cuts)
        me = windows[rank]
        plan = Plan(SHAPE, KERNEL, NB, 0.1, False, 0, *cuts[rank])
        counts, kmin, kmax = _partial_tile_rows(x, cuts[rank], (me.begin, me.end), False)
        ex = S.DistExchange(windows, rank)
        c = torch.from_numpy(counts.copy())
        ex.rows(c, "sum")
        keys = torch.from_numpy(np.stack([kmin, kmax], -1).copy())
        ex.rows(keys, "max")
        # global range all-reduce of the rank-local keys
        xl = x[cuts[rank][0]:cuts[rank][1]].astype(np.float64)
        rk = torch.tensor([~_okey(xl.min()), _okey(xl.max()), 0, 0], dtype=torch.int64)
        ex.allreduce_max(rk)
        # reference: the full-volume tile statistics
        full = O.tile_stats(x, KERNEL, NB, 0.1, False, "c")
        grid = full["grid"]
        fc = full["counts"].reshape(grid[0], -1, NB)
        need = range(plan.info.need_row_begin, plan.info.need_row_end)
        ok_counts = all(np.array_equal(c[t - me.begin].numpy(), fc[t]) for t in need)
        fa = O.tile_stats(x, KERNEL, NB, 0.1, True, "c")
        flo, fhi = fa["lo"].reshape(grid[0], -1), fa["hi"].reshape(grid[0], -1)
        ok_keys = all(
            np.array_equal(keys[t - me.begin, :, 0].numpy(), [~_okey(v) for v in flo[t]]) and
            np.array_equal(keys[t - me.begin, :, 1].numpy(), [_okey(v) for v in fhi[t]])
            for t in need)
        ok_range = (rk[0].item() == ~_okey(float(x.min()))) and (rk[1].item() == _okey(float(x.max())))
        q.put((rank, ok_counts, ok_keys, ok_range, plan.info.need_row_begin, plan.info.need_row_end))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 3])
def test_slab_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 6, r
        rank, ok_counts, ok_keys, ok_range, a, b = r
        assert ok_counts and ok_keys and ok_range, r
    # every tile row some rank blends is covered exactly
    covered = sorted(t for r in res for t in range(r[4], r[5]))
    assert covered[0] == 0
