"""Pins the full-size gate's tools (tests/test_fullsize_gate.py) on CPU: the
reference's per-tile intermediates from a dim-0 crop, and its per-voxel loop
over a window of rows, must equal the reference run on the whole volume.
Test infrastructure only (oracle/_ref is the reference compiled from its own
sources)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")


@pytest.mark.parametrize("adaptive", [False, True])
@pytest.mark.parametrize("b0", [4, 5])
def test_crop_windows_equal_full_volume(adaptive, b0):
    rng = np.random.default_rng(7 + b0 + adaptive)
    shape = (8 * b0, 6, 10)
    kernel = (b0, 3, 4)
    x = np.round(rng.random(shape) * 40) / 40
    full = O.tile_stats(x, kernel, 32, 0.05, adaptive, "ref")
    g0 = full["grid"][0]
    per_row = len(full["lo"]) // g0
    rng_g = (float(x.min()), float(x.max()))
    for t0, t1 in [(0, 2), (0, 3), (3, 4), (2, 5), (g0 - 2, g0), (g0 - 3, g0), (0, g0)]:
        st, _ = O.ref_tile_rows_by_crop(x, kernel, 32, 0.05, adaptive, t0, t1, rng_g)
        sl = slice(t0 * per_row, t1 * per_row)
        for k in ("lo", "hi", "counts", "clipped", "lut", "degenerate"):
            assert np.array_equal(st[k], full[k][sl]), (t0, t1, k)


@pytest.mark.parametrize("adaptive", [False, True])
def test_window_stats_and_blend_rows_equal_full_run(adaptive):
    rng = np.random.default_rng(3 + adaptive)
    shape = (24, 10, 12)
    kernel = (4, 5, 3)
    x = rng.poisson(3.0, shape) / 7.0
    full = O.tile_stats(x, kernel, 16, 0.1, adaptive, "ref")
    win = O.ref_tile_stats_window(x, kernel, 16, 0.1, adaptive, 0, full["grid"][0], threads=3)
    for k in ("lo", "hi", "counts", "clipped", "lut", "degenerate"):
        assert np.array_equal(win[k], full[k]), k
    want = O.mclahe(x, kernel, 16, 0.1, adaptive, "ref", threads=2)
    per_row = len(full["lo"]) // full["grid"][0]
    for r0, r1 in [(0, 24), (0, 5), (9, 14), (20, 24)]:
        t0 = r0 // 4  # cells are b0-aligned here (24 % 4 == 0): rows [r0, r1) use tiles t0..
        t1 = min(full["grid"][0], (r1 - 1) // 4 + 2)
        sub = {k: v[t0 * per_row:t1 * per_row] for k, v in win.items()}
        got = O.ref_blend_rows(x[r0:r1], shape, kernel, r0, 16, t0, sub, threads=2)
        assert np.array_equal(got, want[r0:r1]), (r0, r1)
