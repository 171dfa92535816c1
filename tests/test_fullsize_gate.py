"""Full-size parity gate: the sm_100a path against the COMPILED REFERENCE
(oracle/_ref, built from /root/reference sources) on the BASELINE.json
configs at their full sizes, seed 0.

* 2D, 3D, 4D, 5D: every tile's range, degenerate flag, raw counts, clipped
  histogram and f64 LUT bit-exact (reference symmetric_pad / kernelize /
  build_mappings / compute_histogram / clip_histogram,
  src/histogram.cpp:72-106), and every voxel of the output within 1e-5 of the
  reference's mclahe::mclahe (src/pipeline.cpp:73-129, all host threads).
* Large 4D (2.15G voxels; the reference's padded + kernelized float64 copies
  alone would be ~61 GB): tile rows {0,1}, {4,5} and {7,8} -- both boundary
  rows and an interior pair -- through dim-0 crops that reproduce those tile
  rows exactly (oracle.ref_tile_rows_by_crop, pinned on CPU by
  tests/test_oracle_window.py), every tile bit-exact; every voxel of rows
  [0, 32), [256, 288) and [480, 512) through the reference's own per-voxel
  loop (neighbor_kernels / interp_coefficients / transform_pixel) over those
  mappings, within 1e-5.  The Global range is the full volume's min/max.
  MCLAHE_GATE_L4D_ALL=1 walks every tile row and every voxel the same way, one
  interpolation cell of rows at a time (~5 min of reference time; recorded in
  profiles/r02_fullsize_gate.txt).

Prints one summary line per config (run with -s to see it).
"""
import os
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")]
OUT_TOL = 1e-5
STAT_KEYS = ("lo", "hi", "counts", "clipped", "lut", "degenerate")


@pytest.fixture(scope="module")
def M():
    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import _native
    _native.lib()
    return M


def _assert_tiles(st, ref, sl, ctx):
    for k in STAT_KEYS:
        got = st[k][sl]
        if k == "counts":
            got = got.astype(np.float64)
        bad = np.flatnonzero(~(got == ref[k]).reshape(len(ref["lo"]), -1).all(axis=1))
        assert bad.size == 0, f"{ctx}: {k} differs in {bad.size} tiles (first {bad[:5]})"


@pytest.mark.parametrize("name", ["2d", "3d", "4d", "5d"])
def test_fullsize_every_tile_and_voxel_vs_reference(M, name):
    from paper_1906_11355_b200 import datasets
    cfg = datasets.CONFIGS[name]
    kernel, nb, clip, ad = cfg["kernel"], cfg["n_bins"], cfg["clip_limit"], cfg["adaptive"]
    xt = datasets.make(name, seed=0, device="cuda")
    assert tuple(xt.shape) == tuple(cfg["shape"])
    plan = M.Plan(xt.shape, kernel, nb, clip, ad)
    st = plan.tile_stats(xt)
    out = M.enhance(xt, kernel, nb, clip, ad).cpu().numpy().astype(np.float64)
    x = xt.cpu().numpy()
    del xt
    t0 = time.perf_counter()
    g0 = int(plan.info.grid[0])
    ref = O.ref_tile_stats_window(x, kernel, nb, clip, ad, 0, g0)
    t_stats = time.perf_counter() - t0
    _assert_tiles(st, ref, slice(None), name)
    t0 = time.perf_counter()
    want = O.mclahe(x, kernel, nb, clip, ad, "ref", threads=0)
    t_ref = time.perf_counter() - t0
    err = float(np.max(np.abs(out - want)))
    print(f"[gate] {name}: {x.size} voxels, {len(ref['lo'])} tiles bit-exact "
          f"(lo/hi/degenerate/counts/clipped/lut), {int(ref['degenerate'].sum())} degenerate, "
          f"max|out - ref| = {err:.3e} over every voxel; reference {t_ref:.1f} s "
          f"(+{t_stats:.1f} s tile stats)")
    assert err <= OUT_TOL


def test_fullsize_l4d_tile_row_windows_vs_reference(M):
    from paper_1906_11355_b200 import datasets
    name = "l4d"
    cfg = datasets.CONFIGS[name]
    shape, kernel = tuple(cfg["shape"]), tuple(cfg["kernel"])
    nb, clip, ad = cfg["n_bins"], cfg["clip_limit"], cfg["adaptive"]
    xt = datasets.make(name, seed=0, device="cuda")
    plan = M.Plan(shape, kernel, nb, clip, ad)
    st = plan.tile_stats(xt)
    out_t = M.enhance(xt, kernel, nb, clip, ad)
    x = xt.cpu().numpy()
    del xt
    grange = (float(x.min()), float(x.max()))  # NdImage::min_max is exact: same values
    per_row = int(np.prod([int(plan.info.grid[j]) for j in range(1, len(shape))]))
    b0 = kernel[0]
    total_tiles = total_vox = 0
    worst = 0.0
    t0s = time.perf_counter()
    windows = [((0, 2), (0, b0 // 2)), ((4, 6), (4 * b0, 4 * b0 + b0 // 2)),
               ((7, 9), (shape[0] - b0 // 2, shape[0]))]
    every = os.environ.get("MCLAHE_GATE_L4D_ALL") == "1"
    if every:  # every tile row and every voxel, one interpolation cell of rows at a time
        windows = [((t, t + 2), (t * b0, min(shape[0], (t + 1) * b0))) for t in range(shape[0] // b0)]
    for (ta, tb), (ra, rb) in windows:
        ref, _ = O.ref_tile_rows_by_crop(x, kernel, nb, clip, ad, ta, tb, grange)
        _assert_tiles(st, ref, slice(ta * per_row, tb * per_row), f"{name} tile rows {ta}-{tb}")
        want = O.ref_blend_rows(x[ra:rb], shape, kernel, ra, nb, ta, ref)
        got = out_t[ra:rb].cpu().numpy().astype(np.float64)
        err = float(np.max(np.abs(got - want)))
        assert err <= OUT_TOL, (ra, rb, err)
        worst = max(worst, err)
        total_tiles += len(ref["lo"])
        total_vox += want.size
    what = ("every tile row (windows " + ", ".join(f"{a}-{b - 1}" for (a, b), _ in windows) + ")"
            if every else "tile rows 0-1, 4-5, 7-8")
    rows = "every row" if every else "rows 0-31, 256-287, 480-511"
    print(f"[gate] l4d: {what} ({total_tiles} tile checks) bit-exact, "
          f"{total_vox} voxels ({rows}) max|out - ref| = {worst:.3e}; "
          f"reference {time.perf_counter() - t0s:.1f} s")
