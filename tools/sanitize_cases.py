"""Small runs of every kernel family, for compute-sanitizer (memcheck /
racecheck / synccheck): tools/sanitize.sh runs this file under each tool.
Each case checks its result against the oracle so a silent corruption under
the tool also fails."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_11355_b200 as M  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1906_11355_b200 import _native as N  # noqa: E402
from paper_1906_11355_b200 import datasets  # noqa: E402

TOL = 1e-5


def check(name, got, want):
    err = float(np.max(np.abs(np.asarray(got, np.float64) - want)))
    print(f"{name}: max|err| = {err:.2e}", flush=True)
    assert err <= TOL, name


def case_pencils():
    for name, shape, kernel, nb, clip, ad in [
        ("4d-dict-mdict", (64, 64, 32, 32), (8, 8, 4, 4), 256, 0.02, True),
        ("l4d-global-mdict", (32, 64, 32, 32), (8, 8, 4, 8), 512, 0.01, False),
        ("5d-nb", (16, 16, 16, 16, 16), (4, 4, 2, 4, 4), 128, 0.03, True),
        ("3d-global", (64, 48, 40), (8, 8, 8), 256, 0.02, False),
    ]:
        base = name.split("-")[0]
        x = datasets.make(base, seed=2, shape=shape).numpy()
        plan = M.Plan(x.shape, kernel, nb, clip, ad)
        xt = torch.from_numpy(x).cuda()
        ws = plan.new_workspace()
        out = torch.empty_like(xt)
        plan.enqueue(xt, out, ws)
        plan.check(ws)
        print(name, plan.dict_state(ws), flush=True)
        st = plan.tile_stats(xt)
        ref = O.tile_stats(x, kernel, nb, clip, ad, "c")
        for k in ("lo", "hi", "clipped", "lut", "degenerate"):
            assert np.array_equal(st[k], ref[k]), (name, k)
        check(name, out.cpu().numpy(), O.mclahe(x, kernel, nb, clip, ad, "c"))


def case_generic():
    rng = np.random.default_rng(3)
    x = rng.random((20, 18, 16))  # float64: generic kernels
    check("f64-generic", M.enhance(x, (5, 6, 4), 32, 0.1, True), O.mclahe(x, (5, 6, 4), 32, 0.1, True, "c"))
    x6 = np.round(rng.random((4, 3, 5, 4, 3, 4)) * 20).astype(np.float32) / 20
    check("rank6-generic", M.enhance(x6, (2, 3, 2, 2, 3, 2), 16, 0.2, False),
          O.mclahe(x6, (2, 3, 2, 2, 3, 2), 16, 0.2, False, "c"))


def case_streamed_and_framewise():
    x = datasets.make("4d", seed=3, shape=(128, 64, 32, 32)).numpy()  # 32 MB: streamed chunks
    check("streamed-host", M.enhance(x, (16, 8, 4, 4), 256, 0.02, True),
          O.mclahe(x, (16, 8, 4, 4), 256, 0.02, True, "c"))
    rng = np.random.default_rng(4)
    v = (rng.poisson(3.0, (8, 24, 20)) / 9.0).astype(np.float32)
    p = M.EnhanceParams(0.05, 32, M.RangeMode.Global)
    out = M.mclahe_framewise(v, 0, M.KernelSpec((6, 5)), p)
    want = np.stack([O.mclahe(v[f].astype(np.float64), (6, 5), 32, 0.05, False, "c") for f in range(8)])
    check("framewise-global", out, want)


def case_filters_and_ops():
    rng = np.random.default_rng(5)
    x = rng.random((12, 14, 10))
    g = M.gaussian_filter(x, M.GaussianSpec((1.0, 0.5, 0.0)))
    check("gaussian", g, O.gaussian_filter_np(x, (1.0, 0.5, 0.0)))
    m = M.median_filter(x, M.MedianSpec((3, 2, 1)))
    check("median", m, O.median_filter_np(x, (3, 2, 1)))
    M.compute_metrics(g, x, 64)
    L = N.lib()
    blocks = np.ascontiguousarray(rng.random((6, 500)))
    lo, hi, deg = np.zeros(6), np.zeros(6), np.zeros(6, np.uint8)
    lut = np.zeros((6, 64))
    f64p = C.POINTER(C.c_double)
    rc = L.mclahe_block_mappings(blocks.ctypes.data_as(f64p), C.c_int64(6), C.c_int64(500),
                                 C.c_int64(64), C.c_double(0.05), C.c_int32(1), C.c_double(0.0),
                                 C.c_double(1.0), lo.ctypes.data_as(f64p), hi.ctypes.data_as(f64p),
                                 None, None, lut.ctypes.data_as(f64p),
                                 deg.ctypes.data_as(C.POINTER(C.c_uint8)))
    assert rc == 0
    for k in range(6):  # build_mappings restated: own min/max, bins, clip, CDF
        b = blocks[k]
        assert lo[k] == b.min() and hi[k] == b.max() and deg[k] == 0, k
        cnt = np.bincount(O.bin_index_array(b, b.min(), b.max(), 64), minlength=64)
        want, _ = O.normalized_cdf(O.clip_histogram(cnt.astype(np.float64), 0.05))
        assert np.array_equal(lut[k], want), k
    print("block_mappings: ok", flush=True)
    shp = np.array([12, 14, 10], np.int64)
    bef, aft = np.array([3, 0, 4], np.int64), np.array([2, 5, 1], np.int64)
    out = np.zeros((17, 19, 15))
    i64p = C.POINTER(C.c_int64)
    assert L.mclahe_nd_gather(0, 3, shp.ctypes.data_as(i64p), bef.ctypes.data_as(i64p),
                              aft.ctypes.data_as(i64p), x.ctypes.data_as(f64p),
                              out.ctypes.data_as(f64p)) == 0
    idx = [O.mirror_index_array(np.arange(-bef[j], shp[j] + aft[j]), shp[j]) for j in range(3)]
    assert np.array_equal(out, x[np.ix_(*idx)])
    print("nd_gather: ok", flush=True)


if __name__ == "__main__":
    for fn in (case_pencils, case_generic, case_streamed_and_framewise, case_filters_and_ops):
        fn()
    print("SANITIZE_CASES_OK", flush=True)
