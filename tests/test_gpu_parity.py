"""GPU parity: the sm_100a path against the oracle (oracle/) and the golden
fixtures the reference generated (tests/golden).

Bars (BASELINE.json north_star): bin indices, raw counts and clipped
histograms bit-exact; the f64 CDF/LUT is also bit-exact here (sequential f64
sums in bin order); the float32 output within 1e-5 absolute of the reference
float64 output (OUT_TOL).  Full-size configs are checked through
size-independent properties plus exact spot checks of sampled tiles/voxels.
"""
import glob
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
OUT_TOL = 1e-5
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


@pytest.fixture(scope="module")
def M():
    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import _native
    _native.lib()  # fails loudly if the CUDA library is missing
    return M


def gpu_stats(M, x, kernel, nb, clip, ad):
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    code = 1 if xt.dtype == torch.float64 else 0
    plan = M.Plan(x.shape, kernel, nb, clip, ad, code)
    st = plan.tile_stats(xt)
    return st, plan


def assert_stats_equal(st, ref, ctx=""):
    assert np.array_equal(st["degenerate"], ref["degenerate"]), ctx
    assert np.array_equal(st["lo"], ref["lo"]), ctx
    assert np.array_equal(st["hi"], ref["hi"]), ctx
    assert np.array_equal(st["counts"].astype(np.float64), ref["counts"]), ctx + " counts"
    assert np.array_equal(st["clipped"], ref["clipped"]), ctx + " clipped"
    assert np.array_equal(st["lut"], ref["lut"]), ctx + " lut"


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_golden(M, path):
    g = np.load(path)
    kernel = tuple(int(k) for k in g["kernel"])
    nb, clip, ad = int(g["n_bins"]), float(g["clip_limit"]), bool(g["adaptive"])
    st, _ = gpu_stats(M, g["x"], kernel, nb, clip, ad)
    assert_stats_equal(st, {k: g[k] for k in ("lo", "hi", "counts", "clipped", "lut",
                                               "degenerate")}, os.path.basename(path))
    out = M.enhance(g["x"], kernel, nb, clip, ad)
    assert out.dtype == np.float32
    assert np.max(np.abs(out.astype(np.float64) - g["out"])) <= OUT_TOL


def random_case(seed):
    rng = np.random.default_rng(1000 + seed)
    rank = 1 + seed % 5
    hi = {1: 300, 2: 70, 3: 24, 4: 12, 5: 8}[rank]
    shape = tuple(int(v) for v in rng.integers(2, hi, rank))
    kernel = tuple(int(rng.integers(1, s + 1)) for s in shape)
    nb = int(rng.choice([2, 3, 16, 64, 256]))
    clip = float(rng.choice([0.005, 0.05, 0.3, 1.0]))
    ad = bool(rng.integers(0, 2))
    kind = seed % 4
    if kind == 0:
        x = rng.random(shape)
    elif kind == 1:
        x = np.round(rng.random(shape) * 9) / 9          # values on bin edges
    elif kind == 2:
        x = rng.poisson(2.0, shape) / 7.0                # quantised, many zeros
    else:
        x = rng.normal(0, 3, shape)                      # signed
    return x.astype(np.float32), kernel, nb, clip, ad


@pytest.mark.parametrize("seed", range(40))
def test_random_shapes_vs_oracle(M, seed):
    x, kernel, nb, clip, ad = random_case(seed)
    st, _ = gpu_stats(M, x, kernel, nb, clip, ad)
    ref = O.tile_stats(x, kernel, nb, clip, ad, "c")
    assert_stats_equal(st, ref, f"seed {seed} {x.shape} {kernel} nb={nb} ad={ad}")
    out = M.enhance(x, kernel, nb, clip, ad)
    want = O.mclahe(x, kernel, nb, clip, ad, "c")
    assert np.max(np.abs(out.astype(np.float64) - want)) <= OUT_TOL


# the five BASELINE configs at oracle-sized scale (same structure, every extent / 4)
SCALED = {
    "2d": dict(shape=(256, 256), kernel=(16, 16), n_bins=256, clip_limit=0.01, adaptive=False),
    "3d": dict(shape=(64, 64, 64), kernel=(8, 8, 8), n_bins=256, clip_limit=0.02, adaptive=False),
    "4d": dict(shape=(64, 64, 32, 32), kernel=(8, 8, 4, 4), n_bins=256, clip_limit=0.02,
               adaptive=True),
    "l4d": dict(shape=(64, 64, 32, 32), kernel=(8, 8, 4, 8), n_bins=512, clip_limit=0.01,
                adaptive=False),
    "5d": dict(shape=(32, 32, 16, 16, 16), kernel=(4, 4, 2, 4, 4), n_bins=128, clip_limit=0.03,
               adaptive=True),
}


@pytest.mark.parametrize("name", list(SCALED))
def test_scaled_configs_vs_oracle(M, name):
    from paper_1906_11355_b200 import datasets
    c = SCALED[name]
    x = datasets.make(name, seed=1, shape=c["shape"]).numpy()
    args = (c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"])
    st, plan = gpu_stats(M, x, *args)
    assert plan.info.fast_hist and plan.info.fast_interp, "pencil kernels expected"
    # adaptive float32 single-slab plans count from the fused K2 kernel (k_fused.cu)
    # when it is switched on (opt-in: tests/test_fused_k2.py runs this file so)
    assert plan.flags["fused_k2"] == (c["adaptive"] and os.environ.get("MCLAHE_FUSED_K2") == "1")
    assert_stats_equal(st, O.tile_stats(x, *args, "c"), name)
    out = M.enhance(x, *args)
    want = O.mclahe(x, *args, "c")
    assert np.max(np.abs(out.astype(np.float64) - want)) <= OUT_TOL


def test_bin_index_adversarial(M):
    # values exactly on and one ulp around every bin edge of quantised data
    vals = []
    for m in (7, 12, 200, 500, 255, 1000):
        k = np.arange(0, m + 1, dtype=np.float64) / m
        vals.append(k)
    base = np.concatenate(vals).astype(np.float32)
    up = np.nextafter(base, np.float32(2))
    dn = np.nextafter(base, np.float32(-1))
    rng = np.random.default_rng(5)
    # far outside narrow ranges: y = (v - lo) * n / (hi - lo) spans +-1e38, the
    # magic-number add's whole domain (blend corners evaluate such voxels)
    mag = np.geomspace(1e-9, 3e38, 4000)
    far = np.concatenate([0.3 + mag, 0.3 - mag, mag, -mag]).astype(np.float32)
    v = np.concatenate([base, up, dn, rng.random(200000).astype(np.float32), far,
                        np.array([-1e30, 1e30, 0.0, -0.0, 3.4e38, -3.4e38], np.float32)])
    vt = torch.from_numpy(v).cuda()
    for lo, hi, n in [(0.0, 1.0, 256), (0.0, 1.0, 512), (0.02, 0.98, 128), (1 / 7, 6 / 7, 256),
                      (0.0, 3.0 / 500, 256), (-2.5, 1.0, 7), (0.3, 0.30000003, 64),
                      (0.3, 0.3000001, 256), (1e-30, 3e-30, 16384), (-3e38, 3e38, 256)]:
        lo32, hi32 = float(np.float32(lo)), float(np.float32(hi))
        want = O.bin_index_array(v.astype(np.float64), lo32, hi32, n)
        # generic, packed histogram, packed blend gather, bracketed floors (NB blend)
        for variant in (0, 1, 2, 3):
            got = M.bin_index_device(vt, lo32, hi32, n, variant).cpu().numpy()
            bad = np.flatnonzero(got != want)
            assert bad.size == 0, (lo, hi, n, variant, v[bad[:5]], got[bad[:5]], want[bad[:5]])
    # f64 values that are not float32-representable
    v64 = np.concatenate([np.arange(0, 3001) / 3000.0, rng.random(100000)])
    got = M.bin_index_device(torch.from_numpy(v64).cuda(), 0.0, 1.0, 256).cpu().numpy()
    assert np.array_equal(got, O.bin_index_array(v64, 0.0, 1.0, 256))


@pytest.mark.parametrize("ad", [True, False])
def test_flat_tile_beside_far_values(M, ad):
    # near-constant tiles (ranges of a few ulp) whose blend cells reach into
    # much darker / brighter regions: corners bin voxels with y far outside
    # [0, n) (here y ~ -1e9).  With kernel 32 on 128 columns the tiles cover
    # columns [32t-16, 32t+16) and cell t..t+1 spans [32t, 32t+32).
    rng = np.random.default_rng(21)
    x = np.empty((96, 128), np.float32)
    x[:, :48] = 0.5 + rng.integers(0, 3, (96, 48)) * np.float32(6e-8)
    x[:, 48:] = rng.random((96, 80)) * 0.01
    x[:48, 80:] = 0.9 + rng.random((48, 48)) * 1e-3
    args = ((32, 32), 256, 0.02, ad)
    st, plan = gpu_stats(M, x, *args)
    assert plan.info.fast_hist and plan.info.fast_interp
    assert_stats_equal(st, O.tile_stats(x, *args, "c"), "flat")
    out = M.enhance(x, *args)
    assert np.max(np.abs(out.astype(np.float64) - O.mclahe(x, *args, "c"))) <= OUT_TOL


def test_float64_input(M):
    rng = np.random.default_rng(11)
    x = np.round(rng.random((40, 36, 12)) * 1000) / 1000  # f64 values off the f32 grid
    args = ((8, 6, 4), 64, 0.05, True)
    st, _ = gpu_stats(M, x, *args)
    assert_stats_equal(st, O.tile_stats(x, *args, "c"), "f64")
    out = M.enhance(x, *args)
    assert out.dtype == np.float64
    assert np.max(np.abs(out - O.mclahe(x, *args, "c"))) <= OUT_TOL


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
@pytest.mark.parametrize("adaptive", [False, True])
def test_nonfinite_rejected(M, bad, adaptive):
    x = np.random.default_rng(0).random((32, 32)).astype(np.float32)
    x[5, 7] = bad
    with pytest.raises(M.ValidationError, match="non-finite"):
        M.enhance(x, (8, 8), 16, 0.1, adaptive)
    xt = torch.from_numpy(x).cuda()
    with pytest.raises(M.ValidationError, match="non-finite"):
        M.mclahe(M.McLaheRequest(xt, M.KernelSpec((8, 8)), M.EnhanceParams(0.1, 16)))


def test_constant_image(M):
    for ad in (False, True):
        out = M.enhance(np.full((40, 30, 8), 0.25, np.float32), (8, 8, 4), 32, 0.1, ad)
        assert np.all(out == 0.5)


def test_determinism_and_device_api(M):
    from paper_1906_11355_b200 import datasets
    c = SCALED["4d"]
    x = datasets.make("4d", seed=2, shape=c["shape"]).cuda()
    req = M.McLaheRequest(x, M.KernelSpec(c["kernel"]),
                          M.EnhanceParams(c["clip_limit"], c["n_bins"], M.RangeMode.Adaptive))
    a = M.mclahe(req)
    b = M.mclahe(req)
    assert torch.equal(a, b)
    host = M.mclahe(M.McLaheRequest(x.cpu().numpy(), req.kernel, req.params))
    assert np.array_equal(a.cpu().numpy(), host)


@pytest.mark.parametrize("name,slabs", [("2d", 2), ("3d", 3), ("4d", 4), ("l4d", 2), ("5d", 4),
                                        ("4d", 8)])
def test_fake_slabs_bit_identical(M, name, slabs):
    """The multi-GPU slab path (windows, partial counts, neighbour combine)
    emulated on one device must reproduce the single-GPU output bit for bit."""
    from paper_1906_11355_b200 import datasets, slabs as S
    c = SCALED[name]
    x = datasets.make(name, seed=3, shape=c["shape"]).cuda()
    args = (c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"])
    whole = M.enhance(x, *args)
    parts = S.run_local(x, *args, slabs=slabs)
    assert torch.equal(whole, parts)


@pytest.mark.parametrize("seed", range(6))
def test_fake_slabs_ragged(M, seed):
    from paper_1906_11355_b200 import slabs as S
    rng = np.random.default_rng(77 + seed)
    shape = (int(rng.integers(20, 60)), int(rng.integers(5, 30)), int(rng.integers(4, 12)))
    kernel = (int(rng.integers(2, 9)), int(rng.integers(1, shape[1] + 1)),
              int(rng.integers(1, shape[2] + 1)))
    x = torch.from_numpy(rng.random(shape).astype(np.float32)).cuda()
    ncell = len(S.cell_ranges(shape[0], kernel[0]))
    for g in sorted({2, min(3, ncell), ncell}):
        if g < 2:
            continue
        whole = M.enhance(x, kernel, 32, 0.1, bool(seed % 2))
        assert torch.equal(whole, S.run_local(x, kernel, 32, 0.1, bool(seed % 2), slabs=g))


FULL = ["2d", "3d", "4d", "5d", "l4d"]


@pytest.mark.parametrize("name", FULL)
def test_full_size_properties(M, name):
    """BASELINE sizes: tile mass = prod(kernel) for every binned tile, LUTs
    monotone ending at 1, output in [0, 1], run-to-run bit-identical, and
    exact spot checks of sampled tiles (counts by numpy from the padded
    block) and voxels (f64 blend from the GPU's f64 LUTs)."""
    from paper_1906_11355_b200 import datasets
    c = datasets.CONFIGS[name]
    x = datasets.make(name, seed=0, device="cuda")
    plan = M.Plan(x.shape, c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"])
    assert plan.info.fast_hist and plan.info.fast_interp
    st = plan.tile_stats(x)
    nb = c["n_bins"]
    binned = ~((st["lo"] >= st["hi"]))
    tile_len = int(np.prod(c["kernel"]))
    assert np.all(st["counts"][binned].sum(1) == tile_len)
    lut = st["lut"][~st["degenerate"]]
    assert np.all(np.diff(lut, axis=1) >= 0) and np.all(lut[:, -1] == 1.0)
    ws = plan.new_workspace()
    out = torch.empty_like(x)
    plan.enqueue(x, out, ws)
    plan.check(ws)
    out2 = torch.empty_like(x)
    plan.enqueue(x, out2, ws)
    plan.check(ws)
    assert torch.equal(out, out2)
    assert float(out.min()) >= 0.0 and float(out.max()) <= 1.0
    # spot check: padded tiles rebuilt on the host from the data
    rng = np.random.default_rng(9)
    grid = np.array(st_grid(plan))
    before = np.array(plan.info.before[:x.dim()])
    D = x.dim()
    for t in rng.choice(len(st["lo"]), 24, replace=False):
        tc = np.unravel_index(t, grid)
        idx = []
        for d in range(D):
            o = np.arange(tc[d] * c["kernel"][d], (tc[d] + 1) * c["kernel"][d]) - before[d]
            s = x.shape[d]
            m = np.mod(o, 2 * s)
            m = np.where(m >= s, 2 * s - 1 - m, m)
            idx.append(torch.from_numpy(m).cuda())
        blk = x.index_select(0, idx[0])
        for d in range(1, D):
            blk = blk.index_select(d, idx[d])
        blk = blk.double().cpu().numpy().ravel()
        lo, hi = (st["lo"][t], st["hi"][t])
        if not lo < hi:
            continue
        cnt = np.bincount(O.bin_index_array(blk, lo, hi, nb), minlength=nb)
        assert np.array_equal(cnt, st["counts"][t]), f"tile {t}"
    # spot check voxels: f64 blend with the GPU's f64 LUTs
    flat = rng.choice(x.numel(), 4000, replace=False)
    xs = x.view(-1)[torch.from_numpy(flat).cuda()].double().cpu().numpy()
    got = out.view(-1)[torch.from_numpy(flat).cuda()].double().cpu().numpy()
    gstride = np.cumprod((list(grid[1:]) + [1])[::-1])[::-1]
    shape = np.array(x.shape)
    for f, v, y in zip(flat, xs, got):
        coord = np.array(np.unravel_index(f, shape))
        lower, dlo, dhi, coeff = O.neighbors(coord + before, c["kernel"], grid, "c")
        mapped = []
        for cidx in range(1 << D):
            bits = [(cidx >> (D - 1 - j)) & 1 for j in range(D)]
            t = int(sum((lower[j] + bits[j]) * gstride[j] for j in range(D)))
            if st["degenerate"][t]:
                mapped.append(0.5)
            else:
                mapped.append(st["lut"][t][O.bin_index(float(v), st["lo"][t], st["hi"][t], nb)])
        assert abs(O.blend(coeff, mapped) - y) <= OUT_TOL


def st_grid(plan):
    return [int(plan.info.grid[j]) for j in range(plan.info.rank)]


@pytest.mark.parametrize("name", ["4d", "l4d"])
def test_streamed_host_api_matches_device(M, name):
    """The one-shot host call streams cell-aligned chunks through shared-
    workspace plans (H2D / compute / D2H overlapped); it must equal the
    whole-volume device path bit for bit."""
    from paper_1906_11355_b200 import datasets
    c = dict(SCALED[name])
    shape = (c["shape"][0] * 2,) + tuple(c["shape"][1:])  # >= 16 MB: several chunks
    x = datasets.make(name, seed=4, shape=shape)
    args = (c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"])
    dev = M.enhance(x.cuda(), *args).cpu().numpy()
    host = M.enhance(x.numpy(), *args)
    assert np.array_equal(dev, host)
    xn = x.numpy().copy()
    xn[-1, 3, 2, 1] = np.nan  # non-finite in the LAST chunk is still caught
    with pytest.raises(M.ValidationError, match="non-finite"):
        M.enhance(xn, *args)


@pytest.mark.parametrize("ad", [False, True])
def test_streamed_error_leaves_no_partial_output(M, ad):
    """a non-finite voxel in a late chunk must not leave a partial
    result in the caller's buffer.  Global mode never writes it (the flag is
    read after the range pass, before any blend / D2H); adaptive mode scrubs
    it with NaN (early chunks were already copied back)."""
    import ctypes as C
    from paper_1906_11355_b200 import _native as N
    from paper_1906_11355_b200 import datasets
    c = dict(SCALED["4d"])
    shape = (c["shape"][0] * 2,) + tuple(c["shape"][1:])
    x = datasets.make("4d", seed=5, shape=shape).numpy().copy()
    x[-1, 5, 4, 3] = np.inf
    params = N.make_params(x.shape, c["kernel"], c["n_bins"], c["clip_limit"], ad, 0)
    out = np.full_like(x, 7.0)
    rc = N.lib().mclahe_gpu_run(C.byref(params), x.ctypes.data, out.ctypes.data, None)
    assert rc == 1 and b"non-finite" in N.lib().mclahe_last_error()
    if ad:
        assert np.isnan(out).all()
    else:
        assert np.all(out == 7.0)


def test_framewise_global_rank4_folded_geometry(M):
    """a global framewise call whose per-frame geometry
    would arm the folded-pair blend (one trailing dim, multiple of 32) must
    not launch it -- the frame plan has no dictionary tables."""
    rng = np.random.default_rng(81)
    x = (rng.poisson(3.0, (8, 64, 64, 32)) / 11.0).astype(np.float32)
    kernel = (16, 16, 4)
    params = M.EnhanceParams(0.02, 64, M.RangeMode.Global)
    out = M.mclahe_framewise(x, 0, M.KernelSpec(kernel), params)
    want = _framewise_oracle(x, 0, kernel, 64, 0.02, False, False)
    assert np.max(np.abs(out.astype(np.float64) - want)) <= OUT_TOL


def _run_plan(M, x, kernel, nb, clip, ad, no_dict=False, cell_hist=False):
    old = os.environ.pop("MCLAHE_NO_DICT", None)
    old_c = os.environ.pop("MCLAHE_CELL_HIST", None)
    if no_dict:
        os.environ["MCLAHE_NO_DICT"] = "1"
    if cell_hist:
        os.environ["MCLAHE_CELL_HIST"] = "1"
    try:
        plan = M.Plan(x.shape, kernel, nb, clip, ad)
    finally:
        os.environ.pop("MCLAHE_NO_DICT", None)
        os.environ.pop("MCLAHE_CELL_HIST", None)
        if old is not None:
            os.environ["MCLAHE_NO_DICT"] = old
        if old_c is not None:
            os.environ["MCLAHE_CELL_HIST"] = old_c
    xt = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x)).cuda()
    ws = plan.new_workspace()
    out = torch.empty_like(xt)
    plan.enqueue(xt, out, ws)
    plan.check(ws)
    return out, plan.dict_state(ws)


@pytest.mark.parametrize("case", ["poisson", "rare", "ragged"])
def test_cell_histogram_variant(M, case):
    """K2b by dictionary cell (k_hist_cells, MCLAHE_CELL_HIST=1): voxels counted per
    (tile, value), cell counts turned into bin counts at the unit switch, values the
    sampled dictionary lacks binned on the spot -- the result must equal the
    edge-table K2b's bit for bit (same counts -> same LUTs -> same output)."""
    rng = np.random.default_rng({"poisson": 11, "rare": 12, "ragged": 13}[case])
    if case == "poisson":
        x = (rng.poisson(3.0, (48, 40, 24, 32)) / 11.0).astype(np.float32)
        args = ((12, 10, 6, 4), 256, 0.02, True)
    elif case == "rare":
        x = (rng.poisson(3.0, (32, 32, 16, 32)) / 11.0).astype(np.float32)
        pos = rng.choice(x.size, 400, replace=False)
        x.reshape(-1)[pos] = (0.3 + np.arange(400) * 1e-4).astype(np.float32)
        args = ((8, 8, 4, 4), 256, 0.02, True)
    else:  # mirrored padding in every outer dim: non-uniform row weights
        x = (rng.poisson(5.0, (37, 29, 19, 32)) / 17.0).astype(np.float32)
        x[:6] = 0.25  # degenerate tiles
        args = ((8, 8, 4, 4), 128, 0.03, True)
    a, da = _run_plan(M, x, *args)
    b, db = _run_plan(M, x, *args, cell_hist=True)
    assert da["used"] and db["used"]
    assert torch.equal(a, b)
    want = O.mclahe(x, *args, "c")
    assert np.max(np.abs(b.cpu().numpy().astype(np.float64) - want)) <= OUT_TOL


@pytest.mark.parametrize("case", ["poisson", "edges", "scaled4d", "many", "uneven", "rare", "wide",
                                  "levels"])
def test_value_dictionary_blend(M, case):
    # quantised volumes (few distinct values) take the value-dictionary blend
    # (rank 4 with one trailing dim: the folded-pair kernel k_interp_mdict);
    # it must equal the oracle and, bit for bit, the edge-table blend
    rng = np.random.default_rng({"poisson": 1, "edges": 2, "scaled4d": 3, "many": 4, "uneven": 5,
                                 "rare": 6, "wide": 7, "levels": 8}[case])
    if case == "poisson":
        x = (rng.poisson(3.0, (48, 40, 24, 32)) / 11.0).astype(np.float32)
        args = ((12, 10, 6, 4), 256, 0.02, True)
    elif case == "rare":  # values the sampled dictionary misses: the workspace-LUT path
        x = (rng.poisson(3.0, (32, 32, 16, 32)) / 11.0).astype(np.float32)
        pos = rng.choice(x.size, 400, replace=False)
        x.reshape(-1)[pos] = (0.3 + np.arange(400) * 1e-4).astype(np.float32)
        args = ((8, 8, 4, 4), 256, 0.02, True)
    elif case == "wide":  # trailing cells of two columns, eight 8-float segments
        x = (rng.poisson(2.0, (32, 24, 16, 64)) / 7.0).astype(np.float32)
        args = ((8, 8, 4, 8), 128, 0.03, True)
    elif case == "edges":
        x = (np.round(rng.random((40, 36, 32)) * 9) / 9).astype(np.float32)
        x[:8] = 0.5  # constant (degenerate) tiles too
        args = ((8, 12, 8), 128, 0.05, True)
    elif case == "scaled4d":
        from paper_1906_11355_b200 import datasets
        c = SCALED["4d"]
        x = datasets.make("4d", seed=2, shape=c["shape"]).numpy()
        args = (c["kernel"], c["n_bins"], c["clip_limit"], True)
    elif case == "uneven":  # few values, unevenly spaced: cuckoo lookup
        vals = np.sort(rng.random(300)).astype(np.float32)
        vals[:3] = [0.0, 1e-6, 2e-6]
        x = vals[rng.integers(0, 300, (32, 32, 16, 32))]
        args = ((8, 8, 4, 4), 256, 0.02, True)
    elif case == "levels":  # 1501 levels: too many for the dictionary, quantised (edge mode)
        x = (np.round(rng.random((32, 32, 16, 32)) * 1500) / 1500).astype(np.float32)
        args = ((8, 8, 4, 4), 256, 0.02, True)
    else:  # more distinct values than the dictionary holds: edge-table blend
        x = rng.random((32, 32, 16, 32)).astype(np.float32)
        args = ((8, 8, 4, 4), 256, 0.02, True)
    out, st = _run_plan(M, x, *args)
    ref, st0 = _run_plan(M, x, *args, no_dict=True)
    assert st0["capacity"] == 0 and not st0["used"]
    assert st["capacity"] > 0
    assert st["used"] == (case not in ("many", "levels")), st
    # folded pairs: rank 4, one trailing dim, power-of-two cells (>= 32-row stages)
    assert st["folded"] == (case in ("scaled4d", "uneven", "rare", "wide")), st
    if case not in ("many", "levels"):  # K2a samples one row in eight
        assert 0 < st["values"] <= len(np.unique(x.view(np.uint32))), st
        if case == "rare":
            assert st["values"] < len(np.unique(x.view(np.uint32))), st  # misses exercised
        assert st["affine"] == (case not in ("uneven", "rare")), st  # evenly quantised: direct table
        # counts over a common denominator: the affine cell is the index itself
        assert st["direct"] == (case in ("poisson", "edges", "scaled4d", "wide")), st
    assert torch.equal(out, ref)
    want = O.mclahe(x, *args, "c")
    assert np.max(np.abs(out.cpu().numpy().astype(np.float64) - want)) <= OUT_TOL


def test_value_dictionary_direct_cells_misses(M):
    """Direct-cell dictionary (values numbered by their affine cell): voxels
    whose value is off the lattice or beyond either end of it (cells clamped
    to the last one, negative offsets wrapping) fail the 32-bit check and take
    the workspace-LUT path; the result equals the edge-table blend bit for bit."""
    rng = np.random.default_rng(61)
    x = (rng.poisson(3.0, (32, 32, 16, 32)) / 11.0).astype(np.float32)
    flat = x.reshape(-1)
    pos = rng.choice(x.size, 3, replace=False)
    flat[pos] = np.array([100.0, 0.5 / 11.0, -0.25], np.float32)
    args = ((8, 8, 4, 4), 256, 0.02, True)
    out, st = _run_plan(M, x, *args)
    ref, _ = _run_plan(M, x, *args, no_dict=True)
    assert st["used"] and st["folded"], st
    assert torch.equal(out, ref)
    want = O.mclahe(x, *args, "c")
    assert np.max(np.abs(out.cpu().numpy().astype(np.float64) - want)) <= OUT_TOL
    if st["values"] == len(np.unique(x)) - 3:  # none of the three was sampled
        assert st["direct"], st


@pytest.mark.parametrize("nb", [128, 256, 512])
def test_folded_pair_blend_global_mode(M, nb):
    # global range, one trailing dim, three outer dims: the folded-pair blend
    # (tables per bin) runs; it equals the oracle and, bit for bit, the
    # edge-table kernel of the streamed host call
    rng = np.random.default_rng(nb)
    x = np.clip(rng.normal(0.4, 0.15, (48, 64, 32, 32)), 0, 1).astype(np.float32)
    x[:, :, 20:] = np.round(x[:, :, 20:] * 9) / 9  # values on bin edges too
    args = ((16, 16, 8, 8), nb, 0.01, False)
    out, st = _run_plan(M, x, *args)
    assert st["folded"] and not st["used"] and st["capacity"] == 0, st
    want = O.mclahe(x, *args, "c")
    assert np.max(np.abs(out.cpu().numpy().astype(np.float64) - want)) <= OUT_TOL
    xx = np.concatenate([x] * 4)  # >= 16 MB: the one-shot host call streams chunks
    dev, _ = _run_plan(M, xx, *args)
    host = M.enhance(xx, *args)
    assert np.array_equal(dev.cpu().numpy(), host)


def test_folded_pair_blend_pathological_global_range(M):
    # a global range of denormals (n / (hi - lo) overflows f32): the folded-pair
    # blend bins every voxel by bisecting the edge table
    rng = np.random.default_rng(31)
    x = (rng.integers(1, 9, (32, 32, 16, 32)) * np.float32(1e-40)).astype(np.float32)
    args = ((8, 8, 4, 4), 256, 0.02, False)
    out, st = _run_plan(M, x, *args)
    assert st["folded"], st
    want = O.mclahe(x, *args, "c")
    assert np.max(np.abs(out.cpu().numpy().astype(np.float64) - want)) <= OUT_TOL


@pytest.mark.parametrize("ad", [True, False])
def test_sparse_counts_degenerate_neighbours(M, ad):
    # counts on one half of the trailing dim, zeros on the other: constant
    # (degenerate) tiles beside live ones along the trailing dim, so merged
    # histogram runs meet tiles that build no histogram
    rng = np.random.default_rng(33)
    x = np.zeros((32, 32, 16, 32), np.float32)
    x[..., :2] = rng.poisson(0.7, (32, 32, 16, 2)) / 3.0  # trailing tile 0: x in [0, 2)
    x[..., 20:] = rng.poisson(0.7, (32, 32, 16, 12)) / 3.0
    args = ((8, 8, 4, 4), 256, 0.02, ad)
    st, plan = gpu_stats(M, x, *args)
    assert plan.info.fast_hist and plan.info.fast_interp
    ref = O.tile_stats(x, *args, "c")
    if ad:
        assert ref["degenerate"].any() and not ref["degenerate"].all()
    assert_stats_equal(st, ref, "sparse")
    out = M.enhance(x, *args)
    assert np.max(np.abs(out.astype(np.float64) - O.mclahe(x, *args, "c"))) <= OUT_TOL


def _framewise_oracle(x, axis, kernel, nb, clip, ad, renorm):
    outs = []
    for f in range(x.shape[axis]):
        sl = np.take(x, f, axis=axis).astype(np.float64)
        if renorm:
            lo, hi = sl.min(), sl.max()
            sl = (sl - lo) / (hi - lo) if hi > lo else np.full_like(sl, 0.5)
        outs.append(O.mclahe(sl, kernel, nb, clip, ad, "c"))
    return np.stack(outs, axis=axis)


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("ad", [False, True])
def test_framewise_batched_vs_per_slice_oracle(M, axis, ad):
    # mclahe_framewise (src/pipeline.cpp:131-153) in one batched GPU run
    rng = np.random.default_rng(60 + axis + 3 * ad)
    shape = [20, 24, 28]
    x = (rng.poisson(2.5, shape) / 9.0).astype(np.float32)
    x[..., :3] = 0.4  # constant strips: degenerate tiles / frames
    kernel = tuple(k for j, k in enumerate((6, 8, 7)) if j != axis)
    params = M.EnhanceParams(0.05, 64, M.RangeMode.Adaptive if ad else M.RangeMode.Global)
    out = M.mclahe_framewise(x, axis, M.KernelSpec(kernel), params)
    assert out.dtype == np.float32 and out.shape == x.shape
    want = _framewise_oracle(x, axis, kernel, 64, 0.05, ad, False)
    assert np.max(np.abs(out.astype(np.float64) - want)) <= OUT_TOL


@pytest.mark.parametrize("ad", [False, True])
def test_framewise_renormalized_and_4d(M, ad):
    rng = np.random.default_rng(71 + ad)
    x = (rng.normal(0, 2, (6, 18, 20, 8))).astype(np.float32)
    x[2] = 3.0  # a constant frame
    kernel = (6, 5, 4)
    params = M.EnhanceParams(0.1, 32, M.RangeMode.Adaptive if ad else M.RangeMode.Global)
    for renorm in (False, True):
        out = M.mclahe_framewise(x, 0, M.KernelSpec(kernel), params, renormalize_slices=renorm)
        want = _framewise_oracle(x, 0, kernel, 32, 0.1, ad, renorm)
        assert np.max(np.abs(out.astype(np.float64) - want)) <= OUT_TOL, renorm


@pytest.mark.parametrize("rank", [6, 7, 8])
@pytest.mark.parametrize("ad", [False, True])
def test_high_rank_vs_oracle(M, rank, ad):
    # the reference accepts rank <= 8 (nd_image.cpp:52-58): generic kernels
    rng = np.random.default_rng(90 + rank)
    shape = tuple(int(v) for v in rng.integers(2, 5, rank))
    kernel = tuple(int(rng.integers(1, s + 1)) for s in shape)
    x = (np.round(rng.random(shape) * 20) / 20).astype(np.float32)
    st, _ = gpu_stats(M, x, kernel, 16, 0.2, ad)
    assert_stats_equal(st, O.tile_stats(x, kernel, 16, 0.2, ad, "c"), f"rank {rank}")
    out = M.enhance(x, kernel, 16, 0.2, ad)
    assert np.max(np.abs(out.astype(np.float64) - O.mclahe(x, kernel, 16, 0.2, ad, "c"))) <= OUT_TOL


def test_large_n_bins_and_concurrent_host_calls(M):
    # n_bins up to the GPU limit through the pencil path, and the one-shot C
    # entry called from several host threads at once (its state is locked)
    import threading
    rng = np.random.default_rng(17)
    x = rng.random((48, 40, 32)).astype(np.float32)
    for nb, ad in ((4096, True), (16384, False)):
        out = M.enhance(x, (16, 8, 8), nb, 0.5, ad)
        assert np.max(np.abs(out.astype(np.float64) - O.mclahe(x, (16, 8, 8), nb, 0.5, ad, "c"))) <= OUT_TOL
    want = M.enhance(x, (12, 10, 8), 64, 0.05, True)
    res, errs = [None] * 6, []

    def work(i):
        try:
            res[i] = M.enhance(x, (12, 10, 8), 64, 0.05, True)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    th = [threading.Thread(target=work, args=(i,)) for i in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs and all(np.array_equal(r, want) for r in res)
