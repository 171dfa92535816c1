"""The C++ drop-in (include/mclahe/*.hpp + libmclahe_cpp.so): programs
written against the reference API compile, link and run unchanged.

Two callers: tests/cpp/dropin_example.cpp, and oracle/ref_shim.cpp -- the
test shim that drives the REAL reference library (oracle/_ref) through its
public API (mclahe, build_mappings, compute_histogram, clip_histogram,
normalized_cdf, bin_index, neighbor_kernels, interp_coefficients,
transform_pixel, symmetric_pad, kernelize, min_max, parallel_for, filters,
metrics, NPY, NdImage::values()).  Compiled UNMODIFIED against the B200
headers and linked to libmclahe_cpp.so, it must reproduce the reference bit
for bit (output within 1e-5)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1906_11355_b200", "lib")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    from paper_1906_11355_b200 import _native
    _native.lib()
    if not os.path.exists(os.path.join(LIB, "libmclahe_cpp.so")):
        _native.build()
    out = str(tmp_path_factory.mktemp("cpp") / "dropin_example")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp"), "-L", LIB,
                    "-lmclahe_cpp", "-lmclahe_gpu", f"-Wl,-rpath,{LIB}", "-o", out], check=True)
    return out


def test_compiles_links_and_validates(exe):
    r = subprocess.run([exe, "validate"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "clip_limit must be in (0, 1]" in r.stdout


@pytest.mark.gpu
def test_runs_on_gpu_and_matches_oracle(exe):
    from oracle import oracle as O
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    got = np.array([float(v) for v in r.stdout.split()]).reshape(24, 20, 16)
    i = np.arange(24 * 20 * 16)
    x = (((i * 37) % 101) / 100.0).reshape(24, 20, 16)
    want = O.mclahe(x, (8, 4, 4), 32, 0.05, True, "c")
    assert np.max(np.abs(got - want)) <= 1e-5


@pytest.mark.gpu
def test_framewise_batched_matches_per_slice_oracle(exe):
    from oracle import oracle as O
    r = subprocess.run([exe, "framewise"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    got = np.array([float(v) for v in r.stdout.split()]).reshape(24, 20, 16)
    i = np.arange(24 * 20 * 16)
    x = (((i * 37) % 101) / 100.0).reshape(24, 20, 16)
    want = np.stack([O.mclahe(x[:, f, :], (8, 4), 32, 0.05, False, "c") for f in range(20)], 1)
    assert np.max(np.abs(got - want)) <= 1e-5


@pytest.mark.gpu
def test_filters_and_metrics_match_reference(exe):
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("reference library not built")
    r = subprocess.run([exe, "filters"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    vals = np.array([float(v) for v in r.stdout.split()])
    i = np.arange(24 * 20 * 16)
    x = (((i * 37) % 101) / 100.0).reshape(24, 20, 16)
    g = O.gaussian_filter_ref(x, (1.0, 0.5, 0.0), 4.0)
    m = O.median_filter_ref(g, (3, 1, 2))
    assert np.array_equal(vals[:-4].reshape(x.shape), m)
    want = O.metrics_ref(m, x, 64, 1.0)
    got = vals[-4:]
    assert got[3] == want["entropy_bits"]
    for k, v in zip(("mse", "psnr_db", "std"), got[:3]):
        assert abs(v - want[k]) <= 1e-12 * max(1.0, abs(want[k])), k


@pytest.fixture(scope="module")
def shim_b200(tmp_path_factory):
    """oracle/ref_shim.cpp, unmodified, against include/mclahe/*.hpp."""
    from paper_1906_11355_b200 import _native
    _native.lib()
    if not os.path.exists(os.path.join(LIB, "libmclahe_cpp.so")):
        _native.build()
    out = str(tmp_path_factory.mktemp("shim") / "libshim_b200.so")
    subprocess.run(["g++", "-O3", "-DNDEBUG", "-std=gnu++20", "-fPIC", "-shared", "-pthread",
                    "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "oracle", "ref_shim.cpp"), "-L", LIB, "-lmclahe_cpp",
                    "-lmclahe_gpu", f"-Wl,-rpath,{LIB}", "-o", out], check=True)
    os.environ["MCLAHE_SHIM_B200"] = out
    from oracle import oracle as O
    O._LIBS.pop("b200", None)
    return out


def test_unmodified_reference_caller_compiles_and_links(shim_b200):
    lib = ctypes.CDLL(shim_b200)
    for sym in ("ref_mclahe", "ref_tile_stats", "ref_tile_stats_window", "ref_blend_rows",
                "ref_bin_index", "ref_clip_histogram", "ref_normalized_cdf", "ref_neighbors",
                "ref_transform_pixel", "ref_gaussian", "ref_median", "ref_metrics",
                "ref_write_npy", "ref_read_npy"):
        assert hasattr(lib, sym), sym


def test_scalar_api_matches_reference(shim_b200):
    """Host scalar steps of the per-op API: bit-identical to the reference."""
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("reference library not built")
    rng = np.random.default_rng(11)
    for _ in range(200):
        lo, hi = sorted(rng.normal(0, 2, 2))
        v = float(rng.normal(lo, 3))
        n = int(rng.integers(2, 600))
        assert O.bin_index(v, lo, hi, n, "b200") == O.bin_index(v, lo, hi, n, "ref")
    c = rng.poisson(5.0, 256).astype(np.float64)
    for clip in (0.004, 0.02, 0.3, 1.0):
        a = O.clip_histogram(c, clip, "b200")
        assert np.array_equal(a, O.clip_histogram(c, clip, "ref"))
        assert all(np.array_equal(x, y) for x, y in
                   zip(O.normalized_cdf(a, "b200"), O.normalized_cdf(a, "ref")))
    grid, kernel = (5, 4, 6), (8, 6, 4)
    for _ in range(100):
        px = [int(rng.integers(kernel[j] // 2, (grid[j] - 1) * kernel[j])) for j in range(3)]
        a = O.neighbors(px, kernel, grid, "b200")
        b = O.neighbors(px, kernel, grid, "ref")
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
        luts = rng.random((8, 16))
        los, his = rng.random(8) * 0.1, 0.5 + rng.random(8)
        dg = (rng.random(8) < 0.2).astype(np.uint8)
        v = float(rng.random())
        assert O.transform_pixel_ref(v, luts, los, his, dg, a[3], "b200") == \
            O.transform_pixel_ref(v, luts, los, his, dg, b[3], "ref")


@pytest.mark.gpu
@pytest.mark.parametrize("adaptive", [False, True])
@pytest.mark.parametrize("kind", ["f32", "f64"])
def test_per_op_api_on_gpu_matches_reference(shim_b200, adaptive, kind):
    """symmetric_pad / kernelize / build_mappings / compute_histogram (GPU) and
    mclahe::mclahe through the unmodified reference caller: every per-tile
    array bit-identical to the reference, output within 1e-5."""
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("reference library not built")
    rng = np.random.default_rng(21 + adaptive)
    shape, kernel = (19, 23, 12), (6, 8, 5)
    x = rng.poisson(4.0, shape) / 9.0
    if kind == "f64":
        x = x + rng.normal(0, 1e-3, shape)  # not float32-representable: the f64 path
    x[:4] = 0.25  # constant strips: degenerate tiles in adaptive mode
    a = O.tile_stats(x, kernel, 64, 0.05, adaptive, "b200")
    b = O.tile_stats(x, kernel, 64, 0.05, adaptive, "ref")
    for k in ("lo", "hi", "counts", "clipped", "lut", "degenerate"):
        assert np.array_equal(a[k], b[k]), k
    w = O.ref_tile_stats_window(x, kernel, 64, 0.05, adaptive, 1, 2, threads=3, impl="b200")
    for k in ("lo", "hi", "counts", "clipped", "lut", "degenerate"):
        assert np.array_equal(w[k], O.ref_tile_stats_window(x, kernel, 64, 0.05, adaptive, 1, 2,
                                                            threads=3)[k]), k
    got = O.mclahe(x, kernel, 64, 0.05, adaptive, "b200")
    want = O.mclahe(x, kernel, 64, 0.05, adaptive, "ref")
    assert np.max(np.abs(got - want)) <= 1e-5


@pytest.mark.gpu
def test_filters_metrics_npy_through_unmodified_caller(shim_b200, tmp_path):
    from oracle import oracle as O
    if not O.have_ref():
        pytest.skip("reference library not built")
    rng = np.random.default_rng(5)
    x = rng.random((14, 17, 9))
    g = O.gaussian_filter_ref(x, (1.0, 0.0, 1.5), 4.0, impl="b200")
    assert np.array_equal(g, O.gaussian_filter_ref(x, (1.0, 0.0, 1.5), 4.0))
    m = O.median_filter_ref(x, (3, 2, 1), impl="b200")
    assert np.array_equal(m, O.median_filter_ref(x, (3, 2, 1)))
    ma, mb = O.metrics_ref(g, x, 64, 1.0, impl="b200"), O.metrics_ref(g, x, 64, 1.0)
    assert ma["entropy_bits"] == mb["entropy_bits"]
    for k in ("mse", "psnr_db", "std"):
        assert abs(ma[k] - mb[k]) <= 1e-12 * max(1.0, abs(mb[k])), k
