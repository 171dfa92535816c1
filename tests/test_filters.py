"""The steps either side of the MCLAHE path: the
prefilters gaussian_filter / median_filter (src/filters.cpp) and the contrast
metrics (src/metrics.cpp).

CPU tests pin the numpy restatements (oracle/oracle.py) to the reference
compiled from its sources; GPU tests hold the device kernels to the reference:
bit-exact filters, exact entropy counts, mse / std within 1e-12 relative
(parallel sums)."""
import numpy as np
import pytest

from oracle import oracle as O

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="reference library not built")

CASES = [((37,), (2.0,), (5,)), ((20, 31), (1.5, 0.0), (3, 4)), ((9, 14, 11), (0.7, 2.2, 1.0), (3, 3, 2)),
         ((6, 5, 8, 7), (1.0, 0.0, 0.5, 3.0), (2, 3, 1, 3)), ((3, 200), (0.0, 30.0), (1, 9))]


def _data(shape, seed):
    rng = np.random.default_rng(seed)
    x = rng.random(shape)
    x.flat[:: 7] = np.round(x.flat[:: 7] * 4) / 4  # ties for the median
    return x


@needs_ref
@pytest.mark.parametrize("i", range(len(CASES)))
def test_restatements_match_reference(i):
    shape, sigmas, window = CASES[i]
    x = _data(shape, i)
    assert np.array_equal(O.gaussian_filter_np(x, sigmas, 4.0), O.gaussian_filter_ref(x, sigmas, 4.0))
    assert np.array_equal(O.median_filter_np(x, window), O.median_filter_ref(x, window))
    y = _data(shape, 50 + i)
    a, b = O.metrics_np(x, y, 64, 1.0), O.metrics_ref(x, y, 64, 1.0)
    for k in ("mse", "psnr_db", "std", "entropy_bits"):
        assert abs(a[k] - b[k]) <= 1e-12 * max(1.0, abs(b[k])), k


@needs_ref
def test_reference_validation_messages():
    x = np.zeros((4, 4))
    with pytest.raises(O.OracleValidationError, match="truncate must be positive"):
        O.gaussian_filter_ref(x, (1.0, 1.0), 0.0)
    with pytest.raises(O.OracleValidationError, match="sigma must be non-negative"):
        O.gaussian_filter_ref(x, (1.0, -1.0), 4.0)
    with pytest.raises(O.OracleValidationError, match="window extents must be positive"):
        O.median_filter_ref(x, (0, 1))
    with pytest.raises(O.OracleValidationError, match="psnr peak must be positive"):
        O.metrics_ref(x, x, 8, 0.0)
    with pytest.raises(O.OracleValidationError, match="entropy needs at least 2 bins"):
        O.metrics_ref(x, x, 1, 1.0)


def test_api_validation_before_the_device():
    import paper_1906_11355_b200 as M
    with pytest.raises(M.ValidationError, match="sigma count does not match image rank"):
        M.gaussian_filter(np.zeros((3, 3)), M.GaussianSpec((1.0,)))
    with pytest.raises(M.ValidationError, match="window rank does not match image rank"):
        M.median_filter(np.zeros((3, 3)), M.MedianSpec((3, 3, 3)))
    with pytest.raises(M.ValidationError, match="mse operands differ in shape"):
        M.compute_metrics(np.zeros((3, 3)), np.zeros((3, 4)))


@pytest.fixture(scope="module")
def M():
    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import _native
    _native.lib()
    return M


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("i", range(len(CASES)))
def test_gpu_filters_bit_exact(M, i):
    shape, sigmas, window = CASES[i]
    x = _data(shape, i)
    g = M.gaussian_filter(x, M.GaussianSpec(sigmas, 4.0))
    assert np.array_equal(g, O.gaussian_filter_ref(x, sigmas, 4.0))
    m = M.median_filter(x, M.MedianSpec(window))
    assert np.array_equal(m, O.median_filter_ref(x, window))


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("i", range(len(CASES)))
def test_gpu_metrics(M, i):
    shape = CASES[i][0]
    x, y = _data(shape, i), _data(shape, 90 + i)
    for nb in (2, 64, 256):
        got, want = M.compute_metrics(x, y, nb, 1.0), O.metrics_ref(x, y, nb, 1.0)
        assert got.entropy_bits == want["entropy_bits"], nb  # exact counts, bin-order sum
        for k in ("mse", "psnr_db", "std"):
            assert abs(getattr(got, k) - want[k]) <= 1e-12 * max(1.0, abs(want[k])), (k, nb)
    same = M.compute_metrics(x, x)
    assert same.mse == 0.0 and same.psnr_db == float("inf")
    const = M.compute_metrics(np.full(shape, 0.3))
    ref = O.metrics_ref(np.full(shape, 0.3), np.full(shape, 0.3))
    assert const.entropy_bits == 0.0 == ref["entropy_bits"]  # constant image: 0 by rule
    assert abs(const.std - ref["std"]) <= 1e-12  # (0 up to the sums' rounding)


@pytest.mark.gpu
def test_gpu_device_tensors_and_pipeline(M):
    import torch
    x = _data((24, 30, 16), 7)
    xt = torch.from_numpy(x).cuda()
    g_dev = M.gaussian_filter(xt, M.GaussianSpec((1.0, 1.0, 0.0)))
    assert g_dev.is_cuda and np.array_equal(g_dev.cpu().numpy(),
                                            M.gaussian_filter(x, M.GaussianSpec((1.0, 1.0, 0.0))))
    m_dev = M.median_filter(xt, M.MedianSpec((3, 3, 1)))
    assert np.array_equal(m_dev.cpu().numpy(), M.median_filter(x, M.MedianSpec((3, 3, 1))))
    # the paper's pipeline: smooth, enhance, measure -- all on the device
    out = M.mclahe(M.McLaheRequest(g_dev, M.KernelSpec((8, 10, 8)),
                                   M.EnhanceParams(0.02, 64, M.RangeMode.Adaptive)))
    want = O.mclahe(g_dev.cpu().numpy(), (8, 10, 8), 64, 0.02, True, "c")
    assert np.max(np.abs(out.cpu().numpy() - want)) <= 1e-5
    rep = M.compute_metrics(out, g_dev)
    assert abs(rep.mse - O.metrics_np(out.cpu().numpy(), g_dev.cpu().numpy())["mse"]) <= 1e-12


@pytest.mark.gpu
def test_gpu_filter_errors(M):
    with pytest.raises(M.ValidationError, match="non-finite"):
        M.gaussian_filter(np.array([[1.0, np.nan]]), M.GaussianSpec((1.0, 1.0)))
    with pytest.raises(M.ValidationError, match="non-finite"):
        M.median_filter(np.array([[1.0, np.inf]]), M.MedianSpec((1, 2)))
    with pytest.raises(M.ValidationError, match="truncate must be positive"):
        M.gaussian_filter(np.zeros((3, 3)), M.GaussianSpec((1.0, 1.0), 0.0))
    with pytest.raises(M.ValidationError, match="psnr peak must be positive"):
        M.compute_metrics(np.zeros(4), np.zeros(4), 8, 0.0)
    with pytest.raises(M.ValidationError, match="entropy needs at least 2 bins"):
        M.compute_metrics(np.zeros(4), None, 1)
