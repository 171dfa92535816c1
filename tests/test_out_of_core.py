"""Out-of-core one-shot call (mclahe_gpu_run_out_of_core, SURVEY.md 8(f) 1;
/root/reference/PAPER.md:216 names larger-than-memory volumes as future work):
the volume streams through a ring of chunk slots under a device-memory cap
and must equal the in-core call bit for bit."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    # name: (dataset, shape, kernel, n_bins, clip, adaptive)
    "4d-adaptive": ("4d", (256, 64, 32, 32), (8, 8, 4, 4), 256, 0.02, True),
    "l4d-global": ("l4d", (256, 64, 32, 32), (8, 8, 4, 8), 512, 0.01, False),
    "3d-global": ("3d", (512, 64, 64), (16, 8, 8), 256, 0.02, False),
    "5d-adaptive": ("5d", (128, 32, 16, 16, 16), (4, 4, 2, 4, 4), 128, 0.03, True),
    "4d-ragged": ("4d", (203, 40, 32, 32), (16, 8, 4, 4), 64, 0.05, True),
}


@pytest.fixture(scope="module")
def M():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1906_11355_b200 as m
    return m


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("frac", [0.5, 0.2])
def test_out_of_core_matches_in_core(M, name, frac):
    from paper_1906_11355_b200 import datasets
    ds, shape, kernel, nb, clip, ad = CASES[name]
    x = datasets.make(ds, seed=11, shape=shape).numpy()
    want = M.enhance(x, kernel, nb, clip, ad)
    # in core the call holds the volume, its result and the workspace
    ws = int(M.Plan(x.shape, kernel, nb, clip, ad).info.workspace_bytes)
    cap = ws + int(frac * 2 * x.nbytes)
    try:
        got = M.enhance(x, kernel, nb, clip, ad, max_device_bytes=cap)
    except MemoryError as e:  # a ring of ~2.5 cells of rows may not fit the smallest caps
        assert "does not fit" in str(e), e
        assert frac < 0.5, "half the in-core footprint must be enough for these shapes"
        pytest.skip(f"cap {cap} below the minimal ring: {e}")
    assert np.array_equal(want, got)


def test_out_of_core_reports_too_small_budget(M):
    from paper_1906_11355_b200 import datasets
    ds, shape, kernel, nb, clip, ad = CASES["4d-adaptive"]
    x = datasets.make(ds, seed=3, shape=shape).numpy()
    with pytest.raises(MemoryError, match="does not fit"):
        M.enhance(x, kernel, nb, clip, ad, max_device_bytes=1 << 16)
    with pytest.raises(MemoryError, match="float64"):
        M.enhance(x.astype(np.float64), kernel, nb, clip, ad, max_device_bytes=x.nbytes)  # < 2 x 8 B / voxel


@pytest.mark.parametrize("ad", [False, True])
def test_out_of_core_non_finite(M, ad):
    """Global mode never writes the caller's buffer (both passes' flag is read
    before any blend); adaptive mode scrubs it (early chunks were copied back)."""
    from paper_1906_11355_b200 import _native as N
    from paper_1906_11355_b200 import datasets
    ds, shape, kernel, nb, clip, _ = CASES["4d-adaptive"]
    x = datasets.make(ds, seed=5, shape=shape).numpy().copy()
    x[-1, 5, 4, 3] = np.inf
    params = N.make_params(x.shape, kernel, nb, clip, ad, 0)
    out = np.full_like(x, 7.0)
    ws = int(M.Plan(x.shape, kernel, nb, clip, ad).info.workspace_bytes)
    rc = N.lib().mclahe_gpu_run_out_of_core(C.byref(params), x.ctypes.data, out.ctypes.data,
                                            ws + x.nbytes, None)
    assert rc == 1 and b"non-finite" in N.lib().mclahe_last_error()
    assert np.isnan(out).all() if ad else np.all(out == 7.0)


def test_out_of_core_env_cap(M, monkeypatch):
    """MCLAHE_MAX_DEVICE_BYTES sends the plain one-shot call through the ring."""
    from paper_1906_11355_b200 import datasets
    ds, shape, kernel, nb, clip, ad = CASES["l4d-global"]
    x = datasets.make(ds, seed=9, shape=shape).numpy()
    want = M.enhance(x, kernel, nb, clip, ad)
    ws = int(M.Plan(x.shape, kernel, nb, clip, ad).info.workspace_bytes)
    monkeypatch.setenv("MCLAHE_MAX_DEVICE_BYTES", str(ws + x.nbytes))
    got = M.enhance(x, kernel, nb, clip, ad)
    assert np.array_equal(want, got)
