"""Multi-slab / multi-device runs through the C ABI (mclahe_gpu_run_multi,
SURVEY.md 8(e)).  The exchange kernels read peer snapshots directly (P2P) or
through cudaMemcpyPeerAsync staging; on one GPU the slabs are logical (all on
device 0) and take the identical code path.  The reference promises
bit-identical results for any worker count (pipeline.hpp:10-11,
parallel.hpp:19-22): every slab count must reproduce the one-device output
bit for bit."""
import numpy as np
import pytest

from paper_1906_11355_b200 import slabs as SL

CASES = {
    "4d": dict(shape=(64, 64, 32, 32), kernel=(8, 8, 4, 4), n_bins=256, clip_limit=0.02, adaptive=True),
    "l4d": dict(shape=(64, 64, 32, 32), kernel=(8, 8, 4, 8), n_bins=512, clip_limit=0.01, adaptive=False),
    "5d": dict(shape=(32, 32, 16, 16, 16), kernel=(4, 4, 2, 4, 4), n_bins=128, clip_limit=0.03, adaptive=True),
    "3d": dict(shape=(72, 64, 40), kernel=(9, 8, 8), n_bins=256, clip_limit=0.02, adaptive=False),
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_multi_cuts_match_slab_rule(name, n):
    import paper_1906_11355_b200 as M
    c = CASES[name]
    got = M.multi_cuts(c["shape"], c["kernel"], n, c["n_bins"], c["clip_limit"], c["adaptive"])
    want = SL.slab_cuts(c["shape"][0], c["kernel"][0], n)
    assert got == [a for a, _ in want] + [want[-1][1]]


def test_multi_cuts_too_many_slabs():
    import paper_1906_11355_b200 as M
    with pytest.raises(M.ValidationError, match="interpolation cells"):
        M.multi_cuts((16, 8), (8, 4), 3)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("n", [2, 3, 8])
def test_logical_slabs_bit_identical(name, n):
    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import datasets
    c = CASES[name]
    x = datasets.make(name, seed=6, shape=c["shape"]).numpy()
    args = (c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"])
    one = M.enhance(x, *args)
    multi = M.mclahe_multi(x, *args, devices=[0] * n)
    assert np.array_equal(one, multi), name


@pytest.mark.gpu
def test_multi_device_buffers_and_nonfinite():
    import torch

    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import datasets
    c = CASES["4d"]
    args = (c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"])
    x = datasets.make("4d", seed=7, shape=c["shape"]).cuda()
    one = M.enhance(x, *args)
    cuts = M.multi_cuts(c["shape"], c["kernel"], 4, *args[1:])
    slabs = [x[a:b].contiguous() for a, b in zip(cuts[:-1], cuts[1:])]
    outs = M.mclahe_multi(slabs, *args, devices=[0, 0, 0, 0])
    assert torch.equal(torch.cat(outs, 0), one)
    xn = x.cpu().numpy().copy()
    xn[-1, 2, 3, 4] = np.nan  # non-finite in the last slab: every slab reports it
    with pytest.raises(M.ValidationError, match="non-finite"):
        M.mclahe_multi(xn, *args, devices=[0, 0, 0])
