"""CPU-side checks of the product library (no GPU needed): it loads, exports
every entry point include/mclahe_gpu.h declares, validates requests with the
reference's messages, and plans slabs with the geometry the oracle uses."""
import re
import os

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def N():
    from paper_1906_11355_b200 import _native
    _native.lib()
    return _native


def test_exports_every_declared_symbol(N):
    hdr = open(os.path.join(ROOT, "include", "mclahe_gpu.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int32_t|int64_t|const char\*|void\*|void)\s+(mclahe_\w+)\(",
                              hdr, re.M))
    assert len(declared) >= 15
    L = N.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(N.SIGNATURES), declared ^ set(N.SIGNATURES)


def _plan(shape, kernel, nb=64, clip=0.1, ad=False, rows=None):
    from paper_1906_11355_b200 import Plan
    rows = rows or (0, shape[0])
    return Plan(shape, kernel, nb, clip, ad, 0, rows[0], rows[1])


@pytest.mark.parametrize("shape,kernel", [((1024, 1024), (64, 64)), ((37, 29), (8, 5)),
                                          ((9,), (4,)), ((7, 9, 5, 6), (3, 4, 5, 2)),
                                          ((256, 256, 128, 32), (32, 32, 16, 4))])
def test_geometry_matches_oracle(N, shape, kernel):
    p = _plan(shape, kernel)
    before, after, grid = O.geometry(shape, kernel)
    D = len(shape)
    assert list(p.info.before[:D]) == list(before)
    assert list(p.info.after[:D]) == list(after)
    assert list(p.info.grid[:D]) == list(grid)
    assert p.info.tiles == int(np.prod(grid))
    assert p.window_tiles == p.info.tiles  # whole-volume plan holds every tile


def test_validation_messages(N):
    from paper_1906_11355_b200 import Plan, ValidationError
    with pytest.raises(ValidationError, match=r"kernel size must be in \[1, extent\] along dimension 1"):
        Plan((8, 8), (4, 9))
    with pytest.raises(ValidationError, match=r"clip_limit must be in \(0, 1\]"):
        Plan((8, 8), (4, 4), 16, 1.5)
    with pytest.raises(ValidationError, match="n_bins must be at least 2"):
        Plan((8, 8), (4, 4), 1, 0.5)
    with pytest.raises(ValidationError, match="does not match image rank"):
        Plan((8, 8), (4,))
    with pytest.raises(ValidationError, match="rank must be in"):
        Plan((2,) * 9, (1,) * 9)


def test_host_api_validates_before_touching_the_gpu(N):
    import paper_1906_11355_b200 as M
    with pytest.raises(M.ValidationError, match="clip_limit"):
        M.enhance(np.zeros((8, 8), np.float32), (4, 4), 16, 0.0)


@pytest.mark.parametrize("name", ["2d", "3d", "4d", "l4d", "5d"])
def test_baseline_configs_take_the_pencil_kernels(N, name):
    from paper_1906_11355_b200 import datasets
    c = datasets.CONFIGS[name]
    p = _plan(c["shape"], c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"])
    assert p.info.fast_hist == 1 and p.info.fast_interp == 1
    assert p.info.hist_units > 0 and p.info.interp_units > 0


def test_slab_windows_cover_their_cells(N):
    from paper_1906_11355_b200 import slabs as S
    shape, kernel = (256, 256, 128, 32), (32, 32, 16, 4)
    for world in (2, 4, 8):
        cuts = S.slab_cuts(shape[0], kernel[0], world)
        assert cuts[0][0] == 0 and cuts[-1][1] == shape[0]
        assert all(a < b for a, b in cuts)
        assert all(cuts[i][1] == cuts[i + 1][0] for i in range(world - 1))
        assert len({b - a for a, b in cuts}) == 1  # cell-aligned, perfectly balanced
        for a, b in cuts:
            p = _plan(shape, kernel, 256, 0.02, True, (a, b))
            i = p.info
            # every tile row whose support meets the slab is counted, every
            # tile row a voxel of the slab blends is held
            assert i.tile_row_begin <= i.count_row_begin and i.count_row_end <= i.tile_row_end
            assert i.tile_row_begin <= i.need_row_begin and i.need_row_end <= i.tile_row_end
            assert i.need_row_begin == a // 32 and i.need_row_end == b // 32 + 1


def test_slab_cuts_ragged(N):
    from paper_1906_11355_b200 import slabs as S
    for extent, k in [(37, 8), (100, 7), (64, 64), (9, 2)]:
        cells = S.cell_ranges(extent, k)
        assert cells[0][0] == 0 and cells[-1][1] == extent
        for world in range(1, len(cells) + 1):
            cuts = S.slab_cuts(extent, k, world)
            assert len(cuts) == world and cuts[-1][1] == extent
            starts = {c[0] for c in cells}
            assert all(a in starts for a, _ in cuts)
        with pytest.raises(Exception):
            S.slab_cuts(extent, k, len(cells) + 1)


def test_framewise_validation_messages():
    import paper_1906_11355_b200 as M
    prm = M.EnhanceParams(0.1, 16)
    with pytest.raises(M.ValidationError, match="framewise mode needs rank >= 2"):
        M.mclahe_framewise(np.zeros(5, np.float32), 0, M.KernelSpec(()), prm)
    with pytest.raises(M.ValidationError, match="frame axis 3 out of range for rank 3"):
        M.mclahe_framewise(np.zeros((4, 5, 6), np.float32), 3, M.KernelSpec((2, 2)), prm)
    with pytest.raises(M.ValidationError, match="framewise kernel rank must be image rank - 1"):
        M.mclahe_framewise(np.zeros((4, 5, 6), np.float32), 0, M.KernelSpec((2, 2, 2)), prm)
