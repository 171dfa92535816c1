"""Generates tests/golden/*.npz from the REFERENCE library itself.

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
The reference is compiled from its own sources by oracle/Makefile into
oracle/_ref/libmclahe_ref.so and driven through its public API
(oracle/ref_shim.cpp).  Each fixture holds the float32-valued input, the
request, the per-tile intermediates of build_mappings and the mclahe() output.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

CASES = [
    # name, shape, kernel, n_bins, clip, adaptive, kind
    ("spec_2d_16x16", (16, 16), (4, 4), 8, 0.5, False, "uniform"),
    ("ramp_1d", (64,), (64,), 64, 1.0, False, "ramp"),
    ("ragged_2d", (37, 29), (8, 5), 32, 0.05, True, "uniform"),
    ("quantised_3d", (24, 20, 16), (8, 4, 4), 16, 0.1, False, "quantised"),
    ("adaptive_3d_degenerate", (16, 16, 16), (4, 4, 8), 16, 0.02, True, "sparse"),
    ("small_4d", (16, 16, 8, 8), (8, 8, 4, 4), 32, 0.02, True, "quantised"),
    ("small_5d", (8, 8, 8, 4, 4), (4, 4, 4, 2, 2), 16, 0.03, True, "signed"),
    ("tiny_odd_4d", (7, 9, 5, 6), (3, 4, 5, 2), 8, 0.3, False, "uniform"),
]


def make_input(shape, kind, rng):
    if kind == "uniform":
        return rng.random(shape).astype(np.float32)
    if kind == "ramp":
        return np.linspace(0.0, 1.0, int(np.prod(shape))).reshape(shape).astype(np.float32)
    if kind == "quantised":
        return (rng.poisson(3.0, shape) / 12.0).astype(np.float32)
    if kind == "sparse":
        x = np.zeros(shape, np.float32)
        m = rng.random(shape) < 0.05
        x[m] = rng.integers(1, 5, m.sum()) / 4.0
        return x
    if kind == "signed":
        return (rng.normal(0, 1, shape) * 0.3).astype(np.float32)
    raise ValueError(kind)


def main():
    rng = np.random.default_rng(20190626)
    for name, shape, kernel, nb, clip, ad, kind in CASES:
        x = make_input(shape, kind, rng)
        st = O.tile_stats(x, kernel, nb, clip, ad, impl="ref")
        out = O.mclahe(x, kernel, nb, clip, ad, impl="ref", threads=1)
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), x=x, kernel=np.array(kernel), n_bins=nb,
            clip_limit=clip, adaptive=ad, lo=st["lo"], hi=st["hi"], counts=st["counts"],
            clipped=st["clipped"], lut=st["lut"], degenerate=st["degenerate"],
            grid=np.array(st["grid"]), out=out)
        print(name, x.shape, "tiles", len(st["lo"]))


if __name__ == "__main__":
    main()
