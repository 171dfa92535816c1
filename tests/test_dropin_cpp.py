"""The C++ drop-in (include/mclahe_b200.hpp + libmclahe_cpp.so): a program
written against the reference API compiles, links and runs unchanged."""
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
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
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
