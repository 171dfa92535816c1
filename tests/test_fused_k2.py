"""The fused single-read K2 (csrc/k_fused.cu: tile ranges and counts from one
HBM read, cross-CTA tile-group dependencies) is opt-in (MCLAHE_FUSED_K2=1,
read once per process), so these tests run it in subprocesses:

* the GPU parity suite's golden / random / scaled-config / non-finite /
  determinism cases with the fused kernel switched on (bit-exact stats and
  output <= 1e-5 against the oracle, as for the two-pass path);
* the 4D BASELINE volume at full size: every tile's lo/hi/counts/clipped/LUT
  and every output voxel bit-identical to the two-pass path, over repeated
  runs (a scheduling race or lost arrival would show up as a difference or a
  hang, bounded by the subprocess timeout).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env(on):
    env = dict(os.environ)
    env["MCLAHE_FUSED_K2"] = "1" if on else "0"
    return env


def test_parity_suite_with_fused_k2():
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-m", "gpu", "-x", "-q",
                        "-k", "golden or random or scaled or nonfinite or determinism or sparse or dictionary"],
                       cwd=ROOT, env=_env(True), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


_RUN = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1906_11355_b200 as M
from paper_1906_11355_b200 import datasets
c = datasets.CONFIGS["4d"]
x = datasets.make("4d", seed=0, device="cuda")
plan = M.Plan(x.shape, c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"])
ws = plan.new_workspace()
out = torch.empty_like(x)
for _ in range({iters}):
    plan.enqueue(x, out, ws)
plan.check(ws)
st = plan.tile_stats(x)
assert plan.flags["fused_k2"] == {on}
np.savez({path!r}, out=out.cpu().numpy(), **{{k: np.asarray(v) for k, v in st.items()}})
"""


def _run(tmp_path, on, iters):
    path = str(tmp_path / f"r{int(on)}.npz")
    code = _RUN.format(root=ROOT, iters=iters, on=on, path=path)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=_env(on), capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    return np.load(path)


def test_full_size_4d_bit_identical_to_two_pass(tmp_path):
    a = _run(tmp_path, True, 12)
    b = _run(tmp_path, False, 1)
    for k in ("lo", "hi", "counts", "clipped", "lut", "degenerate", "out"):
        assert np.array_equal(a[k], b[k]), k


def test_parity_with_match_any_histograms():
    """The __match_any_sync warp-aggregated K2b (MCLAHE_K2_MATCH=1, an A/B kept
    for the record: 17x slower) counts exactly like the run-merged adds."""
    env = dict(os.environ)
    env["MCLAHE_K2_MATCH"] = "1"
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-m", "gpu", "-x", "-q",
                        "-k", "golden or random or scaled"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_parity_with_carried_runs_in_adaptive_mode():
    """The carried-run K2b (default in global mode) forced on in adaptive mode
    too (MCLAHE_K2_CARRY=1) counts exactly like the per-row merge."""
    env = dict(os.environ)
    env["MCLAHE_K2_CARRY"] = "1"
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-m", "gpu", "-x", "-q",
                        "-k", "golden or random or scaled or adversarial"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
