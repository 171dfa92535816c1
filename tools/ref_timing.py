"""Times the compiled reference (oracle/_ref) on full BASELINE configs on the
host cores (test/measurement infrastructure; not part of the product)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1906_11355_b200 import datasets  # noqa: E402

for name in sys.argv[1:]:
    cfg = datasets.CONFIGS[name]
    x = datasets.make(name, seed=0, device="cuda" if torch.cuda.is_available() else "cpu").cpu().numpy()
    x64 = x.astype(np.float64)
    t = [0.0, 0.0, 0.0]
    t0 = time.perf_counter()
    O.mclahe(x64, cfg["kernel"], cfg["n_bins"], cfg["clip_limit"], cfg["adaptive"], "ref",
             threads=0, timings=t)
    dt = time.perf_counter() - t0
    print(f"{name}: {x.size} voxels, {dt:.2f} s, {x.size / dt / 1e6:.2f} Mvox/s, phases {t}", flush=True)
    t0 = time.perf_counter()
    O.tile_stats(x64, cfg["kernel"], cfg["n_bins"], cfg["clip_limit"], cfg["adaptive"], "ref")
    print(f"{name}: ref tile_stats {time.perf_counter() - t0:.2f} s", flush=True)
