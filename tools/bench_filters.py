"""Device throughput of the steps either side of the path
on the 4D bench volume widened to float64 (the reference's type), against the
compiled reference on a sample (one thread, as its filters' default).

    python tools/bench_filters.py [--reps 5]
Prints one JSON line per operation."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import numpy as np
    import torch
    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import datasets
    from oracle import oracle as O
    x32 = datasets.make("4d", seed=0, device="cuda")
    x = x32.to(torch.float64)
    n = x.numel()
    sample = x[:4].cpu().numpy()  # 4 of 256 dim-0 rows for the CPU reference
    ops = {
        "gaussian_filter sigma=(1,1,1,1)": (
            lambda t: M.gaussian_filter(t, M.GaussianSpec((1.0, 1.0, 1.0, 1.0))),
            lambda s: O.gaussian_filter_ref(s, (1.0, 1.0, 1.0, 1.0)), 4 * 16),
        "median_filter window=(3,3,3,1)": (
            lambda t: M.median_filter(t, M.MedianSpec((3, 3, 3, 1))),
            lambda s: O.median_filter_ref(s, (3, 3, 3, 1)), 16),
        "compute_metrics n_bins=256": (
            lambda t: M.compute_metrics(t, t, 256),
            lambda s: O.metrics_ref(s, s, 256), 16 + 8 * 3),
    }
    for name, (dev, ref, bytes_per_voxel) in ops.items():
        dev(x)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.reps):
            dev(x)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / a.reps * 1e3
        c0 = time.perf_counter()
        ref(sample)
        cpu_s = time.perf_counter() - c0
        print(json.dumps({"op": name, "voxels": n, "dtype": "f64", "ms": ms,
                          "voxels_per_s": n / (ms * 1e-3),
                          "algo_gbs": n * bytes_per_voxel / (ms * 1e-3) / 1e9,
                          "cpu_reference_voxels_per_s": sample.size / cpu_s,
                          "cpu_reference": "compiled reference, 1 thread, 4 dim-0 rows"}),
              flush=True)


if __name__ == "__main__":
    main()
