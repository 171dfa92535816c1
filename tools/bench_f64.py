"""float64 volumes (the reference's own element type) through the device
passes: per-pass CUDA-event times and voxels/s for each BASELINE config, data
= the config's generator widened to float64 plus a 1e-12 ramp so the values
are not float32-representable (the exact f64 kernels: tile-major K2,
cell-major blend).  One JSON line per config.

    python tools/bench_f64.py [--configs 3d 4d 5d] [--steps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["2d", "3d", "4d", "5d"])
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    import torch
    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import datasets
    for name in a.configs:
        c = datasets.CONFIGS[name]
        x = datasets.make(name, seed=0, device="cuda").double()
        x = (x + torch.arange(x.numel(), device="cuda", dtype=torch.float64).reshape(x.shape) * 1e-12
             / x.numel()).contiguous()
        plan = M.Plan(x.shape, c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"], 1)
        ws = plan.new_workspace()
        out = torch.empty_like(x)
        st = torch.cuda.current_stream()

        def step(ev=None):
            if ev: ev[0].record(st)
            plan.reset(ws)
            plan.range(x, ws)
            plan.make_params(ws)
            if ev: ev[1].record(st)
            plan.histograms(x, ws)
            if ev: ev[2].record(st)
            plan.mappings(ws)
            if ev: ev[3].record(st)
            plan.interpolate(x, out, ws)
            if ev: ev[4].record(st)

        for _ in range(2):
            step()
        plan.check(ws)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(a.steps)]
        torch.cuda.synchronize()
        for e in evs:
            step(e)
        torch.cuda.synchronize()
        names = ["range", "hist", "map", "interp"]
        passes = {n: sorted(e[i].elapsed_time(e[i + 1]) for e in evs)[a.steps // 2]
                  for i, n in enumerate(names)}
        tot = sorted(e[0].elapsed_time(e[4]) for e in evs)[a.steps // 2]
        print(json.dumps({"config": name, "dtype": "f64", "voxels": x.numel(), "ms_per_step": tot,
                          "gvox_s": x.numel() / tot / 1e6, "passes_ms": passes,
                          "blend_gbs": 16 * x.numel() / passes["interp"] / 1e6}), flush=True)


if __name__ == "__main__":
    main()
