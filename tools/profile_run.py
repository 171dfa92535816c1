"""Runs the MCLAHE passes on one BASELINE config a few times (for ncu / nsight).

    python tools/profile_run.py --config 4d --iters 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="4d")
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--f64", action="store_true", help="float64 volume (the f64 kernels)")
    ap.add_argument("--time", action="store_true",
                    help="time the blend pass alone (CUDA events, 20 launches) -- for A/B builds")
    a = ap.parse_args()
    import torch
    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import datasets
    c = datasets.CONFIGS[a.config]
    x = datasets.make(a.config, seed=0, device="cuda")
    if a.f64:
        x = x.double()
    plan = M.Plan(x.shape, c["kernel"], c["n_bins"], c["clip_limit"], c["adaptive"], 1 if a.f64 else 0)
    ws = plan.new_workspace()
    out = torch.empty_like(x)
    for _ in range(a.iters):
        plan.enqueue(x, out, ws)
    plan.check(ws)
    torch.cuda.synchronize()
    if a.time:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
        for k in range(20):
            ev[k].record()
            plan.interpolate(x, out, ws)
        ev[20].record()
        torch.cuda.synchronize()
        ms = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(20))
        print(f"interp ms median {ms[10]:.4f} min {ms[0]:.4f}")
    print("ok", a.config, float(out.mean()))


if __name__ == "__main__":
    main()
