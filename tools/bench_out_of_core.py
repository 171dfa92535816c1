"""End-to-end time of the out-of-core one-shot call (mclahe_gpu_run_out_of_core)
against the in-core call on the BASELINE volumes, pinned host buffers, results
compared bit for bit.  One JSON line per (config, device-memory cap).

    python tools/bench_out_of_core.py [--configs 4d,l4d,5d] [--steps 5]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1906_11355_b200 as M
from paper_1906_11355_b200 import _native as Nat
from paper_1906_11355_b200 import datasets


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="4d,l4d,5d")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--fracs", default="0.5,0.25")
    args = ap.parse_args()
    L = Nat.lib()
    for name in args.configs.split(","):
        cfg = datasets.CONFIGS[name]
        x = datasets.make(name, seed=0)
        host_in = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
        host_in.copy_(x)
        del x
        host_ref = torch.empty_like(host_in).pin_memory()
        host_out = torch.empty_like(host_in).pin_memory()
        params = Nat.make_params(cfg["shape"], cfg["kernel"], cfg["n_bins"], cfg["clip_limit"],
                                 cfg["adaptive"], Nat.F32)
        ws = int(M.Plan(cfg["shape"], cfg["kernel"], cfg["n_bins"], cfg["clip_limit"],
                        cfg["adaptive"]).info.workspace_bytes)
        nbytes = host_in.numel() * 4

        def timed(fn):
            fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                fn()
            torch.cuda.synchronize()
            return (time.perf_counter() - t0) / args.steps

        t_in = timed(lambda: Nat.check(L.mclahe_gpu_run(C.byref(params), host_in.data_ptr(),
                                                       host_ref.data_ptr(), None)))
        print(json.dumps({"config": name, "mode": "in core", "device_bytes": 2 * nbytes + ws,
                          "ms": t_in * 1e3, "gvox_s": host_in.numel() / t_in / 1e9}), flush=True)
        for frac in [float(f) for f in args.fracs.split(",")]:
            cap = ws + int(frac * 2 * nbytes)
            host_out.zero_()
            try:
                t = timed(lambda: Nat.check(L.mclahe_gpu_run_out_of_core(
                    C.byref(params), host_in.data_ptr(), host_out.data_ptr(), cap, None)))
            except MemoryError as e:
                print(json.dumps({"config": name, "mode": "out of core", "cap_bytes": cap,
                                  "error": str(e)}), flush=True)
                continue
            same = bool(torch.equal(host_out, host_ref))
            print(json.dumps({"config": name, "mode": "out of core", "cap_bytes": cap,
                              "cap_frac_of_in_core": frac, "ms": t * 1e3,
                              "gvox_s": host_in.numel() / t / 1e9, "vs_in_core": t / t_in,
                              "bit_identical": same,
                              "host_passes": 1 if cfg["adaptive"] else 2}), flush=True)
            assert same


if __name__ == "__main__":
    main()
