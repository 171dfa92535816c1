#!/usr/bin/env python
"""MCLAHE throughput on B200 -- the bench contract (one JSON line on rank 0).

Workload: BASELINE.json configs[2], the 4D photoemission-like volume
256x256x128x32 float32, kernel (32,32,16,4), 256 bins, clip 0.02, adaptive
range -- the config north_star names for slab scaling (``--config`` picks
another; the rest are parity cases).  A step = the full hot path (range,
binning parameters, per-tile histograms, clip/CDF/LUT, 2^D blend) over the
whole volume.  Inputs (1.07 GB) exceed the 126 MB L2, so no flush is needed.

* value    voxels/s, inputs resident in HBM, K steps timed with CUDA events
           (barrier + synchronize both sides, max over ranks).
* e2e      same metric through the C-ABI one-shot call (mclahe_gpu_run) with
           pinned HOST buffers: H2D input + passes + D2H output every step.
* roofline dominant kernel (the blend, K4): algorithmic bytes 8*N + 4*T*n per
           launch / its CUDA-event time, vs MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline  the reference library (oracle/_ref, compiled from the
           reference sources) on the whole volume (one run, ~12 s for 4D), all
           host cores; lscpu model / sockets / threads recorded.

``--impl reference`` times that reference CPU implementation alone, one full
volume per timed step.
N > 1 (torchrun): the volume is split into cell-aligned slabs along dim 0
(paper_1906_11355_b200/slabs.py): global range all-reduce / neighbour
exchange of shared tile rows over NCCL; scaling "strong" (fixed total work).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "mclahe_voxels_per_s"
UNIT = "voxel/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="4d", choices=["2d", "3d", "4d", "l4d", "5d"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager pass launches instead of one CUDA graph per step")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test the multi-rank path with ranks sharing GPUs")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled while the bench runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.samples, self.proc = [], None
        self.gpu = gpu_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[3:7])
                          if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_reference_sample(x_host_rows, cfg, threads=0):
    """Times the reference library (oracle/_ref) -- or, if it is absent, the C
    oracle port -- on host data; returns (voxels/s, kind, cores, secs)."""
    import numpy as np
    from oracle import oracle as O
    x64 = np.ascontiguousarray(x_host_rows, dtype=np.float64)
    impl, kind = ("ref", "reference") if O.have_ref() else ("c", "port")
    cores = (os.cpu_count() or 1) if impl == "ref" else 1
    t0 = time.perf_counter()
    O.mclahe(x64, cfg["kernel"], cfg["n_bins"], cfg["clip_limit"], cfg["adaptive"], impl,
             threads=threads if threads else cores)
    dt = time.perf_counter() - t0
    return x64.size / dt, kind, cores, dt


def host_cpu_info():
    """Host CPU model / sockets / threads (lscpu), for the CPU baseline."""
    info = {"threads": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "Model name":
                info["model"] = v
            elif k == "Socket(s)":
                info["sockets"] = int(v)
            elif k == "Core(s) per socket":
                info["cores_per_socket"] = int(v)
            elif k == "Thread(s) per core":
                info["threads_per_core"] = int(v)
    except Exception:
        pass
    return info


def sample_rows(cfg, budget_voxels):
    """Rows of dim 0 (a multiple of the dim-0 kernel) for a bounded CPU sample."""
    import numpy as np
    per_row = int(np.prod(cfg["shape"][1:]))
    b0 = cfg["kernel"][0]
    rows = max(b0, (budget_voxels // per_row) // b0 * b0)
    return min(rows, cfg["shape"][0])


def run_reference_arm(args, cfg):
    """The reference's own CPU implementation (oracle/_ref: the reference
    library compiled from its sources) on the FULL workload volume, all host
    threads.  Each timed step is one mclahe::mclahe call over the whole volume
    (~12 s for 4D on 16 threads); the warm-up steps run one dim-0 kernel row
    (page-in, thread start-up), so the default run stays within a few minutes."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    import torch
    from paper_1906_11355_b200 import datasets
    x = datasets.make(args.config, seed=0,
                      device="cuda" if torch.cuda.is_available() else "cpu").cpu().numpy()
    for _ in range(args.warmup):
        cpu_reference_sample(x[: cfg["kernel"][0]], cfg)
    times = []
    kind = cores = None
    for _ in range(args.steps):
        v, kind, cores, dt = cpu_reference_sample(x, cfg)
        times.append(dt)
    ms = 1e3 * statistics.median(times)
    value = x.size / (ms * 1e-3)
    sample = (f"the full {args.config} volume ({x.size} voxels) every timed step, float32 values "
              f"widened to float64; median of {args.steps} runs; warm-up steps on "
              f"{cfg['kernel'][0]} dim-0 rows")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args, cfg, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample, "host": host_cpu_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def small_volume(cfg):
    return 4 * _numel(cfg) <= 126e6


def workload_config(args, cfg, world):
    return {"workload": f"mclahe-{args.config}", "shape": list(cfg["shape"]),
            "kernel_size": list(cfg["kernel"]), "n_bins": cfg["n_bins"],
            "clip_limit": cfg["clip_limit"], "adaptive_hist_range": cfg["adaptive"],
            "parallelism": f"slab{world}" if world > 1 else "single",
            "l2": "L2 flushed (256 MB write) before every step, steps timed alone"
            if small_volume(cfg) else "inputs larger than L2 (no flush)"}


def _numel(cfg):
    n = 1
    for s in cfg["shape"]:
        n *= s
    return n


def main():
    args = parse()
    from paper_1906_11355_b200 import datasets
    cfg = datasets.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import slabs as S

    rank, world, local = dist_env()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    shape, kernel = tuple(cfg["shape"]), tuple(cfg["kernel"])
    nb, clip, ad = cfg["n_bins"], cfg["clip_limit"], cfg["adaptive"]
    N_total = _numel(cfg)

    # ---- input: seeded synthetic volume, generated on the device ----
    x_full = datasets.make(args.config, seed=0, device=dev)
    if world > 1:
        cuts = S.slab_cuts(shape[0], kernel[0], world)
        a, b = cuts[rank]
        x = x_full[a:b].contiguous()
        plan = M.Plan(shape, kernel, nb, clip, ad, 0, a, b)
        windows = S.all_windows(shape, kernel, nb, clip, ad, cuts)
    else:
        x = x_full
        plan = M.Plan(shape, kernel, nb, clip, ad)
        windows = None
    if world > 1:
        del x_full
    ws = plan.new_workspace(dev)
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    T, n = plan.window_tiles, nb

    def step(evs=None):
        if world > 1:
            S.run_rank(x, shape, kernel, nb, clip, ad, rank, world, out=out, plan=plan, ws=ws,
                       windows=windows)
            return
        if evs is None:
            # the whole step through the public call (mclahe_plan_enqueue): every
            # pass, the dictionary numbering on its side branch
            plan.enqueue(x, out, ws)
            return
        evs[0].record(stream)
        plan.reset(ws)
        plan.range(x, ws)
        plan.make_params(ws)
        if evs is not None:
            evs[1].record(stream)
        plan.histograms(x, ws)
        if evs is not None:
            evs[2].record(stream)
        plan.mappings(ws)
        if evs is not None:
            evs[3].record(stream)
        plan.interpolate(x, out, ws)
        if evs is not None:
            evs[4].record(stream)

    gpu_index = local
    if os.environ.get("CUDA_VISIBLE_DEVICES"):
        try:
            gpu_index = int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local])
        except ValueError:
            pass
    sampler = ClockSampler(gpu_index)
    with sampler:
        for _ in range(max(args.warmup, 3)):
            step()
        plan.check(ws)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
        # one process per GPU: the whole step (every pass, no host sync) is
        # captured once into a CUDA graph and replayed, so the timed region
        # holds device work only (small volumes are otherwise host-launch bound)
        graph = None
        if world == 1 and not args.no_graph:
            try:
                torch.cuda.synchronize()
                l_a = M.launch_count()
                step()
                per_step = M.launch_count() - l_a
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    step()
                for _ in range(max(args.warmup, 3)):
                    graph.replay()
                torch.cuda.synchronize()
                plan.check(ws)
            except Exception as exc:  # keep the eager loop if capture is refused
                print(f"[bench] CUDA graph capture failed ({exc}); timing eager steps",
                      file=sys.stderr)
                graph = None
        # volumes smaller than the 126 MB L2: write a 256 MB buffer before every
        # step and time the steps alone (events around each step)
        flush = small_volume(cfg)
        l2buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = M.launch_count()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)] if flush else None
        t0.record(stream)
        for k in range(args.steps):
            if flush:
                l2buf.zero_()
                step_ev[k][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step(evs[k] if world == 1 else None)
            if flush:
                step_ev[k][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
        launches = per_step * args.steps if graph is not None else M.launch_count() - l0
        if flush:
            ms_local = sum(a.elapsed_time(b) for a, b in step_ev) / args.steps
        else:
            ms_local = t0.elapsed_time(t1) / args.steps
        if graph is not None:  # per-pass breakdown: the same steps eagerly, events between passes
            for k in range(args.steps):
                step(evs[k])
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        plan.check(ws)
        ms_t = torch.tensor([ms_local], device=dev if args.dist_backend == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        ms = float(ms_t.item())

        # ---- e2e: host pinned buffers through the C ABI one-shot call ----
        e2e = None
        if world == 1:
            host_in = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
            host_in.copy_(x)
            host_out = torch.empty_like(host_in).pin_memory()
            req = M.McLaheRequest(host_in.numpy(), M.KernelSpec(kernel),
                                  M.EnhanceParams(clip, nb, M.RangeMode(int(ad))))
            from paper_1906_11355_b200 import _native as Nat
            import ctypes as C
            params = Nat.make_params(shape, kernel, nb, clip, ad, Nat.F32)
            L = Nat.lib()

            def e2e_call():
                Nat.check(L.mclahe_gpu_run(C.byref(params), host_in.data_ptr(),
                                           host_out.data_ptr(), None))
            e2e_call()
            # enough calls for ~1 s
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            e2e_call()
            torch.cuda.synchronize()
            first = time.perf_counter() - w0
            k_e2e = args.e2e_steps or max(5, min(40, int(1.0 / max(first, 1e-4))))
            per_call = []
            w0 = time.perf_counter()
            for _ in range(k_e2e):
                c0 = time.perf_counter()
                e2e_call()  # synchronous: returns when the result is in host_out
                per_call.append(time.perf_counter() - c0)
            torch.cuda.synchronize()
            e2e_s = (time.perf_counter() - w0) / k_e2e
            if os.environ.get("BENCH_E2E_TRACE"):
                print("[bench] e2e per-call ms: " + " ".join(f"{t * 1e3:.1f}" for t in per_call),
                      file=sys.stderr)
            assert torch.equal(host_out, out.cpu()), "e2e result differs from device result"
            # every call is timed on its own (it is synchronous); the value is the MEDIAN
            # call -- on this pool's shared hosts a few calls in a run take 2-4x as long
            # (other tenants' load; the per-call trace, BENCH_E2E_TRACE=1, is flat
            # otherwise) -- with the mean and the slowest call reported beside it
            med_s = statistics.median(per_call)
            e2e = {"value": N_total / med_s, "unit": UNIT, "h2d_bytes_per_step": 4 * N_total,
                   "d2h_bytes_per_step": 4 * N_total + 8, "ms_per_step": med_s * 1e3,
                   "steps": k_e2e, "stat": f"median of {k_e2e} synchronous calls",
                   "mean_ms": e2e_s * 1e3, "max_ms": max(per_call) * 1e3,
                   "api": "mclahe_gpu_run (C ABI, pinned host buffers)"}
            del req
        else:
            # each rank: its slab from pinned host memory, the slab path
            # (passes + neighbour exchange), its output rows back to the host;
            # device events around the whole step, max over ranks
            host_in = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
            host_in.copy_(x)
            host_out = torch.empty_like(host_in).pin_memory()

            def e2e_step():
                x.copy_(host_in, non_blocking=True)
                S.run_rank(x, shape, kernel, nb, clip, ad, rank, world, out=out, plan=plan,
                           ws=ws, windows=windows)
                host_out.copy_(out, non_blocking=True)
            e2e_step()
            torch.cuda.synchronize()
            k_e2e = args.e2e_steps or max(3, min(args.steps, 10))
            dist.barrier()
            torch.cuda.synchronize()
            a_ev = torch.cuda.Event(enable_timing=True)
            b_ev = torch.cuda.Event(enable_timing=True)
            a_ev.record(stream)
            for _ in range(k_e2e):
                e2e_step()
            b_ev.record(stream)
            torch.cuda.synchronize()
            e_t = torch.tensor([a_ev.elapsed_time(b_ev) / k_e2e],
                               device=dev if args.dist_backend == "nccl" else "cpu")
            dist.all_reduce(e_t, op=dist.ReduceOp.MAX)
            e2e_ms = float(e_t.item())
            e2e = {"value": N_total / (e2e_ms * 1e-3), "unit": UNIT,
                   "h2d_bytes_per_step": 4 * N_total, "d2h_bytes_per_step": 4 * N_total,
                   "ms_per_step": e2e_ms, "steps": k_e2e,
                   "api": "slabs.run_rank per rank (pinned host slabs, H2D + D2H inside)"}
    clocks = sampler.summary()

    line = None
    if rank == 0:
        peak, peak_kind = peaks()
        line = {"metric": METRIC, "value": N_total / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, generated "
                "on device; stands in for the paper's photoemission set)",
                "config": workload_config(args, cfg, world),
                "launch_mode": "one CUDA graph per step" if graph is not None else "eager pass calls",
                "gpu_launches": launches,
                "clocks": clocks}
        if world == 1:
            per = np.array([[a.elapsed_time(b) for a, b in zip(e[:-1], e[1:])] for e in evs])
            med = np.median(per, 0)  # range+params, hist, mappings, interp (ms)
            Tn = 4 * plan.window_tiles * n
            algo = {"range": 4 * N_total, "hist": 4 * N_total + Tn, "map": 12 * Tn,
                    "interp": 8 * N_total + Tn}
            names = ["range", "hist", "map", "interp"]
            passes = {k: {"ms": float(m), "algo_bytes": algo[k],
                          "gbs": algo[k] / (m * 1e-3) / 1e9} for k, m in zip(names, med)}
            ach = passes["interp"]["gbs"]
            traffic = None
            tp = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
            if os.path.exists(tp):
                with open(tp) as f:
                    traffic = json.load(f).get("interp")
            ds = plan.dict_state(ws)
            kname = ("k_interp_mdict (K4 folded-pair dictionary blend)" if ds["folded"] and ds["used"] else
                     "k_interp_mdict (K4 folded-pair blend, global range)" if ds["folded"] else
                     "k_interp_pencil<DICT> (K4 dictionary blend)" if ds["used"] else
                     "k_interp_pencil (K4 blend)")
            line["roofline"] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                                "frac": ach / peak, "traffic": traffic,
                                "kernel": kname,
                                "algo_bytes_per_launch": algo["interp"],
                                "peak_source": f"{peak_kind} hbm_gbs"}
            line["passes"] = passes
            line["e2e"] = e2e
            if not args.no_cpu_baseline:
                # the whole volume when the reference finishes it in ~30 s on
                # the host (4D: ~12 s), else a dim-0 sample of whole kernel rows
                rows = sample_rows(cfg, 600_000_000)
                xs = x[:rows].cpu().numpy()
                v, kind, cores, dt = cpu_reference_sample(xs, cfg)
                what = ("the whole volume" if rows == cfg["shape"][0]
                        else f"first {rows} of {cfg['shape'][0]} dim-0 rows")
                line["cpu_baseline"] = {
                    "value": v, "unit": UNIT, "cores": cores, "kind": kind,
                    "sample": f"{what} ({xs.size} voxels), one run, {dt:.2f} s",
                    "host": host_cpu_info()}
        else:
            line["e2e"] = e2e
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
