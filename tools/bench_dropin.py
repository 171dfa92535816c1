"""The C++ drop-in end to end, as a reference user sees it: the reference's
own test shim (oracle/ref_shim.cpp: NdImage in, mclahe::mclahe, NdImage out)
compiled unmodified against include/mclahe/*.hpp and linked to
libmclahe_cpp.so ("b200"), against the same shim on the compiled reference
("ref").  float64 input (the reference's element type): once with
float32-representable values (the f32 GPU path) and once with values that
are not (the f64 GPU path).  Prints one JSON line per case."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1906_11355_b200 import datasets  # noqa: E402

LIB = os.path.join(ROOT, "paper_1906_11355_b200", "lib")
shim = "/tmp/libshim_b200_bench.so"
subprocess.run(["g++", "-O3", "-DNDEBUG", "-std=gnu++20", "-fPIC", "-shared", "-pthread",
                "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "oracle", "ref_shim.cpp"),
                "-L", LIB, "-lmclahe_cpp", "-lmclahe_gpu", f"-Wl,-rpath,{LIB}", "-o", shim],
               check=True)
os.environ["MCLAHE_SHIM_B200"] = shim

configs = sys.argv[1:] or ["4d"]
for name in configs:
    cfg = datasets.CONFIGS[name]
    x32 = datasets.make(name, seed=0, device="cuda").cpu().numpy()
    args = (cfg["kernel"], cfg["n_bins"], cfg["clip_limit"], cfg["adaptive"])
    for kind in ("f32-exact", "f64"):
        x = x32.astype(np.float64)
        if kind == "f64":
            x = x + np.random.default_rng(1).normal(0, 1e-9, x.shape)
        O.mclahe(x, *args, "b200")  # warm: plan, library, pinned buffers
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            out = O.mclahe(x, *args, "b200")
        dt = (time.perf_counter() - t0) / reps
        line = {"config": name, "input": kind, "voxels": int(x.size), "b200_s": dt,
                "b200_vox_per_s": x.size / dt}
        if os.environ.get("WITH_REF"):
            t0 = time.perf_counter()
            want = O.mclahe(x, *args, "ref", threads=0)
            line["ref_s"] = time.perf_counter() - t0
            line["max_abs_err"] = float(np.max(np.abs(out - want)))
        # the GPU passes alone, device-resident (same dtype path as above)
        import paper_1906_11355_b200 as M
        xt = torch.from_numpy(x if kind == "f64" else x32).cuda()
        M.enhance(xt, *args)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            M.enhance(xt, *args)
        torch.cuda.synchronize()
        line["device_s"] = (time.perf_counter() - t0) / reps
        print(json.dumps(line), flush=True)
        del x, out, xt
