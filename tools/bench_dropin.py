"""The C++ drop-in end to end, as a reference user sees it: tools/dropin_timer.cpp
(NdImage from an NPY file, mclahe::mclahe timed alone) linked once against the
compiled reference (oracle/_ref/libmclahe_ref.so, all host threads) and once
against the B200 drop-in (libmclahe_cpp.so).  float64 input, the reference's
element type: with float32-representable values (the f32 GPU path) and with
values that are not (the f64 GPU path).  Also the GPU passes alone on a
device-resident tensor of the same dtype.  One JSON line per case."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_11355_b200 as M  # noqa: E402
from paper_1906_11355_b200 import datasets  # noqa: E402

LIB = os.path.join(ROOT, "paper_1906_11355_b200", "lib")
REF = os.path.join(ROOT, "oracle", "_ref")
SRC = os.path.join(ROOT, "tools", "dropin_timer.cpp")


def build(out, ref):
    cmd = ["g++", "-O3", "-DNDEBUG", "-std=gnu++20", "-pthread", SRC, "-o", out]
    if ref:  # the reference's own headers are not shipped; its API is ours, declaration for declaration
        cmd[5:5] = ["-I", os.path.join(ROOT, "include")]
        cmd += ["-L", REF, "-lmclahe_ref", f"-Wl,-rpath,{REF}"]
    else:
        cmd[5:5] = ["-I", os.path.join(ROOT, "include")]
        cmd += ["-L", LIB, "-lmclahe_cpp", "-lmclahe_gpu", f"-Wl,-rpath,{LIB}"]
    subprocess.run(cmd, check=True)


exe_b200, exe_ref = "/tmp/dropin_timer_b200", "/tmp/dropin_timer_ref"
build(exe_b200, False)
have_ref = os.path.exists(os.path.join(REF, "libmclahe_ref.so"))
if have_ref:
    build(exe_ref, True)

for name in sys.argv[1:] or ["4d"]:
    cfg = datasets.CONFIGS[name]
    x32 = datasets.make(name, seed=0, device="cuda").cpu().numpy()
    kern = ",".join(str(k) for k in cfg["kernel"])
    for kind in ("f32-exact", "f64"):
        x = x32.astype(np.float64)
        if kind == "f64":
            x = x + np.random.default_rng(1).normal(0, 1e-9, x.shape)
        path = f"/tmp/dropin_{name}_{kind}.npy"
        np.save(path, x)
        argv = [path, kern, str(cfg["n_bins"]), str(cfg["clip_limit"]), str(int(cfg["adaptive"]))]
        line = {"config": name, "input": kind, "voxels": int(x.size)}
        r = subprocess.run([exe_b200] + argv + ["4", "0"], capture_output=True, text=True, check=True,
                           env=dict(os.environ, MCLAHE_DROPIN_TRACE="1"))
        sys.stderr.write(r.stderr)
        b = json.loads(r.stdout)
        line.update(b200_best_s=b["best_s"], b200_mean_s=b["mean_s"], b200_checksum=b["checksum"])
        if have_ref and os.environ.get("WITH_REF"):
            r = subprocess.run([exe_ref] + argv + ["1", "0"], capture_output=True, text=True, check=True)
            q = json.loads(r.stdout)
            line.update(ref_s=q["best_s"], ref_checksum=q["checksum"],
                        speedup=q["best_s"] / b["best_s"])
        xt = torch.from_numpy(x if kind == "f64" else x32).cuda()
        args = (cfg["kernel"], cfg["n_bins"], cfg["clip_limit"], cfg["adaptive"])
        M.enhance(xt, *args)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            M.enhance(xt, *args)
        torch.cuda.synchronize()
        line["device_s"] = (time.perf_counter() - t0) / 3
        print(json.dumps(line), flush=True)
        os.remove(path)
        del x, xt
