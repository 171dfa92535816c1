"""Per-call times of the one-shot host call (mclahe_gpu_run, pinned buffers) on the 4D
config, with and without an `nvidia-smi -lms 100` poller beside it (bench.py samples
clocks that way):  python tools/e2e_jitter.py [calls]"""
import ctypes as C
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1906_11355_b200 import _native as Nat, datasets  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    c = datasets.CONFIGS["4d"]
    x = datasets.make("4d", seed=0, device="cuda")
    host_in = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
    host_in.copy_(x)
    host_out = torch.empty_like(host_in).pin_memory()
    del x
    params = Nat.make_params(tuple(host_in.shape), c["kernel"], c["n_bins"], c["clip_limit"],
                             c["adaptive"], Nat.F32)
    L = Nat.lib()

    def call():
        Nat.check(L.mclahe_gpu_run(C.byref(params), host_in.data_ptr(), host_out.data_ptr(), None))

    for poll in (False, True, False, True):
        p = None
        if poll:
            p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader",
                                  "-lms", "100"], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        call()
        ts = []
        for _ in range(n):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            call()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        if p:
            p.terminate()
            p.wait()
        s = sorted(ts)
        print(f"poller={'on ' if poll else 'off'} calls={n} min {s[0]:.2f} median {s[n // 2]:.2f} "
              f"mean {sum(s) / n:.2f} p90 {s[int(n * 0.9)]:.2f} max {s[-1]:.2f} ms")


if __name__ == "__main__":
    main()
