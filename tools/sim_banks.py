"""Shared-memory bank model of the 4D folded-pair dictionary blend (k_interp_mdict).

Counts, on the BASELINE 4D volume (seed 0), the shared-memory wavefronts a
warp's gathers need under a lane geometry and a dictionary-slot layout:
a 32-bit gather of 32 lanes costs max over banks of the distinct words that
bank serves (same word = broadcast).  Used to pick layouts on the CPU before
spending GPU time.

    python tools/sim_banks.py [--x0 16]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def wavefronts(slot, lanes_axis=-1):
    """slot: int array (..., 32) of 32-bit word addresses; returns (...) wavefronts."""
    s = np.sort(slot, axis=-1)
    uniq = np.ones_like(s, dtype=bool)
    uniq[..., 1:] = s[..., 1:] != s[..., :-1]
    bank = s % 32
    flat = bank.reshape(-1, 32)
    u = uniq.reshape(-1, 32)
    rows = np.repeat(np.arange(flat.shape[0]), 32)
    cnt = np.bincount(rows * 32 + flat.ravel(), weights=u.ravel(), minlength=flat.shape[0] * 32)
    return cnt.reshape(-1, 32).max(axis=1).reshape(slot.shape[:-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--x0", type=int, default=16, help="dim-0 rows sampled (every 256/x0-th)")
    a = ap.parse_args()
    import torch
    from paper_1906_11355_b200 import datasets
    x = datasets.make("4d", seed=0).numpy()
    vals, inv = np.unique(x, return_inverse=True)
    idx = inv.reshape(x.shape).astype(np.int64)
    print("distinct values", len(vals))
    rows = np.linspace(0, 255, a.x0).astype(int)
    sub = idx[rows]  # (x0, ky, E, t)
    X0, KY, E, T = sub.shape
    res = {}

    def geom(name, e_l, ky_l):
        # lanes: e_l consecutive E positions x ky_l consecutive ky rows (inside a cell)
        v = sub.reshape(X0, KY // ky_l, ky_l, E // e_l, e_l, T)
        v = v.transpose(0, 1, 3, 5, 2, 4).reshape(X0, KY // ky_l, E // e_l, T, 32)
        return v

    for name, e_l, ky_l in (("16E x 2ky (current)", 16, 2), ("8E x 4ky", 8, 4), ("32E", 32, 1),
                            ("4E x 8ky", 4, 8), ("2E x 16ky", 2, 16)):
        v = geom(name, e_l, ky_l)
        w = wavefronts(v)
        distinct = np.array([len(np.unique(r)) for r in v.reshape(-1, 32)[:: max(1, v.size // 32 // 20000)]])
        res[name] = w.mean()
        print(f"{name:22s} gather wavefronts / warp access {w.mean():.3f}  distinct/warp {distinct.mean():.2f}")
    v = geom("", 16, 2)
    # slot remaps of the current geometry
    for name, f in (("idx ^ ((idx>>5)&1)<<4", lambda d: d ^ (((d >> 5) & 1) << 4)),
                    ("idx*33 (pad word /32)", lambda d: d + (d >> 5)),
                    ("idx ^ (idx>>5)&31", lambda d: d ^ ((d >> 5) & 31)),
                    ("idx ^ (idx>>5)*7&31", lambda d: d ^ (((d >> 5) * 7) & 31))):
        w = wavefronts(f(v))
        print(f"remap {name:26s} {w.mean():.3f}")
    # frames mixed across lanes: lane l takes frame (k + l) & 3 of its column at step k
    vt = sub.reshape(X0, KY // 2, 2, E // 16, 16, T // 4, 4).transpose(0, 1, 3, 5, 6, 2, 4)
    vt = vt.reshape(X0, KY // 2, E // 16, T // 4, 4, 32)
    lane = np.arange(32)
    for skew in (0, 8, 16):
        tot = 0.0
        for k in range(4):
            fr = (k + lane) & 3
            d = vt[..., fr, lane]
            tot += wavefronts(d + fr * (576 + skew)).mean()
        print(f"frames mixed over lanes, table skew {skew:2d}: {tot / 4:.3f}")


if __name__ == "__main__":
    main()
