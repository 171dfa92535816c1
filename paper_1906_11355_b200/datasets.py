"""Seeded synthetic inputs for the five BASELINE.json configurations.

The paper's photoemission and fluorescence datasets are not available, so
these generators stand in for them with the shapes, value ranges and value
statistics BASELINE.json specifies (quantised Poisson counts, saturated
pixels, all-zero regions that make adaptive tiles degenerate, negative
values in 5D).  Constants BASELINE.json leaves open are fixed here once.

Everything is torch, so the same code runs on the CPU (tests, oracle-sized
cases) and on the GPU (full-size bench inputs; 8.6 GB for Large 4D).  A
``scale`` < 1 shrinks every extent (and the kernel) for CPU-sized parity runs.
"""
from __future__ import annotations

import math

import torch

CONFIGS = {
    "2d": dict(shape=(1024, 1024), kernel=(64, 64), n_bins=256, clip_limit=0.01, adaptive=False),
    "3d": dict(shape=(256, 256, 256), kernel=(32, 32, 32), n_bins=256, clip_limit=0.02,
               adaptive=False),
    "4d": dict(shape=(256, 256, 128, 32), kernel=(32, 32, 16, 4), n_bins=256, clip_limit=0.02,
               adaptive=True),
    "l4d": dict(shape=(512, 512, 256, 32), kernel=(64, 64, 32, 8), n_bins=512, clip_limit=0.01,
                adaptive=False),
    "5d": dict(shape=(128, 128, 64, 16, 16), kernel=(16, 16, 8, 4, 4), n_bins=128,
               clip_limit=0.03, adaptive=True),
}


def scaled(name: str, div: int = 1) -> dict:
    """Config with every extent and kernel size divided by ``div`` (>= 1)."""
    c = dict(CONFIGS[name])
    c["shape"] = tuple(max(1, s // div) for s in c["shape"])
    c["kernel"] = tuple(max(1, min(k // div, s)) for k, s in zip(c["kernel"], c["shape"]))
    return c


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _u(g, n, lo, hi, device):
    return lo + (hi - lo) * torch.rand(n, generator=g, device=device, dtype=torch.float64)


def _add_blobs(vol, g, count, sigma_lo, sigma_hi, amp, anisotropic):
    """Adds separable Gaussian blobs (uniform centres) into vol (float64)."""
    dev = vol.device
    D = vol.dim()
    centres = [_u(g, count, 0, s, dev) for s in vol.shape]
    if anisotropic:
        sig = [_u(g, count, sigma_lo, sigma_hi, dev) for _ in range(D)]
    else:
        s1 = _u(g, count, sigma_lo, sigma_hi, dev)
        sig = [s1] * D
    c_h = [c.cpu() for c in centres]
    s_h = [s.cpu() for s in sig]
    a_h = amp.cpu()
    for b in range(count):
        sl, prof = [], []
        for d in range(D):
            c, s = float(c_h[d][b]), float(s_h[d][b])
            lo, hi = max(0, int(c - 4 * s)), min(vol.shape[d], int(c + 4 * s) + 1)
            if hi <= lo:
                break
            x = torch.arange(lo, hi, device=dev, dtype=torch.float64)
            prof.append(torch.exp(-0.5 * ((x - c) / s) ** 2))
            sl.append(slice(lo, hi))
        else:
            box = prof[0]
            for p in prof[1:]:
                box = box.unsqueeze(-1) * p
            vol[tuple(sl)] += float(a_h[b]) * box
    return vol


def gen_2d(shape=(1024, 1024), seed=0, device="cpu"):
    g = _gen(seed, device)
    H, W = shape
    x = torch.linspace(0.2, 0.6, W, device=device, dtype=torch.float64)
    vol = x.expand(H, W).clone()
    amp = _u(g, 40, 0.1, 0.4, device)
    scale = max(H, W) / 1024.0
    _add_blobs(vol, g, 40, 5 * scale, 30 * scale, amp, anisotropic=False)
    vol += 0.02 * torch.randn(shape, generator=g, device=device, dtype=torch.float64)
    return vol.clamp_(0.0, 1.0).to(torch.float32)


def _poisson_normalised(intensity, peak, g):
    lam = peak * intensity / intensity.max()
    counts = torch.poisson(lam, generator=g)
    m = counts.max()
    return (counts / (m if m > 0 else 1.0)).to(torch.float32)


def gen_3d(shape=(256, 256, 256), seed=0, device="cpu"):
    g = _gen(seed, device)
    vol = torch.full(shape, 0.05, device=device, dtype=torch.float64)
    n = max(8, int(2000 * (shape[0] * shape[1] * shape[2]) / 256 ** 3))
    amp = torch.exp(torch.randn(n, generator=g, device=device, dtype=torch.float64))  # LogNormal(0,1)
    scale = shape[0] / 256.0
    _add_blobs(vol, g, n, 2 * max(scale, 0.25), 6 * max(scale, 0.25), amp, anisotropic=True)
    return _poisson_normalised(vol, 200.0, g)


# 4D photoemission bands (kx, ky in [-1, 1], E in [-1.0, 0.3] relative to E_F = 0)
_BANDS = ((0.45, -0.65), (-0.35, -0.15), (0.80, -0.95))


def gen_4d(shape=(256, 256, 128, 32), seed=0, device="cpu"):
    g = _gen(seed, device)
    nk1, nk2, nE, nt = shape
    kx = torch.linspace(-1, 1, nk1, device=device, dtype=torch.float64)
    ky = torch.linspace(-1, 1, nk2, device=device, dtype=torch.float64)
    E = torch.linspace(-1.0, 0.3, nE, device=device, dtype=torch.float64)
    k2 = kx[:, None] ** 2 + ky[None, :] ** 2
    hwhm, kT, tau = 0.03, 0.02, 8.0
    spec = torch.zeros(nk1, nk2, nE, device=device, dtype=torch.float64)
    for a, e0 in _BANDS:
        d = E[None, None, :] - (a * k2[:, :, None] + e0)
        spec += hwhm ** 2 / (d * d + hwhm ** 2)
    spec *= 1.0 / (1.0 + torch.exp(E / kT))[None, None, :]
    decay = torch.exp(-torch.arange(nt, device=device, dtype=torch.float64) / tau)
    out = torch.empty(shape, device=device, dtype=torch.float32)
    peak = 500.0
    smax = spec.max()
    for t in range(nt):  # frame by frame keeps the float64 working set small
        lam = peak * spec * decay[t] / smax
        out[..., t] = torch.poisson(lam, generator=g).to(torch.float32)
    m = out.max()
    return out / (m if m > 0 else 1.0)


def gen_5d(shape=(128, 128, 64, 16, 16), seed=0, device="cpu"):
    g = _gen(seed, device)
    base = torch.zeros(shape[:3], device=device, dtype=torch.float64)
    n = max(8, int(500 * (shape[0] * shape[1] * shape[2]) / (128 * 128 * 64)))
    amp = _u(g, n, 0.2, 1.0, device)
    scale = shape[0] / 128.0
    _add_blobs(base, g, n, 2 * max(scale, 0.25), 5 * max(scale, 0.25), amp, anisotropic=False)
    i3 = torch.arange(shape[3], device=device, dtype=torch.float64)
    i4 = torch.arange(shape[4], device=device, dtype=torch.float64)
    mod3 = 1.0 + 0.5 * torch.sin(2 * math.pi * i3 / max(shape[3], 1))
    mod4 = 0.25 + 0.75 * i4 / max(shape[4] - 1, 1)
    out = torch.empty(shape, device=device, dtype=torch.float32)
    for a in range(shape[3]):
        for b in range(shape[4]):
            frame = base * (mod3[a] * mod4[b])
            frame = frame + 0.03 * torch.randn(shape[:3], generator=g, device=device,
                                               dtype=torch.float64)
            out[:, :, :, a, b] = frame.to(torch.float32)
    return out


GENERATORS = {"2d": gen_2d, "3d": gen_3d, "4d": gen_4d, "l4d": gen_4d, "5d": gen_5d}


def make(name: str, seed: int = 0, device="cpu", shape=None) -> torch.Tensor:
    """Seeded float32 volume for config ``name`` (optionally another shape)."""
    shape = tuple(shape or CONFIGS[name]["shape"])
    return GENERATORS[name](shape=shape, seed=seed, device=device).contiguous()
