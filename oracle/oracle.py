"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle.

Two checkers live behind one interface (``impl=``):

* ``"c"``   -- ``oracle/liboracle.so``, the plain-C restatement
              (``oracle/mclahe_oracle.c``) of the reference algorithm.
* ``"ref"`` -- ``oracle/_ref/libmclahe_ref.so``, the reference library compiled
              from its own sources (``oracle/Makefile``) behind a C shim
              (``oracle/ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference legs may import this module.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIBS: dict[str, C.CDLL] = {}

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref/ when /root/reference is present)."""
    kw = dict(stdout=subprocess.DEVNULL, stderr=subprocess.STDOUT) if quiet else {}
    subprocess.run(["make", "-s", "-C", HERE], check=True, **kw)


def _lib(impl: str) -> C.CDLL:
    if impl in _LIBS:
        return _LIBS[impl]
    if impl == "c":
        path = os.path.join(HERE, "liboracle.so")
    elif impl == "ref":
        path = os.path.join(HERE, "_ref", "libmclahe_ref.so")
    elif impl == "b200":
        # oracle/ref_shim.cpp compiled UNMODIFIED against the B200 drop-in's
        # headers (include/mclahe/*.hpp) and linked to libmclahe_cpp.so -- a
        # reference caller re-linked to the GPU build (tests/test_dropin_cpp.py
        # builds it); the same ctypes surface as "ref"
        path = os.environ.get("MCLAHE_SHIM_B200", os.path.join(HERE, "_ref", "libshim_b200.so"))
    else:
        raise ValueError(f"unknown oracle impl {impl!r}")
    if not os.path.exists(path):
        build()
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    lib = C.CDLL(path)
    if impl == "c":
        lib.orc_bin_index.restype = C.c_int64
        lib.orc_bin_index.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int64]
        lib.orc_mirror_index.restype = C.c_int64
        lib.orc_mirror_index.argtypes = [C.c_int64, C.c_int64]
        lib.orc_pad_plan.argtypes = [C.c_int, _i64p, _i64p, _i64p, _i64p]
        lib.orc_clip_histogram.argtypes = [_f64p, C.c_int64, C.c_double, _f64p]
        lib.orc_normalized_cdf.argtypes = [_f64p, C.c_int64, _f64p]
        lib.orc_tile_stats.argtypes = [_f64p, C.c_int, _i64p, _i64p, C.c_int64, C.c_double,
                                       C.c_int, _f64p, _f64p, _f64p, _f64p, _f64p, _u8p]
        lib.orc_neighbor_1d.argtypes = [C.c_int64, C.c_int64, C.c_int64, _i64p, _f64p, _f64p]
        lib.orc_interp_coefficients.argtypes = [C.c_int, _f64p, _f64p, _i64p, _f64p]
        lib.orc_blend.restype = C.c_double
        lib.orc_blend.argtypes = [C.c_int, _f64p, _f64p]
        lib.orc_mclahe.argtypes = [_f64p, C.c_int, _i64p, _i64p, C.c_int64, C.c_double,
                                   C.c_int, _f64p, C.c_char_p, C.c_int]
    else:
        lib.ref_mclahe.argtypes = [_f64p, C.c_int, _i64p, _i64p, C.c_int64, C.c_double,
                                   C.c_int, C.c_uint, _f64p, _f64p, C.c_char_p, C.c_int]
        lib.ref_tile_stats.argtypes = [_f64p, C.c_int, _i64p, _i64p, C.c_int64, C.c_double,
                                       C.c_int, _f64p, _f64p, _f64p, _f64p, _f64p, _u8p,
                                       C.c_char_p, C.c_int]
        lib.ref_tile_stats_window.argtypes = [
            _f64p, C.c_int, _i64p, _i64p, C.c_int64, C.c_double, C.c_int, C.c_int, C.c_double,
            C.c_double, C.c_int64, C.c_int64, C.c_uint, _f64p, _f64p, _f64p, _f64p, _f64p, _u8p,
            C.c_char_p, C.c_int]
        lib.ref_blend_rows.argtypes = [
            _f64p, C.c_int, _i64p, _i64p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
            _f64p, _f64p, _f64p, _u8p, C.c_uint, _f64p, C.c_char_p, C.c_int]
        lib.ref_bin_index.restype = C.c_int64
        lib.ref_bin_index.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int64]
        lib.ref_clip_histogram.argtypes = [_f64p, C.c_int64, C.c_double, _f64p]
        lib.ref_normalized_cdf.argtypes = [_f64p, C.c_int64, _f64p]
        lib.ref_neighbors.argtypes = [C.c_int, _i64p, _i64p, _i64p, _i64p, _f64p, _f64p, _f64p]
        lib.ref_transform_pixel.restype = C.c_double
        lib.ref_transform_pixel.argtypes = [C.c_double, C.c_int, _f64p, C.c_int64, _f64p,
                                            _f64p, _u8p, _f64p]
    _LIBS[impl] = lib
    return lib


def have_ref() -> bool:
    try:
        _lib("ref")
        return True
    except (FileNotFoundError, OSError, subprocess.CalledProcessError):
        return False


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _i64(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(seq, dtype=np.int64))


class OracleValidationError(ValueError):
    """The reference rejected the request (ValidationError)."""


def mclahe(data: np.ndarray, kernel, n_bins: int = 256, clip_limit: float = 1.0,
           adaptive: bool = False, impl: str = "c", threads: int = 0,
           timings: list | None = None) -> np.ndarray:
    """Full pipeline; returns float64 of data's shape (mclahe, pipeline.cpp:73)."""
    x = np.ascontiguousarray(data, dtype=np.float64)
    shape, ker = _i64(x.shape), _i64(kernel)
    out = np.empty(x.shape, dtype=np.float64)
    err = C.create_string_buffer(256)
    lib = _lib(impl)
    if impl == "c":
        rc = lib.orc_mclahe(_p(x, _f64p), x.ndim, _p(shape, _i64p), _p(ker, _i64p), int(n_bins),
                            float(clip_limit), int(bool(adaptive)), _p(out, _f64p), err, 256)
    else:
        t = np.zeros(3)
        rc = lib.ref_mclahe(_p(x, _f64p), x.ndim, _p(shape, _i64p), _p(ker, _i64p), int(n_bins),
                            float(clip_limit), int(bool(adaptive)), int(threads), _p(out, _f64p),
                            _p(t, _f64p), err, 256)
        if timings is not None:
            timings[:] = list(t)
    if rc == 1:
        raise OracleValidationError(err.value.decode())
    if rc != 0:
        raise RuntimeError(err.value.decode())
    return out


def geometry(shape, kernel):
    """(before, after, grid) per dimension (compute_pad_plan, nd_image.cpp:85-102)."""
    shape, kernel = _i64(shape), _i64(kernel)
    before, after = np.zeros_like(shape), np.zeros_like(shape)
    if _lib("c").orc_pad_plan(len(shape), _p(shape, _i64p), _p(kernel, _i64p),
                              _p(before, _i64p), _p(after, _i64p)):
        raise OracleValidationError("invalid kernel")
    grid = (shape + before + after) // kernel
    return before, after, grid


def tile_stats(data: np.ndarray, kernel, n_bins: int, clip_limit: float, adaptive: bool,
               impl: str = "c") -> dict:
    """Per-tile lo/hi/counts/clipped/lut/degenerate (build_mappings internals)."""
    x = np.ascontiguousarray(data, dtype=np.float64)
    shape, ker = _i64(x.shape), _i64(kernel)
    _, _, grid = geometry(x.shape, kernel)
    T = int(np.prod(grid))
    lo, hi = np.zeros(T), np.zeros(T)
    counts, clipped, lut = (np.zeros((T, n_bins)) for _ in range(3))
    degen = np.zeros(T, dtype=np.uint8)
    args = [_p(x, _f64p), x.ndim, _p(shape, _i64p), _p(ker, _i64p), int(n_bins),
            float(clip_limit), int(bool(adaptive)), _p(lo, _f64p), _p(hi, _f64p),
            _p(counts, _f64p), _p(clipped, _f64p), _p(lut, _f64p), _p(degen, _u8p)]
    if impl == "c":
        rc = _lib("c").orc_tile_stats(*args)
    else:
        err = C.create_string_buffer(256)
        rc = _lib(impl).ref_tile_stats(*args, err, 256)
    if rc:
        raise OracleValidationError("tile_stats rejected the request")
    return dict(lo=lo, hi=hi, counts=counts, clipped=clipped, lut=lut,
                degenerate=degen.astype(bool), grid=tuple(int(g) for g in grid))


def ref_tile_stats_window(data: np.ndarray, kernel, n_bins: int, clip_limit: float,
                          adaptive: bool, tile_row0: int, tile_rows: int,
                          global_range=None, threads: int = 0, impl: str = "ref") -> dict:
    """The compiled reference's per-tile intermediates for tile rows
    [tile_row0, tile_row0 + tile_rows) along dim 0 of ``data`` (its own
    symmetric_pad / kernelize / build_mappings, multi-threaded).  global_range
    (lo, hi) overrides the Global-mode range -- for dim-0 crops of a larger
    volume (see ref_shim.cpp)."""
    x = np.ascontiguousarray(data, dtype=np.float64)
    shape, ker = _i64(x.shape), _i64(kernel)
    _, _, grid = geometry(x.shape, kernel)
    T = int(tile_rows) * int(np.prod(grid[1:]))
    lo, hi = np.zeros(T), np.zeros(T)
    counts, clipped, lut = (np.zeros((T, n_bins)) for _ in range(3))
    degen = np.zeros(T, dtype=np.uint8)
    err = C.create_string_buffer(256)
    g = global_range is not None
    glo, ghi = (float(global_range[0]), float(global_range[1])) if g else (0.0, 0.0)
    rc = _lib(impl).ref_tile_stats_window(
        _p(x, _f64p), x.ndim, _p(shape, _i64p), _p(ker, _i64p), int(n_bins), float(clip_limit),
        int(bool(adaptive)), int(g), glo, ghi, int(tile_row0), int(tile_rows), int(threads),
        _p(lo, _f64p), _p(hi, _f64p), _p(counts, _f64p), _p(clipped, _f64p), _p(lut, _f64p),
        _p(degen, _u8p), err, 256)
    if rc:
        raise RuntimeError(err.value.decode())
    return dict(lo=lo, hi=hi, counts=counts, clipped=clipped, lut=lut,
                degenerate=degen.astype(bool))


def ref_tile_rows_by_crop(x: np.ndarray, kernel, n_bins: int, clip_limit: float,
                          adaptive: bool, t0: int, t1: int, global_range, threads: int = 0):
    """Reference intermediates of tile rows [t0, t1) of a volume too large for
    the reference's padded + kernelized copies, from one dim-0 crop.

    With shape[0] % b0 == 0 every crop whose length is a multiple of b0 gets
    the full volume's dim-0 padding (compute_pad_plan, nd_image.cpp:97-99:
    before = floor(b0/2)).  Crop [(t0-1)*b0, (t1)*b0) then holds the full
    volume's tile t as its tile t - t0 + 1 (tile rows of the crop away from its
    own mirrored ends); a crop starting at row 0 keeps tile 0, and one ending at
    the last row keeps the last tile.  Global mode takes the full volume's
    range.  Returns (stats, crop_row0)."""
    s0, b0 = int(x.shape[0]), int(kernel[0])
    assert s0 % b0 == 0, "crop windows need shape[0] % kernel[0] == 0"
    g0 = s0 // b0 + 1
    a = max(0, (t0 - 1) * b0)
    e = min(s0, t1 * b0)
    if t1 == g0:  # window reaching the last tile: the crop ends at the last row
        e = s0
    first = t0 - (a // b0)  # crop tile index of full tile t0
    if a > 0:
        first = 1
    st = ref_tile_stats_window(x[a:e], kernel, n_bins, clip_limit, adaptive, first, t1 - t0,
                               global_range=global_range, threads=threads)
    return st, a


def ref_blend_rows(rows: np.ndarray, full_shape, kernel, row0: int, n_bins: int,
                   tile_row0: int, stats: dict, threads: int = 0, impl: str = "ref") -> np.ndarray:
    """The reference's per-voxel loop (pipeline.cpp:94-127) for original rows
    [row0, row0 + len(rows)) of a volume of ``full_shape``, over the mappings of
    ``stats`` (tile rows starting at tile_row0)."""
    x = np.ascontiguousarray(rows, dtype=np.float64)
    shape, ker = _i64(full_shape), _i64(kernel)
    per_row = int(np.prod(geometry(full_shape, kernel)[2][1:]))
    tile_rows = len(stats["lo"]) // per_row
    out = np.empty_like(x)
    err = C.create_string_buffer(256)
    lut = np.ascontiguousarray(stats["lut"], dtype=np.float64)
    degen = np.ascontiguousarray(stats["degenerate"], dtype=np.uint8)
    lo = np.ascontiguousarray(stats["lo"], dtype=np.float64)
    hi = np.ascontiguousarray(stats["hi"], dtype=np.float64)
    rc = _lib(impl).ref_blend_rows(
        _p(x, _f64p), len(full_shape), _p(shape, _i64p), _p(ker, _i64p), int(row0),
        int(row0) + x.shape[0], int(n_bins), int(tile_row0), int(tile_rows), _p(lo, _f64p),
        _p(hi, _f64p), _p(lut, _f64p), _p(degen, _u8p), int(threads), _p(out, _f64p), err, 256)
    if rc:
        raise RuntimeError(err.value.decode())
    return out


def bin_index(value: float, lo: float, hi: float, n_bins: int, impl: str = "c") -> int:
    if impl == "c":
        return int(_lib("c").orc_bin_index(value, lo, hi, n_bins))
    return int(_lib(impl).ref_bin_index(value, lo, hi, n_bins))


def bin_index_array(values: np.ndarray, lo: float, hi: float, n_bins: int) -> np.ndarray:
    """Vectorised restatement of bin_index (histogram.cpp:24-32) in numpy
    float64 (IEEE round-to-nearest, no FMA): floor((v-lo)/(hi-lo)*n), clamped."""
    v = np.asarray(values, dtype=np.float64)
    with np.errstate(invalid="ignore", divide="ignore"):
        scaled = np.floor((v - np.float64(lo)) / (np.float64(hi) - np.float64(lo))
                          * np.float64(n_bins))
    out = np.where(scaled > 0.0, scaled, 0.0)
    out = np.where(out >= n_bins, n_bins - 1, out)
    return out.astype(np.int64)


def clip_histogram(counts, clip_limit: float, impl: str = "c") -> np.ndarray:
    c = np.ascontiguousarray(counts, dtype=np.float64)
    out = np.empty_like(c)
    getattr(_lib(impl), "orc_clip_histogram" if impl == "c" else "ref_clip_histogram")(
        _p(c, _f64p), c.size, float(clip_limit), _p(out, _f64p))
    return out


def normalized_cdf(clipped, impl: str = "c"):
    c = np.ascontiguousarray(clipped, dtype=np.float64)
    out = np.empty_like(c)
    d = getattr(_lib(impl), "orc_normalized_cdf" if impl == "c" else "ref_normalized_cdf")(
        _p(c, _f64p), c.size, _p(out, _f64p))
    return out, bool(d)


def neighbors(pixel, kernel, grid, impl: str = "c"):
    """(lower, dist_lo, dist_hi, coefficients) for one padded pixel."""
    rank = len(pixel)
    px, ker, gr = _i64(pixel), _i64(kernel), _i64(grid)
    lower = np.zeros(rank, dtype=np.int64)
    dlo, dhi = np.zeros(rank), np.zeros(rank)
    coeff = np.zeros(1 << rank)
    if impl == "c":
        lib = _lib("c")
        for j in range(rank):
            lj = C.c_int64()
            a, b = C.c_double(), C.c_double()
            if lib.orc_neighbor_1d(int(px[j]), int(ker[j]), int(gr[j]), C.byref(lj),
                                   C.byref(a), C.byref(b)):
                raise OracleValidationError("pixel outside the valid interpolation region")
            lower[j], dlo[j], dhi[j] = lj.value, a.value, b.value
        lib.orc_interp_coefficients(rank, _p(dlo, _f64p), _p(dhi, _f64p), _p(ker, _i64p),
                                    _p(coeff, _f64p))
    else:
        if _lib(impl).ref_neighbors(rank, _p(px, _i64p), _p(ker, _i64p), _p(gr, _i64p),
                                     _p(lower, _i64p), _p(dlo, _f64p), _p(dhi, _f64p),
                                     _p(coeff, _f64p)):
            raise OracleValidationError("pixel outside the valid interpolation region")
    return lower, dlo, dhi, coeff


def blend(coeff, mapped) -> float:
    """transform_pixel's ascending-order sum and clamp (interpolation.cpp:68-86)."""
    c = np.ascontiguousarray(coeff, dtype=np.float64)
    m = np.ascontiguousarray(mapped, dtype=np.float64)
    return float(_lib("c").orc_blend(c.size, _p(c, _f64p), _p(m, _f64p)))


def transform_pixel_ref(value, luts, lo, hi, degenerate, coeff, impl: str = "ref") -> float:
    luts = np.ascontiguousarray(luts, dtype=np.float64)
    lo, hi, coeff = (np.ascontiguousarray(a, dtype=np.float64) for a in (lo, hi, coeff))
    dg = np.ascontiguousarray(degenerate, dtype=np.uint8)
    return float(_lib(impl).ref_transform_pixel(float(value), coeff.size, _p(luts, _f64p),
                                                 luts.shape[1], _p(lo, _f64p), _p(hi, _f64p),
                                                 _p(dg, _u8p), _p(coeff, _f64p)))


# ---- prefilters and metrics: numpy restatements + the reference ----

def mirror_index_array(idx: np.ndarray, extent: int) -> np.ndarray:
    """mirror_index (nd_image.cpp:27-34), vectorised: period 2n, edge-including."""
    period = 2 * extent
    m = np.mod(idx, period)
    return np.where(m >= extent, period - 1 - m, m)


def gaussian_taps(sigma: float, truncate: float) -> np.ndarray:
    """gaussian_taps (filters.cpp:12-23): exp(-t^2/2) at k/sigma, k in
    [-ceil(truncate*sigma), +], normalised by their sequential sum."""
    import math
    radius = int(math.ceil(truncate * sigma))
    taps = [math.exp(-0.5 * (k / sigma) * (k / sigma)) for k in range(-radius, radius + 1)]
    total = 0.0
    for w in taps:
        total += w
    return np.array([w / total for w in taps])


def gaussian_filter_np(x: np.ndarray, sigmas, truncate: float = 4.0) -> np.ndarray:
    """gaussian_filter (filters.cpp:82-96 over convolve_axis :28-80): one pass per
    axis with sigma > 0, acc += tap * line[mirror(x + k)] for k ascending."""
    out = np.asarray(x, dtype=np.float64).copy()
    for axis, s in enumerate(sigmas):
        if s == 0.0:
            continue
        taps = gaussian_taps(float(s), float(truncate))
        r = (len(taps) - 1) // 2
        n = out.shape[axis]
        src = np.moveaxis(out, axis, -1)
        acc = np.zeros_like(src)
        pos = np.arange(n)
        for k in range(-r, r + 1):  # sequential in k, each product and sum rounded
            acc = acc + taps[k + r] * src[..., mirror_index_array(pos + k, n)]
        out = np.ascontiguousarray(np.moveaxis(acc, -1, axis))
    return out


def median_filter_np(x: np.ndarray, window) -> np.ndarray:
    """median_filter (filters.cpp:98-142): offsets -floor((w-1)/2)..floor(w/2) per
    dim, mirrored; even counts take the mean of the two central values."""
    x = np.asarray(x, dtype=np.float64)
    stack = []
    grids = [range(-((w - 1) // 2), w // 2 + 1) for w in window]
    import itertools
    for offs in itertools.product(*grids):
        idx = np.ix_(*[mirror_index_array(np.arange(n) + o, n) for n, o in zip(x.shape, offs)])
        stack.append(x[idx])
    st = np.sort(np.stack(stack, axis=0), axis=0)
    m = st.shape[0] // 2
    return st[m] if st.shape[0] % 2 else 0.5 * (st[m - 1] + st[m])


def metrics_np(a: np.ndarray, b: np.ndarray, n_bins: int = 256, peak: float = 1.0) -> dict:
    """compute_metrics (metrics.cpp:11-72); sums in numpy order (tolerance-equal)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    d = a - b
    mse_ = float(np.sum(d * d) / a.size)
    psnr_ = float("inf") if mse_ == 0.0 else float(10.0 * np.log10(peak * peak / mse_))
    mean = float(np.sum(a) / a.size)
    std_ = float(np.sqrt(np.sum((a - mean) ** 2) / a.size))
    lo, hi = float(a.min()), float(a.max())
    ent = 0.0
    if hi > lo:
        bins = bin_index_array(a, lo, hi, n_bins)
        counts = np.bincount(bins, minlength=n_bins).astype(np.float64)
        for c in counts:  # bin order, as the reference
            if c > 0:
                p = c / a.size
                ent -= p * np.log2(p)
    return dict(mse=mse_, psnr_db=psnr_, std=std_, entropy_bits=float(ent))


def gaussian_filter_ref(x: np.ndarray, sigmas, truncate: float = 4.0,
                        impl: str = "ref") -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    sg = np.ascontiguousarray(np.asarray(sigmas, dtype=np.float64))
    shape, out, err = _i64(x.shape), np.empty_like(x), C.create_string_buffer(256)
    rc = _lib(impl).ref_gaussian(_p(x, _f64p), x.ndim, _p(shape, _i64p), _p(sg, _f64p),
                                  C.c_double(truncate), _p(out, _f64p), err, 256)
    if rc:
        raise OracleValidationError(err.value.decode())
    return out


def median_filter_ref(x: np.ndarray, window, impl: str = "ref") -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    shape, win = _i64(x.shape), _i64(window)
    out, err = np.empty_like(x), C.create_string_buffer(256)
    rc = _lib(impl).ref_median(_p(x, _f64p), x.ndim, _p(shape, _i64p), _p(win, _i64p),
                                _p(out, _f64p), err, 256)
    if rc:
        raise OracleValidationError(err.value.decode())
    return out


def metrics_ref(a: np.ndarray, b: np.ndarray, n_bins: int = 256, peak: float = 1.0,
                impl: str = "ref") -> dict:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    shape, out, err = _i64(a.shape), np.zeros(4), C.create_string_buffer(256)
    rc = _lib(impl).ref_metrics(_p(a, _f64p), _p(b, _f64p), a.ndim, _p(shape, _i64p),
                                 C.c_int64(n_bins), C.c_double(peak), _p(out, _f64p), err, 256)
    if rc:
        raise OracleValidationError(err.value.decode())
    return dict(mse=out[0], psnr_db=out[1], std=out[2], entropy_bits=out[3])
