"""ctypes binding of the C ABI in include/mclahe_gpu.h (libmclahe_gpu.so).

The shared library is built in-tree (``paper_1906_11355_b200/lib``) by
``__graft_entry__.build()`` / ``csrc/Makefile``.  There is no CPU fallback:
if the library cannot be loaded (or built with nvcc) every entry point
raises :class:`NativeUnavailable`.
"""
from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libmclahe_gpu.so")
CSRC = os.path.join(PKG, "csrc")

MAX_RANK = 8
OK, ERR_VALIDATION, ERR_CUDA, ERR_COMM, ERR_OOM, ERR_UNSUPPORTED = range(6)
F32, F64 = 0, 1


class NativeUnavailable(RuntimeError):
    """The CUDA library is missing and could not be built."""


class ValidationError(ValueError):
    """Mirror of mclahe::ValidationError (include/mclahe/nd_image.hpp:19-22)."""


class CudaError(RuntimeError):
    pass


class Params(C.Structure):
    _fields_ = [("rank", C.c_int32), ("adaptive", C.c_int32), ("dtype", C.c_int32),
                ("reserved", C.c_int32), ("shape", C.c_int64 * MAX_RANK),
                ("kernel", C.c_int64 * MAX_RANK), ("n_bins", C.c_int64),
                ("clip_limit", C.c_double)]


class Timings(C.Structure):
    _fields_ = [("pad_s", C.c_double), ("histograms_s", C.c_double),
                ("interpolation_s", C.c_double)]


class Metrics(C.Structure):
    _fields_ = [("mse", C.c_double), ("psnr_db", C.c_double), ("std", C.c_double),
                ("entropy_bits", C.c_double), ("n_bins_used", C.c_int64)]


class PlanInfo(C.Structure):
    _fields_ = [("rank", C.c_int32), ("fast_hist", C.c_int32), ("fast_interp", C.c_int32),
                ("trailing_dims", C.c_int32), ("before", C.c_int64 * MAX_RANK),
                ("after", C.c_int64 * MAX_RANK), ("grid", C.c_int64 * MAX_RANK),
                ("tiles", C.c_int64), ("row_begin", C.c_int64), ("row_end", C.c_int64),
                ("tile_row_begin", C.c_int64), ("tile_row_end", C.c_int64),
                ("count_row_begin", C.c_int64), ("count_row_end", C.c_int64),
                ("need_row_begin", C.c_int64), ("need_row_end", C.c_int64),
                ("tiles_per_row", C.c_int64), ("n_bins", C.c_int64),
                ("off_range", C.c_int64), ("off_tile_range", C.c_int64),
                ("off_counts", C.c_int64), ("off_tparams", C.c_int64), ("off_lut", C.c_int64),
                ("off_thr", C.c_int64), ("workspace_bytes", C.c_int64), ("hist_units", C.c_int64),
                ("interp_units", C.c_int64)]


class Debug(C.Structure):
    _fields_ = [("lo", C.c_void_p), ("hi", C.c_void_p), ("counts", C.c_void_p),
                ("clipped", C.c_void_p), ("lut", C.c_void_p), ("degenerate", C.c_void_p)]


# the symbols include/mclahe_gpu.h declares, with ctypes signatures
_vp, _i64 = C.c_void_p, C.c_int64
SIGNATURES = {
    "mclahe_gpu_run": (C.c_int, [C.POINTER(Params), _vp, _vp, C.POINTER(Timings)]),
    "mclahe_gpu_run_out_of_core": (C.c_int, [C.POINTER(Params), _vp, _vp, C.c_int64, C.POINTER(Timings)]),
    "mclahe_gpu_run_device": (C.c_int, [C.POINTER(Params), _vp, _vp, _vp, C.POINTER(Timings)]),
    "mclahe_plan_create": (C.c_int, [C.POINTER(Params), _i64, _i64, C.POINTER(_vp)]),
    "mclahe_plan_destroy": (C.c_int, [_vp]),
    "mclahe_plan_get_info": (C.c_int, [_vp, C.POINTER(PlanInfo)]),
    "mclahe_pass_reset": (C.c_int, [_vp, _vp, _vp]),
    "mclahe_pass_range": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mclahe_pass_params": (C.c_int, [_vp, _vp, _vp]),
    "mclahe_pass_histograms": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mclahe_pass_mappings": (C.c_int, [_vp, _vp, C.POINTER(Debug), _vp]),
    "mclahe_pass_interpolate": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "mclahe_plan_enqueue": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "mclahe_plan_check": (C.c_int, [_vp, _vp, _vp]),
    "mclahe_debug_bin_index": (C.c_int, [C.c_int32, _vp, _i64, C.c_double, C.c_double, _i64,
                                         _vp, _vp]),
    "mclahe_gpu_run_framewise": (C.c_int, [_vp, C.c_int32, _vp, _vp, _vp]),
    "mclahe_multi_cuts": (C.c_int, [C.POINTER(Params), C.c_int32, _vp]),
    "mclahe_gpu_run_multi": (C.c_int, [C.POINTER(Params), C.c_int32, _vp, _vp, _vp, _vp]),
    "mclahe_gpu_run_multi_device": (C.c_int, [C.POINTER(Params), C.c_int32, _vp, _vp, _vp, _vp]),
    "mclahe_block_mappings": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                        C.c_int32, C.c_double, C.c_double, _vp, _vp, _vp, _vp,
                                        _vp, _vp]),
    "mclahe_nd_gather": (C.c_int, [C.c_int32, C.c_int32, _vp, _vp, _vp, _vp, _vp]),
    "mclahe_validate": (C.c_int, [C.POINTER(Params)]),
    "mclahe_host_alloc": (C.c_void_p, [C.c_size_t]),
    "mclahe_host_free": (None, [C.c_void_p]),
    "mclahe_gaussian_filter": (C.c_int, [C.c_int32, _vp, _vp, C.c_double, _vp, _vp]),
    "mclahe_gaussian_filter_device": (C.c_int, [C.c_int32, _vp, _vp, C.c_double, _vp, _vp, _vp]),
    "mclahe_median_filter": (C.c_int, [C.c_int32, _vp, _vp, _vp, _vp]),
    "mclahe_median_filter_device": (C.c_int, [C.c_int32, _vp, _vp, _vp, _vp, _vp]),
    "mclahe_metrics": (C.c_int, [C.c_int32, _vp, _vp, _vp, _i64, C.c_double, _vp]),
    "mclahe_metrics_device": (C.c_int, [C.c_int32, _vp, _vp, _vp, _i64, C.c_double, _vp, _vp]),
    "mclahe_plan_dict_state": (C.c_int, [_vp, _vp, C.POINTER(C.c_int32), _vp]),
    "mclahe_plan_flags": (C.c_int32, [_vp]),
    "mclahe_debug_bin_index_packed": (C.c_int, [_vp, _i64, C.c_double, C.c_double, _i64,
                                                C.c_int32, _vp, _vp]),
    "mclahe_launch_count": (C.c_int64, []),
    "mclahe_last_error": (C.c_char_p, []),
    "mclahe_version": (C.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def build(quiet: bool = True, jobs: int = 8) -> str:
    """Compile libmclahe_gpu.so for sm_100a with nvcc (csrc/Makefile)."""
    if shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"):
        raise NativeUnavailable("nvcc not found; cannot build libmclahe_gpu.so")
    env = dict(os.environ)
    env["PATH"] = env.get("PATH", "") + ":/usr/local/cuda/bin"
    kw = dict(stdout=subprocess.PIPE, stderr=subprocess.STDOUT) if quiet else {}
    r = subprocess.run(["make", "-s", "-C", CSRC, f"-j{jobs}"], env=env, **kw)
    if r.returncode != 0:
        out = r.stdout.decode(errors="replace") if quiet and r.stdout else ""
        raise NativeUnavailable(f"building libmclahe_gpu.so failed:\n{out[-4000:]}")
    return LIB_PATH


def lib() -> C.CDLL:
    """Loads the library (building it first if absent). Raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            build()
        try:
            L = C.CDLL(LIB_PATH)
        except OSError as e:
            raise NativeUnavailable(f"cannot load {LIB_PATH}: {e}") from e
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
        return L


def last_error() -> str:
    return lib().mclahe_last_error().decode(errors="replace")


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = last_error()
    if rc == ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == ERR_OOM:
        raise MemoryError(msg)
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise CudaError(f"[{rc}] {msg}")


def make_params(shape, kernel, n_bins: int, clip_limit: float, adaptive: bool,
                dtype: int = F32) -> Params:
    shape, kernel = tuple(int(s) for s in shape), tuple(int(k) for k in kernel)
    p = Params()
    p.rank = len(shape)
    p.adaptive = 1 if adaptive else 0
    p.dtype = dtype
    if not 1 <= len(shape) <= MAX_RANK:
        raise ValidationError(f"rank must be in [1, {MAX_RANK}]")
    if len(kernel) != len(shape):
        # validate_request, src/pipeline.cpp:21-23
        raise ValidationError(f"kernel rank {len(kernel)} does not match image rank {len(shape)}")
    for i, (s, k) in enumerate(zip(shape, kernel)):
        p.shape[i], p.kernel[i] = s, k
    p.n_bins = int(n_bins)
    p.clip_limit = float(clip_limit)
    return p
