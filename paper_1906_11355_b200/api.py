"""Python host mirror of the reference's MCLAHE interface, over the C ABI.

Reference interface (paths relative to /root/reference/proj/core/):

* ``RangeMode`` / ``EnhanceParams``     include/mclahe/histogram.hpp:13-21
* ``KernelSpec``                        include/mclahe/nd_image.hpp:81-83
* ``McLaheRequest`` / ``PhaseTimings``  include/mclahe/pipeline.hpp:12-24
* ``mclahe(request, timings)``          include/mclahe/pipeline.hpp:30
* ``ValidationError``                   include/mclahe/nd_image.hpp:19-22

Same names, argument meaning and error behaviour; the compute is the sm_100a
library (``libmclahe_gpu.so``).  Host ``numpy`` images go through the
one-shot ``mclahe_gpu_run`` (H2D, four passes, D2H); CUDA ``torch`` tensors go
through a cached device-resident :class:`Plan` on the current stream.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import ValidationError  # noqa: F401  (re-export)


class RangeMode(enum.IntEnum):
    Global = 0
    Adaptive = 1


@dataclass
class EnhanceParams:
    clip_limit: float = 1.0
    n_bins: int = 256
    range_mode: RangeMode = RangeMode.Global


@dataclass
class KernelSpec:
    sizes: tuple = ()


@dataclass
class McLaheRequest:
    image: object = None
    kernel: KernelSpec = field(default_factory=KernelSpec)
    params: EnhanceParams = field(default_factory=EnhanceParams)
    threads: int = 0  # accepted for interface parity; the GPU path ignores it


@dataclass
class PhaseTimings:
    pad_s: float = 0.0
    histograms_s: float = 0.0
    interpolation_s: float = 0.0


def _is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _dtype_code(dt) -> int:
    if _is_torch_dtype(dt):
        import torch
        return N.F64 if dt == torch.float64 else N.F32
    return N.F64 if np.dtype(dt) == np.float64 else N.F32


def _is_torch_dtype(dt) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(dt, torch.dtype)


def _stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class Plan:
    """A device-resident plan for one slab (rows [row_begin, row_end) along
    dim 0) of a volume.  Wraps mclahe_plan_* and the pass entry points."""

    def __init__(self, shape, kernel, n_bins=256, clip_limit=1.0, adaptive=False,
                 dtype=N.F32, row_begin: int = 0, row_end: int | None = None):
        self.params = N.make_params(shape, kernel, n_bins, clip_limit, adaptive, dtype)
        self.shape = tuple(int(s) for s in shape)
        self.kernel = tuple(int(k) for k in kernel)
        self.n_bins, self.clip_limit, self.adaptive, self.dtype = int(n_bins), float(clip_limit), \
            bool(adaptive), dtype
        row_end = self.shape[0] if row_end is None else int(row_end)
        L = N.lib()
        h = C.c_void_p()
        N.check(L.mclahe_plan_create(C.byref(self.params), int(row_begin), row_end, C.byref(h)))
        self._h = h
        info = N.PlanInfo()
        N.check(L.mclahe_plan_get_info(h, C.byref(info)))
        self.info = info
        self.row_begin, self.row_end = int(row_begin), row_end

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.lib().mclahe_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    # ---- geometry ----
    @property
    def workspace_bytes(self) -> int:
        return int(self.info.workspace_bytes)

    @property
    def window_tiles(self) -> int:
        i = self.info
        return int((i.tile_row_end - i.tile_row_begin) * i.tiles_per_row)

    @property
    def local_shape(self) -> tuple:
        return (self.row_end - self.row_begin,) + self.shape[1:]

    def new_workspace(self, device=None):
        import torch
        return torch.empty(self.workspace_bytes, dtype=torch.uint8, device=device or "cuda")

    # workspace views (torch), for the slab exchange layer
    def range_view(self, ws):
        import torch
        o = self.info.off_range
        return ws[o:o + 32].view(torch.int64)

    def tile_range_view(self, ws):
        import torch
        o = self.info.off_tile_range
        return ws[o:o + 16 * self.window_tiles].view(torch.int64).view(-1, 2)

    def counts_view(self, ws):
        import torch
        o = self.info.off_counts
        n = self.window_tiles * self.n_bins
        return ws[o:o + 4 * n].view(torch.int32).view(self.window_tiles, self.n_bins)

    def lut_view(self, ws):
        import torch
        o = self.info.off_lut
        n = self.window_tiles * self.n_bins
        return ws[o:o + 4 * n].view(torch.float32).view(self.window_tiles, self.n_bins)

    # ---- passes ----
    def _ptr(self, t) -> int:
        return int(t.data_ptr())

    @staticmethod
    def _same_device(*ts):
        """Buffers of one pass must live on one device (kernels and TMA maps
        address that device's memory); returns a context making it current."""
        import torch
        devs = {t.device for t in ts if t is not None}
        if len(devs) != 1 or next(iter(devs)).type != "cuda":
            raise ValidationError(f"pass buffers must share one CUDA device, got {sorted(map(str, devs))}")
        return torch.cuda.device(next(iter(devs)))

    def reset(self, ws, stream=None):
        N.check(N.lib().mclahe_pass_reset(self._h, self._ptr(ws), _stream_handle(stream)))

    def range(self, x, ws, stream=None):
        with self._same_device(x, ws):
            N.check(N.lib().mclahe_pass_range(self._h, self._ptr(x), self._ptr(ws),
                                              _stream_handle(stream)))

    def make_params(self, ws, stream=None):
        N.check(N.lib().mclahe_pass_params(self._h, self._ptr(ws), _stream_handle(stream)))

    def histograms(self, x, ws, stream=None):
        with self._same_device(x, ws):
            N.check(N.lib().mclahe_pass_histograms(self._h, self._ptr(x), self._ptr(ws),
                                                   _stream_handle(stream)))

    def mappings(self, ws, stream=None, debug: dict | None = None):
        dbg = None
        if debug is not None:
            dbg = N.Debug()
            for k in ("lo", "hi", "counts", "clipped", "lut", "degenerate"):
                t = debug.get(k)
                setattr(dbg, k, self._ptr(t) if t is not None else None)
        N.check(N.lib().mclahe_pass_mappings(self._h, self._ptr(ws),
                                             C.byref(dbg) if dbg is not None else None,
                                             _stream_handle(stream)))

    def interpolate(self, x, out, ws, stream=None):
        with self._same_device(x, out, ws):
            N.check(N.lib().mclahe_pass_interpolate(self._h, self._ptr(x), self._ptr(out),
                                                    self._ptr(ws), _stream_handle(stream)))

    def enqueue(self, x, out, ws, stream=None):
        with self._same_device(x, out, ws):
            N.check(N.lib().mclahe_plan_enqueue(self._h, self._ptr(x), self._ptr(out), self._ptr(ws),
                                                _stream_handle(stream)))

    def check(self, ws, stream=None):
        N.check(N.lib().mclahe_plan_check(self._h, self._ptr(ws), _stream_handle(stream)))

    @property
    def flags(self) -> dict:
        """Kernels the plan runs (valid once a pass has run on a device):
        ``fused_k2`` (ranges + counts in one kernel, one HBM read), ``pencil_hist``,
        ``pencil_blend``, ``dict`` (value dictionary armed), ``folded`` (folded-pair blend)."""
        f = int(N.lib().mclahe_plan_flags(self._h))
        return dict(fused_k2=bool(f & 1), pencil_hist=bool(f & 2), pencil_blend=bool(f & 4),
                    dict=bool(f & 8), folded=bool(f & 16))

    def dict_state(self, ws, stream=None) -> dict:
        """Value-dictionary state after a run on ``ws``: ``used`` (the blend took
        the dictionary path), ``folded`` (through the folded-pair kernel
        k_interp_mdict), ``values`` (distinct values collected), ``capacity``
        (0 when the plan never arms it), ``affine`` (affine-cell lookup), ``direct``
        (the affine cell is the value's index: values numbered by cell)."""
        st = (C.c_int32 * 4)()
        N.check(N.lib().mclahe_plan_dict_state(self._h, self._ptr(ws), st, _stream_handle(stream)))
        return dict(used=st[0] == 1 or (st[0] == 2 and st[2] > 0), folded=st[0] == 2,
                    values=int(st[1]), capacity=int(st[2]), affine=bool(st[3]),
                    direct=st[3] == 2)

    def tile_stats(self, x, stream=None) -> dict:
        """Runs passes 1-3 and returns the per-tile intermediates of the
        workspace window (debug arrays of build_mappings, histogram.cpp:72-106)."""
        import torch
        ws = self.new_workspace(x.device)
        T, n = self.window_tiles, self.n_bins
        dev = x.device
        dbg = dict(lo=torch.empty(T, dtype=torch.float64, device=dev),
                   hi=torch.empty(T, dtype=torch.float64, device=dev),
                   counts=torch.empty(T, n, dtype=torch.int32, device=dev),
                   clipped=torch.empty(T, n, dtype=torch.float64, device=dev),
                   lut=torch.empty(T, n, dtype=torch.float64, device=dev),
                   degenerate=torch.empty(T, dtype=torch.uint8, device=dev))
        self.reset(ws, stream)
        self.range(x, ws, stream)
        self.make_params(ws, stream)
        self.histograms(x, ws, stream)
        self.mappings(ws, stream, debug=dbg)
        self.check(ws, stream)
        out = {k: v.cpu().numpy() for k, v in dbg.items()}
        out["degenerate"] = out["degenerate"].astype(bool)
        out["lut32"] = self.lut_view(ws).cpu().numpy()
        return out


_PLAN_CACHE: dict = {}


def _cached_plan(shape, kernel, n_bins, clip_limit, adaptive, dtype) -> Plan:
    import torch
    key = (tuple(shape), tuple(kernel), int(n_bins), float(clip_limit), bool(adaptive), dtype,
           torch.cuda.current_device())
    p = _PLAN_CACHE.get(key)
    if p is None:
        if len(_PLAN_CACHE) > 32:
            _PLAN_CACHE.clear()
        p = _PLAN_CACHE[key] = Plan(shape, kernel, n_bins, clip_limit, adaptive, dtype)
    return p


def _request_parts(request: McLaheRequest):
    sizes = request.kernel.sizes if isinstance(request.kernel, KernelSpec) else request.kernel
    p = request.params
    return (tuple(int(s) for s in sizes), int(p.n_bins), float(p.clip_limit),
            RangeMode(p.range_mode) == RangeMode.Adaptive)


def mclahe(request: McLaheRequest, timings: PhaseTimings | None = None,
           max_device_bytes: int | None = None):
    """mclahe::mclahe (include/mclahe/pipeline.hpp:30, src/pipeline.cpp:73-129).

    numpy image -> numpy result (float32 for float32 input, float64 for every
    other real dtype, as the reference computes on doubles); CUDA torch
    tensor -> CUDA torch tensor on the current stream.  Raises
    ValidationError with the reference's messages.

    Host volumes larger than the free device memory stream through a ring of
    chunk slots (out of core, mclahe_gpu_run_out_of_core); ``max_device_bytes``
    caps the device memory the call may use (numpy input only)."""
    kernel, n_bins, clip, adaptive = _request_parts(request)
    img = request.image
    if _is_torch(img):
        return _mclahe_device(img, kernel, n_bins, clip, adaptive, timings)
    x = np.asarray(img)
    if x.dtype != np.float32:
        x = x.astype(np.float64)
    x = np.ascontiguousarray(x)
    params = N.make_params(x.shape, kernel, n_bins, clip, adaptive, _dtype_code(x.dtype))
    out = np.empty_like(x)
    t = N.Timings()
    if max_device_bytes is not None:
        N.check(N.lib().mclahe_gpu_run_out_of_core(C.byref(params), x.ctypes.data, out.ctypes.data,
                                                   int(max_device_bytes), C.byref(t)))
    else:
        N.check(N.lib().mclahe_gpu_run(C.byref(params), x.ctypes.data, out.ctypes.data, C.byref(t)))
    if timings is not None:
        timings.pad_s += t.pad_s
        timings.histograms_s += t.histograms_s
        timings.interpolation_s += t.interpolation_s
    return out


def _mclahe_device(x, kernel, n_bins, clip, adaptive, timings=None):
    import torch
    if not x.is_cuda:
        raise ValidationError("torch input must be a CUDA tensor (use numpy for host data)")
    if x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float64)
    x = x.contiguous()
    # plans, TMA maps and launches belong to the tensor's device, which need
    # not be the current one
    with torch.cuda.device(x.device):
        plan = _cached_plan(x.shape, kernel, n_bins, clip, adaptive, _dtype_code(x.dtype))
        ws = plan.new_workspace(x.device)
        out = torch.empty_like(x)
        plan.enqueue(x, out, ws)
        plan.check(ws)
    return out


def normalize_to_unit(image):
    """normalize_to_unit (src/pipeline.cpp:155-165): affine map of [min, max]
    onto [0, 1] in float64; a constant image maps to 0.5."""
    x = np.asarray(image, dtype=np.float64)
    if not np.all(np.isfinite(x)):
        raise ValidationError("image contains non-finite values")
    lo, hi = float(x.min()), float(x.max())
    if not hi > lo:
        return np.full_like(x, 0.5)
    return (x - lo) / (hi - lo)


def mclahe_framewise(image, frame_axis: int, kernel: KernelSpec, params: EnhanceParams,
                     threads: int = 0, renormalize_slices: bool = False,
                     timings: PhaseTimings | None = None):
    """mclahe_framewise (include/mclahe/pipeline.hpp:37-40, src/pipeline.cpp:131-153):
    mclahe on every slice along frame_axis, batched into one GPU run
    (mclahe_gpu_run_framewise).  numpy in -> numpy out; ``threads`` is
    accepted and ignored.  renormalize_slices maps each slice onto [0, 1]
    (float64) first, as the reference does."""
    x = np.asarray(image)
    if x.ndim < 2:
        raise ValidationError("framewise mode needs rank >= 2")
    if not 0 <= frame_axis < x.ndim:
        raise ValidationError(f"frame axis {frame_axis} out of range for rank {x.ndim}")
    ks = tuple(int(k) for k in kernel.sizes)
    if len(ks) != x.ndim - 1:
        raise ValidationError("framewise kernel rank must be image rank - 1")
    if renormalize_slices:
        x = np.stack([normalize_to_unit(np.take(x, f, axis=frame_axis))
                      for f in range(x.shape[frame_axis])], axis=frame_axis)
    if x.dtype != np.float32:
        x = x.astype(np.float64)
    x = np.ascontiguousarray(x)
    adaptive = params.range_mode == RangeMode.Adaptive
    full_kernel = ks[:frame_axis] + (1,) + ks[frame_axis:]  # slot the ABI ignores
    p = N.make_params(x.shape, full_kernel, params.n_bins, params.clip_limit, adaptive,
                      _dtype_code(x.dtype))
    for i, k in enumerate(ks):  # the ABI takes the slice kernel, frame axis removed
        p.kernel[i] = k
    out = np.empty_like(x)
    t = N.Timings()
    N.check(N.lib().mclahe_gpu_run_framewise(C.byref(p), int(frame_axis), x.ctypes.data,
                                             out.ctypes.data, C.byref(t)))
    if timings is not None:
        timings.pad_s += t.pad_s
        timings.histograms_s += t.histograms_s
        timings.interpolation_s += t.interpolation_s
    return out


# ---- the steps either side of the path: prefilters and metrics (float64) ----

@dataclass
class GaussianSpec:
    """filters.hpp:11-15: sigma per dimension in pixels (0 skips the axis)."""
    sigmas: tuple
    truncate: float = 4.0


@dataclass
class MedianSpec:
    """filters.hpp:17-21: window extents per dimension."""
    window: tuple


@dataclass
class MetricsReport:
    """metrics.hpp:9-17."""
    mse: float = 0.0
    psnr_db: float = 0.0
    std: float = 0.0
    entropy_bits: float = 0.0
    n_bins_used: int = 0


def _shape_arr(shape):
    arr = (C.c_int64 * max(1, len(shape)))(*[int(v) for v in shape])
    return arr


def _filter_call(image, host_fn, dev_fn, *args):
    """numpy -> host ABI -> numpy; CUDA tensor -> device ABI -> CUDA tensor (f64)."""
    if _is_torch(image):
        import torch
        x = image.to(torch.float64).contiguous()
        out = torch.empty_like(x)
        N.check(dev_fn(x.dim(), _shape_arr(x.shape), *args, x.data_ptr(), out.data_ptr(),
                       _stream_handle()))
        return out
    x = np.ascontiguousarray(np.asarray(image, dtype=np.float64))
    out = np.empty_like(x)
    N.check(host_fn(x.ndim, _shape_arr(x.shape), *args, x.ctypes.data, out.ctypes.data))
    return out


def gaussian_filter(image, spec: GaussianSpec):
    """gaussian_filter (filters.hpp:24-25, filters.cpp:82-96) on the GPU, float64."""
    x = image
    rank = x.dim() if _is_torch(x) else np.ndim(x)
    if len(spec.sigmas) != rank:
        raise ValidationError("sigma count does not match image rank")
    sg = (C.c_double * max(1, rank))(*[float(v) for v in spec.sigmas])
    L = N.lib()
    return _filter_call(x, L.mclahe_gaussian_filter, L.mclahe_gaussian_filter_device, sg,
                        C.c_double(float(spec.truncate)))


def median_filter(image, spec: MedianSpec):
    """median_filter (filters.hpp:30-32, filters.cpp:98-142) on the GPU, float64."""
    x = image
    rank = x.dim() if _is_torch(x) else np.ndim(x)
    if len(spec.window) != rank:
        raise ValidationError("window rank does not match image rank")
    win = (C.c_int64 * max(1, rank))(*[int(v) for v in spec.window])
    L = N.lib()
    return _filter_call(x, L.mclahe_median_filter, L.mclahe_median_filter_device, win)


def compute_metrics(a, b=None, n_bins: int = 256, peak: float = 1.0) -> MetricsReport:
    """compute_metrics (metrics.hpp:35-36): std / entropy of a, mse / psnr of (a, b)."""
    L = N.lib()
    rep = N.Metrics()
    if _is_torch(a):
        import torch
        xa = a.to(torch.float64).contiguous()
        xb = None if b is None else b.to(torch.float64).contiguous()
        if xb is not None and tuple(xb.shape) != tuple(xa.shape):
            raise ValidationError("mse operands differ in shape")
        N.check(L.mclahe_metrics_device(xa.dim(), _shape_arr(xa.shape), xa.data_ptr(),
                                        None if xb is None else xb.data_ptr(), int(n_bins),
                                        float(peak), C.byref(rep), _stream_handle()))
    else:
        xa = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
        xb = None if b is None else np.ascontiguousarray(np.asarray(b, dtype=np.float64))
        if xb is not None and xb.shape != xa.shape:
            raise ValidationError("mse operands differ in shape")
        N.check(L.mclahe_metrics(xa.ndim, _shape_arr(xa.shape), xa.ctypes.data,
                                 None if xb is None else xb.ctypes.data, int(n_bins),
                                 float(peak), C.byref(rep)))
    return MetricsReport(rep.mse, rep.psnr_db, rep.std, rep.entropy_bits, int(rep.n_bins_used))


def mse(a, b) -> float:
    """metrics.hpp:19-20."""
    return compute_metrics(a, b).mse


def psnr(a, b, peak: float = 1.0) -> float:
    """metrics.hpp:22-23."""
    return compute_metrics(a, b, peak=peak).psnr_db


def rms_contrast(a) -> float:
    """metrics.hpp:25-26."""
    return compute_metrics(a).std


def shannon_entropy(a, n_bins: int = 256) -> float:
    """metrics.hpp:28-30."""
    return compute_metrics(a, n_bins=n_bins).entropy_bits


def enhance(image, kernel_size, n_bins: int = 256, clip_limit: float = 1.0,
            adaptive_hist_range: bool = False, max_device_bytes: int | None = None):
    """Convenience form with the paper's argument names (data, kernel_size,
    n_bins, clip_limit, adaptive_hist_range)."""
    req = McLaheRequest(image=image, kernel=KernelSpec(tuple(kernel_size)),
                        params=EnhanceParams(clip_limit, n_bins,
                                             RangeMode.Adaptive if adaptive_hist_range
                                             else RangeMode.Global))
    return mclahe(req, max_device_bytes=max_device_bytes)


def multi_cuts(shape, kernel, n_slabs: int, n_bins: int = 256, clip_limit: float = 1.0,
               adaptive: bool = False) -> list:
    """Row boundaries (n_slabs + 1) of the cell-aligned slabs the multi-slab
    run uses along dim 0 (mclahe_multi_cuts; slabs.py slab_cuts' rule)."""
    params = N.make_params(tuple(shape), tuple(kernel), n_bins, clip_limit, adaptive, N.F32)
    cuts = (C.c_int64 * (n_slabs + 1))()
    N.check(N.lib().mclahe_multi_cuts(C.byref(params), int(n_slabs), cuts))
    return [int(c) for c in cuts]


def mclahe_multi(image, kernel, n_bins: int = 256, clip_limit: float = 1.0,
                 adaptive: bool = False, devices=(0,), timings: PhaseTimings | None = None):
    """mclahe::mclahe over slabs along dim 0, slab r on devices[r], in one
    process (mclahe_gpu_run_multi / _multi_device).  Devices
    may repeat (logical slabs on one GPU).  numpy in -> numpy out (host
    buffers); a list of CUDA tensors (slab r's rows on devices[r], see
    multi_cuts) -> a list of output slabs.  Bit-identical to mclahe()."""
    devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
    n = len(devices)
    t = N.Timings()
    if isinstance(image, (list, tuple)):
        import torch
        xs = [s.contiguous() for s in image]
        if len(xs) != n:
            raise ValidationError("one input slab per device")
        shape = (sum(int(s.shape[0]) for s in xs),) + tuple(xs[0].shape[1:])
        params = N.make_params(shape, tuple(kernel), n_bins, clip_limit, adaptive,
                               _dtype_code(xs[0].dtype))
        outs = [torch.empty_like(s) for s in xs]
        ins = (C.c_void_p * n)(*[s.data_ptr() for s in xs])
        ous = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
        N.check(N.lib().mclahe_gpu_run_multi_device(C.byref(params), n, devs, ins, ous,
                                                    C.byref(t)))
        result = outs
    else:
        x = np.asarray(image)
        if x.dtype != np.float32:
            x = x.astype(np.float64)
        x = np.ascontiguousarray(x)
        params = N.make_params(x.shape, tuple(kernel), n_bins, clip_limit, adaptive,
                               _dtype_code(x.dtype))
        result = np.empty_like(x)
        N.check(N.lib().mclahe_gpu_run_multi(C.byref(params), n, devs, x.ctypes.data,
                                             result.ctypes.data, C.byref(t)))
    if timings is not None:
        timings.histograms_s += t.histograms_s
        timings.interpolation_s += t.interpolation_s
    return result


def bin_index_device(values, lo: float, hi: float, n_bins: int, variant: int = 0):
    """bin_index (src/histogram.cpp:24-32) of a CUDA tensor through the kernels'
    binning; int32 result (-1 for a degenerate range).  variant 0: the generic
    kernels' guarded routine (f32 or f64); 1 / 2 / 3: the pencil kernels' packed
    histogram / blend-gather / bracketed-floor (NB blend) routines (float32 only)."""
    import torch
    v = values.contiguous()
    out = torch.empty(v.shape, dtype=torch.int32, device=v.device)
    if variant:
        if v.dtype != torch.float32:
            raise ValidationError("packed binning variants take float32 values")
        N.check(N.lib().mclahe_debug_bin_index_packed(v.data_ptr(), v.numel(), float(lo),
                                                      float(hi), int(n_bins), int(variant),
                                                      out.data_ptr(), _stream_handle()))
        return out
    code = N.F64 if v.dtype == torch.float64 else N.F32
    N.check(N.lib().mclahe_debug_bin_index(code, v.data_ptr(), v.numel(), float(lo), float(hi),
                                           int(n_bins), out.data_ptr(), _stream_handle()))
    return out


def launch_count() -> int:
    return int(N.lib().mclahe_launch_count())
