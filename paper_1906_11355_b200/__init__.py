"""B200-native MCLAHE (arXiv 1906.11355) hot path.

Drop-in for the reference's ``mclahe::mclahe`` entry point: four passes
(range, per-tile histograms over the virtually padded kernel grid, bit-exact
clip/CDF/LUT, 2^D-corner multilinear blend) as sm_100a kernels behind a C ABI
(``include/mclahe_gpu.h``), with a slab decomposition over GPUs
(``slabs.py``).
"""
from ._native import NativeUnavailable, ValidationError  # noqa: F401
from .api import (EnhanceParams, KernelSpec, McLaheRequest, PhaseTimings, Plan,  # noqa: F401
                  RangeMode, bin_index_device, enhance, launch_count, mclahe, mclahe_framewise,
                  normalize_to_unit, GaussianSpec, MedianSpec, MetricsReport, gaussian_filter,
                  median_filter, compute_metrics, mse, psnr, rms_contrast, shannon_entropy,
                  mclahe_multi, multi_cuts)

__all__ = ["EnhanceParams", "KernelSpec", "McLaheRequest", "PhaseTimings", "Plan", "RangeMode",
           "ValidationError", "NativeUnavailable", "mclahe", "enhance", "bin_index_device",
           "launch_count", "mclahe_framewise", "normalize_to_unit", "GaussianSpec", "MedianSpec",
           "MetricsReport", "gaussian_filter", "median_filter", "compute_metrics", "mse", "psnr",
           "rms_contrast", "shannon_entropy", "mclahe_multi", "multi_cuts"]
