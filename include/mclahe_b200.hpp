// include/mclahe_b200.hpp -- umbrella header of the C++ drop-in.
//
// The reference's public headers are rebuilt under include/mclahe/ with the
// same names and declarations (nd_image, histogram, interpolation, pipeline,
// filters, metrics, npy, parallel), so a reference caller keeps
//
//     #include "mclahe/pipeline.hpp"
//     mclahe::NdImage out = mclahe::mclahe(request, &timings);
//
// and only re-links: -lmclahe_cpp -lmclahe_gpu instead of libmclahe.a.  This
// header just includes all of them.  Compute runs on the GPU through the C
// ABI in mclahe_gpu.h: float64 images whose values are all float32-
// representable take the float32 pencil kernels (bit-identical bins, since
// f32 -> f64 is exact), others the exact float64 path.  Errors:
// ValidationError with the reference's messages; CUDA failures as
// std::runtime_error.
#pragma once

#include "mclahe/filters.hpp"
#include "mclahe/histogram.hpp"
#include "mclahe/interpolation.hpp"
#include "mclahe/metrics.hpp"
#include "mclahe/nd_image.hpp"
#include "mclahe/npy.hpp"
#include "mclahe/parallel.hpp"
#include "mclahe/pipeline.hpp"
