/*
 * oracle/mclahe_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference MCLAHE algorithm, used as the parity
 * checker for the CUDA path and as the scalar CPU baseline ("port").  Nothing
 * in the product (paper_1906_11355_b200/) may link or call this; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg do.
 *
 * Pinned against: the reference library compiled from /root/reference
 * (oracle/_ref, see oracle/Makefile) on golden vectors in tests/golden/, and
 * the SPEC.md known-answer examples (tests/test_oracle.py).
 *
 * Every function cites the reference file:line it restates; paths are relative
 * to /root/reference/proj/core/.
 */
#ifndef MCLAHE_ORACLE_H
#define MCLAHE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_RANK 8

/* src/nd_image.cpp:85-102 (compute_pad_plan).  Returns 0, or 1 on bad input. */
int orc_pad_plan(int rank, const int64_t* shape, const int64_t* kernel,
                 int64_t* before, int64_t* after);

/* src/nd_image.cpp:27-34 (mirror_index), edge-including reflection. */
int64_t orc_mirror_index(int64_t index, int64_t extent);

/* src/histogram.cpp:24-32 (bin_index).  Returns -1 for a degenerate range. */
int64_t orc_bin_index(double value, double lo, double hi, int64_t n_bins);

/* src/histogram.cpp:42-55 (clip_histogram). */
void orc_clip_histogram(const double* counts, int64_t n, double clip_limit, double* out);

/* src/histogram.cpp:57-70 (normalized_cdf).  Returns the degenerate flag. */
int orc_normalized_cdf(const double* clipped, int64_t n, double* out);

/* Per-tile intermediates of build_mappings (src/histogram.cpp:72-106) over the
 * materialised padded/kernelized grid (src/nd_image.cpp:104-187).  Arrays are
 * tile-major in row-major grid order: counts/clipped/lut are [T][n_bins],
 * lo/hi/degenerate are [T].  Degenerate-range tiles get zero counts/clipped
 * (the reference builds no histogram for them) and an all-0.5 LUT.  Any
 * output pointer may be NULL.  Returns 0, or 1 on invalid geometry. */
int orc_tile_stats(const double* data, int rank, const int64_t* shape,
                   const int64_t* kernel, int64_t n_bins, double clip_limit,
                   int adaptive, double* lo, double* hi, double* counts,
                   double* clipped, double* lut, uint8_t* degenerate);

/* src/interpolation.cpp:7-42 (neighbor_kernels) for one padded coordinate
 * along one dimension.  Returns 0, or 1 if outside the interpolation span. */
int orc_neighbor_1d(int64_t x_padded, int64_t b, int64_t g, int64_t* lower,
                    double* dist_lo, double* dist_hi);

/* src/interpolation.cpp:44-66 (interp_coefficients); coeff has 2^rank entries. */
void orc_interp_coefficients(int rank, const double* dist_lo, const double* dist_hi,
                             const int64_t* kernel, double* coeff);

/* src/interpolation.cpp:68-86 (transform_pixel) given the per-corner mapped
 * values (apply_mapping results). */
double orc_blend(int corners, const double* coeff, const double* mapped);

/* src/pipeline.cpp:73-129 (mclahe).  out has prod(shape) doubles.  Returns 0,
 * or 1 with a message in err (the reference ValidationError text). */
int orc_mclahe(const double* data, int rank, const int64_t* shape, const int64_t* kernel,
               int64_t n_bins, double clip_limit, int adaptive, double* out,
               char* err, int err_len);

#ifdef __cplusplus
}
#endif

#endif /* MCLAHE_ORACLE_H */
