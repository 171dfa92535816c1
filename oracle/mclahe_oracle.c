/*
 * oracle/mclahe_oracle.c -- TEST INFRASTRUCTURE ONLY (see mclahe_oracle.h).
 *
 * A deliberately naive, single-threaded restatement of the reference
 * algorithm: it materialises the mirror padding implicitly per padded
 * position and walks every tile in padded coordinates, exactly the order the
 * reference's kernelize + compute_histogram visit them.  Build with
 * -ffp-contract=off (oracle/Makefile) so no FMA changes a rounding.
 */
#include "mclahe_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static void set_err(char* err, int err_len, const char* msg) {
  if (err && err_len > 0) {
    strncpy(err, msg, (size_t)err_len - 1);
    err[err_len - 1] = '\0';
  }
}

/* nd_image.cpp:85-102: total = 2b - 1 - ((s - 1) mod b); before = total/2. */
int orc_pad_plan(int rank, const int64_t* shape, const int64_t* kernel,
                 int64_t* before, int64_t* after) {
  for (int i = 0; i < rank; ++i) {
    const int64_t s = shape[i], b = kernel[i];
    if (b <= 0 || b > s) return 1;
    const int64_t total = 2 * b - 1 - ((s - 1) % b);
    before[i] = total / 2;
    after[i] = (total + 1) / 2;
  }
  return 0;
}

/* nd_image.cpp:27-34: fold into [0, 2n) then reflect the upper half. */
int64_t orc_mirror_index(int64_t index, int64_t extent) {
  const int64_t period = 2 * extent;
  int64_t m = index % period;
  if (m < 0) m += period;
  if (m >= extent) m = period - 1 - m;
  return m;
}

/* histogram.cpp:24-32: floor((v - lo) / (hi - lo) * n), IEEE double, no FMA. */
int64_t orc_bin_index(double value, double lo, double hi, int64_t n_bins) {
  if (!(lo < hi)) return -1;
  const double diff = value - lo;
  const double span = hi - lo;
  const double ratio = diff / span;
  const double scaled = floor(ratio * (double)n_bins);
  if (!(scaled > 0.0)) return 0;
  if (scaled >= (double)n_bins) return n_bins - 1;
  return (int64_t)scaled;
}

/* histogram.cpp:42-55: single-pass cap at T = clip * total and uniform
 * redistribution of the excess; both sums run in bin order. */
void orc_clip_histogram(const double* counts, int64_t n, double clip_limit, double* out) {
  double total = 0.0;
  for (int64_t b = 0; b < n; ++b) total += counts[b];
  const double threshold = clip_limit * total;
  double excess = 0.0;
  for (int64_t b = 0; b < n; ++b) {
    const double over = counts[b] - threshold;
    excess += over > 0.0 ? over : 0.0;
  }
  const double share = excess / (double)n;
  for (int64_t b = 0; b < n; ++b)
    out[b] = (counts[b] < threshold ? counts[b] : threshold) + share;
}

/* histogram.cpp:57-70: running prefix sum, then (v - first) / (last - first);
 * a non-positive span gives the constant 0.5 mapping. */
int orc_normalized_cdf(const double* clipped, int64_t n, double* out) {
  double running = 0.0;
  for (int64_t b = 0; b < n; ++b) {
    running += clipped[b];
    out[b] = running;
  }
  const double first = out[0];
  const double span = out[n - 1] - first;
  if (!(span > 0.0)) {
    for (int64_t b = 0; b < n; ++b) out[b] = 0.5;
    return 1;
  }
  for (int64_t b = 0; b < n; ++b) out[b] = (out[b] - first) / span;
  return 0;
}

typedef struct {
  int rank;
  int64_t shape[ORC_MAX_RANK];
  int64_t kernel[ORC_MAX_RANK];
  int64_t before[ORC_MAX_RANK];
  int64_t grid[ORC_MAX_RANK];
  int64_t stride[ORC_MAX_RANK];
  int64_t tiles;
  int64_t tile_len;
  int64_t voxels;
} geom_t;

static int make_geom(geom_t* g, int rank, const int64_t* shape, const int64_t* kernel) {
  int64_t after[ORC_MAX_RANK];
  if (rank < 1 || rank > ORC_MAX_RANK) return 1;
  g->rank = rank;
  if (orc_pad_plan(rank, shape, kernel, g->before, after)) return 1;
  g->tiles = 1;
  g->tile_len = 1;
  g->voxels = 1;
  for (int i = 0; i < rank; ++i) {
    g->shape[i] = shape[i];
    g->kernel[i] = kernel[i];
    g->grid[i] = (shape[i] + g->before[i] + after[i]) / kernel[i];
    g->tiles *= g->grid[i];
    g->tile_len *= kernel[i];
    g->voxels *= shape[i];
  }
  g->stride[rank - 1] = 1;
  for (int i = rank - 1; i > 0; --i) g->stride[i - 1] = g->stride[i] * shape[i];
  return 0;
}

/* Gathers tile k of the padded image (kernelize, nd_image.cpp:146-187) in
 * row-major order within the block; padded coordinates map to the original
 * through mirror_index (symmetric_pad, nd_image.cpp:104-144). */
static void gather_tile(const geom_t* g, const double* data, int64_t k, double* block) {
  int64_t tcoord[ORC_MAX_RANK], bcoord[ORC_MAX_RANK];
  int64_t rem = k;
  for (int i = g->rank - 1; i >= 0; --i) {
    tcoord[i] = rem % g->grid[i];
    rem /= g->grid[i];
    bcoord[i] = 0;
  }
  for (int64_t e = 0; e < g->tile_len; ++e) {
    int64_t flat = 0;
    for (int i = 0; i < g->rank; ++i) {
      const int64_t padded = tcoord[i] * g->kernel[i] + bcoord[i];
      flat += orc_mirror_index(padded - g->before[i], g->shape[i]) * g->stride[i];
    }
    block[e] = data[flat];
    for (int i = g->rank - 1; i >= 0; --i) {
      if (++bcoord[i] < g->kernel[i]) break;
      bcoord[i] = 0;
    }
  }
}

/* build_mappings (histogram.cpp:72-106) per tile, with the global range of
 * the unpadded data (NdImage::min_max, nd_image.cpp:76-83). */
int orc_tile_stats(const double* data, int rank, const int64_t* shape,
                   const int64_t* kernel, int64_t n_bins, double clip_limit,
                   int adaptive, double* lo_out, double* hi_out, double* counts_out,
                   double* clipped_out, double* lut_out, uint8_t* degen_out) {
  geom_t g;
  if (make_geom(&g, rank, shape, kernel) || n_bins < 2) return 1;
  double glo = data[0], ghi = data[0];
  for (int64_t i = 0; i < g.voxels; ++i) {
    if (data[i] < glo) glo = data[i];
    if (data[i] > ghi) ghi = data[i];
  }
  double* block = (double*)malloc(sizeof(double) * (size_t)g.tile_len);
  double* counts = (double*)malloc(sizeof(double) * (size_t)n_bins);
  double* clipped = (double*)malloc(sizeof(double) * (size_t)n_bins);
  double* lut = (double*)malloc(sizeof(double) * (size_t)n_bins);
  for (int64_t k = 0; k < g.tiles; ++k) {
    gather_tile(&g, data, k, block);
    double lo = glo, hi = ghi;
    if (adaptive) {
      lo = hi = block[0];
      for (int64_t e = 0; e < g.tile_len; ++e) {
        if (block[e] < lo) lo = block[e];
        if (block[e] > hi) hi = block[e];
      }
    }
    int degenerate = !(lo < hi);
    for (int64_t b = 0; b < n_bins; ++b) counts[b] = clipped[b] = 0.0;
    if (!degenerate) {
      for (int64_t e = 0; e < g.tile_len; ++e)
        counts[orc_bin_index(block[e], lo, hi, n_bins)] += 1.0;
      orc_clip_histogram(counts, n_bins, clip_limit, clipped);
      degenerate = orc_normalized_cdf(clipped, n_bins, lut);
    } else {
      for (int64_t b = 0; b < n_bins; ++b) lut[b] = 0.5;
    }
    if (lo_out) lo_out[k] = lo;
    if (hi_out) hi_out[k] = hi;
    if (degen_out) degen_out[k] = (uint8_t)degenerate;
    if (counts_out) memcpy(counts_out + k * n_bins, counts, sizeof(double) * (size_t)n_bins);
    if (clipped_out) memcpy(clipped_out + k * n_bins, clipped, sizeof(double) * (size_t)n_bins);
    if (lut_out) memcpy(lut_out + k * n_bins, lut, sizeof(double) * (size_t)n_bins);
  }
  free(block);
  free(counts);
  free(clipped);
  free(lut);
  return 0;
}

/* interpolation.cpp:7-42: lower = floor((2x - b + 1) / 2b) clamped to
 * [0, g-2]; distances to the lower/upper kernel centres. */
int orc_neighbor_1d(int64_t x, int64_t b, int64_t g, int64_t* lower_out,
                    double* dist_lo, double* dist_hi) {
  const int64_t num = 2 * x - b + 1;
  const int64_t den = 2 * b;
  int64_t lower = num >= 0 ? num / den : -((-num + den - 1) / den);
  if (lower < 0) lower = 0;
  if (lower > g - 2) lower = g - 2;
  const double center = (double)lower * (double)b + ((double)b - 1.0) * 0.5;
  const double d_lo = (double)x - center;
  if (d_lo < 0.0 || d_lo > (double)b) return 1;
  *lower_out = lower;
  *dist_lo = d_lo;
  *dist_hi = (double)b - d_lo;
  return 0;
}

/* interpolation.cpp:44-66: corner c selects dist_lo (upper neighbour) when its
 * bit for dimension j (dimension 0 = most significant) is set. */
void orc_interp_coefficients(int rank, const double* dist_lo, const double* dist_hi,
                             const int64_t* kernel, double* coeff) {
  double denom = 1.0;
  for (int j = 0; j < rank; ++j) denom *= (double)kernel[j];
  const int corners = 1 << rank;
  for (int c = 0; c < corners; ++c) {
    double numer = 1.0;
    for (int j = 0; j < rank; ++j) {
      const int upper = (c >> (rank - 1 - j)) & 1;
      numer *= upper ? dist_lo[j] : dist_hi[j];
    }
    coeff[c] = numer / denom;
  }
}

/* interpolation.cpp:68-86: terms summed in ascending value order, clamped. */
double orc_blend(int corners, const double* coeff, const double* mapped) {
  double terms[1 << ORC_MAX_RANK];
  for (int i = 0; i < corners; ++i) terms[i] = coeff[i] * mapped[i];
  for (int i = 1; i < corners; ++i) { /* insertion sort, ascending */
    const double t = terms[i];
    int j = i - 1;
    while (j >= 0 && terms[j] > t) {
      terms[j + 1] = terms[j];
      --j;
    }
    terms[j + 1] = t;
  }
  double sum = 0.0;
  for (int i = 0; i < corners; ++i) sum += terms[i];
  if (sum < 0.0) sum = 0.0;
  if (sum > 1.0) sum = 1.0;
  return sum;
}

/* pipeline.cpp:19-34 (validate_request) then pipeline.cpp:73-129. */
int orc_mclahe(const double* data, int rank, const int64_t* shape, const int64_t* kernel,
               int64_t n_bins, double clip_limit, int adaptive, double* out,
               char* err, int err_len) {
  char msg[160];
  if (rank < 1 || rank > ORC_MAX_RANK) {
    set_err(err, err_len, "rank must be in [1, 8]");
    return 1;
  }
  for (int i = 0; i < rank; ++i) {
    if (kernel[i] <= 0 || kernel[i] > shape[i]) {
      snprintf(msg, sizeof msg, "kernel size must be in [1, extent] along dimension %d", i);
      set_err(err, err_len, msg);
      return 1;
    }
  }
  if (!(clip_limit > 0.0) || !(clip_limit <= 1.0)) {
    set_err(err, err_len, "clip_limit must be in (0, 1]");
    return 1;
  }
  if (n_bins < 2) {
    set_err(err, err_len, "n_bins must be at least 2");
    return 1;
  }
  geom_t g;
  make_geom(&g, rank, shape, kernel);
  for (int64_t i = 0; i < g.voxels; ++i) {
    if (!isfinite(data[i])) {
      set_err(err, err_len, "image contains non-finite values");
      return 1;
    }
  }
  double* lo = (double*)malloc(sizeof(double) * (size_t)g.tiles);
  double* hi = (double*)malloc(sizeof(double) * (size_t)g.tiles);
  double* lut = (double*)malloc(sizeof(double) * (size_t)(g.tiles * n_bins));
  uint8_t* degen = (uint8_t*)malloc((size_t)g.tiles);
  orc_tile_stats(data, rank, shape, kernel, n_bins, clip_limit, adaptive, lo, hi, NULL,
                 NULL, lut, degen);

  int64_t gstride[ORC_MAX_RANK];
  gstride[rank - 1] = 1;
  for (int i = rank - 1; i > 0; --i) gstride[i - 1] = gstride[i] * g.grid[i];
  const int corners = 1 << rank;
  int64_t coord[ORC_MAX_RANK] = {0};
  for (int64_t flat = 0; flat < g.voxels; ++flat) {
    int64_t lower[ORC_MAX_RANK];
    double dlo[ORC_MAX_RANK], dhi[ORC_MAX_RANK], coeff[1 << ORC_MAX_RANK];
    double mapped[1 << ORC_MAX_RANK];
    for (int j = 0; j < rank; ++j)
      orc_neighbor_1d(coord[j] + g.before[j], g.kernel[j], g.grid[j], &lower[j], &dlo[j],
                      &dhi[j]);
    orc_interp_coefficients(rank, dlo, dhi, kernel, coeff);
    for (int c = 0; c < corners; ++c) {
      int64_t t = 0;
      for (int j = 0; j < rank; ++j) t += (lower[j] + ((c >> (rank - 1 - j)) & 1)) * gstride[j];
      /* apply_mapping, histogram.cpp:108-111 */
      mapped[c] = degen[t] ? 0.5 : lut[t * n_bins + orc_bin_index(data[flat], lo[t], hi[t], n_bins)];
    }
    out[flat] = orc_blend(corners, coeff, mapped);
    for (int j = rank - 1; j >= 0; --j) {
      if (++coord[j] < shape[j]) break;
      coord[j] = 0;
    }
  }
  free(lo);
  free(hi);
  free(lut);
  free(degen);
  return 0;
}
