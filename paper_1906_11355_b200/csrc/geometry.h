// geometry.h -- padding / tiling / cell arithmetic shared by host planning and
// the sm_100a kernels.  Everything here is index arithmetic on the ORIGINAL
// (unpadded) coordinates: the reference materialises the mirror-padded image
// (symmetric_pad, src/nd_image.cpp:104-144) and a block-major copy of it
// (kernelize, src/nd_image.cpp:146-187); we never do -- a tile is addressed as
// its "support" box in the original data with a small integer multiplicity per
// voxel (how many padded positions of the tile mirror onto that voxel).
#pragma once

#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define MG_HD __host__ __device__ __forceinline__
#else
#define MG_HD inline
#endif

namespace mg {

constexpr int kMaxRank = 8;

// Monotone signed key of a double, so integer MAX reductions (atomics, NCCL)
// compute float min/max exactly.  Stored as ~key(lo) and key(hi).
MG_HD int64_t okey(double x) {
  int64_t i;
#ifdef __CUDA_ARCH__
  i = __double_as_longlong(x);
#else
  std::memcpy(&i, &x, sizeof i);
#endif
  return i >= 0 ? i : (i ^ INT64_MAX);
}

MG_HD double okey_decode(int64_t k) {
  const int64_t i = k >= 0 ? k : (k ^ INT64_MAX);
#ifdef __CUDA_ARCH__
  return __longlong_as_double(i);
#else
  double x;
  std::memcpy(&x, &i, sizeof x);
  return x;
#endif
}

// Per-dimension geometry (compute_pad_plan, src/nd_image.cpp:85-102).
struct Dim {
  int64_t s, b, before, after, g;
};

MG_HD Dim make_dim(int64_t s, int64_t b) {
  Dim d;
  d.s = s;
  d.b = b;
  const int64_t total = 2 * b - 1 - ((s - 1) % b);
  d.before = total / 2;
  d.after = (total + 1) / 2;
  d.g = (s + total) / b;
  return d;
}

// The padded positions of tile t along one dimension, u = o - before for o in
// [t*b, t*b + b), split by the edge-including mirror (mirror_index,
// src/nd_image.cpp:27-34) into three original-coordinate intervals:
//   identity [id_a, id_e), reflected-below [lo_a, lo_e), reflected-above
//   [hi_a, hi_e).  The multiplicity of original x in the tile is the number of
// intervals containing it (0..3); their union is one contiguous support.
struct TileParts {
  int64_t id_a, id_e, lo_a, lo_e, hi_a, hi_e;

  MG_HD int weight(int64_t x) const {
    return (x >= id_a && x < id_e) + (x >= lo_a && x < lo_e) + (x >= hi_a && x < hi_e);
  }
  MG_HD int64_t support_begin() const {
    int64_t a = INT64_MAX;
    if (id_a < id_e && id_a < a) a = id_a;
    if (lo_a < lo_e && lo_a < a) a = lo_a;
    if (hi_a < hi_e && hi_a < a) a = hi_a;
    return a;
  }
  MG_HD int64_t support_end() const {
    int64_t e = INT64_MIN;
    if (id_a < id_e && id_e > e) e = id_e;
    if (lo_a < lo_e && lo_e > e) e = lo_e;
    if (hi_a < hi_e && hi_e > e) e = hi_e;
    return e;
  }
};

MG_HD TileParts tile_parts(const Dim& d, int64_t t) {
  TileParts p;
  const int64_t u0 = t * d.b - d.before, u1 = u0 + d.b;
  p.id_a = u0 > 0 ? u0 : 0;
  p.id_e = u1 < d.s ? u1 : d.s;
  if (p.id_e < p.id_a) p.id_e = p.id_a;
  if (u0 < 0) {  // u in [u0, min(u1,0)) -> x = -1 - u
    p.lo_a = -(u1 < 0 ? u1 : 0);
    p.lo_e = -u0;
  } else {
    p.lo_a = p.lo_e = 0;
  }
  if (u1 > d.s) {  // u in [max(u0,s), u1) -> x = 2s - 1 - u
    p.hi_a = 2 * d.s - u1;
    p.hi_e = 2 * d.s - (u0 > d.s ? u0 : d.s);
  } else {
    p.hi_a = p.hi_e = 0;
  }
  return p;
}

// The (up to 3, merged) tiles an original voxel x contributes to along one
// dimension, with multiplicities.  Returns the count.
MG_HD int voxel_tiles(const Dim& d, int64_t x, int64_t* tiles, int* weights) {
  int n = 0;
  int64_t cand[3];
  int nc = 0;
  cand[nc++] = (x + d.before) / d.b;
  if (x < d.before) cand[nc++] = (d.before - 1 - x) / d.b;
  if (x >= d.s - d.after) cand[nc++] = (d.before + 2 * d.s - 1 - x) / d.b;
  for (int i = 0; i < nc; ++i) {
    int j = 0;
    while (j < n && tiles[j] != cand[i]) ++j;
    if (j == n) {
      tiles[n] = cand[i];
      weights[n] = 1;
      ++n;
    } else {
      ++weights[j];
    }
  }
  return n;
}

// Interpolation cells (neighbor_kernels, src/interpolation.cpp:24-35): the
// lower neighbour of padded p = x + before is
//   clamp(floor((2p - b + 1) / 2b), 0, g - 2).
MG_HD int64_t cell_of(const Dim& d, int64_t x) {
  const int64_t num = 2 * (x + d.before) - d.b + 1;
  const int64_t den = 2 * d.b;
  int64_t lower = num >= 0 ? num / den : -((-num + den - 1) / den);
  if (lower < 0) lower = 0;
  if (lower > d.g - 2) lower = d.g - 2;
  return lower;
}

// First padded coordinate whose unclamped lower neighbour is >= c.
MG_HD int64_t cell_pmin(const Dim& d, int64_t c) { return (2 * d.b * c + d.b) / 2; }

// Original-coordinate range [a, e) of cell c (may be empty).
MG_HD void cell_range(const Dim& d, int64_t c, int64_t* a, int64_t* e) {
  int64_t lo = c == 0 ? INT64_MIN / 4 : cell_pmin(d, c) - d.before;
  int64_t hi = c == d.g - 2 ? INT64_MAX / 4 : cell_pmin(d, c + 1) - d.before;
  if (lo < 0) lo = 0;
  if (hi > d.s) hi = d.s;
  if (hi < lo) hi = lo;
  *a = lo;
  *e = hi;
}

// Twice the distance from padded p = x + before to the centre of its lower
// neighbour c: 2*d_lo = 2p - 2cb - b + 1 (an exact integer; d_lo is a
// half-integer, src/interpolation.cpp:31-35).
MG_HD int64_t twice_dlo(const Dim& d, int64_t x, int64_t c) {
  return 2 * (x + d.before) - 2 * c * d.b - d.b + 1;
}

// Blend tile block of the NB-specialised K4 kernel (k_pencil.cuh):
// {lo, c_lo, c_hi, c} (one LDS.128; c_lo / c_hi bracket c, see
// binning.cuh: bin_window), the edge table with one pad word after every 32
// entries (entry j at j + j/32, a pad repeats the entry before it), then the
// LUT unpadded (the blend's fast path addresses it straight from the floor
// bits).  Blocks are 16-byte aligned.
struct NbBlock {
  static constexpr MG_HD int pad(int j) { return j + (j >> 5); }
  static constexpr MG_HD int th_words(int n) { return pad(n) + 1; }
  static constexpr MG_HD int lut_words(int n) { return n; }
  static constexpr MG_HD int th_off(int) { return 4; }
  static constexpr MG_HD int lut_off(int n) { return 4 + th_words(n); }
  static constexpr MG_HD int words(int n) { return (lut_off(n) + lut_words(n) + 3) & ~3; }
  // table entry stored at padded position q (pads repeat the entry before)
  static constexpr MG_HD int src(int q) { return 32 * (q / 33) + (q % 33 < 31 ? q % 33 : 31); }
};

}  // namespace mg
