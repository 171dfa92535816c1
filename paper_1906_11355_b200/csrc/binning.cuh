// binning.cuh -- bit-exact bin_index (src/histogram.cpp:24-32) at FP32 speed.
//
// The reference computes  floor(((double)v - lo) / (hi - lo) * n)  in IEEE
// double (divide, then multiply; no FMA) and clamps into [0, n-1].  A double
// divide per voxel per corner does not fit the issue budget of the blend pass,
// and a plain FP32 fused estimate misbins values that sit on (or within a few
// ulp of) a bin edge -- which quantised data does constantly.  So:
//
//   y  = fl32(fl32(v - lo) * c),  c = fl32(n / (hi - lo))
//
// differs from the reference's f64 value q by at most |y| * 1.81e-7 (three
// f32 roundings + O(2^-50)), i.e. by less than tol = 2.5e-7 * n on the only
// interval that matters, y in [0.5, n - 0.5] (outside it the clamp decides the
// bin whatever the rounding).  If frac(y) is further than tol from an integer
// then floor(y) == floor(q) and the fast answer is exact; otherwise (rare) the
// lane recomputes q exactly as the reference does, with __ddiv_rn.  Ranges the
// bound does not cover (c not a normal float, hi - lo overflowing f32, huge n)
// set lim < 0 and always take the exact path.  For f64 data the same scheme
// runs in f64 with tol = 1e-15 * n.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdint>

#include "geometry.h"

namespace mg {

// Per-tile binning parameters.  lim in (0, 0.5): guarded fast path;
// lim < 0: exact path only; lim > 1: degenerate range (no histogram, the
// mapping is the constant 0.5 -- histogram.cpp:95-98).
template <typename T>
struct alignas(4 * sizeof(T)) TileParam {
  T lo, hi, c, lim;
};

MG_HD bool tp_degenerate(float lim) { return lim > 1.0f; }
MG_HD bool tp_degenerate(double lim) { return lim > 1.0; }

// Builds the parameters for range [lo, hi] (exact values of the data type).
MG_HD TileParam<float> make_tile_param_f32(double lo, double hi, int64_t n) {
  TileParam<float> tp;
  tp.lo = static_cast<float>(lo);
  tp.hi = static_cast<float>(hi);
  if (!(lo < hi)) {
    tp.c = 0.0f;
    tp.lim = 2.0f;
    return tp;
  }
  const double c64 = static_cast<double>(n) / (hi - lo);
  const float c = static_cast<float>(c64);
  const float span = tp.hi - tp.lo;  // plain f32 subtraction, no contraction possible
  const bool ok = std::isfinite(c) && c >= FLT_MIN && std::isfinite(span) &&
                  std::isfinite(tp.lo) && std::isfinite(tp.hi) && n <= (int64_t{1} << 20);
  tp.c = ok ? c : 0.0f;
  tp.lim = ok ? 0.5f - static_cast<float>(n) * 2.5e-7f : -1.0f;
  return tp;
}

MG_HD TileParam<double> make_tile_param_f64(double lo, double hi, int64_t n) {
  TileParam<double> tp;
  tp.lo = lo;
  tp.hi = hi;
  if (!(lo < hi)) {
    tp.c = 0.0;
    tp.lim = 2.0;
    return tp;
  }
  const double c = static_cast<double>(n) / (hi - lo);
  const bool ok = std::isfinite(c) && c >= DBL_MIN && n <= (int64_t{1} << 40);
  tp.c = ok ? c : 0.0;
  tp.lim = ok ? 0.5 - static_cast<double>(n) * 1e-15 : -1.0;
  return tp;
}

template <typename T>
MG_HD TileParam<T> make_tile_param(double lo, double hi, int64_t n);
template <>
MG_HD TileParam<float> make_tile_param<float>(double lo, double hi, int64_t n) {
  return make_tile_param_f32(lo, hi, n);
}
template <>
MG_HD TileParam<double> make_tile_param<double>(double lo, double hi, int64_t n) {
  return make_tile_param_f64(lo, hi, n);
}

#ifdef __CUDACC__

// The reference arithmetic, operation for operation (histogram.cpp:27-31).
__device__ __forceinline__ int bin_exact(double v, double lo, double hi, int n) {
  const double scaled = floor(__dmul_rn(__ddiv_rn(__dsub_rn(v, lo), __dsub_rn(hi, lo)),
                                        static_cast<double>(n)));
  if (!(scaled > 0.0)) return 0;
  if (scaled >= static_cast<double>(n)) return n - 1;
  return static_cast<int>(scaled);
}

// nm05 = n - 0.5 (exact in f32 for n < 2^23).  thr = the tile's bin-edge
// table: thr[k] = smallest float whose reference bin is >= k (k in [1, n-1]).
// When y is within tol of an integer k the reference bin is k or k-1 and the
// table decides it with one (L2-resident) load instead of an f64 divide.
__device__ __forceinline__ int bin_of(float v, const TileParam<float>& tp, const float* thr,
                                      int n, float nm05) {
  float y = __fmul_rn(__fsub_rn(v, tp.lo), tp.c);
  y = fminf(fmaxf(y, 0.5f), nm05);
  const float t = __fadd_rd(y, 12582912.0f);  // 1.5 * 2^23: t = floor(y) + M exactly
  const float fr = __fsub_rn(y, __fsub_rn(t, 12582912.0f));
  if (fabsf(__fsub_rn(fr, 0.5f)) < tp.lim) return __float_as_int(t) - 0x4B400000;
  if (tp.lim < 0.0f)
    return bin_exact(static_cast<double>(v), static_cast<double>(tp.lo),
                     static_cast<double>(tp.hi), n);
  const int k = __float2int_rn(y);
  return v >= thr[k] ? k : k - 1;  // thr: shared (pencil kernels) or global memory
}

__device__ __forceinline__ int bin_of(double v, const TileParam<double>& tp, const double*, int n,
                                      double nm05) {
  double y = __dmul_rn(__dsub_rn(v, tp.lo), tp.c);
  y = fmin(fmax(y, 0.5), nm05);
  const double fl = floor(y);
  const double fr = __dsub_rn(y, fl);
  if (fabs(__dsub_rn(fr, 0.5)) < tp.lim) return static_cast<int>(fl);
  return bin_exact(v, tp.lo, tp.hi, n);
}

// Smallest float whose reference bin is >= k (1 <= k <= n-1) for a
// non-degenerate, non-pathological range: guess, walk a few ulps, and fall
// back to bisection over the ordered float keys if the walk is long.
__device__ inline float bin_threshold(double lo, double hi, int n, int k) {
  float v = static_cast<float>(lo + (hi - lo) * static_cast<double>(k) / n);
  v = fminf(fmaxf(v, static_cast<float>(lo)), static_cast<float>(hi));
  int steps = 0;
  if (bin_exact(v, lo, hi, n) >= k) {
    while (steps++ < 16) {
      const float w = nextafterf(v, -INFINITY);
      if (bin_exact(w, lo, hi, n) >= k) v = w;
      else return v;
    }
  } else {
    while (steps++ < 16) {
      v = nextafterf(v, INFINITY);
      if (bin_exact(v, lo, hi, n) >= k) return v;
    }
  }
  // bisection on monotone int keys: bin(lo) = 0 < k <= n-1 = bin(hi)
  auto key = [](float f) { int i = __float_as_int(f); return i >= 0 ? i : (i ^ 0x7FFFFFFF); };
  auto unkey = [](int i) { return __int_as_float(i >= 0 ? i : (i ^ 0x7FFFFFFF)); };
  // bin(a) < k <= bin(b); 64-bit keys (the key span of [-FLT_MAX, FLT_MAX] exceeds INT_MAX)
  long long a = key(static_cast<float>(lo)), b = key(static_cast<float>(hi));
  while (b - a > 1) {
    const long long m = a + (b - a) / 2;
    if (bin_exact(unkey(static_cast<int>(m)), lo, hi, n) >= k) b = m;
    else a = m;
  }
  return unkey(static_cast<int>(b));
}

// ---- packed (f32x2) guarded binning for the pencil kernels ----------------
// Same bound as bin_of, two voxels per FADD2/FMUL2.  Out-of-range y is
// clamped on the integer side (the magic-number floor is exact for
// |y| < 2^22 and monotone beyond, so clamping k is still the reference's
// clamp).  Near an integer the edge table decides (k in [1, n-1]).
// lc = {lo, c}; degenerate tiles use lc = kDegenerateLC (y == 0.5 exactly,
// constant 0.5 LUT), pathological ranges (make_tile_param lim < 0) are
// routed by the caller to bin_search.
typedef unsigned long long u64;

__device__ __forceinline__ u64 pk2(float x, float y) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void upk2(u64 r, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(r));
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 add2rm(u64 a, u64 b) {
  u64 d;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
constexpr int kMagicBits = 0x4B400000;

__device__ __forceinline__ float2 degenerate_lc() {
  return make_float2(-4.2535295865117308e37f /* -2^125 */, 1.1754943508222875e-38f /* 2^-126 */);
}

// k = rint(y) clamped to [0, n], from t = y + kMagic (round to nearest).
// The clamp runs on the raw bits as signed ints, which order every float
// t >= +0 by value and put every negative t (y < -kMagic) below kMagicBits;
// subtracting first would wrap for |t| >= 2^23-ish and misbin voxels far
// outside a narrow tile range (blend corners see such voxels).
__device__ __forceinline__ int clamp_bits(float t, int n) {
  return min(max(__float_as_int(t), kMagicBits), kMagicBits + n) - kMagicBits;
}

// Same value as an opaque max / sub / min sequence, so the compiler cannot
// fold the magic offset into later address arithmetic.
__device__ __forceinline__ int clamp_bits_k(float t, int n) {
  int k;
  asm("{\n\t.reg .s32 x;\n\tmax.s32 x, %1, %2;\n\tsub.s32 x, x, %2;\n\tmin.s32 %0, x, %3;\n\t}"
      : "=r"(k)
      : "r"(__float_as_int(t)), "r"(kMagicBits), "r"(n));
  return k;
}

// Branch-free exact bins of two voxels against one tile, edge table only.
// k = rint(y) (magic-number add in round-to-nearest); since |y - q| < 0.5 for
// every y that matters, the reference bin floor(q) is k or k - 1, and it is k
// iff v >= th[k].  Clamping k to [0, n] against the sentinels th[0] = -inf,
// th[n] = +inf reproduces the reference's clamp for y outside [0, n) (and
// for |y| >= 2^22, where the magic add saturates monotonically).
__device__ __forceinline__ void bins2_edge(u64 V, float v0, float v1, float2 lc, const float* th,
                                           int n, int& b0, int& b1) {
  const u64 y = mul2(sub2(V, pk2(lc.x, lc.x)), pk2(lc.y, lc.y));
  u64 t;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(y), "l"(pk2(kMagic, kMagic)));
  float t0, t1;
  upk2(t, t0, t1);
  const int k0 = clamp_bits(t0, n);
  const int k1 = clamp_bits(t1, n);
  b0 = v0 >= th[k0] ? k0 : k0 - 1;
  b1 = v1 >= th[k1] ? k1 : k1 - 1;
}

// Same rule, fused with the LUT gather: returns LUT[bin] for two voxels.
// thb / Lb are the tile's edge table and LUT (byte pointers, warp-uniform in
// the blend kernel); n4 = 4 * n.  Byte offsets throughout so each gather is a
// single LDS [reg + base].
__device__ __forceinline__ void lut2_edge(u64 V, float v0, float v1, float2 lc, const char* thb,
                                          const char* Lb, int n4, float& m0, float& m1) {
  const u64 y = mul2(sub2(V, pk2(lc.x, lc.x)), pk2(lc.y, lc.y));
  u64 t;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(y), "l"(pk2(kMagic, kMagic)));
  float t0, t1;
  upk2(t, t0, t1);
  const int k0 = clamp_bits(t0, n4 >> 2) << 2;
  const int k1 = clamp_bits(t1, n4 >> 2) << 2;
  const int b0 = v0 >= *reinterpret_cast<const float*>(thb + k0) ? k0 : k0 - 4;
  const int b1 = v1 >= *reinterpret_cast<const float*>(thb + k1) ? k1 : k1 - 4;
  m0 = *reinterpret_cast<const float*>(Lb + b0);
  m1 = *reinterpret_cast<const float*>(Lb + b1);
}

// ---- bracketed floor (the NB blend's fast path) ----------------------------
// With d = fl32(v - lo) and c = fl32(n / (hi - lo)), the exact product d * c
// is within a factor (1 +- 2^-23 (1 + 2^-20)) of the reference's f64 value q
// (two f32 roundings; the f64 ones are ~2^-51).  c_lo = RD(c (1 - 2^-22)) and
// c_hi = RU(c (1 + 2^-22)) therefore bracket q:  d c_lo <= q <= d c_hi for
// d >= 0 (reversed for d < 0).  fma.rm(d, c, M) = floor(d c) + M exactly
// (one rounding, |d c| < 2^22), so when the two floors agree they ARE
// floor(q), no edge table needed; when they differ (q within ~5e-7 |q| of an
// integer) the bin is k or k - 1 with k the upper one and the edge table
// decides.  Out-of-range products clamp on the raw bits (clamp_bits).
constexpr float kWinLo = 0.99999976158142089844f;  // 1 - 2^-22
constexpr float kWinHi = 1.00000023841857910156f;  // 1 + 2^-22

__device__ __forceinline__ float2 bin_window(float c) {
  return make_float2(__fmul_rd(c, kWinLo), __fmul_ru(c, kWinHi));
}

__device__ __forceinline__ u64 fma_rm2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// LUT entry at shared byte address lbase + 4 * bits + OFF (one IMAD + one
// LDS [reg + imm]; lbase already carries -4 * kMagicBits, mod 2^32).
template <int OFF>
__device__ __forceinline__ float lut_at(uint32_t lbase, int bits) {
  float m;
  asm volatile(
      "{\n\t.reg .u32 a;\n\tmad.lo.u32 a, %1, 4, %2;\n\tld.shared.f32 %0, [a+%3];\n\t}"
      : "=f"(m)
      : "r"(bits), "r"(lbase), "n"(OFF));
  return m;
}

// Same entry from the floor bits with one VIADDMNMX.RELU: k = clamp(bits -
// kMagicBits, 0, nm1) at shared byte address base + 4 * k + OFF.  Exact only
// while bits - kMagicBits cannot wrap (t > 0: the caller checks the range).
template <int OFF>
__device__ __forceinline__ float lut_at_relu(uint32_t base, int bits, int nm1) {
  float m;
  asm volatile(
      "{\n\t.reg .s32 k;\n\t.reg .u32 a;\n\t"
      "add.s32 k, %1, %3;\n\t"
      "min.relu.s32 k, k, %4;\n\t"
      "mad.lo.u32 a, k, 4, %2;\n\t"
      "ld.shared.f32 %0, [a+%5];\n\t}"
      : "=f"(m)
      : "r"(bits), "r"(base), "r"(-kMagicBits), "r"(nm1), "n"(OFF));
  return m;
}

// Bins of two voxels by the bracketed floors, as the NB blend computes them
// (fast answer clamp(floor(d c_lo)); where the clamped floors disagree, the
// edge table th (unpadded here) decides between them).  w = bin_window(c).
__device__ __forceinline__ void bins2_bracket(u64 V, float v0, float v1, float lo, float2 w,
                                              const float* th, int n, int& b0, int& b1) {
  const u64 d = sub2(V, pk2(lo, lo));
  const u64 M2 = pk2(kMagic, kMagic);
  float a[2], b[2];
  upk2(fma_rm2(d, pk2(w.x, w.x), M2), a[0], a[1]);
  upk2(fma_rm2(d, pk2(w.y, w.y), M2), b[0], b[1]);
  const float vv[2] = {v0, v1};
  int r[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int ka = clamp_bits(a[i], n - 1), kb = clamp_bits(b[i], n - 1);
    r[i] = (ka != kb && vv[i] >= th[kb]) ? kb : ka;
  }
  b0 = r[0];
  b1 = r[1];
}

// Same rule against an NbBlock (edge table padded one word per 32 entries at
// TH, LUT unpadded at L): the edge test decides k or k - 1, then one gather.
template <int TH, int L>
__device__ __forceinline__ float edge_gather_u(uint32_t base, int k, float v) {
  float m;
  asm volatile(
      "{\n\t.reg .u32 a, b;\n\t.reg .f32 t;\n\t.reg .pred p;\n\t"
      "shr.u32 a, %1, 5;\n\t"
      "add.u32 a, a, %1;\n\t"
      "mad.lo.u32 a, a, 4, %2;\n\t"
      "ld.shared.f32 t, [a+%4];\n\t"
      "mad.lo.u32 b, %1, 4, %2;\n\t"
      "setp.lt.f32 p, %3, t;\n\t"
      "@p sub.u32 b, b, 4;\n\t"
      "ld.shared.f32 %0, [b+%5];\n\t}"
      : "=f"(m)
      : "r"(k), "r"(base), "f"(v), "n"(TH), "n"(L));
  return m;
}

// Reference bin of v given k = rint(y) clamped to [0, n] (clamp_bits_k) and
// the tile's edge table at shared address th: k if v >= th[k], else k - 1.
__device__ __forceinline__ int edge_bin(uint32_t th, int k, float v) {
  int b;
  asm volatile(
      "{\n\t.reg .u32 a;\n\t.reg .f32 t;\n\t.reg .pred p;\n\t"
      "mad.lo.u32 a, %1, 4, %2;\n\t"
      "ld.shared.f32 t, [a];\n\t"
      "setp.lt.f32 p, %3, t;\n\t"
      "selp.s32 %0, 1, 0, p;\n\t"
      "sub.s32 %0, %1, %0;\n\t}"
      : "=r"(b)
      : "r"(k), "r"(th), "f"(v));
  return b;
}

// Histogram word of the reference bin: k as edge_bin, the word at
// h + 4 * bin (h = the tile's row), without materialising the bin.
__device__ __forceinline__ uint32_t edge_hist_addr(uint32_t th, int k, float v, uint32_t h) {
  uint32_t a;
  asm volatile(
      "{\n\t.reg .u32 t;\n\t.reg .f32 x;\n\t.reg .pred p;\n\t"
      "mad.lo.u32 t, %1, 4, %2;\n\t"
      "ld.shared.f32 x, [t];\n\t"
      "mad.lo.u32 %0, %1, 4, %4;\n\t"
      "setp.lt.f32 p, %3, x;\n\t"
      "@p sub.u32 %0, %0, 4;\n\t}"
      : "=r"(a)
      : "r"(k), "r"(th), "f"(v), "r"(h));
  return a;
}

// Unconditional shared-memory add.
__device__ __forceinline__ void red_add(uint32_t addr, uint32_t val) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(val) : "memory");
}
// the same add predicated off where skip is set (no branch; lanes that skip take
// no part in the instruction's bank conflicts)
__device__ __forceinline__ void red_add_unless(uint32_t addr, uint32_t val, bool skip) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %2, 0;\n\t@p red.shared.add.u32 [%0], %1;\n\t}" ::"r"(addr),
      "r"(val), "r"((uint32_t)skip)
      : "memory");
}

// Exact bin from the edge table alone (binary search over thr[1..n-1]);
// used for ranges the float guard does not cover.
__device__ __forceinline__ int bin_search(float v, const float* th, int n) {
  int lo = 0, hi = n - 1;  // answer in [lo, hi]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (v >= th[mid]) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// {lo, c} table entry for a tile (NaN c marks a pathological range).
__device__ __forceinline__ float2 tile_lc(const TileParam<float>& tp) {
  if (tp_degenerate(tp.lim)) return degenerate_lc();
  if (tp.lim < 0.0f) return make_float2(tp.lo, __int_as_float(0x7fc00000));
  return make_float2(tp.lo, tp.c);
}

#endif  // __CUDACC__

}  // namespace mg
