// common.cuh -- kernel-side types and the bulk-copy stage pipeline shared by
// the pencil kernels (K2a tile ranges, K2b histograms, K4 blend).
//
// Pencil work decomposition: a unit is one tile (K2) or one interpolation
// cell (K4) along the KO outer dimensions, all tiles/cells along the KT
// trailing dimensions, and a chunk of dim-0 rows.  A unit's voxels are
// "runs": for every coordinate of the outer dims except the last, the
// ext[KO-1] consecutive rows of P = prod(trailing extents) floats are one
// contiguous span of the input.  The input is described to the TMA engine
// as a (KO + 1 or 2)-D tensor (outer dims, trailing block split into <=256
// wide rows); one producer thread walks each unit in R2 x R1 row boxes and
// issues ONE cp.async.bulk.tensor per pipeline stage (completion counted on an
// mbarrier); eight consumer warps read each stage with conflict-free 16-byte
// LDS, every thread owning a fixed 4-voxel column of the trailing block.
#pragma once

#include <type_traits>

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "binning.cuh"
#include "geometry.h"

namespace mg {

// Compile-time loop: f(std::integral_constant<int, I>) for I in [B, E).
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}


constexpr int kUnitInts = 10;      // unit record: [0..7] tile/cell per outer dim, [8] ra, [9] re
constexpr int kMaxOuterDims = 5;   // pencil kernels: KO in [1, 5]
constexpr int kMaxRuns = 16;       // runs gathered into one stage
constexpr int kMaxStages = 6;
constexpr int kConsumers = 256;    // 8 consumer warps (K2 kernels)
constexpr int kPencilThreads = kConsumers + 32;  // + producer warp
#ifndef BLEND_CONSUMERS
#define BLEND_CONSUMERS 512
#endif
constexpr int kConsumersBlend = BLEND_CONSUMERS;  // consumer warps x 32 (K4: one CTA per SM)
constexpr int kBlendThreads = kConsumersBlend + 32;

// Kernel-side geometry (passed by value).
struct KGeom {
  int rank;         // D
  int kt;           // trailing dims covered by a pencil
  int n_bins;
  int tpr;          // threads per trailing block (P / 4)
  int rpi;          // trailing blocks (rows) per consumer iteration
  int adaptive;
  int nst;          // pipeline stages
  int stage_rows;   // rows of P floats per stage (= R1 * R2)
  int r1, lg_r1;    // box rows along outer dim KO-1 (power of two) and log2
  int r2;           // box rows along outer dim KO-2 (1 if KO == 1)
  int tma_rank;     // rank of the TMA tensor view of the input
  int nseg;         // K4: 32-float segments of the trailing block (one per stage)
  int64_t stage_stride;  // floats between stage buffers (1024-byte multiple)
  int64_t P;        // elements of one trailing block
  int64_t gtr;      // tiles of one trailing block
  Dim d[kMaxRank];
  int64_t vstride[kMaxRank];  // strides of the LOCAL (slab) buffer
  int64_t tstride[kMaxRank];  // row-major strides of the tile grid
  int64_t row0;               // global dim-0 row of local row 0
  int64_t trow0;              // first tile row of the workspace window
  int64_t win_tiles;
  int64_t local_voxels;
  double clip;
  float inv_b[kMaxRank];   // 1 / b per dim (K4 weight factors)
  float inv_2b[kMaxRank];  // 1 / (2 b)
  int dict;                // 1: the value-dictionary blend is armed (K2a builds the dictionary)
  int stiles;              // NB blend: trailing tiles staged at once (one segment's window)
  int dyn_units;           // blend: > 0 = units handed out dynamically (count), via W.range[3]
  int seg_items;           // blend: 1 = a work item is (unit, ONE segment): item / nseg, item % nseg
  int nb_edges;            // NB blend: -1 auto (from the K2a value sample), 0 bracketed floors, 1 edge tables
  int cell_hist;           // K2b: 1 = k_hist_cells is launched beside k_hist_pencil (dictionary state selects)
};

// Value dictionary (adaptive mode, float32): when the volume holds few
// distinct values (quantised counts), K2a collects them, k_dict_finalize
// numbers them and builds a lookup hash, k_dict_luts tabulates every tile's
// LUT[bin(value)] per value, and the blend gathers those directly.
constexpr int kDictHG = 8192;        // global set slots (accepts <= kDictHG / 2 values)
// Shared-memory sets are bucketised: 4 keys per 16-byte bucket, so a present
// value is found with one LDS.128 and four compares (no divergent probe loop).
constexpr int kDictLgBS = 10;        // K2a per-CTA set: 1024 buckets (16 KB)
constexpr int kDictHS = 4 << kDictLgBS;
constexpr int kDictLgHL = 10;        // blend lookup: 1024 {bits, index} (affine direct table or cuckoo hash)
constexpr int kDictHL = 1 << kDictLgHL;
constexpr int kDictKC = 608;         // values (or direct cells) per tile row in the blend (capacity)
constexpr uint32_t kDictEmpty = 0xFFFFFFFFu;  // a NaN pattern: never a finite input
__host__ __device__ __forceinline__ uint32_t dict_hash(uint32_t b, int lg) {
  return (b * 0x9E3779B1u) >> (32 - lg);
}
// meta[0]: values inserted, [1]: overflow, [2]: dictionary usable, [3]: K
// (index slots), [7]: distinct values numbered

// Cuckoo lookup: a value sits at one of two slots (branch-free, two LDS.64);
// -1 when absent.
__host__ __device__ __forceinline__ uint32_t dict_h1(uint32_t b) {
  return (b * 0x9E3779B1u) >> (32 - kDictLgHL);
}
__host__ __device__ __forceinline__ uint32_t dict_h2(uint32_t b) {
  return ((b ^ (b >> 15)) * 0x85EBCA77u) >> (32 - kDictLgHL);
}
__device__ __forceinline__ int dict_lookup(const uint2* t, uint32_t b) {
  const uint2 e1 = t[dict_h1(b)], e2 = t[dict_h2(b)];
  return e1.x == b ? (int)e1.y : e2.x == b ? (int)e2.y : -1;
}

// meta[4]: 1 = affine lookup (meta[5] = bits of v0, meta[6] = bits of S), 0 = cuckoo,
// 2 = direct cells: the affine cell IS the index (values numbered by cell,
// holes hold kDictEmpty), so the folded-pair blend gathers by cell after one
// 32-bit check of the value's bits instead of an LDS.64 {bits, index} lookup.
// Affine cells of two values (packed, as the blend computes them), clamped to
// [0, LIM]; the second value's cell goes to *c1 when c1 != nullptr.
#ifdef __CUDACC__
template <uint32_t LIM = kDictHL - 1>
__device__ __forceinline__ int dict_cell(float a, float b, float v0, float S, int* c1) {
  unsigned long long V, D, Y, T;
  asm("mov.b64 %0, {%1, %2};" : "=l"(V) : "f"(a), "f"(b));
  asm("mov.b64 %0, {%1, %1};" : "=l"(D) : "f"(v0));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(Y) : "l"(V), "l"(D));
  asm("mov.b64 %0, {%1, %1};" : "=l"(D) : "f"(S));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(Y) : "l"(Y), "l"(D));
  asm("mov.b64 %0, {%1, %1};" : "=l"(D) : "f"(12582912.0f));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(T) : "l"(Y), "l"(D));
  float t0, t1;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(t0), "=f"(t1) : "l"(T));
  // one unsigned min (VIADDMNMX): values below v0 wrap to huge and land on the
  // last cell, which the caller's bit comparison rejects like any other miss
  auto cl = [](float t) {
    return (int)min((uint32_t)__float_as_int(t) - 0x4B400000u, LIM);
  };
  if (c1) *c1 = cl(t1);
  return cl(t0);
}
#endif


// Workspace views.
struct WS {
  int64_t* range;       // [4]: ~key(lo), key(hi), nonfinite, unused
  int64_t* trange;      // [win_tiles][2]
  uint32_t* counts;     // [win_tiles][n_bins]
  void* tparams;        // TileParam<T>[adaptive ? win_tiles : 1]
  float* lut;           // [win_tiles][n_bins]
  float* thr;           // [adaptive ? win_tiles : 1][n_bins] bin-edge tables (f32 data)
  int32_t* dmeta;       // [8] value dictionary state (see kDict*)
  uint32_t* dkeys;      // [kDictHG] value bits (open addressing)
  float* dvals;         // [kDictHG / 2] values by index
  uint2* dlt;           // [kDictHL] cuckoo lookup {bits, index}
  float* lutd;          // [win_tiles][kDictKC] LUT[bin(value)] per value
  int32_t* k2g;         // fused K2: [groups] arrivals, then [groups] published flags
  float* k2tab;         // fused K2: [groups] aligned table blocks (k_fused.cu ftab_bytes)
};

struct Debug {
  double* lo;
  double* hi;
  uint32_t* counts;
  double* clipped;
  double* lut;
  uint8_t* degenerate;
};

__device__ __forceinline__ int32_t key32(float x) {
  const int32_t i = __float_as_int(x);
  return i >= 0 ? i : (i ^ 0x7FFFFFFF);
}
__device__ __forceinline__ float key32_decode(int32_t k) {
  return __int_as_float(k >= 0 ? k : (k ^ 0x7FFFFFFF));
}

// ----------------------------------------------------- mbarrier / bulk ---
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "MG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
      "@!p bra MG_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Polling variant (no suspend-time hint): for the blend producer, whose slot
// frees in well under a microsecond, where the suspend / wake round trip of
// the hinted wait is on the critical path.  MG_SPIN_NS > 0 backs off that many
// nanoseconds between polls: a bare spin issues ~3 instructions per poll on
// the SM sub-partition it shares with four consumer warps (5D blend: 6 % of
// all instructions issued).
#ifndef MG_SPIN_NS
#define MG_SPIN_NS 32
#endif
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
    if (MG_SPIN_NS > 0) __nanosleep(MG_SPIN_NS);
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
template <int NC = kConsumers>
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
}

// One pipeline stage = one TMA box of one unit: R2 x R1 rows of P floats.
struct Stage {
  int32_t unit;   // -1: end of stream
  int32_t wuni;   // K2: 1 if the multiplicity is uniform over the box (= wfix)
  int32_t wfix;   // K2: multiplicity over dims < KO-2 (or over the whole box if wuni)
  int32_t seg;    // K4: 32-float segment of the trailing block held by the stage
  int64_t key;    // tile window offset (K2) or cell key (K4) of the unit
  int32_t x[kMaxOuterDims];     // absolute coordinates of the box origin (dim 0 global)
  int32_t cell[kMaxOuterDims];  // K4: cells of the unit (K2: tiles)
  TileParts p1, p2;             // K2: tile parts along dims KO-1 and KO-2
  int32_t tc[6];                // TMA box coordinates of the stage (K4 reuses them to store)
  int32_t ph;                   // fused K2: 0 = range pass over the unit, 1 = counting pass
  int32_t last;                 // fused K2: last box of the unit's pass; NEXT producers: last
                                // box of the work item, the fields below name the next item
  int32_t nunit;                // next work item (-1: none)
  int32_t nseg;                 // its segment
  int64_t nkey;                 // its cell key
  int32_t ncell[kMaxOuterDims]; // its cells
};

// Producer-private per-unit box (kept in shared memory, not registers, so
// the single producer thread does not inflate the kernel's register count).
struct ProdBox {
  int64_t a[kMaxOuterDims];
  int32_t ext[kMaxOuterDims];
  TileParts parts[kMaxOuterDims];
};

struct Pipe {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
  Stage st[kMaxStages];
  ProdBox box;
};

// 1024-byte aligned so stage buffers meet the TMA 128B-swizzle alignment.
__device__ __forceinline__ size_t pipe_bytes() { return (sizeof(Pipe) + 1023) & ~size_t(1023); }

// Initialises the barriers (thread 0) -- call before the role split, then
// __syncthreads().
__device__ __forceinline__ void pipe_init(Pipe& pp, int nst, int consumer_warps = kConsumers / 32) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&pp.full[s], 1);
      mbar_init(&pp.empty[s], consumer_warps);
    }
    fence_barrier_init();
  }
}

// TMA tensor load of one box; coordinates innermost first.
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, int rank, const int* c,
                                         uint64_t* bar) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  const uint32_t d = smem_u32(dst), b = smem_u32(bar);
  switch (rank) {
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(b)
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]),
          "r"(b)
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]),
          "r"(c[2]), "r"(c[3]), "r"(b)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]),
          "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b)
          : "memory");
      break;
  }
}

// Same with an L2 cache-policy hint (createpolicy): the fused K2 keeps the
// boxes of its range walk in L2 (evict_last) for the counting walk that
// re-reads them, which then marks them evict_first.
__device__ __forceinline__ void tma_load_hint(void* dst, const CUtensorMap* map, int rank,
                                              const int* c, uint64_t* bar, uint64_t pol) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  const uint32_t d = smem_u32(dst), b = smem_u32(bar);
  switch (rank) {
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
          " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(b), "l"(pol)
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
          " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]),
          "r"(b), "l"(pol)
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
          " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]),
          "r"(c[2]), "r"(c[3]), "r"(b), "l"(pol)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]),
          "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b), "l"(pol)
          : "memory");
      break;
  }
}

// TMA tensor store of one box from shared memory (bulk-group completion).
__device__ __forceinline__ void tma_store(const CUtensorMap* map, int rank, const int* c,
                                          const void* src) {
  const uint64_t m = reinterpret_cast<uint64_t>(map);
  const uint32_t s = smem_u32(src);
  switch (rank) {
    case 2:
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m),
                   "r"(c[0]), "r"(c[1]), "r"(s)
                   : "memory");
      break;
    case 3:
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(m),
                   "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(s)
                   : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(m),
          "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(s)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(m),
          "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(s)
          : "memory");
      break;
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// Makes this thread's generic-proxy shared-memory writes visible to the TMA.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Producer (one thread): walks the CTA's units box by box (the plan makes
// every unit extent along dims KO-1 / KO-2 a multiple of R1 / R2) and issues
// one TMA box load per stage.  CELLS selects interpolation-cell boxes (K4)
// instead of tile-support boxes (K2).
// Is the multiplicity of tile parts p constant over [x, x + r)?  (no
// interval end strictly inside the range)
__device__ __forceinline__ bool parts_uniform(const TileParts& p, int64_t x, int64_t r) {
  const int64_t e[6] = {p.id_a, p.id_e, p.lo_a, p.lo_e, p.hi_a, p.hi_e};
  bool u = true;
#pragma unroll
  for (int i = 0; i < 6; ++i) u = u && !(e[i] > x && e[i] < x + r);
  return u;
}

// STORE: consumers leave each stage's results in place; before a slot is
// refilled (and after the last stage) its box is written back with a TMA
// tensor store through out_map.
// SEGOUT: segments outermost in a unit (the blend kernels, which stage per
// segment); otherwise every box walks all segments in turn.
// The per-stage path is kept short (one thread issues every stage while 16
// consumer warps share its SM sub-partition): slot / phase counters instead
// of divisions, the unit record and geometry in registers, TMA coordinates in
// registers.
// NEXT: the producer takes the following work item while it starts the
// current one and names it in the record of the current item's last box
// (Stage::last / nunit / nseg / nkey / ncell), so a consumer that rebuilds
// per-item tables can do so as soon as it has finished the item -- while the
// next item's first boxes are still in flight -- instead of after they land.
template <int KO, bool CELLS, bool WEIGHTS = !CELLS, bool STORE = false, bool SEGOUT = STORE,
          bool NEXT = false>
__device__ __noinline__ void pipe_produce(const KGeom& G, const CUtensorMap* map,
                                          const int32_t* __restrict__ units, int u0, int u1,
                                          Pipe& pp, float* bufs,
                                          const CUtensorMap* out_map = nullptr,
                                          unsigned long long* dyn = nullptr,
                                          const TileParam<float>* skip_tp = nullptr) {
  const int nst = G.nst;
  const int nseg = G.nseg;
  const bool segv = G.tma_rank - KO == 2;  // the TMA view has a segment coordinate
  const int tma_rank = G.tma_rank;
  const int seg_items = G.seg_items;
  const int32_t row0 = (int32_t)G.row0;
  const int64_t stage_elems = G.stage_stride;
  const uint32_t box_bytes = (uint32_t)((int64_t)G.stage_rows * (G.P / nseg) * 4);
  const int R1 = G.r1, R2 = G.r2;
  ProdBox& B = pp.box;
  uint32_t it = 0;
  int slot = 0;
  uint32_t phase = 0;  // (it / nst) & 1
  // dyn != nullptr: units are handed out dynamically (one atomic per unit,
  // [u0, u1) is then the whole list); otherwise the CTA's static range
  int u = dyn ? u0 + (int)atomicAdd(dyn, 1ULL) : u0;
  // NEXT: the item after u, taken when u has kNextAhead boxes left to issue --
  // late enough that the handout order stays what it is without the look-ahead
  // (sibling items still start together on different CTAs and share their L2
  // lines; taking it at the start of u gave one CTA two siblings in a row:
  // 4D folded-pair blend 0.64 -> 0.68 ms), early enough to hide the atomic and
  // the record read
  constexpr int kNextAhead = 6;
  int un = 0;
#pragma unroll 1
  for (; u < u1; u = NEXT ? un : (dyn ? u0 + (int)atomicAdd(dyn, 1ULL) : u + 1)) {
    // seg_items: work item u = (unit u / nseg, segment u % nseg)
    const int seg_w = seg_items ? u % nseg : 0;
    const int32_t* U = units + (int64_t)(seg_items ? u / nseg : u) * kUnitInts;
    int32_t cellr[KO];
#pragma unroll
    for (int j = 0; j < KO; ++j) cellr[j] = U[j];
    // NEXT: the following item's identity, for the record of this item's last box
    int32_t ncellr[KO] = {0};
    int64_t nkey = 0;
    int nseg_w = 0;
    bool have_next = false;
    int64_t key = 0;
    B.a[0] = U[8];
    B.ext[0] = U[9] - U[8];
    B.parts[0] = tile_parts(G.d[0], cellr[0]);
#pragma unroll 1
    for (int j = 1; j < KO; ++j) {
      if (CELLS) {
        int64_t ca, ce;
        cell_range(G.d[j], U[j], &ca, &ce);
        B.a[j] = ca;
        B.ext[j] = (int32_t)(ce - ca);
      } else {
        B.parts[j] = tile_parts(G.d[j], U[j]);
        B.a[j] = B.parts[j].support_begin();
        B.ext[j] = (int32_t)(B.parts[j].support_end() - B.a[j]);
      }
    }
    if (CELLS) {
#pragma unroll 1
      for (int j = 0; j < KO; ++j) key = key * G.d[j].g + U[j];
    } else {
      key = (U[0] - G.trow0) * G.tstride[0];
#pragma unroll 1
      for (int j = 1; j < KO; ++j) key += (int64_t)U[j] * G.tstride[j];
      // K2b, adaptive: a unit whose tiles are all degenerate is never binned
      // (build_mappings skips collapsed ranges, src/histogram.cpp:95-98), so
      // its boxes are not even loaded
      if (skip_tp) {
        bool all = true;
#pragma unroll 1
        for (int t = 0; t < G.gtr && all; ++t) all = tp_degenerate(skip_tp[key + t].lim);
        if (all) continue;
      }
    }
    // boxes: dims < KO-2 one coordinate each, dim KO-2 in steps of R2, dim KO-1 of R1
    int64_t nfix = 1;
#pragma unroll 1
    for (int j = 0; j < KO - 2; ++j) nfix *= B.ext[j];
    const int n1 = B.ext[KO - 1] / R1;
    const int n2 = KO >= 2 ? B.ext[KO - 2] / R2 : 1;
    const int32_t a1 = (int32_t)B.a[KO - 1], a2 = KO >= 2 ? (int32_t)B.a[KO - 2] : 0;
    TileParts p1, p2;
    if (WEIGHTS) {
      p1 = B.parts[KO - 1];
      if (KO >= 2) p2 = B.parts[KO - 2];
    }
    // boxes of this work item still to issue (NEXT: the last one carries the next item)
    int64_t left = nfix * n1 * n2 * (SEGOUT ? (seg_items ? 1 : nseg) : nseg);
    // blend (SEGOUT): segments outermost, so a consumer staging per segment
    // restages rarely
#pragma unroll 1
    for (int sego = seg_w; sego < (SEGOUT ? (seg_items ? seg_w + 1 : nseg) : seg_w + 1); ++sego)
#pragma unroll 1
    for (int64_t f = 0; f < nfix; ++f) {
      int32_t xf[kMaxOuterDims];
      int32_t wfix = 1;
      int64_t rem = f;
#pragma unroll
      for (int j = KO - 3; j >= 0; --j) {
        xf[j] = (int32_t)(B.a[j] + rem % B.ext[j]);
        rem /= B.ext[j];
        if (WEIGHTS) wfix *= B.parts[j].weight(xf[j]);
      }
#pragma unroll 1
      for (int i2 = 0; i2 < n2; ++i2) {
        const int32_t x2 = a2 + i2 * R2;
#pragma unroll 1
        for (int i1 = 0; i1 < n1; ++i1) {
          const int32_t x1 = a1 + i1 * R1;
#pragma unroll 1
        for (int segi = 0; segi < (SEGOUT ? 1 : nseg); ++segi) {
          const int seg = SEGOUT ? sego : segi;
          if (STORE || SEGOUT) mbar_wait_spin(&pp.empty[slot], phase ^ 1);  // blend: latency-critical
          else mbar_wait(&pp.empty[slot], phase ^ 1);
          Stage& S = pp.st[slot];
          if (STORE && it >= (uint32_t)nst) {  // write back the slot's previous results
            tma_store(out_map, tma_rank, S.tc, bufs + slot * stage_elems);
            tma_store_wait_read();
          }
          S.unit = u;
          S.seg = seg;
          S.key = key;
          if (NEXT) {
            if (!have_next && left <= kNextAhead) {
              have_next = true;
              un = dyn ? u0 + (int)atomicAdd(dyn, 1ULL) : u + 1;
              if (un < u1) {
                const int32_t* Un = units + (int64_t)(seg_items ? un / nseg : un) * kUnitInts;
                nseg_w = seg_items ? un % nseg : 0;
#pragma unroll
                for (int j = 0; j < KO; ++j) {
                  ncellr[j] = Un[j];
                  nkey = nkey * G.d[j].g + Un[j];
                }
              }
            }
            const bool last = --left == 0;
            S.last = last ? 1 : 0;
            if (last) {
              S.nunit = un < u1 ? un : -1;
              S.nseg = nseg_w;
              S.nkey = nkey;
#pragma unroll
              for (int j = 0; j < KO; ++j) S.ncell[j] = ncellr[j];
            }
          }
#pragma unroll
          for (int j = 0; j < KO - 2; ++j) S.x[j] = xf[j];
          S.x[KO - 1] = x1;
          if (KO >= 2) S.x[KO >= 2 ? KO - 2 : 0] = x2;
#pragma unroll
          for (int j = 0; j < KO; ++j) S.cell[j] = cellr[j];
          if (WEIGHTS) {
            S.p1 = p1;
            if (KO >= 2) S.p2 = p2;
            const bool uni = parts_uniform(p1, x1, R1) && (KO < 2 || parts_uniform(p2, x2, R2));
            S.wuni = uni ? 1 : 0;
            S.wfix = uni ? wfix * p1.weight(x1) * (KO >= 2 ? p2.weight(x2) : 1) : wfix;
          }
          // TMA coordinates, innermost first: trailing block (+ segment),
          // then dims KO-1 .. 0 (dim 0 local to the slab)
          int c[6];
          int co[KO];
#pragma unroll
          for (int j = 0; j < KO; ++j)
            co[j] = j == KO - 1 ? x1 : (KO >= 2 && j == KO - 2 ? x2 : xf[j < KO - 2 ? j : 0]);
          co[0] -= row0;
          c[0] = 0;
          if (segv) {
            c[1] = seg;
#pragma unroll
            for (int j = 0; j < KO; ++j) c[2 + j] = co[KO - 1 - j];
          } else {
#pragma unroll
            for (int j = 0; j < KO; ++j) c[1 + j] = co[KO - 1 - j];
          }
          if (STORE)
#pragma unroll
            for (int i = 0; i < 6; ++i) S.tc[i] = c[i];
          mbar_expect_tx(&pp.full[slot], box_bytes);
          tma_load(bufs + slot * stage_elems, map, tma_rank, c, &pp.full[slot]);
          ++it;
          if (++slot == nst) {
            slot = 0;
            phase ^= 1;
          }
        }
        }
      }
    }
  }
  mbar_wait(&pp.empty[slot], phase ^ 1);
  if (STORE && it >= (uint32_t)nst) {
    tma_store(out_map, tma_rank, pp.st[slot].tc, bufs + slot * stage_elems);
    tma_store_wait_read();
  }
  pp.st[slot].unit = -1;
  mbar_arrive(&pp.full[slot]);
  if (STORE) {  // drain: the stages still in flight after the sentinel
    for (uint32_t j = (it >= (uint32_t)nst ? it - nst + 1 : 0); j < it; ++j) {
      const int s = j % nst;
      mbar_wait(&pp.empty[s], (j / nst) & 1);
      tma_store(out_map, tma_rank, pp.st[s].tc, bufs + s * stage_elems);
    }
    tma_store_wait_all();
  }
}

}  // namespace mg
