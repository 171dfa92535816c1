// common.cuh -- kernel-side types and the bulk-copy stage pipeline shared by
// the pencil kernels (K2a tile ranges, K2b histograms, K4 blend).
//
// Pencil work decomposition: a unit is one tile (K2) or one interpolation
// cell (K4) along the KO outer dimensions, all tiles/cells along the KT
// trailing dimensions, and a chunk of dim-0 rows.  A unit's voxels are
// "runs": for every coordinate of the outer dims except the last, the
// ext[KO-1] consecutive rows of P = prod(trailing extents) floats are one
// contiguous span of the input.  A producer warp streams runs into shared
// memory stages with cp.async.bulk (TMA bulk copy, completion on an
// mbarrier); eight consumer warps read each stage with conflict-free 16-byte
// LDS, every thread owning a fixed 4-voxel column of the trailing block.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "binning.cuh"
#include "geometry.h"

namespace mg {

constexpr int kUnitInts = 10;      // unit record: [0..7] tile/cell per outer dim, [8] ra, [9] re
constexpr int kMaxOuterDims = 5;   // pencil kernels: KO in [1, 5]
constexpr int kMaxRuns = 16;       // runs gathered into one stage
constexpr int kMaxStages = 6;
constexpr int kConsumers = 256;    // 8 consumer warps
constexpr int kPencilThreads = kConsumers + 32;  // + producer warp

// Kernel-side geometry (passed by value).
struct KGeom {
  int rank;         // D
  int kt;           // trailing dims covered by a pencil
  int n_bins;
  int tpr;          // threads per trailing block (P / 4)
  int rpi;          // trailing blocks (rows) per consumer iteration
  int adaptive;
  int nst;          // pipeline stages
  int stage_rows;   // rows of P floats per stage
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
};

// Workspace views.
struct WS {
  int64_t* range;       // [4]: ~key(lo), key(hi), nonfinite, unused
  int64_t* trange;      // [win_tiles][2]
  uint32_t* counts;     // [win_tiles][n_bins]
  void* tparams;        // TileParam<T>[adaptive ? win_tiles : 1]
  float* lut;           // [win_tiles][n_bins]
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
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra MG_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
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
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// One pipeline stage: up to kMaxRuns runs (or one chunk of one run) of one unit.
struct Stage {
  int32_t unit;   // -1: end of stream
  int32_t nruns;  // runs in the stage
  int32_t nr;     // rows per run in the stage
  int32_t r0;     // first row (relative to the box) of each run
  int64_t key;    // tile window offset (K2) or cell key (K4) of the unit
  int64_t a_last; // box start along outer dim KO-1
  TileParts pl;   // K2: tile parts along outer dim KO-1
  int32_t cell[kMaxOuterDims];           // K4: cells of the unit
  int64_t run_off[kMaxRuns];             // local element offset of (run, row r0)
  int32_t run_w[kMaxRuns];               // K2: multiplicity over dims 0..KO-2
  int32_t run_x[kMaxRuns][kMaxOuterDims];  // K4: absolute coords of dims 0..KO-2
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

__device__ __forceinline__ size_t pipe_bytes() { return (sizeof(Pipe) + 127) & ~size_t(127); }

// Initialises the barriers (thread 0) -- call before the role split, then
// __syncthreads().
__device__ __forceinline__ void pipe_init(Pipe& pp, int nst) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&pp.full[s], 1);
      mbar_init(&pp.empty[s], kConsumers / 32);
    }
    fence_barrier_init();
  }
}

// Producer (one thread): walks the CTA's units, cuts their runs into stages
// and issues the bulk copies.  CELLS selects interpolation-cell boxes (K4)
// instead of tile-support boxes (K2).
template <int KO, bool CELLS>
__device__ __noinline__ void pipe_produce(const KGeom& G, const float* __restrict__ in,
                                          const int32_t* __restrict__ units, int u0, int u1,
                                          Pipe& pp, float* bufs) {
  const int nst = G.nst;
  const int srows = G.stage_rows;
  const int64_t stage_elems = (int64_t)srows * G.P;
  ProdBox& B = pp.box;
  uint32_t it = 0;
#pragma unroll 1
  for (int u = u0; u < u1; ++u) {
    const int32_t* U = units + (int64_t)u * kUnitInts;
    int64_t key = 0;
    B.a[0] = U[8];
    B.ext[0] = U[9] - U[8];
    if (!CELLS) B.parts[0] = tile_parts(G.d[0], U[0]);
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
    }
    const int32_t el = B.ext[KO - 1];
    int64_t nrun = 1;
#pragma unroll 1
    for (int j = 0; j < KO - 1; ++j) nrun *= B.ext[j];
    const bool chunked = el >= srows;
    const int32_t m = chunked ? 1 : min(kMaxRuns, srows / el);
#pragma unroll 1
    for (int64_t run = 0; run < nrun; run += m) {
      const int32_t nruns = (int32_t)min((int64_t)m, nrun - run);
#pragma unroll 1
      for (int32_t r0 = 0; r0 < el; r0 += (chunked ? srows : el)) {
        const int32_t nr = chunked ? min(srows, el - r0) : el;
        const int slot = it % nst;
        mbar_wait(&pp.empty[slot], ((it / nst) & 1) ^ 1);
        Stage& S = pp.st[slot];
        S.unit = u;
        S.nruns = nruns;
        S.nr = nr;
        S.r0 = r0;
        S.key = key;
        S.a_last = B.a[KO - 1];
        if (!CELLS) S.pl = B.parts[KO - 1];
#pragma unroll 1
        for (int j = 0; j < KO; ++j) S.cell[j] = U[j];
        const uint32_t run_bytes = (uint32_t)(nr * G.P * 4);
        mbar_expect_tx(&pp.full[slot], run_bytes * nruns);
        float* dst = bufs + slot * stage_elems;
#pragma unroll 1
        for (int k = 0; k < nruns; ++k) {
          int64_t rem = run + k;
          int64_t off = (KO == 1 ? B.a[0] + r0 - G.row0 : B.a[KO - 1] + r0) * G.vstride[KO - 1];
          int32_t w = 1;
#pragma unroll 1
          for (int j = KO - 2; j >= 0; --j) {
            const int64_t x = B.a[j] + rem % B.ext[j];
            rem /= B.ext[j];
            off += (j == 0 ? x - G.row0 : x) * G.vstride[j];
            if (!CELLS) w *= B.parts[j].weight(x);
            S.run_x[k][j] = (int32_t)x;
          }
          S.run_off[k] = off;
          S.run_w[k] = w;
          bulk_g2s(dst + (int64_t)k * nr * G.P, in + off, run_bytes, &pp.full[slot]);
        }
        ++it;
      }
    }
  }
  const int slot = it % nst;
  mbar_wait(&pp.empty[slot], ((it / nst) & 1) ^ 1);
  pp.st[slot].unit = -1;
  mbar_arrive(&pp.full[slot]);
}

}  // namespace mg
