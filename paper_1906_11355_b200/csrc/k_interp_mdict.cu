// k_interp_mdict.cu -- K4, value-dictionary blend with the trailing corners
// folded into per-frame tables (adaptive mode, one trailing dim, KO == 3).
//
// The reference blends 2^D corner LUTs per voxel (src/pipeline.cpp:94-127,
// src/interpolation.cpp:44-86).  With one trailing dim, a voxel at frame i of
// trailing column c (4 frames, one trailing cell) weighs its two trailing
// corners with the column's fixed weights tw[c][i][0..1], so for every
// dictionary value v the pair folds into one number
//
//     M[c][i][co][v] = fma(tw1, L(co, tt_c + 1)[v], tw0 * L(co, tt_c)[v])
//
// and a voxel needs 2^KO gathers instead of 2^(KO+1): the shared-memory
// gathers, which bound the blend, halve.  The tables of all 8 columns would
// not fit in shared memory (590 KB for the 4D config), so a work item is one
// interpolation cell pencil x ONE 8-float segment of the trailing block (two
// columns, 147 KB of tables); the four CTAs holding the segments of one cell
// pencil take consecutive work items, and the tensor map's 256-byte L2
// promotion turns their 32-byte TMA boxes into whole-line DRAM reads.
//
// Summation order per voxel: acc = fma(wo[co], M[co], acc) over co ascending
// -- the edge-table blend (k_interp_pencil, MORD) sums in the same order, so
// both produce the same bits.
#include "k_pencil.cuh"

#ifndef MDICT_BUILD_BATCH
#define MDICT_BUILD_BATCH 4
#endif
// 1: the producer names the next work item in the last box of the current one
// (pipe_produce NEXT) and the consumers rebuild their tables before its first
// box lands.  Measured slower (4D blend 0.641 -> 0.651 ms, Large 4D 4.06 ->
// 4.21 ms; taking the next item at the start of the current one: 0.683 / 4.24,
// the siblings of a pencil then run back to back on one CTA and stop sharing
// their L2 lines), so it stays off: -DMDICT_NEXT=1 for A/B.
#ifndef MDICT_NEXT
#define MDICT_NEXT 0
#endif
// timing probes (results are WRONG; never shipped): 1 = tables built for a CTA's
// first item only, 2 = every gather at index 0 (broadcast), 3 = gathers at
// index = lane (conflict-free, no broadcast), 4 = 1 + 3, 5 = no blend at all (copy)
// 1: an in-place (TSTORE) item is a whole 32-row block, both 16-byte columns per
// lane (outer weights and row geometry once per 8 voxels instead of per 4)
// (-1: in global mode only -- Large 4D blend 4.05 -> 3.89 ms; the adaptive 4D blend
// measured 0.623 -> 0.631 ms with it)
#ifndef MDICT_BOTH
#define MDICT_BOTH -1
#endif
// consumer warps of the folded-pair blend (+ one producer warp): 19 warps are the
// most that keep 96 registers (5 warps per SM sub-partition).  Adaptive 4D blend
// 0.627 (16) / 0.621 (18) / 0.666 ms (20, 80 registers); Large 4D (global mode)
// 3.88 / 3.91 / 3.97 ms
#ifndef MDICT_NWARP_ADAPT
#define MDICT_NWARP_ADAPT 18
#endif
#ifndef MDICT_NWARP_GLOBAL
#define MDICT_NWARP_GLOBAL 16
#endif
// 1: a new item's first batch of table loads is issued before the item barrier (in
// flight while the slower warps finish the previous item).  Measured much slower
// (4D blend 0.623 -> 0.727 ms, Large 4D 3.88 -> 4.14 ms: the batch's 32 registers
// live across the barrier spill into the blend loop), so it stays off.
#ifndef MDICT_EARLY_LOAD
#define MDICT_EARLY_LOAD 0
#endif
#ifndef MDICT_PROBE
#define MDICT_PROBE 0
#endif

namespace mg {

// LDS [reg + imm]: one shared word at a compile-time byte offset from a 32-bit
// shared address
template <int OFF>
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float m;
  asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(m) : "r"(a), "n"(OFF));
  return m;
}
template <int OFF>
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t w;
  asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(w) : "r"(a), "n"(OFF));
  return w;
}

// TSTORE: results written in place into the stage and TMA-stored by the
// producer (otherwise a lane blends both 16-byte columns of its row and
// stores the full 32-byte sector straight to global; stages are released
// right after they are read).
// NWARP consumer warps (+ one producer warp).  ADAPT: value-dictionary tables
// (TK = kDictKC values per row); global mode (!ADAPT): one bin per voxel from
// the global edge table, tables per bin (TK = n_bins).
template <int KO, bool TSTORE, int NWARP, bool ADAPT, int TK>
__global__ void __launch_bounds__(NWARP * 32 + 32, 1)
    k_interp_mdict(const __grid_constant__ KGeom G, const __grid_constant__ CUtensorMap tmap,
                   const __grid_constant__ CUtensorMap omap, const float* __restrict__ in,
                   float* __restrict__ out, const int32_t* __restrict__ units,
                   const int32_t* __restrict__ cta_units, WS W) {
  constexpr int NCO = 1 << KO;
  constexpr int kMdictConsumers = NWARP * 32;
  constexpr int NW = NWARP;
  constexpr int KC = TK;
  constexpr int MB_ = MDICT_BUILD_BATCH;  // table-build tasks per thread per pass (loads in flight)
  if (W.range[2] != 0) return;  // non-finite input: write nothing
  if (ADAPT && W.dmeta[2] == 0) return;  // no usable dictionary: the edge-table blend runs
  extern __shared__ __align__(1024) unsigned char smem[];
  const PencilSmem P = pencil_smem(G, smem);
  const int n = G.n_bins;
  float* Ms = reinterpret_cast<float*>(P.tail);                  // [4 frames][NCO][2 columns][KC]
  uint2* dltS = reinterpret_cast<uint2*>(Ms + 2 * 4 * NCO * KC);  // ADAPT: [kDictHL]
  float* thrS = reinterpret_cast<float*>(dltS);                    // global: edge table [n + 1]
  int* ofS = reinterpret_cast<int*>(dltS + kDictHL);              // [NCO]
  const int ncol = (int)(G.P / 4);
  int* colT = reinterpret_cast<int*>(
      (reinterpret_cast<uintptr_t>(ofS + NCO) + 15) & ~uintptr_t(15));  // [ncol]
  float* colW = reinterpret_cast<float*>(colT + ((ncol + 3) & ~3));    // [ncol][4][2]
  // dictionary scalars in the dynamic tail: the kernel has no static shared
  // memory (1024-aligned, it would cost 1 KB of the opt-in and the fourth stage)
  int* scal = reinterpret_cast<int*>(colW + ncol * 8);
  int& s_dmode = scal[0];
  float& s_dv0 = reinterpret_cast<float*>(scal)[1];
  float& s_dS = reinterpret_cast<float*>(scal)[2];
  int& s_nv = scal[3];
  pipe_init(*P.pipe, G.nst, NW);
  __syncthreads();
  if (threadIdx.x >= kMdictConsumers) {
    if (threadIdx.x == kMdictConsumers)
      pipe_produce<KO, true, false, TSTORE, true, MDICT_NEXT != 0>(G, &tmap, units, 0, G.dyn_units, *P.pipe,
                                                  P.bufs, &omap,
                                                  reinterpret_cast<unsigned long long*>(&W.range[3]));
    return;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Dim& dl = G.d[G.rank - 1];
  for (int col = tid; col < ncol; col += kMdictConsumers) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t x = (int64_t)col * 4 + i;
      const int64_t c = cell_of(dl, x);
      const float f1 = (float)twice_dlo(dl, x, c) / (float)(2 * dl.b);
      if (i == 0) colT[col] = (int)(c * G.tstride[G.rank - 1]);
      colW[(col * 4 + i) * 2 + 0] = 1.0f - f1;
      colW[(col * 4 + i) * 2 + 1] = f1;
    }
  }
  if (ADAPT) {
    if (W.dmeta[4] == 2) {  // direct cells: the values' bits by cell (holes never match)
      // one copy per column, so a voxel's bits sit at a fixed offset from its table address
      uint32_t* bitsS = reinterpret_cast<uint32_t*>(dltS);
      static_assert(2 * KC * 4 <= kDictHL * 8, "two copies of the cell bits fit the lookup area");
      for (int k = tid; k < KC; k += kMdictConsumers)
        bitsS[k] = bitsS[KC + k] = k < W.dmeta[3] ? __float_as_uint(W.dvals[k]) : kDictEmpty;
    } else {
      for (int k = tid; k < kDictHL; k += kMdictConsumers) dltS[k] = W.dlt[k];
    }
    if (tid == 0) {
      s_dmode = W.dmeta[4];
      s_dv0 = __int_as_float(W.dmeta[5]);
      s_dS = __int_as_float(W.dmeta[6]);
      s_nv = min(W.dmeta[3], KC);
    }
  } else {
    for (int k = tid; k <= KC; k += kMdictConsumers) thrS[k] = W.thr[k];
    if (tid == 0) s_nv = KC;
  }
  consumers_sync<kMdictConsumers>();
  // dictionary constants in registers (not re-read from shared memory per item)
  const int dmode = ADAPT ? s_dmode : 0;
  const uint32_t ms32 = (uint32_t)__cvta_generic_to_shared(Ms);
  const float dv0 = ADAPT ? s_dv0 : 0.0f, dS = ADAPT ? s_dS : 0.0f;
  const TileParam<float> g0 = reinterpret_cast<const TileParam<float>*>(W.tparams)[0];
  const float2 glc = tile_lc(g0);
  const bool patho = !ADAPT && isnan(glc.y);  // a range the float guard does not cover
  const float* lsrc = ADAPT ? W.lutd : W.lut;  // rows of KC per tile
  const int tstr1 = (int)G.tstride[G.rank - 1];  // trailing corner: next tile of the last dim
  const int64_t stage_elems = G.stage_stride;
  const int rows = G.stage_rows;
  const int nrb = (rows + 31) >> 5;
  const int r1mask = G.r1 - 1, lg_r1 = G.lg_r1;  // per-item row split, kept in registers
  // a warp's 32 rows: 8 along dim KO-1 x 4 along dim KO-2 when the box has
  // them (neighbouring voxels along dim KO-2 share values more often than
  // those 16-32 rows apart along KO-1: ~8 % fewer gather wavefronts on the 4D
  // volume); 8 consecutive rows per 8 lanes keep the 32-byte swizzled stage
  // accesses conflict-free
  const bool l84 = lg_r1 >= 3 && (rows >> lg_r1) >= 4;
  const int h84 = lg_r1 - 3;
  // row of (row block rb, lane) = a warp-uniform part from rb plus a per-lane
  // constant, for both lane layouts: r1 = ((rb << rs1) & r1mask) + r1L,
  // r2 = ((rb >> rs2a) << rs2b) + r2L, q = (r2 << lg_r1) | r1
  const int rs1 = l84 ? 3 : 5;
  const int rs2a = l84 ? h84 : (lg_r1 >= 5 ? lg_r1 - 5 : 0);
  const int rs2b = l84 ? 2 : (lg_r1 >= 5 ? 0 : 5 - lg_r1);
  const int r1L = l84 ? (lane & 7) : (lane & r1mask);
  const int r2L = l84 ? (lane >> 3) : (lane >> lg_r1);
  const int qL = (r2L << lg_r1) | r1L;
  float ugs[KO], ugt[KO];
  int64_t cur = -1;
  int seg = 0;
  int rot = 0;  // round-robin offset of the item deal
  uint32_t it = 0;
  int cs_slot = 0;
  uint32_t cs_phase = 0;
  // the next work item, named by the record of the current item's last box
  // (pipe_produce NEXT): its tables are rebuilt as soon as this item is done,
  // while its first boxes are still in flight
  bool pend = false;
  int pend_seg = 0;
  int64_t pend_key = 0;
  int32_t pend_cell[KO] = {0};
  while (true) {
    const int s = cs_slot;  // it % nst, (it / nst) & 1 as counters: no division
    const Stage& S = P.pipe->st[s];
    bool build = pend;
    int32_t icell[KO];
    int iseg = pend_seg;
    int64_t ikey = pend_key;
#pragma unroll
    for (int j = 0; j < KO; ++j) icell[j] = pend_cell[j];
    if (!pend) {
      mbar_wait(&P.pipe->full[s], cs_phase);
      if (S.unit < 0) break;
      ikey = S.key * G.nseg + S.seg;
      if (ikey != cur) {  // first item (or an item whose predecessor did not name it)
        build = true;
        iseg = S.seg;
#pragma unroll
        for (int j = 0; j < KO; ++j) icell[j] = S.cell[j];
      }
    }
    if (build) {  // new work item: fold the two columns' corner pairs into M
      seg = iseg;
      // window tile of corner co's trailing row: of0 + sum_j bit_j(co) * tstride[j]
      int64_t of0 = (icell[0] - G.trow0) * G.tstride[0];
#pragma unroll
      for (int j = 1; j < KO; ++j) of0 += icell[j] * G.tstride[j];
      auto ofc = [&](int co) {
        int64_t of = of0;
#pragma unroll
        for (int j = 0; j < KO; ++j) of += ((co >> (KO - 1 - j)) & 1) * G.tstride[j];
        return of;
      };
      const int nv4 = (s_nv + 3) >> 2;
      const int ntask = ((MDICT_PROBE == 1 || MDICT_PROBE == 4) && cur >= 0) ? 0 : 2 * NCO * nv4;
      // a thread's tasks in batches of MB_: all 2 * MB_ L2 loads in flight first
      auto load = [&](int k0, float4 (&L0)[MB_], float4 (&L1)[MB_]) {
#pragma unroll
        for (int b = 0; b < MB_; ++b) {
          const int k = min(k0 + b * kMdictConsumers, ntask - 1);
          const int v4 = k % nv4, cc = k / nv4;  // cc = c * NCO + co
          const int c = cc / NCO, co = cc - c * NCO;
          const int64_t t0 = ofc(co) + colT[min(seg * 2 + c, ncol - 1)];
          L0[b] = __ldg(reinterpret_cast<const float4*>(lsrc + t0 * KC) + v4);
          L1[b] = __ldg(reinterpret_cast<const float4*>(lsrc + (t0 + tstr1) * KC) + v4);
        }
      };
      auto fold = [&](int k0, const float4 (&L0)[MB_], const float4 (&L1)[MB_]) {
#pragma unroll
        for (int b = 0; b < MB_; ++b) {
          const int k = k0 + b * kMdictConsumers;
          if (k >= ntask) break;
          const int v4 = k % nv4, cc = k / nv4;
          const int c = cc / NCO, co = cc - c * NCO;
          const int colc = min(seg * 2 + c, ncol - 1);
          const float a0[4] = {L0[b].x, L0[b].y, L0[b].z, L0[b].w};
          const float a1[4] = {L1[b].x, L1[b].y, L1[b].z, L1[b].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 tw = *reinterpret_cast<const float2*>(colW + (colc * 4 + i) * 2);
            float r[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) r[e] = fmaf(tw.y, a1[e], tw.x * a0[e]);
            reinterpret_cast<float4*>(Ms + ((i * NCO + co) * 2 + c) * KC)[v4] =
                make_float4(r[0], r[1], r[2], r[3]);
          }
        }
      };
      // the first batch's loads are issued BEFORE the barrier: they fly while the
      // slower warps finish the previous item (the tables are only written after it)
      float4 F0[MB_], F1[MB_];
      if (MDICT_EARLY_LOAD && tid < ntask) load(tid, F0, F1);
      consumers_sync<kMdictConsumers>();
      if (tid < NCO) ofS[tid] = (int)ofc(tid);
      if (MDICT_EARLY_LOAD && tid < ntask) fold(tid, F0, F1);
#pragma unroll 1
      for (int k0 = tid + (MDICT_EARLY_LOAD ? MB_ * kMdictConsumers : 0); k0 < ntask;
           k0 += MB_ * kMdictConsumers) {
        float4 L0[MB_], L1[MB_];
        load(k0, L0, L1);
        fold(k0, L0, L1);
      }
      consumers_sync<kMdictConsumers>();
      cur = ikey;
#pragma unroll
      for (int jd = 0; jd < KO; ++jd) {
        const Dim& d = G.d[jd];
        ugs[jd] = G.inv_b[jd];
        ugt[jd] = (float)(2 * d.before - 2 * (int64_t)icell[jd] * d.b - d.b + 1) * G.inv_2b[jd];
      }
    }
    if (pend) {  // tables ready: now wait for the item's first box
      pend = false;
      mbar_wait(&P.pipe->full[s], cs_phase);
      if (S.unit < 0) break;
    }
    // this item's last box names the next item (read before the stage is released)
    if (MDICT_NEXT && S.last && S.nunit >= 0) {
      pend = true;
      pend_seg = S.nseg;
      pend_key = S.nkey * G.nseg + S.nseg;
#pragma unroll
      for (int j = 0; j < KO; ++j) pend_cell[j] = S.ncell[j];
    }
    // outer weights exactly as k_interp_pencil computes them
    float wfix[NCO / 4];
    const float s1 = ugs[KO - 1], t1 = ugt[KO - 1];
    const float s2 = ugs[KO - 2], t2 = ugt[KO - 2];
    {
      float ff[KO - 2 > 0 ? KO - 2 : 1];
#pragma unroll
      for (int j = 0; j < KO - 2; ++j) ff[j] = fmaf((float)S.x[j], ugs[j], ugt[j]);
#pragma unroll
      for (int cf = 0; cf < NCO / 4; ++cf) {
        float w = 1.0f;
#pragma unroll
        for (int j = 0; j < KO - 2; ++j) w *= ((cf >> (KO - 3 - j)) & 1) ? ff[j] : 1.0f - ff[j];
        wfix[cf] = w;
      }
    }
    const int xb1 = S.x[KO - 1], xb2 = S.x[KO - 2];
    // results go straight to global memory (16 bytes per lane and row; a
    // stage is free once read, so loads never wait on a write-back)
    int64_t gbase = (int64_t)(S.x[0] - G.row0) * G.vstride[0];
#pragma unroll
    for (int j = 1; j < KO - 2; ++j) gbase += (int64_t)S.x[j] * G.vstride[j];
    gbase += (int64_t)xb2 * G.vstride[KO - 2] + (int64_t)xb1 * G.vstride[KO - 1];
    unsigned char* buf = reinterpret_cast<unsigned char*>(P.bufs + s * stage_elems);
    // items of consecutive stages dealt round-robin over the warps (the item
    // count need not be a multiple of NW).  TSTORE: an item is one 16-byte
    // column of a 32-row block, results in place (TMA-stored by the
    // producer).  Otherwise an item is a whole 32-row block: a lane blends
    // both columns of its row (one full 32-byte sector) and stores them
    // straight to global memory; the stage is released as soon as the warp's
    // last item has been read, so the producer refills it during the math.
    constexpr bool BOTH = TSTORE && (MDICT_BOTH == 1 || (MDICT_BOTH < 0 && !ADAPT));
    constexpr bool HALF = TSTORE && !BOTH;  // items are single columns
    const int nitems = HALF ? 2 * nrb : nrb;
    const int first = warp >= rot ? warp - rot : warp + NW - rot;
    rot += nitems % NW;  // items dealt so far, mod NW
    if (rot >= NW) rot -= NW;
    // one column's 4 voxels (frames) of row q against its tables
    auto blend_col = [&](const int c, const float4 v4, const float (&wo)[NCO]) -> float4 {
      if (MDICT_PROBE == 5) return v4;  // pipeline only: stage in, stage out
      const int col = seg * 2 + c;
      const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
      float acc[4];
      int miss = 0;  // voxels the dictionary does not hold (bit i)
      // ONE shared address per voxel, a = Ms + 4 * (c * KC + index): its 2^KO
      // folded-pair entries (and, for direct cells, the cell's value bits) sit at
      // compile-time offsets from it (LDS [reg + imm])
      const uint32_t mcs = ms32 + (uint32_t)(c * KC * 4);
      uint32_t a[4];
      bool direct = false;
      if constexpr (ADAPT) direct = dmode == 2;
      if (direct) {
        // direct cells: the cell's value bits (one copy per column) are checked
        // against the voxel; a voxel whose bits differ still gathers (valid cell,
        // wrong value) and is redone below
        constexpr int kBitsOff = 2 * 4 * NCO * KC * 4;  // dltS - Ms in bytes
        int cl[4];
        cl[0] = dict_cell<KC - 1>(vv[0], vv[1], dv0, dS, &cl[1]);
        cl[2] = dict_cell<KC - 1>(vv[2], vv[3], dv0, dS, &cl[3]);
        bool bad = false;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a[i] = mcs + 4u * (uint32_t)cl[i];
          bad |= lds_u32<kBitsOff>(a[i]) != __float_as_uint(vv[i]);
        }
        if (bad) {
#pragma unroll
          for (int i = 0; i < 4; ++i) miss |= (lds_u32<kBitsOff>(a[i]) != __float_as_uint(vv[i])) << i;
        }
      } else {
        int di[4];
        if (!ADAPT) {  // one bin per voxel: the global edge table
          if (!patho) {
            bins2_edge(pk2(vv[0], vv[1]), vv[0], vv[1], glc, thrS, KC, di[0], di[1]);
            bins2_edge(pk2(vv[2], vv[3]), vv[2], vv[3], glc, thrS, KC, di[2], di[3]);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) di[i] = bin_search(vv[i], thrS, KC);
          }
        } else if (dmode) {  // affine cells: one LDS.64 per voxel
          int cl[4];
          cl[0] = dict_cell(vv[0], vv[1], dv0, dS, &cl[1]);
          cl[2] = dict_cell(vv[2], vv[3], dv0, dS, &cl[3]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint2 e = dltS[cl[i]];
            di[i] = e.x == __float_as_uint(vv[i]) ? (int)e.y : -1;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) di[i] = dict_lookup(dltS, __float_as_uint(vv[i]));
        }
        if (ADAPT && (di[0] | di[1] | di[2] | di[3]) < 0) {  // a missing value is -1
#pragma unroll
          for (int i = 0; i < 4; ++i) miss |= (di[i] < 0) << i;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = mcs + 4u * (uint32_t)(ADAPT ? max(di[i], 0) : di[i]);
      }
      if (MDICT_PROBE == 2 || MDICT_PROBE >= 3) {
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = mcs + (MDICT_PROBE == 2 ? (a[i] & 0) : ((a[i] & 0) + 4 * lane));
      }
      {
        // two voxels per packed FFMA2 (same per-voxel order and rounding as
        // fmaf: acc = fma(wo[co], M, acc), co ascending)
        u64 acc01 = 0, acc23 = 0;
        static_for<0, NCO>([&](auto coc) {
          constexpr int co = decltype(coc)::value;
          constexpr int kOff = co * 2 * KC * 4, kFrame = NCO * 2 * KC * 4;
          float m[4];
          m[0] = lds_f32<kOff>(a[0]);
          m[1] = lds_f32<kOff + kFrame>(a[1]);
          m[2] = lds_f32<kOff + 2 * kFrame>(a[2]);
          m[3] = lds_f32<kOff + 3 * kFrame>(a[3]);
          const u64 w2 = pk2(wo[co], wo[co]);
          acc01 = fma2(pk2(m[0], m[1]), w2, acc01);
          acc23 = fma2(pk2(m[2], m[3]), w2, acc23);
        });
        upk2(acc01, acc[0], acc[1]);
        upk2(acc23, acc[2], acc[3]);
      }
      if (miss) {  // values the (sampled) dictionary lacks: from the workspace LUTs
        const int colc = min(col, ncol - 1);
        const int tt = colT[colc];
        float a[4] = {0.f, 0.f, 0.f, 0.f};
        static_for<0, NCO>([&](auto coc) {  // same order as the gathers above
          constexpr int co = decltype(coc)::value;
          const int t0 = ofS[co] + tt;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if ((miss >> i) & 1) {
              const float2 tw = *reinterpret_cast<const float2*>(colW + (colc * 4 + i) * 2);
              const float L0 = lut_value_global(W, n, t0, vv[i]);
              const float L1 = lut_value_global(W, n, t0 + tstr1, vv[i]);
              a[i] = fmaf(wo[co], fmaf(tw.y, L1, tw.x * L0), a[i]);
            }
        });
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if ((miss >> i) & 1) acc[i] = a[i];
      }
      float4 r;
      r.x = fminf(fmaxf(acc[0], 0.f), 1.f);
      r.y = fminf(fmaxf(acc[1], 0.f), 1.f);
      r.z = fminf(fmaxf(acc[2], 0.f), 1.f);
      r.w = fminf(fmaxf(acc[3], 0.f), 1.f);
      return r;
    };
    if (!TSTORE && first >= nitems) {  // no item for this warp in this stage
      __syncwarp();
      if (lane == 0) mbar_arrive(&P.pipe->empty[s]);
    }
    static_assert(NW % 2 == 0, "a warp's items of a stage share their column parity");
    const int c = HALF ? (first & 1) : 0;  // item & 1 for every item of this warp in this stage
    for (int item = first; item < nitems; item += NW) {
      const int rb = HALF ? item >> 1 : item;
      // stages hold a power of two >= 32 rows (plan_mdict): every lane has a row
      const int r1u = (rb << rs1) & r1mask, r2u = (rb >> rs2a) << rs2b;
      const int r1 = r1u + r1L, r2 = r2u + r2L;
      const int q = ((r2u << lg_r1) | r1u) + qL;
      const float f1 = fmaf((float)(xb1 + r1), s1, t1);
      const float f2 = fmaf((float)(xb2 + r2), s2, t2);
      // wo[co] = (g1[co & 1] * g2[(co >> 1) & 1]) * wfix[co >> 2], two corners per
      // packed multiply (same products, same rounding)
      float wo[NCO];
      {
        const u64 g1p = pk2(1.0f - f1, f1);
        const float g20 = 1.0f - f2;
        const u64 wa = mul2(g1p, pk2(g20, g20)), wb = mul2(g1p, pk2(f2, f2));
#pragma unroll
        for (int cf = 0; cf < NCO / 4; ++cf) {
          const u64 wf = pk2(wfix[cf], wfix[cf]);
          upk2(mul2(wa, wf), wo[4 * cf + 0], wo[4 * cf + 1]);
          upk2(mul2(wb, wf), wo[4 * cf + 2], wo[4 * cf + 3]);
        }
      }
      // 32B-swizzled stage row (32 bytes): 16-byte chunk c of row q at c ^ ((q >> 2) & 1)
      if constexpr (BOTH) {
        const int sw = (q >> 2) & 1;
        float4* pa = reinterpret_cast<float4*>(buf + q * 32 + (sw << 4));
        float4* pb = reinterpret_cast<float4*>(buf + q * 32 + ((1 ^ sw) << 4));
        const float4 va = *pa, vb = *pb;
        *pa = blend_col(0, va, wo);
        *pb = blend_col(1, vb, wo);
      } else if constexpr (TSTORE) {
        float4* slot4 = reinterpret_cast<float4*>(buf + q * 32 + ((c ^ ((q >> 2) & 1)) << 4));
        // in place; the producer TMA-stores the box
        *slot4 = blend_col(c, *slot4, wo);
      } else {
        const int sw = (q >> 2) & 1;
        const float4 va = *reinterpret_cast<const float4*>(buf + q * 32 + (sw << 4));
        const float4 vb = *reinterpret_cast<const float4*>(buf + q * 32 + ((1 ^ sw) << 4));
        if (item + NW >= nitems) {  // the warp's last read of this stage
          __syncwarp();
          if (lane == 0) mbar_arrive(&P.pipe->empty[s]);
        }
        const float4 ra = blend_col(0, va, wo);
        const float4 rbv = blend_col(1, vb, wo);
        float* o = out + gbase + (int64_t)r2 * G.vstride[KO - 2] + (int64_t)r1 * G.vstride[KO - 1] +
                   seg * 8;
        if (seg * 2 < ncol) __stcs(reinterpret_cast<float4*>(o), ra);
        if (seg * 2 + 1 < ncol) __stcs(reinterpret_cast<float4*>(o) + 1, rbv);
      }
    }
    if (TSTORE) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&P.pipe->empty[s]);
    }
    ++it;
    if (++cs_slot == G.nst) {
      cs_slot = 0;
      cs_phase ^= 1;
    }
  }
}

PencilInterpFn get_interp_mdict(int ko, bool tma_store, bool adaptive, int n_bins) {
  if (ko != 3) return nullptr;
  if (adaptive)
    return tma_store ? k_interp_mdict<3, true, MDICT_NWARP_ADAPT, true, kDictKC>
                     : k_interp_mdict<3, false, MDICT_NWARP_ADAPT, true, kDictKC>;
  switch (n_bins) {
    case 128: return tma_store ? k_interp_mdict<3, true, MDICT_NWARP_GLOBAL, false, 128> : k_interp_mdict<3, false, MDICT_NWARP_GLOBAL, false, 128>;
    case 256: return tma_store ? k_interp_mdict<3, true, MDICT_NWARP_GLOBAL, false, 256> : k_interp_mdict<3, false, MDICT_NWARP_GLOBAL, false, 256>;
    case 512: return tma_store ? k_interp_mdict<3, true, MDICT_NWARP_GLOBAL, false, 512> : k_interp_mdict<3, false, MDICT_NWARP_GLOBAL, false, 512>;
    default: return nullptr;
  }
}

int interp_mdict_threads(bool adaptive) {
  return (adaptive ? MDICT_NWARP_ADAPT : MDICT_NWARP_GLOBAL) * 32 + 32;
}

}  // namespace mg
