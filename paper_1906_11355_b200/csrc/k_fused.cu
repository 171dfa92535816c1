// k_fused.cu -- fused adaptive K2: per-tile ranges and counts from ONE HBM
// read of the input (single-slab float32 adaptive pencil plans).
//
// The reference derives a tile's range and its histogram from the same block
// (src/histogram.cpp:86-99: min/max of the block, then compute_histogram over
// it).  The two-pass build (K2a k_range_pencil, then K2b k_hist_pencil after
// k_params / k_thresholds) streams the volume from HBM twice.  Here one
// persistent kernel walks every unit twice:
//
//   range walk    TMA-stage the unit's support boxes from HBM (L2 evict_last),
//                 per-tile min/max, the dictionary sample and the finiteness
//                 check (as K2a); the unit then arrives on its tile GROUP (the
//                 units sharing one key: one KO-outer tile, every trailing
//                 tile).  When the last unit of a group arrives, the group's
//                 binning parameters and bin-edge tables are built (k_params +
//                 k_thresholds, exact f64 rule) and published (release flag).
//   count walk    once the group is published, the same boxes again -- read a
//                 few microseconds earlier, so from L2 -- counted exactly as
//                 K2b does.
//
// The range walk of one unit and the count walk of an earlier one interleave
// box by box, so every CTA keeps streaming from HBM while it counts from L2.
// Units are small (the bytes between a box's two reads must fit L2 over all
// CTAs), so the per-unit bookkeeping is taken off the consumer warps: the CTA
// is 8 consumer warps + a producer warp (TMA) + a bookkeeping warp (flushes
// ranges, arrives on groups, stages the count walk's tables, flushes and
// zeroes histograms), talking through mbarriers and a shared-memory event
// ring; histograms, tables and range slots are double-buffered.  The f64
// edge-table build of a completed group is shared by the consumer warps (1/8
// each, picked up between stages): one warp alone would take tens of
// microseconds.
//
// Units are handed out in order by an atomic counter and a group's units are
// consecutive, so a unit waits only for units already handed out to running
// CTAs (no deadlock while at least max-units-per-group CTAs run: host check).
// Counts are integer sums: bit-identical to K2a + K2b.
#include "k_pencil.cuh"
#ifdef FK2_WATCHDOG
#include <cstdio>
#endif

namespace mg {

constexpr int kFusedThreads = kConsumers + 64;  // + producer warp + bookkeeping warp
constexpr int kEvRing = 16;
constexpr int kNRS = 4;  // range slots = units allowed between their two walks
enum { EV_RANGE = 0, EV_FLUSH = 2, EV_QUIT = 3 };

// One unit walk of the producer (in shared memory: the single producer
// thread's registers would count against every consumer thread).
struct FWalk {
  int32_t u;  // unit (-1: idle)
  int32_t grp;
  int64_t key;
  int64_t a[kMaxOuterDims];
  int32_t ext[kMaxOuterDims];
  TileParts parts[kMaxOuterDims];
  int32_t nfix, f, bi, nbox;
  int32_t n1, n2, i1, i2;
};

struct FCtl {
  uint64_t rdone[kNRS];  // consumers' last stage of a range walk in slot b (8 warps)
  uint64_t hdone[2];  // ... of a count walk into histogram buffer b
  uint64_t pdone;     // consumer warps' shares of a group's edge tables (8 warps)
  int ev_type[kEvRing], ev_unit[kEvRing], ev_buf[kEvRing], ev_seq[kEvRing];
  int ev_head, ev_tail;  // producer / bookkeeper ring positions
  int r_fin;             // range walks finalised (bookkeeper -> producer)
  int h_free[2];         // count walk seq + 1 last flushed out of buffer b
  int p_seq;             // edge-table build requests (bookkeeper -> consumers)
  int64_t p_key;         // ... the group's first tile
  int p_grp;             // ... and the group
  FWalk walks[2];
  // unit records in shared memory (global loads would stall the producer)
  int32_t rnext[kUnitInts + 2];           // prefetched (cp.async) record of the next unit
  int32_t rcur[kUnitInts + 2];            // the range walk's unit
  int32_t prec[kNRS][kUnitInts + 2];      // units between their walks (ring)
  int pend_u[kNRS];
  int pend_head, pend_tail;               // producer-owned ring positions
  int front;                              // bookkeeper: (unit << 2) | 1 group published, | 2 skip
};

// A group's count-walk tables, built once (group_tables) into an aligned
// workspace block so one bulk copy stages them: [gtr] TileParam<float>, then
// [gtr][n1p] bin-edge rows (n1p = n + 1 rounded up to 4 floats).
__host__ __device__ __forceinline__ int64_t ftab_n1p(int64_t n) { return (n + 1 + 3) & ~int64_t(3); }
__host__ __device__ __forceinline__ int64_t ftab_bytes(int64_t gtr, int64_t n) {
  return gtr * 16 + gtr * ftab_n1p(n) * 4;
}

template <int KO>
__device__ __forceinline__ int64_t unit_key(const KGeom& G, const int32_t* U) {
  int64_t key = (U[0] - G.trow0) * G.tstride[0];
#pragma unroll
  for (int j = 1; j < KO; ++j) key += (int64_t)U[j] * G.tstride[j];
  return key;
}

template <int KO>
__device__ __forceinline__ void fwalk_start(const KGeom& G, const int32_t* U, int u, FWalk& w) {
  w.u = u;
  w.grp = U[6];
  w.key = unit_key<KO>(G, U);
  w.a[0] = U[8];
  w.ext[0] = U[9] - U[8];
  w.parts[0] = tile_parts(G.d[0], U[0]);
#pragma unroll 1
  for (int j = 1; j < KO; ++j) {
    w.parts[j] = tile_parts(G.d[j], U[j]);
    w.a[j] = w.parts[j].support_begin();
    w.ext[j] = (int32_t)(w.parts[j].support_end() - w.a[j]);
  }
  int32_t nfix = 1;
#pragma unroll 1
  for (int j = 0; j < KO - 2; ++j) nfix *= w.ext[j];
  w.nfix = nfix;
  w.n1 = w.ext[KO - 1] / G.r1;
  w.n2 = KO >= 2 ? w.ext[KO - 2] / G.r2 : 1;
  w.f = 0;
  w.i1 = w.i2 = 0;
  w.bi = 0;
  w.nbox = nfix * w.n1 * w.n2;
}

// FK2_WATCHDOG (debug builds): a wait longer than 0.5 s prints the waiting
// role's state and traps, so a scheduling deadlock shows up as an error
// instead of a hung GPU.
#ifdef FK2_WATCHDOG
__device__ __forceinline__ uint64_t wd_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define WD_BEGIN uint64_t wd_t0 = wd_now();
#define WD_CHECK(...)                            \
  if (wd_now() - wd_t0 > 500000000ull) {         \
    printf(__VA_ARGS__);                         \
    __trap();                                    \
  }
#else
#define WD_BEGIN
#define WD_CHECK(...)
#endif
// One thread's wait (the producer).
__device__ __forceinline__ void mbar_wait_wd1(uint64_t* bar, uint32_t parity, int who) {
  WD_BEGIN
  while (!mbar_try_wait(bar, parity)) {
    WD_CHECK("cta %d: %d waits on an mbarrier (parity %u)\n", blockIdx.x, who, parity)
  }
}
// Warp-wide wait (every lane leaves together).
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity, int who) {
  WD_BEGIN
  while (!__all_sync(0xffffffffu, mbar_try_wait(bar, parity))) {
    WD_CHECK("cta %d: %d waits on an mbarrier (parity %u)\n", blockIdx.x, who, parity)
  }
}

__device__ __forceinline__ int ld_relaxed_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ int vld(const int& x) { return *reinterpret_cast<const volatile int*>(&x); }
__device__ __forceinline__ void vst(int& x, int v) { *reinterpret_cast<volatile int*>(&x) = v; }

// ------------------------------------------------------------ producer ----
template <int KO>
__device__ __noinline__ void produce_fused(const KGeom& G, const CUtensorMap* map,
                                           const int32_t* __restrict__ units, int nunits,
                                           Pipe& pp, float* bufs, unsigned long long* dyn,
                                           const TileParam<float>* tparams,
                                           const int32_t* gready, const float* gtab,
                                           float* htab0, float* htab1, FCtl& ctl) {
  const int nst = G.nst;
  const bool segv = G.tma_rank - KO == 2;
  const int32_t row0 = (int32_t)G.row0;
  const int64_t stage_elems = G.stage_stride;
  const uint32_t box_bytes = (uint32_t)((int64_t)G.stage_rows * G.P * 4);
  const int R1 = G.r1, R2 = G.r2;
  uint64_t pol_keep, pol_drop;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_drop));
  FWalk& wr = ctl.walks[0];
  FWalk& wh = ctl.walks[1];
  wr.u = -1;
  wh.u = -1;
  int npend = 0, ptail = 0, phead = 0;
  int nr = 0, nh = 0;    // range / count walks started
  bool r_done = false, turn = false;
  // The next unit is taken from the counter ahead of time only when it can
  // start without waiting for any group (room for it between the walks);
  // a unit held but not started while this CTA waits on groups could close a
  // wait cycle with another CTA (handing out in order is what rules them out).
  int next_u = (int)atomicAdd(dyn, 1ULL);
  bool have_next = true, pf = false;
  int ev = 0;
  auto push = [&](int type, int unit, int buf, int seq) {
    WD_BEGIN
    while (ev - vld(ctl.ev_tail) >= kEvRing) {
      __nanosleep(64);
      WD_CHECK("cta %d: producer ring full ev %d tail %d\n", blockIdx.x, ev, vld(ctl.ev_tail))
    }
    const int k = ev % kEvRing;
    ctl.ev_type[k] = type;
    ctl.ev_unit[k] = unit;
    ctl.ev_buf[k] = buf;
    ctl.ev_seq[k] = seq;
    __threadfence_block();
    vst(ctl.ev_head, ++ev);
  };
  auto copy_rec = [](int32_t* d, const int32_t* s_) {
#pragma unroll
    for (int i = 0; i < kUnitInts; ++i) d[i] = s_[i];
  };
  int slot = 0;
  uint32_t phase = 0;
#ifdef FK2_WATCHDOG
  long idle_spins = 0;
  WD_BEGIN
#endif
#pragma unroll 1
  while (true) {
    // next range walk: its min/max slot (nr % kNRS) must be finalised (walk
    // nr - kNRS), and at most kNRS - 1 units wait between their walks (L2)
    if (wr.u < 0 && !r_done && npend < kNRS - 1 && vld(ctl.r_fin) >= nr - kNRS + 1) {
      if (!have_next) {
        next_u = (int)atomicAdd(dyn, 1ULL);
        pf = false;
      }
      have_next = false;
      if (next_u >= nunits) {
        r_done = true;
      } else {
        if (!pf) {
          copy_rec(ctl.rcur, units + (int64_t)next_u * kUnitInts);
        } else {
          asm volatile("cp.async.wait_all;" ::: "memory");
          copy_rec(ctl.rcur, ctl.rnext);
        }
        fwalk_start<KO>(G, ctl.rcur, next_u, wr);
        ++nr;
        if (npend <= kNRS - 3) {  // it will be startable: take it now, record after the next box
          next_u = (int)atomicAdd(dyn, 1ULL);
          have_next = true;
          pf = false;
        }
      }
    }
    // next count walk: group published (the bookkeeper polls it) and the
    // histogram buffer flushed; its tables ride on the walk's first box
    bool hfirst = false;
    if (wh.u < 0 && npend > 0 && (nh < 2 || vld(ctl.h_free[nh & 1]) >= nh - 1)) {
      const int pos = phead % kNRS;
      const int u = ctl.pend_u[pos];
      const int fr = vld(ctl.front);
      if ((fr >> 2) == u && (fr & 3) != 0) {
        ++phead;
        --npend;
        vst(ctl.pend_head, phead);
        if ((fr & 3) == 2) continue;  // every tile degenerate: not counted at all
        fwalk_start<KO>(G, ctl.prec[pos], u, wh);
        ++nh;
        hfirst = true;
      }
    }
    const bool canR = wr.u >= 0, canH = wh.u >= 0;
    if (!canR && !canH) {
      if (r_done && npend == 0) break;
      __nanosleep(128);
#ifdef FK2_WATCHDOG
      if (++idle_spins > 2000000)
        WD_CHECK("cta %d: producer idle nr %d nh %d npend %d r_done %d next_u %d have %d r_fin %d front %d "
                 "pend_u %d h_free %d %d grp %d ready %d\n",
                 blockIdx.x, nr, nh, npend, (int)r_done, next_u, (int)have_next, vld(ctl.r_fin),
                 vld(ctl.front), ctl.pend_u[phead % kNRS], vld(ctl.h_free[0]), vld(ctl.h_free[1]),
                 ctl.prec[phead % kNRS][6], ld_relaxed_gpu(gready + ctl.prec[phead % kNRS][6]))
#endif
      continue;
    }
    const bool doH = hfirst || (canH && (!canR || turn));
    turn = !doH;
    FWalk& w = doH ? wh : wr;
    // box (f, i2, i1) of the walk
    int32_t xf[kMaxOuterDims];
    int32_t wfix = 1;
    int32_t rem = w.f;
#pragma unroll
    for (int j = KO - 3; j >= 0; --j) {
      xf[j] = (int32_t)w.a[j] + rem % w.ext[j];
      rem /= w.ext[j];
      wfix *= w.parts[j].weight(xf[j]);
    }
    const int32_t x1 = (int32_t)w.a[KO - 1] + w.i1 * R1;
    const int32_t x2 = KO >= 2 ? (int32_t)w.a[KO >= 2 ? KO - 2 : 0] + w.i2 * R2 : 0;
    const bool lastbox = ++w.bi == w.nbox;
    if (++w.i1 == w.n1) {
      w.i1 = 0;
      if (++w.i2 == w.n2) {
        w.i2 = 0;
        ++w.f;
      }
    }
    const int buf = doH ? ((nh - 1) & 1) : ((nr - 1) % kNRS);
    mbar_wait_wd1(&pp.empty[slot], phase ^ 1, 1);
    Stage& S = pp.st[slot];
    S.unit = w.u;
    S.seg = buf;
    S.key = w.key;
    S.ph = doH ? 1 : 0;
    S.last = lastbox ? 1 : 0;
#pragma unroll
    for (int j = 0; j < KO - 2; ++j) S.x[j] = xf[j];
    S.x[KO - 1] = x1;
    if (KO >= 2) S.x[KO >= 2 ? KO - 2 : 0] = x2;
    const TileParts p1 = w.parts[KO - 1];
    S.p1 = p1;
    TileParts p2;
    if (KO >= 2) {
      p2 = w.parts[KO >= 2 ? KO - 2 : 0];
      S.p2 = p2;
    }
    const bool uni = parts_uniform(p1, x1, R1) && (KO < 2 || parts_uniform(p2, x2, R2));
    S.wuni = uni ? 1 : 0;
    S.wfix = uni ? wfix * p1.weight(x1) * (KO >= 2 ? p2.weight(x2) : 1) : wfix;
    int c[6];
    int co[KO];
#pragma unroll
    for (int j = 0; j < KO; ++j)
      co[j] = j == KO - 1 ? x1 : (KO >= 2 && j == KO - 2 ? x2 : xf[j < KO - 2 ? j : 0]);
    co[0] -= row0;
    c[0] = 0;
    if (segv) {
      c[1] = 0;
#pragma unroll
      for (int j = 0; j < KO; ++j) c[2 + j] = co[KO - 1 - j];
    } else {
#pragma unroll
      for (int j = 0; j < KO; ++j) c[1 + j] = co[KO - 1 - j];
    }
    if (hfirst) {  // the group's tables into the walk's buffer with this box
      const uint32_t tb = (uint32_t)ftab_bytes(G.gtr, G.n_bins);
      mbar_expect_tx(&pp.full[slot], box_bytes + tb);
      bulk_g2s(buf ? htab1 : htab0, gtab + (int64_t)wh.grp * (tb / 4), tb, &pp.full[slot]);
    } else {
      mbar_expect_tx(&pp.full[slot], box_bytes);
    }
    tma_load_hint(bufs + slot * stage_elems, map, G.tma_rank, c, &pp.full[slot],
                  doH ? pol_drop : pol_keep);
    if (++slot == nst) {
      slot = 0;
      phase ^= 1;
    }
    if (lastbox) {
      if (doH) {
        push(EV_FLUSH, w.u, buf, nh - 1);
        wh.u = -1;
      } else {
        const int pos = ptail % kNRS;
        ctl.pend_u[pos] = w.u;
        copy_rec(ctl.prec[pos], ctl.rcur);
        __threadfence_block();
        vst(ctl.pend_tail, ++ptail);
        ++npend;
        push(EV_RANGE, w.u, buf, nr - 1);
        wr.u = -1;
      }
    }
    if (have_next && !pf && next_u < nunits) {  // the next unit's record, async into shared memory
      const uint32_t d = smem_u32(ctl.rnext);
      const int32_t* src = units + (int64_t)next_u * kUnitInts;
#pragma unroll
      for (int i = 0; i < kUnitInts / 2; ++i)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d + 8 * i), "l"(src + 2 * i)
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      pf = true;
    }
  }
  push(EV_QUIT, -1, 0, 0);
  mbar_wait(&pp.empty[slot], phase ^ 1);
  pp.st[slot].unit = -1;
  mbar_arrive(&pp.full[slot]);
}

// Shared-memory layout of the fused kernel's tail (after the stages).
struct FTail {
  uint32_t* hist[2];  // [gtr][n + 1]
  float* tab[2];      // the count walk's tables (ftab_bytes: TileParams, then edge rows)
  int32_t* rmin[kNRS];  // [gtr] ~key32(lo)
  int32_t* rmax[kNRS];  // [gtr] key32(hi)
  uint32_t dummy_s;   // shared address of [kConsumers] discard words (run tails)
  uint32_t* sset;     // dictionary sample set
};

__device__ __forceinline__ FTail fused_tail(const KGeom& G, unsigned char* p) {
  FTail t;
  const int64_t hb = (G.gtr * (G.n_bins + 1) * 4 + 15) & ~15LL;
  const int64_t tb = ftab_bytes(G.gtr, G.n_bins);
  const int64_t lb = (G.gtr * 8 + 15) & ~15LL;
  for (int b = 0; b < 2; ++b) {
    t.tab[b] = reinterpret_cast<float*>(p);
    p += tb;
    t.hist[b] = reinterpret_cast<uint32_t*>(p);
    p += hb;
  }
  for (int b = 0; b < kNRS; ++b) {
    t.rmin[b] = reinterpret_cast<int32_t*>(p);
    t.rmax[b] = t.rmin[b] + G.gtr;
    p += lb;
  }
  t.dummy_s = (uint32_t)__cvta_generic_to_shared(p);
  p += kConsumers * 4;
  t.sset = reinterpret_cast<uint32_t*>(p);
  return t;
}

__device__ __forceinline__ TileParam<float> tab_tp(const float* tab, int t) {
  const float4 q = reinterpret_cast<const float4*>(tab)[t];
  TileParam<float> tp;
  tp.lo = q.x;
  tp.hi = q.y;
  tp.c = q.z;
  tp.lim = q.w;
  return tp;
}

// Edge tables + binning parameters of tiles [key, key + gtr) from their
// published ranges (k_params + k_thresholds), entries i0, i0 + step, ...
__device__ __forceinline__ void group_tables(const KGeom& G, WS W, int64_t key, int64_t grp, int i0,
                                             int step) {
  const int n = G.n_bins, n1 = n + 1;
  const int n1p = (int)ftab_n1p(n);
  TileParam<float>* tparams = reinterpret_cast<TileParam<float>*>(W.tparams);
  float* tab = W.k2tab + grp * (ftab_bytes(G.gtr, n) / 4);
  TileParam<float>* ttp = reinterpret_cast<TileParam<float>*>(tab);
  float* tthr = tab + G.gtr * 4;
  long long mkey = LLONG_MIN;
  for (int64_t t = i0; t < G.gtr; t += step) {
    const long long* r = reinterpret_cast<const long long*>(W.trange + 2 * (key + t));
    const long long r0 = __ldcg(r), r1 = __ldcg(r + 1);
    const TileParam<float> p = make_tile_param<float>(okey_decode(~r0), okey_decode(r1), n);
    tparams[key + t] = p;
    ttp[t] = p;
    if (r0 != LLONG_MIN) mkey = max(mkey, r0);
  }
  // the group's ranges: one load per lane, then shuffled to each entry's lane
  const int lane = threadIdx.x & 31;
  const bool bc = G.gtr <= 32;
  long long q0 = 0, q1 = 0;
  if (bc && lane < G.gtr) {
    const long long* r = reinterpret_cast<const long long*>(W.trange + 2 * (key + lane));
    q0 = __ldcg(r);
    q1 = __ldcg(r + 1);
  }
  const int64_t total = G.gtr * n1;
  for (int64_t b0 = i0 - lane; b0 < total; b0 += step) {  // warp-uniform trip count
    const int64_t i = b0 + lane;
    const int64_t t = (i < total ? i : total - 1) / n1;
    const int k = (int)(i - t * n1);
    long long r0, r1;
    if (bc) {
      r0 = __shfl_sync(0xffffffffu, q0, (int)t);
      r1 = __shfl_sync(0xffffffffu, q1, (int)t);
    } else {
      const long long* r = reinterpret_cast<const long long*>(W.trange + 2 * (key + t));
      r0 = __ldcg(r);
      r1 = __ldcg(r + 1);
    }
    if (i >= total) continue;
    const TileParam<float> p = make_tile_param<float>(okey_decode(~r0), okey_decode(r1), n);
    const float th = k == n ? INFINITY
                            : (k == 0 || tp_degenerate(p.lim))
                                  ? -INFINITY
                                  : bin_threshold((double)p.lo, (double)p.hi, n, k);
    W.thr[key * n1 + i] = th;
    tthr[t * n1p + k] = th;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mkey = max(mkey, __shfl_xor_sync(0xffffffffu, mkey, o));
  if ((threadIdx.x & 31) == 0 && mkey != LLONG_MIN)
    atomicMax(reinterpret_cast<long long*>(&W.range[0]), mkey);
}

// ---------------------------------------------------------- bookkeeper ----
template <int KO>
__device__ __noinline__ void bookkeep(const KGeom& G, WS W, const int32_t* __restrict__ units,
                                      FCtl& ctl, const FTail& T) {
  const int lane = threadIdx.x & 31;
  const int n = G.n_bins, n1 = n + 1;
  const int gtr = (int)G.gtr;
  int32_t* gcnt = W.k2g;
  int32_t* gready = W.k2g + G.win_tiles / G.gtr;
  uint32_t rpar[kNRS] = {0, 0, 0, 0}, hpar[2] = {0, 0}, ppar = 0;
  int pseq = 0;
  int pub = -1;  // group whose edge tables the consumer warps are building
  // publish a completed build: tables visible device-wide, then the flag
  const TileParam<float>* tparams = reinterpret_cast<const TileParam<float>*>(W.tparams);
  // the producer's oldest waiting unit: poll its group's flag (relaxed; the
  // latency is the bookkeeper's, not the producer's) and tell the producer
  // once it is published, and whether every tile of the unit is degenerate
  auto poll_front = [&]() {
    int st = 0, u = -1;
    if (lane == 0) {
      const int h = vld(ctl.pend_head);
      if (h < vld(ctl.pend_tail)) {
        const int pos = h % kNRS;
        u = vld(ctl.pend_u[pos]);
        if ((vld(ctl.front) >> 2) != u && ld_relaxed_gpu(gready + ctl.prec[pos][6]) != 0) {
          fence_acq_rel_gpu();
          const int64_t key = unit_key<KO>(G, ctl.prec[pos]);
          bool all = true;
          for (int t = 0; t < gtr && all; ++t) all = tp_degenerate(__ldcg(&tparams[key + t].lim));
          st = all ? 2 : 1;
        }
      }
      if (st) vst(ctl.front, (u << 2) | st);
    }
    __syncwarp();
  };
  auto publish = [&]() {
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicExch(&gready[pub], 1);
    pub = -1;
    ppar ^= 1;
  };
#pragma unroll 1
  for (int tail = 0;; ++tail) {
    // every decision is lane 0's, broadcast: the warp's control flow (and
    // with it pub / ppar) stays uniform
    WD_BEGIN
    while (__shfl_sync(0xffffffffu, vld(ctl.ev_head), 0) <= tail) {
      if (pub >= 0 && __shfl_sync(0xffffffffu, (int)mbar_try_wait(&ctl.pdone, ppar), 0)) publish();
      poll_front();
      __nanosleep(32);
      WD_CHECK("cta %d: bookkeeper idle tail %d pub %d pseq %d\n", blockIdx.x, tail, pub, pseq)
    }
    poll_front();
    __threadfence_block();
    const int k = tail % kEvRing;
    const int type = ctl.ev_type[k], unit = ctl.ev_unit[k], b = ctl.ev_buf[k], seq = ctl.ev_seq[k];
    __syncwarp();
    if (lane == 0) vst(ctl.ev_tail, tail + 1);
    if (type == EV_QUIT) {
      if (pub >= 0) {
#ifdef FK2_WATCHDOG
        if (lane == 0)
          printf("cta %d: quit with build of group %d pending: gcnt %d gready %d pseq %d units %d\n",
                 blockIdx.x, pub, ld_relaxed_gpu(gcnt + pub), ld_relaxed_gpu(gready + pub), pseq,
                 0);
#endif
        mbar_wait_wd(&ctl.pdone, ppar, 20);
        publish();
      }
      return;
    }
    const int32_t* U = units + (int64_t)unit * kUnitInts;
    const int64_t key = unit_key<KO>(G, U);
    if (type == EV_RANGE) {
      mbar_wait_wd(&ctl.rdone[b], rpar[b], 21);
      rpar[b] ^= 1;
      for (int t = lane; t < gtr; t += 32) {
        const int32_t mn = T.rmin[b][t], mx = T.rmax[b][t];
        if (mx != INT32_MIN) {
          long long* r = reinterpret_cast<long long*>(W.trange + 2 * (key + t));
          atomicMax(r, (long long)~okey((double)key32_decode(~mn)));
          atomicMax(r + 1, (long long)okey((double)key32_decode(mx)));
        }
        T.rmin[b][t] = T.rmax[b][t] = INT32_MIN;
      }
      __threadfence();
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        const int old = atomicAdd(&gcnt[U[6]], 1);
        last = old == U[7] - 1;
#ifdef FK2_WATCHDOG
        if (old >= U[7]) printf("cta %d: group %d over-arrived: %d of %d (unit %d)\n", blockIdx.x, U[6], old + 1, U[7], unit);
#endif
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        // the group's edge tables: 1/8 per consumer warp, picked up between
        // stages; published once all eight are in (one build in flight)
        if (pub >= 0) {
          mbar_wait_wd(&ctl.pdone, ppar, 22);
          publish();
        }
        __threadfence();
        if (lane == 0) {
          *reinterpret_cast<volatile int64_t*>(&ctl.p_key) = key;
          vst(ctl.p_grp, U[6]);
          __threadfence_block();
          vst(ctl.p_seq, ++pseq);
        }
        pub = U[6];
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        vst(ctl.r_fin, seq + 1);
      }
    } else {  // EV_FLUSH: the count walk's histogram into the workspace, then zeroed
      mbar_wait_wd(&ctl.hdone[b], hpar[b], 23);
      hpar[b] ^= 1;
      uint32_t* h = T.hist[b];
#pragma unroll 1
      for (int t = 0; t < gtr; ++t) {
        // degenerate tiles are counted by the hot path but never used
        const bool deg = tp_degenerate(tab_tp(T.tab[b], t).lim);
        uint32_t* dst = W.counts + (key + t) * n;
        uint32_t* row = h + t * n1;
        int kb = lane;
#pragma unroll 1
        for (; kb + 7 * 32 < n; kb += 8 * 32) {
          uint32_t c[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) c[j] = row[kb + j * 32];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (c[j]) {
              if (!deg) atomicAdd(dst + kb + j * 32, c[j]);
              row[kb + j * 32] = 0;
            }
        }
        for (; kb < n; kb += 32) {
          const uint32_t c = row[kb];
          if (c) {
            if (!deg) atomicAdd(dst + kb, c);
            row[kb] = 0;
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        vst(ctl.h_free[b], seq + 1);
      }
    }
  }
}

// ------------------------------------------------------------- kernel ----
template <int KO, bool DICT>
__global__ void __launch_bounds__(kFusedThreads, 2)
    k_k2_fused(const __grid_constant__ KGeom G, const __grid_constant__ CUtensorMap tmap,
               const float* __restrict__ in, const int32_t* __restrict__ units,
               const int32_t* __restrict__ cta_units, WS W) {
  extern __shared__ __align__(128) unsigned char smem[];
  const PencilSmem P = pencil_smem(G, smem);
  const FTail T = fused_tail(G, P.tail);
  const int n = G.n_bins;
  const int n1 = n + 1;
  __shared__ FCtl ctl;
  __shared__ int s_n, s_over;
  uint32_t* sset = T.sset;
  if (DICT) {
    for (int k = threadIdx.x; k < kDictHS; k += blockDim.x) sset[k] = kDictEmpty;
    if (threadIdx.x == 0) s_n = s_over = 0;
  }
  for (int b = 0; b < 2; ++b)
    for (int k = threadIdx.x; k < G.gtr * n1; k += blockDim.x) T.hist[b][k] = 0;
  for (int b = 0; b < kNRS; ++b)
    for (int t = threadIdx.x; t < G.gtr; t += blockDim.x) T.rmin[b][t] = T.rmax[b][t] = INT32_MIN;
  if (threadIdx.x == 0) {
    for (int b = 0; b < kNRS; ++b) mbar_init(&ctl.rdone[b], kConsumers / 32);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ctl.hdone[b], kConsumers / 32);
      ctl.h_free[b] = 0;
    }
    mbar_init(&ctl.pdone, kConsumers / 32);
    ctl.ev_head = ctl.ev_tail = 0;
    ctl.r_fin = 0;
    ctl.p_seq = 0;
    ctl.pend_head = ctl.pend_tail = 0;
    ctl.front = -4;
  }
  pipe_init(*P.pipe, G.nst);
  __syncthreads();
  TileParam<float>* tparams = reinterpret_cast<TileParam<float>*>(W.tparams);
  if (threadIdx.x >= kConsumers + 32) {
    bookkeep<KO>(G, W, units, ctl, T);
    return;
  }
  if (threadIdx.x >= kConsumers) {
    if (threadIdx.x == kConsumers)
      produce_fused<KO>(G, &tmap, units, G.dyn_units, *P.pipe, P.bufs,
                        reinterpret_cast<unsigned long long*>(&W.range[3]), tparams,
                        W.k2g + G.win_tiles / G.gtr, W.k2tab, T.tab[0], T.tab[1], ctl);
    return;
  }
  const int tid = threadIdx.x, lane = tid & 31;
  const int slot = tid / G.tpr;
  const int64_t e0 = (int64_t)(tid % G.tpr) * 4;
  const bool lane_on = slot < G.rpi;
  const int64_t stage_elems = G.stage_stride;
  const int trips = slot < G.stage_rows ? (G.stage_rows - slot + G.rpi - 1) / G.rpi : 0;
  const uint32_t dummy_s = T.dummy_s + 4u * tid;
  int trt[4], trw[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) trailing_tile(G, e0 + i, &trt[i], &trw[i]);
  const bool same_pairs = trt[0] == trt[1] && trt[2] == trt[3];
  const float kDegC = degenerate_lc().y;

  auto dict_add = [&](float f) {  // bucketised insert, as k_range_pencil
    const uint32_t b = __float_as_uint(f);
    uint32_t bk = dict_hash(b, kDictLgBS);
    const uint4 q = reinterpret_cast<const uint4*>(sset)[bk];
    if (q.x == b || q.y == b || q.z == b || q.w == b) return;
    for (int probe = 0; probe < (1 << kDictLgBS); ++probe) {
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
        uint32_t* sl = sset + bk * 4 + j;
        const uint32_t k = *reinterpret_cast<volatile uint32_t*>(sl);
        if (k == b) return;
        if (k == kDictEmpty) {
          const uint32_t old = atomicCAS(sl, kDictEmpty, b);
          if (old == kDictEmpty) {
            if (atomicAdd(&s_n, 1) >= kDictHS / 2) s_over = 1;
            return;
          }
          if (old == b) return;
        }
      }
      bk = (bk + 1) & ((1u << kDictLgBS) - 1);
    }
    s_over = 1;
  };
  float mn[4], mx[4], mn2[4], mx2[4];
  int bad = 0;
  u64 nf01 = 0, nf23 = 0;
  const u64 zero2 = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    mn[i] = mn2[i] = INFINITY;
    mx[i] = mx2[i] = -INFINITY;
  }
  // count-walk state (K2b, adaptive)
  float2 lc0 = degenerate_lc(), lc2 = degenerate_lc();
  int hbx[4] = {-1, -1, -1, -1};
  bool patho = false;
  int cur_h = -1, hsel = 0;
  int my_pseq = 0;
  auto params_share = [&]() {  // this warp's 1/8 of a completed group's tables (warp-uniform)
    const int ps = __shfl_sync(0xffffffffu, vld(ctl.p_seq), 0);
    if (ps == my_pseq) return;
    my_pseq = ps;
    __threadfence_block();
    const int64_t key = *reinterpret_cast<volatile int64_t*>(&ctl.p_key);
    group_tables(G, W, key, vld(ctl.p_grp), tid, kConsumers);
    __threadfence();
    __syncwarp();
    if (lane == 0) mbar_arrive(&ctl.pdone);
  };

  uint32_t it = 0;
  int cs_slot = 0;
  uint32_t cs_phase = 0;
  while (true) {
    const int s = cs_slot;
    // wait for the stage; between polls take a share of any group's tables
    // (warp-uniform: the table build shuffles across the whole warp)
    {
      WD_BEGIN
      while (!__all_sync(0xffffffffu, mbar_try_wait(&P.pipe->full[s], cs_phase))) {
        params_share();
        WD_CHECK("cta %d warp %d: consumer waits stage %d it %u pseq %d/%d\n", blockIdx.x,
                 threadIdx.x / 32, s, it, my_pseq, vld(ctl.p_seq))
      }
    }
    params_share();
    const Stage& S = P.pipe->st[s];
    if (S.unit < 0) break;
    const int ph = S.ph, last = S.last, buf = S.seg, unit = S.unit;
    const float* sb = P.bufs + s * stage_elems;
    if (ph == 0) {
      if (lane_on) {
        const int P4 = (int)G.P;
        const int rstep = G.rpi * P4;
        const float* rp = sb + slot * P4 + e0;
        const int jd = (int)((0u - it) & 3u);
        int k = 0;
#pragma unroll 1
        for (; k + 4 <= trips; k += 4, rp += 4 * rstep) {
          float4 v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = *reinterpret_cast<const float4*>(rp + j * rstep);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float a[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
            float* m0 = (j & 1) ? mn2 : mn;
            float* m1 = (j & 1) ? mx2 : mx;
            nf01 = fma2(pk2(a[0], a[1]), zero2, nf01);
            nf23 = fma2(pk2(a[2], a[3]), zero2, nf23);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              m0[i] = fminf(m0[i], a[i]);
              m1[i] = fmaxf(m1[i], a[i]);
            }
          }
          if (DICT && (K2A_SAMPLE_GROUPS == 1 || ((k >> 2) + it) % K2A_SAMPLE_GROUPS == 0) &&
              !*reinterpret_cast<volatile int*>(&s_over)) {
            const float4 w = jd == 0 ? v[0] : jd == 1 ? v[1] : jd == 2 ? v[2] : v[3];
            const float a[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (i == 0 || a[i] != a[i - 1]) dict_add(a[i]);
          }
        }
        for (; k < trips; ++k, rp += rstep) {
          const float4 v = *reinterpret_cast<const float4*>(rp);
          const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            bad |= !isfinite(a[i]);
            mn[i] = fminf(mn[i], a[i]);
            mx[i] = fmaxf(mx[i], a[i]);
          }
          if (DICT && ((k + it) & 3) == 0 && !*reinterpret_cast<volatile int*>(&s_over)) {
#pragma unroll
            for (int i = 0; i < 4; ++i) dict_add(a[i]);
          }
        }
      }
    } else {
      if (unit != cur_h) {  // a new count walk: its tables are staged (producer waited)
        cur_h = unit;
        hsel = buf;
        patho = false;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 lc = tile_lc(tab_tp(T.tab[buf], trt[i]));
          if (i == 0) lc0 = lc;
          if (i == 2) lc2 = lc;
          patho |= isnan(lc.y);  // a range the f32 guard does not cover: bin_search
          hbx[i] = lc.y != kDegC ? trt[i] * n1 : -1;
        }
      }
      uint32_t* hist = T.hist[hsel];
      const int n1p = (int)ftab_n1p(n);
      const float* thrS = T.tab[hsel] + G.gtr * 4;
      const uint32_t hist_s = (uint32_t)__cvta_generic_to_shared(hist);
      if (lane_on && !patho && same_pairs && S.wuni != 0) {
        // hot path (K2b adaptive): edge-table bins, runs of equal (tile, bin)
        // merged into one shared add, run tails to the thread's discard word
        const uint32_t wf = (uint32_t)S.wfix;
        uint32_t w[4], ha[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          w[i] = wf * (uint32_t)trw[i];
          ha[i] = hist_s + (uint32_t)(trt[i] * n1) * 4u;
        }
        const uint32_t th0 = (uint32_t)__cvta_generic_to_shared(thrS + trt[0] * n1p);
        const uint32_t th2 = (uint32_t)__cvta_generic_to_shared(thrS + trt[2] * n1p);
        const u64 L0 = pk2(lc0.x, lc0.x), C0 = pk2(lc0.y, lc0.y);
        const u64 L2 = pk2(lc2.x, lc2.x), C2 = pk2(lc2.y, lc2.y);
        const float* rp = sb + slot * G.P + e0;
        const int64_t rstep = (int64_t)G.rpi * G.P;
#pragma unroll 4
        for (int k = 0; k < trips; ++k, rp += rstep) {
          const float4 v = *reinterpret_cast<const float4*>(rp);
          u64 t01, t23;
          asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t01) : "l"(mul2(sub2(pk2(v.x, v.y), L0), C0)), "l"(pk2(kMagic, kMagic)));
          asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t23) : "l"(mul2(sub2(pk2(v.z, v.w), L2), C2)), "l"(pk2(kMagic, kMagic)));
          float tf[4];
          upk2(t01, tf[0], tf[1]);
          upk2(t23, tf[2], tf[3]);
          const float vv[4] = {v.x, v.y, v.z, v.w};
          uint32_t a[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            a[i] = edge_hist_addr(i < 2 ? th0 : th2, clamp_bits_k(tf[i], n), vv[i], ha[i]);
          const bool e01 = a[0] == a[1], e12 = a[1] == a[2], e23 = a[2] == a[3];
          const uint32_t s3 = w[3];
          const uint32_t s2 = w[2] + (e23 ? s3 : 0u);
          const uint32_t s1 = w[1] + (e12 ? s2 : 0u);
          const uint32_t s0 = w[0] + (e01 ? s1 : 0u);
          red_add(a[0], s0);
          red_add(e01 ? dummy_s : a[1], s1);
          red_add(e12 ? dummy_s : a[2], s2);
          red_add(e23 ? dummy_s : a[3], s3);
        }
      } else if (lane_on) {
        const bool wuni = S.wuni != 0;
        const int32_t wfix = S.wfix;
        auto lcv = [&](int i) { return tile_lc(tab_tp(T.tab[hsel], trt[i])); };
        for (int q = slot; q < G.stage_rows; q += G.rpi) {
          uint32_t wrow;
          if (wuni) {
            wrow = (uint32_t)wfix;
          } else {
            const int r1 = q & (G.r1 - 1), r2 = q >> G.lg_r1;
            int32_t wv = wfix * S.p1.weight(S.x[KO - 1] + r1);
            if (KO >= 2) wv *= S.p2.weight(S.x[KO >= 2 ? KO - 2 : 0] + r2);
            wrow = (uint32_t)wv;
          }
          const float4 v = *reinterpret_cast<const float4*>(sb + q * G.P + e0);
          int b[4];
          const float a4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float* th = thrS + trt[i] * n1p;
            if (isnan(lcv(i).y)) b[i] = bin_search(a4[i], th, n);
            else bins2_edge(pk2(a4[i], a4[i]), a4[i], a4[i], lcv(i), th, n, b[i], b[i]);
          }
          int kprev = -1;
          uint32_t acc = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int key2 = hbx[i] >= 0 ? hbx[i] + b[i] : -2 - i;
            const uint32_t wv = wrow * (uint32_t)trw[i];
            if (key2 == kprev) {
              acc += wv;
            } else {
              if (kprev >= 0) atomicAdd(&hist[kprev], acc);
              kprev = key2;
              acc = wv;
            }
          }
          if (kprev >= 0) atomicAdd(&hist[kprev], acc);
        }
      }
    }
    if (last && ph == 0) {  // the walk's per-thread min/max into its range slot
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        mn[i] = fminf(mn[i], mn2[i]);
        mx[i] = fmaxf(mx[i], mx2[i]);
        if (lane_on && mn[i] <= mx[i]) {
          atomicMax(&T.rmin[buf][trt[i]], ~key32(mn[i]));
          atomicMax(&T.rmax[buf][trt[i]], key32(mx[i]));
        }
        mn[i] = mn2[i] = INFINITY;
        mx[i] = mx2[i] = -INFINITY;
      }
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&P.pipe->empty[s]);
      if (last) mbar_arrive(ph == 0 ? &ctl.rdone[buf] : &ctl.hdone[buf]);
    }
    ++it;
    if (++cs_slot == G.nst) {
      cs_slot = 0;
      cs_phase ^= 1;
    }
  }
  {
    float z0, z1, z2, z3;
    upk2(nf01, z0, z1);
    upk2(nf23, z2, z3);
    bad |= isnan(z0) || isnan(z1) || isnan(z2) || isnan(z3);
  }
  if (bad) atomicMax(reinterpret_cast<long long*>(&W.range[2]), 1LL);
  if (DICT) {  // merge the CTA's sampled values into the workspace set (as K2a)
    consumers_sync();
    if (s_over) {
      if (tid == 0) atomicExch(&W.dmeta[1], 1);
      return;
    }
    for (int k = tid; k < kDictHS; k += kConsumers) {
      const uint32_t b = sset[k];
      if (b == kDictEmpty) continue;
      uint32_t h = dict_hash(b, 13);
      for (int probe = 0; probe < kDictHG; ++probe) {
        const uint32_t old = atomicCAS(&W.dkeys[h], kDictEmpty, b);
        if (old == b) break;
        if (old == kDictEmpty) {
          if (atomicAdd(&W.dmeta[0], 1) >= kDictHG / 2) atomicExch(&W.dmeta[1], 1);
          break;
        }
        h = (h + 1) & (kDictHG - 1);
      }
    }
  }
}

template <bool DICT>
static PencilRangeFn fused_t(int ko) {
  switch (ko) {
    case 1: return k_k2_fused<1, DICT>;
    case 2: return k_k2_fused<2, DICT>;
    case 3: return k_k2_fused<3, DICT>;
    case 4: return k_k2_fused<4, DICT>;
    default: return k_k2_fused<5, DICT>;
  }
}

PencilRangeFn get_k2_fused(int ko, bool dict) { return dict ? fused_t<true>(ko) : fused_t<false>(ko); }
int k2_fused_threads() { return kFusedThreads; }
int64_t k2_fused_tail_bytes(int64_t gtr, int64_t n_bins, bool dict) {
  const int64_t hb = (gtr * (n_bins + 1) * 4 + 15) & ~15LL;
  const int64_t lb = (gtr * 8 + 15) & ~15LL;
  return 2 * (hb + ftab_bytes(gtr, n_bins)) + kNRS * lb + kConsumers * 4 + (dict ? kDictHS * 4 : 0);
}
int64_t k2_fused_tab_bytes(int64_t gtr, int64_t n_bins) { return ftab_bytes(gtr, n_bins);
}

}  // namespace mg
