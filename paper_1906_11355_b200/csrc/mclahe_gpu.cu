// mclahe_gpu.cu -- host side of the C ABI (include/mclahe_gpu.h): request
// validation, slab planning (tile windows, pencil units, CTA balancing),
// pass launches and the one-shot drop-in.  Kernels live in kernels.cuh.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/mclahe_gpu.h"
#include "k_misc.cuh"
#include "k_pencil.cuh"

namespace mg {
// k_tile.cu
void launch_tile_major(int dtype_f64, int mode, int grid, cudaStream_t st, const KGeom& G,
                       const void* in, WS W, int accum);
cudaError_t tile_major_smem_cap(int max_smem);
void launch_interp_cell(int dtype_f64, int adaptive, int grid, cudaStream_t st, const KGeom& G,
                        const void* in, void* out, WS W, int64_t cell0, int64_t ncells);
}  // namespace mg

namespace {

using namespace mg;

thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? MCLAHE_ERR_OOM : MCLAHE_ERR_CUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

#define MG_CUDA(call)                                 \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

#define MG_LAUNCHED_AT(what)                                  \
  do {                                                        \
    ++g_launches;                                             \
    cudaError_t e_ = cudaGetLastError();                      \
    if (e_ != cudaSuccess) return cuda_fail(e_, what);        \
  } while (0)
#define MG_LAUNCHED() MG_LAUNCHED_AT(__func__)

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// NVTX range over one host-side pass / call (header-only NVTX v3: free unless
// a profiler is attached), so an nsys / ncu timeline shows which pass a
// kernel launch belongs to (mclahe.range, mclahe.histograms, ...).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace

// error / launch bookkeeping shared with the other host translation units
// (host_err.h)
namespace mg {
int host_fail(int code, const std::string& msg) { return fail(code, msg); }
int host_cuda_fail(cudaError_t e, const char* where) { return cuda_fail(e, where); }
void host_count_launch() { ++g_launches; }
}  // namespace mg

namespace {

// validate_request (src/pipeline.cpp:19-34) minus the finiteness scan, which
// runs on the device; plus the NdImage invariants (src/nd_image.cpp:52-58).
int validate(const mclahe_params_t* p) {
  if (!p) return fail(MCLAHE_ERR_VALIDATION, "null params");
  if (p->rank < 1 || p->rank > MCLAHE_MAX_RANK)
    return fail(MCLAHE_ERR_VALIDATION, "rank must be in [1, 8]");
  for (int i = 0; i < p->rank; ++i)
    if (p->shape[i] <= 0) return fail(MCLAHE_ERR_VALIDATION, "shape extents must be positive");
  for (int i = 0; i < p->rank; ++i) {
    if (p->kernel[i] <= 0 || p->kernel[i] > p->shape[i])
      return fail(MCLAHE_ERR_VALIDATION,
                  "kernel size must be in [1, extent] along dimension " + std::to_string(i));
  }
  if (!(p->clip_limit > 0.0) || !(p->clip_limit <= 1.0))
    return fail(MCLAHE_ERR_VALIDATION, "clip_limit must be in (0, 1]");
  if (p->n_bins < 2) return fail(MCLAHE_ERR_VALIDATION, "n_bins must be at least 2");
  if (p->n_bins > 16384)
    return fail(MCLAHE_ERR_UNSUPPORTED, "n_bins above 16384 is not supported on the GPU path");
  if (p->dtype != MCLAHE_F32 && p->dtype != MCLAHE_F64)
    return fail(MCLAHE_ERR_VALIDATION, "dtype must be MCLAHE_F32 or MCLAHE_F64");
  int64_t tile = 1;
  for (int i = 0; i < p->rank; ++i) tile *= p->kernel[i];
  if (tile >= (int64_t{1} << 31))
    return fail(MCLAHE_ERR_UNSUPPORTED, "kernel volume too large for 32-bit tile counts");
  if (p->shape[0] >= (int64_t{1} << 31))
    return fail(MCLAHE_ERR_UNSUPPORTED, "dim-0 extent must be below 2^31");
  return MCLAHE_OK;
}

// Pencil configuration for one kernel family.
struct Pencil {
  bool on = false;
  int kt = 0, ko = 0;
  int64_t P = 0, gtr = 0;
  int tpr = 0, rpi = 0;
  int nst = 0, stage_rows = 0;
  int r1 = 1, lg_r1 = 0, r2 = 1;  // TMA box rows along outer dims KO-1, KO-2
  int tma_rank = 0, width = 0;    // TMA view: [outer dims..., P/width, width]
  int nseg = 1;                   // blend: 32-float segments per trailing block
  int64_t stage_stride = 0;       // floats per stage buffer
  int64_t tail = 0;               // kernel-specific shared memory (hist / LUTs)
  int64_t stage_budget = 0;
  int64_t smem = 0;
  bool hist_family = false;
};

constexpr int64_t kPipeBytes = (sizeof(mg::Pipe) + 1023) & ~int64_t(1023);
constexpr int64_t kStageBytes = 16384;
constexpr int kMaxChunks = 32;  // streamed one-shot: chunks per call (events are sized for it)

// dictionary workspace: meta[8] | keys[HG] | vals[HG/2] | lookup[HL] | lutd[tiles][KC]
constexpr int64_t kDictOffKeys = 256;
constexpr int64_t kDictOffVals = kDictOffKeys + kDictHG * 4;
constexpr int64_t kDictOffLt = kDictOffVals + kDictHG / 2 * 4;
constexpr int64_t kDictOffLutd = kDictOffLt + kDictHL * 8;
int64_t dict_bytes(int64_t win_tiles) { return kDictOffLutd + win_tiles * kDictKC * 4; }

}  // namespace

struct mclahe_plan_s {
  mclahe_params_t p{};
  mclahe_plan_info_t info{};
  Dim d[kMaxRank];
  KGeom G{};  // base geometry (kt/tpr/rpi/P/gtr filled per kernel)
  Pencil hist, interp;
  std::vector<int32_t> hist_units, interp_units;
  std::vector<int64_t> hist_vox, interp_vox;  // voxels per unit (balancing)
  // device state (lazy)
  int device = -1;
  int sms = 0;
  int32_t* d_tables = nullptr;
  int64_t off_hist_units = 0, off_hist_cta = 0, off_interp_units = 0, off_interp_cta = 0;
  int hist_grid = 0, interp_grid = 0, range_grid = 0, map_grid = 0, map_block = 128;
  int hist_dyn_grid = 0;  // K2 grid when units are handed out dynamically (occupancy x SMs)
  int64_t map_smem = 0;
  // tile-major K2 (k_tile.cu) for the non-pencil paths: fused range + counts
  // in one kernel for single-slab adaptive plans; shared_ws: a chunk plan of
  // the streamed call (workspace shared with the other chunks: combine, not store)
  bool fused_k2 = false, shared_ws = false;
  // fused pencil K2 (k_fused.cu): single-slab float32 adaptive pencil plans;
  // workspace [groups] arrival counters + [groups] published flags at off_k2g
  bool fused_pencil = false, fused_try = false;
  int64_t off_k2g = 0, off_k2tab = 0, k2_groups = 0, fused_smem = 0;
  int fused_grid = 0, k2_group_units = 0;
  int tile_grid = 0;
  // batched framewise, global mode: tiles take their frame's range (-1: off)
  int frame_axis = -1;
  int64_t off_frange = 0;
  // value dictionary (kDict*): armed when the blend's tables fit shared memory
  int dict_cap = 0, dict_nst = 0;
  int64_t dict_smem = 0, off_dict = 0;
  // folded-pair dictionary blend (k_interp_mdict): one 8-float segment per work item
  Pencil interp_m;
  bool mdict = false;
  bool cell_hist = false;        // K2b by dictionary cell launched beside the edge-table K2b
  int64_t cell_hist_smem = 0;
  std::vector<int32_t> mdict_units;  // whole cells (the interp units' dim-0 chunks merged)
  int64_t off_mdict_units = 0;
  // TMA views of the last input buffer (re-encoded when the pointer changes)
  const void* map_ptr[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  CUtensorMap map[5];  // [0] hist view of the input, [1] blend view of the input, [2] of the
                       // output, [3] / [4] the folded-pair blend's 8-float views of both
  bool f32() const { return p.dtype == MCLAHE_F32; }
  mclahe_plan_s() = default;
  mclahe_plan_s(const mclahe_plan_s&) = delete;
  mclahe_plan_s& operator=(const mclahe_plan_s&) = delete;
  // side branch of a whole-step enqueue: the dictionary numbering runs beside
  // params / edge tables / histograms (created on first use)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  ~mclahe_plan_s() {
    if (d_tables) cudaFree(d_tables);
    if (side) cudaStreamDestroy(side);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
  }
};

namespace {

int64_t nb_seg_tiles(const mclahe_plan_s& pl, const Pencil& c);

KGeom pencil_geom(const mclahe_plan_s& pl, const Pencil& pc) {
  KGeom G = pl.G;
  G.kt = pc.kt;
  G.P = pc.P;
  G.gtr = pc.gtr;
  G.tpr = pc.tpr;
  G.rpi = pc.rpi;
  G.nst = pc.nst;
  G.stage_rows = pc.stage_rows;
  G.r1 = pc.r1;
  G.lg_r1 = pc.lg_r1;
  G.r2 = pc.r2;
  G.tma_rank = pc.tma_rank;
  G.nseg = pc.nseg;
  G.stage_stride = pc.stage_stride;
  G.dict = pl.dict_cap > 0 ? 1 : 0;
  G.cell_hist = pl.cell_hist ? 1 : 0;
  static const int nb_edges = getenv("MCLAHE_NB_EDGES") ? atoi(getenv("MCLAHE_NB_EDGES")) : -1;
  G.nb_edges = nb_edges;
  G.stiles = (int)(pc.kt > 0 && !pc.hist_family ? nb_seg_tiles(pl, pc) : pc.gtr);
  for (int j = 0; j < G.rank; ++j) {
    G.inv_b[j] = 1.0f / (float)G.d[j].b;
    G.inv_2b[j] = 1.0f / (float)(2 * G.d[j].b);
  }
  return G;
}

bool trailing_merged(const Dim& d) {
  for (int64_t x = 0; x < d.before && x < d.s; ++x)
    if ((d.before - 1 - x) / d.b != (x + d.before) / d.b) return false;
  for (int64_t x = std::max<int64_t>(0, d.s - d.after); x < d.s; ++x)
    if ((d.before + 2 * d.s - 1 - x) / d.b != (x + d.before) / d.b) return false;
  return true;
}

bool nb_specialised(int64_t n) {
  static const bool no_nb = getenv("MCLAHE_NO_NB") != nullptr;
  return !no_nb && (n == 128 || n == 256);
}

// Trailing tiles the NB blend stages at once: all of them for one segment
// (32 floats of the trailing block; nseg == 1: every trailing tile), i.e.
// the span of the segment's columns' first tiles plus the far corner.
int64_t nb_seg_tiles(const mclahe_plan_s& pl, const Pencil& c) {
  const int D = pl.p.rank;
  if (c.nseg <= 1) return c.gtr;
  int64_t ts[kMaxRank], corner = 0;
  int64_t st = 1;
  for (int j = D - 1; j >= D - c.kt; --j) {
    ts[j] = st;
    corner += st;
    st *= pl.d[j].g;
  }
  int64_t best = 0;
  for (int seg = 0; seg < c.nseg; ++seg) {
    int64_t lo = INT64_MAX, hi = INT64_MIN;
    for (int k = 0; k < 8; ++k) {
      int64_t e = (int64_t)(seg * 8 + k) * 4, t = 0;
      for (int j = D - 1; j >= D - c.kt; --j) {
        const int64_t x = e % pl.d[j].s;
        e /= pl.d[j].s;
        t += cell_of(pl.d[j], x) * ts[j];
      }
      lo = std::min(lo, t);
      hi = std::max(hi, t);
    }
    best = std::max(best, hi + corner - lo + 1);
  }
  return std::min(best, c.gtr);
}

// Chooses how many trailing dims one pencil covers for a kernel family
// (box rows and pipeline depth are fixed later, once the units are known).
Pencil choose_pencil(const mclahe_plan_s& pl, bool for_hist) {
  Pencil best;
  const int D = pl.p.rank;
  const int64_t n = pl.p.n_bins;
  if (!pl.f32() || D < 2) return best;
  std::vector<Pencil> ok;
  for (int kt = 1; kt <= D - 1; ++kt) {
    const int ko = D - kt;
    if (ko > kMaxOuterDims) continue;
    if (!for_hist && (kt > 2 || ko > 4)) continue;
    Pencil c;
    c.kt = kt;
    c.ko = ko;
    c.P = 1;
    c.gtr = 1;
    bool merged = true;
    for (int j = D - kt; j < D; ++j) {
      c.P *= pl.d[j].s;
      c.gtr *= pl.d[j].g;
      merged = merged && trailing_merged(pl.d[j]);
    }
    if (c.P % 4 != 0 || c.P / 4 > 256) continue;
    c.width = (int)std::min<int64_t>(c.P, 256);
    if (c.P % c.width != 0) continue;
    c.tma_rank = ko + (c.P > 256 ? 2 : 1);
    if (c.tma_rank > 5) continue;
    c.tpr = (int)(c.P / 4);
    c.rpi = 256 / c.tpr;
    c.hist_family = for_hist;
    if (for_hist) {
      if (!merged) continue;
      if (c.gtr * n >= (int64_t{1} << 31) / 2) continue;
      c.tail = align_up(c.gtr * (n + 1) * 4, 16) + kConsumers * 4 + c.gtr * 16 +
               (pl.p.adaptive ? c.gtr : 1) * (n + 1) * 4;
      if (c.tail > 64 * 1024) continue;
      static const int64_t k2_stage =
          getenv("MCLAHE_K2_STAGE_KB") ? atoi(getenv("MCLAHE_K2_STAGE_KB")) * 1024 : kStageBytes;
      c.stage_budget = k2_stage;  // 3 stages, ~3 CTAs per SM
    } else {
      if (n % 4 != 0 || c.P % 32 != 0) continue;
      c.nseg = (int)(c.P / 32);
      c.tma_rank = ko + (c.nseg > 1 ? 2 : 1);
      if (c.tma_rank > 5) continue;
      // a thread's 4 columns must share their trailing cell
      const Dim& dl = pl.d[D - 1];
      if (dl.s % 4 != 0) continue;
      bool shared = true;
      for (int64_t cc = 1; cc <= dl.g - 2 && shared; ++cc) {
        int64_t ca, ce;
        cell_range(dl, cc, &ca, &ce);
        shared = (ca % 4) == 0;
      }
      if (!shared) continue;
      // LUTs (+ bin-edge tables: per tile when adaptive, one row when global)
      // + per-tile ranges; one CTA per SM with 16 consumer warps
      const int64_t luts1 = (int64_t{1} << ko) * c.gtr * (n + 1);  // rows padded to n+1
      const int64_t pairs = (int64_t{1} << ko) * (c.gtr - 1) * (n + 1) * 2;  // global, KT == 1
      c.tail = align_up((pl.p.adaptive ? 2 * luts1 : (kt == 1 ? pairs : luts1) + n + 1) * 4, 16) +
               (int64_t{1} << ko) * c.gtr * 16 + (c.P / 4) * (4 + 16 * (int64_t{1} << kt));
      c.tail += 16;  // column tables start 16-byte aligned
      if (pl.p.adaptive && nb_specialised(n)) {
        // NB-specialised kernel (the only adaptive blend launched): padded
        // per-tile blocks (NbBlock) for the trailing tiles of one segment
        c.tail = (int64_t{1} << ko) * nb_seg_tiles(pl, c) * NbBlock::words((int)n) * 4 +
                 (c.P / 4) * (4 + 16 * (int64_t{1} << kt)) + 16;
      }
      c.rpi = kConsumersBlend / c.tpr;
      const int64_t avail = 226 * 1024 - kPipeBytes - c.tail;
      if (avail >= 4 * 4096) c.stage_budget = std::min<int64_t>(kStageBytes, avail / 4);
      else if (avail >= 2 * 4096) c.stage_budget = avail / 2;
      else continue;
    }
    if (c.stage_budget < c.P * 4) continue;
    c.on = true;
    ok.push_back(c);
  }
  for (const Pencil& c : ok)
    if (c.P >= 32) return c;
  if (!ok.empty()) return ok.back();
  return best;
}

int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    const int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

int64_t pow2_divisor(int64_t g, int64_t cap) {
  int64_t r = 1;
  while (r * 2 <= cap && g % (r * 2) == 0) r *= 2;
  return r;
}

// Natural per-unit extents along an outer dim: tile supports (K2) or
// interpolation-cell ranges (K4), dim 0 clipped to the slab.
void extents(const mclahe_plan_s& pl, bool cells, int j, std::vector<std::pair<int64_t, int64_t>>& out) {
  const Dim& d = pl.d[j];
  out.clear();
  const int64_t n = cells ? d.g - 1 : d.g;
  for (int64_t t = 0; t < n; ++t) {
    int64_t a, e;
    if (cells) {
      cell_range(d, t, &a, &e);
    } else {
      const TileParts tp = tile_parts(d, t);
      a = tp.support_begin();
      e = tp.support_end();
    }
    if (j == 0) {
      a = std::max(a, pl.info.row_begin);
      e = std::min(e, pl.info.row_end);
    }
    if (e > a) out.push_back({a, e});
  }
}

// Box rows (powers of two dividing every unit extent, so boxes never cross a
// unit), pipeline depth and shared memory of a pencil family.
void size_boxes(const mclahe_plan_s& pl, Pencil& c, bool cells) {
  const int64_t row_bytes = cells ? 128 : c.P * 4;  // blend stages hold one 32-float segment
  const int64_t rows_cap = std::max<int64_t>(1, std::min<int64_t>(c.stage_budget / row_bytes, 256));
  std::vector<std::pair<int64_t, int64_t>> ex;
  int64_t g1 = 0, g2 = 0;
  extents(pl, cells, c.ko - 1, ex);
  for (auto& p : ex) g1 = gcd64(g1, p.second - p.first);
  // when dim 0 is a box dim (KO <= 2) keep >= ~2 units per SM: cap its box rows
  int64_t n_other = 1;
  for (int j = 1; j < c.ko; ++j) n_other *= cells ? pl.d[j].g - 1 : pl.d[j].g;
  const int64_t local_rows = pl.info.row_end - pl.info.row_begin;
  int64_t cap0 = 1;
  while (cap0 * 2 <= std::max<int64_t>(1, local_rows * n_other / 296)) cap0 *= 2;
  if (cells) cap0 = std::max<int64_t>(cap0, 32);  // blend: keep a warp's worth of rows per box
  c.r1 = (int)pow2_divisor(g1, std::min<int64_t>(std::min<int64_t>(rows_cap, 256),
                                                 c.ko == 1 ? cap0 : 256));
  c.r2 = 1;
  if (c.ko >= 2) {
    extents(pl, cells, c.ko - 2, ex);
    for (auto& p : ex) g2 = gcd64(g2, p.second - p.first);
    c.r2 = (int)pow2_divisor(g2, std::min<int64_t>(std::min<int64_t>(rows_cap / c.r1, 256),
                                                   c.ko == 2 ? cap0 : 256));
  }
  c.lg_r1 = 0;
  while ((1 << c.lg_r1) < c.r1) ++c.lg_r1;
  c.stage_rows = c.r1 * c.r2;
  c.stage_stride = cells ? align_up(c.stage_rows * 128, 1024) / 4 : align_up(c.stage_rows * c.P * 4, 128) / 4;
  const int64_t stage = c.stage_stride * 4;
  if (!cells) {
    static const int k2_nst = getenv("MCLAHE_K2_NST") ? atoi(getenv("MCLAHE_K2_NST")) : 3;
    c.nst = k2_nst;
  } else {
    c.nst = (int)std::max<int64_t>(2, std::min<int64_t>(4, (226 * 1024 - kPipeBytes - c.tail) / stage));
  }
  c.smem = kPipeBytes + c.nst * stage + c.tail;
}

// Arms the value-dictionary blend (adaptive float32 pencils) when its value
// tables, lookup hash and two pipeline stages fit one CTA's shared memory, and
// appends the dictionary state to the workspace.  MCLAHE_NO_DICT=1 disarms it.
void plan_dict(mclahe_plan_s* pl) {
  pl->dict_cap = 0;
  const Pencil& c = pl->interp;
  if (!pl->p.adaptive || !pl->f32() || !c.on || !pl->hist.on || getenv("MCLAHE_NO_DICT")) return;
  const int64_t nco = int64_t{1} << c.ko, nct = int64_t{1} << c.kt;
  const int64_t tail =  // value blocks + cuckoo table + corner rows + column tables
      nco * c.gtr * kDictKC * 4 + kDictHL * 8 + nco * 4 + (c.P / 4) * (4 + 16 * nct) + 16;
  const int64_t stage = c.stage_stride * 4;
  const int64_t nst = std::min<int64_t>(4, (226 * 1024 - kPipeBytes - tail) / stage);
  if (nst < 2) return;
  pl->dict_cap = kDictKC;
  pl->dict_nst = (int)nst;
  pl->dict_smem = kPipeBytes + nst * stage + tail;
  mclahe_plan_info_t& I = pl->info;
  pl->off_dict = align_up(I.workspace_bytes, 256);
  I.workspace_bytes = align_up(pl->off_dict + dict_bytes(pl->G.win_tiles), 256);
}

// Arms the folded-pair dictionary blend (k_interp_mdict) over the dictionary
// blend: one trailing dim, three outer dims, 8-float segments.  Its stages
// hold R2 x R1 rows of one segment (32 bytes); MCLAHE_NO_MDICT=1 disarms it.
void plan_mdict(mclahe_plan_s* pl) {
  pl->mdict = false;
  const Pencil& c = pl->interp;
  const bool A = pl->p.adaptive != 0;
  if ((A && !pl->dict_cap) || !pl->f32() || !c.on || c.kt != 1 || c.ko != 3 || c.P % 8 != 0 ||
      !get_interp_mdict(c.ko, false, A, (int)pl->p.n_bins) || getenv("MCLAHE_NO_MDICT"))
    return;
  const int64_t tk = A ? kDictKC : pl->p.n_bins;  // table row: dictionary values or bins
  Pencil m = c;
  m.nseg = (int)(c.P / 8);
  m.tma_rank = c.ko + 2;
  if (m.tma_rank > 5) return;
  // rows along dim KO-2: a power of two dividing every cell extent, R1 x R2 <= 512
  std::vector<std::pair<int64_t, int64_t>> ex;
  int64_t g2 = 0;
  extents(*pl, true, c.ko - 2, ex);
  for (auto& p : ex) g2 = gcd64(g2, p.second - p.first);
  m.r1 = c.r1;
  m.lg_r1 = c.lg_r1;
  static const int rows_cap = getenv("MCLAHE_MDICT_ROWS") ? atoi(getenv("MCLAHE_MDICT_ROWS")) : 512;
  static const int nst_cap = getenv("MCLAHE_MDICT_NST") ? atoi(getenv("MCLAHE_MDICT_NST")) : 4;
  m.r2 = (int)pow2_divisor(g2, std::min<int64_t>(256, std::max(1, rows_cap / m.r1)));
  m.stage_rows = m.r1 * m.r2;
  // the kernel has no per-lane row clamp: every box must be full, i.e. the
  // stage is whole warps of rows (a power of two >= 32) and R1 / R2 divide
  // every cell extent along dims KO-1 / KO-2 (else the TMA box would cross
  // into the next cell and lanes would read / write past it)
  if (m.stage_rows < 32 || (m.stage_rows & (m.stage_rows - 1)) != 0) return;
  for (auto& p : ex)
    if ((p.second - p.first) % m.r2 != 0) return;
  {
    std::vector<std::pair<int64_t, int64_t>> ex1;
    extents(*pl, true, c.ko - 1, ex1);
    for (auto& p : ex1)
      if ((p.second - p.first) % m.r1 != 0) return;
  }
  m.stage_stride = align_up(m.stage_rows * 32, 1024) / 4;
  const int64_t nco = int64_t{1} << c.ko;
  m.tail = 2 * 4 * nco * tk * 4 + kDictHL * 8 + nco * 4 + 16 + ((c.P / 4 + 3) & ~int64_t(3)) * 4 +
           (c.P / 4) * 32 + 16 + 16;  // ... | colW | dictionary scalars [4]
  const int64_t stage = m.stage_stride * 4;
  // 227 KB opt-in less the kernel's few static words (the other pencils keep
  // 1 KB of headroom: 226 KB); with kDictKC = 608 the fourth stage needs it
  const int64_t nst = std::min<int64_t>(std::min(nst_cap, kMaxStages), (227 * 1024 - 128 - kPipeBytes - m.tail) / stage);
  if (nst < 2) return;
  m.nst = (int)nst;
  m.smem = kPipeBytes + nst * stage + m.tail;
  // a work item rebuilds its tables, so units are merged from the interp
  // units' dim-0 chunks of one cell up to ~1M voxels (the 4D config: whole
  // cell pencils); larger ones would let the four CTAs sharing a pencil's rows
  // (one segment each) drift apart by more than L2 holds (Large 4D read
  // twice its input with whole 16 MB pencils)
  std::vector<int32_t>& mu = pl->mdict_units;
  mu.clear();
  const std::vector<int32_t>& iu = pl->interp_units;
  static const int lg_item = getenv("MCLAHE_MDICT_LG_ITEM") ? atoi(getenv("MCLAHE_MDICT_LG_ITEM")) : 20;
  int64_t mvox = 0;
  for (size_t k = 0, u = 0; k < iu.size(); k += kUnitInts, ++u) {
    const size_t last = mu.size();
    const int64_t v = pl->interp_vox[u];
    if (last && std::equal(iu.begin() + k, iu.begin() + k + c.ko, mu.begin() + last - kUnitInts) &&
        mu[last - 1] == iu[k + 8] && mvox + v <= (int64_t{1} << lg_item)) {
      mu[last - 1] = iu[k + 9];  // contiguous dim-0 chunk of the same cell
      mvox += v;
      continue;
    }
    mu.insert(mu.end(), iu.begin() + k, iu.begin() + k + kUnitInts);
    mvox = v;
  }
  if (mu.empty() || (int64_t)(mu.size() / kUnitInts) * m.nseg > INT32_MAX) return;
  pl->interp_m = m;
  pl->mdict = true;
}

void push_unit(std::vector<int32_t>& units, std::vector<int64_t>& vox, const int64_t* idx, int ko,
               int64_t ra, int64_t re, int64_t vox_per_row, int64_t target, int64_t quantum) {
  int64_t rows = std::max<int64_t>(1, target / std::max<int64_t>(1, vox_per_row));
  rows = std::max<int64_t>(quantum, rows / quantum * quantum);
  for (int64_t a = ra; a < re; a += rows) {
    const int64_t e = std::min(re, a + rows);
    int32_t rec[kUnitInts] = {0};
    for (int j = 0; j < ko; ++j) rec[j] = (int32_t)idx[j];
    rec[8] = (int32_t)a;
    rec[9] = (int32_t)e;
    units.insert(units.end(), rec, rec + kUnitInts);
    vox.push_back((e - a) * vox_per_row);
  }
}

// K2 units (range and histogram passes) handed out by an atomic counter
// (W.range[3], reset before each pass) on volumes of >= 2^26 voxels: 2^18-voxel
// units in global mode (Large 4D hist 2.18 -> 1.93 ms), 2^17 in adaptive mode
// (4D range + hist 0.564 -> 0.539 ms, 5D 0.601 -> 0.588; 2^16 / 2^18 slower:
// more flushes / a longer tail).  The static voxel-balanced split left SMs
// idle 18 % of the 4D histogram pass (ncu: active vs elapsed cycles) because
// CTAs with the same voxel count finish at data-dependent times.
// MCLAHE_STATIC_UNITS keeps the static split everywhere.
bool k2_dynamic(const mclahe_plan_s& pl, int64_t local_voxels) {
  static const bool static_units = getenv("MCLAHE_STATIC_UNITS") != nullptr;
  (void)pl;
  return !static_units && local_voxels >= (int64_t{1} << 26);
}

void build_units(mclahe_plan_s& pl) {
  const int64_t local = pl.G.local_voxels;
  const int64_t target = std::min<int64_t>(std::max<int64_t>(local / (148 * 16), 4096), 1 << 18);
  // blend units: the n_bins-specialised blend restages its tables per (unit,
  // segment), so on volumes whose blend units are handed out dynamically
  // (>= 2^26 voxels, do_interp) they are 2^18 voxels (5D: 4.22 -> 3.72 ms; 2^19:
  // 4.10 ms); MCLAHE_INTERP_UNIT overrides (voxels, A/B)
  static const int64_t interp_unit =
      getenv("MCLAHE_INTERP_UNIT") ? atoll(getenv("MCLAHE_INTERP_UNIT")) : 0;
  const int64_t interp_target =
      interp_unit > 0 ? interp_unit : (local >= (int64_t{1} << 26) ? int64_t{1} << 18 : target);
  // K2 units likewise (handed out by a counter on such volumes, k2_dynamic):
  // fewer per-unit histogram flushes
  static const int64_t k2_unit = getenv("MCLAHE_K2_UNIT") ? atoll(getenv("MCLAHE_K2_UNIT")) : 0;
  // fused K2: 2^14-voxel units (the bytes read between a box's two walks,
  // ~2 units per CTA over every CTA, must stay in L2: 2^15 re-read 30 % from
  // HBM, 2^16 and up nearly all of it)
  static const int64_t fk2_unit = getenv("MCLAHE_FK2_UNIT") ? atoll(getenv("MCLAHE_FK2_UNIT")) : 0;
  const int64_t hist_target =
      pl.fused_try ? (fk2_unit > 0 ? fk2_unit : std::min<int64_t>(target, int64_t{1} << 14))
      : k2_unit > 0 ? k2_unit
                  : (k2_dynamic(pl, local) ? (pl.p.adaptive ? int64_t{1} << 17 : int64_t{1} << 18) : target);
  for (int fam = 0; fam < 2; ++fam) {
    Pencil& pc = fam == 0 ? pl.hist : pl.interp;
    if (!pc.on) continue;
    const bool cells = fam == 1;
    size_boxes(pl, pc, cells);
    // dim-0 chunks must stay multiples of the box rows along dim 0
    const int64_t quantum = pc.ko == 1 ? pc.r1 : (pc.ko == 2 ? pc.r2 : 1);
    std::vector<int32_t>& units = fam == 0 ? pl.hist_units : pl.interp_units;
    std::vector<int64_t>& vox = fam == 0 ? pl.hist_vox : pl.interp_vox;
    const int ko = pc.ko;
    int64_t idx[kMaxRank] = {0};
    int64_t lo0, hi0;
    if (cells) {
      lo0 = cell_of(pl.d[0], pl.info.row_begin);
      hi0 = cell_of(pl.d[0], pl.info.row_end - 1) + 1;
    } else {
      lo0 = pl.info.count_row_begin;
      hi0 = pl.info.count_row_end;
    }
    idx[0] = lo0;
    const int64_t lim_j = cells ? -1 : 0;  // cells: g-1 per dim, tiles: g
    while (true) {
      int64_t per_row = pc.P;
      bool empty = false;
      for (int j = 1; j < ko; ++j) {
        int64_t a, e;
        if (cells) {
          cell_range(pl.d[j], idx[j], &a, &e);
        } else {
          const TileParts tp = tile_parts(pl.d[j], idx[j]);
          a = tp.support_begin();
          e = tp.support_end();
        }
        per_row *= e - a;
        empty = empty || e <= a;
      }
      int64_t a0, e0;
      if (cells) {
        cell_range(pl.d[0], idx[0], &a0, &e0);
      } else {
        const TileParts t0 = tile_parts(pl.d[0], idx[0]);
        a0 = t0.support_begin();
        e0 = t0.support_end();
      }
      const int64_t ra = std::max(a0, pl.info.row_begin), re = std::min(e0, pl.info.row_end);
      if (!empty && re > ra)
        push_unit(units, vox, idx, ko, ra, re, per_row, cells ? interp_target : hist_target, quantum);
      int j = ko - 1;
      while (j >= 1 && ++idx[j] == pl.d[j].g + lim_j) idx[j--] = 0;
      if (j == 0 && ++idx[0] == hi0) break;
    }
  }
}

// Contiguous, voxel-balanced unit ranges per CTA.
std::vector<int32_t> balance(const std::vector<int64_t>& vox, int grid) {
  std::vector<int32_t> cta(grid + 1, 0);
  int64_t total = 0;
  for (int64_t v : vox) total += v;
  int64_t acc = 0;
  int c = 1;
  for (size_t u = 0; u < vox.size() && c < grid; ++u) {
    acc += vox[u];
    while (c < grid && acc * grid >= total * c) cta[c++] = (int32_t)(u + 1);
  }
  while (c <= grid) cta[c++] = (int32_t)vox.size();
  cta[grid] = (int32_t)vox.size();
  return cta;
}

// ---- TMA tensor view of the (slab) input --------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// K2: [outer dims KO-1..0][P/width][width], box [R2 x R1 rows][P].
// K4: [outer dims KO-1..0][P/32 segments][32], box [R2 x R1 rows][1][32], 128B swizzle.
int tensor_map(mclahe_plan_s* pl, int fam, const void* in) {
  if (pl->map_ptr[fam] == in) return MCLAHE_OK;
  const int slot = fam;
  if (fam == 2) fam = 1;  // output view of the blend family
  if (fam == 4) fam = 3;  // output view of the folded-pair blend
  const Pencil& c = fam == 0 ? pl->hist : (fam == 3 ? pl->interp_m : pl->interp);
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(MCLAHE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[5], strides[5];
  cuuint32_t box[5], es[5];
  int r = 0;
  const bool seg = fam == 1 || fam == 3;
  const int64_t inner = fam == 1 ? 32 : (fam == 3 ? 8 : c.width);
  dims[r] = (cuuint64_t)inner;
  box[r] = (cuuint32_t)inner;
  ++r;
  if (c.tma_rank - c.ko == 2) {
    dims[r] = (cuuint64_t)(c.P / inner);
    strides[r - 1] = (cuuint64_t)inner * 4;
    box[r] = seg ? 1 : (cuuint32_t)(c.P / inner);
    ++r;
  }
  for (int j = c.ko - 1; j >= 0; --j) {
    dims[r] = (cuuint64_t)(j == 0 ? pl->info.row_end - pl->info.row_begin : pl->d[j].s);
    strides[r - 1] = (cuuint64_t)pl->G.vstride[j] * 4;
    box[r] = (cuuint32_t)(j == c.ko - 1 ? c.r1 : (j == c.ko - 2 ? c.r2 : 1));
    ++r;
  }
  for (int i = 0; i < r; ++i) es[i] = 1;
  const CUresult res = enc(&pl->map[slot], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)r,
                           const_cast<void*>(in), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           fam == 1 ? CU_TENSOR_MAP_SWIZZLE_128B
                                    : (fam == 3 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE),
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (res != CUDA_SUCCESS)
    return fail(MCLAHE_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)res) + ")");
  pl->map_ptr[slot] = in;
  return MCLAHE_OK;
}

// full_window: the workspace holds every tile row (chunks of a streamed
// single-GPU run share one workspace); otherwise only the rows the slab
// counts into or blends from.
void plan_fused_pencil(mclahe_plan_s* pl, bool full_window);

int plan_describe(const mclahe_params_t* params, int64_t row_begin, int64_t row_end,
                  mclahe_plan_s* pl, bool full_window = false) {
  int rc = validate(params);
  if (rc) return rc;
  if (row_begin < 0 || row_end > params->shape[0] || row_begin >= row_end)
    return fail(MCLAHE_ERR_VALIDATION, "slab rows must satisfy 0 <= begin < end <= shape[0]");
  pl->p = *params;
  const int D = params->rank;
  mclahe_plan_info_t& I = pl->info;
  std::memset(&I, 0, sizeof I);
  I.rank = D;
  I.tiles = 1;
  for (int j = 0; j < D; ++j) {
    pl->d[j] = make_dim(params->shape[j], params->kernel[j]);
    I.before[j] = pl->d[j].before;
    I.after[j] = pl->d[j].after;
    I.grid[j] = pl->d[j].g;
    I.tiles *= pl->d[j].g;
  }
  I.row_begin = row_begin;
  I.row_end = row_end;
  I.n_bins = params->n_bins;
  // tile rows whose support meets the slab
  int64_t cb = INT64_MAX, ce = INT64_MIN;
  for (int64_t t = 0; t < pl->d[0].g; ++t) {
    const TileParts tp = tile_parts(pl->d[0], t);
    if (tp.support_begin() < row_end && tp.support_end() > row_begin) {
      cb = std::min(cb, t);
      ce = std::max(ce, t + 1);
    }
  }
  I.count_row_begin = cb;
  I.count_row_end = ce;
  I.need_row_begin = cell_of(pl->d[0], row_begin);
  I.need_row_end = cell_of(pl->d[0], row_end - 1) + 2;
  I.tile_row_begin = full_window ? 0 : std::min(I.count_row_begin, I.need_row_begin);
  I.tile_row_end = full_window ? pl->d[0].g : std::max(I.count_row_end, I.need_row_end);
  I.tiles_per_row = I.tiles / pl->d[0].g;
  const int64_t win_tiles = (I.tile_row_end - I.tile_row_begin) * I.tiles_per_row;
  const int64_t n = params->n_bins;
  const int64_t tp_size = pl->f32() ? sizeof(TileParam<float>) : sizeof(TileParam<double>);
  I.off_range = 0;
  I.off_tile_range = 256;
  I.off_counts = align_up(I.off_tile_range + (params->adaptive ? win_tiles * 16 : 16), 256);
  I.off_tparams = align_up(I.off_counts + win_tiles * n * 4, 256);
  I.off_lut = align_up(I.off_tparams + (params->adaptive ? win_tiles : 1) * tp_size, 256);
  I.off_thr = align_up(I.off_lut + win_tiles * n * 4, 256);
  I.workspace_bytes =
      align_up(I.off_thr + (pl->f32() ? (params->adaptive ? win_tiles : 1) * (n + 1) * 4 : 0), 256);

  KGeom& G = pl->G;
  std::memset(&G, 0, sizeof G);
  G.rank = D;
  G.n_bins = (int)n;
  G.adaptive = params->adaptive ? 1 : 0;
  for (int j = 0; j < D; ++j) G.d[j] = pl->d[j];
  G.vstride[D - 1] = 1;
  G.tstride[D - 1] = 1;
  for (int j = D - 1; j > 0; --j) {
    G.vstride[j - 1] = G.vstride[j] * params->shape[j];
    G.tstride[j - 1] = G.tstride[j] * pl->d[j].g;
  }
  G.row0 = row_begin;
  G.trow0 = I.tile_row_begin;
  G.win_tiles = win_tiles;
  G.local_voxels = (row_end - row_begin) * G.vstride[0];
  G.clip = params->clip_limit;

  pl->hist = choose_pencil(*pl, true);
  pl->interp = choose_pencil(*pl, false);
  I.fast_hist = pl->hist.on;
  I.fast_interp = pl->interp.on;
  I.trailing_dims = pl->interp.on ? pl->interp.kt : pl->hist.kt;
  {  // the fused pencil K2 (plan_fused_pencil; opt-in, see k_fused.cu) wants small units
    static const bool on = getenv("MCLAHE_FUSED_K2") != nullptr && atoi(getenv("MCLAHE_FUSED_K2")) != 0;
    pl->fused_try = on && pl->hist.on && params->adaptive && pl->f32() && !full_window &&
                    row_begin == 0 && row_end == params->shape[0];
  }
  build_units(*pl);
  I.hist_units = (int64_t)pl->hist_vox.size();
  I.interp_units = (int64_t)pl->interp_vox.size();
  // streamed chunk plans (full_window) interleave range passes with mappings,
  // so a dictionary numbered per chunk would not be stable: edge tables only
  if (!full_window) plan_dict(pl);
  if (!full_window) plan_mdict(pl);
  pl->shared_ws = full_window && (row_begin != 0 || row_end != params->shape[0]);
  plan_fused_pencil(pl, full_window);
  pl->fused_k2 = !pl->hist.on && params->adaptive && !pl->f32() && !pl->shared_ws &&
                 row_begin == 0 && row_end == params->shape[0];
  return MCLAHE_OK;
}

// Arms the fused pencil K2 (k_fused.cu) for single-slab float32 adaptive plans:
// numbers the tile groups (units sharing a key: one KO-outer tile, every
// trailing tile) in the unit records ([6] group, [7] units in the group) and
// appends the group counters to the workspace.  Every window tile must belong
// to a group with at least one unit (the kernel writes every tile's binning
// parameters).  Opt-in (MCLAHE_FUSED_K2=1): it halves the HBM reads of the
// range + count passes but measured slower than the two passes (k_fused.cu).
void plan_fused_pencil(mclahe_plan_s* pl, bool full_window) {
  pl->fused_pencil = false;
  if (!pl->fused_try) return;
  (void)full_window;
  const Pencil& c = pl->hist;
  const int64_t groups = pl->G.win_tiles / c.gtr;
  if (groups * c.gtr != pl->G.win_tiles || groups <= 0) return;
  std::vector<int32_t>& U = pl->hist_units;
  const int64_t nu = (int64_t)U.size() / kUnitInts;
  std::vector<int32_t> per(groups, 0);
  std::vector<int64_t> gid(nu);
  for (int64_t u = 0; u < nu; ++u) {
    const int32_t* r = &U[u * kUnitInts];
    int64_t key = (r[0] - pl->G.trow0) * pl->G.tstride[0];
    for (int j = 1; j < c.ko; ++j) key += (int64_t)r[j] * pl->G.tstride[j];
    if (key % c.gtr != 0 || key / c.gtr >= groups || key < 0) return;
    gid[u] = key / c.gtr;
    if (u > 0 && gid[u] != gid[u - 1] && per[gid[u]] > 0) return;  // units of a group consecutive
    ++per[gid[u]];
  }
  int mx = 0;
  for (int64_t g = 0; g < groups; ++g) {
    if (per[g] == 0) return;
    mx = std::max(mx, per[g]);
  }
  if (c.ko > 5) return;  // record slots 6 / 7 hold the group
  for (int64_t u = 0; u < nu; ++u) {
    U[u * kUnitInts + 6] = (int32_t)gid[u];
    U[u * kUnitInts + 7] = per[gid[u]];
  }
  pl->k2_groups = groups;
  pl->k2_group_units = mx;
  pl->off_k2g = align_up(pl->info.workspace_bytes, 256);
  pl->off_k2tab = align_up(pl->off_k2g + 2 * groups * 4, 256);
  pl->info.workspace_bytes =
      align_up(pl->off_k2tab + groups * k2_fused_tab_bytes(c.gtr, pl->p.n_bins), 256);
  pl->fused_smem = kPipeBytes + c.nst * c.stage_stride * 4 +
                   k2_fused_tail_bytes(c.gtr, pl->p.n_bins, pl->dict_cap > 0);
  pl->fused_pencil = true;
}

using RangeFn = PencilRangeFn;
using HistFn = PencilHistFn;
using InterpFn = PencilInterpFn;
RangeFn range_fn(int ko, bool dict) { return get_range_pencil(ko, dict); }
// MCLAHE_K2_MATCH=1: the warp-aggregated (__match_any_sync) histogram adds (A/B).
// Runs carried across a thread's rows (k_hist_pencil CARRY) in global mode:
// Large 4D hist 1.93 -> 1.80 ms; adaptive 4D / 5D unchanged (0.307 / 0.311,
// 0.375 / 0.377 ms), so they keep the per-row merge.  MCLAHE_K2_CARRY=0/1
// forces either (A/B).
HistFn hist_fn(int ko, bool a) {
  static const bool match = getenv("MCLAHE_K2_MATCH") && atoi(getenv("MCLAHE_K2_MATCH")) != 0;
  static const int carry_env = getenv("MCLAHE_K2_CARRY") ? atoi(getenv("MCLAHE_K2_CARRY")) : -1;
  const bool carry = carry_env < 0 ? !a : carry_env != 0;
  return get_hist_pencil(ko, a, match ? 1 : carry ? 2 : 0);
}
// MCLAHE_NO_NB=1 forces the runtime-n_bins blend kernel (A/B measurements).
InterpFn interp_fn(int ko, int kt, bool a, int64_t n_bins) {
  return get_interp_pencil(ko, kt, a, nb_specialised(n_bins) ? (int)n_bins : 0);
}

WS ws_view(const mclahe_plan_s* pl, void* ws) {
  char* b = static_cast<char*>(ws);
  WS W;
  W.range = reinterpret_cast<int64_t*>(b + pl->info.off_range);
  W.trange = reinterpret_cast<int64_t*>(b + pl->info.off_tile_range);
  W.counts = reinterpret_cast<uint32_t*>(b + pl->info.off_counts);
  W.tparams = b + pl->info.off_tparams;
  W.lut = reinterpret_cast<float*>(b + pl->info.off_lut);
  W.thr = reinterpret_cast<float*>(b + pl->info.off_thr);
  W.dmeta = nullptr;
  W.dkeys = nullptr;
  W.dvals = nullptr;
  W.dlt = nullptr;
  W.lutd = nullptr;
  W.k2g = pl->fused_pencil ? reinterpret_cast<int32_t*>(b + pl->off_k2g) : nullptr;
  W.k2tab = pl->fused_pencil ? reinterpret_cast<float*>(b + pl->off_k2tab) : nullptr;
  if (pl->dict_cap) {
    char* d = b + pl->off_dict;
    W.dmeta = reinterpret_cast<int32_t*>(d);
    W.dkeys = reinterpret_cast<uint32_t*>(d + kDictOffKeys);
    W.dvals = reinterpret_cast<float*>(d + kDictOffVals);
    W.dlt = reinterpret_cast<uint2*>(d + kDictOffLt);
    W.lutd = reinterpret_cast<float*>(d + kDictOffLutd);
  }
  return W;
}

int64_t range_smem(const mclahe_plan_s* pl) {
  return kPipeBytes + pl->hist.nst * pl->hist.stage_stride * 4 + align_up(pl->hist.gtr * 8, 16) +
         (pl->dict_cap ? kDictHS * 4 : 0);
}

// Raises a kernel's dynamic shared-memory cap to the device opt-in maximum
// minus its static shared memory.
template <typename F>
cudaError_t raise_smem_cap(F f, int optin) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(f));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(reinterpret_cast<const void*>(f),
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - (int)fa.sharedSizeBytes);
}

int device_init(mclahe_plan_s* pl) {
  int dev;
  MG_CUDA(cudaGetDevice(&dev));
  if (pl->device == dev) return MCLAHE_OK;
  if (pl->device >= 0) return fail(MCLAHE_ERR_CUDA, "plan used on a different device");
  MG_CUDA(cudaDeviceGetAttribute(&pl->sms, cudaDevAttrMultiProcessorCount, dev));
  // Shared-memory caps are per kernel, not per plan: raise them to the
  // device's opt-in maximum once so plans sharing an instantiation never
  // undercut each other (occupancy still follows each launch's real size).
  int max_smem = 0;
  MG_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const bool A = pl->p.adaptive != 0;
  if (pl->dict_cap > 0 && !pl->side) {  // side branch of enqueue_all (made here: not under capture)
    MG_CUDA(cudaStreamCreateWithFlags(&pl->side, cudaStreamNonBlocking));
    MG_CUDA(cudaEventCreateWithFlags(&pl->ev_fork, cudaEventDisableTiming));
    MG_CUDA(cudaEventCreateWithFlags(&pl->ev_join, cudaEventDisableTiming));
  }
  std::vector<int32_t> hist_cta, interp_cta;
  if (pl->hist.on) {
    int occ = 0;
    HistFn f = hist_fn(pl->hist.ko, A);
    MG_CUDA(raise_smem_cap(f, max_smem));
    MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, kPencilThreads, pl->hist.smem));
    if (A) {
      RangeFn r = range_fn(pl->hist.ko, pl->dict_cap > 0);
      MG_CUDA(raise_smem_cap(r, max_smem));
    }
    // K2b by dictionary cell (k_hist_cells), opt-in with MCLAHE_CELL_HIST=1: whole-volume
    // adaptive float32 plans with the value dictionary armed, when its [gtr][kDictKC + 1]
    // counters keep the CTAs per SM.  Exact (parity suites green with it) but slower than the
    // edge-table K2b on the 4D volume (0.340 vs 0.299 ms): per-cell keys merge far fewer
    // neighbouring voxels than per-bin keys, so more lanes take part in every shared add.
    pl->cell_hist = false;
    if (A && pl->dict_cap > 0 && pl->f32() && !pl->fused_pencil && pl->frame_axis < 0 &&
        !pl->shared_ws && pl->info.row_begin == 0 && pl->info.row_end == pl->p.shape[0] &&
        getenv("MCLAHE_CELL_HIST")) {
      const int64_t tail = align_up(pl->hist.gtr * (kDictKC + 1) * 4, 16) + kDictKC * 4;
      const int64_t smem = pl->hist.smem - pl->hist.tail + tail;
      HistFn fc = get_hist_cells(pl->hist.ko);
      int occ_c = 0;
      if (smem <= max_smem && raise_smem_cap(fc, max_smem) == cudaSuccess &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, fc, kPencilThreads, smem) == cudaSuccess &&
          occ_c >= occ) {
        pl->cell_hist = true;
        pl->cell_hist_smem = smem;
      }
    }
    pl->hist_grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)pl->hist_vox.size(), (int64_t)std::max(occ, 1) * pl->sms));
    pl->hist_dyn_grid = pl->hist_grid;
    hist_cta = balance(pl->hist_vox, pl->hist_grid);
    if (pl->fused_pencil) {
      RangeFn fk = get_k2_fused(pl->hist.ko, pl->dict_cap > 0);
      int focc = 0;
      MG_CUDA(raise_smem_cap(fk, max_smem));
      MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&focc, fk, k2_fused_threads(), pl->fused_smem));
      pl->fused_grid = (int)std::min<int64_t>((int64_t)pl->hist_vox.size(), (int64_t)focc * pl->sms);
      // a group's units wait for each other: they must all be able to run
      if (focc < 1 || pl->fused_grid < pl->k2_group_units) pl->fused_pencil = false;
    }
  }
  if (pl->interp.on) {
    int occ = 0;
    InterpFn f = interp_fn(pl->interp.ko, pl->interp.kt, A, pl->p.n_bins);
    MG_CUDA(raise_smem_cap(f, max_smem));
    if (pl->dict_cap) MG_CUDA(raise_smem_cap(get_interp_pencil_dict(pl->interp.ko, pl->interp.kt), max_smem));
    if (pl->mdict) {
      MG_CUDA(raise_smem_cap(get_interp_mdict(pl->interp.ko, false, A, (int)pl->p.n_bins), max_smem));
      MG_CUDA(raise_smem_cap(get_interp_mdict(pl->interp.ko, true, A, (int)pl->p.n_bins), max_smem));
    }
    MG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, kBlendThreads, pl->interp.smem));
    pl->interp_grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)pl->interp_vox.size(), (int64_t)std::max(occ, 1) * pl->sms));
    interp_cta = balance(pl->interp_vox, pl->interp_grid);
  }
  const size_t total = pl->hist_units.size() + hist_cta.size() + pl->interp_units.size() +
                       interp_cta.size() + pl->mdict_units.size() + 4;
  MG_CUDA(cudaMalloc(&pl->d_tables, total * sizeof(int32_t)));
  std::vector<int32_t> host;
  host.reserve(total);
  pl->off_hist_units = (int64_t)host.size();
  host.insert(host.end(), pl->hist_units.begin(), pl->hist_units.end());
  pl->off_hist_cta = (int64_t)host.size();
  host.insert(host.end(), hist_cta.begin(), hist_cta.end());
  pl->off_interp_units = (int64_t)host.size();
  host.insert(host.end(), pl->interp_units.begin(), pl->interp_units.end());
  pl->off_interp_cta = (int64_t)host.size();
  host.insert(host.end(), interp_cta.begin(), interp_cta.end());
  pl->off_mdict_units = (int64_t)host.size();
  host.insert(host.end(), pl->mdict_units.begin(), pl->mdict_units.end());
  host.resize(total, 0);
  MG_CUDA(cudaMemcpy(pl->d_tables, host.data(), total * sizeof(int32_t), cudaMemcpyHostToDevice));
  pl->range_grid = pl->sms * 4;
  if (!pl->hist.on || !pl->interp.on) {
    MG_CUDA(tile_major_smem_cap(max_smem));
    pl->tile_grid = (int)std::max<int64_t>(1, std::min<int64_t>(pl->G.win_tiles, (int64_t)pl->sms * 8));
  }
  // mappings: one warp per tile, f64 scratch of n_bins per warp
  const int64_t n = pl->p.n_bins;
  int warps = (int)std::max<int64_t>(1, std::min<int64_t>(4, (96 * 1024) / (n * 8)));
  pl->map_block = warps * 32;
  pl->map_smem = (int64_t)warps * n * 8;
  if (pl->f32())
    MG_CUDA(raise_smem_cap(k_mappings<float>, max_smem));
  else
    MG_CUDA(raise_smem_cap(k_mappings<double>, max_smem));
  const int64_t tiles = pl->G.win_tiles;
  pl->map_grid = (int)std::max<int64_t>(1, std::min<int64_t>((tiles + warps - 1) / warps, 1 << 20));
  pl->device = dev;
  return MCLAHE_OK;
}

int generic_grid(const mclahe_plan_s* pl) {
  return (int)std::max<int64_t>(
      1, std::min<int64_t>((pl->G.local_voxels + 255) / 256, (int64_t)pl->sms * 32));
}

int do_reset(mclahe_plan_s* pl, void* ws, cudaStream_t st) {
  NvtxRange nvtx("mclahe.reset");
  WS W = ws_view(pl, ws);
  const int64_t ntr = pl->p.adaptive ? pl->G.win_tiles * 2 : 0;
  MG_CUDA(cudaMemsetAsync(W.counts, 0, (size_t)pl->G.win_tiles * pl->p.n_bins * 4, st));
  const int64_t nr = std::max<int64_t>(ntr, pl->dict_cap ? kDictHG : 0);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nr + 255) / 256, 1024));
  k_reset<<<grid, 256, 0, st>>>(W.range, W.trange, ntr, W, pl->dict_cap > 0 ? 1 : 0);
  MG_LAUNCHED();
  return MCLAHE_OK;
}

// fork: the dictionary numbering (k_dict_finalize, only read by k_dict_luts and
// the blend) goes to the plan's side stream and ev_join is recorded there; the
// caller must make `st` wait for ev_join before the mappings pass.
int do_range(mclahe_plan_s* pl, const void* in, void* ws, cudaStream_t st, bool fork = false) {
  NvtxRange nvtx("mclahe.range");
  WS W = ws_view(pl, ws);
  if (pl->frame_axis >= 0) {  // framewise global mode: per-frame ranges
    const int ax = pl->frame_axis;
    int64_t outer = 1, inner = 1;
    for (int j = 0; j < ax; ++j) outer *= pl->p.shape[j];
    for (int j = ax + 1; j < pl->p.rank; ++j) inner *= pl->p.shape[j];
    const int64_t frames = pl->p.shape[ax];
    int64_t* frange = reinterpret_cast<int64_t*>(static_cast<char*>(ws) + pl->off_frange);
    k_reset<<<(int)std::max<int64_t>(1, std::min<int64_t>((2 * frames + 255) / 256, 1024)), 256, 0, st>>>(
        W.range, frange, 2 * frames, W, 0);
    MG_LAUNCHED();
    const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((inner + 255) / 256, 64)),
                    (unsigned)std::max<int64_t>(1, std::min<int64_t>(outer * frames, 65535)));
    if (pl->f32())
      k_frame_range<float><<<grid, 256, 0, st>>>(static_cast<const float*>(in), outer, frames, inner,
                                                 frange, W.range);
    else
      k_frame_range<double><<<grid, 256, 0, st>>>(static_cast<const double*>(in), outer, frames,
                                                  inner, frange, W.range);
    MG_LAUNCHED();
    const int tg = (int)std::max<int64_t>(1, std::min<int64_t>((pl->G.win_tiles + 255) / 256, 4096));
    k_frame_tiles<<<tg, 256, 0, st>>>(pl->G, W, frange, ax);
    MG_LAUNCHED();
    return MCLAHE_OK;
  }
  if (!pl->p.adaptive) {
    if (pl->f32())
      k_global_range<float><<<pl->range_grid, 256, 0, st>>>(static_cast<const float*>(in),
                                                            pl->G.local_voxels, W.range);
    else
      k_global_range<double><<<pl->range_grid, 256, 0, st>>>(static_cast<const double*>(in),
                                                             pl->G.local_voxels, W.range);
    MG_LAUNCHED();
    return MCLAHE_OK;
  }
  if (pl->fused_pencil) {  // ranges + counts, one DRAM read (k_fused.cu)
    KGeom G = pencil_geom(*pl, pl->hist);
    G.dyn_units = (int)pl->hist_vox.size();
    MG_CUDA(cudaMemsetAsync(W.range + 3, 0, sizeof(int64_t), st));
    MG_CUDA(cudaMemsetAsync(W.k2g, 0, (size_t)pl->k2_groups * 8, st));
    int rc = tensor_map(pl, 0, in);
    if (rc) return rc;
    get_k2_fused(pl->hist.ko, pl->dict_cap > 0)<<<pl->fused_grid, k2_fused_threads(), pl->fused_smem, st>>>(
        G, pl->map[0], static_cast<const float*>(in), pl->d_tables + pl->off_hist_units,
        pl->d_tables + pl->off_hist_cta, W);
    MG_LAUNCHED();
    if (pl->dict_cap) {
      k_dict_finalize<<<1, 1024, 0, st>>>(W, pl->dict_cap);
      MG_LAUNCHED();
    }
    return MCLAHE_OK;
  }
  if (pl->hist.on) {
    KGeom G = pencil_geom(*pl, pl->hist);
    G.dyn_units = k2_dynamic(*pl, pl->G.local_voxels) ? (int)pl->hist_vox.size() : 0;
    if (G.dyn_units) MG_CUDA(cudaMemsetAsync(W.range + 3, 0, sizeof(int64_t), st));
    RangeFn f = range_fn(pl->hist.ko, pl->dict_cap > 0);
    int rc = tensor_map(pl, 0, in);
    if (rc) return rc;
    f<<<G.dyn_units ? pl->hist_dyn_grid : pl->hist_grid, kPencilThreads, range_smem(pl), st>>>(G, pl->map[0], static_cast<const float*>(in),
                                                    pl->d_tables + pl->off_hist_units,
                                                    pl->d_tables + pl->off_hist_cta, W);
    MG_LAUNCHED();
    if (pl->dict_cap) {  // number the collected values once the slab's range pass is in
      cudaStream_t fs = st;
      if (fork) {
        MG_CUDA(cudaEventRecord(pl->ev_fork, st));
        MG_CUDA(cudaStreamWaitEvent(pl->side, pl->ev_fork, 0));
        fs = pl->side;
      }
      k_dict_finalize<<<1, 1024, 0, fs>>>(W, pl->dict_cap);
      MG_LAUNCHED();
      if (fork) MG_CUDA(cudaEventRecord(pl->ev_join, pl->side));
    }
    return MCLAHE_OK;
  }
  // tile-major range (+ counts when fused: single-slab float64 plans)
  launch_tile_major(pl->f32() ? 0 : 1, pl->fused_k2 ? 2 : 0, pl->tile_grid, st, pl->G, in, W,
                    pl->shared_ws ? 1 : 0);
  MG_LAUNCHED();
  return MCLAHE_OK;
}

// Binning parameters + edge tables for window tiles [t0, t0 + nt) (adaptive;
// nt < 0: the whole window) or the global range.
int do_params(mclahe_plan_s* pl, void* ws, cudaStream_t st, int64_t t0 = 0, int64_t nt = -1) {
  NvtxRange nvtx("mclahe.params");
  WS W = ws_view(pl, ws);
  if (pl->fused_pencil) return MCLAHE_OK;  // built by the fused K2 kernel
  if (nt < 0) nt = pl->G.win_tiles - t0;
  if (pl->p.adaptive && nt <= 0) return MCLAHE_OK;
  const int64_t n = pl->p.adaptive ? nt : 1;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 127) / 128, 4096));
  if (pl->f32()) k_params<float><<<grid, 128, 0, st>>>(pl->G, W, t0, nt);
  else k_params<double><<<grid, 128, 0, st>>>(pl->G, W, t0, nt);
  MG_LAUNCHED();
  if (pl->f32()) {
    const int64_t total = n * (pl->p.n_bins + 1);
    const int tg = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 8192));
    k_thresholds<<<tg, 256, 0, st>>>(pl->G, W, t0, nt);
    MG_LAUNCHED();
  }
  return MCLAHE_OK;
}

int do_hist(mclahe_plan_s* pl, const void* in, void* ws, cudaStream_t st) {
  NvtxRange nvtx("mclahe.histograms");
  WS W = ws_view(pl, ws);
  const bool A = pl->p.adaptive != 0;
  if (pl->fused_pencil) return MCLAHE_OK;  // counted by the fused range pass
  if (pl->hist.on) {
    KGeom G = pencil_geom(*pl, pl->hist);
    G.dyn_units = k2_dynamic(*pl, pl->G.local_voxels) ? (int)pl->hist_vox.size() : 0;
    if (G.dyn_units) MG_CUDA(cudaMemsetAsync(W.range + 3, 0, sizeof(int64_t), st));
    HistFn f = hist_fn(pl->hist.ko, A);
    int rc = tensor_map(pl, 0, in);
    if (rc) return rc;
    f<<<G.dyn_units ? pl->hist_dyn_grid : pl->hist_grid, kPencilThreads, pl->hist.smem, st>>>(G, pl->map[0], static_cast<const float*>(in),
                                                 pl->d_tables + pl->off_hist_units,
                                                 pl->d_tables + pl->off_hist_cta, W);
    MG_LAUNCHED();
    if (pl->cell_hist) {  // the dictionary state selects which of the two counts the volume
      get_hist_cells(pl->hist.ko)<<<G.dyn_units ? pl->hist_dyn_grid : pl->hist_grid, kPencilThreads,
                                    pl->cell_hist_smem, st>>>(
          G, pl->map[0], static_cast<const float*>(in), pl->d_tables + pl->off_hist_units,
          pl->d_tables + pl->off_hist_cta, W);
      MG_LAUNCHED();
    }
    return MCLAHE_OK;
  }
  if (pl->fused_k2) return MCLAHE_OK;  // counted by the range pass
  (void)A;
  launch_tile_major(pl->f32() ? 0 : 1, 1, pl->tile_grid, st, pl->G, in, W, pl->shared_ws ? 1 : 0);
  MG_LAUNCHED();
  return MCLAHE_OK;
}

// Mappings of window tiles [t0, t0 + nt) (nt < 0: the whole window).
int do_map(mclahe_plan_s* pl, void* ws, const mclahe_debug_t* dbg, cudaStream_t st,
           int64_t t0 = 0, int64_t nt = -1) {
  NvtxRange nvtx("mclahe.mappings");
  if (nt < 0) nt = pl->G.win_tiles - t0;
  if (nt <= 0) return MCLAHE_OK;
  WS W = ws_view(pl, ws);
  Debug D{};
  if (dbg) {
    D.lo = dbg->lo;
    D.hi = dbg->hi;
    D.counts = dbg->counts;
    D.clipped = dbg->clipped;
    D.lut = dbg->lut;
    D.degenerate = dbg->degenerate;
    if ((D.lo == nullptr) != (D.hi == nullptr))
      return fail(MCLAHE_ERR_VALIDATION, "debug lo and hi must both be set or both NULL");
  }
  const int warps = pl->map_block / 32;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nt + warps - 1) / warps, pl->map_grid));
  // per-value LUT rows of the mapped tiles: written by the mappings warps themselves
  // (MCLAHE_SPLIT_DLUT=1: by k_dict_luts in a launch of its own, A/B)
  static const bool split_dlut = getenv("MCLAHE_SPLIT_DLUT") != nullptr;
  const int fused_rows = (pl->dict_cap && pl->f32() && !split_dlut) ? 1 : 0;
  if (pl->f32())
    k_mappings<float><<<grid, pl->map_block, pl->map_smem, st>>>(pl->G, W, D, t0, nt, fused_rows);
  else k_mappings<double><<<grid, pl->map_block, pl->map_smem, st>>>(pl->G, W, D, t0, nt, 0);
  MG_LAUNCHED();
  if (pl->dict_cap && !fused_rows) {  // per-value LUT rows of the mapped tiles
    WS Wt = W;
    Wt.tparams = static_cast<char*>(W.tparams) + t0 * (int64_t)sizeof(TileParam<float>);
    Wt.lut = W.lut + t0 * pl->p.n_bins;
    Wt.lutd = W.lutd + t0 * kDictKC;
    Wt.thr = W.thr + t0 * (pl->p.n_bins + 1);
    // CTAs per SM for the per-value rows (a thread's entries are chains of dependent loads)
    static const int dl_mult = getenv("MCLAHE_DLUT_GRID") ? std::max(1, atoi(getenv("MCLAHE_DLUT_GRID"))) : 16;
    const int g = (int)std::min<int64_t>((nt * kDictKC + 255) / 256, (int64_t)pl->sms * dl_mult);
    k_dict_luts<float><<<g, 256, 0, st>>>(Wt, nt, (int)pl->p.n_bins);
    MG_LAUNCHED();
  }
  return MCLAHE_OK;
}

int do_interp(mclahe_plan_s* pl, const void* in, void* out, void* ws, cudaStream_t st) {
  NvtxRange nvtx("mclahe.interpolate");
  if (getenv("MCLAHE_DEBUG"))
    fprintf(stderr, "[mclahe] do_interp pencil=%d pending=%s\n", (int)pl->interp.on,
            cudaGetErrorString(cudaPeekAtLastError()));
  WS W = ws_view(pl, ws);
  const bool A = pl->p.adaptive != 0;
  if (pl->interp.on) {
    KGeom G = pencil_geom(*pl, pl->interp);
    // Large volumes hand units out dynamically (one atomic per unit): corner
    // tables and tile shapes make per-unit cost uneven, and a static split left
    // some SMs 30% idle at the tail. Below ~64M voxels the memset + atomics
    // cost more than the imbalance (3D config: 0.063 -> 0.068 ms), so the
    // balanced static split stays. MCLAHE_STATIC_UNITS forces static.
    static const bool static_units = getenv("MCLAHE_STATIC_UNITS") != nullptr;
    G.dyn_units = (static_units || pl->G.local_voxels < (int64_t{1} << 26)) ? 0 : (int)pl->interp_vox.size();
    if (G.dyn_units) MG_CUDA(cudaMemsetAsync(W.range + 3, 0, sizeof(int64_t), st));
    InterpFn f = interp_fn(pl->interp.ko, pl->interp.kt, A, pl->p.n_bins);
    int rc = tensor_map(pl, 1, in);
    if (rc) return rc;
    if ((rc = tensor_map(pl, 2, out))) return rc;
    if (getenv("MCLAHE_DEBUG")) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(f));
      fprintf(stderr,
              "[mclahe] interp ko=%d kt=%d grid=%d block=%d smem=%lld nst=%d rows=%d P=%lld regs=%d "
              "maxthr=%d static=%zu maxdyn=%d\n",
              pl->interp.ko, pl->interp.kt, pl->interp_grid, kBlendThreads,
              (long long)pl->interp.smem, pl->interp.nst, pl->interp.stage_rows,
              (long long)pl->interp.P, fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes,
              fa.maxDynamicSharedSizeBytes);
    }
    if (pl->mdict) {  // folded-pair dictionary blend; exits at once when the dictionary is unusable
      if ((rc = tensor_map(pl, 3, in))) return rc;
      if ((rc = tensor_map(pl, 4, out))) return rc;
      KGeom Gm = pencil_geom(*pl, pl->interp_m);
      Gm.seg_items = 1;
      Gm.dyn_units = (int)(pl->mdict_units.size() / kUnitInts) * pl->interp_m.nseg;
      if (!G.dyn_units) MG_CUDA(cudaMemsetAsync(W.range + 3, 0, sizeof(int64_t), st));
      const int grid = (int)std::min<int64_t>(Gm.dyn_units, pl->sms);
      // in-place results + TMA store (MCLAHE_MDICT_STG=1: per-lane global stores, A/B)
      static const bool tstore = getenv("MCLAHE_MDICT_STG") == nullptr;
      get_interp_mdict(pl->interp.ko, tstore, A, (int)pl->p.n_bins)<<<grid, interp_mdict_threads(A),
                                                                  pl->interp_m.smem, st>>>(
          Gm, pl->map[3], pl->map[4], static_cast<const float*>(in), static_cast<float*>(out),
          pl->d_tables + pl->off_mdict_units, pl->d_tables + pl->off_interp_cta, W);
      MG_LAUNCHED();
      if (!A) return MCLAHE_OK;  // global mode: the folded-pair blend is the blend
    } else if (pl->dict_cap) {  // value-dictionary blend; exits at once when the dictionary is unusable
      KGeom Gd = G;
      Gd.nst = pl->dict_nst;
      get_interp_pencil_dict(pl->interp.ko, pl->interp.kt)<<<pl->interp_grid, kBlendThreads,
                                                            pl->dict_smem, st>>>(
          Gd, pl->map[1], pl->map[2], static_cast<const float*>(in), static_cast<float*>(out),
          pl->d_tables + pl->off_interp_units, pl->d_tables + pl->off_interp_cta, W);
      MG_LAUNCHED();
    }
    f<<<pl->interp_grid, kBlendThreads, pl->interp.smem, st>>>(G, pl->map[1], pl->map[2], static_cast<const float*>(in),
                                                     static_cast<float*>(out),
                                                     pl->d_tables + pl->off_interp_units,
                                                     pl->d_tables + pl->off_interp_cta, W);
    MG_LAUNCHED();
    return MCLAHE_OK;
  }
  // cell-major blend when the 2^D corner LUTs fit shared memory
  if (((int64_t{1} << pl->p.rank) * pl->p.n_bins * 4) <= 200 * 1024 && !getenv("MCLAHE_GENERIC_BLEND")) {
    const Dim& d0 = pl->d[0];
    const int64_t c0 = cell_of(d0, pl->info.row_begin);
    const int64_t c1 = cell_of(d0, pl->info.row_end - 1);
    int64_t ncells = c1 - c0 + 1;
    for (int j = 1; j < pl->p.rank; ++j) ncells *= pl->d[j].g - 1;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ncells, (int64_t)pl->sms * 8));
    launch_interp_cell(pl->f32() ? 0 : 1, A ? 1 : 0, grid, st, pl->G, in, out, W, c0, c1 - c0 + 1);
    MG_LAUNCHED();
    return MCLAHE_OK;
  }
  const int grid = generic_grid(pl);
  if (pl->f32()) {
    if (A) k_interp_generic<float, true><<<grid, 256, 0, st>>>(pl->G, static_cast<const float*>(in), static_cast<float*>(out), W);
    else k_interp_generic<float, false><<<grid, 256, 0, st>>>(pl->G, static_cast<const float*>(in), static_cast<float*>(out), W);
  } else {
    if (A) k_interp_generic<double, true><<<grid, 256, 0, st>>>(pl->G, static_cast<const double*>(in), static_cast<double*>(out), W);
    else k_interp_generic<double, false><<<grid, 256, 0, st>>>(pl->G, static_cast<const double*>(in), static_cast<double*>(out), W);
  }
  MG_LAUNCHED();
  return MCLAHE_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int check_ptrs(const mclahe_plan_s* pl, const void* in, const void* out) {
  if (!in) return fail(MCLAHE_ERR_VALIDATION, "null input buffer");
  if ((pl->hist.on || pl->interp.on) && (!aligned16(in) || (out && !aligned16(out))))
    return fail(MCLAHE_ERR_VALIDATION, "device buffers must be 16-byte aligned");
  return MCLAHE_OK;
}

int64_t elem_size(const mclahe_params_t* p) { return p->dtype == MCLAHE_F64 ? 8 : 4; }

int64_t volume(const mclahe_params_t* p) {
  int64_t n = 1;
  for (int i = 0; i < p->rank; ++i) n *= p->shape[i];
  return n;
}

// ---- streamed one-shot (single GPU): chunked H2D -> passes -> D2H -------
// The volume is cut into cell-aligned chunks along dim 0, each with its own
// full-window plan over ONE shared workspace (counts and range keys are
// combined by the kernels' atomics).  H2D, compute and D2H run on three
// streams so PCIe in both directions overlaps the kernels; a pass for a tile
// row runs as soon as every chunk its support meets has been through the
// previous pass.
struct Streamed {
  std::vector<std::unique_ptr<mclahe_plan_s>> chunks;
  std::vector<int64_t> cuts;      // chunk row boundaries (C + 1)
  std::vector<int> last_chunk;    // per tile row: last chunk its support meets
  int64_t tiles_per_row = 0;
  // Out-of-core ring (in_slots > 0): the device holds in_slots input and
  // out_slots output chunk slots instead of the whole volume; chunk k's rows
  // live in input slot k % in_slots until it has been blended, its results in
  // output slot k % out_slots until they are back on the host.
  int in_slots = 0, out_slots = 0;
  int64_t slot_bytes = 0;
  std::vector<cudaEvent_t> rev;   // ring events: [0,C) landed, [C,2C) slot free, [2C,3C) D2H done, 3C..3C+2
  Streamed() = default;
  Streamed(const Streamed&) = delete;
  Streamed& operator=(const Streamed&) = delete;
  ~Streamed() {
    for (cudaEvent_t e : rev)
      if (e) cudaEventDestroy(e);
  }
};

int build_streamed(const mclahe_params_t* p, Streamed& S, int want_chunks = 0) {
  const Dim d0 = make_dim(p->shape[0], p->kernel[0]);
  std::vector<std::pair<int64_t, int64_t>> cells;
  for (int64_t c = 0; c + 1 < d0.g; ++c) {
    int64_t a, e;
    cell_range(d0, c, &a, &e);
    if (e > a) cells.push_back({a, e});
  }
  const int64_t bytes = volume(p) * elem_size(p);
  // Row-balanced chunks, not cell-aligned: a chunk's blend waits for the tile
  // rows its last cell touches, so the D2H tail after the final H2D is about
  // one cell of rows plus one chunk; more, smaller chunks shorten it.  Cuts on
  // multiples of 8 rows (or 1 for short volumes) keep TMA boxes whole.
  const int64_t S0 = p->shape[0];
  const int64_t align = S0 >= 128 ? 8 : 1;
  static const int max_chunks = std::max(
      2, std::min(kMaxChunks, getenv("MCLAHE_CHUNKS") ? atoi(getenv("MCLAHE_CHUNKS")) : 16));
  int C = (int)std::max<int64_t>(
      1, std::min<int64_t>({S0 / align, (int64_t)max_chunks, std::max<int64_t>(1, bytes / (8 << 20))}));
  if (want_chunks > 0) C = (int)std::max<int64_t>(1, std::min<int64_t>(S0 / align, want_chunks));
  if (C < 2 || cells.size() < 2) return MCLAHE_ERR_UNSUPPORTED;
  S.cuts.assign(1, 0);
  for (int k = 1; k < C; ++k) {
    const int64_t cut = (S0 * k / C) / align * align;
    if (cut > S.cuts.back() && cut < S0) S.cuts.push_back(cut);
  }
  S.cuts.push_back(S0);
  C = (int)S.cuts.size() - 1;
  S.chunks.clear();
  for (int k = 0; k < C; ++k) {
    auto pl = std::make_unique<mclahe_plan_s>();
    const int rc = plan_describe(p, S.cuts[k], S.cuts[k + 1], pl.get(), true);
    if (rc) return rc;
    S.chunks.push_back(std::move(pl));
  }
  S.tiles_per_row = S.chunks[0]->info.tiles_per_row;
  S.last_chunk.assign((size_t)d0.g, 0);
  for (int64_t t = 0; t < d0.g; ++t) {
    const TileParts tp = tile_parts(d0, t);
    const int64_t last_row = tp.support_end() - 1;
    int k = 0;
    while (k + 1 < C && S.cuts[k + 1] <= last_row) ++k;
    S.last_chunk[(size_t)t] = k;
  }
  return MCLAHE_OK;
}

// The step (index of the chunk whose arrival triggers it) at which each chunk
// is blended, by the rules run_streamed applies; `main_pass_global`: the
// second pass of a global-mode ring run (ranges known, a chunk is counted when
// it lands again).
std::vector<int> blend_steps(const Streamed& S, bool adaptive) {
  const int C = (int)S.chunks.size();
  const int64_t g0 = (int64_t)S.last_chunk.size();
  std::vector<int> step((size_t)C, -1);
  int hist = 0, blended = 0;
  int64_t params_rows = adaptive ? 0 : g0, mapped_rows = 0;
  for (int k = 0; k < C; ++k) {
    if (adaptive) {
      while (params_rows < g0 && S.last_chunk[(size_t)params_rows] < k + 1) ++params_rows;
      while (hist < C && S.chunks[(size_t)hist]->info.count_row_end <= params_rows) ++hist;
    } else {
      hist = k + 1;
    }
    while (mapped_rows < g0 && S.last_chunk[(size_t)mapped_rows] < hist) ++mapped_rows;
    while (blended < C && S.chunks[(size_t)blended]->info.need_row_end <= mapped_rows)
      step[(size_t)blended++] = k;
  }
  return step;
}

// Out-of-core plan: the finest chunking is tried last; the first chunk count
// whose ring (the chunks a blend waits for, one more to keep H2D running, and
// the output slots) fits `budget` bytes beside the workspace wins.
int build_ring(const mclahe_params_t* p, int64_t budget, std::unique_ptr<Streamed>& out) {
  const int64_t S0 = p->shape[0];
  const int64_t row_bytes = volume(p) / S0 * elem_size(p);
  int64_t best_need = INT64_MAX;
  for (int want = 16; ; want *= 2) {
    auto S = std::make_unique<Streamed>();
    const int rc = build_streamed(p, *S, want);
    if (rc != MCLAHE_OK && rc != MCLAHE_ERR_UNSUPPORTED) return rc;
    if (rc == MCLAHE_ERR_UNSUPPORTED)
      return fail(MCLAHE_ERR_OOM, "volume does not fit the device memory budget and cannot be chunked along dim 0");
    const int C = (int)S->chunks.size();
    const std::vector<int> step = blend_steps(*S, p->adaptive != 0);
    int lag = 0;
    for (int b = 0; b < C; ++b) {
      if (step[(size_t)b] < 0) return fail(MCLAHE_ERR_CUDA, "streamed schedule does not complete");
      lag = std::max(lag, step[(size_t)b] - b);
    }
    int64_t slot = 0;
    for (int k = 0; k < C; ++k) slot = std::max(slot, (S->cuts[(size_t)k + 1] - S->cuts[(size_t)k]) * row_bytes);
    slot = align_up(slot, 1024);
    const int64_t wsb = align_up(S->chunks[0]->info.workspace_bytes, 256);
    // preferred / minimal ring: lag + 2 in, 3 out / lag + 1 in, 2 out
    for (int slack = 1; slack >= 0; --slack) {
      const int ni = std::min(C, lag + 1 + slack), no = std::min(C, 2 + slack);
      const int64_t need = (ni + no) * slot + wsb;
      best_need = std::min(best_need, need);
      if (need <= budget) {
        S->in_slots = ni;
        S->out_slots = no;
        S->slot_bytes = slot;
        out = std::move(S);
        return MCLAHE_OK;
      }
    }
    if (C < want || want >= 4096) break;  // no finer chunking exists
  }
  return fail(MCLAHE_ERR_OOM, "volume does not fit the device memory budget: the out-of-core ring needs at least " +
                                  std::to_string(best_need) + " bytes (about 2.5 interpolation cells of dim-0 rows)");
}

int run_streamed(Streamed& S, const mclahe_params_t* p, const void* in, void* out, void* d_in,
                 void* d_out, void* ws, cudaStream_t s_in, cudaStream_t s_comp, cudaStream_t s_out,
                 std::vector<cudaEvent_t>& ev_shared, mclahe_timings_t* timings) {
  const int C = (int)S.chunks.size();
  const bool ring = S.in_slots > 0;
  // events: [0, C) inputs landed, [C, 2C) chunk blended (its input slot is
  // free), [2C, 3C) ring: output back on the host, 3C / 3C+1 timing, 3C+2 ring
  // pass boundary
  if (ring && S.rev.empty()) {
    S.rev.assign((size_t)(3 * C + 3), nullptr);
    for (auto& e : S.rev) MG_CUDA(cudaEventCreate(&e));
  }
  std::vector<cudaEvent_t>& ev = ring ? S.rev : ev_shared;
  const int T0 = ring ? 3 * C : 2 * C;
  if (ev.size() < (size_t)(T0 + 2)) return fail(MCLAHE_ERR_CUDA, "streamed run: too few events");
  const int64_t row_bytes = volume(p) / p->shape[0] * elem_size(p);
  const int64_t g0 = (int64_t)S.last_chunk.size();
  const int64_t tpr = S.tiles_per_row;
  const bool A = p->adaptive != 0;
  mclahe_plan_s* M = S.chunks[0].get();  // any chunk plan: same full-window layout
  int rc;
  for (auto& c : S.chunks)
    if ((rc = device_init(c.get()))) return rc;
  auto host_off = [&](int k) { return S.cuts[(size_t)k] * row_bytes; };
  auto chunk_len = [&](int k) { return (S.cuts[(size_t)k + 1] - S.cuts[(size_t)k]) * row_bytes; };
  auto in_ptr = [&](int k) {
    return static_cast<char*>(d_in) + (ring ? (k % S.in_slots) * S.slot_bytes : host_off(k));
  };
  auto out_ptr = [&](int k) {
    return static_cast<char*>(d_out) + (ring ? (k % S.out_slots) * S.slot_bytes : host_off(k));
  };
  // ring: a wait is only enqueued on an event recorded earlier in THIS call
  std::vector<char> freed((size_t)C, 0), back((size_t)C, 0), landed((size_t)C, 0);
  auto load = [&](int k) -> int {
    if (ring && k >= S.in_slots) {
      if (!freed[(size_t)(k - S.in_slots)]) return fail(MCLAHE_ERR_CUDA, "ring schedule: input slot still in use");
      MG_CUDA(cudaStreamWaitEvent(s_in, ev[(size_t)(C + k - S.in_slots)], 0));
    }
    MG_CUDA(cudaMemcpyAsync(in_ptr(k), static_cast<const char*>(in) + host_off(k), (size_t)chunk_len(k),
                            cudaMemcpyHostToDevice, s_in));
    MG_CUDA(cudaEventRecord(ev[(size_t)k], s_in));
    landed[(size_t)k] = 1;
    return MCLAHE_OK;
  };
  MG_CUDA(cudaEventRecord(ev[(size_t)T0], s_comp));
  if ((rc = do_reset(M, ws, s_comp))) return rc;
  bool gparams = false;
  if (ring && !A) {
    // global mode out of core: the range needs every voxel before any bin
    // exists, so the volume streams through the ring twice (range; counts + blend)
    for (int k = 0; k < C; ++k) {
      if ((rc = load(k))) return rc;
      MG_CUDA(cudaStreamWaitEvent(s_comp, ev[(size_t)k], 0));
      if ((rc = do_range(S.chunks[(size_t)k].get(), in_ptr(k), ws, s_comp))) return rc;
      MG_CUDA(cudaEventRecord(ev[(size_t)(C + k)], s_comp));
      freed[(size_t)k] = 1;
    }
    int64_t gflag = 0;
    MG_CUDA(cudaMemcpyAsync(&gflag, static_cast<char*>(ws) + M->info.off_range + 16, sizeof gflag,
                            cudaMemcpyDeviceToHost, s_comp));
    MG_CUDA(cudaStreamSynchronize(s_comp));  // every slot is free again
    if (gflag) return fail(MCLAHE_ERR_VALIDATION, "image contains non-finite values");
    if ((rc = do_params(M, ws, s_comp))) return rc;
    gparams = true;
    std::fill(freed.begin(), freed.end(), 0);
    std::fill(landed.begin(), landed.end(), 0);
  }
  if (!ring)
    for (int k = 0; k < C; ++k)
      if ((rc = load(k))) return rc;
  int ranged = gparams ? C : 0, hist = 0, blended = 0;
  int64_t params_rows = 0, mapped_rows = 0;
  for (int k = 0; k < C; ++k) {
    if (ring) {
      // first pass of a ring: in_slots chunks in flight; later chunks are
      // loaded as the blends free their slots (enqueued below, in order)
      if (k == 0)
        for (int j = 0; j < std::min(C, S.in_slots); ++j)
          if ((rc = load(j))) return rc;
    }
    if (ring && !landed[(size_t)k]) return fail(MCLAHE_ERR_CUDA, "ring schedule: chunk not loaded");
    MG_CUDA(cudaStreamWaitEvent(s_comp, ev[(size_t)k], 0));
    mclahe_plan_s* pk = S.chunks[(size_t)k].get();
    if (!gparams || A) {
      if ((rc = do_range(pk, in_ptr(k), ws, s_comp))) return rc;
      ranged = k + 1;
    }
    // binning parameters: tile rows whose support is fully ranged (adaptive),
    // or the global range once every chunk is in
    if (A) {
      int64_t r = params_rows;
      while (r < g0 && S.last_chunk[(size_t)r] < ranged) ++r;
      if (r > params_rows) {
        if ((rc = do_params(M, ws, s_comp, params_rows * tpr, (r - params_rows) * tpr))) return rc;
        params_rows = r;
      }
    } else if (ranged == C && !gparams) {
      // global mode: every voxel has been through the range pass before any
      // bin exists, so the non-finite flag is final here -- report it before
      // any blend or D2H touches the caller's buffer (the reference throws
      // before it writes anything, src/pipeline.cpp:33)
      int64_t gflag = 0;
      MG_CUDA(cudaMemcpyAsync(&gflag, static_cast<char*>(ws) + M->info.off_range + 16,
                              sizeof gflag, cudaMemcpyDeviceToHost, s_comp));
      MG_CUDA(cudaStreamSynchronize(s_comp));
      if (gflag) return fail(MCLAHE_ERR_VALIDATION, "image contains non-finite values");
      if ((rc = do_params(M, ws, s_comp))) return rc;
      gparams = true;
    }
    // histograms of chunks whose counted tile rows all have parameters (the
    // second pass of a global-mode ring counts a chunk when it lands again)
    while (hist < C) {
      mclahe_plan_s* ph = S.chunks[(size_t)hist].get();
      const bool ready = A ? ph->info.count_row_end <= params_rows : (gparams && (!ring || hist <= k));
      if (!ready) break;
      if ((rc = do_hist(ph, in_ptr(hist), ws, s_comp))) return rc;
      ++hist;
    }
    // mappings of tile rows whose every counting chunk is done
    int64_t r = mapped_rows;
    while (r < g0 && S.last_chunk[(size_t)r] < hist) ++r;
    if (r > mapped_rows) {
      if ((rc = do_map(M, ws, nullptr, s_comp, mapped_rows * tpr, (r - mapped_rows) * tpr)))
        return rc;
      mapped_rows = r;
    }
    // blend + D2H of chunks whose tile rows are all mapped
    while (blended < C && S.chunks[(size_t)blended]->info.need_row_end <= mapped_rows) {
      mclahe_plan_s* pb = S.chunks[(size_t)blended].get();
      if (ring && blended >= S.out_slots) {
        if (!back[(size_t)(blended - S.out_slots)]) return fail(MCLAHE_ERR_CUDA, "ring schedule: output slot still in use");
        MG_CUDA(cudaStreamWaitEvent(s_comp, ev[(size_t)(2 * C + blended - S.out_slots)], 0));
      }
      if ((rc = do_interp(pb, in_ptr(blended), out_ptr(blended), ws, s_comp))) return rc;
      MG_CUDA(cudaEventRecord(ev[(size_t)(C + blended)], s_comp));
      freed[(size_t)blended] = 1;
      MG_CUDA(cudaStreamWaitEvent(s_out, ev[(size_t)(C + blended)], 0));
      MG_CUDA(cudaMemcpyAsync(static_cast<char*>(out) + host_off(blended), out_ptr(blended),
                              (size_t)chunk_len(blended), cudaMemcpyDeviceToHost, s_out));
      if (ring) {
        MG_CUDA(cudaEventRecord(ev[(size_t)(2 * C + blended)], s_out));
        back[(size_t)blended] = 1;
        // the freed input slot takes the next chunk not yet on its way
        const int nxt = blended + S.in_slots;
        if (nxt < C && (rc = load(nxt))) return rc;
      }
      ++blended;
    }
  }
  if (blended != C) return fail(MCLAHE_ERR_CUDA, "streamed schedule did not complete");
  MG_CUDA(cudaEventRecord(ev[(size_t)(T0 + 1)], s_comp));
  int64_t flag = 0;
  MG_CUDA(cudaMemcpyAsync(&flag, static_cast<char*>(ws) + M->info.off_range + 16, sizeof flag,
                          cudaMemcpyDeviceToHost, s_comp));
  MG_CUDA(cudaStreamSynchronize(s_comp));
  MG_CUDA(cudaStreamSynchronize(s_out));
  if (flag) {
    // adaptive mode: early chunks were blended and copied back while later
    // chunks were still arriving; scrub the caller's buffer so no partial
    // result survives the error (NaN is never a valid output)
    const int64_t n = volume(p);
    if (p->dtype == MCLAHE_F64)
      std::fill_n(static_cast<double*>(out), n, std::numeric_limits<double>::quiet_NaN());
    else
      std::fill_n(static_cast<float*>(out), n, std::numeric_limits<float>::quiet_NaN());
    return fail(MCLAHE_ERR_VALIDATION, "image contains non-finite values");
  }
  if (timings) {
    float total = 0.f;
    MG_CUDA(cudaEventElapsedTime(&total, ev[(size_t)T0], ev[(size_t)(T0 + 1)]));
    timings->histograms_s += total * 1e-3;  // interleaved passes: reported as one span
  }
  return MCLAHE_OK;
}

// ---- one-shot context: cached plan + buffers ----
struct OneShot {
  std::mutex mu;
  std::map<std::string, std::unique_ptr<mclahe_plan_s>> plans;
  void* buf = nullptr;
  size_t buf_bytes = 0;
  int buf_dev = -1;
  cudaStream_t stream = nullptr;
  int stream_dev = -1;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t s_in = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> sev;  // streamed-run events
  std::map<std::string, std::unique_ptr<Streamed>> streamed;
};
OneShot& oneshot() {
  static OneShot* o = new OneShot();  // intentionally leaked (process lifetime)
  return *o;
}

std::string plan_key(const mclahe_params_t* p, int dev) {
  std::string k(reinterpret_cast<const char*>(p), sizeof *p);
  k.append(reinterpret_cast<const char*>(&dev), sizeof dev);
  return k;
}

mclahe_plan_s* cached_plan(OneShot& o, const mclahe_params_t* p, int* rc, int frame_axis = -1) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    *rc = cuda_fail(e, "cudaGetDevice");
    return nullptr;
  }
  mclahe_params_t q = *p;
  q.reserved = 0;
  for (int i = q.rank; i < MCLAHE_MAX_RANK; ++i) q.shape[i] = q.kernel[i] = 0;
  std::string key = plan_key(&q, dev);
  key.append(reinterpret_cast<const char*>(&frame_axis), sizeof frame_axis);
  auto it = o.plans.find(key);
  if (it != o.plans.end()) return it->second.get();
  auto pl = std::make_unique<mclahe_plan_s>();
  *rc = plan_describe(&q, 0, q.shape[0], pl.get());
  if (*rc) return nullptr;
  if (frame_axis >= 0) {  // per-frame global ranges: K2a and the dictionary stay off
    pl->frame_axis = frame_axis;
    pl->dict_cap = 0;
    // the plan was described as adaptive, so plan_mdict may have armed the
    // folded-pair dictionary blend; with no dictionary it has no tables
    pl->mdict = false;
    // the frame range pass sets the tiles' ranges; the counts come from the
    // histogram pass (no fused tile-major range + counts)
    pl->fused_k2 = false;
    pl->fused_pencil = false;
    pl->off_frange = align_up(pl->info.workspace_bytes, 256);
    pl->info.workspace_bytes = align_up(pl->off_frange + q.shape[frame_axis] * 16, 256);
  }
  *rc = device_init(pl.get());
  if (*rc) return nullptr;
  if (o.plans.size() > 32) o.plans.clear();
  mclahe_plan_s* raw = pl.get();
  o.plans[key] = std::move(pl);
  return raw;
}

int ensure_buf(OneShot& o, size_t bytes) {
  int dev;
  MG_CUDA(cudaGetDevice(&dev));
  if (o.buf && o.buf_bytes >= bytes && o.buf_dev == dev) return MCLAHE_OK;
  if (o.buf) {
    cudaFree(o.buf);
    o.buf = nullptr;
  }
  MG_CUDA(cudaMalloc(&o.buf, bytes));
  o.buf_bytes = bytes;
  o.buf_dev = dev;
  return MCLAHE_OK;
}

int ensure_stream(OneShot& o) {
  int dev;
  MG_CUDA(cudaGetDevice(&dev));
  if (o.stream && o.stream_dev == dev) return MCLAHE_OK;
  MG_CUDA(cudaStreamCreateWithFlags(&o.stream, cudaStreamNonBlocking));
  MG_CUDA(cudaStreamCreateWithFlags(&o.s_in, cudaStreamNonBlocking));
  MG_CUDA(cudaStreamCreateWithFlags(&o.s_out, cudaStreamNonBlocking));
  for (auto& e : o.ev) MG_CUDA(cudaEventCreate(&e));
  o.sev.resize(2 * kMaxChunks + 2);
  for (auto& e : o.sev) MG_CUDA(cudaEventCreate(&e));
  o.stream_dev = dev;
  return MCLAHE_OK;
}

int enqueue_all(mclahe_plan_s* pl, const void* in, void* out, void* ws, cudaStream_t st,
                cudaEvent_t* ev) {
  int rc;
  // the dictionary numbering (~14 us, one CTA) leaves the critical path: it
  // runs on a side branch beside params / edge tables / histograms and joins
  // before the mappings pass (MCLAHE_NO_FORK=1 keeps one stream)
  static const bool no_fork = getenv("MCLAHE_NO_FORK") != nullptr;
  const bool fork = !no_fork && pl->dict_cap > 0 && pl->hist.on && !pl->fused_pencil &&
                    pl->frame_axis < 0 && pl->side != nullptr;
  if (ev) MG_CUDA(cudaEventRecord(ev[0], st));
  if ((rc = do_reset(pl, ws, st))) return rc;
  if ((rc = do_range(pl, in, ws, st, fork))) return rc;
  if ((rc = do_params(pl, ws, st))) return rc;
  // (the cell-counting K2b reads the numbered dictionary: it joins before the histograms)
  if (fork && pl->cell_hist) MG_CUDA(cudaStreamWaitEvent(st, pl->ev_join, 0));
  if ((rc = do_hist(pl, in, ws, st))) return rc;
  if (fork && !pl->cell_hist) MG_CUDA(cudaStreamWaitEvent(st, pl->ev_join, 0));
  if ((rc = do_map(pl, ws, nullptr, st))) return rc;
  if (ev) MG_CUDA(cudaEventRecord(ev[1], st));
  if ((rc = do_interp(pl, in, out, ws, st))) return rc;
  if (ev) MG_CUDA(cudaEventRecord(ev[2], st));
  return MCLAHE_OK;
}

int read_status(const mclahe_plan_s* pl, const void* ws, cudaStream_t st) {
  int64_t flag = 0;
  MG_CUDA(cudaMemcpyAsync(&flag, static_cast<const char*>(ws) + pl->info.off_range + 16,
                          sizeof flag, cudaMemcpyDeviceToHost, st));
  MG_CUDA(cudaStreamSynchronize(st));
  if (flag) return fail(MCLAHE_ERR_VALIDATION, "image contains non-finite values");
  return MCLAHE_OK;
}





}  // namespace

namespace {

// One plan over the whole volume: H2D, every pass, non-finite check, D2H.
int run_plan_host(OneShot& o, mclahe_plan_s* pl, const void* in, void* out, size_t bytes,
                  size_t io, mclahe_timings_t* timings) {
  int rc;
  if ((rc = ensure_buf(o, 2 * io + (size_t)pl->info.workspace_bytes))) return rc;
  if ((rc = ensure_stream(o))) return rc;
  char* base = static_cast<char*>(o.buf);
  void* d_in = base;
  void* d_out = base + io;
  void* ws = base + 2 * io;
  cudaStream_t st = o.stream;
  MG_CUDA(cudaMemcpyAsync(d_in, in, bytes, cudaMemcpyHostToDevice, st));
  if ((rc = enqueue_all(pl, d_in, d_out, ws, st, timings ? o.ev : nullptr))) return rc;
  int64_t flag = 0;
  MG_CUDA(cudaMemcpyAsync(&flag, static_cast<char*>(ws) + pl->info.off_range + 16, sizeof flag,
                          cudaMemcpyDeviceToHost, st));
  MG_CUDA(cudaStreamSynchronize(st));
  if (flag) return fail(MCLAHE_ERR_VALIDATION, "image contains non-finite values");
  MG_CUDA(cudaMemcpyAsync(out, d_out, bytes, cudaMemcpyDeviceToHost, st));
  MG_CUDA(cudaStreamSynchronize(st));
  if (timings) {
    float a = 0, b = 0;
    MG_CUDA(cudaEventElapsedTime(&a, o.ev[0], o.ev[1]));
    MG_CUDA(cudaEventElapsedTime(&b, o.ev[1], o.ev[2]));
    timings->histograms_s += a * 1e-3;
    timings->interpolation_s += b * 1e-3;
  }
  return MCLAHE_OK;
}

}  // namespace

// ---- multi-slab / multi-device run ---------------------
// The volume is cut along dim 0 at interpolation-cell boundaries into
// row-balanced slabs (the cut rule of slabs.py: slab_cuts).  Each slab has its
// own window plan, device buffers and stream on its device; devices may
// repeat (logical slabs on one GPU run the identical code path).  The only
// cross-slab traffic:
//   * range keys (~key(lo), key(hi), non-finite): MAX over all slabs;
//   * adaptive: per-tile range keys of tile rows two windows share: MAX;
//   * the partial integer counts of shared tile rows: SUM.
// Each slab snapshots the rows it shares into its own exchange buffer (so a
// neighbour's in-place combine never feeds back), records an event, and the
// combine kernel of every slab reads its peers' snapshots directly -- peer
// memory over NVLink / NVSwitch when the device differs (P2P enabled),
// local memory for logical slabs; when P2P is unavailable the snapshot is
// first staged with cudaMemcpyPeerAsync.  Integer MAX / SUM are order-free,
// so every slab's counts, LUTs and output equal the one-device run bit for bit.
namespace {

__global__ void k_combine_max(int64_t* __restrict__ dst, const int64_t* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = max(dst[i], src[i]);
}

__global__ void k_combine_sum(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src,
                              int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

// Cell-aligned, row-balanced cuts (slabs.py: slab_cuts).
int multi_cuts(const mclahe_params_t* p, int slabs, std::vector<int64_t>& cuts) {
  const Dim d0 = make_dim(p->shape[0], p->kernel[0]);
  std::vector<std::pair<int64_t, int64_t>> cells;
  for (int64_t c = 0; c + 1 < d0.g; ++c) {
    int64_t a, e;
    cell_range(d0, c, &a, &e);
    if (e > a) cells.push_back({a, e});
  }
  if (slabs < 1 || slabs > (int)cells.size())
    return fail(MCLAHE_ERR_VALIDATION, "cannot split " + std::to_string(cells.size()) +
                                           " interpolation cells along dim 0 over " +
                                           std::to_string(slabs) + " slabs");
  cuts.assign(1, 0);
  int ci = 0;
  for (int r = 0; r < slabs; ++r) {
    int e = (int)cells.size();
    if (r < slabs - 1) {
      const double target = (double)p->shape[0] * (r + 1) / slabs;
      const int lo_e = ci + 1, hi_e = (int)cells.size() - (slabs - r - 1);
      e = lo_e;
      for (int k = lo_e; k <= hi_e; ++k)
        if (std::fabs((double)cells[k - 1].second - target) <
            std::fabs((double)cells[e - 1].second - target))
          e = k;
    }
    cuts.push_back(cells[e - 1].second);
    ci = e;
  }
  return MCLAHE_OK;
}

struct Slab {
  std::unique_ptr<mclahe_plan_s> plan;
  int dev = 0;
  cudaStream_t st = nullptr;
  cudaEvent_t ev_range = nullptr, ev_counts = nullptr, ev_t[3] = {nullptr, nullptr, nullptr};
  void* buf = nullptr;            // d_in | d_out | workspace | snapshots | staging
  char *d_in = nullptr, *d_out = nullptr, *ws = nullptr;
  int64_t* snap_keys = nullptr;   // range keys [4]
  int64_t* snap_trange = nullptr; // tile range keys of rows [ov_a, ov_b)
  uint32_t* snap_counts = nullptr;// counts of rows [ov_a, ov_b)
  char* stage = nullptr;          // peer snapshots staged here when P2P is unavailable
  int64_t ov_a = 0, ov_b = 0;     // union of the tile rows shared with any peer
  int64_t rows = 0;
};

struct Multi {
  std::vector<Slab> slabs;
  std::vector<int64_t> cuts;
  size_t stage_bytes = 0;
  ~Multi() {
    for (Slab& s : slabs) {
      cudaSetDevice(s.dev);
      if (s.buf) cudaFree(s.buf);
      if (s.st) cudaStreamDestroy(s.st);
      for (cudaEvent_t e : {s.ev_range, s.ev_counts, s.ev_t[0], s.ev_t[1], s.ev_t[2]})
        if (e) cudaEventDestroy(e);
    }
  }
};

bool can_read(int dev, int peer) {
  if (dev == peer) return true;
  int ok = 0;
  return cudaDeviceCanAccessPeer(&ok, dev, peer) == cudaSuccess && ok;
}

int build_multi(const mclahe_params_t* p, int n, const int32_t* devices, Multi& M) {
  int rc = multi_cuts(p, n, M.cuts);
  if (rc) return rc;
  int ndev = 0;
  MG_CUDA(cudaGetDeviceCount(&ndev));
  for (int r = 0; r < n; ++r)
    if (devices[r] < 0 || devices[r] >= ndev)
      return fail(MCLAHE_ERR_VALIDATION, "device id " + std::to_string(devices[r]) + " out of range");
  // peer access between every pair of distinct devices
  for (int r = 0; r < n; ++r)
    for (int q = 0; q < n; ++q) {
      if (devices[r] == devices[q] || !can_read(devices[r], devices[q])) continue;
      MG_CUDA(cudaSetDevice(devices[r]));
      const cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      cudaGetLastError();
    }
  M.slabs.resize((size_t)n);
  const int64_t row_bytes = volume(p) / p->shape[0] * elem_size(p);
  const int64_t n_bins = p->n_bins;
  for (int r = 0; r < n; ++r) {
    Slab& S = M.slabs[(size_t)r];
    S.dev = devices[r];
    MG_CUDA(cudaSetDevice(S.dev));
    S.plan = std::make_unique<mclahe_plan_s>();
    if ((rc = plan_describe(p, M.cuts[r], M.cuts[r + 1], S.plan.get()))) return rc;
    if ((rc = device_init(S.plan.get()))) return rc;
    S.rows = M.cuts[r + 1] - M.cuts[r];
    const mclahe_plan_info_t& I = S.plan->info;
    S.ov_a = INT64_MAX;
    S.ov_b = INT64_MIN;
    for (int q = 0; q < n; ++q) {
      if (q == r) continue;
      mclahe_plan_s tmp;
      if ((rc = plan_describe(p, M.cuts[q], M.cuts[q + 1], &tmp))) return rc;
      const int64_t a = std::max(I.tile_row_begin, tmp.info.tile_row_begin);
      const int64_t b = std::min(I.tile_row_end, tmp.info.tile_row_end);
      if (b > a) {
        S.ov_a = std::min(S.ov_a, a);
        S.ov_b = std::max(S.ov_b, b);
      }
    }
    if (S.ov_b <= S.ov_a) S.ov_a = S.ov_b = I.tile_row_begin;
  }
  // one allocation per slab: in | out | workspace | snapshots | staging
  int64_t max_ov = 0;
  for (Slab& S : M.slabs) max_ov = std::max(max_ov, S.ov_b - S.ov_a);
  const int64_t tpr = M.slabs[0].plan->info.tiles_per_row;
  const int64_t snap_tr = max_ov * tpr * 16, snap_cnt = max_ov * tpr * n_bins * 4;
  M.stage_bytes = (size_t)align_up(32 + snap_tr + snap_cnt, 256);
  for (Slab& S : M.slabs) {
    MG_CUDA(cudaSetDevice(S.dev));
    const int64_t io = align_up(S.rows * row_bytes, 256);
    const int64_t wsb = align_up(S.plan->info.workspace_bytes, 256);
    const int64_t total = 2 * io + wsb + 4 * (int64_t)M.stage_bytes;  // snapshots + 3 staging slots
    MG_CUDA(cudaMalloc(&S.buf, (size_t)total));
    char* b = static_cast<char*>(S.buf);
    S.d_in = b;
    S.d_out = b + io;
    S.ws = b + 2 * io;
    char* snap = S.ws + wsb;
    S.snap_keys = reinterpret_cast<int64_t*>(snap);
    S.snap_trange = reinterpret_cast<int64_t*>(snap + 32);
    S.snap_counts = reinterpret_cast<uint32_t*>(snap + 32 + snap_tr);
    S.stage = snap + M.stage_bytes;  // staging slots 0 / 1 / 2: keys, tile ranges, counts
    MG_CUDA(cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking));
    MG_CUDA(cudaEventCreateWithFlags(&S.ev_range, cudaEventDisableTiming));
    MG_CUDA(cudaEventCreateWithFlags(&S.ev_counts, cudaEventDisableTiming));
    for (cudaEvent_t& e : S.ev_t) MG_CUDA(cudaEventCreate(&e));
  }
  return MCLAHE_OK;
}

// Pointer of peer q's snapshot readable by slab r's device: direct, or
// staged into r's staging slot with a peer copy on r's stream.
int peer_view(Multi& M, int r, int q, const void* src, int64_t bytes, int slot, const void** out) {
  Slab& S = M.slabs[(size_t)r];
  const Slab& Q = M.slabs[(size_t)q];
  if (can_read(S.dev, Q.dev)) {
    *out = src;
    return MCLAHE_OK;
  }
  char* dst = S.stage + slot * (int64_t)M.stage_bytes;
  MG_CUDA(cudaMemcpyPeerAsync(dst, S.dev, src, Q.dev, (size_t)bytes, S.st));
  *out = dst;
  return MCLAHE_OK;
}

int grid_n(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 2048)); }

// Slab r's combine of the rows [a, b) it shares with peer q (op 0: MAX of the
// tile range keys, 1: SUM of counts).
int combine_rows(Multi& M, int r, int q, int op, int slot) {
  Slab& S = M.slabs[(size_t)r];
  const Slab& Q = M.slabs[(size_t)q];
  const mclahe_plan_info_t& I = S.plan->info;
  const mclahe_plan_info_t& J = Q.plan->info;
  const int64_t a = std::max(I.tile_row_begin, J.tile_row_begin);
  const int64_t b = std::min(I.tile_row_end, J.tile_row_end);
  if (b <= a) return MCLAHE_OK;
  const int64_t tpr = I.tiles_per_row, nb = I.n_bins;
  const int64_t per = op == 0 ? tpr * 2 : tpr * nb;  // elements per tile row
  const int64_t n = (b - a) * per;
  const void* src;
  int rc;
  if (op == 0) {
    const int64_t* qs = Q.snap_trange + (a - Q.ov_a) * per;
    if ((rc = peer_view(M, r, q, qs, n * 8, slot, &src))) return rc;
    int64_t* dst = reinterpret_cast<int64_t*>(S.ws + I.off_tile_range) + (a - I.tile_row_begin) * per;
    k_combine_max<<<grid_n(n), 256, 0, S.st>>>(dst, static_cast<const int64_t*>(src), n);
  } else {
    const uint32_t* qs = Q.snap_counts + (a - Q.ov_a) * per;
    if ((rc = peer_view(M, r, q, qs, n * 4, slot, &src))) return rc;
    uint32_t* dst = reinterpret_cast<uint32_t*>(S.ws + I.off_counts) + (a - I.tile_row_begin) * per;
    k_combine_sum<<<grid_n(n), 256, 0, S.st>>>(dst, static_cast<const uint32_t*>(src), n);
  }
  MG_LAUNCHED();
  return MCLAHE_OK;
}

// One multi-slab run.  host_in / host_out: whole-volume HOST buffers (each
// slab copies its rows on its own stream), else in_dev / out_dev: per-slab
// DEVICE buffers (slab r's rows on devices[r]).
int run_multi(Multi& M, const mclahe_params_t* p, const void* host_in, void* host_out,
              const void* const* in_dev, void* const* out_dev, mclahe_timings_t* timings) {
  const int n = (int)M.slabs.size();
  const int64_t row_bytes = volume(p) / p->shape[0] * elem_size(p);
  const bool A = p->adaptive != 0;
  int rc;
  auto in_of = [&](int r) -> const void* { return host_in ? M.slabs[(size_t)r].d_in : in_dev[r]; };
  auto out_of = [&](int r) -> void* { return host_out ? M.slabs[(size_t)r].d_out : out_dev[r]; };
  // pass 1 per slab, then its snapshots
  for (int r = 0; r < n; ++r) {
    Slab& S = M.slabs[(size_t)r];
    MG_CUDA(cudaSetDevice(S.dev));
    if (host_in)
      MG_CUDA(cudaMemcpyAsync(S.d_in, static_cast<const char*>(host_in) + M.cuts[r] * row_bytes,
                              (size_t)(S.rows * row_bytes), cudaMemcpyHostToDevice, S.st));
    MG_CUDA(cudaEventRecord(S.ev_t[0], S.st));
    if ((rc = do_reset(S.plan.get(), S.ws, S.st))) return rc;
    if ((rc = do_range(S.plan.get(), in_of(r), S.ws, S.st))) return rc;
    const mclahe_plan_info_t& I = S.plan->info;
    MG_CUDA(cudaMemcpyAsync(S.snap_keys, S.ws + I.off_range, 32, cudaMemcpyDeviceToDevice, S.st));
    if (A && S.ov_b > S.ov_a)
      MG_CUDA(cudaMemcpyAsync(S.snap_trange,
                              S.ws + I.off_tile_range + (S.ov_a - I.tile_row_begin) * I.tiles_per_row * 16,
                              (size_t)((S.ov_b - S.ov_a) * I.tiles_per_row * 16),
                              cudaMemcpyDeviceToDevice, S.st));
    MG_CUDA(cudaEventRecord(S.ev_range, S.st));
  }
  // range exchange: keys MAX over every slab, shared tile ranges MAX with the neighbours
  for (int r = 0; r < n; ++r) {
    Slab& S = M.slabs[(size_t)r];
    MG_CUDA(cudaSetDevice(S.dev));
    for (int q = 0; q < n; ++q) {
      if (q == r) continue;
      MG_CUDA(cudaStreamWaitEvent(S.st, M.slabs[(size_t)q].ev_range, 0));
      const void* src;
      if ((rc = peer_view(M, r, q, M.slabs[(size_t)q].snap_keys, 24, 0, &src))) return rc;
      k_combine_max<<<1, 32, 0, S.st>>>(reinterpret_cast<int64_t*>(S.ws + S.plan->info.off_range),
                                        static_cast<const int64_t*>(src), 3);
      MG_LAUNCHED();
      if (A && (rc = combine_rows(M, r, q, 0, 1))) return rc;
    }
    if ((rc = do_params(S.plan.get(), S.ws, S.st))) return rc;
    if ((rc = do_hist(S.plan.get(), in_of(r), S.ws, S.st))) return rc;
    const mclahe_plan_info_t& I = S.plan->info;
    if (S.ov_b > S.ov_a)
      MG_CUDA(cudaMemcpyAsync(S.snap_counts,
                              S.ws + I.off_counts + (S.ov_a - I.tile_row_begin) * I.tiles_per_row * I.n_bins * 4,
                              (size_t)((S.ov_b - S.ov_a) * I.tiles_per_row * I.n_bins * 4),
                              cudaMemcpyDeviceToDevice, S.st));
    MG_CUDA(cudaEventRecord(S.ev_counts, S.st));
  }
  // counts exchange (SUM with the neighbours), mappings, blend
  for (int r = 0; r < n; ++r) {
    Slab& S = M.slabs[(size_t)r];
    MG_CUDA(cudaSetDevice(S.dev));
    for (int q = 0; q < n; ++q) {
      if (q == r) continue;
      MG_CUDA(cudaStreamWaitEvent(S.st, M.slabs[(size_t)q].ev_counts, 0));
      if ((rc = combine_rows(M, r, q, 1, 2))) return rc;
    }
    if ((rc = do_map(S.plan.get(), S.ws, nullptr, S.st))) return rc;
    MG_CUDA(cudaEventRecord(S.ev_t[1], S.st));
    if ((rc = do_interp(S.plan.get(), in_of(r), out_of(r), S.ws, S.st))) return rc;
    MG_CUDA(cudaEventRecord(S.ev_t[2], S.st));
  }
  // every slab's flag is the combined (global) one: read slab 0's
  int64_t flag = 0;
  {
    Slab& S = M.slabs[0];
    MG_CUDA(cudaSetDevice(S.dev));
    MG_CUDA(cudaMemcpyAsync(&flag, S.ws + S.plan->info.off_range + 16, 8, cudaMemcpyDeviceToHost, S.st));
    MG_CUDA(cudaStreamSynchronize(S.st));
  }
  for (Slab& S : M.slabs) {
    MG_CUDA(cudaSetDevice(S.dev));
    MG_CUDA(cudaStreamSynchronize(S.st));
  }
  if (flag) return fail(MCLAHE_ERR_VALIDATION, "image contains non-finite values");
  if (host_out)
    for (int r = 0; r < n; ++r) {
      Slab& S = M.slabs[(size_t)r];
      MG_CUDA(cudaSetDevice(S.dev));
      MG_CUDA(cudaMemcpyAsync(static_cast<char*>(host_out) + M.cuts[r] * row_bytes, S.d_out,
                              (size_t)(S.rows * row_bytes), cudaMemcpyDeviceToHost, S.st));
    }
  double hist_s = 0, interp_s = 0;
  for (Slab& S : M.slabs) {
    MG_CUDA(cudaSetDevice(S.dev));
    MG_CUDA(cudaStreamSynchronize(S.st));
    float a = 0, b = 0;
    MG_CUDA(cudaEventElapsedTime(&a, S.ev_t[0], S.ev_t[1]));
    MG_CUDA(cudaEventElapsedTime(&b, S.ev_t[1], S.ev_t[2]));
    hist_s = std::max(hist_s, a * 1e-3);
    interp_s = std::max(interp_s, b * 1e-3);
  }
  if (timings) {
    timings->histograms_s += hist_s;
    timings->interpolation_s += interp_s;
  }
  return MCLAHE_OK;
}

std::mutex g_multi_mu;
std::map<std::string, std::unique_ptr<Multi>>& multi_cache() {
  static auto* c = new std::map<std::string, std::unique_ptr<Multi>>();
  return *c;
}

int multi_get(const mclahe_params_t* params, int32_t n, const int32_t* devices, Multi** out) {
  int rc = validate(params);
  if (rc) return rc;
  if (n < 1 || !devices) return fail(MCLAHE_ERR_VALIDATION, "need at least one slab and a device list");
  mclahe_params_t q = *params;
  q.reserved = 0;
  for (int i = q.rank; i < MCLAHE_MAX_RANK; ++i) q.shape[i] = q.kernel[i] = 0;
  std::string key(reinterpret_cast<const char*>(&q), sizeof q);
  key.append(reinterpret_cast<const char*>(devices), sizeof(int32_t) * (size_t)n);
  auto& C = multi_cache();
  auto it = C.find(key);
  if (it == C.end()) {
    int cur = 0;
    MG_CUDA(cudaGetDevice(&cur));
    auto M = std::make_unique<Multi>();
    rc = build_multi(&q, n, devices, *M);
    cudaSetDevice(cur);
    if (rc) return rc;
    if (C.size() > 4) C.clear();
    it = C.emplace(key, std::move(M)).first;
  }
  *out = it->second.get();
  return MCLAHE_OK;
}

}  // namespace

extern "C" {

const char* mclahe_last_error(void) { return g_last_error.c_str(); }
const char* mclahe_version(void) { return "mclahe-b200 0.1 (sm_100a)"; }
int64_t mclahe_launch_count(void) { return g_launches.load(); }

int mclahe_plan_create(const mclahe_params_t* params, int64_t row_begin, int64_t row_end,
                       mclahe_plan_t* plan) {
  if (!plan) return fail(MCLAHE_ERR_VALIDATION, "null plan pointer");
  *plan = nullptr;
  try {
    auto pl = std::make_unique<mclahe_plan_s>();
    const int rc = plan_describe(params, row_begin, row_end, pl.get());
    if (rc) return rc;
    *plan = pl.release();
    return MCLAHE_OK;
  } catch (const std::bad_alloc&) {
    return fail(MCLAHE_ERR_OOM, "host allocation failed");
  }
}

int mclahe_plan_destroy(mclahe_plan_t plan) {
  if (!plan) return MCLAHE_OK;
  delete plan;
  return MCLAHE_OK;
}

int mclahe_plan_get_info(mclahe_plan_t plan, mclahe_plan_info_t* info) {
  if (!plan || !info) return fail(MCLAHE_ERR_VALIDATION, "null plan or info");
  *info = plan->info;
  return MCLAHE_OK;
}

#define MG_PLAN_INIT(pl)                       \
  do {                                         \
    if (!(pl)) return fail(MCLAHE_ERR_VALIDATION, "null plan"); \
    int rc_ = device_init(pl);                 \
    if (rc_) return rc_;                       \
  } while (0)

int mclahe_pass_reset(mclahe_plan_t plan, void* ws, void* stream) {
  MG_PLAN_INIT(plan);
  return do_reset(plan, ws, static_cast<cudaStream_t>(stream));
}

int mclahe_pass_range(mclahe_plan_t plan, const void* in, void* ws, void* stream) {
  MG_PLAN_INIT(plan);
  int rc = check_ptrs(plan, in, nullptr);
  if (rc) return rc;
  return do_range(plan, in, ws, static_cast<cudaStream_t>(stream));
}

int mclahe_pass_params(mclahe_plan_t plan, void* ws, void* stream) {
  MG_PLAN_INIT(plan);
  return do_params(plan, ws, static_cast<cudaStream_t>(stream));
}

int mclahe_pass_histograms(mclahe_plan_t plan, const void* in, void* ws, void* stream) {
  MG_PLAN_INIT(plan);
  int rc = check_ptrs(plan, in, nullptr);
  if (rc) return rc;
  return do_hist(plan, in, ws, static_cast<cudaStream_t>(stream));
}

int mclahe_pass_mappings(mclahe_plan_t plan, void* ws, const mclahe_debug_t* debug, void* stream) {
  MG_PLAN_INIT(plan);
  return do_map(plan, ws, debug, static_cast<cudaStream_t>(stream));
}

int mclahe_pass_interpolate(mclahe_plan_t plan, const void* in, void* out, void* ws, void* stream) {
  MG_PLAN_INIT(plan);
  int rc = check_ptrs(plan, in, out);
  if (rc) return rc;
  if (!out) return fail(MCLAHE_ERR_VALIDATION, "null output buffer");
  return do_interp(plan, in, out, ws, static_cast<cudaStream_t>(stream));
}

int mclahe_plan_enqueue(mclahe_plan_t plan, const void* in, void* out, void* ws, void* stream) {
  MG_PLAN_INIT(plan);
  if (plan->info.row_begin != 0 || plan->info.row_end != plan->p.shape[0])
    return fail(MCLAHE_ERR_VALIDATION, "mclahe_plan_enqueue needs a whole-volume plan");
  int rc = check_ptrs(plan, in, out);
  if (rc) return rc;
  if (!out) return fail(MCLAHE_ERR_VALIDATION, "null output buffer");
  return enqueue_all(plan, in, out, ws, static_cast<cudaStream_t>(stream), nullptr);
}

int mclahe_plan_check(mclahe_plan_t plan, const void* ws, void* stream) {
  if (!plan) return fail(MCLAHE_ERR_VALIDATION, "null plan");
  return read_status(plan, ws, static_cast<cudaStream_t>(stream));
}

int mclahe_gpu_run_device(const mclahe_params_t* params, const void* in, void* out, void* stream,
                          mclahe_timings_t* timings) {
  NvtxRange nvtx("mclahe_gpu_run_device");
  int rc = validate(params);
  if (rc) return rc;
  OneShot& o = oneshot();
  std::lock_guard<std::mutex> lock(o.mu);
  mclahe_plan_s* pl = cached_plan(o, params, &rc);
  if (!pl) return rc;
  if ((rc = check_ptrs(pl, in, out))) return rc;
  if ((rc = ensure_buf(o, (size_t)pl->info.workspace_bytes))) return rc;
  if ((rc = ensure_stream(o))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((rc = enqueue_all(pl, in, out, o.buf, st, timings ? o.ev : nullptr))) return rc;
  if ((rc = read_status(pl, o.buf, st))) return rc;
  if (timings) {
    float a = 0, b = 0;
    MG_CUDA(cudaEventElapsedTime(&a, o.ev[0], o.ev[1]));
    MG_CUDA(cudaEventElapsedTime(&b, o.ev[1], o.ev[2]));
    timings->histograms_s += a * 1e-3;
    timings->interpolation_s += b * 1e-3;
  }
  return MCLAHE_OK;
}

namespace {

// Device bytes a one-shot call may use: `cap` when given, else what is free
// now plus the cached one-shot buffer (it is reallocated to fit), less a margin
// for the chunk plans' tables; MCLAHE_MAX_DEVICE_BYTES caps both.
int device_budget(const OneShot& o, int64_t cap, int64_t* budget) {
  size_t free_b = 0, total_b = 0;
  MG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  int64_t b = (int64_t)free_b + (int64_t)o.buf_bytes;
  b -= std::min<int64_t>(b / 16, int64_t{1} << 30);
  if (const char* e = getenv("MCLAHE_MAX_DEVICE_BYTES")) b = std::min<int64_t>(b, atoll(e));
  if (cap > 0) b = std::min(b, cap);
  *budget = b;
  return MCLAHE_OK;
}

int run_host(const mclahe_params_t* params, const void* in, void* out, int64_t max_device_bytes,
             mclahe_timings_t* timings) {
  int rc = validate(params);
  if (rc) return rc;
  if (!in || !out) return fail(MCLAHE_ERR_VALIDATION, "null host buffer");
  OneShot& o = oneshot();
  std::lock_guard<std::mutex> lock(o.mu);
  mclahe_plan_s* pl = cached_plan(o, params, &rc);
  if (!pl) return rc;
  const size_t bytes = (size_t)(volume(params) * elem_size(params));
  const size_t io = (size_t)align_up((int64_t)bytes, 256);
  int dev = 0;
  MG_CUDA(cudaGetDevice(&dev));
  mclahe_params_t q = *params;
  q.reserved = 0;
  for (int i = q.rank; i < MCLAHE_MAX_RANK; ++i) q.shape[i] = q.kernel[i] = 0;
  int64_t budget = 0;
  if ((rc = device_budget(o, max_device_bytes, &budget))) return rc;
  if ((int64_t)(2 * io) + pl->info.workspace_bytes > budget) {
    // out of core: the volume streams through a ring of chunk slots
    if (!pl->f32())
      return fail(MCLAHE_ERR_OOM, "float64 volume does not fit the device memory budget (the out-of-core ring takes float32 volumes)");
    std::string key = plan_key(&q, dev);
    key.append("ring");
    auto it = o.streamed.find(key);
    if (it != o.streamed.end() && it->second) {
      const Streamed& S = *it->second;
      const int64_t need = (S.in_slots + S.out_slots) * S.slot_bytes +
                           align_up(S.chunks[0]->info.workspace_bytes, 256);
      if (need > budget) {
        o.streamed.erase(it);
        it = o.streamed.end();
      }
    }
    if (it == o.streamed.end()) {
      std::unique_ptr<Streamed> S;
      if ((rc = build_ring(params, budget, S))) return rc;
      if (o.streamed.size() > 8) o.streamed.clear();
      it = o.streamed.emplace(key, std::move(S)).first;
    }
    Streamed& S = *it->second;
    const int64_t in_b = S.in_slots * S.slot_bytes, out_b = S.out_slots * S.slot_bytes;
    const size_t wsb = (size_t)S.chunks[0]->info.workspace_bytes;
    if (o.buf && (int64_t)o.buf_bytes > budget) {  // a larger cached buffer breaks the cap
      cudaFree(o.buf);
      o.buf = nullptr;
      o.buf_bytes = 0;
    }
    if ((rc = ensure_buf(o, (size_t)(in_b + out_b) + wsb))) return rc;
    if ((rc = ensure_stream(o))) return rc;
    char* base = static_cast<char*>(o.buf);
    return run_streamed(S, params, in, out, base, base + in_b, base + in_b + out_b, o.s_in, o.stream,
                        o.s_out, o.sev, timings);
  }
  // float32 volumes large enough to chunk: streamed H2D / compute / D2H
  if (pl->f32() && getenv("MCLAHE_NO_STREAM") == nullptr) {
    const std::string key = plan_key(&q, dev);
    auto it = o.streamed.find(key);
    if (it == o.streamed.end()) {
      auto S = std::make_unique<Streamed>();
      const int brc = build_streamed(params, *S);
      if (brc != MCLAHE_OK && brc != MCLAHE_ERR_UNSUPPORTED) return brc;
      if (brc == MCLAHE_ERR_UNSUPPORTED) S.reset();
      if (o.streamed.size() > 8) o.streamed.clear();
      it = o.streamed.emplace(key, std::move(S)).first;
    }
    if (it->second) {
      Streamed& S = *it->second;
      const size_t wsb = (size_t)S.chunks[0]->info.workspace_bytes;
      if ((rc = ensure_buf(o, 2 * io + wsb))) return rc;
      if ((rc = ensure_stream(o))) return rc;
      char* base = static_cast<char*>(o.buf);
      return run_streamed(S, params, in, out, base, base + io, base + 2 * io, o.s_in, o.stream,
                          o.s_out, o.sev, timings);
    }
  }
  return run_plan_host(o, pl, in, out, bytes, io, timings);
}

}  // namespace

int mclahe_gpu_run(const mclahe_params_t* params, const void* in, void* out,
                   mclahe_timings_t* timings) {
  NvtxRange nvtx("mclahe_gpu_run");
  return run_host(params, in, out, 0, timings);
}

int mclahe_gpu_run_out_of_core(const mclahe_params_t* params, const void* in, void* out,
                               int64_t max_device_bytes, mclahe_timings_t* timings) {
  NvtxRange nvtx("mclahe_gpu_run_out_of_core");
  if (max_device_bytes <= 0) return fail(MCLAHE_ERR_VALIDATION, "max_device_bytes must be positive");
  return run_host(params, in, out, max_device_bytes, timings);
}

int mclahe_gpu_run_framewise(const mclahe_params_t* params, int32_t frame_axis, const void* in,
                             void* out, mclahe_timings_t* timings) {
  NvtxRange nvtx("mclahe_gpu_run_framewise");
  if (!params) return fail(MCLAHE_ERR_VALIDATION, "null params");
  const int D = params->rank;
  if (D < 2) return fail(MCLAHE_ERR_VALIDATION, "framewise mode needs rank >= 2");
  if (frame_axis < 0 || frame_axis >= D)
    return fail(MCLAHE_ERR_VALIDATION, "frame axis " + std::to_string(frame_axis) +
                                           " out of range for rank " + std::to_string(D));
  // the slice request first, so messages match the reference's per-slice checks
  mclahe_params_t sl = *params;
  sl.rank = D - 1;
  for (int j = 0, k = 0; j < D; ++j)
    if (j != frame_axis) sl.shape[k++] = params->shape[j];
  for (int j = D - 1; j < MCLAHE_MAX_RANK; ++j) sl.shape[j] = sl.kernel[j] = 0;
  int rc = validate(&sl);
  if (rc) return rc;
  if (!in || !out) return fail(MCLAHE_ERR_VALIDATION, "null host buffer");
  // the volume with kernel 1 along the frame axis: each tile is one frame
  // thick and the blend weight across frames is exactly 0 / 1
  mclahe_params_t q = *params;
  for (int j = 0, k = 0; j < D; ++j) q.kernel[j] = j == frame_axis ? 1 : params->kernel[k++];
  if (params->adaptive) return mclahe_gpu_run(&q, in, out, timings);
  q.adaptive = 1;  // per-tile parameters, each tile's range = its frame's global range
  OneShot& o = oneshot();
  std::lock_guard<std::mutex> lock(o.mu);
  mclahe_plan_s* pl = cached_plan(o, &q, &rc, frame_axis);
  if (!pl) return rc;
  const size_t bytes = (size_t)(volume(&q) * elem_size(&q));
  return run_plan_host(o, pl, in, out, bytes, (size_t)align_up((int64_t)bytes, 256), timings);
}

int mclahe_validate(const mclahe_params_t* params) { return validate(params); }

void* mclahe_host_alloc(size_t bytes) {
  void* p = nullptr;
  const cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cuda_fail(e, "cudaHostAlloc");
    return nullptr;
  }
  return p;
}

void mclahe_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int mclahe_multi_cuts(const mclahe_params_t* params, int32_t n_slabs, int64_t* cuts) {
  int rc = validate(params);
  if (rc) return rc;
  if (!cuts) return fail(MCLAHE_ERR_VALIDATION, "null cuts");
  std::vector<int64_t> c;
  if ((rc = multi_cuts(params, n_slabs, c))) return rc;
  std::copy(c.begin(), c.end(), cuts);
  return MCLAHE_OK;
}

int mclahe_gpu_run_multi(const mclahe_params_t* params, int32_t n_slabs, const int32_t* devices,
                         const void* host_in, void* host_out, mclahe_timings_t* timings) {
  NvtxRange nvtx("mclahe_gpu_run_multi");
  if (!host_in || !host_out) return fail(MCLAHE_ERR_VALIDATION, "null host buffer");
  std::lock_guard<std::mutex> lock(g_multi_mu);
  int cur = 0;
  MG_CUDA(cudaGetDevice(&cur));
  Multi* M = nullptr;
  int rc = multi_get(params, n_slabs, devices, &M);
  if (!rc) rc = run_multi(*M, params, host_in, host_out, nullptr, nullptr, timings);
  cudaSetDevice(cur);
  return rc;
}

int mclahe_gpu_run_multi_device(const mclahe_params_t* params, int32_t n_slabs,
                                const int32_t* devices, const void* const* in_dev,
                                void* const* out_dev, mclahe_timings_t* timings) {
  if (!in_dev || !out_dev) return fail(MCLAHE_ERR_VALIDATION, "null device buffer list");
  for (int r = 0; r < n_slabs; ++r)
    if (!in_dev[r] || !out_dev[r] || !aligned16(in_dev[r]) || !aligned16(out_dev[r]))
      return fail(MCLAHE_ERR_VALIDATION, "slab buffers must be non-NULL and 16-byte aligned");
  std::lock_guard<std::mutex> lock(g_multi_mu);
  int cur = 0;
  MG_CUDA(cudaGetDevice(&cur));
  Multi* M = nullptr;
  int rc = multi_get(params, n_slabs, devices, &M);
  if (!rc) rc = run_multi(*M, params, nullptr, nullptr, in_dev, out_dev, timings);
  cudaSetDevice(cur);
  return rc;
}

int mclahe_debug_bin_index(int32_t dtype, const void* values, int64_t n, double lo, double hi,
                           int64_t n_bins, int32_t* out, void* stream) {
  if (n_bins < 2 || n_bins > 16384) return fail(MCLAHE_ERR_VALIDATION, "n_bins out of range");
  if (n <= 0) return MCLAHE_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 4096);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == MCLAHE_F32) {
    float* thr = nullptr;
    MG_CUDA(cudaMallocAsync(&thr, (size_t)(n_bins + 1) * sizeof(float), st));
    k_debug_thresholds<<<(int)((n_bins + 128) / 128), 128, 0, st>>>(lo, hi, (int)n_bins, thr);
    MG_LAUNCHED();
    k_debug_bins<float><<<grid, 256, 0, st>>>(static_cast<const float*>(values), n, lo, hi,
                                              (int)n_bins, thr, out);
    MG_LAUNCHED();
    MG_CUDA(cudaFreeAsync(thr, st));
  } else {
    k_debug_bins<double><<<grid, 256, 0, st>>>(static_cast<const double*>(values), n, lo, hi,
                                               (int)n_bins, nullptr, out);
    MG_LAUNCHED();
  }
  return MCLAHE_OK;
}

int32_t mclahe_plan_flags(mclahe_plan_t plan) {
  if (!plan) return 0;
  return (plan->fused_pencil ? 1 : 0) | (plan->hist.on ? 2 : 0) | (plan->interp.on ? 4 : 0) |
         (plan->dict_cap ? 8 : 0) | (plan->mdict ? 16 : 0);
}

int mclahe_plan_dict_state(mclahe_plan_t plan, const void* workspace, int32_t* state,
                           void* stream) {
  if (!plan || !state) return fail(MCLAHE_ERR_VALIDATION, "plan and state must be non-NULL");
  state[0] = state[1] = state[3] = 0;
  state[2] = plan->dict_cap;
  if (!plan->dict_cap) {  // global mode: the folded-pair blend runs whenever it is armed
    state[0] = plan->mdict ? 2 : 0;
    return MCLAHE_OK;
  }
  if (!workspace) return fail(MCLAHE_ERR_VALIDATION, "workspace must be non-NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t m[8];
  MG_CUDA(cudaMemcpyAsync(m, static_cast<const char*>(workspace) + plan->off_dict, sizeof m,
                          cudaMemcpyDeviceToHost, st));
  MG_CUDA(cudaStreamSynchronize(st));
  state[0] = m[2] ? (plan->mdict ? 2 : 1) : 0;
  state[1] = m[7];
  state[3] = m[2] ? m[4] : 0;
  return MCLAHE_OK;
}

int mclahe_debug_bin_index_packed(const float* values, int64_t n, double lo, double hi,
                                  int64_t n_bins, int32_t variant, int32_t* out, void* stream) {
  if (n_bins < 2 || n_bins > 16384) return fail(MCLAHE_ERR_VALIDATION, "n_bins out of range");
  if (variant < 1 || variant > 3) return fail(MCLAHE_ERR_VALIDATION, "variant must be 1, 2 or 3");
  if (n <= 0) return MCLAHE_OK;
  const int grid = (int)std::min<int64_t>((n / 2 + 256) / 256, 4096);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* thr = nullptr;
  MG_CUDA(cudaMallocAsync(&thr, (size_t)(2 * n_bins + 1) * sizeof(float), st));
  float* lut = thr + n_bins + 1;
  k_debug_thresholds<<<(int)((n_bins + 128) / 128), 128, 0, st>>>(lo, hi, (int)n_bins, thr);
  MG_LAUNCHED();
  k_debug_identity<<<(int)((n_bins + 127) / 128), 128, 0, st>>>(lut, (int)n_bins);
  MG_LAUNCHED();
  k_debug_bins_packed<<<grid, 256, 0, st>>>(values, n, lo, hi, (int)n_bins, thr, lut, variant,
                                            out);
  MG_LAUNCHED();
  MG_CUDA(cudaFreeAsync(thr, st));
  return MCLAHE_OK;
}

}  // extern "C"
