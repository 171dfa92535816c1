/*
 * include/mclahe_gpu.h -- C ABI of the B200-native MCLAHE hot path.
 *
 * Plain pointers and sizes only (no C++/torch types), so it binds from C++,
 * ctypes, cgo or JNI alike.  Every entry point cites the reference interface
 * it replaces (paths relative to /root/reference/proj/core/).
 *
 * Status codes: MCLAHE_OK (0), MCLAHE_ERR_VALIDATION (1; message = the
 * reference ValidationError text), MCLAHE_ERR_CUDA (2), MCLAHE_ERR_COMM (3),
 * MCLAHE_ERR_OOM (4), MCLAHE_ERR_UNSUPPORTED (5).  No function throws across
 * the ABI; mclahe_last_error() returns the message of the calling thread's
 * last failure.
 *
 * Two ways in:
 *   1. mclahe_gpu_run()        one-shot, HOST buffers: the drop-in for
 *                              mclahe::mclahe (include/mclahe/pipeline.hpp:30).
 *   2. mclahe_plan_* + passes  device-resident, stream-ordered, caller-owned
 *                              workspace; the slab (multi-GPU) layer inserts
 *                              its collectives between the passes.
 */
#ifndef MCLAHE_GPU_H
#define MCLAHE_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCLAHE_MAX_RANK 8

enum {
  MCLAHE_OK = 0,
  MCLAHE_ERR_VALIDATION = 1,
  MCLAHE_ERR_CUDA = 2,
  MCLAHE_ERR_COMM = 3,
  MCLAHE_ERR_OOM = 4,
  MCLAHE_ERR_UNSUPPORTED = 5
};

enum { MCLAHE_F32 = 0, MCLAHE_F64 = 1 };

/* McLaheRequest (include/mclahe/pipeline.hpp:12-17) + EnhanceParams
 * (include/mclahe/histogram.hpp:17-21) flattened to POD.  `adaptive` is
 * RangeMode (histogram.hpp:13): 0 = Global, 1 = Adaptive.  `dtype` is the
 * element type of both the input and the output buffer. */
typedef struct {
  int32_t rank;
  int32_t adaptive;
  int32_t dtype;
  int32_t reserved;
  int64_t shape[MCLAHE_MAX_RANK];
  int64_t kernel[MCLAHE_MAX_RANK];
  int64_t n_bins;
  double clip_limit;
} mclahe_params_t;

/* PhaseTimings (include/mclahe/pipeline.hpp:20-24), filled from CUDA events:
 * pad = 0 (padding is virtual), histograms = range + counts + mappings,
 * interpolation = blend.  Accumulates (+=) like the reference. */
typedef struct {
  double pad_s;
  double histograms_s;
  double interpolation_s;
} mclahe_timings_t;

/* Geometry and workspace layout of a plan, for the slab exchange layer. */
typedef struct {
  int32_t rank;
  int32_t fast_hist;      /* 1 if the pencil histogram kernel is used */
  int32_t fast_interp;    /* 1 if the pencil interpolation kernel is used */
  int32_t trailing_dims;  /* k: trailing dims covered by one pencil */
  int64_t before[MCLAHE_MAX_RANK];
  int64_t after[MCLAHE_MAX_RANK];
  int64_t grid[MCLAHE_MAX_RANK];
  int64_t tiles;          /* all tiles of the full volume */
  int64_t row_begin, row_end;           /* slab rows along dim 0 (original) */
  int64_t tile_row_begin, tile_row_end; /* tile-row window held in workspace */
  int64_t count_row_begin, count_row_end; /* tile rows this slab counts into */
  int64_t need_row_begin, need_row_end;   /* tile rows the slab's voxels blend */
  int64_t tiles_per_row;  /* prod_{j>=1} grid[j] */
  int64_t n_bins;
  /* workspace byte offsets */
  int64_t off_range;      /* int64[4]: ~key(lo), key(hi), nonfinite, blend unit counter (MAX-reducible) */
  int64_t off_tile_range; /* int64[window tiles][2]: ~key(lo), key(hi)   (MAX-reducible) */
  int64_t off_counts;     /* int32[window tiles][n_bins]                 (SUM-reducible) */
  int64_t off_tparams;    /* per-tile binning parameters */
  int64_t off_lut;        /* float32[window tiles][n_bins] */
  int64_t off_thr;        /* float32[adaptive ? window tiles : 1][n_bins] bin-edge tables */
  int64_t workspace_bytes;
  int64_t hist_units, interp_units;
} mclahe_plan_info_t;

typedef struct mclahe_plan_s* mclahe_plan_t;

/* Optional per-tile intermediates (device pointers, any may be NULL), tile
 * index = window tile (tile-row window of the plan).  Mirrors what
 * build_mappings (src/histogram.cpp:72-106) produces per KernelMapping plus
 * the compute_histogram / clip_histogram arrays. */
typedef struct {
  double* lo;            /* [tiles]  IntensityRange.lo */
  double* hi;            /* [tiles]  IntensityRange.hi */
  uint32_t* counts;      /* [tiles][n_bins] raw counts (compute_histogram) */
  double* clipped;       /* [tiles][n_bins] clip_histogram output */
  double* lut;           /* [tiles][n_bins] normalized_cdf values (f64) */
  uint8_t* degenerate;   /* [tiles]  KernelMapping.degenerate */
} mclahe_debug_t;

/* ---- one-shot drop-in ------------------------------------------------- */

/* Replaces mclahe::mclahe(const McLaheRequest&, PhaseTimings*)
 * (include/mclahe/pipeline.hpp:30, src/pipeline.cpp:73-129).  `in` and `out`
 * are HOST buffers of prod(shape) elements of `dtype`; validation
 * (src/pipeline.cpp:19-34) happens first, with the reference messages.
 * Pinned host buffers are copied asynchronously; pageable ones through the
 * driver's staging path.  timings may be NULL.
 * On MCLAHE_ERR_VALIDATION for non-finite input `out` holds no result: in
 * global mode it is never written (the flag is read after the range pass,
 * before any blend); in adaptive mode the streamed call has already copied
 * early chunks back, so it fills `out` with NaN before returning. */
int mclahe_gpu_run(const mclahe_params_t* params, const void* in, void* out,
                   mclahe_timings_t* timings);

/* Out of core (src/pipeline.cpp:73-129 has no size limit beyond host memory;
 * PAPER.md:216 names larger-than-memory volumes as future work).  When the
 * volume, its result and the workspace do not fit the device memory that is
 * free (or MCLAHE_MAX_DEVICE_BYTES), mclahe_gpu_run streams float32 volumes
 * through a ring of chunk slots along dim 0 instead of full-size device
 * buffers: a chunk stays resident until the tile rows its voxels blend from are
 * complete (about 1.5 interpolation cells of rows later), then its slot takes
 * the next chunk.  Adaptive mode reads the host volume once; global mode
 * twice (the range needs every voxel before any bin exists).  Results are
 * bit-identical to the in-core call.  This entry point is the same call with an
 * explicit device-memory cap (bytes, > 0); MCLAHE_ERR_OOM if even the smallest
 * ring (about 2.5 cells of dim-0 rows plus the workspace) does not fit. */
int mclahe_gpu_run_out_of_core(const mclahe_params_t* params, const void* in, void* out,
                               int64_t max_device_bytes, mclahe_timings_t* timings);

/* Same, with DEVICE buffers on `stream` (cudaStream_t; NULL = legacy).  The
 * library allocates (and caches) its workspace.  Synchronises `stream` before
 * returning so the non-finite check can be reported. */
int mclahe_gpu_run_device(const mclahe_params_t* params, const void* in_dev, void* out_dev,
                          void* stream, mclahe_timings_t* timings);

/* ---- plans and passes (device-resident) --------------------------------- */

/* Plans one slab: original rows [row_begin, row_end) along dim 0 of the
 * volume described by params (the whole volume: 0, shape[0]).  The input and
 * output buffers given to the passes hold exactly those rows.  Validates
 * like src/pipeline.cpp:19-33 (the non-finite check runs on the device). */
int mclahe_plan_create(const mclahe_params_t* params, int64_t row_begin, int64_t row_end,
                       mclahe_plan_t* plan);
int mclahe_plan_destroy(mclahe_plan_t plan);
int mclahe_plan_get_info(mclahe_plan_t plan, mclahe_plan_info_t* info);

/* Resets the workspace (ranges, counts) -- first pass of every run. */
int mclahe_pass_reset(mclahe_plan_t plan, void* workspace, void* stream);

/* Pass 1.  Global mode: min/max + finiteness of the slab
 * (NdImage::min_max / all_finite, src/nd_image.cpp:70-83).  Adaptive mode:
 * per-tile min/max over the padded tiles this slab touches
 * (src/histogram.cpp:86-94).  Results land MAX-reducible at off_range /
 * off_tile_range for the exchange layer. */
int mclahe_pass_range(mclahe_plan_t plan, const void* in_dev, void* workspace, void* stream);

/* Turns the (exchanged) ranges into per-tile binning parameters. */
int mclahe_pass_params(mclahe_plan_t plan, void* workspace, void* stream);

/* Pass 2.  Per-tile counts over the virtually padded kernel grid
 * (kernelize + compute_histogram + bin_index, src/nd_image.cpp:146-187,
 * src/histogram.cpp:24-40).  Partial (SUM-reducible) for slabs. */
int mclahe_pass_histograms(mclahe_plan_t plan, const void* in_dev, void* workspace,
                           void* stream);

/* Pass 3.  clip_histogram + normalized_cdf per tile (src/histogram.cpp:42-70),
 * bit-exact f64, LUT stored as f32.  debug may be NULL. */
int mclahe_pass_mappings(mclahe_plan_t plan, void* workspace, const mclahe_debug_t* debug,
                         void* stream);

/* Pass 4.  Per-voxel multilinear blend of the 2^D neighbour LUTs
 * (src/pipeline.cpp:94-127, src/interpolation.cpp:7-86).  Writes nothing if
 * pass 1 saw a non-finite value. */
int mclahe_pass_interpolate(mclahe_plan_t plan, const void* in_dev, void* out_dev,
                            void* workspace, void* stream);

/* All passes for a single-slab plan, stream-ordered, no host sync. */
int mclahe_plan_enqueue(mclahe_plan_t plan, const void* in_dev, void* out_dev,
                        void* workspace, void* stream);

/* Synchronises `stream` and reports MCLAHE_ERR_VALIDATION ("image contains
 * non-finite values") if pass 1 flagged the input. */
int mclahe_plan_check(mclahe_plan_t plan, const void* workspace, void* stream);

/* Exact bin_index (src/histogram.cpp:24-32) of n device values through the
 * same fast-guarded routine the kernels use; out is int32[n].  For testing
 * the binning on adversarial values. */
int mclahe_debug_bin_index(int32_t dtype, const void* values_dev, int64_t n, double lo,
                           double hi, int64_t n_bins, int32_t* out_dev, void* stream);

/* Value-dictionary state after a run on `workspace` (synchronises `stream`):
 * state[0] = 1 if the last blend used the dictionary path, 2 if it used the
 * folded-pair blend k_interp_mdict (adaptive: with the dictionary; global
 * mode, capacity 0: always when the plan arms it), 0 otherwise, state[1] = number
 * of distinct values collected, state[2] = the plan's capacity (0: never),
 * state[3] = 1 if values were looked up through the affine direct table
 * (0: cuckoo hash).  state has 4 entries. */
int mclahe_plan_dict_state(mclahe_plan_t plan, const void* workspace, int32_t* state,
                           void* stream);

/* Which kernels a plan runs (bit mask, after the plan's first pass on a
 * device): 1 = fused pencil K2 (tile ranges and counts in one kernel, one read
 * of the input from HBM; k_fused.cu), 2 = pencil histogram kernel, 4 = pencil
 * blend, 8 = value dictionary armed, 16 = folded-pair blend armed. */
int32_t mclahe_plan_flags(mclahe_plan_t plan);

/* The pencil kernels' packed f32x2 binning on n device float32 values (pairs
 * of consecutive values): variant 1 = the histogram routine, 2 = the blend
 * gather (through an identity LUT), 3 = the bracketed floors of the
 * n_bins-specialised adaptive blend.  Must equal mclahe_debug_bin_index. */
int mclahe_debug_bin_index_packed(const float* values_dev, int64_t n, double lo, double hi,
                                  int64_t n_bins, int32_t variant, int32_t* out_dev,
                                  void* stream);

/* Batched mclahe_framewise (src/pipeline.cpp:131-153, renormalize_slices =
 * false): every slice along frame_axis enhanced on its own, in one run.
 * params->shape / rank describe the whole volume; params->kernel holds the
 * rank-1 slice kernel (the frame axis removed), as in the reference.  The
 * frames run as one volume with kernel 1 along the frame axis (tiles one
 * frame thick, blend weight across frames exactly 0/1); in global mode each
 * tile takes its frame's own min/max.  Host buffers, like mclahe_gpu_run. */
int mclahe_gpu_run_framewise(const mclahe_params_t* params, int32_t frame_axis,
                             const void* host_in, void* host_out, mclahe_timings_t* timings);

/* ---- The steps either side of the path, float64 ----
 * gaussian_filter (src/filters.cpp:82-96): separable, per-axis sigma (0 skips
 *   the axis), radius ceil(truncate * sigma), mirror boundary; bit-identical
 *   to the reference (taps from the host libm, unfused sequential sums).
 * median_filter (src/filters.cpp:98-142): window extents per dimension
 *   (offsets -floor((w-1)/2) .. floor(w/2)), mirror boundary, even windows take
 *   the mean of the two central values; at most 343 values per window here.
 * metrics (src/metrics.cpp:11-72): mse and psnr of (a, b) (b may be NULL:
 *   both 0), population standard deviation of a, Shannon entropy of a over
 *   [min, max] in n_bins bins (exact counts; sum in bin order on the host).
 * *_device forms take device buffers and synchronise `stream`; the plain forms
 * take host buffers. */
typedef struct {
  double mse;
  double psnr_db;
  double std;
  double entropy_bits;
  int64_t n_bins_used;
} mclahe_metrics_t;

int mclahe_gaussian_filter(int32_t rank, const int64_t* shape, const double* sigmas,
                           double truncate, const double* host_in, double* host_out);
int mclahe_gaussian_filter_device(int32_t rank, const int64_t* shape, const double* sigmas,
                                  double truncate, const double* in_dev, double* out_dev,
                                  void* stream);
int mclahe_median_filter(int32_t rank, const int64_t* shape, const int64_t* window,
                         const double* host_in, double* host_out);
int mclahe_median_filter_device(int32_t rank, const int64_t* shape, const int64_t* window,
                                const double* in_dev, double* out_dev, void* stream);
int mclahe_metrics(int32_t rank, const int64_t* shape, const double* host_a,
                   const double* host_b, int64_t n_bins, double peak, mclahe_metrics_t* report);
int mclahe_metrics_device(int32_t rank, const int64_t* shape, const double* a_dev,
                          const double* b_dev, int64_t n_bins, double peak,
                          mclahe_metrics_t* report, void* stream);

/* ---- Multi-slab / multi-device --------------------------
 * The volume is cut along dim 0 at interpolation-cell boundaries into
 * n_slabs row-balanced slabs (mclahe_multi_cuts: n_slabs + 1 row
 * boundaries); slab r runs on devices[r] with its own plan, stream and
 * buffers.  Devices may repeat: logical slabs on one GPU take the identical
 * code path (the 1-GPU test of the exchange).  Cross-slab traffic: the range
 * keys (MAX over all slabs), the per-tile range keys of shared tile rows
 * (adaptive, MAX with the neighbours) and the partial integer counts of
 * shared tile rows (SUM with the neighbours) -- read by a combine kernel
 * straight from the peers' snapshot buffers over NVLink / NVSwitch (P2P), or
 * staged by cudaMemcpyPeerAsync where P2P is unavailable.  Integer combines
 * are order-free: results are bit-identical to mclahe_gpu_run for any slab
 * count and device list (the reference's worker-count promise,
 * include/mclahe/pipeline.hpp:10-11, parallel.hpp:19-22).
 * mclahe_gpu_run_multi: whole-volume HOST buffers.
 * mclahe_gpu_run_multi_device: per-slab DEVICE buffers (slab r's rows
 * [cuts[r], cuts[r+1]) resident on devices[r]). */
int mclahe_multi_cuts(const mclahe_params_t* params, int32_t n_slabs, int64_t* cuts);
int mclahe_gpu_run_multi(const mclahe_params_t* params, int32_t n_slabs, const int32_t* devices,
                         const void* host_in, void* host_out, mclahe_timings_t* timings);
int mclahe_gpu_run_multi_device(const mclahe_params_t* params, int32_t n_slabs,
                                const int32_t* devices, const void* const* in_dev,
                                void* const* out_dev, mclahe_timings_t* timings);

/* ---- The reference's per-operation API on the device (csrc/ops.cu) -------
 * For callers of include/mclahe/{histogram,nd_image}.hpp that use the
 * building blocks instead of mclahe::mclahe.  Host buffers, float64.
 *
 * mclahe_block_mappings: build_mappings (src/histogram.cpp:72-106) over
 *   n_blocks contiguous blocks of block_len values (KernelGrid::blocks):
 *   adaptive = each block's own min/max (first of the minimal class, NaN
 *   never wins unless it is the block's front element), else
 *   [global_lo, global_hi]; lo / hi / counts (compute_histogram) / clipped
 *   (clip_histogram) / lut (normalized_cdf values or 0.5) / degenerate per
 *   block, bit-identical to the reference.  Any output may be NULL, except
 *   that lut and degenerate go together; lut == NULL skips clip / CDF (the
 *   compute_histogram form).
 * mclahe_nd_gather: op 0 = symmetric_pad (a = before, b = after,
 *   src/nd_image.cpp:104-144), op 1 = kernelize (a = kernel sizes, b unused,
 *   :146-187), op 2 = crop (a = offset, b = out shape, :189-218). */
int mclahe_block_mappings(const double* host_blocks, int64_t n_blocks, int64_t block_len,
                          int64_t n_bins, double clip_limit, int32_t adaptive, double global_lo,
                          double global_hi, double* lo, double* hi, double* counts,
                          double* clipped, double* lut, uint8_t* degenerate);
int mclahe_nd_gather(int32_t op, int32_t rank, const int64_t* in_shape, const int64_t* a,
                     const int64_t* b, const double* host_in, double* host_out);

/* The request checks of validate_request (src/pipeline.cpp:19-33, minus the
 * finiteness scan that runs on the device), on the host only: no CUDA call,
 * so a caller can reject a bad request before staging any data. */
int mclahe_validate(const mclahe_params_t* params);

/* Page-locked host memory (cudaHostAlloc, portable): buffers from here make
 * the host-buffer calls copy at full PCIe rate and overlap H2D / compute /
 * D2H; the C++ drop-in stages its float64 <-> float32 conversions in them.
 * NULL on failure (mclahe_last_error() says why). */
void* mclahe_host_alloc(size_t bytes);
void mclahe_host_free(void* p);

/* Number of kernel launches the last pass call on this thread issued. */
int64_t mclahe_launch_count(void);

const char* mclahe_last_error(void);
const char* mclahe_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MCLAHE_GPU_H */
