/*
 * gridshift_cuda.h -- C ABI of the B200-native MeanShift++ grid-shift engine
 * (libgridshift_cuda.so, sm_100a).
 *
 * Plain pointers and sizes only; no torch/numpy types cross this boundary.
 * Every entry point replaces one function of the reference's Python engine
 * interface (`/root/reference/pkg/src/gridshift/`), and a binding (ctypes,
 * cgo, JNI, ...) re-raises the status codes exactly as the reference does:
 *
 *   GS_OK            0  success
 *   GS_EINVAL        1  invalid input -> ValueError (message via gs_last_error)
 *   GS_ERUNTIME      2  CUDA / device failure -> RuntimeError
 *   GS_EUNSUPPORTED  3  valid input outside this engine's envelope
 *                       (d > 8, n >= 2^32, lattice >= 2^62 cells) -> ValueError
 *
 * Threading: a gs_ctx owns its device buffers and stream and serialises the
 * calls made on it; use one context per host thread for concurrency (the
 * reference's batch segmentation runs engines from a thread pool,
 * cli.py:206-216).  Device work runs without the caller holding any lock.
 *
 * Host-pointer entry points copy inputs host->device and results
 * device->host inside the call (pinned host buffers make those copies
 * full-speed).  The *_device / gs_shard_* variants take device pointers and
 * a cudaStream_t (as void*, NULL = legacy default stream) and leave results
 * on the device.
 */
#ifndef GRIDSHIFT_CUDA_H
#define GRIDSHIFT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GS_API __attribute__((visibility("default")))
#else
#define GS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define GS_OK 0
#define GS_EINVAL 1
#define GS_ERUNTIME 2
#define GS_EUNSUPPORTED 3

#define GS_DTYPE_F64 0
#define GS_DTYPE_F32 1

typedef struct gs_ctx gs_ctx;

/* Last error message of the calling thread ("" if none). */
GS_API const char* gs_last_error(void);

/* Library version string, e.g. "gridshift-b200 0.1 sm_100a". */
GS_API const char* gs_version(void);

/* Create / destroy an engine context bound to CUDA device `device`. */
GS_API int gs_ctx_create(int device, gs_ctx** out);
GS_API void gs_ctx_destroy(gs_ctx* ctx);

/*
 * Full MeanShift++ run: replaces gridshift.modeseek.meanshiftpp
 * (modeseek.py:125-146) as registered in ENGINES["meanshiftpp"]
 * (modeseek.py:288); the per-iteration step is modeseek.py:105-111 and the
 * labelling is _extract (modeseek.py:256-272).
 *
 *   x          (n, d) row-major points, float64 (PointSet.data, grid.py:43)
 *   h          bandwidth (ShiftConfig.h; must be finite > 0, grid.py:25-29)
 *   eta        absolute movement tolerance, already resolved
 *              (ShiftConfig.resolve_eta, modeseek.py:71-74); must be > 0
 *   max_iters  >= 1 (ShiftConfig.max_iters)
 * Outputs:
 *   labels_out     (n,) int64, dense in [0, k), numbered by first appearance
 *   k_out          number of clusters (modes are fetched with gs_fetch_modes)
 *   iters_out      iterations executed (ShiftTrace.iterations)
 *   movement_out   (max_iters,) float64; first *iters_out entries valid
 *                  (ShiftTrace.total_movement_per_iter)
 *   converged_out  1 if movement < eta was reached (ShiftTrace.converged)
 */
GS_API int gs_meanshiftpp(gs_ctx* ctx, const double* x, int64_t n, int32_t d, double h, double eta,
                   int32_t max_iters, int64_t* labels_out, int64_t* k_out, int32_t* iters_out,
                   double* movement_out, int32_t* converged_out);

/* Host input in float64 or float32 (GS_DTYPE_*): float32 rows are copied
 * as-is and upcast on device, exactly as PointSet upcasts on the host
 * (grid.py:43) -- half the host->device bytes for float32 data. */
GS_API int gs_meanshiftpp_host(gs_ctx* ctx, const void* x, int32_t dtype, int64_t n, int32_t d,
                               double h, double eta, int32_t max_iters, int64_t* labels_out,
                               int64_t* k_out, int32_t* iters_out, double* movement_out,
                               int32_t* converged_out);

/* Same engine on device-resident input (x_dev: (n,d) row-major, dtype
 * GS_DTYPE_F64 or GS_DTYPE_F32 -- f32 is upcast on device as PointSet
 * does on the host, grid.py:43).  labels_dev: (n,) int64 device buffer.
 * stream: the cudaStream_t to run on, taken literally (NULL = the legacy
 * default stream, e.g. torch's default stream).  Returns after the stream
 * work completed. */
GS_API int gs_meanshiftpp_device(gs_ctx* ctx, const void* x_dev, int32_t dtype, int64_t n, int32_t d,
                          double h, double eta, int32_t max_iters, int64_t* labels_dev,
                          int64_t* k_out, int32_t* iters_out, double* movement_out,
                          int32_t* converged_out, void* stream);

/* Segmentation front end fused into the engine: uint8 (height, width, 3)
 * pixels -> features image_to_features (segment.py:82-92; mode 0 = "rgb",
 * 1 = "rgbxy" with spatial factor `scale`) -> meanshiftpp.  Replaces
 * segment_image's feature build + ENGINES dispatch (segment.py:95-106). */
GS_API int gs_segment_image(gs_ctx* ctx, const uint8_t* pixels, int32_t height, int32_t width,
                     int32_t mode, double scale, double h, double eta, int32_t max_iters,
                     int64_t* labels_out, int64_t* k_out, int32_t* iters_out,
                     double* movement_out, int32_t* converged_out);

/* Context options.  GS_OPT_COLLAPSED (0/1, default 0): run iterations
 * t >= 1 of gs_meanshiftpp* in the collapsed-group formulation (SURVEY.md
 * 8f): after iteration 0 all points of a run of the spatial sort share one
 * position, so each iteration updates one position per run (the tables and
 * movement are the same exact integers; results are bit-identical).  The
 * per-point iterate is then not materialised after iteration 0. */
#define GS_OPT_COLLAPSED 1
/* GS_OPT_SUMS: how the per-cell coordinate sums (np.bincount, sequential in
 * fp64 in point order from 0.0, grid.py:186-187) are formed.  Neighbourhood
 * sums follow the reference's lexicographic offset order (grid.py:253-258)
 * in modes 0 and 2.
 *   2 (default) = sequential model: the reference's sequential sums without
 *     the point order -- a cell holding c copies of one value (every cell a
 *     single source cell moved into) gets the reference's sum bit for bit
 *     (closed form per binade); a cell that received several source cells
 *     folds them interleaved proportionally instead of in point order
 *     (O(sources), no sort); the first table (distinct input values) is the
 *     exact sum rounded once.  Cells, counts and labels equal the
 *     reference's; modes within 1e-9*h on every BASELINE configuration
 *     (measured: <= 2e-10*h).  Assumes the points of a
 *     mixed cell are well mixed in index order (shuffled rows); for large
 *     spatially sorted inputs use 0.
 *   0 = the reference's summation order, bit for bit: mixed cells are summed
 *     in point-index order (index-ordered point lists, radix sort for long
 *     cells); every iterate equals the reference's bitwise.
 *   1 = order-independent exact sums rounded once (the row-sharded
 *     multi-GPU runs always use these: their result does not depend on how
 *     points are split across ranks). */
#define GS_OPT_SUMS 2
#define GS_SUMS_REFERENCE 0
#define GS_SUMS_EXACT 1
#define GS_SUMS_SEQMODEL 2
GS_API int gs_ctx_set_option(gs_ctx* ctx, int32_t option, int64_t value);

/* Mean colours (k, 3) of the segments of the last gs_segment_image on this
 * context: SegmentMap.mean_colors as segment_map_from_labeling computes them
 * (segment.py:109-117: np.bincount sums of the uint8 colours per label /
 * counts).  The per-label sums are accumulated on the device as integers, so
 * the quotients equal the reference's bit for bit. */
GS_API int gs_fetch_mean_colors(gs_ctx* ctx, double* colors_out, int64_t cap_rows);

/* Modes (k, d) of the last run on this context (Labeling.modes). */
GS_API int gs_fetch_modes(gs_ctx* ctx, double* modes_out, int64_t cap_rows);

/* Per-iteration occupied-cell count and (cells, counts) fingerprint of the
 * last run (observability; pins per-iteration tables bit for bit). */
GS_API int gs_fetch_trace(gs_ctx* ctx, int64_t* k_per_iter, uint64_t* fp_per_iter, int32_t cap);

/* Bytes the shift kernel stored per iteration of the last per-point run (the
 * iterate is updated in place and bitwise-unchanged coordinate pairs are not
 * rewritten; reads are always 8*d bytes per point).  Roofline accounting. */
GS_API int gs_fetch_shift_bytes(gs_ctx* ctx, uint64_t* bytes_per_iter, int32_t cap);

/* Final iterate y_T of the last per-point gs_meanshiftpp* run, in ORIGINAL
 * point order, (n, d) row-major fp64 into host memory (modeseek.py:136-141:
 * the `y` the reference hands to _extract).  Test observability: with
 * GS_SUMS_REFERENCE it equals the reference's iterate bit for bit.  Not
 * available after a collapsed-mode run (the per-point iterate is not
 * materialised) -> GS_EINVAL. */
GS_API int gs_fetch_iterate(gs_ctx* ctx, double* y_out, int64_t n);

/* Reference-order sums of the last run (observability): per table (row 0 =
 * the first table, row t+1 = the table derived in iteration t) five
 * counters: segments folded in index order, of those the long ones taking
 * the global radix sort, their points, the longest segment, and the
 * single-source cells whose closed form was recomputed (not cached). */
GS_API int gs_fetch_refsum_stats(gs_ctx* ctx, uint32_t* out, int32_t rows);

/* Host<->device bytes of the last host entry point call (gs_meanshiftpp,
 * gs_meanshiftpp_host, gs_segment_image): the input upload, and the label
 * delivery -- either 8 bytes per point, or on the sorted dense path 4 bytes
 * per point (initial-cell index, copied while the loop runs) plus 4 bytes per
 * lattice cell (per-cell labels) -- plus the modes.  End-to-end accounting. */
GS_API int gs_fetch_transfer_bytes(gs_ctx* ctx, int64_t* h2d_bytes, int64_t* d2h_bytes);

/* Kernel accounting.  mode 1: enable per-launch CUDA-event timing (and
 * reset counters); mode 0: disable (and reset); mode 2: write the
 * accumulated device milliseconds and launch counts per kernel kind
 * (index -> name via gs_profile_kind) into ms_out / launches_out[cap]. */
GS_API int gs_profile(gs_ctx* ctx, int32_t mode, double* ms_out, int64_t* launches_out, int32_t cap);
GS_API const char* gs_profile_kind(int32_t kind);

/* One grid-mean update: replaces meanshiftpp_step (modeseek.py:114-122). */
GS_API int gs_shift_step(gs_ctx* ctx, const double* y, int64_t n, int32_t d, double h, double* y_out,
                  double* movement_out);

/* Occupied-cell tables of a point set: replaces build_cell_tables /
 * _tables_from_data (grid.py:179-196) and, when nbr_* are non-NULL, the
 * 3^d neighbour statistics _neighbor_stats_cells (grid.py:230-273).
 * Two-phase: call with cap=0 to get *k_out, then with cap >= k.
 * Rows are lexicographically sorted by cell (CellTables.cells order). */
GS_API int gs_build_tables(gs_ctx* ctx, const double* y, int64_t n, int32_t d, double h, int64_t cap,
                    int64_t* cells_out, int64_t* counts_out, double* sums_out,
                    int64_t* nbr_counts_out, double* nbr_sums_out, int64_t* k_out);

/* Cluster extraction of converged positions: replaces extract_clusters
 * (modeseek.py:275-285).  Modes via gs_fetch_modes. */
GS_API int gs_extract_clusters(gs_ctx* ctx, const double* y, int64_t n, int32_t d, double h,
                        int64_t* labels_out, int64_t* k_out);

/*
 * Window tracker over a resident frame sequence: replaces the per-frame
 * loop of track_sequence / track_frame (track.py:147-205) after
 * init_tracker (track.py:110-135) produced the bin set.
 *   frames      (T, H, W, 3) uint8, frame 0 is the init frame
 *   win         initial window (cx, cy) and extents (w, h_px)
 *   bins        (nb, 3) int64 colour cells of B (BinSet.bins)
 *   h           colour bandwidth; update_bins as in track_frame
 * Outputs per frame (row 0 = the init state): cx, cy, lost, match count,
 * and the number of bins of B after the frame; optionally (non-NULL) the
 * bin set of every row as a bitmap over the colour lattice [0, L)^3,
 * L = floor(255/h) + 1, code = (b0*L + b1)*L + b2, ceil(L^3/32) uint32
 * words per frame.
 */
GS_API int gs_track_sequence(gs_ctx* ctx, const uint8_t* frames, int32_t n_frames, int32_t height,
                      int32_t width, double cx, double cy, int32_t w, int32_t h_px,
                      const int64_t* bins, int32_t nb, double h, int32_t update_bins,
                      int32_t init_matches, double tol, int32_t max_iters, double* cx_out,
                      double* cy_out, int32_t* lost_out, int64_t* matches_out,
                      int64_t* nbins_out, uint32_t* bitmap_hist_out);

/* Bin set B after the last gs_track_sequence frame (two-phase like
 * gs_build_tables). */
GS_API int gs_fetch_track_bins(gs_ctx* ctx, int64_t* bins_out, int32_t cap, int32_t* nb_out);

/*
 * Row-sharded run (one process per GPU; cfg4-style strong scaling).  The
 * caller owns the collectives (e.g. NCCL through torch.distributed) and
 * drives:
 *   gs_shard_init        local input -> per-axis cell range / max|x| / flags
 *   (all-reduce MIN cmin, MAX cmax, MAX absmax, OR flags)
 *   gs_shard_plan        global plan; local spatial sort; local first table
 *   gs_shard_table_io    export (0) / import (1) the table words (int64)
 *   (all-reduce SUM of the table words: exact integer merge)
 *   per iteration t:     gs_shard_iterate -> (all-reduce SUM of 4 int64
 *                        limbs) -> gs_shard_converge; gs_shard_status between
 *                        chunks
 *   gs_shard_components  local first-appearance minima per component root
 *   (all-reduce MIN of the int64 minima, slots entries)
 *   gs_shard_finish      labels of the local rows (global first-appearance
 *                        numbering), k, trace; modes via gs_fetch_modes.
 * Every rank derives identical tables, so no per-iteration table exchange is
 * needed.  Same reference semantics as gs_meanshiftpp (modeseek.py:125-146).
 */
GS_API int gs_shard_init(gs_ctx* ctx, const void* x_dev, int32_t dtype, int64_t n_local, int32_t d,
                         double h, void* stream, int64_t* cmin_out, int64_t* cmax_out,
                         double* absmax_out, int32_t* flags_out);
GS_API int gs_shard_plan(gs_ctx* ctx, const int64_t* cmin, const int64_t* cmax, const double* absmax,
                         int32_t flags, int64_t n_total, int32_t max_iters, void* stream,
                         int64_t* table_words_out);
GS_API int gs_shard_table_io(gs_ctx* ctx, void* buf_dev, int32_t to_device_table, void* stream);
GS_API int gs_shard_iterate(gs_ctx* ctx, int32_t t, void* limbs_dev, void* stream);
GS_API int gs_shard_converge(gs_ctx* ctx, int32_t t, const void* limbs_dev, double eta, void* stream);
GS_API int gs_shard_status(gs_ctx* ctx, int32_t* done_out, int32_t* iters_out, void* stream);
GS_API int gs_shard_components(gs_ctx* ctx, int64_t global_offset, void* minima_dev, void* stream,
                               int64_t* slots_out);
GS_API int gs_shard_finish(gs_ctx* ctx, const void* minima_dev, int64_t* labels_dev, void* stream,
                           int64_t* k_out, int32_t* iters_out, double* movement_out,
                           int32_t* converged_out);

#ifdef __cplusplus
}
#endif

#endif /* GRIDSHIFT_CUDA_H */
