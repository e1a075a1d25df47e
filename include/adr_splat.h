/*
 * adr_splat.h — C ABI of the B200 AdR-Gaussian forward rasterizer
 * (libadrsplat.so, sm_100a).
 *
 * The reference (splatbench 0.1.0, /root/reference/pkg/src/splatbench/) is a
 * pure-Python package with no FFI.  These entry points are what its Python
 * stage functions bind to (see INTEGRATION.md for the ctypes stubs); each
 * cites the reference function it replaces.  Conventions:
 *
 *  - every pointer named d_* is DEVICE memory owned by the caller; h_* is host;
 *  - every call is asynchronous on `stream` (a cudaStream_t passed as void*),
 *    except the ones documented as synchronising;
 *  - scratch memory is caller-provided: call the matching *_scratch_bytes()
 *    first (cub-style two-phase API); the library never allocates device
 *    memory itself;
 *  - return value is an adr_status; adr_last_error() gives the message.
 *    ADR_ERR_VALUE maps to ValueError, ADR_ERR_CAPACITY to CapacityError,
 *    ADR_ERR_INTERNAL to InternalError (sb/errors.py:4-17).
 */
#ifndef ADR_SPLAT_H
#define ADR_SPLAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADR_ABI_VERSION 3

typedef enum {
    ADR_OK = 0,
    ADR_ERR_VALUE = 1,     /* bad argument            -> ValueError    */
    ADR_ERR_CAPACITY = 2,  /* key / index overflow    -> CapacityError */
    ADR_ERR_INTERNAL = 3,  /* invariant violated      -> InternalError */
    ADR_ERR_CUDA = 4       /* CUDA runtime failure    -> RuntimeError  */
} adr_status;

/* CullingMode (sb/projection.py:46-49). */
typedef enum { ADR_MODE_BASELINE = 0, ADR_MODE_CIRCLE = 1, ADR_MODE_AABB = 2 } adr_mode;

/* Scene storage dtype. Math is fp64 either way (bit-exact with the reference
 * when the stored values are the reference's values). */
typedef enum { ADR_F32 = 0, ADR_F64 = 1 } adr_dtype;

/* Camera constants, computed on the host with the reference's own
 * expressions (sb/projection.py:341-355, sb/scene.py:147-158). */
typedef struct {
    double rot[9];        /* world->camera rotation, row-major */
    double trans[3];
    double center[3];     /* -R^T t */
    double fx, fy;
    double lim_x, lim_y;  /* FOV_CLAMP_FACTOR * (0.5 * W / f) */
    double cx, cy;        /* 0.5 * (W - 1), 0.5 * (H - 1) */
    double near_plane;
    float background[3];
    int32_t width, height;
} adr_camera;

/* Scene arrays (SceneArrays, sb/scene.py:105-110), device, row-major:
 * centers (N,3), scales (N,3), rotations (N,4) wxyz, opacities (N,),
 * sh (N,K,3) with K = (sh_degree+1)^2. */
typedef struct {
    const void* d_centers;
    const void* d_scales;
    const void* d_rotations;
    const void* d_opacities;
    const void* d_sh;
    int64_t n;
    int32_t sh_degree;
    int32_t dtype;        /* adr_dtype */
} adr_scene;

/* Projection (sb/projection.py:86-112), device, index-aligned with the scene. */
typedef struct {
    uint8_t* d_valid;       /* (N,)   bool  */
    float* d_mean2d;        /* (N,2)        */
    float* d_cov2d;         /* (N,3)  sxx, syy, sxy */
    float* d_conic;         /* (N,3)  a, b, c       */
    float* d_depth;         /* (N,)         */
    float* d_color;         /* (N,3)        */
    float* d_opacity;       /* (N,)         */
    float* d_lambda_max;    /* (N,)         */
    int32_t* d_ext_x;       /* (N,)         */
    int32_t* d_ext_y;       /* (N,)         */
} adr_projection;

/* ---------------------------------------------------------------- utils */
int32_t adr_abi_version(void);
const char* adr_last_error(void);
/* Running total of kernels this library has launched (all entry points). */
int64_t adr_kernel_launches(void);
/* Number of SMs of the current device (for diagnostics). */
int32_t adr_device_sm_count(void);

/* ------------------------------------------------------- stage functions */

/* Stage 1 — preprocess (sb/projection.py:291-420). Writes every Projection
 * field; rows that do not survive are zeroed (valid = 0). */
int32_t adr_preprocess(const adr_scene* scene, const adr_camera* cam, int32_t mode,
                       double alpha_low, double dilation, const adr_projection* out,
                       void* stream);

/* Stage 2a — touched-tile counts (sb/tiling.py:111-114, rects :77-99). */
int32_t adr_touched_counts(const adr_projection* proj, int64_t n, int32_t tiles_x,
                           int32_t tiles_y, int64_t* d_counts, void* stream);

/* Stage 2b — inclusive sum (sb/tiling.py:117-122), int64.  The overflow
 * check of the reference becomes a device flag: *d_overflow is set to 1 when
 * the running sum exceeds INT64_MAX (caller maps it to CapacityError). */
size_t adr_inclusive_sum_scratch_bytes(int64_t n);
int32_t adr_inclusive_sum(const int64_t* d_counts, int64_t n, int64_t* d_offsets,
                          int32_t* d_overflow, void* d_scratch, size_t scratch_bytes,
                          void* stream);

/* Stage 3 — duplicate with keys (sb/tiling.py:125-156): entries of Gaussian g
 * fill [offsets[g]-count, offsets[g]) row-major over its tile rectangle,
 * key = tile << 32 | float32 depth bits, gidx = g. */
int32_t adr_duplicate_with_keys(const adr_projection* proj, int64_t n,
                                const int64_t* d_offsets, int32_t tiles_x, int32_t tiles_y,
                                uint64_t* d_keys, int64_t* d_gidx, void* stream);

/* Stage 4 — stable ascending sort by key (sb/tiling.py:159-164): LSD radix
 * sort over bits [0, end_bit) (end_bit <= 64; pass 64 for arbitrary keys).
 * Inputs are not modified. */
size_t adr_sort_pairs_scratch_bytes(int64_t p);
int32_t adr_sort_pairs(const uint64_t* d_keys, const int64_t* d_gidx, int64_t p,
                       int32_t end_bit, uint64_t* d_keys_out, int64_t* d_gidx_out,
                       void* d_scratch, size_t scratch_bytes, void* stream);

/* Stage 5 — tile ranges (sb/tiling.py:167-177): ranges (n_tiles,2) int64,
 * empty tiles (k,k).  *d_error gets 1 if keys are unsorted, 2 if a key
 * references a tile >= n_tiles (caller maps both to InternalError). */
int32_t adr_identify_tile_ranges(const uint64_t* d_sorted_keys, int64_t p, int64_t n_tiles,
                                 int64_t* d_ranges, int32_t* d_error, void* stream);

/* Load-map statistics produced by the render epilogue (LoadStats,
 * sb/metrics.py:59-86): exact integer moments, min, max.  The histogram is
 * optional (d_hist may be NULL); when given it has hist_bins entries and
 * counts >= hist_bins are clamped into the last bin. */
typedef struct {
    int64_t sum;
    int64_t sum_sq;
    int32_t min;
    int32_t max;
} adr_load_stats;

/* Stage 6 — render (sb/render.py:128-171): per-tile front-to-back blend and
 * per-pixel composited count.  d_gidx lists, per sorted pair, the Gaussian
 * index into the projection; d_ranges is the (n_tiles,2) span table. */
int32_t adr_render(const adr_projection* proj, int64_t n, const int64_t* d_gidx, int64_t p,
                   const int64_t* d_ranges, const adr_camera* cam, double alpha_low,
                   double term_threshold, float* d_pixels, int32_t* d_counts,
                   adr_load_stats* d_stats, int32_t* d_hist, int32_t hist_bins, void* stream);

/* ------------------------------------------------------- numerics checks */

/* The render's float32 exp (restatement of numpy's, sb/render.py:96) on n
 * device floats, for golden-vector tests. */
int32_t adr_exp_np_f32(const float* d_x, float* d_y, int64_t n, void* stream);

/* Exhaustive check of the render's exp fast path against the full exp on
 * every float32 in [-87, 88]: d_result[0] = mismatches, d_result[1] = inputs
 * checked, d_result[2] = smallest mismatching bit pattern (all-ones if none). */
int32_t adr_selftest_exp(uint64_t* d_result, void* stream);

/* Exhaustive pin of the render's exp against numpy's: *d_out = sum over the
 * float32 bit patterns u in [lo, hi) of (bits(exp(u)) + 1) *
 * (u * 0x9E3779B97F4A7C15 | 1) mod 2^64 — the checksum
 * tests/golden/make_exp_exhaustive.py computes over np.exp(float32). */
int32_t adr_exp_checksum(uint64_t lo, uint64_t hi, uint64_t* d_out, void* stream);

/* The PLY loader's float64 activations (test infrastructure): over every
 * non-NaN float32 bit pattern u in [lo, hi) widened to float64, the sum of
 * (bits(f(u)) + 1) * (u * 0x9E3779B97F4A7C15 | 1) mod 2^64 with f = np.exp
 * (kind 0) or scipy.special.expit (kind 1) as adr_ply_activate evaluates
 * them; tests/golden/make_exp64_exhaustive.py sums numpy / scipy. */
int32_t adr_exp64_checksum(int32_t kind, uint64_t lo, uint64_t hi, uint64_t* d_out, void* stream);

/* Render self-check (test infrastructure, no reference counterpart).  With
 * enable != 0 the following frames launch the counting instantiation of the
 * tile blend, which iterates each warp's plain bounding box and counts every
 * splat the 8x8-quadrant tau-ellipse mask would have skipped although one of
 * the warp's pixels passes the exact power test (an unsafe removal).
 * host_out (8 counters, may be NULL) receives the counters accumulated since
 * the previous call (synchronises the device); the call also resets them.
 * [2] = warp iterations the mask removes, [6] = batches + 1e9 x unsafe
 * removals (must stay < 1e9). */
int32_t adr_render_selfcheck(int32_t enable, unsigned long long* host_out);

/* ------------------------------------------------------------ PLY ingest */

/* load_ply (sb/scene.py:316-398), device half: activates rows
 * [row0, row0 + rows) of the float32 property matrix (d_raw = row row0's
 * first property, 16-byte aligned, n_props <= 1536 floats per row, file
 * order) into the float64
 * scene *out (dtype ADR_F64, out->n = all rows): centers = (x, y, z),
 * scales = np.exp(scale_*), rotations = rot / np.linalg.norm(rot),
 * opacities = scipy expit(opacity), sh = (f_dc, f_rest) gathered to (K, 3),
 * bit-identical to the reference's numpy / scipy arithmetic.  cols (host,
 * 11 + 3K entries): the property column of x, y, z, scale_0..2, rot_0..3,
 * opacity, then each SH coefficient in (k, channel) order.  d_status
 * (device, 2 int64, reset to INT64_MAX by adr_ply_status_reset) receives the
 * smallest row with a non-finite property (scene.py:370-373) and with a
 * quaternion norm < 1e-12 (scene.py:388-391); the caller raises from them. */
int32_t adr_ply_status_reset(int64_t* d_status, void* stream);
int32_t adr_ply_activate(const float* d_raw, int64_t row0, int64_t rows, int32_t n_props,
                         const int32_t* cols, const adr_scene* out, int64_t* d_status, void* stream);

/* ----------------------------------------------- brute-force reference path */

/* render_reference (sb/oracle.py:23-78) on the GPU: given a BASELINE-mode
 * Projection of n Gaussians, sort the valid ones globally by (float32 depth
 * bits, index) and blend every pixel over the Gaussians whose footprint
 * rectangle overlaps its tile, with no tile binning.  Writes the (H,W,3)
 * image and (H,W) load map; bit-identical to adr_render_frame's when stages
 * 2-5 are correct.  Asynchronous; scratch from
 * adr_render_reference_scratch_bytes(n). */
size_t adr_render_reference_scratch_bytes(int64_t n);
int32_t adr_render_reference(const adr_projection* proj, int64_t n, const adr_camera* cam,
                             double alpha_low, double term_threshold, float* d_pixels,
                             int32_t* d_load, void* d_scratch, size_t scratch_bytes, void* stream);

/* ------------------------------------------------- load-balancing objective */

/* Image terms of total_loss (sb/metrics.py:94-143) in fp64: d_out[0] =
 * l1_loss(a, b) (mean |a - b| over H*W*3), d_out[1] = ssim(a, b) (11-tap
 * Gaussian window given in h_window — the host computes it with the
 * reference's numpy expression, sb/metrics.py:108-111 — applied as
 * scipy.ndimage.correlate1d along rows then columns with zero padding; SSIM
 * constants c1, c2).  a, b: (H,W,3) float32 device images.  Asynchronous;
 * scratch from adr_image_loss_scratch_bytes(). */
size_t adr_image_loss_scratch_bytes(int32_t width, int32_t height);
int32_t adr_image_losses(const float* d_a, const float* d_b, int32_t width, int32_t height,
                         const double* h_window, double c1, double c2, double* d_out,
                         void* d_scratch, size_t scratch_bytes, void* stream);

/* --------------------------------------------- fused pipeline (run_pipeline)
 * sb/pipeline.py:85-124.  The frame runs as a fixed kernel sequence with no
 * host synchronisation, so it can be captured into a CUDA graph.  Pair
 * buffers have a caller-chosen capacity; when the frame needs more pairs the
 * frame still completes (no out-of-bounds writes), *d_pair_count holds the
 * true P and the caller re-runs with a larger capacity.
 */
typedef struct {
    /* outputs (device) */
    adr_projection proj;          /* Projection                           */
    float* d_pixels;              /* (H,W,3)                              */
    int32_t* d_load;              /* (H,W)                                */
    uint64_t* d_keys;             /* (pair_capacity,) sorted keys, optional */
    int32_t* d_gidx;              /* (pair_capacity,) sorted Gaussian indices (required) */
    int64_t* d_ranges;            /* (n_tiles,2)                           */
    int64_t* d_counters;          /* 8 entries: [0]=P, [1]=culled, [2]=M (Gaussians with
                                     pairs), [3]=min(P, capacity), [4]=valid rows with a NaN
                                     colour, [5]=ceil-ambiguous culling extents (log fence:
                                     0 proves the extents equal numpy's), [6]=1 when
                                     P > pair_capacity (frame truncated, re-run larger) */
    adr_load_stats* d_stats;
    int32_t* d_hist;              /* optional, hist_bins entries           */
    int32_t hist_bins;
    /* workspace */
    void* d_scratch;
    size_t scratch_bytes;
    int64_t pair_capacity;
    /* optional per-stage CUDA events (7 cudaEvent_t as void*), may be NULL */
    void* const* events;
    /* nonzero: the Projection's mean2d, conic, opacity and color are written
     * only into the render record — row i is 12 float32 at byte offset
     * adr_frame_record_offset(...) + 48 i of d_scratch: mean2d = [0:2],
     * conic = [2:5], opacity = [5], color = [6:9] (rows of invalid Gaussians
     * zero) — and proj.d_mean2d / d_conic / d_opacity / d_color are not
     * touched (the caller views the record instead: 36 bytes per Gaussian
     * fewer to write).  0: every Projection array is written. */
    int32_t projection_in_record;
} adr_frame_buffers;

size_t adr_frame_scratch_bytes(int64_t n, int32_t width, int32_t height, int64_t pair_capacity);
/* Byte offset of the render record array inside the frame scratch. */
size_t adr_frame_record_offset(int64_t n, int32_t width, int32_t height, int64_t pair_capacity);
int32_t adr_render_frame(const adr_scene* scene, const adr_camera* cam, int32_t mode,
                         double alpha_low, double dilation, double term_threshold,
                         const adr_frame_buffers* buf, void* stream);

/* Batched frames of one scene (no reference counterpart to replace: the
 * reference renders one view per run_pipeline call, sb/pipeline.py:85-124;
 * this is that call split at its stage-1 boundary, sb/pipeline.py:98).
 *
 * adr_preprocess_views: stage 1 of n_views (1..8) frames in ONE launch.  Each
 * Gaussian's row and SH coefficients are read once and its view-independent
 * terms (cov3d, ln(sigma / alpha_low)) evaluated once; every view's
 * Projection, render record, tile rect and depth key are written into bufs[v]
 * (an array of n_views frame buffers, each its own scratch and counters),
 * bit-identical to adr_render_frame's stage 1 for (scene, cams[v]).
 * adr_render_frame_post: stages 2-6 of a frame whose stage 1 ran through
 * adr_preprocess_views (same scene, camera, mode, alpha_low; enqueue it after
 * that launch, e.g. on another stream behind an event).  Together they give
 * exactly adr_render_frame's outputs.  Events [0] and [1] are not recorded. */
int32_t adr_preprocess_views(const adr_scene* scene, const adr_camera* cams, int32_t n_views,
                             int32_t mode, double alpha_low, double dilation,
                             const adr_frame_buffers* bufs, void* stream);
int32_t adr_render_frame_post(const adr_scene* scene, const adr_camera* cam, int32_t mode,
                              double alpha_low, double dilation, double term_threshold,
                              const adr_frame_buffers* buf, void* stream);

#ifdef __cplusplus
}
#endif
#endif
