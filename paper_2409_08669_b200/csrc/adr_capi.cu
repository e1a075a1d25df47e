// adr_capi.cu — extern "C" entry points of libadrsplat (include/adr_splat.h)
// and the fused frame (sb/pipeline.py:85-124).
#include <atomic>
#include <cmath>
#include <climits>
#include <string>

#include "adr_binning.cuh"
#include "adr_kernels.cuh"

namespace adr {

namespace {
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const std::string& msg) { g_last_error = msg; }

int32_t fail(int32_t code, const std::string& msg) {
    set_error(msg);
    return code;
}

namespace {

inline int32_t tiles_of(int32_t v) { return (v + kTile - 1) / kTile; }

// Workspace carve-up of the fused frame (must match adr_frame_scratch_bytes).
struct FrameLayout {
    uint32_t* dkey;
    uint32_t* order;
    Record* rec;
    size_t rec_offset;   // byte offset of rec inside the scratch
    uint2* gpack;
    uint32_t* kminmax;
    uint32_t* plan_mm;
    uint32_t* tile_order;
    void* binning;
    size_t binning_bytes;
};

size_t frame_bytes(int64_t n, int32_t tx, int32_t ty, int64_t cap, FrameLayout* out, void* base, size_t cap_bytes) {
    const int64_t n_tiles = (int64_t)tx * ty;
    Carver c(base, cap_bytes);
    FrameLayout l;
    l.dkey = c.take<uint32_t>(n);
    l.order = c.take<uint32_t>(n);
    l.rec_offset = c.used;
    l.rec = c.take<Record>(n);
    l.gpack = c.take<uint2>(n);
    l.kminmax = c.take<uint32_t>(2 * 4 * ceil_div(n > 0 ? n : 1, 128));   // per preprocess warp
    l.plan_mm = c.take<uint32_t>(2);
    l.tile_order = c.take<uint32_t>(n_tiles);
    l.binning_bytes = frame_binning_scratch(n, cap, tx, ty);
    l.binning = c.take<char>((int64_t)l.binning_bytes);
    if (out) *out = l;
    return c.used;
}

}  // namespace

}  // namespace adr


namespace adr {
namespace {

// Per-frame layout and the fused stage-1 extras of one frame's buffers.
struct FrameSetup {
    FrameLayout L;
    FusedPre fp;
    cudaEvent_t ev[7] = {};
    int32_t tx = 0, ty = 0;
    int64_t n_tiles = 0;
    double alpha_low = 0.0;
};

int32_t frame_setup(const adr_scene* scene, const adr_camera* cam, double alpha_low, const adr_frame_buffers* buf,
                    FrameSetup* f) {
    if (!scene || !cam || !buf) return fail(ADR_ERR_VALUE, "null argument");
    if (cam->width < 1 || cam->height < 1) return fail(ADR_ERR_VALUE, "grid dimensions must be positive");
    f->tx = tiles_of(cam->width);
    f->ty = tiles_of(cam->height);
    f->n_tiles = (int64_t)f->tx * f->ty;
    if (f->n_tiles >= (int64_t(1) << 32)) return fail(ADR_ERR_CAPACITY, "tile count does not fit the 32-bit key field");
    const size_t need = frame_bytes(scene->n, f->tx, f->ty, buf->pair_capacity, &f->L, buf->d_scratch,
                                    buf->scratch_bytes);
    if (need > buf->scratch_bytes) return fail(ADR_ERR_VALUE, "render_frame: scratch too small");
    if (buf->events)
        for (int i = 0; i < 7; ++i) f->ev[i] = reinterpret_cast<cudaEvent_t>(buf->events[i]);
    f->alpha_low = alpha_low;
    FusedPre& fp = f->fp;
    fp.rec = f->L.rec;
    fp.gpack = f->L.gpack;
    fp.dkey = f->L.dkey;
    fp.d_m = buf->d_counters + 2;
    fp.culled = reinterpret_cast<unsigned long long*>(buf->d_counters + 1);
    fp.nan_colors = reinterpret_cast<unsigned long long*>(buf->d_counters + 4);
    fp.ambiguous = reinterpret_cast<unsigned long long*>(buf->d_counters + 5);
    fp.tiles_x = f->tx;
    fp.tiles_y = f->ty;
    fp.kminmax = supertile_path(f->n_tiles, f->tx, f->ty) ? f->L.kminmax : nullptr;
    fp.rec_only = buf->projection_in_record != 0;
    fp.ln_a32_a64 = std::log((double)(float)alpha_low / alpha_low);
    fp.plan_mm = fp.kminmax ? f->L.plan_mm : nullptr;
    return ADR_OK;
}

// Stages 2-6 of a frame whose stage 1 (fused) has run on `st` or before it.
int32_t frame_post(const adr_scene& scene, const adr_camera& cam, double term_threshold,
                   const adr_frame_buffers* buf, const FrameSetup& f, cudaStream_t st) {
    const int64_t n = scene.n;
    const FrameLayout& L = f.L;
    const cudaEvent_t* ev = f.ev;
    int32_t rc = ADR_OK;
    if (n > 0) {
        FrameBinning fb;
        fb.proj = buf->proj;
        fb.n = n;
        fb.cap = buf->pair_capacity;
        fb.n_tiles = f.n_tiles;
        fb.tiles_x = f.tx;
        fb.tiles_y = f.ty;
        fb.dkey = L.dkey;
        fb.order = L.order;
        fb.gpack = L.gpack;
        fb.kminmax = f.fp.kminmax;
        fb.plan_mm = f.fp.plan_mm;
        fb.ranges = buf->d_ranges;
        fb.keys = buf->d_keys;
        fb.gidx = buf->d_gidx;
        fb.counters = buf->d_counters;
        fb.stats = buf->d_hist ? nullptr : buf->d_stats;   // with a histogram the init kernel runs
        fb.scratch = L.binning;
        fb.scratch_bytes = L.binning_bytes;
        fb.ev_after_scan = ev[2];
        fb.ev_after_dup = ev[3];
        fb.ev_after_sort = ev[4];
        fb.ev_after_ranges = ev[5];
        rc = frame_binning(fb, st);
        if (rc) return rc;
    } else {
        ADR_CUDA_TRY(cudaMemsetAsync(buf->d_ranges, 0, sizeof(int64_t) * 2 * f.n_tiles, st));
        for (int i = 2; i <= 5; ++i)
            if (ev[i]) ADR_CUDA_TRY(cudaEventRecord(ev[i], st));
    }

    if (n <= 0 || buf->d_hist) {
        rc = launch_init_stats(buf->d_stats, buf->d_hist, buf->hist_bins, st);
        if (rc) return rc;
    }
    RenderArgs ra;
    ra.rec = L.rec;
    ra.idx = reinterpret_cast<const uint32_t*>(buf->d_gidx);
    ra.ranges = buf->d_ranges;
    ra.order = nullptr;  // longest-span-first order measured no gain (profiles/r01_notes.md)
    ra.width = cam.width;
    ra.height = cam.height;
    ra.tiles_x = f.tx;
    ra.tiles_y = f.ty;
    for (int i = 0; i < 3; ++i) ra.bg[i] = cam.background[i];
    ra.alpha_low = (float)f.alpha_low;
    ra.term = (float)term_threshold;
    ra.pixels = buf->d_pixels;
    ra.load = buf->d_load;
    ra.stats = buf->d_stats;
    ra.hist = buf->d_hist;
    ra.hist_bins = buf->hist_bins;
    ra.nan_flag = buf->d_counters + 4;
    rc = launch_render(ra, st);
    if (rc) return rc;
    if (ev[6]) ADR_CUDA_TRY(cudaEventRecord(ev[6], st));
    return ADR_OK;
}

}  // namespace
}  // namespace adr

using namespace adr;

extern "C" {

int32_t adr_abi_version(void) { return ADR_ABI_VERSION; }

int64_t adr_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

const char* adr_last_error(void) { return g_last_error.c_str(); }

int32_t adr_device_sm_count(void) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return sms;
}

int32_t adr_preprocess(const adr_scene* scene, const adr_camera* cam, int32_t mode, double alpha_low,
                       double dilation, const adr_projection* out, void* stream) {
    if (!scene || !cam || !out) return fail(ADR_ERR_VALUE, "null argument");
    return launch_preprocess(*scene, *cam, mode, alpha_low, dilation, *out, nullptr, as_stream(stream));
}

int32_t adr_touched_counts(const adr_projection* proj, int64_t n, int32_t tiles_x, int32_t tiles_y,
                           int64_t* d_counts, void* stream) {
    if (!proj) return fail(ADR_ERR_VALUE, "null argument");
    return stage_touched_counts(*proj, n, tiles_x, tiles_y, d_counts, as_stream(stream));
}

size_t adr_inclusive_sum_scratch_bytes(int64_t n) { return stage_inclusive_sum_scratch(n); }

int32_t adr_inclusive_sum(const int64_t* d_counts, int64_t n, int64_t* d_offsets, int32_t* d_overflow,
                          void* d_scratch, size_t scratch_bytes, void* stream) {
    return stage_inclusive_sum(d_counts, n, d_offsets, d_overflow, d_scratch, scratch_bytes, as_stream(stream));
}

int32_t adr_duplicate_with_keys(const adr_projection* proj, int64_t n, const int64_t* d_offsets, int32_t tiles_x,
                                int32_t tiles_y, uint64_t* d_keys, int64_t* d_gidx, void* stream) {
    if (!proj) return fail(ADR_ERR_VALUE, "null argument");
    return stage_duplicate(*proj, n, d_offsets, tiles_x, tiles_y, d_keys, d_gidx, as_stream(stream));
}

size_t adr_sort_pairs_scratch_bytes(int64_t p) { return stage_sort_scratch(p); }

int32_t adr_sort_pairs(const uint64_t* d_keys, const int64_t* d_gidx, int64_t p, int32_t end_bit,
                       uint64_t* d_keys_out, int64_t* d_gidx_out, void* d_scratch, size_t scratch_bytes,
                       void* stream) {
    return stage_sort(d_keys, d_gidx, p, end_bit, d_keys_out, d_gidx_out, d_scratch, scratch_bytes,
                      as_stream(stream));
}

int32_t adr_identify_tile_ranges(const uint64_t* d_sorted_keys, int64_t p, int64_t n_tiles, int64_t* d_ranges,
                                 int32_t* d_error, void* stream) {
    return stage_ranges(d_sorted_keys, p, n_tiles, d_ranges, d_error, as_stream(stream));
}

int32_t adr_render(const adr_projection* proj, int64_t n, const int64_t* d_gidx, int64_t p, const int64_t* d_ranges,
                   const adr_camera* cam, double alpha_low, double term_threshold, float* d_pixels,
                   int32_t* d_counts, adr_load_stats* d_stats, int32_t* d_hist, int32_t hist_bins, void* stream) {
    if (!proj || !cam) return fail(ADR_ERR_VALUE, "null argument");
    (void)n;
    (void)p;
    cudaStream_t st = as_stream(stream);
    int32_t rc = launch_init_stats(d_stats, d_hist, hist_bins, st);
    if (rc) return rc;
    return launch_render_proj(*proj, d_gidx, d_ranges, cam->width, cam->height, cam->background, (float)alpha_low,
                              (float)term_threshold, d_pixels, d_counts, d_stats, d_hist, hist_bins, st);
}

size_t adr_frame_record_offset(int64_t n, int32_t width, int32_t height, int64_t pair_capacity) {
    FrameLayout L;
    frame_bytes(n, tiles_of(width), tiles_of(height), pair_capacity, &L, nullptr, 0);
    return L.rec_offset;
}

size_t adr_frame_scratch_bytes(int64_t n, int32_t width, int32_t height, int64_t pair_capacity) {
    return frame_bytes(n, tiles_of(width), tiles_of(height), pair_capacity, nullptr, nullptr, 0) + 1024;
}

int32_t adr_render_frame(const adr_scene* scene, const adr_camera* cam, int32_t mode, double alpha_low,
                         double dilation, double term_threshold, const adr_frame_buffers* buf, void* stream) {
    FrameSetup f;
    int32_t rc = frame_setup(scene, cam, alpha_low, buf, &f);
    if (rc) return rc;
    cudaStream_t st = as_stream(stream);
    ADR_CUDA_TRY(cudaMemsetAsync(buf->d_counters, 0, 8 * sizeof(int64_t), st));
    if (f.ev[0]) ADR_CUDA_TRY(cudaEventRecord(f.ev[0], st));
    rc = launch_preprocess(*scene, *cam, mode, alpha_low, dilation, buf->proj, &f.fp, st);
    if (rc) return rc;
    if (f.ev[1]) ADR_CUDA_TRY(cudaEventRecord(f.ev[1], st));
    return frame_post(*scene, *cam, term_threshold, buf, f, st);
}

int32_t adr_preprocess_views(const adr_scene* scene, const adr_camera* cams, int32_t n_views, int32_t mode,
                             double alpha_low, double dilation, const adr_frame_buffers* bufs, void* stream) {
    if (!scene || !cams || !bufs) return fail(ADR_ERR_VALUE, "null argument");
    if (n_views < 1 || n_views > kMaxBatchViews) return fail(ADR_ERR_VALUE, "n_views must lie in 1..8");
    cudaStream_t st = as_stream(stream);
    PreViews pv;
    pv.nv = n_views;
    for (int v = 0; v < n_views; ++v) {
        FrameSetup f;
        int32_t rc = frame_setup(scene, &cams[v], alpha_low, &bufs[v], &f);
        if (rc) return rc;
        for (int u = 0; u < v; ++u)
            if (bufs[u].d_scratch == bufs[v].d_scratch || bufs[u].d_counters == bufs[v].d_counters ||
                bufs[u].proj.d_valid == bufs[v].proj.d_valid)
                return fail(ADR_ERR_VALUE, "preprocess_views: every view needs its own frame buffers");
        ADR_CUDA_TRY(cudaMemsetAsync(bufs[v].d_counters, 0, 8 * sizeof(int64_t), st));
        pv.cam[v] = cams[v];
        pv.out[v] = bufs[v].proj;
        pv.fused[v] = f.fp;
    }
    return launch_preprocess_views(*scene, pv, mode, alpha_low, dilation, st);
}

int32_t adr_render_frame_post(const adr_scene* scene, const adr_camera* cam, int32_t mode, double alpha_low,
                              double dilation, double term_threshold, const adr_frame_buffers* buf, void* stream) {
    (void)mode;
    (void)dilation;
    FrameSetup f;
    int32_t rc = frame_setup(scene, cam, alpha_low, buf, &f);
    if (rc) return rc;
    return frame_post(*scene, *cam, term_threshold, buf, f, as_stream(stream));
}

}  // extern "C"
