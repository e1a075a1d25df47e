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
    l.kminmax = c.take<uint32_t>(2 * ceil_div(n > 0 ? n : 1, 128));
    l.plan_mm = c.take<uint32_t>(2);
    l.tile_order = c.take<uint32_t>(n_tiles);
    l.binning_bytes = frame_binning_scratch(n, cap, tx, ty);
    l.binning = c.take<char>((int64_t)l.binning_bytes);
    if (out) *out = l;
    return c.used;
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
    if (!scene || !cam || !buf) return fail(ADR_ERR_VALUE, "null argument");
    if (cam->width < 1 || cam->height < 1) return fail(ADR_ERR_VALUE, "grid dimensions must be positive");
    cudaStream_t st = as_stream(stream);
    const int32_t tx = tiles_of(cam->width), ty = tiles_of(cam->height);
    const int64_t n_tiles = (int64_t)tx * ty;
    if (n_tiles >= (int64_t(1) << 32)) return fail(ADR_ERR_CAPACITY, "tile count does not fit the 32-bit key field");
    const int64_t n = scene->n;
    FrameLayout L;
    const size_t need = frame_bytes(n, tx, ty, buf->pair_capacity, &L, buf->d_scratch, buf->scratch_bytes);
    if (need > buf->scratch_bytes) return fail(ADR_ERR_VALUE, "render_frame: scratch too small");
    cudaEvent_t ev[7] = {};
    if (buf->events)
        for (int i = 0; i < 7; ++i) ev[i] = reinterpret_cast<cudaEvent_t>(buf->events[i]);

    ADR_CUDA_TRY(cudaMemsetAsync(buf->d_counters, 0, 8 * sizeof(int64_t), st));
    if (ev[0]) ADR_CUDA_TRY(cudaEventRecord(ev[0], st));
    FusedPre fp;
    fp.rec = L.rec;
    fp.gpack = L.gpack;
    fp.dkey = L.dkey;
    fp.d_m = buf->d_counters + 2;
    fp.culled = reinterpret_cast<unsigned long long*>(buf->d_counters + 1);
    fp.nan_colors = reinterpret_cast<unsigned long long*>(buf->d_counters + 4);
    fp.ambiguous = reinterpret_cast<unsigned long long*>(buf->d_counters + 5);
    fp.tiles_x = tx;
    fp.tiles_y = ty;
    fp.kminmax = supertile_path(n_tiles, tx, ty) ? L.kminmax : nullptr;
    fp.rec_only = buf->projection_in_record != 0;
    fp.ln_a32_a64 = std::log((double)(float)alpha_low / alpha_low);
    fp.plan_mm = fp.kminmax ? L.plan_mm : nullptr;
    int32_t rc = launch_preprocess(*scene, *cam, mode, alpha_low, dilation, buf->proj, &fp, st);
    if (rc) return rc;
    if (ev[1]) ADR_CUDA_TRY(cudaEventRecord(ev[1], st));

    if (n > 0) {
        FrameBinning fb;
        fb.proj = buf->proj;
        fb.n = n;
        fb.cap = buf->pair_capacity;
        fb.n_tiles = n_tiles;
        fb.tiles_x = tx;
        fb.tiles_y = ty;
        fb.dkey = L.dkey;
        fb.order = L.order;
        fb.gpack = L.gpack;
        fb.kminmax = fp.kminmax;
        fb.plan_mm = fp.plan_mm;
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
        ADR_CUDA_TRY(cudaMemsetAsync(buf->d_ranges, 0, sizeof(int64_t) * 2 * n_tiles, st));
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
    ra.width = cam->width;
    ra.height = cam->height;
    ra.tiles_x = tx;
    ra.tiles_y = ty;
    for (int i = 0; i < 3; ++i) ra.bg[i] = cam->background[i];
    ra.alpha_low = (float)alpha_low;
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

}  // extern "C"
