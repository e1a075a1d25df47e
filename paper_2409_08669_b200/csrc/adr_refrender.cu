// adr_refrender.cu — brute-force reference renderer on the GPU
// (sb/oracle.py:23-78): a large-N self-check of stages
// 2-5 that bypasses the tile binning entirely.
//
//   1. every valid Gaussian sorted once, globally, by (float32 depth bits,
//      index) — keys built here, the library's stable LSD radix sort;
//   2. per 16-row pixel band, the Gaussians that can reach the band
//      (sb/oracle.py:54-58, fp64 interval tests) are compacted in depth
//      order (stable: flag, inclusive scan, scatter);
//   3. one CTA per tile of the band walks that list; a Gaussian exists for
//      the tile only when its footprint rectangle overlaps the tile — the
//      reference's own independent interval comparison (sb/oracle.py:
//      64-70), not the binning code — and pixels blend with the exact
//      scalar recurrence (numpy float32 exp, no culling shortcuts).
//
// Bitwise equality with the fused frame therefore checks counting, prefix
// sum, key packing, both sorts and range identification.
#include "adr_binning.cuh"
#include "adr_sort.cuh"

namespace adr {
namespace {

__global__ void k_ref_keys(const uint8_t* __restrict__ valid, const float* __restrict__ depth, int64_t n,
                           uint64_t* __restrict__ keys, int64_t* __restrict__ vals,
                           unsigned long long* __restrict__ m) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool v = i < n && valid[i];
    if (i < n) {
        keys[i] = v ? (uint64_t)__float_as_uint(depth[i]) : 0xffffffffull;
        vals[i] = i;
    }
    const uint32_t b = __ballot_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(m, (unsigned long long)__popc(b));
}

struct RefGeom {
    const float2* mean2d;
    const int32_t* ext_x;
    const int32_t* ext_y;
};

// reachable(g) for the band [row_top, row_top + 16) (sb/oracle.py:54-58)
__device__ __forceinline__ bool reaches_band(const RefGeom& g, int64_t i, double row_top, double grid_right) {
    const float2 m = g.mean2d[i];
    const double mx = m.x, my = m.y, ex = g.ext_x[i], ey = g.ext_y[i];
    return (__dsub_rn(my, ey) < __dadd_rn(row_top, 16.0)) && (__dadd_rn(my, ey) >= row_top) &&
           (__dsub_rn(mx, ex) < grid_right) && (__dadd_rn(mx, ex) >= 0.0);
}

__global__ void k_band_flags(RefGeom g, const int64_t* __restrict__ order, const unsigned long long* __restrict__ d_m,
                             int64_t n, double row_top, double grid_right, int64_t* __restrict__ flags) {
    const int64_t m = (int64_t)*d_m;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) flags[p] = (p < m && reaches_band(g, order[p], row_top, grid_right)) ? 1 : 0;
}

__global__ void k_band_scatter(const int64_t* __restrict__ order, const int64_t* __restrict__ flags,
                               const int64_t* __restrict__ incl, const unsigned long long* __restrict__ d_m,
                               int64_t* __restrict__ band_list, int64_t* __restrict__ band_len) {
    const int64_t m = (int64_t)*d_m;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < m && flags[p]) band_list[incl[p] - 1] = order[p];
    if (p == 0) *band_len = m > 0 ? incl[m - 1] : 0;  // flags are 0 past m
}

constexpr int kRefBatch = 256;

__global__ void __launch_bounds__(kTilePixels)
k_ref_blend(adr_projection proj, const int64_t* __restrict__ band_list, const int64_t* __restrict__ band_len,
            int32_t band, int32_t width, int32_t height, float bg0, float bg1, float bg2, float alpha_low,
            float term, float* __restrict__ pixels, int32_t* __restrict__ load) {
    __shared__ float4 sG[kRefBatch];   // mx, my, a, b
    __shared__ float4 sW[kRefBatch];   // c, sigma, r, g
    __shared__ float sB[kRefBatch];    // blue
    __shared__ uint8_t sP[kRefBatch];  // present in this tile
    const int tx = blockIdx.x;
    const int px = tx * kTile + (threadIdx.x & (kTile - 1));
    const int py = band * kTile + (threadIdx.x >> 4);
    const bool inside = px < width && py < height;
    const float fpx = (float)px, fpy = (float)py;
    // the pixel's tile span (sb/oracle.py:61-62)
    const double tile_x0 = (double)(tx * kTile), tile_y0 = (double)(band * kTile);
    const int64_t len = *band_len;
    float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
    int cnt = 0;
    bool done = !inside;
    for (int64_t b0 = 0; b0 < len; b0 += kRefBatch) {
        if (__syncthreads_count(done) == kTilePixels) break;
        const int nb = (int)((len - b0) < kRefBatch ? (len - b0) : kRefBatch);
        if ((int)threadIdx.x < nb) {
            const int64_t g = band_list[b0 + threadIdx.x];
            const float2 m = reinterpret_cast<const float2*>(proj.d_mean2d)[g];
            const double mx = m.x, my = m.y, ex = proj.d_ext_x[g], ey = proj.d_ext_y[g];
            // present(): footprint rectangle vs the tile (sb/oracle.py:64-70)
            const bool present = (__dsub_rn(mx, ex) < __dadd_rn(tile_x0, 16.0)) && (__dadd_rn(mx, ex) >= tile_x0) &&
                                 (__dsub_rn(my, ey) < __dadd_rn(tile_y0, 16.0)) && (__dadd_rn(my, ey) >= tile_y0);
            sP[threadIdx.x] = present;
            sG[threadIdx.x] = make_float4(m.x, m.y, proj.d_conic[3 * g], proj.d_conic[3 * g + 1]);
            sW[threadIdx.x] = make_float4(proj.d_conic[3 * g + 2], proj.d_opacity[g], proj.d_color[3 * g],
                                          proj.d_color[3 * g + 1]);
            sB[threadIdx.x] = proj.d_color[3 * g + 2];
        }
        __syncthreads();
        for (int j = 0; j < nb && !done; ++j) {
            if (!sP[j]) continue;
            const float4 G = sG[j];
            const float4 W = sW[j];
            const float dx = __fsub_rn(fpx, G.x);
            const float dy = __fsub_rn(fpy, G.y);
            const float q = __fadd_rn(__fmul_rn(__fmul_rn(G.z, dx), dx), __fmul_rn(__fmul_rn(W.x, dy), dy));
            const float power = __fsub_rn(__fmul_rn(-0.5f, q), __fmul_rn(__fmul_rn(G.w, dx), dy));
            float alpha = __fmul_rn(W.y, exp_np(power));
            alpha = alpha < 0.99f ? alpha : (alpha != alpha ? alpha : 0.99f);
            if (!(alpha >= alpha_low)) continue;
            const float w = __fmul_rn(alpha, T);
            C0 = __fadd_rn(C0, __fmul_rn(w, W.z));
            C1 = __fadd_rn(C1, __fmul_rn(w, W.w));
            C2 = __fadd_rn(C2, __fmul_rn(w, sB[j]));
            T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
            ++cnt;
            if (T < term) done = true;
        }
    }
    if (inside) {
        const int64_t pix = (int64_t)py * width + px;
        float o0 = __fadd_rn(C0, __fmul_rn(T, bg0)), o1 = __fadd_rn(C1, __fmul_rn(T, bg1)),
              o2 = __fadd_rn(C2, __fmul_rn(T, bg2));
        pixels[3 * pix] = o0 < 0.f ? 0.f : (o0 > 1.f ? 1.f : o0);
        pixels[3 * pix + 1] = o1 < 0.f ? 0.f : (o1 > 1.f ? 1.f : o1);
        pixels[3 * pix + 2] = o2 < 0.f ? 0.f : (o2 > 1.f ? 1.f : o2);
        load[pix] = cnt;
    }
}

}  // namespace
}  // namespace adr

using namespace adr;

extern "C" {

size_t adr_render_reference_scratch_bytes(int64_t n) {
    const int64_t nn = n > 0 ? n : 1;
    return 6 * align_up(sizeof(int64_t) * (size_t)nn) + radix_scratch_bytes<uint64_t, int64_t>(nn) +
           stage_inclusive_sum_scratch(nn) + 4096;
}

int32_t adr_render_reference(const adr_projection* proj, int64_t n, const adr_camera* cam, double alpha_low,
                             double term_threshold, float* d_pixels, int32_t* d_load, void* d_scratch,
                             size_t scratch_bytes, void* stream) {
    if (!proj || !cam || !d_pixels || !d_load) return fail(ADR_ERR_VALUE, "null argument");
    if (scratch_bytes < adr_render_reference_scratch_bytes(n)) return fail(ADR_ERR_VALUE, "scratch too small");
    cudaStream_t st = as_stream(stream);
    const int32_t width = cam->width, height = cam->height;
    const int32_t tiles_x = (width + kTile - 1) / kTile, tiles_y = (height + kTile - 1) / kTile;
    const int64_t nn = n > 0 ? n : 1;
    Carver c(d_scratch, scratch_bytes);
    uint64_t* keys = c.take<uint64_t>(nn);
    int64_t* vals = c.take<int64_t>(nn);
    uint64_t* skeys = c.take<uint64_t>(nn);
    int64_t* order = c.take<int64_t>(nn);
    int64_t* flags = c.take<int64_t>(nn);
    int64_t* incl = c.take<int64_t>(nn);
    const size_t rs = radix_scratch_bytes<uint64_t, int64_t>(nn);
    void* rscratch = c.take<char>((int64_t)rs);
    const size_t ss = stage_inclusive_sum_scratch(nn);
    void* sscratch = c.take<char>((int64_t)ss);
    unsigned long long* d_m = c.take<unsigned long long>(1);
    int64_t* band_len = c.take<int64_t>(1);
    int32_t* overflow = c.take<int32_t>(1);
    if (!c.ok()) return fail(ADR_ERR_VALUE, "scratch too small");
    ADR_CUDA_TRY(cudaMemsetAsync(d_m, 0, sizeof(unsigned long long), st));
    if (n > 0) {
        k_ref_keys<<<ceil_div(n, 256), 256, 0, st>>>(proj->d_valid, proj->d_depth, n, keys, vals, d_m);
        ADR_LAUNCH_CHECK();
        // stable sort by (depth bits, index); invalid rows (all-ones) last
        int32_t rc = radix_sort<uint64_t, int64_t>(keys, vals, skeys, order, nullptr, n, 32, rscratch, rs, st);
        if (rc) return rc;
    }
    const double grid_right = (double)tiles_x * kTile;  // sb/oracle.py:81-83
    RefGeom geom{reinterpret_cast<const float2*>(proj->d_mean2d), proj->d_ext_x, proj->d_ext_y};
    int64_t* band_list = reinterpret_cast<int64_t*>(keys);  // reuse: the unsorted keys are dead after the sort
    for (int32_t band = 0; band < tiles_y; ++band) {
        ADR_CUDA_TRY(cudaMemsetAsync(band_len, 0, sizeof(int64_t), st));
        if (n > 0) {
            k_band_flags<<<ceil_div(n, 256), 256, 0, st>>>(geom, order, d_m, n, (double)band * kTile, grid_right,
                                                           flags);
            ADR_LAUNCH_CHECK();
            int32_t rc = stage_inclusive_sum(flags, n, incl, overflow, sscratch, ss, st);
            if (rc) return rc;
            k_band_scatter<<<ceil_div(n, 256), 256, 0, st>>>(order, flags, incl, d_m, band_list, band_len);
            ADR_LAUNCH_CHECK();
        }
        k_ref_blend<<<tiles_x, kTilePixels, 0, st>>>(*proj, band_list, band_len, band, width, height,
                                                     cam->background[0], cam->background[1], cam->background[2],
                                                     (float)alpha_low, (float)term_threshold, d_pixels, d_load);
        ADR_LAUNCH_CHECK();
    }
    return ADR_OK;
}

}  // extern "C"
