// adr_render.cu — stage 6 (sb/render.py:57-171): per-tile front-to-back
// blending and the per-pixel load map, with the load-statistics epilogue
// (LoadStats / load_loss, sb/metrics.py:59-86).
//
// One CTA per 16x16 tile, one thread per pixel.  Each batch of 256 pairs is
// gathered into shared memory; every pixel then walks the batch in order with
// the exact fp32 recurrence of SURVEY.md App. A.3 (numpy float32 exp, no FMA
// contraction), so the image and load map equal the reference bit for bit.
#include "adr_kernels.cuh"
#include "adr_scan.cuh"

namespace adr {

namespace {

constexpr int kRenderBlock = kTilePixels;  // 256

// Record source for the fused frame: records by rank + per-pair rank list.
struct RecSource {
    const Record* rec;
    const uint32_t* idx;
    __device__ __forceinline__ Record load(int64_t j) const { return rec[idx[j]]; }
};

// Record source for the stage API: Projection SoA + int64 Gaussian indices.
struct ProjSource {
    const float2* mean2d;
    const float* conic;
    const float* opacity;
    const float* color;
    const int64_t* gidx;
    float alpha_low;
    __device__ __forceinline__ Record load(int64_t j) const {
        const int64_t g = gidx[j];
        const float2 m = mean2d[g];
        Record r;
        const float a = conic[3 * g], b = conic[3 * g + 1], c = conic[3 * g + 2], op = opacity[g];
        float tau, hx, hy;
        cull_params(a, b, c, op, alpha_low, &tau, &hx, &hy);
        r.a = make_float4(m.x, m.y, a, b);
        r.b = make_float4(c, op, color[3 * g], color[3 * g + 1]);
        r.c = make_float4(color[3 * g + 2], tau, hx, hy);
        return r;
    }
};

// Rows 2w, 2w+1 of the tile belong to warp w: bit w of the mask is set when
// the splat's conservative box (mx +- hx, my +- hy) meets those pixel rows
// and the tile's pixel columns.
__device__ __forceinline__ uint32_t warp_mask(const Record& r, float x_lo, float y_lo) {
    const float mx = r.a.x, my = r.a.y, hx = r.c.z, hy = r.c.w;
    if (!(mx - hx <= x_lo + (kTile - 1)) || !(mx + hx >= x_lo)) return 0u;
    const float lo = fmaxf(fminf(ceilf(0.5f * ((my - hy) - y_lo - 1.0f)), 8.0f), 0.0f);
    const float hi = fmaxf(fminf(floorf(0.5f * ((my + hy) - y_lo)), 7.0f), -1.0f);
    const int w0 = (int)lo, w1 = (int)hi;
    if (w1 < w0) return 0u;
    return ((2u << w1) - 1u) & ~((1u << w0) - 1u);
}

template <class Src>
__global__ void __launch_bounds__(kRenderBlock)
k_render(Src src, const int64_t* __restrict__ ranges, int32_t width, int32_t height, int32_t tiles_x, float bg0,
         float bg1, float bg2, float alpha_low, float term, float* __restrict__ pixels, int32_t* __restrict__ load,
         adr_load_stats* stats, int32_t* hist, int32_t hist_bins) {
    // shared-memory batch, split by use: the power test needs (mx, my, a, b)
    // + (c, tau); only contributions that pass it read (sigma, r, g, b)
    __shared__ float4 sG[kRenderBlock];   // mx, my, a, b
    __shared__ float2 sT[kRenderBlock];   // c, tau
    __shared__ float4 sW[kRenderBlock];   // sigma, r, g, b
    __shared__ uint8_t smask[kRenderBlock];
    __shared__ unsigned long long ssum[kRenderBlock / 32], ssq[kRenderBlock / 32];
    __shared__ int smin[kRenderBlock / 32], smax[kRenderBlock / 32];
    const int tile = blockIdx.x;
    const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
    const int px = tx * kTile + (threadIdx.x & (kTile - 1));
    const int py = ty * kTile + (threadIdx.x >> 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool inside = px < width && py < height;
    const int64_t start = ranges[2 * tile], end = ranges[2 * tile + 1];
    const float fpx = (float)px, fpy = (float)py;
    const float x_lo = (float)(tx * kTile), y_lo = (float)(ty * kTile);

    float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
    int cnt = 0;
    bool done = !inside;
    for (int64_t b = start; b < end; b += kRenderBlock) {
        if (__syncthreads_count(done) == kRenderBlock) break;
        const int nb = (int)((end - b) < kRenderBlock ? (end - b) : kRenderBlock);
        if ((int)threadIdx.x < nb) {
            const Record r = src.load(b + threadIdx.x);
            sG[threadIdx.x] = r.a;
            sT[threadIdx.x] = make_float2(r.b.x, r.c.y);
            sW[threadIdx.x] = make_float4(r.b.y, r.b.z, r.b.w, r.c.x);
            smask[threadIdx.x] = (uint8_t)warp_mask(r, x_lo, y_lo);
        }
        __syncthreads();
        if (__any_sync(kFull, !done)) {
            for (int c0 = 0; c0 < nb; c0 += 32) {
                uint32_t m = __ballot_sync(kFull, c0 + lane < nb && ((smask[c0 + lane] >> warp) & 1u));
                while (m) {
                    const int j = c0 + __ffs(m) - 1;
                    m &= m - 1u;
                    if (done) continue;
                    const float4 G = sG[j];
                    const float2 Tc = sT[j];
                    const float dx = __fsub_rn(fpx, G.x);
                    const float dy = __fsub_rn(fpy, G.y);
                    const float q = __fadd_rn(__fmul_rn(__fmul_rn(G.z, dx), dx), __fmul_rn(__fmul_rn(Tc.x, dy), dy));
                    const float power = __fsub_rn(__fmul_rn(-0.5f, q), __fmul_rn(__fmul_rn(G.w, dx), dy));
                    if (power < Tc.y) continue;  // alpha < alpha_low for sure (cull_params)
                    const float4 W = sW[j];
                    const float e = (power >= -87.0f && power <= 88.0f) ? exp_np_fast(power) : exp_np(power);
                    float alpha = __fmul_rn(W.x, e);
                    alpha = alpha < 0.99f ? alpha : (alpha != alpha ? alpha : 0.99f);
                    if (!(alpha >= alpha_low)) continue;
                    const float w = __fmul_rn(alpha, T);
                    C0 = __fadd_rn(C0, __fmul_rn(w, W.y));
                    C1 = __fadd_rn(C1, __fmul_rn(w, W.z));
                    C2 = __fadd_rn(C2, __fmul_rn(w, W.w));
                    T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                    ++cnt;
                    if (T < term) done = true;
                }
                if (__all_sync(kFull, done)) break;
            }
        }
    }
    if (inside) {
        const int64_t pix = (int64_t)py * width + px;
        float o0 = __fadd_rn(C0, __fmul_rn(T, bg0));
        float o1 = __fadd_rn(C1, __fmul_rn(T, bg1));
        float o2 = __fadd_rn(C2, __fmul_rn(T, bg2));
        o0 = o0 < 0.f ? 0.f : (o0 > 1.f ? 1.f : o0);
        o1 = o1 < 0.f ? 0.f : (o1 > 1.f ? 1.f : o1);
        o2 = o2 < 0.f ? 0.f : (o2 > 1.f ? 1.f : o2);
        pixels[3 * pix] = o0;
        pixels[3 * pix + 1] = o1;
        pixels[3 * pix + 2] = o2;
        load[pix] = cnt;
        if (hist) atomicAdd(hist + (cnt < hist_bins ? cnt : hist_bins - 1), 1);
    }
    if (stats) {
        unsigned long long s = inside ? (unsigned long long)cnt : 0ull;
        unsigned long long s2 = inside ? (unsigned long long)cnt * (unsigned long long)cnt : 0ull;
        int mn = inside ? cnt : INT_MAX, mx = inside ? cnt : INT_MIN;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_xor_sync(kFull, s, o);
            s2 += __shfl_xor_sync(kFull, s2, o);
            mn = min(mn, __shfl_xor_sync(kFull, mn, o));
            mx = max(mx, __shfl_xor_sync(kFull, mx, o));
        }
        const int w = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) {
            ssum[w] = s;
            ssq[w] = s2;
            smin[w] = mn;
            smax[w] = mx;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < kRenderBlock / 32; ++k) {
                s += ssum[k];
                s2 += ssq[k];
                mn = min(mn, smin[k]);
                mx = max(mx, smax[k]);
            }
            atomicAdd(reinterpret_cast<unsigned long long*>(&stats->sum), s);
            atomicAdd(reinterpret_cast<unsigned long long*>(&stats->sum_sq), s2);
            atomicMin(&stats->min, mn);
            atomicMax(&stats->max, mx);
        }
    }
}

__global__ void k_init_stats(adr_load_stats* stats, int32_t* hist, int32_t bins) {
    if (stats && blockIdx.x == 0 && threadIdx.x == 0) {
        stats->sum = 0;
        stats->sum_sq = 0;
        stats->min = INT_MAX;
        stats->max = INT_MIN;
    }
    if (hist)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < bins; i += (int64_t)gridDim.x * blockDim.x)
            hist[i] = 0;
}

}  // namespace

int32_t launch_init_stats(adr_load_stats* stats, int32_t* hist, int32_t bins, cudaStream_t st) {
    if (!stats && !hist) return ADR_OK;
    const int blocks = hist ? (int)((bins + 255) / 256 < 1024 ? (bins + 255) / 256 : 1024) : 1;
    k_init_stats<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(stats, hist, bins);
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

int32_t launch_render(const RenderArgs& a, cudaStream_t st) {
    const int64_t n_tiles = (int64_t)a.tiles_x * a.tiles_y;
    if (n_tiles <= 0) return ADR_OK;
    RecSource src{a.rec, a.idx};
    k_render<RecSource><<<n_tiles, kRenderBlock, 0, st>>>(src, a.ranges, a.width, a.height, a.tiles_x, a.bg[0], a.bg[1],
                                                         a.bg[2], a.alpha_low, a.term, a.pixels, a.load, a.stats,
                                                         a.hist, a.hist_bins);
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

int32_t launch_render_proj(const adr_projection& p, const int64_t* gidx, const int64_t* ranges, int32_t width,
                           int32_t height, const float* bg, float alpha_low, float term, float* pixels,
                           int32_t* load, adr_load_stats* stats, int32_t* hist, int32_t bins, cudaStream_t st) {
    const int32_t tx = (width + kTile - 1) / kTile, ty = (height + kTile - 1) / kTile;
    const int64_t n_tiles = (int64_t)tx * ty;
    if (n_tiles <= 0) return ADR_OK;
    ProjSource src{reinterpret_cast<const float2*>(p.d_mean2d), p.d_conic, p.d_opacity, p.d_color, gidx, alpha_low};
    k_render<ProjSource><<<n_tiles, kRenderBlock, 0, st>>>(src, ranges, width, height, tx, bg[0], bg[1], bg[2],
                                                          alpha_low, term, pixels, load, stats, hist, bins);
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

}  // namespace adr
