// adr_render.cu — stage 6 (sb/render.py:57-171): per-tile front-to-back
// blending and the per-pixel load map, with the load-statistics epilogue
// (LoadStats / load_loss, sb/metrics.py:59-86).
//
// One CTA (128 threads) per 16x16 tile; each thread owns two horizontally
// adjacent pixels and evaluates them together in packed fp32x2 arithmetic
// (FADD2/FMUL2/FFMA2: two IEEE round-to-nearest ops per instruction, see
// adr_f32x2.cuh), which halves the issue slots of the exact blend.  Each batch
// of 256 pairs is gathered into shared memory; every pixel walks the batch in
// order with the exact fp32 recurrence of SURVEY.md App. A.3 (numpy float32
// exp, no FMA contraction), so the image and load map equal the reference bit
// for bit.
#include "adr_f32x2.cuh"
#include "adr_kernels.cuh"
#include "adr_scan.cuh"

#ifndef ADR_RENDER_MINB
#define ADR_RENDER_MINB 8
#endif

namespace adr {

// Self-check instantiation (k_render<Src, true>, selected at run time by
// adr_render_selfcheck): warp-iteration outcome counters of the blend loop,
// including every quad_mask removal that would have skipped a contributing
// pixel (must stay 0; tests/test_gpu_parity.py, tools/render_profile.py).
// The frame path launches the PROF = false instantiation, which has none of it.
__device__ unsigned long long g_render_prof[8];
#define RPROF(i, v)                          \
    do {                                     \
        if constexpr (PROF) rp[i] += (v);    \
    } while (0)

namespace {

constexpr int kRenderThreads = 128;       // 2 pixels per thread
#ifndef ADR_RBATCH
#define ADR_RBATCH 256
#endif
constexpr int kBatch = ADR_RBATCH;        // pairs staged per round

// Record source for the fused frame: records by rank + per-pair rank list.
struct RecSource {
    static constexpr int kMinBlocks = ADR_RENDER_MINB;   // 8: 64 registers (8 blocks/SM: +0.6% frames/s over 7, notes exp. 9)
    const Record* rec;
    const uint32_t* idx;
    __device__ __forceinline__ Record load(int64_t j) const { return rec[idx[j]]; }
    __device__ __forceinline__ uint32_t nan_bits(int64_t j) const {
        const float* r = reinterpret_cast<const float*>(rec + idx[j]);
        return (uint32_t)(r[6] != r[6]) | ((uint32_t)(r[7] != r[7]) << 1) | ((uint32_t)(r[8] != r[8]) << 2);
    }
};

// Record source for the stage API: Projection SoA + int64 Gaussian indices.
struct ProjSource {
    static constexpr int kMinBlocks = 6;   // the inline cull_params needs more registers
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
        const float c0 = color[3 * g], c1 = color[3 * g + 1], c2 = color[3 * g + 2];
        float tau, hx, hy;
        cull_params(a, b, c, op, alpha_low, c0, c1, c2, &tau, &hx, &hy);
        r.a = make_float4(m.x, m.y, a, b);
        r.b = make_float4(c, op, c0, c1);
        r.c = make_float4(c2, tau, hx, hy);
        return r;
    }
    __device__ __forceinline__ uint32_t nan_bits(int64_t j) const {
        const float* c = color + 3 * gidx[j];
        return (uint32_t)(c[0] != c[0]) | ((uint32_t)(c[1] != c[1]) << 1) | ((uint32_t)(c[2] != c[2]) << 2);
    }
};

constexpr int kPairChunk = 2048;   // sb/render.py:36 _PAIR_CHUNK (frozen-break granularity)

// NaN-colour poisoning (sb/render.py:106-108, 119-120): the reference adds
// weight * colour for EVERY pair of every chunk it processes, frozen pixel or
// not, and 0 * NaN = NaN, so a NaN colour channel among the pairs
// [start, processed_end) turns that channel NaN for every pixel of the tile.
// processed_end is the end of the 2048-pair chunk in which the tile's last
// pixel froze (frozen.all() break), or the span end.  Returns the 3 channel
// bits (block-uniform; every thread must call it).
template <class Src>
__device__ __forceinline__ uint32_t poison_bits(const Src& src, int64_t start, int64_t processed_end) {
    uint32_t bits = 0;
    for (int64_t j = start + threadIdx.x; j < processed_end; j += blockDim.x) bits |= src.nan_bits(j);
    return (uint32_t)(__syncthreads_or(bits & 1u) != 0) | ((uint32_t)(__syncthreads_or(bits & 2u) != 0) << 1) |
           ((uint32_t)(__syncthreads_or(bits & 4u) != 0) << 2);
}

// predicated increment (keeps the counter in place: no select + copy)
__device__ __forceinline__ void inc_if(int& c, bool p) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %1, 0;\n\t@q add.s32 %0, %0, 1;\n\t}" : "+r"(c) : "r"((int)p));
}

template <int kOff>
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+%5];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a), "n"(kOff));
    return v;
}
template <int kOff>
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2+%3];" : "=f"(v.x), "=f"(v.y) : "r"(a), "n"(kOff));
    return v;
}

// Warp w owns the 8x8 quadrant (qx, qy) = (w & 1, w >> 1) of the tile (a
// square footprint meets fewer small splats than a 4x16 strip): bit w of the
// mask is set when the splat's conservative box (mx +- hx, my +- hy) meets the
// quadrant's pixel columns and rows.
__device__ __forceinline__ uint32_t warp_mask(const Record& r, float x_lo, float y_lo) {
    // pixel centres are integers: only the integer columns ceil(l)..floor(r)
    // and rows ceil(t)..floor(b) of the box can contribute, so a box that
    // straddles no pixel centre of a quadrant (small splats between centres)
    // does not enter it (each pixel's own test is unchanged: px >= l <=>
    // px >= ceil(l) for integer px)
    const float mx = r.a.x, my = r.a.y, hx = r.c.z, hy = r.c.w;
    const float l = ceilf(mx - hx), rr = floorf(mx + hx), t = ceilf(my - hy), b = floorf(my + hy);
    if (!(l <= rr && t <= b)) return 0u;
    const uint32_t xm = (uint32_t)(l <= x_lo + 7.0f && rr >= x_lo) | ((uint32_t)(l <= x_lo + 15.0f && rr >= x_lo + 8.0f) << 1);
    const uint32_t ym = (uint32_t)(t <= y_lo + 7.0f && b >= y_lo) | ((uint32_t)(t <= y_lo + 15.0f && b >= y_lo + 8.0f) << 1);
    return (xm * ((ym & 1u) | ((ym & 2u) << 1)));  // bits: (qy,qx) = 0:(0,0) 1:(0,1) 2:(1,0) 3:(1,1)
}

// warp_mask refined by the tau-ellipse itself: for each 8-row band of the
// tile, the x-extent of the ellipse over the band's pixel rows (concave in y:
// the rightmost point if its row lies inside the band, otherwise the larger
// of the two band-end rows; leftmost alike), widened by a margin far above
// the evaluation error, decides which column halves can hold a
// contributing pixel.  The ellipse is Q(d) <= K' with K' = hx^2 det / c: the
// same inflated ellipse whose x half-extent is hx, so it contains every pixel
// whose fp32 power reaches tau (cull_params).  Slow splats keep the box.
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t quad_mask(const Record& r, float x_lo, float y_lo) {
    const uint32_t m = warp_mask(r, x_lo, y_lo);
    if (m == 0u || !(r.c.y > -3.0e38f)) return m;
    const float hx = r.c.z;
    // per-splat constants in fp64 (det cancels), then fp32: every fp32 error
    // below is a few ulp of aK or of the extents, far inside eps
    const double a = r.a.z, b = r.a.w, c = r.b.x;
    const double det64 = a * c - b * b;
    if (!(det64 > 0.0 && a > 0.0 && c > 0.0 && hx < 1e30f)) return m;
    const float det = (float)det64;
    const float aK = (float)(a * ((double)hx * (double)hx * det64 / c));
    const float dyr = (float)(-b * (double)hx / c);   // row offset of the rightmost point (leftmost: -dyr)
    const float ia = (float)(1.0 / a), bf = r.a.w;
    const float mx = r.a.x, my = r.a.y;
    const float eps = 1e-3f + 2e-3f * hx + 4e-6f * fabsf(mx);
    const float t = ceilf(my - r.c.w), bt = floorf(my + r.c.w);
    uint32_t out = 0u;
#pragma unroll
    for (int band = 0; band < 2; ++band) {
        const uint32_t bits = m & (3u << (2 * band));
        if (!bits) continue;
        const float d0 = fmaxf(y_lo + 8.0f * band, t) - my;
        const float d1 = fminf(y_lo + 8.0f * band + 7.0f, bt) - my;
        const float D0 = aK - det * d0 * d0, D1 = aK - det * d1 * d1;
        float xr = hx, xl = -hx;
        if (D0 >= 0.0f && D1 >= 0.0f) {
            const float s0 = sqrt_approx(D0), s1 = sqrt_approx(D1);
            if (!(dyr >= d0 && dyr <= d1)) xr = fmaxf(-bf * d0 + s0, -bf * d1 + s1) * ia;
            if (!(-dyr >= d0 && -dyr <= d1)) xl = fminf(-bf * d0 - s0, -bf * d1 - s1) * ia;
        }
        const float L = ceilf(mx + xl - eps), R = floorf(mx + xr + eps);
        if (!(L <= R)) continue;
        const uint32_t xm = (uint32_t)(L <= x_lo + 7.0f && R >= x_lo) | ((uint32_t)(L <= x_lo + 15.0f && R >= x_lo + 8.0f) << 1);
        out |= bits & (xm << (2 * band));
    }
    return out;
}

// One pixel's blend step with the full exp_np (slow splats).
__device__ __forceinline__ void blend_scalar(float fpx, float fpy, const float4& G, const float2& Tc, const float4& W,
                                             float alpha_low, float term, float& T, float& C0, float& C1, float& C2,
                                             int& cnt, bool& done) {
    if (done) return;
    const float dx = __fsub_rn(fpx, G.x);
    const float dy = __fsub_rn(fpy, G.y);
    const float q = __fadd_rn(__fmul_rn(__fmul_rn(G.z, dx), dx), __fmul_rn(__fmul_rn(Tc.x, dy), dy));
    const float power = __fsub_rn(__fmul_rn(-0.5f, q), __fmul_rn(__fmul_rn(G.w, dx), dy));
    if (power < Tc.y) return;
    const float e = (power >= -87.0f && power <= 88.0f) ? exp_np_fast(power) : exp_np(power);
    float alpha = __fmul_rn(W.x, e);
    alpha = alpha < 0.99f ? alpha : (alpha != alpha ? alpha : 0.99f);
    if (!(alpha >= alpha_low)) return;
    const float w = __fmul_rn(alpha, T);
    C0 = __fadd_rn(C0, __fmul_rn(w, W.y));
    C1 = __fadd_rn(C1, __fmul_rn(w, W.z));
    C2 = __fadd_rn(C2, __fmul_rn(w, W.w));
    T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
    ++cnt;
    if (T < term) done = true;
}

// term_threshold <= 1 (the render path of every frame): a pixel's "done"
// (frozen) state is implied by T itself — T starts at 1 >= term, only
// contributing blends change it and the reference tests T < term right after
// each of them (render.py:110-112).  term > 1 or NaN is k_render_unlit below.
// nan_flag: null = always check NaN-colour poisoning (stage API); otherwise
// only when *nan_flag != 0 (the fused frame's count of NaN-colour rows).
template <class Src, bool PROF = false>
__global__ void __launch_bounds__(kRenderThreads, Src::kMinBlocks)
k_render(Src src, const int64_t* __restrict__ ranges, int32_t width, int32_t height, int32_t tiles_x, float bg0,
         float bg1, float bg2, float alpha_low, float term, float* __restrict__ pixels, int32_t* __restrict__ load,
         adr_load_stats* stats, int32_t* hist, int32_t hist_bins, F2K K, const uint32_t* __restrict__ order,
         const int64_t* __restrict__ nan_flag) {
    // shared-memory batch, split by use: the power test needs (mx, my, a, b)
    // + (c, tau); only splats that pass it read (sigma, r, g, b)
    // batch arrays at a 16-byte stride, one array after the other, so one
    // address register per splat reaches all three (immediate offsets)
    __shared__ __align__(16) float4 sB[3 * kBatch];   // G: mx, my, a, b | W: sigma, r, g, b | T: c, tau
    float4* const sG = sB;
    float4* const sW = sB + kBatch;
    float4* const sT = sB + 2 * kBatch;
    __shared__ uint8_t smask[kBatch];
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(sB);
    __shared__ unsigned long long ssum[kRenderThreads / 32], ssq[kRenderThreads / 32];
    __shared__ int smin[kRenderThreads / 32], smax[kRenderThreads / 32];
    const int tile = order ? (int)order[blockIdx.x] : (int)blockIdx.x;
    const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px0 = tx * kTile + 8 * (warp & 1) + 2 * (lane & 3);
    const int py = ty * kTile + 8 * (warp >> 1) + (lane >> 2);
    const bool in0 = px0 < width && py < height, in1 = px0 + 1 < width && py < height;
    const int64_t start = ranges[2 * tile], end = ranges[2 * tile + 1];
    const float fpx0 = (float)px0, fpx1 = (float)(px0 + 1), fpy = (float)py;
    const f2 PX = pk(fpx0, fpx1);
    const float x_lo = (float)(tx * kTile), y_lo = (float)(ty * kTile);

    // pixels outside the image start done (T = 0 in the implied mode: they
    // are never written)
    f2 T = pk(in0 ? 1.0f : 0.0f, in1 ? 1.0f : 0.0f), C0 = 0ull, C1 = 0ull, C2 = 0ull;
    int cnt0 = 0, cnt1 = 0;
    unsigned long long rp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define DONE0 (lo_of(T) < term)
#define DONE1 (hi_of(T) < term)
    int64_t stop = end;   // first batch at whose start every pixel was done
    for (int64_t b = start; b < end; b += kBatch) {
        if (__syncthreads_count(DONE0 && DONE1) == kRenderThreads) {
            stop = b;
            break;
        }
        const int nb = (int)((end - b) < kBatch ? (end - b) : kBatch);
        for (int i = threadIdx.x; i < nb; i += kRenderThreads) {
            const Record r = src.load(b + i);
            sG[i] = r.a;
            sT[i] = make_float4(r.b.x, r.c.y, 0.f, 0.f);
            sW[i] = make_float4(r.b.y, r.b.z, r.b.w, r.c.x);
            if constexpr (PROF)
                smask[i] = (uint8_t)(quad_mask(r, x_lo, y_lo) | (warp_mask(r, x_lo, y_lo) << 4));
            else
                smask[i] = (uint8_t)quad_mask(r, x_lo, y_lo);
        }
        __syncthreads();
        RPROF(6, 1);
        if (__any_sync(kFull, !(DONE0 && DONE1))) {
            for (int c0 = 0; c0 < nb; c0 += 32) {
                // PROF: iterate the plain box (bits 4-7) and remember the quadrant mask
                const uint32_t qm = __ballot_sync(kFull, c0 + lane < nb && ((smask[c0 + lane] >> warp) & 1u));
                uint32_t m = PROF ? __ballot_sync(kFull, c0 + lane < nb && ((smask[c0 + lane] >> (4 + warp)) & 1u))
                                  : qm;
                while (m) {
                    const int j = c0 + __ffs(m) - 1;
                    m &= m - 1u;
                    RPROF(0, 1);
                    RPROF(3, (unsigned)!DONE0 + (unsigned)!DONE1);
                    const uint32_t sa = s_base + 16u * j;
                    const float4 G = lds_f4<0>(sa);
                    const float2 Tc = lds_f2<2 * 16 * kBatch>(sa);
                    const float tau = Tc.y;
                    if (tau < -3.0e38f) {  // slow splat: full exp_np, scalar per pixel
                        const float4 W = lds_f4<16 * kBatch>(sa);
                        float t0 = lo_of(T), t1 = hi_of(T);
                        float a0 = lo_of(C0), a1 = hi_of(C0), b0 = lo_of(C1), b1 = hi_of(C1);
                        float d0 = lo_of(C2), d1 = hi_of(C2);
                        bool d0f = DONE0, d1f = DONE1;
                        blend_scalar(fpx0, fpy, G, Tc, W, alpha_low, term, t0, a0, b0, d0, cnt0, d0f);
                        blend_scalar(fpx1, fpy, G, Tc, W, alpha_low, term, t1, a1, b1, d1, cnt1, d1f);
                        T = pk(t0, t1);
                        C0 = pk(a0, a1);
                        C1 = pk(b0, b1);
                        C2 = pk(d0, d1);
                        continue;
                    }
                    // power = (-0.5 * ((a*dx)*dx + (c*dy)*dy)) - ((b*dx)*dy), both lanes
                    const float dy = __fsub_rn(fpy, G.y);
                    const float cdd = __fmul_rn(__fmul_rn(Tc.x, dy), dy);
                    const f2 dx = sub2(PX, bc(G.x), K);
                    const f2 q = add2(mul2(mul2(bc(G.z), dx, K), dx, K), bc(cdd), K);
                    const f2 bd = mul2(mul2(bc(G.w), dx, K), bc(dy), K);
                    const f2 pw = sub2(mul2(bc(-0.5f), q, K), bd, K);
                    bool p0 = !DONE0 && lo_of(pw) >= tau;
                    bool p1 = !DONE1 && hi_of(pw) >= tau;
                    RPROF(4, (unsigned)p0 + (unsigned)p1);
                    RPROF(1, __all_sync(kFull, !(p0 || p1)));
                    RPROF(7, __all_sync(kFull, !(p0 || p1)) && __all_sync(kFull, !DONE0 && !DONE1));
                    if constexpr (PROF) {
                        // slot 2: iterations quad_mask removes; slot 6 += 1e9 per unsafe removal
                        if (!((qm >> (j - c0)) & 1u)) {
                            RPROF(2, lane == 0);
                            if (__any_sync(kFull, p0 || p1) && lane == 0) rp[6] += 1000000000ull;
                        }
                    }
                    if (!(p0 || p1)) continue;  // both alphas < alpha_low for sure
                    const float4 W = lds_f4<16 * kBatch>(sa);
                    const f2 al = mul2(bc(W.x), exp2_np_fast(pw, K), K);
                    float a0 = fminf(lo_of(al), 0.99f), a1 = fminf(hi_of(al), 0.99f);  // finite here
                    p0 = p0 && a0 >= alpha_low;
                    p1 = p1 && a1 >= alpha_low;
                    RPROF(5, (unsigned)p0 + (unsigned)p1);
                    if (!(p0 || p1)) continue;
                    // a lane that does not contribute blends alpha = 0 — an exact
                    // no-op (T * 1 = T, C + 0 * colour = C for finite colours),
                    // which is also what the reference does (render.py:98-109)
                    const f2 A = pk(p0 ? a0 : 0.0f, p1 ? a1 : 0.0f);
                    const f2 w = mul2(A, T, K);
                    C0 = add2(C0, mul2(w, bc(W.y), K), K);
                    C1 = add2(C1, mul2(w, bc(W.z), K), K);
                    C2 = add2(C2, mul2(w, bc(W.w), K), K);
                    T = mul2(T, sub2(K.one, A, K), K);
                    inc_if(cnt0, p0);
                    inc_if(cnt1, p1);
                }
                if (__all_sync(kFull, DONE0 && DONE1)) break;
            }
        }
    }
#undef DONE0
#undef DONE1
    if constexpr (PROF) {
        // per-warp events (0, 1, 2, 6) counted once per warp; per-pixel sums (3, 4, 5) summed over lanes
        for (int k = 0; k < 8; ++k) {
            unsigned long long v = rp[k];
            if (k == 3 || k == 4 || k == 5)
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane == 0) atomicAdd(&g_render_prof[k], v);
        }
    }
    uint32_t poison = 0;
    if (!nan_flag || *nan_flag != 0) {
        // every pixel was done at the start of batch `stop`, not at the start
        // of the batch before: the last freeze lies in [stop - kBatch, stop)
        int64_t pe = end;
        if (stop < end) {
            const int64_t rel = stop - kBatch - start > 0 ? stop - kBatch - start : 0;
            const int64_t ce = start + (rel / kPairChunk + 1) * kPairChunk;
            pe = ce < end ? ce : end;
        }
        poison = poison_bits(src, start, pe);
    }
    const float t0 = lo_of(T), t1 = hi_of(T);
    const float o[2][3] = {{__fadd_rn(lo_of(C0), __fmul_rn(t0, bg0)), __fadd_rn(lo_of(C1), __fmul_rn(t0, bg1)),
                            __fadd_rn(lo_of(C2), __fmul_rn(t0, bg2))},
                           {__fadd_rn(hi_of(C0), __fmul_rn(t1, bg0)), __fadd_rn(hi_of(C1), __fmul_rn(t1, bg1)),
                            __fadd_rn(hi_of(C2), __fmul_rn(t1, bg2))}};
    const bool ins[2] = {in0, in1};
    const int cnts[2] = {cnt0, cnt1};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (!ins[k]) continue;
        const int64_t pix = (int64_t)py * width + px0 + k;
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const float v = o[k][ch];
            pixels[3 * pix + ch] = (poison >> ch) & 1u ? __int_as_float(0x7fc00000) : (v < 0.f ? 0.f : (v > 1.f ? 1.f : v));
        }
        load[pix] = cnts[k];
        if (hist) atomicAdd(hist + (cnts[k] < hist_bins ? cnts[k] : hist_bins - 1), 1);
    }
    if (stats) {
        unsigned long long s = (in0 ? (unsigned long long)cnt0 : 0ull) + (in1 ? (unsigned long long)cnt1 : 0ull);
        unsigned long long s2 = (in0 ? (unsigned long long)cnt0 * (unsigned long long)cnt0 : 0ull) +
                                (in1 ? (unsigned long long)cnt1 * (unsigned long long)cnt1 : 0ull);
        int mn = INT_MAX, mx = INT_MIN;
        if (in0) {
            mn = min(mn, cnt0);
            mx = max(mx, cnt0);
        }
        if (in1) {
            mn = min(mn, cnt1);
            mx = max(mx, cnt1);
        }
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) {
            s += __shfl_xor_sync(kFull, s, o2);
            s2 += __shfl_xor_sync(kFull, s2, o2);
            mn = min(mn, __shfl_xor_sync(kFull, mn, o2));
            mx = max(mx, __shfl_xor_sync(kFull, mx, o2));
        }
        if (lane == 0) {
            ssum[warp] = s;
            ssq[warp] = s2;
            smin[warp] = mn;
            smax[warp] = mx;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < kRenderThreads / 32; ++k) {
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

// term_threshold > 1 or NaN (sb/render.py:100-120 taken literally): no pair
// is ever live (T_before = 1 < term, or any comparison with NaN), so nothing
// is composited and no count accrues.  With term > 1 every pixel freezes at
// the span's first pair with T = 1 - eff(first pair); with a NaN term nothing
// freezes and T = prod(1 - eff) over the whole span.  Output T * bg (C = 0),
// plus NaN-colour poisoning over the processed chunks.  One thread per pixel.
template <class Src>
__global__ void __launch_bounds__(kTilePixels)
k_render_unlit(Src src, const int64_t* __restrict__ ranges, int32_t width, int32_t height, int32_t tiles_x,
               float bg0, float bg1, float bg2, float alpha_low, float term, float* __restrict__ pixels,
               int32_t* __restrict__ load, adr_load_stats* stats, int32_t* hist, int32_t hist_bins,
               const int64_t* __restrict__ nan_flag) {
    const int tile = blockIdx.x;
    const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
    const int px = tx * kTile + (threadIdx.x & (kTile - 1)), py = ty * kTile + (threadIdx.x >> 4);
    const bool in = px < width && py < height;
    const int64_t start = ranges[2 * tile], end = ranges[2 * tile + 1];
    const bool first_only = term > 1.0f;
    const int64_t last = first_only ? (start < end ? start + 1 : start) : end;
    const float fpx = (float)px, fpy = (float)py;
    float T = 1.0f;
    for (int64_t j = start; j < last; ++j) {
        const Record r = src.load(j);
        const float dx = __fsub_rn(fpx, r.a.x), dy = __fsub_rn(fpy, r.a.y);
        const float q = __fadd_rn(__fmul_rn(__fmul_rn(r.a.z, dx), dx), __fmul_rn(__fmul_rn(r.b.x, dy), dy));
        const float power = __fsub_rn(__fmul_rn(-0.5f, q), __fmul_rn(__fmul_rn(r.a.w, dx), dy));
        float alpha = __fmul_rn(r.b.y, exp_np(power));
        alpha = alpha < 0.99f ? alpha : (alpha != alpha ? alpha : 0.99f);
        T = __fmul_rn(T, __fsub_rn(1.0f, alpha >= alpha_low ? alpha : 0.0f));
    }
    uint32_t poison = 0;
    if (!nan_flag || *nan_flag != 0) {
        const int64_t ce = start + kPairChunk;
        poison = poison_bits(src, start, first_only && ce < end ? ce : end);
    }
    if (in) {
        const int64_t pix = (int64_t)py * width + px;
        const float bg[3] = {bg0, bg1, bg2};
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const float v = __fadd_rn(0.0f, __fmul_rn(T, bg[ch]));
            pixels[3 * pix + ch] = (poison >> ch) & 1u ? __int_as_float(0x7fc00000) : (v < 0.f ? 0.f : (v > 1.f ? 1.f : v));
        }
        load[pix] = 0;
    }
    const int n_in = __syncthreads_count(in);
    if (threadIdx.x == 0 && n_in > 0) {
        if (stats) {
            atomicMin(&stats->min, 0);
            atomicMax(&stats->max, 0);
        }
        if (hist && hist_bins > 0) atomicAdd(hist, n_in);
    }
}

// Longest-span-first launch order of the tiles (LPT scheduling): tiles are
// bucketed by floor(log2(span + 1)), heaviest bucket first, so the heavy
// tiles of the image centre start in the first wave instead of forming the
// tail.  Order within a bucket is arbitrary; every tile's output depends only
// on its own span, so results are unaffected.
__global__ void __launch_bounds__(1024) k_tile_order(const int64_t* __restrict__ ranges, int32_t n_tiles,
                                                     uint32_t* __restrict__ order) {
    __shared__ uint32_t cnt[64], pos[64];
    if (threadIdx.x < 64) cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
        const uint64_t len = (uint64_t)(ranges[2 * t + 1] - ranges[2 * t]);
        atomicAdd(&cnt[__clzll(len + 1)], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int k = 0; k < 64; ++k) {
            pos[k] = s;
            s += cnt[k];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
        const uint64_t len = (uint64_t)(ranges[2 * t + 1] - ranges[2 * t]);
        order[atomicAdd(&pos[__clzll(len + 1)], 1u)] = (uint32_t)t;
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

static int g_render_selfcheck = 0;

int32_t launch_render(const RenderArgs& a, cudaStream_t st) {
    const int64_t n_tiles = (int64_t)a.tiles_x * a.tiles_y;
    if (n_tiles <= 0) return ADR_OK;
    RecSource src{a.rec, a.idx};
    if (!(a.term <= 1.0f)) {
        k_render_unlit<RecSource><<<n_tiles, kTilePixels, 0, st>>>(src, a.ranges, a.width, a.height, a.tiles_x,
                                                                   a.bg[0], a.bg[1], a.bg[2], a.alpha_low, a.term,
                                                                   a.pixels, a.load, a.stats, a.hist, a.hist_bins,
                                                                   a.nan_flag);
        ADR_LAUNCH_CHECK();
        return ADR_OK;
    }
    if (a.order) {
        k_tile_order<<<1, 1024, 0, st>>>(a.ranges, (int32_t)n_tiles, a.order);
        ADR_LAUNCH_CHECK();
    }
    auto kern = g_render_selfcheck ? k_render<RecSource, true> : k_render<RecSource, false>;
    kern<<<n_tiles, kRenderThreads, 0, st>>>(src, a.ranges, a.width, a.height, a.tiles_x, a.bg[0], a.bg[1], a.bg[2],
                                             a.alpha_low, a.term, a.pixels, a.load, a.stats, a.hist, a.hist_bins,
                                             f2k_host(), a.order, a.nan_flag);
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
    if (!(term <= 1.0f)) {
        k_render_unlit<ProjSource><<<n_tiles, kTilePixels, 0, st>>>(src, ranges, width, height, tx, bg[0], bg[1],
                                                                    bg[2], alpha_low, term, pixels, load, stats,
                                                                    hist, bins, nullptr);
    } else {
        k_render<ProjSource><<<n_tiles, kRenderThreads, 0, st>>>(src, ranges, width, height, tx, bg[0], bg[1], bg[2],
                                                                 alpha_low, term, pixels, load, stats, hist, bins,
                                                                 f2k_host(), nullptr, nullptr);
    }
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

}  // namespace adr

extern "C" int32_t adr_render_selfcheck(int32_t enable, unsigned long long* host_out) {
    // counters: [0] warp iterations, [1] iterations with no pixel passing tau,
    // [2] iterations quad_mask removed, [3] live pixel visits, [4] pixels passing
    // tau, [5] contributing pixels, [6] batches + 1e9 x unsafe quad_mask removals,
    // [7] all-fail iterations with no done pixel
    if (host_out) {
        ADR_CUDA_TRY(cudaDeviceSynchronize());
        ADR_CUDA_TRY(cudaMemcpyFromSymbol(host_out, adr::g_render_prof, sizeof(unsigned long long) * 8));
    }
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    ADR_CUDA_TRY(cudaMemcpyToSymbol(adr::g_render_prof, z, sizeof(z)));
    adr::g_render_selfcheck = enable ? 1 : 0;
    return ADR_OK;
}
