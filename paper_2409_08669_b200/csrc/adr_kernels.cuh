// adr_kernels.cuh — host-side launchers shared between translation units.
#pragma once

#include "adr_common.cuh"

namespace adr {

// Render-side per-Gaussian record (indexed by Gaussian), 48 bytes.
//   a = (mx, my, conic_a, conic_b)
//   b = (conic_c, opacity, r, g)
//   c = (b, tau, hx, hy)   -- conservative culling parameters, see cull_params
struct __align__(16) Record {
    float4 a, b, c;
};

// Exact-safe culling parameters of one splat for the fp32 blend of
// sb/render.py:93-97 (alpha = min(sigma * exp_np(power), 0.99), skipped when
// alpha < alpha_low):
//   tau      : power < tau  =>  alpha < alpha_low.  exp_np is within 2 ulp of
//              exp and the product adds one rounding, so
//              ln(alpha_low / sigma) - 1e-5 (rounded down) is a strict bound;
//              it is raised to -87 (sigma < 1e30 makes alpha < alpha_low there
//              too), so every power the render evaluates lies in [-87, 0+].
//              Special values:
//                +inf : sigma <= 0 (or NaN) — the splat never contributes;
//                -inf : "slow" splat — no tau culling and the full exp_np:
//                       sigma >= 1e30 or non-finite, a colour non-finite, or
//                       a conic that is not positive definite and well
//                       conditioned (its fp32 power may exceed 88).
//   (hx, hy) : every pixel with |px - mx| > hx or |py - my| > hy has
//              power < tau *as computed in fp32*: the box of the ellipse
//              Q(d) <= -2 tau, inflated by s = sqrt((1 + 1e-4) / (1 - eta))
//              where eta bounds the relative fp32 evaluation error of power
//              (8 ulp * (max|a|,|c| + |b|/2) / lambda_min), plus 1e-3 px.
//              Slow splats get an infinite box (no culling).
// A contribution is only skipped when the reference provably skips it, so
// the image and load map stay bit-identical.
// ln_a_over_op: ln(alpha_low32 / op) when the caller already has it (the
// fused preprocess derives it from the extent's ln(sigma / alpha_low) plus a
// per-frame constant, within ~1e-7 — inside the 1e-5 margin, which is
// widened by 2e-7 on that path); >= 1e300: computed here.
#ifndef ADR_CULL_FAST
#define ADR_CULL_FAST 1
#endif
__device__ inline void cull_params(float a, float b, float c, float op, float alpha_low32, float c0, float c1,
                                   float c2, float* tau, float* hx, float* hy,
                                   double ln_a_over_op = 1e300) {
    const float kInf = __int_as_float(0x7f800000);
    if (!(op > 0.0f)) {
        *tau = kInf;
        *hx = *hy = 0.0f;
        return;
    }
    *tau = -kInf;
    *hx = *hy = kInf;
    if (!(op < 1e30f) || !isfinite(c0) || !isfinite(c1) || !isfinite(c2)) return;
    const double da = a, db = b, dc = c;
    const double det = da * dc - db * db;   // fp64: no cancellation loss for near-singular conics
    if (!(det > 0.0) || !(da > 0.0) || !(dc > 0.0)) return;
#if ADR_CULL_FAST
    // The bounds below need not be correctly rounded, only conservative: they
    // are evaluated in fp32 (a few ulp each) and every result that must not
    // be too small is enlarged by a relative 1e-5 / 2e-6 that covers those
    // errors many times over; the 1 + 1e-4 slack of s is left intact.
    const float det32 = (float)det;
    if (!(det32 > 0.0f)) return;   // fp32 underflow: slow splat (no culling)
    const float dh = 0.5f * (a - c);
    const float lmin = det32 / (0.5f * (a + c) + sqrtf(dh * dh + b * b));   // det / lambda_max
    if (!(lmin > 0.0f)) return;
    const float eta = (16.0f * 5.9604644775390625e-08f) * ((fmaxf(a, c) + 0.5f * fabsf(b)) / lmin) * 1.00001f;
    if (!(eta < 0.25f)) return;
#else
    const double half = 0.5 * (da + dc), rad = sqrt(0.25 * (da - dc) * (da - dc) + db * db);
    const double lmin = half - rad;
    if (!(lmin > 0.0)) return;
    const double M = (da > dc ? da : dc) + 0.5 * fabs(db);
    const double eta = 2.0 * 8.0 * 5.9604644775390625e-08 * M / lmin;
    if (!(eta < 0.25)) return;
#endif
    const double t = ln_a_over_op < 1e299 ? ln_a_over_op - 1.02e-5
                                                  : log((double)alpha_low32 / (double)op) - 1e-5;
    float t32 = __double2float_rd(t);
    t32 = t32 > -87.0f ? t32 : -87.0f;
    *tau = t32;
    const double K = -2.0 * (double)t32;
    if (K <= 0.0) {
        *hx = *hy = 1.0f;
        return;
    }
#if ADR_CULL_FAST
    const float s = sqrtf((1.0f + 1e-4f) / (1.0f - eta)) * 1.000002f;
    const float k_det = (float)K / det32;
    *hx = __fadd_ru(s * sqrtf(k_det * c), 1e-3f);
    *hy = __fadd_ru(s * sqrtf(k_det * a), 1e-3f);
#else
    const double s = sqrt((1.0 + 1e-4) / (1.0 - eta));
    *hx = __double2float_ru(s * sqrt(K * dc / det) + 1e-3);
    *hy = __double2float_ru(s * sqrt(K * da / det) + 1e-3);
#endif
}

// Extra per-Gaussian outputs the fused frame needs from stage 1.
struct FusedPre {
    Record* rec = nullptr;                    // render record (valid rows)
    uint2* gpack = nullptr;                   // tile rect (x0 | x1 << 16, y0 | y1 << 16)
    unsigned long long* culled = nullptr;     // += number of !valid rows
    uint32_t* dkey = nullptr;                 // depth-sort key (all-ones: no pairs)
    int64_t* d_m = nullptr;                   // += number of Gaussians with pairs (zeroed)
    unsigned long long* nan_colors = nullptr; // += valid rows with a NaN colour channel
    unsigned long long* ambiguous = nullptr;  // += ceil-ambiguous extents (log fence)
    uint32_t* kminmax = nullptr;              // per preprocess warp: min and max depth key of the selected rows
                                              // ([2 b] = min, [2 b + 1] = max; none: all-ones, 0)
    uint32_t* plan_mm = nullptr;              // the depth plan's (min, max), reset to (all-ones, 0) here
    bool rec_only = false;                    // mean2d / conic / opacity / color only in the record
    double ln_a32_a64 = 0.0;                  // ln((double)(float)alpha_low / alpha_low), for cull_params
    int32_t tiles_x = 0, tiles_y = 0;
};

int32_t launch_preprocess(const adr_scene& scene, const adr_camera& cam, int32_t mode,
                          double alpha_low, double dilation, const adr_projection& out,
                          const FusedPre* fused, cudaStream_t st);

// Stage 1 of several frames of one scene in one launch (adr_preprocess_views).
constexpr int kMaxBatchViews = 8;
struct PreViews {
    int32_t nv = 0;
    adr_camera cam[kMaxBatchViews];
    adr_projection out[kMaxBatchViews];
    FusedPre fused[kMaxBatchViews];
};
int32_t launch_preprocess_views(const adr_scene& scene, const PreViews& views, int32_t mode, double alpha_low,
                                double dilation, cudaStream_t st);

struct RenderArgs {
    const Record* rec;        // records
    const uint32_t* idx;      // per sorted pair: record index
    const int64_t* ranges;    // (n_tiles, 2) int64 spans
    uint32_t* order;          // scratch (n_tiles): tiles by decreasing span, or null
    int32_t width, height, tiles_x, tiles_y;
    float bg[3];
    float alpha_low;
    float term;
    float* pixels;
    int32_t* load;
    adr_load_stats* stats;    // may be null
    int32_t* hist;            // may be null
    int32_t hist_bins;
    const int64_t* nan_flag;  // device count of NaN-colour rows (null: always check poisoning)
};

int32_t launch_render(const RenderArgs& a, cudaStream_t st);
int32_t launch_render_proj(const adr_projection& p, const int64_t* gidx, const int64_t* ranges, int32_t width,
                           int32_t height, const float* bg, float alpha_low, float term, float* pixels,
                           int32_t* load, adr_load_stats* stats, int32_t* hist, int32_t bins, cudaStream_t st);
int32_t launch_init_stats(adr_load_stats* stats, int32_t* hist, int32_t bins, cudaStream_t st);

}  // namespace adr
