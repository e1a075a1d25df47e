/*
 * adr_oracle.c — CPU restatement of splatbench's forward rasterizer.
 *
 * TEST INFRASTRUCTURE ONLY (see adr_oracle.h).  Compiled with
 * -ffp-contract=off so every + - * / is one IEEE operation, exactly like a
 * numpy elementwise ufunc; FMAs appear only where the reference's BLAS calls
 * evaluate fused or inside numpy's float32 exp (A.2).
 *
 * Reference paths below are relative to /root/reference/pkg/src/splatbench/.
 */
#include "adr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TILE 16
#define PAIR_CHUNK 2048 /* render.py:36 _PAIR_CHUNK: the blend's frozen-break granularity */

/* numpy's float64 -> int32 astype on x86 (cvttsd2si): out-of-range and NaN
 * give INT32_MIN ("integer indefinite"), projection.py:419-420. */
static inline int32_t np_i32(double v) {
    return (v >= -2147483648.0 && v < 2147483648.0) ? (int32_t)v : INT32_MIN;
}

/* Culling extents are ceil(min(sqrt(2 s log_ratio), r_o)) (projection.py:
 * 387-396).  numpy's fp64 log and orc_log are both faithfully rounded, so
 * they differ by at most 2 ulp; that moves the sqrt by far less than
 * v * 2^-48.  An extent is "ceil-ambiguous" when the sqrt that min() can
 * select lies within that margin of a positive integer: only then can the
 * log's last bit change the output.  The count proves per frame that it
 * does not. */
int32_t orc_ceil_ambiguous(double v, double r_o) {
    if (!(v == v) || v > r_o * (1.0 + 0x1p-46) + 1e-300) return 0;
    const double m = nearbyint(v);
    return m >= 1.0 && fabs(v - m) <= v * 0x1p-48;
}

static int64_t g_ambiguous = 0;
int64_t orc_preprocess_ambiguous(void) { return g_ambiguous; }

/* ------------------------------------------------------------------------ */
/* numpy float32 exp (render.py:96 calls np.exp on f32). */
/* ------------------------------------------------------------------------ */

static inline float f_from_bits(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint32_t bits_from_f(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* v * 2^k with a single rounding (what AVX512 scalef / ldexpf produce). */
static inline float scale_pow2(float v, int k) {
    if (k > 127) return (v * 0x1p127f) * f_from_bits((uint32_t)(k - 127 + 127) << 23);
    if (k >= -126) return v * f_from_bits((uint32_t)(k + 127) << 23);
    return (v * f_from_bits((uint32_t)(k + 64 + 127) << 23)) * 0x1p-64f;
}

float orc_exp_np(float x) {
    if (x != x) return f_from_bits(0x7fc00000u);   /* numpy returns the canonical quiet NaN for every NaN */
    if (x > 88.72283935546875f) return INFINITY;
    if (x < -103.97208404541015625f) return 0.0f;
    float q = x * 1.442695040888963407359924681001892137f;
    q = (q + 0x1.8p23f) - 0x1.8p23f;                /* round to nearest int */
    float r = fmaf(q, -6.93145752e-1f, x);          /* Cody-Waite ln2 split */
    r = fmaf(q, -1.42860677e-6f, r);
    float num = fmaf(5.082762527590693718096e-04f, r, 6.757896990527504603057e-03f);
    num = fmaf(num, r, 5.114512081637298353406e-02f);
    num = fmaf(num, r, 2.473615434895520810817e-01f);
    num = fmaf(num, r, 7.257664613233124478488e-01f);
    num = fmaf(num, r, 9.999999999980870924916e-01f);
    float den = fmaf(2.159509375685829852307e-02f, r, -2.742335390411667452936e-01f);
    den = fmaf(den, r, 1.0f);
    return scale_pow2(num / den, (int)q);
}

/* ------------------------------------------------------------------------ */
/* fp64 log: the classic fdlibm argument reduction + Lg1..Lg7 polynomial,   */
/* written with plain IEEE ops so the CUDA kernel reproduces it bit for bit. */
/* The reference calls np.log (projection.py:389); its result only feeds      */
/* ceil(sqrt(...)) so sub-ulp differences from numpy never reach an output    */
/* in practice (checked against the goldens).                                */
/* ------------------------------------------------------------------------ */
double orc_log(double x) {
    const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
    const double Lg1 = 6.666666666666735130e-01, Lg2 = 3.999999999940941908e-01,
                 Lg3 = 2.857142874366239149e-01, Lg4 = 2.222219843214978396e-01,
                 Lg5 = 1.818357216161805012e-01, Lg6 = 1.531383769920937332e-01,
                 Lg7 = 1.479819860511658591e-01;
    uint64_t ux; memcpy(&ux, &x, 8);
    int32_t hx = (int32_t)(ux >> 32);
    uint32_t lx = (uint32_t)ux;
    int32_t k = 0;
    if (hx < 0x00100000) {
        if (((hx & 0x7fffffff) | lx) == 0) return -INFINITY;
        if (hx < 0) return NAN;
        k -= 54; x *= 1.80143985094819840000e+16;
        memcpy(&ux, &x, 8); hx = (int32_t)(ux >> 32);
    }
    if (hx >= 0x7ff00000) return x + x;
    k += (hx >> 20) - 1023;
    hx &= 0x000fffff;
    int32_t i = (hx + 0x95f64) & 0x100000;
    memcpy(&ux, &x, 8);
    ux = ((uint64_t)(uint32_t)(hx | (i ^ 0x3ff00000)) << 32) | (ux & 0xffffffffu);
    memcpy(&x, &ux, 8);
    k += (i >> 20);
    double f = x - 1.0;
    double dk;
    if ((0x000fffff & (2 + hx)) < 3) {
        if (f == 0.0) {
            if (k == 0) return 0.0;
            dk = (double)k; return dk * ln2_hi + dk * ln2_lo;
        }
        double R = f * f * (0.5 - 0.33333333333333333 * f);
        if (k == 0) return f - R;
        dk = (double)k; return dk * ln2_hi - ((R - dk * ln2_lo) - f);
    }
    double s = f / (2.0 + f);
    dk = (double)k;
    double z = s * s;
    i = hx - 0x6147a;
    double w = z * z;
    int32_t j = 0x6b851 - hx;
    double t1 = w * (Lg2 + w * (Lg4 + w * Lg6));
    double t2 = z * (Lg1 + w * (Lg3 + w * (Lg5 + w * Lg7)));
    i |= j;
    double R = t2 + t1;
    if (i > 0) {
        double hfsq = 0.5 * f * f;
        if (k == 0) return f - (hfsq - s * (hfsq + R));
        return dk * ln2_hi - ((hfsq - (s * (hfsq + R) + dk * ln2_lo)) - f);
    }
    if (k == 0) return f - s * (f - R);
    return dk * ln2_hi - ((s * (f - R) - dk * ln2_lo) - f);
}

/* numpy's NaN-propagating minimum/maximum (np.minimum / np.maximum). */
/* numpy's minimum / maximum (ties give the second operand, a NaN operand is
 * returned) and clip (v unless strictly outside [lo, hi]; NaN stays), as the
 * AVX-512 array loops behave, signed zeros included. */
static inline double np_min(double a, double b) { return (a < b || a != a) ? a : b; }
static inline double np_max(double a, double b) { return (a > b || a != a) ? a : b; }
static inline double np_clip(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* SH constants, projection.py:119-125. */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* projection.py:140-163, one channel; Python left-to-right precedence. */
static double sh_channel(const double* c /* (K,3) row-major */, int ch, int deg,
                         double x, double y, double z) {
#define C(k) c[(k) * 3 + ch]
    double r = SH_C0 * C(0);
    if (deg > 0) {
        r = ((r - (SH_C1 * y) * C(1)) + (SH_C1 * z) * C(2)) - (SH_C1 * x) * C(3);
        if (deg > 1) {
            double xx = x * x, yy = y * y, zz = z * z;
            double xy = x * y, yz = y * z, xz = x * z;
            r = r + (SH_C2[0] * xy) * C(4);
            r = r + (SH_C2[1] * yz) * C(5);
            r = r + (SH_C2[2] * ((2.0 * zz - xx) - yy)) * C(6);
            r = r + (SH_C2[3] * xz) * C(7);
            r = r + (SH_C2[4] * (xx - yy)) * C(8);
            if (deg > 2) {
                r = r + ((SH_C3[0] * y) * (3.0 * xx - yy)) * C(9);
                r = r + ((SH_C3[1] * xy) * z) * C(10);
                r = r + ((SH_C3[2] * y) * ((4.0 * zz - xx) - yy)) * C(11);
                r = r + ((SH_C3[3] * z) * ((2.0 * zz - 3.0 * xx) - 3.0 * yy)) * C(12);
                r = r + ((SH_C3[4] * x) * ((4.0 * zz - xx) - yy)) * C(13);
                r = r + ((SH_C3[5] * z) * (xx - yy)) * C(14);
                r = r + ((SH_C3[6] * x) * (xx - 3.0 * yy)) * C(15);
            }
        }
    }
#undef C
    return np_clip(r + 0.5, 0.0, 1.0);
}

/* projection.py:337-420 for a single row i. */
static void project_row(int64_t i, int32_t deg, const double* centers, const double* scales,
                        const double* rotations, const double* opacities, const double* sh,
                        const orc_camera* cam, int32_t mode, double alpha_low, double dilation,
                        uint8_t* valid, float* mean2d, float* cov2d, float* conic, float* depth_o,
                        float* color, float* opacity_o, float* lambda_max, int32_t* ext_x,
                        int32_t* ext_y) {
    const double* R = cam->rot;
    const double c0 = centers[3 * i], c1 = centers[3 * i + 1], c2 = centers[3 * i + 2];
    /* p_view = centers @ R.T + t (:342): OpenBLAS dgemm inner product order. */
    double pv[3];
    for (int k = 0; k < 3; ++k)
        pv[k] = fma(c2, R[3 * k + 2], fma(c1, R[3 * k + 1], c0 * R[3 * k + 0])) + cam->trans[k];
    const double depth = pv[2];
    int alive = depth > cam->near_plane;                                   /* :344 */

    /* quaternion_to_rotation (:170-184) and m = rot * scale (:348). */
    const double w = rotations[4 * i], x = rotations[4 * i + 1], y = rotations[4 * i + 2],
                 z = rotations[4 * i + 3];
    double rq[9];
    rq[0] = 1.0 - 2.0 * (y * y + z * z);
    rq[1] = 2.0 * (x * y - w * z);
    rq[2] = 2.0 * (x * z + w * y);
    rq[3] = 2.0 * (x * y + w * z);
    rq[4] = 1.0 - 2.0 * (x * x + z * z);
    rq[5] = 2.0 * (y * z - w * x);
    rq[6] = 2.0 * (x * z - w * y);
    rq[7] = 2.0 * (y * z + w * x);
    rq[8] = 1.0 - 2.0 * (x * x + y * y);
    double m[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) m[3 * a + b] = rq[3 * a + b] * scales[3 * i + b];
    /* cov3d = m @ m^T (:349), batched dgemm order. */
    double cov[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            cov[3 * a + b] = fma(m[3 * a + 2], m[3 * b + 2],
                                 fma(m[3 * a + 1], m[3 * b + 1], m[3 * a + 0] * m[3 * b + 0]));

    /* :351-372 */
    const double safe_z = alive ? depth : 1.0;
    const double inv_z = 1.0 / safe_z;
    const double tx = np_clip(pv[0] * inv_z, -cam->lim_x, cam->lim_x) * safe_z;
    const double ty = np_clip(pv[1] * inv_z, -cam->lim_y, cam->lim_y) * safe_z;
    const double j0 = cam->fx * inv_z;
    const double j2x = (((-cam->fx) * tx) * inv_z) * inv_z;
    const double j1 = cam->fy * inv_z;
    const double j2y = (((-cam->fy) * ty) * inv_z) * inv_z;
    double t0[3], t1[3];
    for (int k = 0; k < 3; ++k) {
        t0[k] = j0 * R[0 + k] + j2x * R[6 + k];
        t1[k] = j1 * R[3 + k] + j2y * R[6 + k];
    }
    /* c_t = cov3d @ t (:368-369): batched dgemv order. */
    double ct0[3], ct1[3];
    for (int a = 0; a < 3; ++a) {
        ct0[a] = fma(cov[3 * a + 2], t0[2], fma(cov[3 * a + 0], t0[0], cov[3 * a + 1] * t0[1]));
        ct1[a] = fma(cov[3 * a + 2], t1[2], fma(cov[3 * a + 0], t1[0], cov[3 * a + 1] * t1[1]));
    }
    const double sxx = ((t0[0] * ct0[0] + t0[1] * ct0[1]) + t0[2] * ct0[2]) + dilation;
    const double syy = ((t1[0] * ct1[0] + t1[1] * ct1[1]) + t1[2] * ct1[2]) + dilation;
    const double sxy = (t0[0] * ct1[0] + t0[1] * ct1[1]) + t0[2] * ct1[2];

    /* :374-397 */
    const double det = sxx * syy - sxy * sxy;
    const double mid = 0.5 * (sxx + syy);
    const double disc = sqrt(np_max(mid * mid - det, 0.0));
    const double lam_max = mid + disc;
    const double mx = ((cam->fx * pv[0]) * inv_z) + cam->cx;
    const double my = ((cam->fy * pv[1]) * inv_z) + cam->cy;
    const double r_o_real = 3.0 * sqrt(np_max(lam_max, 0.0));
    const double sigma = opacities[i];
    double ex, ey;
    if (mode == ORC_BASELINE) {
        ex = ceil(r_o_real);
        ey = ex;
    } else {
        alive = alive && (sigma > alpha_low);
        const double log_ratio = orc_log(np_max(sigma / alpha_low, 1e-300));
        int32_t amb = 0;
        if (mode == ORC_CIRCLE) {
            const double r_ad = sqrt((2.0 * lam_max) * log_ratio);
            ex = ceil(np_min(r_ad, r_o_real));
            ey = ex;
            amb = orc_ceil_ambiguous(r_ad, r_o_real);
        } else {
            const double vx = sqrt((2.0 * sxx) * log_ratio), vy = sqrt((2.0 * syy) * log_ratio);
            ex = ceil(np_min(vx, r_o_real));
            ey = ceil(np_min(vy, r_o_real));
            amb = orc_ceil_ambiguous(vx, r_o_real) + orc_ceil_ambiguous(vy, r_o_real);
        }
        if (alive && amb) {
#ifdef _OPENMP
#pragma omp atomic
#endif
            g_ambiguous += amb;
        }
    }
    alive = alive && (ex >= 1.0) && (ey >= 1.0);

    valid[i] = (uint8_t)alive;
    if (!alive) {
        mean2d[2 * i] = mean2d[2 * i + 1] = 0.0f;
        cov2d[3 * i] = cov2d[3 * i + 1] = cov2d[3 * i + 2] = 0.0f;
        conic[3 * i] = conic[3 * i + 1] = conic[3 * i + 2] = 0.0f;
        depth_o[i] = 0.0f;
        color[3 * i] = color[3 * i + 1] = color[3 * i + 2] = 0.0f;
        opacity_o[i] = 0.0f;
        lambda_max[i] = 0.0f;
        ext_x[i] = ext_y[i] = 0;
        return;
    }
    /* SH view direction (:399-402): dirs = (c - cam.center) / ||.|| */
    double d0 = c0 - cam->center[0], d1 = c1 - cam->center[1], d2 = c2 - cam->center[2];
    const double nrm = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
    const double dn = nrm > 0 ? nrm : 1.0;
    d0 = d0 / dn; d1 = d1 / dn; d2 = d2 / dn;
    const int64_t K = (int64_t)(deg + 1) * (deg + 1);
    const double* coeffs = sh + i * K * 3;

    /* :406-420 */
    mean2d[2 * i] = (float)mx;
    mean2d[2 * i + 1] = (float)my;
    cov2d[3 * i] = (float)sxx;
    cov2d[3 * i + 1] = (float)syy;
    cov2d[3 * i + 2] = (float)sxy;
    conic[3 * i] = (float)(syy / det);
    conic[3 * i + 1] = (float)(-sxy / det);
    conic[3 * i + 2] = (float)(sxx / det);
    depth_o[i] = (float)depth;
    for (int ch = 0; ch < 3; ++ch) color[3 * i + ch] = (float)sh_channel(coeffs, ch, deg, d0, d1, d2);
    opacity_o[i] = (float)sigma;
    lambda_max[i] = (float)lam_max;
    ext_x[i] = np_i32(ex);
    ext_y[i] = np_i32(ey);
}

void orc_preprocess(int64_t n, int32_t sh_degree, const double* centers, const double* scales,
                    const double* rotations, const double* opacities, const double* sh,
                    const orc_camera* cam, int32_t mode, double alpha_low, double dilation,
                    uint8_t* valid, float* mean2d, float* cov2d, float* conic, float* depth,
                    float* color, float* opacity, float* lambda_max, int32_t* ext_x,
                    int32_t* ext_y, int32_t nthreads) {
    g_ambiguous = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t i = 0; i < n; ++i)
        project_row(i, sh_degree, centers, scales, rotations, opacities, sh, cam, mode, alpha_low,
                    dilation, valid, mean2d, cov2d, conic, depth, color, opacity, lambda_max,
                    ext_x, ext_y);
    (void)nthreads;
}

/* tiling.py:77-99 — rectangle of one row, exact in fp64. */
static inline void tile_rect(float mx32, float my32, int32_t ex32, int32_t ey32, int v,
                             int32_t tiles_x, int32_t tiles_y, int64_t* x0, int64_t* x1,
                             int64_t* y0, int64_t* y1) {
    const double mx = mx32, my = my32, ex = ex32, ey = ey32;
    const double fx0 = np_clip(floor((mx - ex) / TILE), 0, tiles_x);
    const double fx1 = np_clip(floor((mx + ex) / TILE) + 1, 0, tiles_x);
    const double fy0 = np_clip(floor((my - ey) / TILE), 0, tiles_y);
    const double fy1 = np_clip(floor((my + ey) / TILE) + 1, 0, tiles_y);
    int64_t a0 = (int64_t)fx0, a1 = (int64_t)fx1, b0 = (int64_t)fy0, b1 = (int64_t)fy1;
    if (a1 < a0) a1 = a0;
    if (b1 < b0) b1 = b0;
    if (!v) { a1 = a0; b1 = b0; }
    *x0 = a0; *x1 = a1; *y0 = b0; *y1 = b1;
}

void orc_touched_counts(int64_t n, const float* mean2d, const int32_t* ext_x,
                        const int32_t* ext_y, const uint8_t* valid, int32_t tiles_x,
                        int32_t tiles_y, int64_t* counts) {
    for (int64_t i = 0; i < n; ++i) {
        int64_t x0, x1, y0, y1;
        tile_rect(mean2d[2 * i], mean2d[2 * i + 1], ext_x[i], ext_y[i], valid[i], tiles_x,
                  tiles_y, &x0, &x1, &y0, &y1);
        counts[i] = (x1 - x0) * (y1 - y0);
    }
}

int32_t orc_inclusive_sum(int64_t n, const int64_t* counts, int64_t* offsets) {
    int64_t acc = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (counts[i] > INT64_MAX - acc) return 1;
        acc += counts[i];
        offsets[i] = acc;
    }
    return 0;
}

void orc_duplicate_with_keys(int64_t n, const float* mean2d, const int32_t* ext_x,
                             const int32_t* ext_y, const uint8_t* valid, const float* depth,
                             const int64_t* offsets, int32_t tiles_x, int32_t tiles_y,
                             uint64_t* keys, int64_t* gidx) {
    for (int64_t g = 0; g < n; ++g) {
        int64_t x0, x1, y0, y1;
        tile_rect(mean2d[2 * g], mean2d[2 * g + 1], ext_x[g], ext_y[g], valid[g], tiles_x,
                  tiles_y, &x0, &x1, &y0, &y1);
        const int64_t cnt = (x1 - x0) * (y1 - y0);
        int64_t o = offsets[g] - cnt;
        const uint64_t dbits = bits_from_f(depth[g]);
        for (int64_t ty = y0; ty < y1; ++ty)
            for (int64_t tx = x0; tx < x1; ++tx) {
                keys[o] = ((uint64_t)(ty * tiles_x + tx) << 32) | dbits;
                gidx[o] = g;
                ++o;
            }
    }
}

void orc_sort_pairs(int64_t p, const uint64_t* keys, const int64_t* gidx, uint64_t* keys_out,
                    int64_t* gidx_out) {
    if (p <= 0) return;
    uint64_t kmax = 0;
    for (int64_t i = 0; i < p; ++i) kmax |= keys[i];
    uint64_t* ka = (uint64_t*)malloc((size_t)p * 8);
    int64_t* va = (int64_t*)malloc((size_t)p * 8);
    uint64_t* kb = (uint64_t*)malloc((size_t)p * 8);
    int64_t* vb = (int64_t*)malloc((size_t)p * 8);
    memcpy(ka, keys, (size_t)p * 8);
    memcpy(va, gidx, (size_t)p * 8);
    for (int shift = 0; shift < 64 && (kmax >> shift) != 0; shift += 8) {
        int64_t hist[257] = {0};
        for (int64_t i = 0; i < p; ++i) hist[((ka[i] >> shift) & 0xff) + 1]++;
        for (int d = 0; d < 256; ++d) hist[d + 1] += hist[d];
        for (int64_t i = 0; i < p; ++i) {
            const int64_t dst = hist[(ka[i] >> shift) & 0xff]++;
            kb[dst] = ka[i];
            vb[dst] = va[i];
        }
        uint64_t* tk = ka; ka = kb; kb = tk;
        int64_t* tv = va; va = vb; vb = tv;
    }
    memcpy(keys_out, ka, (size_t)p * 8);
    memcpy(gidx_out, va, (size_t)p * 8);
    free(ka); free(va); free(kb); free(vb);
}

int32_t orc_identify_tile_ranges(int64_t p, const uint64_t* sorted_keys, int64_t n_tiles,
                                 int64_t* ranges) {
    for (int64_t i = 1; i < p; ++i)
        if (sorted_keys[i] < sorted_keys[i - 1]) return 1;
    if (p > 0 && (int64_t)(sorted_keys[p - 1] >> 32) >= n_tiles) return 2;
    /* ranges[t] = (lower_bound(t), lower_bound(t+1)) over the tile ids. */
    int64_t k = 0;
    for (int64_t t = 0; t <= n_tiles; ++t) {
        while (k < p && (int64_t)(sorted_keys[k] >> 32) < t) ++k;
        if (t < n_tiles) ranges[2 * t] = k;
        if (t > 0) ranges[2 * (t - 1) + 1] = k;
    }
    return 0;
}

/* render.py:57-125 restated per pixel as the scalar recurrence the chunked
 * numpy kernel reproduces, and render.py:128-171.
 *
 * Per pixel, pair k of the tile's span (render.py:89-120):
 *   eff   = alpha >= alpha_low ? alpha : 0          (:96-97; NaN alpha -> 0)
 *   live  = T_before >= term                        (:104)
 *   C    += live ? (eff * T_before) * colour : 0    (:105-108)
 *   count+= live && eff > 0                         (:109)
 *   T     = T_before * (1 - eff)                    (:102, cumprod)
 *   the pixel freezes right after the first pair with T < term (:113-120).
 * With term <= 1 only contributing pairs change T, so this is the familiar
 * "composite, then stop once T < term".  With term > 1 no pair is ever live
 * and every pixel freezes at the span's first pair with T = 1 - eff(first);
 * with a NaN term nothing is live and nothing freezes.
 *
 * NaN colours (NaN SH coefficients pass np.clip, projection.py:163): the
 * reference adds weight * colour for EVERY pair of every processed chunk,
 * frozen or not, and 0 * NaN = NaN, so a NaN colour channel among the pairs
 * of the chunks the tile processes — up to the end of the 2048-pair chunk in
 * which its last pixel froze (frozen.all() break, :119-120), else the whole
 * span — turns that channel NaN for every pixel of the tile. */
void orc_render(int32_t width, int32_t height, int32_t tiles_x, int32_t tiles_y,
                const float* mean2d, const float* conic, const float* opacity,
                const float* color, const int64_t* gidx, const int64_t* ranges,
                const float* background, double alpha_low, double term_threshold,
                float* pixels, int32_t* counts, int32_t tile_stride, int32_t tile_phase,
                int32_t nthreads) {
    const float alpha_low32 = (float)alpha_low;
    const float term32 = (float)term_threshold;
    const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
    if (tile_stride < 1) tile_stride = 1;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t tile = tile_phase; tile < n_tiles; tile += tile_stride) {
        const int32_t ty = (int32_t)(tile / tiles_x), tx = (int32_t)(tile % tiles_x);
        const int32_t x0 = tx * TILE, y0 = ty * TILE;
        const int32_t x1 = x0 + TILE < width ? x0 + TILE : width;
        const int32_t y1 = y0 + TILE < height ? y0 + TILE : height;
        const int64_t start = ranges[2 * tile], end = ranges[2 * tile + 1];
        int all_frozen = 1;
        int64_t last_freeze = -1;
        for (int32_t py = y0; py < y1; ++py)
            for (int32_t px = x0; px < x1; ++px) {
                float T = 1.0f, C0 = 0.0f, C1 = 0.0f, C2 = 0.0f;
                int32_t cnt = 0;
                int64_t froze = -1;
                const float fpx = (float)px, fpy = (float)py;
                for (int64_t k = start; k < end; ++k) {
                    const int64_t g = gidx[k];
                    const float dx = fpx - mean2d[2 * g];
                    const float dy = fpy - mean2d[2 * g + 1];
                    const float a = conic[3 * g], b = conic[3 * g + 1], c = conic[3 * g + 2];
                    const float power = (-0.5f * ((a * dx) * dx + (c * dy) * dy)) - ((b * dx) * dy);
                    float alpha = opacity[g] * orc_exp_np(power);
                    alpha = (alpha != alpha) ? alpha : (alpha < 0.99f ? alpha : 0.99f);
                    const float eff = alpha >= alpha_low32 ? alpha : 0.0f;   /* :97 */
                    if (T >= term32 && eff > 0.0f) {                         /* :104-109 */
                        const float wgt = eff * T;
                        C0 = C0 + wgt * color[3 * g];
                        C1 = C1 + wgt * color[3 * g + 1];
                        C2 = C2 + wgt * color[3 * g + 2];
                        ++cnt;
                    }
                    T = T * (1.0f - eff);
                    if (T < term32) {                                        /* :113-120 */
                        froze = k - start;
                        break;
                    }
                }
                if (froze < 0) all_frozen = 0;
                else if (froze > last_freeze) last_freeze = froze;
                float* out = pixels + 3 * ((int64_t)py * width + px);
                float o0 = C0 + T * background[0], o1 = C1 + T * background[1],
                      o2 = C2 + T * background[2];
                out[0] = o0 < 0.0f ? 0.0f : (o0 > 1.0f ? 1.0f : o0);       /* :122-124 */
                out[1] = o1 < 0.0f ? 0.0f : (o1 > 1.0f ? 1.0f : o1);
                out[2] = o2 < 0.0f ? 0.0f : (o2 > 1.0f ? 1.0f : o2);
                counts[(int64_t)py * width + px] = cnt;
            }
        /* NaN-colour poisoning over the processed chunks */
        int64_t processed = end - start;
        if (all_frozen && last_freeze >= 0) {
            const int64_t chunk_end = (last_freeze / PAIR_CHUNK + 1) * PAIR_CHUNK;
            if (chunk_end < processed) processed = chunk_end;
        }
        int poison = 0;
        for (int64_t k = start; k < start + processed; ++k)
            for (int ch = 0; ch < 3; ++ch)
                if (color[3 * gidx[k] + ch] != color[3 * gidx[k] + ch]) poison |= 1 << ch;
        if (poison)
            for (int32_t py = y0; py < y1; ++py)
                for (int32_t px = x0; px < x1; ++px)
                    for (int ch = 0; ch < 3; ++ch)
                        if (poison >> ch & 1) pixels[3 * ((int64_t)py * width + px) + ch] = NAN;
    }
    (void)tiles_y;
    (void)nthreads;
}

/* Exhaustive pin of orc_exp_np (test infrastructure): over every float32 bit
 * pattern u in [lo, hi), H = sum of (y + 1) * (u * 0x9E3779B97F4A7C15 | 1)
 * mod 2^64 with y = the output bits (order-independent; any changed output
 * changes H).  tests/golden/make_exp_exhaustive.py computes the same sum over
 * numpy's own np.exp(float32). */
uint64_t orc_exp_checksum(uint64_t lo, uint64_t hi) {
    uint64_t total = 0;
#pragma omp parallel for reduction(+ : total) schedule(static)
    for (int64_t c = (int64_t)(lo >> 20); c < (int64_t)((hi + 0xfffff) >> 20); ++c) {
        uint64_t s = 0;
        const uint64_t a = (uint64_t)c << 20, b = ((uint64_t)c + 1) << 20;
        for (uint64_t u = a < lo ? lo : a; u < (b < hi ? b : hi); ++u) {
            float x;
            uint32_t ub = (uint32_t)u, yb;
            memcpy(&x, &ub, 4);
            const float y = orc_exp_np(x);
            memcpy(&yb, &y, 4);
            s += ((uint64_t)yb + 1u) * ((u * 0x9E3779B97F4A7C15ull) | 1u);
        }
        total += s;
    }
    return total;
}

/* ------------------------------------------------------------------------ */
/* float64 exp of the PLY loader (scene.py:385-386), test infrastructure.    */
/* numpy 2.3.5's np.exp(float64) on this AVX512_SKX host is Intel SVML's     */
/* __svml_exp8_ha (vendored in numpy); scipy's expit(x) is                    */
/* 1 / (1 + exp(-x)) with glibc 2.39's exp (its FMA variant).  Both are      */
/* restated operation by operation from the disassembly of those library     */
/* builds; the tables come from tools/gen_exp64_tables.py (first principles). */
/* ------------------------------------------------------------------------ */

#include "../paper_2409_08669_b200/csrc/adr_exp64_tab.h"

static const uint64_t k_s16_hi[16] = ADR_SVML16_HI;
static const uint64_t k_s16_lo[16] = ADR_SVML16_LO;
static const uint64_t k_s64[128] = ADR_SVML64_HILO;
static const uint64_t k_g128[256] = ADR_GLIBC128;

static inline double d_from_bits(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static inline uint64_t bits_from_d(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }

/* SVML's scalar path for |x| >= 0x1.61da04cbafe44p+9 and +-inf (plain SSE
 * arithmetic, no FMA): 2^(j/64) table, degree-5 polynomial, and a split
 * rounding for subnormal results. */
static double svml_exp_rare(double x) {
    const uint64_t ux = bits_from_d(x);
    if (((ux >> 52) & 0x7ff) == 0x7ff) return ux == 0xfff0000000000000ull ? 0.0 : x * x;
    if (x > 0x1.62e42fefa39efp+9) return 0x1.fffffffffffffp+1023 * 0x1.fffffffffffffp+1023;
    if (x < -0x1.74910d52d3051p+9) return 0x1.0000000000001p-1022 * 0x1.0000000000001p-1022;
    const double t1 = x * 0x1.71547652b82fep+6 + 0x1.8p52;   /* two roundings (no contraction) */
    const uint32_t n32 = (uint32_t)bits_from_d(t1);
    const uint32_t j = n32 & 63u, k = n32 >> 6;
    const double nf = t1 - 0x1.8p52;
    double r = x - nf * 0x1.62e42fefa0000p-7;
    r = r - nf * 0x1.cf79abc9e3b3ap-46;
    const double hi = d_from_bits(k_s64[2 * j]), lo = d_from_bits(k_s64[2 * j + 1]);
    double p = 0x1.6c16a1c2a3ffdp-10 * r + 0x1.111123aaf20d3p-7;
    p = p * r + 0x1.5555555558fccp-5;
    p = p * r + 0x1.55555555548f8p-3;
    p = p * r + 0x1.0p-1;
    p = p * r * r + r;
    p = (p + lo) * hi;
    if (!(x < -0x1.6232bdd7abcd2p+9)) {
        uint32_t e = (k + 0x3ffu) & 0x7ffu;
        const double y = p + hi;
        if (e > 0x7fe) {
            e = (e - 1) & 0x7ffu;
            return y * d_from_bits((uint64_t)e << 52) * 2.0;
        }
        return y * d_from_bits((uint64_t)e << 52);
    }
    const uint32_t e = (k + 0x43bu) & 0x7ffu;          /* scaled by 2^60 */
    const double sc = d_from_bits((uint64_t)e << 52);
    const double a = p * sc, b = sc * hi, s = b + a;
    if (e <= 0x32) return s * 0x1p-60;
    const double l = (b - s) + a;
    const double c = s * 0x1.8p32, h = (s + c) - c;
    const double el = l + (s - h);
    return h * 0x1p-60 + el * 0x1p-60;
}

/* np.exp(float64) = __svml_exp8_ha: z = RZ(x / ln2 + shifter) puts
 * floor16(x / ln2) and its 1/16 index in z's low bits; r = x - N ln2 (two
 * FMA steps); exp(r) by a degree-6 polynomial; result scaled by 2^floor(N). */
double orc_exp_svml(double x) {
    const double shifter = 0x1.8000000003ff0p+48;
    if (fabs(x) >= 0x1.61da04cbafe44p+9) return svml_exp_rare(x);
    double z = fma(x, 0x1.71547652b82fep+0, shifter);
    /* round toward zero (z > 0): step down when RN rounded up */
    if (fma(x, 0x1.71547652b82fep+0, -(z - shifter)) < 0.0) z = d_from_bits(bits_from_d(z) - 1);
    const uint32_t j = (uint32_t)(bits_from_d(z) & 15u);
    const double n = z - shifter;
    double r = fma(-n, 0x1.62e42fefa39efp-1, x);
    r = fma(-n, 0x1.abc9e3b39803fp-56, r);
    r = d_from_bits(bits_from_d(r) & 0xbfffffffffffffffull);
    const double r2 = r * r;
    double a = fma(0x1.7411836940c04p-10, r, 0x1.1101cbbc265c0p-7);
    const double b = fma(0x1.55557242d68fep-5, r, 0x1.5555553939732p-3);
    const double c = fma(0x1.000000000d008p-1, r, 0x1.fffffffffff70p-1);
    a = fma(r2, a, b);
    a = fma(r2, a, c);
    const double hi = d_from_bits(k_s16_hi[j]), lo = d_from_bits(k_s16_lo[j]);
    const double v = fma(a, r, lo);
    const double m = fma(hi, v, hi);
    return ldexp(m, (int)floor(n));   /* vscalefpd; normal for this range */
}

/* glibc 2.39 exp (sysdeps/ieee754/dbl-64/e_exp.c design, FMA build). */
double orc_exp_glibc(double x) {
    const uint64_t ux = bits_from_d(x);
    uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x3fu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x;
        if (abstop >= 0x409) {
            if (ux == 0xfff0000000000000ull) return 0.0;
            if (abstop == 0x7ff) return 1.0 + x;
            return (ux >> 63) ? 0x1p-767 * 0x1p-767 : 0x1p769 * 0x1p769;
        }
        abstop = 0;   /* |x| in [512, 1024): the scaled special case */
    }
    double kd = fma(x, 0x1.71547652b82fep+7, 0x1.8p52);
    const uint64_t ki = bits_from_d(kd);
    kd -= 0x1.8p52;
    double r = fma(kd, -0x1.62e42fefa0000p-8, x);
    r = fma(kd, -0x1.cf79abc9e3b3ap-47, r);
    const uint32_t idx = 2u * (uint32_t)(ki & 127u);
    const uint64_t top = ki << 45;
    const double tail = d_from_bits(k_g128[idx]);
    uint64_t sbits = k_g128[idx + 1] + top;
    const double a = fma(r, 0x1.555555555543cp-3, 0x1.ffffffffffdbdp-2);
    const double t = r + tail;
    const double r2 = r * r;
    const double b = fma(r, 0x1.1111167a4d017p-7, 0x1.55555cf172b91p-5);
    const double t2 = fma(a, r2, t);
    const double tmp = fma(r2 * r2, b, t2);
    if (abstop == 0) {
        if ((ki & 0x80000000ull) == 0) {
            sbits -= 1009ull << 52;
            const double scale = d_from_bits(sbits);
            return 0x1p1009 * fma(scale, tmp, scale);
        }
        sbits += 1022ull << 52;
        const double scale = d_from_bits(sbits);
        const double st = scale * tmp;
        double y = scale + st;
        if (y < 1.0) {
            const double lo = (scale - y) + st;
            const double hi = 1.0 + y;
            const double l2 = ((1.0 - hi) + y) + lo;
            y = (hi + l2) - 1.0;
            if (y == 0.0) y = 0.0;
        }
        return y * 0x1p-1022;
    }
    const double scale = d_from_bits(sbits);
    return fma(scale, tmp, scale);
}

/* scipy.special.expit(float64) (scene.py:385). */
double orc_expit(double x) { return 1.0 / (1.0 + orc_exp_glibc(-x)); }

/* Exhaustive pin over float32 inputs widened to float64 (a PLY stores
 * float32): H = sum over non-NaN bit patterns u in [lo, hi) of
 * (bits(f(u)) + 1) * (u * 0x9E3779B97F4A7C15 | 1) mod 2^64; kind 0 = np.exp,
 * 1 = expit.  tests/golden/make_exp64_exhaustive.py sums numpy / scipy. */
uint64_t orc_exp64_checksum(int32_t kind, uint64_t lo, uint64_t hi) {
    uint64_t total = 0;
#pragma omp parallel for reduction(+ : total) schedule(dynamic, 16)
    for (int64_t c = (int64_t)(lo >> 20); c < (int64_t)((hi + 0xfffff) >> 20); ++c) {
        uint64_t s = 0;
        const uint64_t a = (uint64_t)c << 20, b = ((uint64_t)c + 1) << 20;
        for (uint64_t u = a < lo ? lo : a; u < (b < hi ? b : hi); ++u) {
            const uint32_t ub = (uint32_t)u;
            if ((ub & 0x7fffffffu) > 0x7f800000u) continue;
            const double x = (double)f_from_bits(ub);
            const double y = kind == 0 ? orc_exp_svml(x) : orc_expit(x);
            s += (bits_from_d(y) + 1u) * ((u * 0x9E3779B97F4A7C15ull) | 1u);
        }
        total += s;
    }
    return total;
}
