// adr_exp64.cuh — the float64 exponentials of the reference's PLY loader
// (sb/scene.py:385-386), bit-exact on the device:
//   exp_svml : numpy 2.3.5's np.exp(float64) on an AVX512_SKX host, which is
//              Intel SVML's __svml_exp8_ha (vendored in numpy);
//   expit_glibc : scipy.special.expit(float64) = 1 / (1 + exp(-x)) with
//              glibc 2.39's exp (the FMA build of sysdeps/ieee754/dbl-64/e_exp.c).
// Operation by operation as those library builds evaluate (every step an
// explicit IEEE intrinsic, so nvcc cannot contract or reorder), with the
// 2^(k/N) tables from tools/gen_exp64_tables.py.  Pinned exhaustively over
// all float32 inputs (a PLY stores float32) by tests/golden/exp64_exhaustive.json.
#pragma once

#include <cstdint>

#include "adr_exp64_tab.h"

namespace adr {

static __device__ const uint64_t g_s16_hi[16] = ADR_SVML16_HI;
static __device__ const uint64_t g_s16_lo[16] = ADR_SVML16_LO;
static __device__ const uint64_t g_s64[128] = ADR_SVML64_HILO;
static __device__ const uint64_t g_g128[256] = ADR_GLIBC128;

__device__ __forceinline__ double dbits(uint64_t u) { return __longlong_as_double((long long)u); }
__device__ __forceinline__ uint64_t ubits(double d) { return (uint64_t)__double_as_longlong(d); }

// SVML's scalar special-case path (|x| >= 0x1.61da04cbafe44p+9, +-inf): plain
// SSE arithmetic (no FMA), 2^(j/64) table, split rounding for subnormals.
static __device__ __noinline__ double exp_svml_rare(double x) {
    const uint64_t ux = ubits(x);
    if (((ux >> 52) & 0x7ff) == 0x7ff) return ux == 0xfff0000000000000ull ? 0.0 : __dmul_rn(x, x);
    if (x > 0x1.62e42fefa39efp+9) return dbits(0x7ff0000000000000ull);   // DBL_MAX^2
    if (x < -0x1.74910d52d3051p+9) return 0.0;                           // (2^-1022)^2
    const double t1 = __dadd_rn(__dmul_rn(x, 0x1.71547652b82fep+6), 0x1.8p52);
    const uint32_t n32 = (uint32_t)ubits(t1);
    const uint32_t j = n32 & 63u, k = n32 >> 6;
    const double nf = __dsub_rn(t1, 0x1.8p52);
    double r = __dsub_rn(x, __dmul_rn(nf, 0x1.62e42fefa0000p-7));
    r = __dsub_rn(r, __dmul_rn(nf, 0x1.cf79abc9e3b3ap-46));
    const double hi = dbits(g_s64[2 * j]), lo = dbits(g_s64[2 * j + 1]);
    double p = __dadd_rn(__dmul_rn(0x1.6c16a1c2a3ffdp-10, r), 0x1.111123aaf20d3p-7);
    p = __dadd_rn(__dmul_rn(p, r), 0x1.5555555558fccp-5);
    p = __dadd_rn(__dmul_rn(p, r), 0x1.55555555548f8p-3);
    p = __dadd_rn(__dmul_rn(p, r), 0x1.0p-1);
    p = __dadd_rn(__dmul_rn(__dmul_rn(p, r), r), r);
    p = __dmul_rn(__dadd_rn(p, lo), hi);
    if (!(x < -0x1.6232bdd7abcd2p+9)) {
        uint32_t e = (k + 0x3ffu) & 0x7ffu;
        const double y = __dadd_rn(p, hi);
        if (e > 0x7fe) {
            e = (e - 1) & 0x7ffu;
            return __dmul_rn(__dmul_rn(y, dbits((uint64_t)e << 52)), 2.0);
        }
        return __dmul_rn(y, dbits((uint64_t)e << 52));
    }
    const uint32_t e = (k + 0x43bu) & 0x7ffu;   // scaled by 2^60
    const double sc = dbits((uint64_t)e << 52);
    const double a = __dmul_rn(p, sc), b = __dmul_rn(sc, hi), s = __dadd_rn(b, a);
    if (e <= 0x32) return __dmul_rn(s, 0x1p-60);
    const double l = __dadd_rn(__dsub_rn(b, s), a);
    const double c = __dmul_rn(s, 0x1.8p32), h = __dsub_rn(__dadd_rn(s, c), c);
    const double el = __dadd_rn(l, __dsub_rn(s, h));
    return __dadd_rn(__dmul_rn(h, 0x1p-60), __dmul_rn(el, 0x1p-60));
}

// np.exp(float64): z = RZ(x / ln2 + shifter) holds floor16(x / ln2) and its
// 1/16 index; r = x - N ln2 in two FMA steps; degree-6 polynomial; scaled by
// 2^floor(N) (vscalefpd; the result is normal on this path).
__device__ __forceinline__ double exp_svml(double x) {
    const double shifter = 0x1.8000000003ff0p+48;
    if (fabs(x) >= 0x1.61da04cbafe44p+9) return exp_svml_rare(x);
    const double z = __fma_rz(x, 0x1.71547652b82fep+0, shifter);
    const uint32_t j = (uint32_t)(ubits(z) & 15u);
    const double n = __dsub_rn(z, shifter);
    double r = __fma_rn(-n, 0x1.62e42fefa39efp-1, x);
    r = __fma_rn(-n, 0x1.abc9e3b39803fp-56, r);
    r = dbits(ubits(r) & 0xbfffffffffffffffull);
    const double r2 = __dmul_rn(r, r);
    double a = __fma_rn(0x1.7411836940c04p-10, r, 0x1.1101cbbc265c0p-7);
    const double b = __fma_rn(0x1.55557242d68fep-5, r, 0x1.5555553939732p-3);
    const double c = __fma_rn(0x1.000000000d008p-1, r, 0x1.fffffffffff70p-1);
    a = __fma_rn(r2, a, b);
    a = __fma_rn(r2, a, c);
    const double hi = dbits(__ldg(reinterpret_cast<const unsigned long long*>(g_s16_hi) + j));
    const double lo = dbits(__ldg(reinterpret_cast<const unsigned long long*>(g_s16_lo) + j));
    const double m = __fma_rn(hi, __fma_rn(a, r, lo), hi);
    const int kf = (int)floor(n);   // in [-1022, 1021]
    return __dmul_rn(m, dbits((uint64_t)(kf + 1023) << 52));
}

// glibc 2.39 exp, FMA build.
__device__ __forceinline__ double exp_glibc(double x) {
    const uint64_t ux = ubits(x);
    uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x3fu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) return __dadd_rn(1.0, x);
        if (abstop >= 0x409) {
            if (ux == 0xfff0000000000000ull) return 0.0;
            if (abstop == 0x7ff) return __dadd_rn(1.0, x);
            return (ux >> 63) ? 0.0 : dbits(0x7ff0000000000000ull);
        }
        abstop = 0;   // |x| in [512, 1024): scaled special case
    }
    double kd = __fma_rn(x, 0x1.71547652b82fep+7, 0x1.8p52);
    const uint64_t ki = ubits(kd);
    kd = __dsub_rn(kd, 0x1.8p52);
    double r = __fma_rn(kd, -0x1.62e42fefa0000p-8, x);
    r = __fma_rn(kd, -0x1.cf79abc9e3b3ap-47, r);
    const uint32_t idx = 2u * (uint32_t)(ki & 127u);
    const double tail = dbits(__ldg(reinterpret_cast<const unsigned long long*>(g_g128) + idx));
    uint64_t sbits = __ldg(reinterpret_cast<const unsigned long long*>(g_g128) + idx + 1) + (ki << 45);
    const double a = __fma_rn(r, 0x1.555555555543cp-3, 0x1.ffffffffffdbdp-2);
    const double t = __dadd_rn(r, tail);
    const double r2 = __dmul_rn(r, r);
    const double b = __fma_rn(r, 0x1.1111167a4d017p-7, 0x1.55555cf172b91p-5);
    const double tmp = __fma_rn(__dmul_rn(r2, r2), b, __fma_rn(a, r2, t));
    if (abstop == 0) {
        if ((ki & 0x80000000ull) == 0) {
            const double scale = dbits(sbits - (1009ull << 52));
            return __dmul_rn(0x1p1009, __fma_rn(scale, tmp, scale));
        }
        const double scale = dbits(sbits + (1022ull << 52));
        const double st = __dmul_rn(scale, tmp);
        double y = __dadd_rn(scale, st);
        if (y < 1.0) {
            const double lo = __dadd_rn(__dsub_rn(scale, y), st);
            const double hi = __dadd_rn(1.0, y);
            const double l2 = __dadd_rn(__dadd_rn(__dsub_rn(1.0, hi), y), lo);
            y = __dsub_rn(__dadd_rn(hi, l2), 1.0);
            if (y == 0.0) y = 0.0;
        }
        return __dmul_rn(y, 0x1p-1022);
    }
    const double scale = dbits(sbits);
    return __fma_rn(scale, tmp, scale);
}

__device__ __forceinline__ double expit_glibc(double x) {
    return __ddiv_rn(1.0, __dadd_rn(1.0, exp_glibc(-x)));
}

}  // namespace adr
