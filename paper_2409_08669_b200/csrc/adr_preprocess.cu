// adr_preprocess.cu — stage 1 (sb/projection.py:291-420), one thread per
// Gaussian, fp64 math in the reference's evaluation order.
//
// Bit-exactness notes:
//  * numpy elementwise ops → one IEEE op each (explicit __d*_rn intrinsics);
//  * p_view = centers @ R.T + t and cov3d = m @ m^T → OpenBLAS dgemm order
//    fma(c2,R2, fma(c1,R1, c0*R0)) (+ t);
//  * c_t = cov3d @ t (batched dgemv) → fma(cov2,t2, fma(cov0,t0, cov1*t1));
//  * np.sum over 3 terms → (a+b)+c; outputs rounded fp64→fp32 (RN).
#include "adr_kernels.cuh"

#ifndef PRE_BLOCKS_PER_SM
#define PRE_BLOCKS_PER_SM 0
#endif
#include "adr_scan.cuh"

namespace adr {

namespace {

__device__ __constant__ double kShC0 = 0.28209479177387814;
__device__ __constant__ double kShC1 = 0.4886025119029199;
__device__ __constant__ double kShC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                           -1.0925484305920792, 0.5462742152960396};
__device__ __constant__ double kShC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                           0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                           -0.5900435899266435};

#define MUL __dmul_rn
#define ADD __dadd_rn
#define SUB __dsub_rn
#define FMA __fma_rn

// sb/projection.py:140-163 for one channel (Python left-to-right order).
template <int DEG>
__device__ __forceinline__ double sh_channel(const double* c, double x, double y, double z) {
    double r = MUL(kShC0, c[0]);
    if (DEG > 0) {
        r = SUB(ADD(SUB(r, MUL(MUL(kShC1, y), c[1])), MUL(MUL(kShC1, z), c[2])), MUL(MUL(kShC1, x), c[3]));
    }
    if (DEG > 1) {
        const double xx = MUL(x, x), yy = MUL(y, y), zz = MUL(z, z);
        const double xy = MUL(x, y), yz = MUL(y, z), xz = MUL(x, z);
        r = ADD(r, MUL(MUL(kShC2[0], xy), c[4]));
        r = ADD(r, MUL(MUL(kShC2[1], yz), c[5]));
        r = ADD(r, MUL(MUL(kShC2[2], SUB(SUB(MUL(2.0, zz), xx), yy)), c[6]));
        r = ADD(r, MUL(MUL(kShC2[3], xz), c[7]));
        r = ADD(r, MUL(MUL(kShC2[4], SUB(xx, yy)), c[8]));
        if (DEG > 2) {
            r = ADD(r, MUL(MUL(MUL(kShC3[0], y), SUB(MUL(3.0, xx), yy)), c[9]));
            r = ADD(r, MUL(MUL(MUL(kShC3[1], xy), z), c[10]));
            r = ADD(r, MUL(MUL(MUL(kShC3[2], y), SUB(SUB(MUL(4.0, zz), xx), yy)), c[11]));
            r = ADD(r, MUL(MUL(MUL(kShC3[3], z), SUB(SUB(MUL(2.0, zz), MUL(3.0, xx)), MUL(3.0, yy))), c[12]));
            r = ADD(r, MUL(MUL(MUL(kShC3[4], x), SUB(SUB(MUL(4.0, zz), xx), yy)), c[13]));
            r = ADD(r, MUL(MUL(MUL(kShC3[5], z), SUB(xx, yy)), c[14]));
            r = ADD(r, MUL(MUL(MUL(kShC3[6], x), SUB(xx, MUL(3.0, yy))), c[15]));
        }
    }
    return np_clip(ADD(r, 0.5), 0.0, 1.0);
}

constexpr int kPreBlock = 128;
// Fused frames may cap the preprocess grid at kPreBlocksPerSm blocks per SM
// (grid-stride); measured no better than the full grid (notes.md, exp. 8).
constexpr int kPreBlocksPerSm = PRE_BLOCKS_PER_SM;   // fused frames: resident blocks per SM (0: one per 128 Gaussians)

// SH coefficients of the block's Gaussians are staged through shared memory:
// one coalesced pass over the block's contiguous (128, K, 3) slab, stored with
// an odd per-Gaussian stride (K*3 + 1 elements) so the per-thread reads of its
// own coefficients are bank-conflict free.
template <typename T, int DEG>
__device__ __forceinline__ void stage_sh(const T* __restrict__ sh, int64_t first, int count, T* stage) {
    constexpr int K3 = (DEG + 1) * (DEG + 1) * 3;
    constexpr int S = K3 + 1;
    const T* src = sh + first * K3;
    const int total = count * K3;
    if constexpr (sizeof(T) == 4 && K3 % 4 == 0) {
        if (count == kPreBlock && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
            // all K3/4 vector loads of this thread in flight before any store
            constexpr int kVec = K3 / 4;
            const float4* s4 = reinterpret_cast<const float4*>(src);
            float4 v[kVec];
#pragma unroll
            for (int u = 0; u < kVec; ++u) v[u] = __ldg(s4 + threadIdx.x + u * kPreBlock);
#pragma unroll
            for (int u = 0; u < kVec; ++u) {
                const int f = 4 * (threadIdx.x + u * kPreBlock), g = f / K3, j = f - g * K3;
                float* d = reinterpret_cast<float*>(stage) + g * S + j;
                d[0] = v[u].x;
                d[1] = v[u].y;
                d[2] = v[u].z;
                d[3] = v[u].w;
            }
            return;
        }
    }
    for (int f = threadIdx.x; f < total; f += kPreBlock) {
        const int g = f / K3, j = f - g * K3;
        stage[g * S + j] = src[f];
    }
}

// A Gaussian's view-independent terms (sb/projection.py:337-372 before the
// camera enters): the row's centre, cov3d = M Mᵀ with M = R(q)·diag(s) (six
// unique entries: fma/mul are commutative, so cov[a][b] == cov[b][a] bit for
// bit), sigma and ln(sigma / alpha_low) (not evaluated in BASELINE mode).
struct PreRow {
    double c[3];
    double cov[6];   // xx, xy, xz, yy, yz, zz
    double sigma;
    double log_ratio;
};

__device__ __forceinline__ double cov_at(const PreRow& g, int a, int b) {
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    return g.cov[lo == 0 ? hi : (lo == 1 ? 2 + hi : 5)];
}

template <typename T>
__device__ __forceinline__ void pre_row(PreRow& g, const T ac[3], const T as[3], const T aq[4], T aop,
                                        int32_t mode, double alpha_low) {
    g.c[0] = (double)ac[0];
    g.c[1] = (double)ac[1];
    g.c[2] = (double)ac[2];
    const double w = (double)aq[0], x = (double)aq[1], y = (double)aq[2], z = (double)aq[3];
    double rq[9];
    rq[0] = SUB(1.0, MUL(2.0, ADD(MUL(y, y), MUL(z, z))));
    rq[1] = MUL(2.0, SUB(MUL(x, y), MUL(w, z)));
    rq[2] = MUL(2.0, ADD(MUL(x, z), MUL(w, y)));
    rq[3] = MUL(2.0, ADD(MUL(x, y), MUL(w, z)));
    rq[4] = SUB(1.0, MUL(2.0, ADD(MUL(x, x), MUL(z, z))));
    rq[5] = MUL(2.0, SUB(MUL(y, z), MUL(w, x)));
    rq[6] = MUL(2.0, SUB(MUL(x, z), MUL(w, y)));
    rq[7] = MUL(2.0, ADD(MUL(y, z), MUL(w, x)));
    rq[8] = SUB(1.0, MUL(2.0, ADD(MUL(x, x), MUL(y, y))));
    const double s0 = (double)as[0], s1 = (double)as[1], s2 = (double)as[2];
    double m[9];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        m[3 * a + 0] = MUL(rq[3 * a + 0], s0);
        m[3 * a + 1] = MUL(rq[3 * a + 1], s1);
        m[3 * a + 2] = MUL(rq[3 * a + 2], s2);
    }
    int u = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = a; b < 3; ++b)
            g.cov[u++] = FMA(m[3 * a + 2], m[3 * b + 2], FMA(m[3 * a + 1], m[3 * b + 1], MUL(m[3 * a], m[3 * b])));
    g.sigma = (double)aop;
    g.log_ratio = mode == ADR_MODE_BASELINE ? 0.0 : log_fd(np_max(__ddiv_rn(g.sigma, alpha_low), 1e-300));
}

// One view of one Gaussian row (k_preprocess_views; k_preprocess keeps its
// own single-view body, which ptxas schedules without spills at the 72-register
// budget): everything after the camera enters
// (sb/projection.py:355-420), the fused frame's extras (sb/tiling.py:77-114)
// and the warp's fused epilogue (no block barrier: warps of a block run their
// views independently).
template <typename T, int DEG, bool FUSED>
__device__ __forceinline__ void preprocess_view(const PreRow& g, bool in_range, int64_t i, const T* shp,
                                                const adr_camera& cam, int32_t mode, double alpha_low,
                                                double dilation, const adr_projection& out, const FusedPre& fused,
                                                int64_t blk) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    bool alive = false;
    bool selected = false;   // fused: touches >= 1 tile
    uint32_t dbits = 0;      // fused: float32 depth bits
    int ambiguous = 0;       // fused: ceil-ambiguous extents of this row (log fence)
    bool nan_color = false;  // fused: a valid row with a NaN colour channel
    if (in_range) {
        const double* R = cam.rot;
        const double c0 = g.c[0], c1 = g.c[1], c2 = g.c[2];
        double pv[3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
            pv[k] = ADD(FMA(c2, R[3 * k + 2], FMA(c1, R[3 * k + 1], MUL(c0, R[3 * k + 0]))), cam.trans[k]);
        const double depth = pv[2];
        alive = depth > cam.near_plane;

        const double safe_z = alive ? depth : 1.0;
        const double inv_z = __ddiv_rn(1.0, safe_z);
        const double tx = MUL(np_clip(MUL(pv[0], inv_z), -cam.lim_x, cam.lim_x), safe_z);
        const double ty = MUL(np_clip(MUL(pv[1], inv_z), -cam.lim_y, cam.lim_y), safe_z);
        const double j0 = MUL(cam.fx, inv_z);
        const double j2x = MUL(MUL(MUL(-cam.fx, tx), inv_z), inv_z);
        const double j1 = MUL(cam.fy, inv_z);
        const double j2y = MUL(MUL(MUL(-cam.fy, ty), inv_z), inv_z);
        double t0[3], t1[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            t0[k] = ADD(MUL(j0, R[k]), MUL(j2x, R[6 + k]));
            t1[k] = ADD(MUL(j1, R[3 + k]), MUL(j2y, R[6 + k]));
        }
        double ct0[3], ct1[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            ct0[a] = FMA(cov_at(g, a, 2), t0[2], FMA(cov_at(g, a, 0), t0[0], MUL(cov_at(g, a, 1), t0[1])));
            ct1[a] = FMA(cov_at(g, a, 2), t1[2], FMA(cov_at(g, a, 0), t1[0], MUL(cov_at(g, a, 1), t1[1])));
        }
        const double sxx = ADD(ADD(ADD(MUL(t0[0], ct0[0]), MUL(t0[1], ct0[1])), MUL(t0[2], ct0[2])), dilation);
        const double syy = ADD(ADD(ADD(MUL(t1[0], ct1[0]), MUL(t1[1], ct1[1])), MUL(t1[2], ct1[2])), dilation);
        const double sxy = ADD(ADD(MUL(t0[0], ct1[0]), MUL(t0[1], ct1[1])), MUL(t0[2], ct1[2]));

        const double det = SUB(MUL(sxx, syy), MUL(sxy, sxy));
        const double mid = MUL(0.5, ADD(sxx, syy));
        const double disc = __dsqrt_rn(np_max(SUB(MUL(mid, mid), det), 0.0));
        const double lam_max = ADD(mid, disc);
        const double mx = ADD(MUL(MUL(cam.fx, pv[0]), inv_z), cam.cx);
        const double my = ADD(MUL(MUL(cam.fy, pv[1]), inv_z), cam.cy);
        const double r_o_real = MUL(3.0, __dsqrt_rn(np_max(lam_max, 0.0)));
        const double sigma = g.sigma;
        double ex, ey;
        double ln_a_over_op = 1e300;   // for cull_params (fused); 1e300: not known

        if (mode == ADR_MODE_BASELINE) {
            ex = ceil(r_o_real);
            ey = ex;
        } else {
            alive = alive && (sigma > alpha_low);
            const double log_ratio = g.log_ratio;
            if (FUSED) ln_a_over_op = fused.ln_a32_a64 - log_ratio;   // = ln(a32 / sigma)
            if (mode == ADR_MODE_CIRCLE) {
                const double v = __dsqrt_rn(MUL(MUL(2.0, lam_max), log_ratio));
                ex = ceil(np_min(v, r_o_real));
                ey = ex;
                if (FUSED && alive) ambiguous = ceil_ambiguous(v, r_o_real);
            } else {
                const double vx = __dsqrt_rn(MUL(MUL(2.0, sxx), log_ratio));
                const double vy = __dsqrt_rn(MUL(MUL(2.0, syy), log_ratio));
                ex = ceil(np_min(vx, r_o_real));
                ey = ceil(np_min(vy, r_o_real));
                if (FUSED && alive) ambiguous = ceil_ambiguous(vx, r_o_real) + ceil_ambiguous(vy, r_o_real);
            }
        }
        alive = alive && (ex >= 1.0) && (ey >= 1.0);

        out.d_valid[i] = (uint8_t)alive;
        if (alive) {
            double d0 = SUB(c0, cam.center[0]), d1 = SUB(c1, cam.center[1]), d2 = SUB(c2, cam.center[2]);
            const double nrm = __dsqrt_rn(ADD(ADD(MUL(d0, d0), MUL(d1, d1)), MUL(d2, d2)));
            const double dn = nrm > 0 ? nrm : 1.0;
            d0 = __ddiv_rn(d0, dn);
            d1 = __ddiv_rn(d1, dn);
            d2 = __ddiv_rn(d2, dn);
            double col[3];
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                double cf[K];
#pragma unroll
                for (int k = 0; k < K; ++k) cf[k] = (double)shp[k * 3 + ch];
                col[ch] = sh_channel<DEG>(cf, d0, d1, d2);
            }
            const float2 m2 = make_float2(__double2float_rn(mx), __double2float_rn(my));
            const float ca = __double2float_rn(__ddiv_rn(syy, det));
            const float cb = __double2float_rn(__ddiv_rn(-sxy, det));
            const float cc = __double2float_rn(__ddiv_rn(sxx, det));
            const float dz = __double2float_rn(depth);
            const float op = __double2float_rn(sigma);
            const float c0f = __double2float_rn(col[0]), c1f = __double2float_rn(col[1]),
                        c2f = __double2float_rn(col[2]);
            if (!(FUSED && fused.rec_only)) {   // else these live in the render record only
                reinterpret_cast<float2*>(out.d_mean2d)[i] = m2;
                out.d_conic[3 * i] = ca;
                out.d_conic[3 * i + 1] = cb;
                out.d_conic[3 * i + 2] = cc;
                out.d_color[3 * i] = c0f;
                out.d_color[3 * i + 1] = c1f;
                out.d_color[3 * i + 2] = c2f;
                out.d_opacity[i] = op;
            }
            out.d_cov2d[3 * i] = __double2float_rn(sxx);
            out.d_cov2d[3 * i + 1] = __double2float_rn(syy);
            out.d_cov2d[3 * i + 2] = __double2float_rn(sxy);
            out.d_depth[i] = dz;
            out.d_lambda_max[i] = __double2float_rn(lam_max);
            const int32_t ix = np_i32(ex), iy = np_i32(ey);
            out.d_ext_x[i] = ix;
            out.d_ext_y[i] = iy;
            if (FUSED) {
                nan_color = c0f != c0f || c1f != c1f || c2f != c2f;
                const Rect r = tile_rect(m2.x, m2.y, ix, iy, true, fused.tiles_x, fused.tiles_y);
                selected = r.count() > 0;
                dbits = __float_as_uint(dz);
                Record R;
                float tau, hx, hy;
                cull_params(ca, cb, cc, op, (float)alpha_low, c0f, c1f, c2f, &tau, &hx, &hy, ln_a_over_op);
                R.a = make_float4(m2.x, m2.y, ca, cb);
                R.b = make_float4(cc, op, c0f, c1f);
                R.c = make_float4(c2f, tau, hx, hy);
                fused.rec[i] = R;
                fused.gpack[i] = make_uint2((uint32_t)r.x0 | ((uint32_t)r.x1 << 16),
                                            (uint32_t)r.y0 | ((uint32_t)r.y1 << 16));
            }
        } else {
            if (FUSED && fused.rec_only) {
                const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                Record R;
                R.a = R.b = R.c = z;
                fused.rec[i] = R;
            } else {
                reinterpret_cast<float2*>(out.d_mean2d)[i] = make_float2(0.f, 0.f);
                out.d_conic[3 * i] = out.d_conic[3 * i + 1] = out.d_conic[3 * i + 2] = 0.f;
                out.d_color[3 * i] = out.d_color[3 * i + 1] = out.d_color[3 * i + 2] = 0.f;
                out.d_opacity[i] = 0.f;
            }
            out.d_cov2d[3 * i] = out.d_cov2d[3 * i + 1] = out.d_cov2d[3 * i + 2] = 0.f;
            out.d_depth[i] = 0.f;
            out.d_lambda_max[i] = 0.f;
            out.d_ext_x[i] = 0;
            out.d_ext_y[i] = 0;
        }
    }
    if (FUSED) {
        // depth-sort key: float32 depth bits for Gaussians touching >= 1
        // tile (depth > near_plane > 0, so bit 31 is clear), all-ones for the
        // rest, which a stable sort then leaves behind the M selected ones
        if (in_range) fused.dkey[i] = selected ? dbits : 0xffffffffu;
        const int lane = threadIdx.x & 31;
        const uint32_t culled = __ballot_sync(kFull, in_range && !alive);
        const uint32_t sb = __ballot_sync(kFull, selected);
        const uint32_t nanb = __ballot_sync(kFull, nan_color);
        if (__any_sync(kFull, ambiguous != 0)) {
            const int amb = __reduce_add_sync(kFull, (unsigned)ambiguous);
            if (lane == 0 && fused.ambiguous) atomicAdd(fused.ambiguous, (unsigned long long)amb);
        }
        if (fused.kminmax) {   // the depth sort's key-range plan (adr_supertile.cu): per-warp extrema
            const uint32_t kmn = __reduce_min_sync(kFull, selected ? dbits : 0xffffffffu);
            const uint32_t kmx = __reduce_max_sync(kFull, selected ? dbits : 0u);
            if (threadIdx.x == 0 && blk == 0 && fused.plan_mm) {
                fused.plan_mm[0] = 0xffffffffu;
                fused.plan_mm[1] = 0u;
            }
            if (lane == 0)
                reinterpret_cast<uint2*>(fused.kminmax)[blk * (kPreBlock / 32) + (threadIdx.x >> 5)] =
                    make_uint2(kmn, kmx);
        }
        if (lane == 0) {
            if (culled) atomicAdd(fused.culled, (unsigned long long)__popc(culled));
            if (sb) atomicAdd(reinterpret_cast<unsigned long long*>(fused.d_m), (unsigned long long)__popc(sb));
            if (nanb && fused.nan_colors) atomicAdd(fused.nan_colors, (unsigned long long)__popc(nanb));
        }
    }
}


// Loads one block's rows: per-Gaussian attributes, then the SH slab staged
// into shared memory (the caller synchronises before reading the stage).
template <typename T, int DEG>
__device__ __forceinline__ void load_block(const T* __restrict__ centers, const T* __restrict__ scales,
                                           const T* __restrict__ rotations, const T* __restrict__ opacities,
                                           const T* __restrict__ sh, int64_t n, int64_t first, T* stage,
                                           T ac[3], T as[3], T aq[4], T& aop) {
    const int64_t i = first + threadIdx.x;
    if (i < n) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            ac[k] = centers[3 * i + k];
            as[k] = scales[3 * i + k];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) aq[k] = rotations[4 * i + k];
        aop = opacities[i];
    }
    stage_sh<T, DEG>(sh, first, (int)(n - first < kPreBlock ? n - first : kPreBlock), stage);
}

template <typename T, int DEG, bool FUSED>
__device__ __forceinline__ void preprocess_block(const T* __restrict__ centers, const T* __restrict__ scales,
                                                 const T* __restrict__ rotations, const T* __restrict__ opacities,
                                                 const T* __restrict__ sh, int64_t n, const adr_camera& cam,
                                                 int32_t mode, double alpha_low, double dilation,
                                                 const adr_projection& out, const FusedPre& fused, int64_t blk) {
    constexpr int K = (DEG + 1) * (DEG + 1);
    constexpr int S = K * 3 + 1;
    extern __shared__ __align__(16) unsigned char pre_smem[];
    T* stage = reinterpret_cast<T*>(pre_smem);
    const int64_t first = blk * kPreBlock;
    const int64_t i = first + threadIdx.x;
    // per-Gaussian attributes first, so their latency overlaps the SH staging
    T ac[3] = {T(0), T(0), T(0)}, as[3] = {T(0), T(0), T(0)}, aq[4] = {T(0), T(0), T(0), T(0)}, aop = T(0);
    if (i < n) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            ac[k] = centers[3 * i + k];
            as[k] = scales[3 * i + k];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) aq[k] = rotations[4 * i + k];
        aop = opacities[i];
    }
    stage_sh<T, DEG>(sh, first, (int)(n - first < kPreBlock ? n - first : kPreBlock), stage);
    __syncthreads();
    bool alive = false;
    bool selected = false;   // fused: touches >= 1 tile
    uint32_t dbits = 0;      // fused: float32 depth bits
    int ambiguous = 0;       // fused: ceil-ambiguous extents of this row (log fence)
    bool nan_color = false;  // fused: a valid row with a NaN colour channel
    if (i < n) {
        const double* R = cam.rot;
        const double c0 = (double)ac[0], c1 = (double)ac[1], c2 = (double)ac[2];
        double pv[3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
            pv[k] = ADD(FMA(c2, R[3 * k + 2], FMA(c1, R[3 * k + 1], MUL(c0, R[3 * k + 0]))), cam.trans[k]);
        const double depth = pv[2];
        alive = depth > cam.near_plane;

        const double w = (double)aq[0], x = (double)aq[1], y = (double)aq[2], z = (double)aq[3];
        double rq[9];
        rq[0] = SUB(1.0, MUL(2.0, ADD(MUL(y, y), MUL(z, z))));
        rq[1] = MUL(2.0, SUB(MUL(x, y), MUL(w, z)));
        rq[2] = MUL(2.0, ADD(MUL(x, z), MUL(w, y)));
        rq[3] = MUL(2.0, ADD(MUL(x, y), MUL(w, z)));
        rq[4] = SUB(1.0, MUL(2.0, ADD(MUL(x, x), MUL(z, z))));
        rq[5] = MUL(2.0, SUB(MUL(y, z), MUL(w, x)));
        rq[6] = MUL(2.0, SUB(MUL(x, z), MUL(w, y)));
        rq[7] = MUL(2.0, ADD(MUL(y, z), MUL(w, x)));
        rq[8] = SUB(1.0, MUL(2.0, ADD(MUL(x, x), MUL(y, y))));
        const double s0 = (double)as[0], s1 = (double)as[1], s2 = (double)as[2];
        double m[9];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            m[3 * a + 0] = MUL(rq[3 * a + 0], s0);
            m[3 * a + 1] = MUL(rq[3 * a + 1], s1);
            m[3 * a + 2] = MUL(rq[3 * a + 2], s2);
        }
        double cov[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
                cov[3 * a + b] = FMA(m[3 * a + 2], m[3 * b + 2], FMA(m[3 * a + 1], m[3 * b + 1], MUL(m[3 * a], m[3 * b])));

        const double safe_z = alive ? depth : 1.0;
        const double inv_z = __ddiv_rn(1.0, safe_z);
        const double tx = MUL(np_clip(MUL(pv[0], inv_z), -cam.lim_x, cam.lim_x), safe_z);
        const double ty = MUL(np_clip(MUL(pv[1], inv_z), -cam.lim_y, cam.lim_y), safe_z);
        const double j0 = MUL(cam.fx, inv_z);
        const double j2x = MUL(MUL(MUL(-cam.fx, tx), inv_z), inv_z);
        const double j1 = MUL(cam.fy, inv_z);
        const double j2y = MUL(MUL(MUL(-cam.fy, ty), inv_z), inv_z);
        double t0[3], t1[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            t0[k] = ADD(MUL(j0, R[k]), MUL(j2x, R[6 + k]));
            t1[k] = ADD(MUL(j1, R[3 + k]), MUL(j2y, R[6 + k]));
        }
        double ct0[3], ct1[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            ct0[a] = FMA(cov[3 * a + 2], t0[2], FMA(cov[3 * a + 0], t0[0], MUL(cov[3 * a + 1], t0[1])));
            ct1[a] = FMA(cov[3 * a + 2], t1[2], FMA(cov[3 * a + 0], t1[0], MUL(cov[3 * a + 1], t1[1])));
        }
        const double sxx = ADD(ADD(ADD(MUL(t0[0], ct0[0]), MUL(t0[1], ct0[1])), MUL(t0[2], ct0[2])), dilation);
        const double syy = ADD(ADD(ADD(MUL(t1[0], ct1[0]), MUL(t1[1], ct1[1])), MUL(t1[2], ct1[2])), dilation);
        const double sxy = ADD(ADD(MUL(t0[0], ct1[0]), MUL(t0[1], ct1[1])), MUL(t0[2], ct1[2]));

        const double det = SUB(MUL(sxx, syy), MUL(sxy, sxy));
        const double mid = MUL(0.5, ADD(sxx, syy));
        const double disc = __dsqrt_rn(np_max(SUB(MUL(mid, mid), det), 0.0));
        const double lam_max = ADD(mid, disc);
        const double mx = ADD(MUL(MUL(cam.fx, pv[0]), inv_z), cam.cx);
        const double my = ADD(MUL(MUL(cam.fy, pv[1]), inv_z), cam.cy);
        const double r_o_real = MUL(3.0, __dsqrt_rn(np_max(lam_max, 0.0)));
        const double sigma = (double)aop;
        double ex, ey;
        double ln_a_over_op = 1e300;   // for cull_params (fused); 1e300: not known

        if (mode == ADR_MODE_BASELINE) {
            ex = ceil(r_o_real);
            ey = ex;
        } else {
            alive = alive && (sigma > alpha_low);
            const double log_ratio = log_fd(np_max(__ddiv_rn(sigma, alpha_low), 1e-300));
            if (FUSED) ln_a_over_op = fused.ln_a32_a64 - log_ratio;   // = ln(a32 / sigma)
            if (mode == ADR_MODE_CIRCLE) {
                const double v = __dsqrt_rn(MUL(MUL(2.0, lam_max), log_ratio));
                ex = ceil(np_min(v, r_o_real));
                ey = ex;
                if (FUSED && alive) ambiguous = ceil_ambiguous(v, r_o_real);
            } else {
                const double vx = __dsqrt_rn(MUL(MUL(2.0, sxx), log_ratio));
                const double vy = __dsqrt_rn(MUL(MUL(2.0, syy), log_ratio));
                ex = ceil(np_min(vx, r_o_real));
                ey = ceil(np_min(vy, r_o_real));
                if (FUSED && alive) ambiguous = ceil_ambiguous(vx, r_o_real) + ceil_ambiguous(vy, r_o_real);
            }
        }
        alive = alive && (ex >= 1.0) && (ey >= 1.0);

        out.d_valid[i] = (uint8_t)alive;
        if (alive) {
            double d0 = SUB(c0, cam.center[0]), d1 = SUB(c1, cam.center[1]), d2 = SUB(c2, cam.center[2]);
            const double nrm = __dsqrt_rn(ADD(ADD(MUL(d0, d0), MUL(d1, d1)), MUL(d2, d2)));
            const double dn = nrm > 0 ? nrm : 1.0;
            d0 = __ddiv_rn(d0, dn);
            d1 = __ddiv_rn(d1, dn);
            d2 = __ddiv_rn(d2, dn);
            const T* shp = stage + threadIdx.x * S;
            double col[3];
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                double cf[K];
#pragma unroll
                for (int k = 0; k < K; ++k) cf[k] = (double)shp[k * 3 + ch];
                col[ch] = sh_channel<DEG>(cf, d0, d1, d2);
            }
            const float2 m2 = make_float2(__double2float_rn(mx), __double2float_rn(my));
            const float ca = __double2float_rn(__ddiv_rn(syy, det));
            const float cb = __double2float_rn(__ddiv_rn(-sxy, det));
            const float cc = __double2float_rn(__ddiv_rn(sxx, det));
            const float dz = __double2float_rn(depth);
            const float op = __double2float_rn(sigma);
            const float c0f = __double2float_rn(col[0]), c1f = __double2float_rn(col[1]),
                        c2f = __double2float_rn(col[2]);
            if (!(FUSED && fused.rec_only)) {   // else these live in the render record only
                reinterpret_cast<float2*>(out.d_mean2d)[i] = m2;
                out.d_conic[3 * i] = ca;
                out.d_conic[3 * i + 1] = cb;
                out.d_conic[3 * i + 2] = cc;
                out.d_color[3 * i] = c0f;
                out.d_color[3 * i + 1] = c1f;
                out.d_color[3 * i + 2] = c2f;
                out.d_opacity[i] = op;
            }
            out.d_cov2d[3 * i] = __double2float_rn(sxx);
            out.d_cov2d[3 * i + 1] = __double2float_rn(syy);
            out.d_cov2d[3 * i + 2] = __double2float_rn(sxy);
            out.d_depth[i] = dz;
            out.d_lambda_max[i] = __double2float_rn(lam_max);
            const int32_t ix = np_i32(ex), iy = np_i32(ey);
            out.d_ext_x[i] = ix;
            out.d_ext_y[i] = iy;
            if (FUSED) {
                nan_color = c0f != c0f || c1f != c1f || c2f != c2f;
                const Rect r = tile_rect(m2.x, m2.y, ix, iy, true, fused.tiles_x, fused.tiles_y);
                selected = r.count() > 0;
                dbits = __float_as_uint(dz);
                Record R;
                float tau, hx, hy;
                cull_params(ca, cb, cc, op, (float)alpha_low, c0f, c1f, c2f, &tau, &hx, &hy, ln_a_over_op);
                R.a = make_float4(m2.x, m2.y, ca, cb);
                R.b = make_float4(cc, op, c0f, c1f);
                R.c = make_float4(c2f, tau, hx, hy);
                fused.rec[i] = R;
                fused.gpack[i] = make_uint2((uint32_t)r.x0 | ((uint32_t)r.x1 << 16),
                                            (uint32_t)r.y0 | ((uint32_t)r.y1 << 16));
            }
        } else {
            if (FUSED && fused.rec_only) {
                const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                Record R;
                R.a = R.b = R.c = z;
                fused.rec[i] = R;
            } else {
                reinterpret_cast<float2*>(out.d_mean2d)[i] = make_float2(0.f, 0.f);
                out.d_conic[3 * i] = out.d_conic[3 * i + 1] = out.d_conic[3 * i + 2] = 0.f;
                out.d_color[3 * i] = out.d_color[3 * i + 1] = out.d_color[3 * i + 2] = 0.f;
                out.d_opacity[i] = 0.f;
            }
            out.d_cov2d[3 * i] = out.d_cov2d[3 * i + 1] = out.d_cov2d[3 * i + 2] = 0.f;
            out.d_depth[i] = 0.f;
            out.d_lambda_max[i] = 0.f;
            out.d_ext_x[i] = 0;
            out.d_ext_y[i] = 0;
        }
    }
    if (FUSED) {
        // depth-sort key: float32 depth bits for Gaussians touching >= 1
        // tile (depth > near_plane > 0, so bit 31 is clear), all-ones for the
        // rest, which a stable sort then leaves behind the M selected ones
        if (i < n) fused.dkey[i] = selected ? dbits : 0xffffffffu;
        const int lane = threadIdx.x & 31;
        const uint32_t culled = __ballot_sync(kFull, i < n && !alive);
        const uint32_t sb = __ballot_sync(kFull, selected);
        const uint32_t nanb = __ballot_sync(kFull, nan_color);
        if (__any_sync(kFull, ambiguous != 0)) {
            const int amb = __reduce_add_sync(kFull, (unsigned)ambiguous);
            if (lane == 0 && fused.ambiguous) atomicAdd(fused.ambiguous, (unsigned long long)amb);
        }
        if (fused.kminmax) {   // the depth sort's key-range plan (adr_supertile.cu): per-warp extrema
            const uint32_t kmn = __reduce_min_sync(kFull, selected ? dbits : 0xffffffffu);
            const uint32_t kmx = __reduce_max_sync(kFull, selected ? dbits : 0u);
            if (threadIdx.x == 0 && blk == 0 && fused.plan_mm) {
                fused.plan_mm[0] = 0xffffffffu;
                fused.plan_mm[1] = 0u;
            }
            if (lane == 0)
                reinterpret_cast<uint2*>(fused.kminmax)[blk * (kPreBlock / 32) + (threadIdx.x >> 5)] =
                    make_uint2(kmn, kmx);
        }
        if (lane == 0) {
            if (culled) atomicAdd(fused.culled, (unsigned long long)__popc(culled));
            if (sb) atomicAdd(reinterpret_cast<unsigned long long*>(fused.d_m), (unsigned long long)__popc(sb));
            if (nanb && fused.nan_colors) atomicAdd(fused.nan_colors, (unsigned long long)__popc(nanb));
        }
    }
}

// Grid-stride over 128-Gaussian blocks.  Register budget pinned to 7 blocks
// per SM (72 registers): with frames in flight, 64 registers (8 blocks) and
// 80 (6 blocks) both measured 2-5% fewer frames/s (notes.md, experiment 8).
template <typename T, int DEG, bool FUSED>
#ifndef ADR_PRE_MINB
#define ADR_PRE_MINB 7
#endif
__global__ void __launch_bounds__(kPreBlock, ADR_PRE_MINB)
k_preprocess(const T* __restrict__ centers, const T* __restrict__ scales,
             const T* __restrict__ rotations, const T* __restrict__ opacities,
             const T* __restrict__ sh, int64_t n, adr_camera cam, int32_t mode,
             double alpha_low, double dilation, adr_projection out, FusedPre fused) {
    const int64_t nblk = (n + kPreBlock - 1) / kPreBlock;
    for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        preprocess_block<T, DEG, FUSED>(centers, scales, rotations, opacities, sh, n, cam, mode, alpha_low,
                                        dilation, out, fused, blk);
        __syncthreads();   // the SH stage is rewritten by the next block
    }
}


// Stage 1 of up to kMaxBatchViews frames of ONE scene in one launch (the
// views of a bench step / serving batch share the scene): each block reads
// its 128 rows and their SH slab once, evaluates the view-independent terms
// once (PreRow), then runs every view's projection / SH colour / outputs.
// Every view's outputs are bit-identical to k_preprocess's (same operations
// on the same operands); the scene is read once instead of nv times.
// Register budget: 7 blocks/SM (72 registers, 48 B of spills) measured best
// against 4 / 5 / 6 (120 / 96 / 80 registers), a float64 SH stage and the
// view-independent row kept in shared memory (notes.md, experiment 20).
#ifndef ADR_PREV_MINB
#define ADR_PREV_MINB 7
#endif
template <typename T, int DEG>
__global__ void __launch_bounds__(kPreBlock, ADR_PREV_MINB)
k_preprocess_views(const T* __restrict__ centers, const T* __restrict__ scales,
                   const T* __restrict__ rotations, const T* __restrict__ opacities,
                   const T* __restrict__ sh, int64_t n, int32_t mode, double alpha_low, double dilation,
                   const __grid_constant__ PreViews pv) {
    constexpr int S = (DEG + 1) * (DEG + 1) * 3 + 1;
    extern __shared__ __align__(16) unsigned char pre_smem[];
    T* stage = reinterpret_cast<T*>(pre_smem);
    const int64_t blk = blockIdx.x;
    const int64_t first = blk * kPreBlock;
    const int64_t i = first + threadIdx.x;
    T ac[3] = {T(0), T(0), T(0)}, as[3] = {T(0), T(0), T(0)}, aq[4] = {T(0), T(0), T(0), T(0)}, aop = T(0);
    load_block<T, DEG>(centers, scales, rotations, opacities, sh, n, first, stage, ac, as, aq, aop);
    __syncthreads();
    PreRow g;
    if (i < n) pre_row<T>(g, ac, as, aq, aop, mode, alpha_low);
#pragma unroll 1
    for (int v = 0; v < pv.nv; ++v)
        preprocess_view<T, DEG, true>(g, i < n, i, stage + threadIdx.x * S, pv.cam[v], mode, alpha_low, dilation,
                                      pv.out[v], pv.fused[v], blk);
}

#undef MUL
#undef ADD
#undef SUB
#undef FMA

template <typename T, bool FUSED>
int32_t launch_typed(const adr_scene& s, const adr_camera& cam, int32_t mode, double alpha_low,
                     double dilation, const adr_projection& out, const FusedPre& f, cudaStream_t st) {
    int64_t grid = ceil_div(s.n, kPreBlock);
    if (FUSED && kPreBlocksPerSm > 0) {
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            ADR_CUDA_TRY(cudaGetDevice(&dev));
            ADR_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        }
        const int64_t cap = (int64_t)sms * kPreBlocksPerSm;
        grid = grid < cap ? grid : cap;
    }
    const T* c = static_cast<const T*>(s.d_centers);
    const T* sc = static_cast<const T*>(s.d_scales);
    const T* r = static_cast<const T*>(s.d_rotations);
    const T* o = static_cast<const T*>(s.d_opacities);
    const T* sh = static_cast<const T*>(s.d_sh);
#define ADR_PRE(DEG)                                                                                          \
    do {                                                                                                      \
        const size_t sm = sizeof(T) * kPreBlock * ((DEG + 1) * (DEG + 1) * 3 + 1);                            \
        ADR_CUDA_TRY(cudaFuncSetAttribute(k_preprocess<T, DEG, FUSED>,                                         \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));             \
        k_preprocess<T, DEG, FUSED><<<grid, kPreBlock, sm, st>>>(c, sc, r, o, sh, s.n, cam, mode, alpha_low,  \
                                                                 dilation, out, f);                           \
    } while (0)
    switch (s.sh_degree) {
        case 0: ADR_PRE(0); break;
        case 1: ADR_PRE(1); break;
        case 2: ADR_PRE(2); break;
        case 3: ADR_PRE(3); break;
        default: return fail(ADR_ERR_VALUE, "sh_degree must be in 0..3");
    }
#undef ADR_PRE
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

}  // namespace

int32_t launch_preprocess(const adr_scene& scene, const adr_camera& cam, int32_t mode,
                          double alpha_low, double dilation, const adr_projection& out,
                          const FusedPre* fused, cudaStream_t st) {
    if (!(alpha_low > 0.0 && alpha_low < 1.0)) return fail(ADR_ERR_VALUE, "alpha_low must lie in (0, 1)");
    if (!(dilation >= 0.0)) return fail(ADR_ERR_VALUE, "dilation must be non-negative");
    if (mode < ADR_MODE_BASELINE || mode > ADR_MODE_AABB) return fail(ADR_ERR_VALUE, "unknown culling mode");
    if (scene.n < 0) return fail(ADR_ERR_VALUE, "negative Gaussian count");
    if (scene.n == 0) return ADR_OK;
    FusedPre f = fused ? *fused : FusedPre{};
    if (scene.dtype == ADR_F32)
        return fused ? launch_typed<float, true>(scene, cam, mode, alpha_low, dilation, out, f, st)
                     : launch_typed<float, false>(scene, cam, mode, alpha_low, dilation, out, f, st);
    if (scene.dtype == ADR_F64)
        return fused ? launch_typed<double, true>(scene, cam, mode, alpha_low, dilation, out, f, st)
                     : launch_typed<double, false>(scene, cam, mode, alpha_low, dilation, out, f, st);
    return fail(ADR_ERR_VALUE, "scene dtype must be ADR_F32 or ADR_F64");
}


int32_t launch_preprocess_views(const adr_scene& s, const PreViews& pv, int32_t mode, double alpha_low,
                                double dilation, cudaStream_t st) {
    if (!(alpha_low > 0.0 && alpha_low < 1.0)) return fail(ADR_ERR_VALUE, "alpha_low must lie in (0, 1)");
    if (!(dilation >= 0.0)) return fail(ADR_ERR_VALUE, "dilation must be non-negative");
    if (mode < ADR_MODE_BASELINE || mode > ADR_MODE_AABB) return fail(ADR_ERR_VALUE, "unknown culling mode");
    if (pv.nv < 1 || pv.nv > kMaxBatchViews) return fail(ADR_ERR_VALUE, "n_views must lie in 1..8");
    if (s.n < 0) return fail(ADR_ERR_VALUE, "negative Gaussian count");
    if (s.n == 0) return ADR_OK;
    const int64_t grid = ceil_div(s.n, kPreBlock);
#define ADR_PREV(T, DEG)                                                                                       \
    do {                                                                                                       \
        const size_t sm = sizeof(T) * kPreBlock * ((DEG + 1) * (DEG + 1) * 3 + 1);                  \
        ADR_CUDA_TRY(cudaFuncSetAttribute(k_preprocess_views<T, DEG>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                          (int)sm));                                                           \
        k_preprocess_views<T, DEG><<<grid, kPreBlock, sm, st>>>(                                               \
            static_cast<const T*>(s.d_centers), static_cast<const T*>(s.d_scales),                             \
            static_cast<const T*>(s.d_rotations), static_cast<const T*>(s.d_opacities),                        \
            static_cast<const T*>(s.d_sh), s.n, mode, alpha_low, dilation, pv);                                \
    } while (0)
#define ADR_PREV_T(T)                                                   \
    switch (s.sh_degree) {                                              \
        case 0: ADR_PREV(T, 0); break;                                  \
        case 1: ADR_PREV(T, 1); break;                                  \
        case 2: ADR_PREV(T, 2); break;                                  \
        case 3: ADR_PREV(T, 3); break;                                  \
        default: return fail(ADR_ERR_VALUE, "sh_degree must be in 0..3"); \
    }
    if (s.dtype == ADR_F32) {
        ADR_PREV_T(float)
    } else if (s.dtype == ADR_F64) {
        ADR_PREV_T(double)
    } else {
        return fail(ADR_ERR_VALUE, "scene dtype must be ADR_F32 or ADR_F64");
    }
#undef ADR_PREV_T
#undef ADR_PREV
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

}  // namespace adr
