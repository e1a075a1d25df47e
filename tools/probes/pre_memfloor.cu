// Memory floor of k_preprocess's access pattern (config 3: N = 5.8M, SH3, fp32):
// the same loads (attributes as strided scalars, the SH slab as 12 coalesced
// 16-byte loads per thread through an odd-stride shared row) and the same
// stores (Projection SoA incl. the stride-12 B 3-float arrays, the 48 B record,
// the 8 B rect, the depth key), with trivial arithmetic instead of the fp64
// projection.  Prints the kernel time and GB/s against the 2.06 GB it moves.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int B = 128, K3 = 48, S = K3 + 1;
template <int MODE>  // 0: full pattern, 1: loads only, 2: SH slab only, 3: attributes only, 4: stores only,
                     // 5: full pattern with warp-transposed (coalesced 16 B) 3-float and record stores
__global__ void __launch_bounds__(B) k_floor(const float* c, const float* s, const float* r, const float* o,
                                            const float* sh, long n, float* mean2d, float* cov, float* conic,
                                            float* depth, float* color, float* opac, float* lam, int* ex, int* ey,
                                            unsigned char* valid, float4* rec, uint2* rect, unsigned* dkey) {
    __shared__ float st[B * S];
    const long first = (long)blockIdx.x * B, i = first + threadIdx.x;
    float a = 0.f;
    if (i < n && MODE != 2 && MODE != 4) {
        for (int k = 0; k < 3; ++k) a += c[3 * i + k] + s[3 * i + k];
        for (int k = 0; k < 4; ++k) a += r[4 * i + k];
        a += o[i];
    }
    const float4* s4 = reinterpret_cast<const float4*>(sh + first * K3);
    float4 v[K3 / 4];
    if (first + B <= n && MODE != 3 && MODE != 4) {
#pragma unroll
        for (int u = 0; u < K3 / 4; ++u) v[u] = __ldg(s4 + threadIdx.x + u * B);
#pragma unroll
        for (int u = 0; u < K3 / 4; ++u) {
            const int f = 4 * (threadIdx.x + u * B), g = f / K3, j = f - g * K3;
            float* d = st + g * S + j;
            d[0] = v[u].x; d[1] = v[u].y; d[2] = v[u].z; d[3] = v[u].w;
        }
    }
    __syncthreads();
    if (i >= n) return;
    float csum = 0.f;
    for (int k = 0; k < K3; ++k) csum += st[threadIdx.x * S + k];
    const float x = a + csum;
    if (MODE == 1 || MODE == 2 || MODE == 3) {
        if (x == 123.456f) depth[i] = x;   // keeps the loads live, (almost) never stores
        return;
    }
    reinterpret_cast<float2*>(mean2d)[i] = make_float2(x, x + 1.f);
    if (MODE == 5) {
        // warp-private staging in the warp's own (already consumed) SH rows
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        __syncwarp();
        float* ws = st + w * 32 * S;
        for (int k = 0; k < 3; ++k) { ws[3 * lane + k] = x + k; ws[96 + 3 * lane + k] = x - k; ws[192 + 3 * lane + k] = x * k; }
        float4* wr = reinterpret_cast<float4*>(ws + 288);
        for (int k = 0; k < 3; ++k) wr[3 * lane + k] = make_float4(x, x, x, x);
        __syncwarp();
        const long wfirst = first + 32 * w;
        if (lane < 24) {
            reinterpret_cast<float4*>(cov + 3 * wfirst)[lane] = reinterpret_cast<const float4*>(ws)[lane];
            reinterpret_cast<float4*>(conic + 3 * wfirst)[lane] = reinterpret_cast<const float4*>(ws + 96)[lane];
            reinterpret_cast<float4*>(color + 3 * wfirst)[lane] = reinterpret_cast<const float4*>(ws + 192)[lane];
        }
        for (int k = 0; k < 3; ++k) rec[3 * wfirst + 32 * k + lane] = wr[32 * k + lane];
    } else {
    for (int k = 0; k < 3; ++k) { cov[3 * i + k] = x + k; conic[3 * i + k] = x - k; color[3 * i + k] = x * k; }
    rec[3 * i] = make_float4(x, x, x, x); rec[3 * i + 1] = make_float4(x, x, x, x); rec[3 * i + 2] = make_float4(x, x, x, x);
    }
    depth[i] = x; opac[i] = x; lam[i] = x; ex[i] = (int)x; ey[i] = (int)x; valid[i] = x > 0.f;
    rect[i] = make_uint2((unsigned)x, (unsigned)x + 1u);
    dkey[i] = __float_as_uint(x);
}
int main() {
    const long n = 5800000;
    float *c, *s, *r, *o, *sh, *m2, *cv, *cn, *dp, *cl, *op, *lm; int *ex, *ey; unsigned char* vl; float4* rc; uint2* rt; unsigned* dk;
    cudaMalloc(&c, 12 * n); cudaMalloc(&s, 12 * n); cudaMalloc(&r, 16 * n); cudaMalloc(&o, 4 * n); cudaMalloc(&sh, 192 * n);
    cudaMalloc(&m2, 8 * n); cudaMalloc(&cv, 12 * n); cudaMalloc(&cn, 12 * n); cudaMalloc(&dp, 4 * n); cudaMalloc(&cl, 12 * n);
    cudaMalloc(&op, 4 * n); cudaMalloc(&lm, 4 * n); cudaMalloc(&ex, 4 * n); cudaMalloc(&ey, 4 * n); cudaMalloc(&vl, n);
    cudaMalloc(&rc, 48 * n); cudaMalloc(&rt, 8 * n); cudaMalloc(&dk, 4 * n);
    cudaMemset(c, 0, 12 * n); cudaMemset(s, 0, 12 * n); cudaMemset(r, 0, 16 * n); cudaMemset(o, 0, 4 * n); cudaMemset(sh, 0, 192 * n);
    void* flush; cudaMalloc(&flush, 512l << 20);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int grid = (int)((n + B - 1) / B);
    const char* names[6] = {"full pattern", "loads only", "SH slab only", "attributes only", "stores only", "full, coalesced"};
    const double mb[6] = {2.09e9, 236.0 * n, 192.0 * n, 44.0 * n, 125.0 * n, 2.09e9};
    for (int mode = 0; mode < 6; ++mode) {
        float best = 1e9f;
        for (int rep = 0; rep < 8; ++rep) {
            cudaMemset(flush, rep, 512l << 20);   // evict L2
            cudaEventRecord(e0);
            if (mode == 0) k_floor<0><<<grid, B>>>(c, s, r, o, sh, n, m2, cv, cn, dp, cl, op, lm, ex, ey, vl, rc, rt, dk);
            if (mode == 1) k_floor<1><<<grid, B>>>(c, s, r, o, sh, n, m2, cv, cn, dp, cl, op, lm, ex, ey, vl, rc, rt, dk);
            if (mode == 2) k_floor<2><<<grid, B>>>(c, s, r, o, sh, n, m2, cv, cn, dp, cl, op, lm, ex, ey, vl, rc, rt, dk);
            if (mode == 3) k_floor<3><<<grid, B>>>(c, s, r, o, sh, n, m2, cv, cn, dp, cl, op, lm, ex, ey, vl, rc, rt, dk);
            if (mode == 4) k_floor<4><<<grid, B>>>(c, s, r, o, sh, n, m2, cv, cn, dp, cl, op, lm, ex, ey, vl, rc, rt, dk);
            if (mode == 5) k_floor<5><<<grid, B>>>(c, s, r, o, sh, n, m2, cv, cn, dp, cl, op, lm, ex, ey, vl, rc, rt, dk);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep > 1 && ms < best) best = ms;
        }
        printf("pre_memfloor %-16s %7.1f us  %6.0f GB/s  (%.2f GB)  %s\n", names[mode], best * 1e3,
               mb[mode] / (best * 1e-3) / 1e9, mb[mode] / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
