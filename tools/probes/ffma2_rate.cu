// Throughput probe: scalar FFMA vs packed FFMA2 (sm_100a), 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
struct K2 { unsigned long long a, b; float fa, fb; };
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__global__ void k_scalar(float* out, int iters, K2 k) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __fmaf_rn(x[i], k.fa, k.fb);
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_packed(float* out, int iters, K2 k) {
    unsigned long long x[8];
    for (int i = 0; i < 8; ++i) x[i] = (unsigned long long)(threadIdx.x + i) * 0x100000001ull;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma2(x[i], k.a, k.b);
    unsigned long long s = 0; for (int i = 0; i < 8; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(s & 0xffff);
}
int main() {
    float* d; cudaMalloc(&d, 148 * 8 * 1024 * 4);
    K2 k; k.fa = 0.999f; k.fb = 0.001f;
    unsigned int ua, ub; memcpy(&ua, &k.fa, 4); memcpy(&ub, &k.fb, 4);
    k.a = ((unsigned long long)ua << 32) | ua; k.b = ((unsigned long long)ub << 32) | ub;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); k_scalar<<<148 * 8, 1024>>>(d, iters, k); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 148.0 * 8 * 1024 * iters * 8 * 2;
        printf("scalar FFMA : %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
        cudaEventRecord(e0); k_packed<<<148 * 8, 1024>>>(d, iters, k); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("packed FFMA2: %.3f ms  %.1f TFLOP/s (lanes x2)\n", ms, 2 * fl / ms / 1e9);
    }
    return 0;
}
