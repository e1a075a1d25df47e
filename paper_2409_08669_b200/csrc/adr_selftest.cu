// adr_selftest.cu — numerics self-tests exposed through the C ABI.
//
//   adr_exp_np_f32    : the render's float32 exp (numpy's AVX512F restatement)
//                       on arbitrary inputs, for golden-vector tests.
//   adr_selftest_exp  : exhaustive check that exp_np_fast and the packed
//                       exp2_np_fast (both render fast paths; the packed one
//                       evaluated with a different partner value in the other
//                       lane) equal exp_np on every float32 in [-87, 88].
#include "adr_common.cuh"
#include "adr_f32x2.cuh"
#include "adr_scan.cuh"
#include "adr_exp64.cuh"

namespace adr {
namespace {

__global__ void k_exp_np(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = exp_np(x[i]);
}

__global__ void k_selftest_exp(unsigned long long* mismatches, unsigned int* first_bad,
                               unsigned long long* checked, F2K k) {
    unsigned long long bad = 0, seen = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < (1ull << 32); u += stride) {
        const float x = __uint_as_float((uint32_t)u);
        if (!(x >= -87.0f && x <= 88.0f)) continue;
        ++seen;
        const float partner = __fmul_rn(-0.5f, x);  // also in [-87, 88]
        const f2 v = exp2_np_fast(pk(x, partner), k);
        const uint32_t ref = __float_as_uint(exp_np(x));
        if (__float_as_uint(exp_np_fast(x)) != ref || __float_as_uint(lo_of(v)) != ref ||
            __float_as_uint(hi_of(v)) != __float_as_uint(exp_np(partner))) {
            ++bad;
            atomicMin(first_bad, (uint32_t)u);
        }
    }
    if (bad) atomicAdd(mismatches, bad);
    atomicAdd(checked, seen);
}

// Exhaustive pin against numpy: H = sum over u in [lo, hi) of
// (bits(exp_np(u)) + 1) * (u * 0x9E3779B97F4A7C15 | 1) mod 2^64, the same
// checksum tests/golden/make_exp_exhaustive.py computes over np.exp.
__global__ void k_exp_checksum(uint64_t lo, uint64_t hi, unsigned long long* out) {
    uint64_t s = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t u = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < hi; u += stride) {
        const uint32_t y = __float_as_uint(exp_np(__uint_as_float((uint32_t)u)));
        s += ((uint64_t)y + 1u) * ((u * 0x9E3779B97F4A7C15ull) | 1u);
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)s);
}

// The PLY loader's float64 activations over every non-NaN float32 input u
// in [lo, hi) widened to float64: H = sum of (bits(f(u)) + 1) *
// (u * 0x9E3779B97F4A7C15 | 1) mod 2^64, kind 0 = np.exp (exp_svml),
// 1 = scipy expit (expit_glibc); tests/golden/make_exp64_exhaustive.py.
__global__ void k_exp64_checksum(int32_t kind, uint64_t lo, uint64_t hi, unsigned long long* out) {
    uint64_t s = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t u = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < hi; u += stride) {
        const uint32_t ub = (uint32_t)u;
        if ((ub & 0x7fffffffu) > 0x7f800000u) continue;
        const double x = (double)__uint_as_float(ub);
        const double y = kind == 0 ? exp_svml(x) : expit_glibc(x);
        s += (ubits(y) + 1u) * ((u * 0x9E3779B97F4A7C15ull) | 1u);
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)s);
}

}  // namespace
}  // namespace adr

using namespace adr;

extern "C" {

int32_t adr_exp_np_f32(const float* d_x, float* d_y, int64_t n, void* stream) {
    if (n <= 0) return ADR_OK;
    const int64_t blocks = ceil_div(n, 256) < 4096 ? ceil_div(n, 256) : 4096;
    k_exp_np<<<blocks, 256, 0, as_stream(stream)>>>(d_x, d_y, n);
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

int32_t adr_exp_checksum(uint64_t lo, uint64_t hi, uint64_t* d_out, void* stream) {
    cudaStream_t st = as_stream(stream);
    ADR_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(uint64_t), st));
    if (hi <= lo) return ADR_OK;
    k_exp_checksum<<<148 * 8, 256, 0, st>>>(lo, hi, reinterpret_cast<unsigned long long*>(d_out));
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

int32_t adr_exp64_checksum(int32_t kind, uint64_t lo, uint64_t hi, uint64_t* d_out, void* stream) {
    if (kind != 0 && kind != 1) return fail(ADR_ERR_VALUE, "adr_exp64_checksum: kind must be 0 or 1");
    cudaStream_t st = as_stream(stream);
    ADR_CUDA_TRY(cudaMemsetAsync(d_out, 0, sizeof(uint64_t), st));
    if (hi <= lo) return ADR_OK;
    k_exp64_checksum<<<148 * 8, 256, 0, st>>>(kind, lo, hi, reinterpret_cast<unsigned long long*>(d_out));
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

int32_t adr_selftest_exp(uint64_t* d_result, void* stream) {
    // d_result[0] = mismatches, d_result[1] = float inputs checked,
    // d_result[2] (low 32 bits) = smallest mismatching bit pattern
    cudaStream_t st = as_stream(stream);
    ADR_CUDA_TRY(cudaMemsetAsync(d_result, 0, 2 * sizeof(uint64_t), st));
    ADR_CUDA_TRY(cudaMemsetAsync(d_result + 2, 0xff, sizeof(uint64_t), st));
    k_selftest_exp<<<148 * 8, 256, 0, st>>>(reinterpret_cast<unsigned long long*>(d_result),
                                            reinterpret_cast<unsigned int*>(d_result + 2),
                                            reinterpret_cast<unsigned long long*>(d_result + 1), f2k_host());
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

}  // extern "C"
