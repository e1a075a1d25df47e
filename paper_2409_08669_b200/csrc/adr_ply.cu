// adr_ply.cu — device half of the PLY checkpoint loader (sb/scene.py:316-398).
//
// The host parses the header and streams the float32 property matrix (one
// row of n_props floats per Gaussian, file order) to the device in chunks;
// this kernel activates each chunk into the float64 SoA scene the frame
// consumes, bit-identical to the reference's numpy / scipy arithmetic:
//   centers   = (x, y, z)                              scene.py:376
//   opacities = expit(opacity)                          scene.py:385 (scipy -> glibc exp)
//   scales    = exp(scale_0..2)                          scene.py:386 (numpy -> SVML exp8_ha)
//   rotations = rot / ||rot||, ||.|| = sqrt(((w2 + x2) + y2) + z2)   scene.py:387-392
//   sh[:, 0]  = f_dc_c, sh[:, 1 + j, c] = f_rest_{c (K-1) + j}        scene.py:380-384
// and reports the first row with a non-finite property (scene.py:370-373,
// every column) and the first zero-norm quaternion (scene.py:388-391).
//
// HBM-bound: per row 4 P bytes in, 8 (11 + 3K) bytes out (P = 62, K = 16:
// 248 + 472 B).  A block streams tiles of whole rows into shared memory by
// TMA bulk copies (double-buffered), then writes every output array with
// consecutive threads on consecutive elements (streaming stores); the fp64 exp / expit / divide work is ~0.3 kflop per
// row, far below the B200's fp64 rate at this byte count.
#include "adr_common.cuh"
#include "adr_exp64.cuh"
#include "adr_tma.cuh"

namespace adr {
namespace {

constexpr int kPlyThreads = 256;
constexpr int kPlyTileFloats = 6144;   // 24 KB per buffer, two buffers: rows = min(64, 6144 / P) & ~3

struct PlyCols {
    int32_t c[11 + 48];   // x y z | scale 0..2 | rot 0..3 | opacity | sh (k, channel)
};

// Tiles of T whole rows stream into two shared-memory buffers by 1-D bulk
// copies (TMA): tile i + 1 is in flight while the block activates tile i.
// A tile whose byte count is not a multiple of 16 (only the last one) copies
// the rounded-down part in bulk and its last <= 3 floats with plain loads.
template <int K>
__global__ void __launch_bounds__(kPlyThreads)
k_ply_activate(const float* __restrict__ raw, int64_t row0, int64_t rows, int32_t P, int32_t T,
               const __grid_constant__ PlyCols cols, double* __restrict__ ctr, double* __restrict__ scl,
               double* __restrict__ rot, double* __restrict__ op, double* __restrict__ sh,
               unsigned long long* __restrict__ status) {
    extern __shared__ __align__(16) float s_buf[];   // [2][T * P], each 16-byte aligned
    __shared__ int32_t s_col[11 + 3 * K];
    __shared__ double s_norm[64];
    __shared__ __align__(8) uint64_t s_bar[2];
    constexpr int Q = 3 * K;
    const int stride_f = (T * P + 3) & ~3;
    const int64_t tiles = (rows + T - 1) / T;
    if (blockIdx.x >= tiles) return;
    for (int i = threadIdx.x; i < 11 + Q; i += kPlyThreads) s_col[i] = cols.c[i];
    auto issue = [&](int64_t tile, int b) {   // thread 0 only
        const int64_t r0 = tile * T;
        const int nr = rows - r0 < T ? (int)(rows - r0) : T;
        const uint32_t bytes = (uint32_t)(nr * P * 4) & ~15u;
        fence_proxy_async_smem();
        if (bytes) {
            mbar_expect_tx(&s_bar[b], bytes);
            bulk_g2s(s_buf + b * stride_f, raw + r0 * P, bytes, &s_bar[b]);
        } else {
            mbar_expect_tx(&s_bar[b], 0);
        }
    };
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_proxy_async_smem();
        issue(blockIdx.x, 0);
    }
    __syncthreads();
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
        const int b = it & 1;
        if (threadIdx.x == 0 && tile + gridDim.x < tiles) issue(tile + gridDim.x, b ^ 1);
        const int64_t r0 = tile * T;
        const int nr = rows - r0 < T ? (int)(rows - r0) : T;
        const int nf = nr * P;
        float* s_tile = s_buf + b * stride_f;
        mbar_wait(&s_bar[b], (it >> 1) & 1);
        const int bulk_f = (nf * 4 & ~15) / 4;
        if (threadIdx.x < nf - bulk_f) s_tile[bulk_f + threadIdx.x] = __ldcs(raw + r0 * P + bulk_f + threadIdx.x);
        __syncthreads();
        for (int i = threadIdx.x; i < nf; i += kPlyThreads)
            if (!isfinite(s_tile[i])) atomicMin(status, (unsigned long long)(row0 + r0 + i / P));
        if (threadIdx.x < nr) {
            const float* row = s_tile + threadIdx.x * P;
            double n2 = 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double v = row[s_col[6 + q]];
                n2 = __dadd_rn(n2, __dmul_rn(v, v));
            }
            const double nrm = __dsqrt_rn(n2);
            s_norm[threadIdx.x] = nrm;
            if (nrm < 1e-12) atomicMin(status + 1, (unsigned long long)(row0 + r0 + threadIdx.x));
        }
        __syncthreads();
        const int64_t g0 = row0 + r0;
        for (int e = threadIdx.x; e < nr * 3; e += kPlyThreads) {
            const int r = e / 3, c = e - 3 * r;
            const float* row = s_tile + r * P;
            __stcs(ctr + g0 * 3 + e, (double)row[s_col[c]]);
            __stcs(scl + g0 * 3 + e, exp_svml((double)row[s_col[3 + c]]));
        }
        for (int e = threadIdx.x; e < nr * 4; e += kPlyThreads) {
            const int r = e >> 2;
            __stcs(rot + g0 * 4 + e, __ddiv_rn((double)s_tile[r * P + s_col[6 + (e & 3)]], s_norm[r]));
        }
        for (int r = threadIdx.x; r < nr; r += kPlyThreads)
            __stcs(op + g0 + r, expit_glibc((double)s_tile[r * P + s_col[10]]));
        for (int e = threadIdx.x; e < nr * Q; e += kPlyThreads) {
            const int r = e / Q;
            __stcs(sh + g0 * Q + e, (double)s_tile[r * P + s_col[11 + (e - r * Q)]]);
        }
        __syncthreads();   // buffer b and s_norm free before the next issue / tile
    }
}

__global__ void k_status_reset(unsigned long long* status) {
    if (threadIdx.x < 2) status[threadIdx.x] = 0x7fffffffffffffffull;
}

template <int K>
int32_t launch_ply(const float* raw, int64_t row0, int64_t rows, int32_t P, const PlyCols& cols,
                   const adr_scene& out, unsigned long long* status, cudaStream_t st) {
    // T a multiple of 4: every tile's first row is 16-byte aligned for the bulk copy
    const int T = (kPlyTileFloats / P < 64 ? kPlyTileFloats / P : 64) & ~3;
    const size_t smem = 2 * (size_t)((T * P + 3) & ~3) * sizeof(float);
    // one wave of resident blocks (a second partial wave would double the
    // grid-stride loop's tail)
    int per_sm = 0, dev = 0, sms = 0;
    ADR_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ply_activate<K>, kPlyThreads, smem));
    ADR_CUDA_TRY(cudaGetDevice(&dev));
    ADR_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t tiles = ceil_div(rows, T), wave = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    const int grid = (int)(tiles < wave ? tiles : wave);
    k_ply_activate<K><<<grid, kPlyThreads, smem, st>>>(
        raw, row0, rows, P, T, cols, (double*)out.d_centers, (double*)out.d_scales, (double*)out.d_rotations,
        (double*)out.d_opacities, (double*)out.d_sh, status);
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

}  // namespace
}  // namespace adr

using namespace adr;

extern "C" {

int32_t adr_ply_status_reset(int64_t* d_status, void* stream) {
    if (!d_status) return fail(ADR_ERR_VALUE, "adr_ply_status_reset: null status");
    k_status_reset<<<1, 32, 0, as_stream(stream)>>>(reinterpret_cast<unsigned long long*>(d_status));
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

int32_t adr_ply_activate(const float* d_raw, int64_t row0, int64_t rows, int32_t n_props, const int32_t* cols,
                         const adr_scene* out, int64_t* d_status, void* stream) {
    if (!out || !cols || !d_status) return fail(ADR_ERR_VALUE, "adr_ply_activate: null argument");
    if (out->dtype != ADR_F64) return fail(ADR_ERR_VALUE, "adr_ply_activate: the scene must be float64");
    if (out->sh_degree < 0 || out->sh_degree > 3) return fail(ADR_ERR_VALUE, "adr_ply_activate: sh_degree outside 0..3");
    if (rows < 0 || row0 < 0 || row0 + rows > out->n) return fail(ADR_ERR_VALUE, "adr_ply_activate: rows outside the scene");
    if (n_props < 1 || n_props > kPlyTileFloats / 4) return fail(ADR_ERR_VALUE, "adr_ply_activate: bad property count");
    const int K = (out->sh_degree + 1) * (out->sh_degree + 1);
    PlyCols pc{};
    for (int i = 0; i < 11 + 3 * K; ++i) {
        if (cols[i] < 0 || cols[i] >= n_props) return fail(ADR_ERR_VALUE, "adr_ply_activate: column out of range");
        pc.c[i] = cols[i];
    }
    if (rows == 0) return ADR_OK;
    if (!d_raw || (reinterpret_cast<uintptr_t>(d_raw) & 15))
        return fail(ADR_ERR_VALUE, "adr_ply_activate: raw matrix null or not 16-byte aligned");
    auto* status = reinterpret_cast<unsigned long long*>(d_status);
    cudaStream_t st = as_stream(stream);
    switch (K) {
        case 1: return launch_ply<1>(d_raw, row0, rows, n_props, pc, *out, status, st);
        case 4: return launch_ply<4>(d_raw, row0, rows, n_props, pc, *out, status, st);
        case 9: return launch_ply<9>(d_raw, row0, rows, n_props, pc, *out, status, st);
        default: return launch_ply<16>(d_raw, row0, rows, n_props, pc, *out, status, st);
    }
}

}  // extern "C"
