// adr_scan.cuh — single-pass device-wide scan (decoupled look-back) and the
// warp/block helpers the binning kernels share.
#pragma once

#include "adr_common.cuh"

namespace adr {

constexpr uint32_t kFull = 0xffffffffu;

// Status word of one block in the look-back chain:
// bits [63:62] = 0 not ready, 1 aggregate only, 2 inclusive prefix; [61:0] value.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPre = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// Block-wide exclusive sum of one value per thread.  `smem` holds >= 33
// entries.  Returns the exclusive prefix; *total receives the block sum.
template <typename T, int BLOCK>
__device__ __forceinline__ T block_exclusive_sum(T v, T* smem, T* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kWarps = BLOCK / 32;
    T inc = warp_inclusive_sum(v);
    if (lane == 31) smem[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < kWarps ? smem[lane] : T(0);
        T wi = warp_inclusive_sum(w);
        if (lane < kWarps) smem[lane] = wi - w;
        if (lane == kWarps - 1) smem[32] = wi;
    }
    __syncthreads();
    T r = smem[warp] + inc - v;
    *total = smem[32];
    __syncthreads();
    return r;
}

// Decoupled look-back (called by all 32 lanes of ONE warp).  Publishes this
// block's aggregate, resolves the exclusive prefix of all earlier blocks and
// publishes the inclusive prefix.  Returns the exclusive prefix on all lanes.
__device__ __forceinline__ uint64_t lookback(uint64_t* status, int64_t bid, uint64_t agg) {
    const int lane = threadIdx.x & 31;
    if (bid == 0) {
        if (lane == 0) st_relaxed(status, kFlagPre | agg);
        return 0;
    }
    if (lane == 0) st_relaxed(status + bid, kFlagAgg | agg);
    uint64_t excl = 0;
    int64_t end = bid - 1;
    while (true) {
        const int64_t idx = end - lane;
        uint64_t s = idx >= 0 ? ld_relaxed(status + idx) : kFlagPre;
        while (__any_sync(kFull, (s >> 62) == 0)) {
            if ((s >> 62) == 0) s = ld_relaxed(status + idx);
        }
        const uint32_t pre = __ballot_sync(kFull, (s >> 62) == 2);
        const int stop = pre ? __ffs(pre) - 1 : 31;
        uint64_t v = lane <= stop ? (s & kValMask) : 0;
        excl += warp_sum(v);
        if (pre) break;
        end -= 32;
    }
    if (lane == 0) st_relaxed(status + bid, kFlagPre | (excl + agg));
    return excl;
}

// Dynamic block index in launch order (forward-progress guarantee for the
// look-back chain).  counter must be zero before the launch.
__device__ __forceinline__ int64_t dynamic_block_id(unsigned long long* counter, int64_t* smem) {
    if (threadIdx.x == 0) *smem = (int64_t)atomicAdd(counter, 1ull);
    __syncthreads();
    const int64_t b = *smem;
    __syncthreads();
    return b;
}

// Scratch needed by one look-back scan over `n_blocks` blocks.
inline size_t lookback_bytes(int64_t n_blocks) {
    return align_up(sizeof(uint64_t) * (size_t)(n_blocks + 1)) + 256;
}

}  // namespace adr
