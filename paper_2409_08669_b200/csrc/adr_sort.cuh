// adr_sort.cuh — stable LSD radix sort (key, value) for sm_100a.
//
// Each pass = upsweep (per-block digit histogram) → look-back scan of the
// digit-major histogram → downsweep (warp-level match_any ranking, block
// reorder in shared memory, coalesced scatter).  Stability: items keep their
// input order inside a digit, which is what np.argsort(kind="stable") gives
// (sb/tiling.py:159-164).  Used by the stage API (64-bit keys) and by the
// fused frame (32-bit depth keys of Gaussians, 16-bit tile keys of pairs).
//
// Item counts may live on the device (`d_n`): grids are sized for the static
// upper bound and blocks beyond the live count contribute empty histograms, so
// a whole frame can be captured into one CUDA graph without host syncs.
#pragma once

#include "adr_scan.cuh"

namespace adr {

constexpr int kSortBlock = 256;
constexpr int kSortWarps = kSortBlock / 32;

template <typename K>
struct SortCfg {
    static constexpr int kIpt = sizeof(K) >= 8 ? 8 : 16;
    static constexpr int kTileItems = kSortBlock * kIpt;
};

__device__ __forceinline__ int64_t live_count(const int64_t* d_n, int64_t n_static) {
    return d_n ? *d_n : n_static;
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int bit, uint32_t mask) {
    return (uint32_t)(key >> bit) & mask;
}

// Upsweep: hist[d * n_blocks + b] = #items of block b with digit d.
template <typename K, int RADIX_BITS>
__global__ void __launch_bounds__(kSortBlock)
radix_upsweep(const K* __restrict__ keys, const int64_t* d_n, int64_t n_static, int bit,
              uint32_t* __restrict__ hist) {
    constexpr int R = 1 << RADIX_BITS;
    constexpr int kIpt = SortCfg<K>::kIpt;
    __shared__ uint32_t sh[kSortWarps][R];
    const int64_t n = live_count(d_n, n_static);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kSortWarps * R; i += kSortBlock) (&sh[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * SortCfg<K>::kTileItems;
    const uint32_t mask = R - 1;
#pragma unroll
    for (int k = 0; k < kIpt; ++k) {
        const int64_t i = base + (int64_t)k * kSortBlock + threadIdx.x;
        if (i < n) atomicAdd(&sh[warp][digit_of(keys[i], bit, mask)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < R; d += kSortBlock) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) s += sh[w][d];
        hist[(int64_t)d * gridDim.x + blockIdx.x] = s;
    }
    (void)lane;
}

// Exclusive scan of the digit-major histogram (length R * n_blocks), one
// decoupled look-back pass.
template <int IPT>
__global__ void __launch_bounds__(256)
scan_u32_exclusive(uint32_t* __restrict__ data, int64_t n, uint64_t* status,
                   unsigned long long* counter) {
    __shared__ int64_t sbid;
    __shared__ uint64_t sred[33];
    __shared__ uint64_t sexcl;
    const int64_t bid = dynamic_block_id(counter, &sbid);
    const int64_t base = bid * 256 * IPT + (int64_t)threadIdx.x * IPT;
    uint32_t v[IPT];
    uint64_t tsum = 0;
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        v[k] = base + k < n ? data[base + k] : 0u;
        tsum += v[k];
    }
    uint64_t btotal;
    const uint64_t tpre = block_exclusive_sum<uint64_t, 256>(tsum, sred, &btotal);
    if (threadIdx.x < 32) {
        const uint64_t e = lookback(status, bid, btotal);
        if (threadIdx.x == 0) sexcl = e;
    }
    __syncthreads();
    uint64_t run = sexcl + tpre;
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        if (base + k < n) data[base + k] = (uint32_t)run;
        run += v[k];
    }
}

// Downsweep: stable scatter of one pass.
template <typename K, typename V, int RADIX_BITS>
__global__ void __launch_bounds__(kSortBlock)
radix_downsweep(const K* __restrict__ keys_in, const V* __restrict__ vals_in,
                K* __restrict__ keys_out, V* __restrict__ vals_out, const int64_t* d_n,
                int64_t n_static, int bit, const uint32_t* __restrict__ offsets) {
    constexpr int R = 1 << RADIX_BITS;
    constexpr int kIpt = SortCfg<K>::kIpt;
    constexpr int kTile = SortCfg<K>::kTileItems;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* skeys = reinterpret_cast<K*>(smem_raw);
    V* svals = reinterpret_cast<V*>(smem_raw + sizeof(K) * kTile);
    uint32_t* wh = reinterpret_cast<uint32_t*>(smem_raw + (sizeof(K) + sizeof(V)) * kTile);
    uint32_t* bstart = wh + kSortWarps * R;   // [R] block-local digit starts
    uint32_t* goff = bstart + R;              // [R] global digit offsets of this block
    __shared__ uint32_t sred[33];

    const int64_t n = live_count(d_n, n_static);
    const int64_t base = (int64_t)blockIdx.x * kTile;
    if (base >= n) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t mask = R - 1;
    for (int i = threadIdx.x; i < kSortWarps * R; i += kSortBlock) wh[i] = 0;
    for (int d = threadIdx.x; d < R; d += kSortBlock)
        goff[d] = offsets[(int64_t)d * gridDim.x + blockIdx.x];
    __syncthreads();

    // Warp w owns items [base + w*32*kIpt, base + (w+1)*32*kIpt), processed in
    // rounds of 32 consecutive items so (round, lane) order == input order.
    const int64_t wbase = base + (int64_t)warp * 32 * kIpt;
    K k_reg[kIpt];
    V v_reg[kIpt];
    uint32_t d_reg[kIpt], r_reg[kIpt];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < kIpt; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        const bool live = i < n;
        K key = live ? keys_in[i] : K(0);
        V val = live ? vals_in[i] : V(0);
        const uint32_t d = live ? digit_of(key, bit, mask) : (uint32_t)R;
        const uint32_t peers = __match_any_sync(kFull, d);
        const uint32_t before = live ? wh[warp * R + d] : 0u;
        __syncwarp();
        if (live && lane == __ffs(peers) - 1) wh[warp * R + d] = before + __popc(peers);
        __syncwarp();
        k_reg[r] = key;
        v_reg[r] = val;
        d_reg[r] = d;
        r_reg[r] = before + __popc(peers & lt);
    }
    __syncthreads();
    // Per digit: exclusive prefix over warps, then exclusive prefix over digits.
    constexpr int kDpt = (R + kSortBlock - 1) / kSortBlock;  // digits per thread
    uint32_t dtot[kDpt];
    uint32_t tsum = 0;
#pragma unroll
    for (int j = 0; j < kDpt; ++j) {
        const int d = threadIdx.x * kDpt + j;
        uint32_t run = 0;
        if (d < R) {
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) {
                const uint32_t t = wh[w * R + d];
                wh[w * R + d] = run;
                run += t;
            }
        }
        dtot[j] = run;
        tsum += run;
    }
    uint32_t btot;
    uint32_t pre = block_exclusive_sum<uint32_t, kSortBlock>(tsum, sred, &btot);
#pragma unroll
    for (int j = 0; j < kDpt; ++j) {
        const int d = threadIdx.x * kDpt + j;
        if (d < R) bstart[d] = pre;
        pre += dtot[j];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kIpt; ++r) {
        if (d_reg[r] < (uint32_t)R) {
            const uint32_t pos = bstart[d_reg[r]] + wh[warp * R + d_reg[r]] + r_reg[r];
            skeys[pos] = k_reg[r];
            svals[pos] = v_reg[r];
        }
    }
    __syncthreads();
    const int live_items = (int)((n - base) < kTile ? (n - base) : kTile);
    for (int i = threadIdx.x; i < live_items; i += kSortBlock) {
        const K key = skeys[i];
        const uint32_t d = digit_of(key, bit, mask);
        const int64_t g = (int64_t)goff[d] + (i - (int64_t)bstart[d]);
        keys_out[g] = key;
        vals_out[g] = svals[i];
    }
}

template <typename K, typename V, int RADIX_BITS>
inline size_t downsweep_smem() {
    constexpr int R = 1 << RADIX_BITS;
    return (sizeof(K) + sizeof(V)) * SortCfg<K>::kTileItems + sizeof(uint32_t) * (kSortWarps * R + 2 * R);
}

// Scratch for sorting up to n_max items: alternate key/value buffers, the
// digit histogram and the look-back status of its scan.
template <typename K, typename V>
inline size_t radix_scratch_bytes(int64_t n_max) {
    const int64_t nb = ceil_div(n_max > 0 ? n_max : 1, SortCfg<K>::kTileItems);
    const int64_t hist = nb * 256;
    const int64_t scan_blocks = ceil_div(hist, 256 * 8);
    return align_up(sizeof(K) * n_max) + align_up(sizeof(V) * n_max) +
           align_up(sizeof(uint32_t) * hist) + lookback_bytes(scan_blocks) + 256;
}

// Host driver: sorts n items (live count optionally on device) on bits
// [0, end_bit) with 8-bit digits (the last digit may be narrower).  Output
// lands in keys_out/vals_out; inputs are untouched.
template <typename K, typename V>
int32_t radix_sort(const K* keys_in, const V* vals_in, K* keys_out, V* vals_out,
                   const int64_t* d_n, int64_t n_max, int end_bit, void* scratch,
                   size_t scratch_bytes, cudaStream_t st) {
    if (n_max <= 0) return ADR_OK;
    if (end_bit <= 0) {
        // Nothing to order: the stable sort is the identity.
        ADR_CUDA_TRY(cudaMemcpyAsync(keys_out, keys_in, sizeof(K) * n_max, cudaMemcpyDeviceToDevice, st));
        ADR_CUDA_TRY(cudaMemcpyAsync(vals_out, vals_in, sizeof(V) * n_max, cudaMemcpyDeviceToDevice, st));
        return ADR_OK;
    }
    Carver c(scratch, scratch_bytes);
    K* alt_k = c.take<K>(n_max);
    V* alt_v = c.take<V>(n_max);
    const int64_t nb = ceil_div(n_max, SortCfg<K>::kTileItems);
    uint32_t* hist = c.take<uint32_t>(nb * 256);
    const int64_t hist_len_max = nb * 256;
    const int64_t scan_blocks_max = ceil_div(hist_len_max, 256 * 8);
    uint64_t* status = c.take<uint64_t>(scan_blocks_max + 1);
    unsigned long long* counter = reinterpret_cast<unsigned long long*>(status + scan_blocks_max);
    if (!c.ok()) return fail(ADR_ERR_VALUE, "radix_sort: scratch too small");

    const int passes = (end_bit + 7) / 8;
    const K* src_k = keys_in;
    const V* src_v = vals_in;
    for (int p = 0; p < passes; ++p) {
        const int bit = p * 8;
        const int bits = end_bit - bit < 8 ? end_bit - bit : 8;
        // Ping-pong so the final pass writes keys_out.
        const bool to_out = ((passes - 1 - p) % 2) == 0;
        K* dst_k = to_out ? keys_out : alt_k;
        V* dst_v = to_out ? vals_out : alt_v;
        const int radix = 1 << bits;
        (void)radix;
        const int64_t hist_len = nb * 256;  // digit-major with stride nb; unused digits are zero
        ADR_CUDA_TRY(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * hist_len, st));
        ADR_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(uint64_t) * (scan_blocks_max + 1), st));
        // Use 8-bit digit kernels with a narrower mask when bits < 8 by
        // shifting: digits above `bits` are zero after masking the key range.
#define ADR_SORT_PASS(RB)                                                                          \
    do {                                                                                           \
        radix_upsweep<K, RB><<<nb, kSortBlock, 0, st>>>(src_k, d_n, n_max, bit, hist);             \
        ADR_LAUNCH_CHECK();                                                                        \
        const int64_t hl = nb * (1 << RB);                                                         \
        const int64_t sb = ceil_div(hl, 256 * 8);                                                  \
        scan_u32_exclusive<8><<<sb, 256, 0, st>>>(hist, hl, status, counter);                      \
        ADR_LAUNCH_CHECK();                                                                        \
        const size_t sm = downsweep_smem<K, V, RB>();                                              \
        ADR_CUDA_TRY(cudaFuncSetAttribute(radix_downsweep<K, V, RB>,                               \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));  \
        radix_downsweep<K, V, RB><<<nb, kSortBlock, sm, st>>>(src_k, src_v, dst_k, dst_v, d_n,     \
                                                              n_max, bit, hist);                   \
        ADR_LAUNCH_CHECK();                                                                        \
    } while (0)
        switch (bits) {
            case 1: ADR_SORT_PASS(1); break;
            case 2: ADR_SORT_PASS(2); break;
            case 3: ADR_SORT_PASS(3); break;
            case 4: ADR_SORT_PASS(4); break;
            case 5: ADR_SORT_PASS(5); break;
            case 6: ADR_SORT_PASS(6); break;
            case 7: ADR_SORT_PASS(7); break;
            default: ADR_SORT_PASS(8); break;
        }
#undef ADR_SORT_PASS
        src_k = dst_k;
        src_v = dst_v;
    }
    return ADR_OK;
}

}  // namespace adr
