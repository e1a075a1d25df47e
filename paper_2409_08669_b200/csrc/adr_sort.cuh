// adr_sort.cuh — stable LSD radix sort (key, value) for sm_100a.
//
// Reduce-then-scan per digit pass (<= 8-bit digits):
//
//   upsweep   : block digit histogram with shared-memory atomics ->
//               digit-major histogram over blocks.
//   scan      : exclusive scan of the digit-major histogram (look-back).
//   downsweep : warp-striped rounds of 32 items; peers with the same digit
//               come from one ballot per digit bit, the lowest peer bumps
//               the warp's counter, so each item gets its rank among equal
//               digits; warp prefixes + block digit starts place the tile in
//               shared memory in digit order; coalesced digit runs go out.
//
// Ballots run on the ALU pipe; MATCH.ANY (MIO pipe) and thread-private
// counter columns (64 KB of shared memory, 2 blocks/SM) both measured slower.
// Stable: (round, lane) order is input order, so equal digits keep their
// input order — np.argsort(kind="stable") (sb/tiling.py:159-164).  Item
// counts may live on the device (`d_n`) so whole frames can be captured into
// one CUDA graph.
#pragma once

#include "adr_scan.cuh"

namespace adr {

constexpr int kSortBlock = 256;
constexpr int kSortWarps = kSortBlock / 32;
constexpr int kMaxRadixBits = 8;

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

// Peers of this lane among the warp's lanes with the same digit: one
// ballot per digit bit (vote.sync on the ALU pipe; MATCH.ANY issues through
// the MIO pipe and measured slower).
template <int RB>
__device__ __forceinline__ uint32_t digit_peers(uint32_t d) {
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < RB; ++b) {
        uint32_t m;
        asm("{\n\t.reg .pred p;\n\t.reg .b32 q;\n\t"
            "and.b32 q, %1, %2;\n\tsetp.ne.u32 p, q, 0;\n\t"
            "vote.sync.ballot.b32 q, p, 0xffffffff;\n\t@!p not.b32 q, q;\n\tmov.b32 %0, q;\n\t}"
            : "=r"(m) : "r"(d), "r"(1u << b));
        peers &= m;
    }
    return peers;
}

// Key-range plan of the fused frame's depth sort.  With kmin = the smallest
// selected depth key rounded down to a multiple of 256, the keys "fit" when
// every selected key lies within 2^24 - 1 of kmin.  Then the
// sort runs on 24-bit keys t = key - kmin (all-ones "no pairs" keys ->
// 0xFFFFFF, still last): pass 0 sorts the raw low byte (equal to t's, kmin
// being a multiple of 256), pass 1 transforms as it loads, pass 2 is the last
// pass and restores key = t + kmin, pass 3's kernels exit at once.  Otherwise
// the 4 passes run on the raw keys.  Decided on the device, so a frame stays
// one fixed launch sequence (one CUDA graph); the (min, max) pair is reduced
// by kPlanBlocks extra blocks of pass 0's upsweep from the preprocess's
// per-block minima / maxima (the preprocess resets it).
struct DepthPlan {
    const uint32_t* plan = nullptr;       // (min, max) selected depth key; reset by the preprocess
    int pass = 0;
    uint32_t* plan_out = nullptr;         // pass 0 upsweep: the extra blocks' atomic min / max target
    const uint32_t* kminmax = nullptr;    // per preprocess warp: (min, max) selected key
    int64_t nkb = 0;                      // number of preprocess warps (4 per block)
};

constexpr int kPlanBlocks = 16;           // extra blocks of pass 0's upsweep that reduce the plan

// -> fits (three passes suffice), kmin (the key offset, a multiple of 256)
__device__ __forceinline__ bool plan_decode(const DepthPlan& dp, uint32_t* kmin) {
    *kmin = 0;
    if (!dp.plan) return false;
    const uint2 mm = *reinterpret_cast<const uint2*>(dp.plan);
    if (mm.x > mm.y) return true;   // no selected Gaussian: every key is all-ones
    *kmin = mm.x & ~0xffu;
    return mm.y - *kmin < 0xffffffu;
}

__device__ __forceinline__ bool plan_fits(const DepthPlan& dp) {
    uint32_t k;
    return plan_decode(dp, &k);
}

// Pass-1 key transform of a register array of keys, applied after all of
// them were loaded (a per-key plan test between the loads serialises them).
template <typename K, int N>
__device__ __forceinline__ void plan_transform(K (&kr)[N], const DepthPlan& dp) {
    if constexpr (sizeof(K) == 4) {
        if (dp.pass != 1 || !dp.plan) return;
        uint32_t kmin;
        if (!plan_decode(dp, &kmin)) return;
#pragma unroll
        for (int r = 0; r < N; ++r) kr[r] = kr[r] == K(0xffffffffu) ? K(0xffffffu) : K((uint32_t)kr[r] - kmin);
    }
}

// A plan block (pass 0 upsweep, the last kPlanBlocks blocks of the grid):
// min / max over its slice of the preprocess warps' extrema, merged with
// two atomics.
template <int BLOCK>
__device__ __forceinline__ void plan_reduce(const DepthPlan& dp, int slice) {
    __shared__ uint32_t smn[BLOCK / 32], smx[BLOCK / 32];
    uint32_t mn = 0xffffffffu, mx = 0u;
    for (int64_t b = (int64_t)slice * BLOCK + threadIdx.x; b < dp.nkb; b += (int64_t)kPlanBlocks * BLOCK) {
        const uint2 v = reinterpret_cast<const uint2*>(dp.kminmax)[b];
        mn = v.x < mn ? v.x : mn;
        mx = v.y > mx ? v.y : mx;
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) {
        smn[threadIdx.x >> 5] = mn;
        smx[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < BLOCK / 32; ++w) {
            mn = smn[w] < mn ? smn[w] : mn;
            mx = smx[w] > mx ? smx[w] : mx;
        }
        atomicMin(dp.plan_out, mn);
        atomicMax(dp.plan_out + 1, mx);
    }
}

// Block digit histogram: plain shared-memory atomics (no ranking needed).
template <typename K, int RB>
__global__ void __launch_bounds__(kSortBlock)
radix_upsweep(const K* __restrict__ keys, const int64_t* d_n, int64_t n_static, int bit,
              uint32_t* __restrict__ hist, DepthPlan dp = DepthPlan()) {
    constexpr int R = 1 << RB;
    constexpr int kIpt = SortCfg<K>::kIpt;
    __shared__ uint32_t h[R];
    if (dp.plan_out && blockIdx.x >= gridDim.x - kPlanBlocks) {
        plan_reduce<kSortBlock>(dp, blockIdx.x - (gridDim.x - kPlanBlocks));
        return;
    }
    if (dp.pass == 3 && plan_fits(dp)) return;
    const int64_t n = live_count(d_n, n_static);
    for (int i = threadIdx.x; i < R; i += kSortBlock) h[i] = 0;
    const int64_t base = (int64_t)blockIdx.x * SortCfg<K>::kTileItems;
    K kr[kIpt];
#pragma unroll
    for (int r = 0; r < kIpt; ++r) {
        const int64_t i = base + (int64_t)r * kSortBlock + threadIdx.x;
        kr[r] = i < n ? keys[i] : K(0);
    }
    plan_transform(kr, dp);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kIpt; ++r) {
        if (base + (int64_t)r * kSortBlock + threadIdx.x < n) atomicAdd(&h[digit_of(kr[r], bit, R - 1)], 1u);
    }
    __syncthreads();
    const int64_t nbh = dp.plan_out ? gridDim.x - kPlanBlocks : gridDim.x;   // histogram blocks
    for (int d = threadIdx.x; d < R; d += kSortBlock) hist[(int64_t)d * nbh + blockIdx.x] = h[d];
}

// Exclusive scan of the digit-major histogram (length R * n_blocks), one
// decoupled look-back pass.
template <int IPT>
__global__ void __launch_bounds__(256)
scan_u32_exclusive(uint32_t* __restrict__ data, int64_t n, uint64_t* status, unsigned long long* counter,
                   DepthPlan dp = DepthPlan()) {
    if (dp.pass == 3 && plan_fits(dp)) return;
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

// Downsweep of one pass (warp-striped: round r, lane l -> item wbase+32r+l,
// so (round, lane) order is input order).  vals_in == nullptr means the
// identity (value = input index).  Last-pass extras (MODE):
//   1: exp_keys[g] = key << 32 | float bits of exp_depth[value]  (reference keys)
//   2: gdst[g] = gsrc[value] (8-byte gather) and vals_out[g] = value; no key output
//   3: rinfo[g] = {value, key, gsrc[value]} (16-byte rank record); no key/value output
struct SortExtra {
    int mode = 0;
    const float* exp_depth = nullptr;
    uint64_t* exp_keys = nullptr;
    bool skip_keys_out = false;   // MODE 1: the exported keys carry the tile ids, no separate copy
    DepthPlan dp;                 // depth-sort key-range plan (MODE 0 / 3 passes of the fused frame)
    const uint2* gsrc = nullptr;
    uint2* gdst = nullptr;
    uint4* rinfo = nullptr;
};

template <typename K, typename V, int RB, int MODE>
__global__ void __launch_bounds__(kSortBlock, 3)
radix_downsweep(const K* __restrict__ keys_in, const V* __restrict__ vals_in, K* __restrict__ keys_out,
                V* __restrict__ vals_out, const int64_t* d_n, int64_t n_static, int bit,
                const uint32_t* __restrict__ offsets, SortExtra ex) {
    constexpr int R = 1 << RB;
    constexpr int kIpt = SortCfg<K>::kIpt;
    constexpr int kTile = SortCfg<K>::kTileItems;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* skeys = reinterpret_cast<K*>(smem_raw);
    V* svals = reinterpret_cast<V*>(smem_raw + sizeof(K) * kTile);
    __shared__ uint32_t wh[kSortWarps][R];
    __shared__ uint32_t dstart[R];
    __shared__ int64_t goff[R];
    __shared__ uint32_t sred[33];

    const int64_t n = live_count(d_n, n_static);
    const int64_t base = (int64_t)blockIdx.x * kTile;
    if (base >= n) return;
    // depth-sort plan: pass 3 is skipped and pass 2 becomes the last (MODE 3)
    // pass when the keys fit 24 bits
    uint32_t kmin = 0;
    const bool fits = ex.dp.pass >= 2 && plan_decode(ex.dp, &kmin);   // passes 2 and 3 change with it
    if (ex.dp.pass == 3 && fits) return;
    const bool as_last = MODE == 3 || (ex.dp.pass == 2 && fits);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kSortWarps * R; i += kSortBlock) (&wh[0][0])[i] = 0;
    const int64_t wbase = base + (int64_t)warp * 32 * kIpt;
    K kr[kIpt];
    V vr[kIpt];
#pragma unroll
    for (int r = 0; r < kIpt; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        kr[r] = i < n ? keys_in[i] : K(0);
        vr[r] = i < n ? (vals_in ? vals_in[i] : V(i)) : V(0);
    }
    plan_transform(kr, ex.dp);
    __syncthreads();
    // ranks packed two per register (rank within warp < 32 * kIpt <= 512)
    uint32_t rank2[(kIpt + 1) / 2];
    const uint32_t lt = (1u << lane) - 1u;
    const bool full = base + kTile <= n;
    const uint32_t live_mask = full ? 0xffffffffu : 0u;
#pragma unroll
    for (int r = 0; r < kIpt; ++r) {
        const bool live = full || wbase + r * 32 + lane < n;
        const uint32_t d = digit_of(kr[r], bit, R - 1);
        uint32_t peers = digit_peers<RB>(d);
        if (!full) peers &= __ballot_sync(kFull, live) | live_mask;
        const uint32_t before = wh[warp][d];
        __syncwarp();
        if (live && (peers & lt) == 0) wh[warp][d] = before + __popc(peers);
        __syncwarp();
        const uint32_t rk = before + __popc(peers & lt);
        if (r & 1) rank2[r >> 1] |= rk << 16; else rank2[r >> 1] = rk;
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, block total, block-local start
    uint32_t tot = 0;
    const int dd = threadIdx.x;
    if (dd < R) {
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t t = wh[w][dd];
            wh[w][dd] = tot;
            tot += t;
        }
    }
    uint32_t btot;
    const uint32_t dpre = block_exclusive_sum<uint32_t, kSortBlock>(dd < R ? tot : 0u, sred, &btot);
    if (dd < R) {
        dstart[dd] = dpre;
        goff[dd] = (int64_t)offsets[(int64_t)dd * gridDim.x + blockIdx.x] - (int64_t)dpre;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kIpt; ++r) {
        if (wbase + r * 32 + lane < n) {
            const uint32_t d = digit_of(kr[r], bit, R - 1);
            const uint32_t pos = dstart[d] + wh[warp][d] + ((rank2[r >> 1] >> (16 * (r & 1))) & 0xffffu);
            skeys[pos] = kr[r];
            svals[pos] = vr[r];
        }
    }
    __syncthreads();
    const int live = (int)((n - base) < kTile ? (n - base) : kTile);
    for (int i = threadIdx.x; i < live; i += kSortBlock) {
        const K key = skeys[i];
        const V val = svals[i];
        const int64_t g = goff[digit_of(key, bit, R - 1)] + i;
        if (MODE == 3 || (MODE == 0 && as_last)) {
            const uint2 r = __ldg(ex.gsrc + val);
            uint32_t kk = (uint32_t)key;
            if (fits) kk = kk == 0xffffffu ? 0xffffffffu : kk + kmin;
            ex.rinfo[g] = make_uint4((uint32_t)val, kk, r.x, r.y);
        } else if (MODE == 2) {
            vals_out[g] = val;
            ex.gdst[g] = __ldg(ex.gsrc + val);
        } else {
            if (MODE != 1 || !ex.skip_keys_out) keys_out[g] = key;
            vals_out[g] = val;
            if (MODE == 1 && ex.exp_keys)
                ex.exp_keys[g] = ((uint64_t)key << 32) | __float_as_uint(__ldcg(ex.exp_depth + val));
        }
    }
}

template <typename K, typename V, int RB>
inline size_t downsweep_smem() {
    return (sizeof(K) + sizeof(V)) * SortCfg<K>::kTileItems;
}

// Scratch for sorting up to n_max items.
template <typename K, typename V>
inline size_t radix_scratch_bytes(int64_t n_max) {
    const int64_t nb = ceil_div(n_max > 0 ? n_max : 1, SortCfg<K>::kTileItems);
    const int64_t hist = nb << kMaxRadixBits;
    const int64_t scan_blocks = ceil_div(hist, 256 * 8);
    return align_up(sizeof(K) * n_max) + align_up(sizeof(V) * n_max) + align_up(sizeof(uint32_t) * hist) +
           lookback_bytes(scan_blocks) + 512;
}

// Digit width per pass: end_bit split into ceil(end_bit / 7) near-equal digits.
inline int pass_count(int end_bit) { return (end_bit + kMaxRadixBits - 1) / kMaxRadixBits; }

// Host driver: sorts n items (live count optionally on device) on bits
// [0, end_bit).  Output lands in keys_out/vals_out (unless extra.mode == 2);
// inputs are untouched; vals_in == nullptr sorts the identity permutation.
template <typename K, typename V>
int32_t radix_sort(const K* keys_in, const V* vals_in, K* keys_out, V* vals_out, const int64_t* d_n,
                   int64_t n_max, int end_bit, void* scratch, size_t scratch_bytes, cudaStream_t st,
                   const SortExtra& extra = SortExtra()) {
    if (n_max <= 0) return ADR_OK;
    const int passes = pass_count(end_bit);
    if (extra.dp.plan && (passes != 4 || sizeof(K) != 4))
        return fail(ADR_ERR_VALUE, "radix_sort: a depth plan needs 32-bit keys and 4 passes");
    if (passes == 0 && (!vals_in || extra.mode != 0))
        return fail(ADR_ERR_VALUE, "radix_sort: identity values / extras need >= 1 pass");
    if (passes == 0) {
        ADR_CUDA_TRY(cudaMemcpyAsync(keys_out, keys_in, sizeof(K) * n_max, cudaMemcpyDeviceToDevice, st));
        ADR_CUDA_TRY(cudaMemcpyAsync(vals_out, vals_in, sizeof(V) * n_max, cudaMemcpyDeviceToDevice, st));
        return ADR_OK;
    }
    Carver c(scratch, scratch_bytes);
    K* alt_k = c.take<K>(n_max);
    V* alt_v = c.take<V>(n_max);
    const int64_t nb = ceil_div(n_max, SortCfg<K>::kTileItems);
    uint32_t* hist = c.take<uint32_t>(nb << kMaxRadixBits);
    const int64_t scan_blocks_max = ceil_div(nb << kMaxRadixBits, 256 * 8);
    uint64_t* status = c.take<uint64_t>(scan_blocks_max + 1);
    unsigned long long* counter = reinterpret_cast<unsigned long long*>(status + scan_blocks_max);
    if (!c.ok()) return fail(ADR_ERR_VALUE, "radix_sort: scratch too small");

    const K* src_k = keys_in;
    const V* src_v = vals_in;
    int bit = 0;
    for (int p = 0; p < passes; ++p) {
        const int bits = (end_bit - bit) / (passes - p);  // near-equal split, wider digits last
        const bool to_out = ((passes - 1 - p) % 2) == 0;
        const bool last = p == passes - 1;
        K* dst_k = to_out ? keys_out : alt_k;
        V* dst_v = to_out ? vals_out : alt_v;
        SortExtra pex = extra;
        pex.dp.pass = p;
        const bool plan_block = p == 0 && extra.dp.plan_out;   // pass 0: one extra upsweep block reduces the plan
        if (!plan_block) pex.dp.plan_out = nullptr;
        ADR_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(uint64_t) * (scan_blocks_max + 1), st));
#define ADR_SORT_PASS(RB)                                                                                     \
    do {                                                                                                      \
        radix_upsweep<K, RB><<<nb + (plan_block ? kPlanBlocks : 0), kSortBlock, 0, st>>>(src_k, d_n, n_max,   \
                                                                                          bit, hist,          \
                                                                            pex.dp);                          \
        ADR_LAUNCH_CHECK();                                                                                   \
        const int64_t hl = nb << RB;                                                                          \
        scan_u32_exclusive<8><<<ceil_div(hl, 256 * 8), 256, 0, st>>>(hist, hl, status, counter, pex.dp);      \
        ADR_LAUNCH_CHECK();                                                                                   \
        const size_t dsm = downsweep_smem<K, V, RB>();                                                        \
        const int mode = last ? extra.mode : 0;                                                               \
        (void)mode;                                                                                           \
        if (mode == 1) {                                                                                      \
            ADR_CUDA_TRY(cudaFuncSetAttribute(radix_downsweep<K, V, RB, 1>,                                   \
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));        \
            radix_downsweep<K, V, RB, 1><<<nb, kSortBlock, dsm, st>>>(src_k, src_v, dst_k, dst_v, d_n, n_max,  \
                                                                      bit, hist, pex);                        \
        } else if (mode == 3) {                                                                               \
            ADR_CUDA_TRY(cudaFuncSetAttribute(radix_downsweep<K, V, RB, 3>,                                   \
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));        \
            radix_downsweep<K, V, RB, 3><<<nb, kSortBlock, dsm, st>>>(src_k, src_v, dst_k, dst_v, d_n, n_max,  \
                                                                      bit, hist, pex);                        \
        } else if (mode == 2) {                                                                               \
            ADR_CUDA_TRY(cudaFuncSetAttribute(radix_downsweep<K, V, RB, 2>,                                   \
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));        \
            radix_downsweep<K, V, RB, 2><<<nb, kSortBlock, dsm, st>>>(src_k, src_v, dst_k, dst_v, d_n, n_max,  \
                                                                      bit, hist, pex);                        \
        } else {                                                                                              \
            ADR_CUDA_TRY(cudaFuncSetAttribute(radix_downsweep<K, V, RB, 0>,                                   \
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));        \
            radix_downsweep<K, V, RB, 0><<<nb, kSortBlock, dsm, st>>>(src_k, src_v, dst_k, dst_v, d_n, n_max,  \
                                                                      bit, hist, pex);                        \
        }                                                                                                     \
        ADR_LAUNCH_CHECK();                                                                                   \
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
        bit += bits;
        src_k = dst_k;
        src_v = dst_v;
    }
    return ADR_OK;
}

}  // namespace adr
