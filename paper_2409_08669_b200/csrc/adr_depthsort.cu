// adr_depthsort.cu — the fused frame's depth-rank sort as a onesweep LSD
// radix sort (stable, 8-bit digits) of the N depth keys with the identity as
// values (sb/tiling.py:159-164 ordering: (float32 depth bits, index)).
//
//   k_ds_plan  : kPlanBlocks blocks reduce the preprocess's per-warp key
//                extrema into the key-range plan (adr_sort.cuh DepthPlan:
//                24-bit keys t = key - kmin when they fit, three passes);
//   k_ds_hist0 : the digit histogram of pass 0 (the raw low byte, equal to
//                t's because kmin is a multiple of 256);
//   k_ds_pass  : one kernel per pass.  A block (dynamic id: launch order)
//                ranks its 4096 keys by warp ballots, publishes its per-digit
//                counts, resolves their global offsets by decoupled look-back
//                over the earlier blocks (thread per digit), stages the tile in
//                digit order and writes it out coalesced; meanwhile it
//                histograms the NEXT pass's digit of the keys it holds (order
//                does not matter for a histogram), so no pass needs an upsweep
//                or a histogram scan.  The last pass writes the 16-byte rank
//                records {index, depth bits, tile rect} of adr_supertile.cu.
//
// Decided on the device (fits or not, which pass is last), so the frame stays
// one fixed launch sequence / CUDA graph.
#include "adr_binning.cuh"
#include "adr_sort.cuh"

namespace adr {

namespace {

constexpr int kDsR = 256;                         // 8-bit digits
#ifndef ADR_DS_IPT
#define ADR_DS_IPT 16
#endif
constexpr int kDsIpt = ADR_DS_IPT;                // keys per thread
constexpr int kDsTile = kSortBlock * kDsIpt;      // 4096 keys per block

struct DsBufs {
    uint32_t* hist;        // [4][256] digit histograms (zeroed per frame)
    unsigned long long* tick;  // [4] dynamic block counters (zeroed per frame)
    uint64_t* status;      // [4][nb][256] look-back words (zeroed per frame)
    int64_t nb;
};

__global__ void __launch_bounds__(kSortBlock) k_ds_plan(DepthPlan dp) {
    plan_reduce<kSortBlock>(dp, blockIdx.x);
}

// Pass 0's digit histogram over the raw keys (low byte == t's low byte).
__global__ void __launch_bounds__(kSortBlock) k_ds_hist0(const uint32_t* __restrict__ keys, int64_t n,
                                                         uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kSortWarps][kDsR];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kSortWarps * kDsR; i += kSortBlock) (&h[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kDsTile;
    uint32_t k[kDsIpt];
#pragma unroll
    for (int r = 0; r < kDsIpt; ++r) {
        const int64_t i = base + (int64_t)r * kSortBlock + threadIdx.x;
        k[r] = i < n ? keys[i] : 0u;
    }
#pragma unroll
    for (int r = 0; r < kDsIpt; ++r)
        if (base + (int64_t)r * kSortBlock + threadIdx.x < n) atomicAdd(&h[warp][k[r] & 0xffu], 1u);
    __syncthreads();
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) s += h[w][threadIdx.x];
    if (s) atomicAdd(hist + threadIdx.x, s);
}

// One onesweep pass (see the file comment).  vals_in == nullptr: identity.
#ifndef ADR_DS_MINB
#define ADR_DS_MINB 3
#endif
__global__ void __launch_bounds__(kSortBlock, ADR_DS_MINB)
k_ds_pass(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
          uint32_t* __restrict__ vals_out, int64_t n, int pass, DepthPlan dp, DsBufs b,
          const uint2* __restrict__ gsrc, uint4* __restrict__ rinfo) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* skeys = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* svals = skeys + kDsTile;
    __shared__ uint32_t wh[kSortWarps][kDsR];
    __shared__ uint32_t hn[kSortWarps][kDsR];     // next pass's digit histogram
    __shared__ uint32_t dstart[kDsR];
    __shared__ int64_t goff[kDsR];
    __shared__ uint32_t sred[33];
    __shared__ int64_t sbid;

    uint32_t kmin = 0;
    const bool fits = plan_decode(dp, &kmin);
    if (pass == 3 && fits) return;                // three passes suffice
    const int last_pass = fits ? 2 : 3;
    const bool last = pass == last_pass;
    const int bit = 8 * pass;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kSortWarps * kDsR; i += kSortBlock) {
        (&wh[0][0])[i] = 0;
        (&hn[0][0])[i] = 0;
    }
    const int64_t bid = dynamic_block_id(b.tick + pass, &sbid);   // includes a barrier
    const int64_t base = bid * kDsTile;
    const int64_t wbase = base + (int64_t)warp * 32 * kDsIpt;
    uint32_t kr[kDsIpt], vr[kDsIpt];
#pragma unroll
    for (int r = 0; r < kDsIpt; ++r) {
        const int64_t i = wbase + r * 32 + lane;
        kr[r] = i < n ? keys_in[i] : 0u;
        vr[r] = i < n ? (vals_in ? vals_in[i] : (uint32_t)i) : 0u;
    }
    if (pass == 1 && fits) {   // keys become t = key - kmin (all-ones -> 0xFFFFFF, still last)
#pragma unroll
        for (int r = 0; r < kDsIpt; ++r) kr[r] = kr[r] == 0xffffffffu ? 0xffffffu : kr[r] - kmin;
    }
    const bool full = base + kDsTile <= n;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t live_mask = full ? 0xffffffffu : 0u;
    uint32_t rank2[kDsIpt / 2];
#pragma unroll
    for (int r = 0; r < kDsIpt; ++r) {
        const bool live = full || wbase + r * 32 + lane < n;
        const uint32_t d = (kr[r] >> bit) & 0xffu;
        uint32_t peers = digit_peers<8>(d);
        if (!full) peers &= __ballot_sync(kFull, live) | live_mask;
        const uint32_t before = wh[warp][d];
        __syncwarp();
        if (live && (peers & lt) == 0) wh[warp][d] = before + __popc(peers);
        __syncwarp();
        const uint32_t rk = before + __popc(peers & lt);
        if (r & 1) rank2[r >> 1] |= rk << 16; else rank2[r >> 1] = rk;
        if (!last && live) {   // next pass's digit (pass 0 still holds raw keys: transform for it)
            const uint32_t t = (pass == 0 && fits) ? (kr[r] == 0xffffffffu ? 0xffffffu : kr[r] - kmin) : kr[r];
            atomicAdd(&hn[warp][(t >> (bit + 8)) & 0xffu], 1u);
        }
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, block total, block-local start
    const int dd = threadIdx.x;   // kSortBlock == kDsR
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
        const uint32_t t = wh[w][dd];
        wh[w][dd] = tot;
        tot += t;
    }
    // publish this block's per-digit count, then resolve its exclusive prefix
    // over the earlier blocks (decoupled look-back, thread per digit)
    uint64_t* st = b.status + ((int64_t)pass * b.nb) * kDsR;
    if (bid == 0) {
        st_relaxed(st + dd, kFlagPre | tot);
    } else {
        st_relaxed(st + bid * kDsR + dd, kFlagAgg | tot);
    }
    uint32_t btot;
    const uint32_t dpre = block_exclusive_sum<uint32_t, kSortBlock>(tot, sred, &btot);
    // the pass's global digit starts from its histogram
    uint32_t gtot;
    const uint32_t gstart = block_exclusive_sum<uint32_t, kSortBlock>(__ldcg(b.hist + pass * kDsR + dd), sred, &gtot);
    uint64_t excl = 0;
    if (bid > 0) {
        for (int64_t j = bid - 1;; --j) {   // (8 words per round trip measured no faster)
            uint64_t w = ld_relaxed(st + j * kDsR + dd);
            while ((w >> 62) == 0) w = ld_relaxed(st + j * kDsR + dd);
            excl += w & kValMask;
            if ((w >> 62) == 2) break;
        }
        st_relaxed(st + bid * kDsR + dd, kFlagPre | (excl + tot));
    }
    dstart[dd] = dpre;
    goff[dd] = (int64_t)gstart + (int64_t)excl - (int64_t)dpre;
    if (!last) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) s += hn[w][dd];
        if (s) atomicAdd(b.hist + (pass + 1) * kDsR + dd, s);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kDsIpt; ++r) {
        if (wbase + r * 32 + lane < n) {
            const uint32_t d = (kr[r] >> bit) & 0xffu;
            const uint32_t pos = dstart[d] + wh[warp][d] + ((rank2[r >> 1] >> (16 * (r & 1))) & 0xffffu);
            skeys[pos] = kr[r];
            svals[pos] = vr[r];
        }
    }
    __syncthreads();
    const int live = (int)((n - base) < kDsTile ? (n - base) : kDsTile);
    if (last) {
        // the tile-rect gathers of ADR_DS_GATHER items in flight per thread
        // before their rank records are written
#ifndef ADR_DS_GATHER
#define ADR_DS_GATHER 4
#endif
        constexpr int U = ADR_DS_GATHER;
        for (int i0 = threadIdx.x; i0 < live; i0 += U * kSortBlock) {
            uint32_t key[U], val[U];
            uint2 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * kSortBlock;
                key[u] = i < live ? skeys[i] : 0u;
                val[u] = i < live ? svals[i] : 0u;
                r[u] = i < live ? __ldg(gsrc + val[u]) : make_uint2(0u, 0u);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * kSortBlock;
                if (i < live) {
                    const int64_t g = goff[(key[u] >> bit) & 0xffu] + i;
                    const uint32_t kk = fits ? (key[u] == 0xffffffu ? 0xffffffffu : key[u] + kmin) : key[u];
                    rinfo[g] = make_uint4(val[u], kk, r[u].x, r[u].y);
                }
            }
        }
        return;
    }
    for (int i = threadIdx.x; i < live; i += kSortBlock) {
        const uint32_t key = skeys[i];
        const int64_t g = goff[(key >> bit) & 0xffu] + i;
        keys_out[g] = key;
        vals_out[g] = svals[i];
    }
}

}  // namespace

size_t depth_sort_scratch(int64_t n) {
    const int64_t nb = ceil_div(n > 0 ? n : 1, kDsTile);
    return 2 * align_up(4 * (size_t)n) * 2                      // keys / values ping-pong
           + align_up(4 * 4 * kDsR + 8 * 4)                      // histograms + tick counters
           + align_up(8 * (size_t)(4 * nb * kDsR)) + 1024;       // look-back status
}

int32_t depth_sort_onesweep(const uint32_t* dkey, int64_t n, const DepthPlan& dp_in, const uint2* gpack,
                            uint4* rinfo, void* scratch, size_t scratch_bytes, cudaStream_t st) {
    if (n <= 0) return ADR_OK;
    const int64_t nb = ceil_div(n, kDsTile);
    Carver c(scratch, scratch_bytes);
    uint32_t* ka = c.take<uint32_t>(n);
    uint32_t* va = c.take<uint32_t>(n);
    uint32_t* kb = c.take<uint32_t>(n);
    uint32_t* vb = c.take<uint32_t>(n);
    char* zero0 = reinterpret_cast<char*>(c.take<uint32_t>(4 * kDsR + 8));
    uint64_t* status = c.take<uint64_t>(4 * nb * kDsR);
    if (!c.ok()) return fail(ADR_ERR_VALUE, "depth sort: scratch too small");
    DsBufs b;
    b.hist = reinterpret_cast<uint32_t*>(zero0);
    b.tick = reinterpret_cast<unsigned long long*>(b.hist + 4 * kDsR);
    b.status = status;
    b.nb = nb;
    // histograms, counters and look-back words start at zero (one memset:
    // they are contiguous in the scratch)
    const size_t zbytes = reinterpret_cast<char*>(status + 4 * nb * kDsR) - zero0;
    ADR_CUDA_TRY(cudaMemsetAsync(zero0, 0, zbytes, st));
    DepthPlan dp = dp_in;
    if (dp.plan_out) {
        k_ds_plan<<<kPlanBlocks, kSortBlock, 0, st>>>(dp);
        ADR_LAUNCH_CHECK();
    }
    dp.plan_out = nullptr;
    k_ds_hist0<<<(unsigned)nb, kSortBlock, 0, st>>>(dkey, n, b.hist);
    ADR_LAUNCH_CHECK();
    const size_t sm = 2 * sizeof(uint32_t) * kDsTile;
    static bool attr = false;
    if (!attr) {
        ADR_CUDA_TRY(cudaFuncSetAttribute(k_ds_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr = true;
    }
    const uint32_t* kin[4] = {dkey, ka, kb, ka};
    const uint32_t* vin[4] = {nullptr, va, vb, va};
    uint32_t* kout[4] = {ka, kb, ka, kb};
    uint32_t* vout[4] = {va, vb, va, vb};
    for (int p = 0; p < 4; ++p) {
        k_ds_pass<<<(unsigned)nb, kSortBlock, sm, st>>>(kin[p], vin[p], kout[p], vout[p], n, p, dp, b, gpack,
                                                        rinfo);
        ADR_LAUNCH_CHECK();
    }
    return ADR_OK;
}

}  // namespace adr
