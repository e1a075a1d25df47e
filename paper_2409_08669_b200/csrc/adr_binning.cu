// adr_binning.cu — stages 2-5 (sb/tiling.py) as stage-API kernels, plus the
// fused frame's binning kernels (compaction, rank-ordered emission, ranges).
#include "adr_binning.cuh"
#include "adr_sort.cuh"

namespace adr {

// ------------------------------------------------------------- stage API

namespace {

__global__ void k_touched_counts(const float2* __restrict__ mean2d, const int32_t* __restrict__ ext_x,
                                 const int32_t* __restrict__ ext_y, const uint8_t* __restrict__ valid,
                                 int64_t n, int32_t tiles_x, int32_t tiles_y, int64_t* __restrict__ counts) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float2 m = mean2d[i];
    counts[i] = tile_rect(m.x, m.y, ext_x[i], ext_y[i], valid[i] != 0, tiles_x, tiles_y).count();
}

// int64 inclusive sum, reduce-then-scan.  Phase 1: per-block sums (wrapping
// int64) plus exact __int128 totals for the overflow check of
// sb/tiling.py:120-121.
constexpr int kScanBlock = 256, kScanIpt = 8, kScanTile = kScanBlock * kScanIpt;

__global__ void k_sum64_reduce(const int64_t* __restrict__ in, int64_t n, int64_t* __restrict__ bsum,
                               __int128* __restrict__ bsum_exact) {
    __shared__ __int128 sh[kScanBlock / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    __int128 acc = 0;
    for (int k = 0; k < kScanIpt; ++k) {
        const int64_t i = base + (int64_t)k * kScanBlock + threadIdx.x;
        if (i < n) acc += in[i];
    }
    // warp reduce of 128-bit via two 64-bit shuffles
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t lo = __shfl_xor_sync(kFull, (uint64_t)acc, o);
        const int64_t hi = __shfl_xor_sync(kFull, (int64_t)(acc >> 64), o);
        acc += ((__int128)hi << 64) | (__int128)lo;
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        __int128 t = 0;
        for (int w = 0; w < kScanBlock / 32; ++w) t += sh[w];
        bsum_exact[blockIdx.x] = t;
        bsum[blockIdx.x] = (int64_t)(uint64_t)t;
    }
}

// Phase 2: one block scans the block sums (exclusive, wrapping) and checks the
// exact total against INT64_MAX.
__global__ void k_sum64_blocks(int64_t* __restrict__ bsum, const __int128* __restrict__ bsum_exact,
                               int64_t nb, int32_t* __restrict__ overflow) {
    __shared__ int64_t sred[33];
    __shared__ __int128 sexact;
    if (threadIdx.x == 0) sexact = 0;
    __syncthreads();
    int64_t carry = 0;
    __int128 exact = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += kScanBlock) {
        const int64_t b = b0 + threadIdx.x;
        const int64_t v = b < nb ? bsum[b] : 0;
        if (b < nb) exact += bsum_exact[b];
        int64_t tot;
        const int64_t ex = (int64_t)block_exclusive_sum<uint64_t, kScanBlock>((uint64_t)v, (uint64_t*)sred, (uint64_t*)&tot);
        if (b < nb) bsum[b] = (int64_t)((uint64_t)carry + (uint64_t)ex);
        carry = (int64_t)((uint64_t)carry + (uint64_t)tot);
    }
    // exact total across threads
    for (int t = 0; t < kScanBlock; ++t) {
        if (threadIdx.x == t) sexact += exact;
        __syncthreads();
    }
    if (threadIdx.x == 0 && overflow) *overflow = sexact > (__int128)INT64_MAX ? 1 : 0;
}

// Phase 3: per-block inclusive scan seeded by the block prefix.
__global__ void k_sum64_scan(const int64_t* __restrict__ in, int64_t n, const int64_t* __restrict__ bpre,
                             int64_t* __restrict__ out) {
    __shared__ uint64_t sred[33];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIpt;
    uint64_t v[kScanIpt];
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanIpt; ++k) {
        v[k] = base + k < n ? (uint64_t)in[base + k] : 0;
        s += v[k];
    }
    uint64_t tot;
    uint64_t run = block_exclusive_sum<uint64_t, kScanBlock>(s, sred, &tot) + (uint64_t)bpre[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanIpt; ++k) {
        run += v[k];
        if (base + k < n) out[base + k] = (int64_t)run;
    }
}

__global__ void k_duplicate(const float2* __restrict__ mean2d, const int32_t* __restrict__ ext_x,
                            const int32_t* __restrict__ ext_y, const uint8_t* __restrict__ valid,
                            const float* __restrict__ depth, const int64_t* __restrict__ offsets, int64_t n,
                            int32_t tiles_x, int32_t tiles_y, uint64_t* __restrict__ keys,
                            int64_t* __restrict__ gidx) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const float2 m = mean2d[g];
    const Rect r = tile_rect(m.x, m.y, ext_x[g], ext_y[g], valid[g] != 0, tiles_x, tiles_y);
    int64_t o = offsets[g] - r.count();
    const uint64_t db = __float_as_uint(depth[g]);
    for (int32_t ty = r.y0; ty < r.y1; ++ty)
        for (int32_t tx = r.x0; tx < r.x1; ++tx) {
            keys[o] = ((uint64_t)((int64_t)ty * tiles_x + tx) << 32) | db;
            gidx[o] = g;
            ++o;
        }
}

// ranges[t] = (lower_bound(t), lower_bound(t+1)) over tile ids of sorted
// keys; one thread per boundary position i in [0, P].
template <typename Tile>
__device__ __forceinline__ void write_bounds(int64_t i, int64_t t_prev, int64_t t_cur, int64_t n_tiles,
                                             int64_t* ranges) {
    for (int64_t t = t_prev + 1; t <= t_cur; ++t) {
        if (t < n_tiles) ranges[2 * t] = i;
        if (t > 0) ranges[2 * (t - 1) + 1] = i;
    }
}

__global__ void k_ranges_u64(const uint64_t* __restrict__ keys, int64_t p, int64_t n_tiles,
                             int64_t* __restrict__ ranges, int32_t* __restrict__ error) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > p) return;
    const int64_t t_prev = i == 0 ? -1 : (int64_t)(keys[i - 1] >> 32);
    int64_t t_cur = n_tiles;
    if (i < p) {
        const uint64_t k = keys[i];
        t_cur = (int64_t)(k >> 32);
        if (i > 0 && k < keys[i - 1]) atomicMax(error, 1);
        if (i == p - 1 && t_cur >= n_tiles) atomicMax(error, 2);
        if (t_cur > n_tiles) t_cur = n_tiles;
    }
    write_bounds<uint64_t>(i, t_prev < n_tiles ? t_prev : n_tiles, t_cur, n_tiles, ranges);
}

}  // namespace

int32_t stage_touched_counts(const adr_projection& p, int64_t n, int32_t tx, int32_t ty, int64_t* counts,
                             cudaStream_t st) {
    if (n <= 0) return ADR_OK;
    k_touched_counts<<<ceil_div(n, 256), 256, 0, st>>>(reinterpret_cast<const float2*>(p.d_mean2d), p.d_ext_x,
                                                       p.d_ext_y, p.d_valid, n, tx, ty, counts);
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

size_t stage_inclusive_sum_scratch(int64_t n) {
    const int64_t nb = ceil_div(n > 0 ? n : 1, kScanTile);
    return align_up(sizeof(int64_t) * nb) + align_up(sizeof(__int128) * nb) + 256;
}

int32_t stage_inclusive_sum(const int64_t* in, int64_t n, int64_t* out, int32_t* overflow, void* scratch,
                            size_t bytes, cudaStream_t st) {
    if (overflow) ADR_CUDA_TRY(cudaMemsetAsync(overflow, 0, sizeof(int32_t), st));
    if (n <= 0) return ADR_OK;
    const int64_t nb = ceil_div(n, kScanTile);
    Carver c(scratch, bytes);
    int64_t* bsum = c.take<int64_t>(nb);
    __int128* bex = c.take<__int128>(nb);
    if (!c.ok()) return fail(ADR_ERR_VALUE, "inclusive_sum: scratch too small");
    k_sum64_reduce<<<nb, kScanBlock, 0, st>>>(in, n, bsum, bex);
    ADR_LAUNCH_CHECK();
    k_sum64_blocks<<<1, kScanBlock, 0, st>>>(bsum, bex, nb, overflow);
    ADR_LAUNCH_CHECK();
    k_sum64_scan<<<nb, kScanBlock, 0, st>>>(in, n, bsum, out);
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

int32_t stage_duplicate(const adr_projection& p, int64_t n, const int64_t* offsets, int32_t tx, int32_t ty,
                        uint64_t* keys, int64_t* gidx, cudaStream_t st) {
    if (n <= 0) return ADR_OK;
    k_duplicate<<<ceil_div(n, 128), 128, 0, st>>>(reinterpret_cast<const float2*>(p.d_mean2d), p.d_ext_x,
                                                  p.d_ext_y, p.d_valid, p.d_depth, offsets, n, tx, ty, keys, gidx);
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

size_t stage_sort_scratch(int64_t p) { return radix_scratch_bytes<uint64_t, int64_t>(p); }

int32_t stage_sort(const uint64_t* k, const int64_t* v, int64_t p, int32_t end_bit, uint64_t* ko, int64_t* vo,
                   void* scratch, size_t bytes, cudaStream_t st) {
    if (end_bit < 0 || end_bit > 64) return fail(ADR_ERR_VALUE, "end_bit must be in [0, 64]");
    return radix_sort<uint64_t, int64_t>(k, v, ko, vo, nullptr, p, end_bit, scratch, bytes, st);
}

int32_t stage_ranges(const uint64_t* keys, int64_t p, int64_t n_tiles, int64_t* ranges, int32_t* error,
                     cudaStream_t st) {
    ADR_CUDA_TRY(cudaMemsetAsync(error, 0, sizeof(int32_t), st));
    if (n_tiles <= 0) return ADR_OK;
    k_ranges_u64<<<ceil_div(p + 1, 256), 256, 0, st>>>(keys, p, n_tiles, ranges, error);
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

// ------------------------------------------------------------ fused frame

namespace {

constexpr int kLbBlock = 256, kLbIpt = 8, kLbTile = kLbBlock * kLbIpt;

// Generic single-pass exclusive scan with decoupled look-back; Op supplies
// load(i) -> u64, store(i, exclusive, value) and total(sum).
template <class Op>
__global__ void __launch_bounds__(kLbBlock)
k_scan_lookback(Op op, const int64_t* d_n, int64_t n_static, uint64_t* status, unsigned long long* counter) {
    __shared__ int64_t sbid;
    __shared__ uint64_t sred[33];
    __shared__ uint64_t sexcl;
    const int64_t n = d_n ? *d_n : n_static;
    const int64_t bid = dynamic_block_id(counter, &sbid);
    const int64_t base = bid * kLbTile + (int64_t)threadIdx.x * kLbIpt;
    uint64_t v[kLbIpt];
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < kLbIpt; ++k) {
        v[k] = base + k < n ? op.load(base + k) : 0ull;
        s += v[k];
    }
    uint64_t btot;
    const uint64_t tpre = block_exclusive_sum<uint64_t, kLbBlock>(s, sred, &btot);
    if (threadIdx.x < 32) {
        const uint64_t e = lookback(status, bid, btot);
        if (threadIdx.x == 0) sexcl = e;
    }
    __syncthreads();
    uint64_t run = sexcl + tpre;
#pragma unroll
    for (int k = 0; k < kLbIpt; ++k) {
        if (base + k < n) op.store(base + k, run, v[k]);
        run += v[k];
    }
    if (bid == (int64_t)gridDim.x - 1 && threadIdx.x == kLbBlock - 1) op.total(run);
}

// Compaction of the Gaussians that touch >= 1 tile, in index order, keyed by
// their float32 depth bits (positive: depth > near_plane > 0).
struct SelectOp {
    const uint32_t* cnt;
    const float* depth;
    uint32_t* sel_key;
    uint32_t* sel_idx;
    int64_t* d_m;
    __device__ uint64_t load(int64_t i) const { return cnt[i] != 0u ? 1ull : 0ull; }
    __device__ void store(int64_t i, uint64_t ex, uint64_t v) const {
        if (v) {
            sel_key[ex] = __float_as_uint(depth[i]);
            sel_idx[ex] = (uint32_t)i;
        }
    }
    __device__ void total(uint64_t t) const { *d_m = (int64_t)t; }
};

// Pair offsets in depth-rank order: off[r] = sum_{r' < r} cnt[order[r']].
struct OffsetsOp {
    const uint32_t* cnt;
    const uint32_t* order;
    uint32_t* off;
    int64_t* d_p;        // true pair count
    int64_t* d_pc;       // pair count clamped to capacity
    int64_t cap;
    __device__ uint64_t load(int64_t r) const { return cnt[order[r]]; }
    __device__ void store(int64_t r, uint64_t ex, uint64_t) const {
        off[r] = ex < (uint64_t)cap ? (uint32_t)ex : (uint32_t)cap;
    }
    __device__ void total(uint64_t t) const {
        *d_p = (int64_t)t;
        *d_pc = t < (uint64_t)cap ? (int64_t)t : cap;
    }
};

// Emission in depth-rank order: rank r writes (tile, r) for every tile of its
// rectangle, row-major, and its render record.  Because ranks are ordered by
// (depth bits, Gaussian index), a stable sort of this stream by tile alone is
// exactly np.argsort(keys, kind="stable") of the reference (tiling.py:159-164).
template <typename TileT>
__global__ void k_emit(const uint32_t* __restrict__ order, const uint32_t* __restrict__ off,
                       const int64_t* __restrict__ d_m, const adr_projection proj, int32_t tiles_x,
                       int32_t tiles_y, int64_t cap, TileT* __restrict__ tiles, uint32_t* __restrict__ ranks,
                       Record* __restrict__ rec) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= *d_m) return;
    const uint32_t g = order[r];
    const float2 m = reinterpret_cast<const float2*>(proj.d_mean2d)[g];
    const Rect rc = tile_rect(m.x, m.y, proj.d_ext_x[g], proj.d_ext_y[g], true, tiles_x, tiles_y);
    int64_t o = off[r];
    for (int32_t ty = rc.y0; ty < rc.y1; ++ty)
        for (int32_t tx = rc.x0; tx < rc.x1; ++tx) {
            if (o < cap) {
                tiles[o] = (TileT)(ty * tiles_x + tx);
                ranks[o] = (uint32_t)r;
            }
            ++o;
        }
    Record R;
    R.a = make_float4(m.x, m.y, proj.d_conic[3 * g], proj.d_conic[3 * g + 1]);
    R.b = make_float4(proj.d_conic[3 * g + 2], proj.d_opacity[g], proj.d_color[3 * g], proj.d_color[3 * g + 1]);
    R.c = make_float4(proj.d_color[3 * g + 2], 0.f, 0.f, 0.f);
    rec[r] = R;
}

template <typename TileT>
__global__ void k_ranges_tiles(const TileT* __restrict__ tiles, const int64_t* __restrict__ d_p, int64_t n_tiles,
                               int64_t* __restrict__ ranges) {
    const int64_t p = *d_p;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= p; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t_prev = i == 0 ? -1 : (int64_t)tiles[i - 1];
        const int64_t t_cur = i < p ? (int64_t)tiles[i] : n_tiles;
        write_bounds<TileT>(i, t_prev, t_cur, n_tiles, ranges);
    }
}

template <typename TileT>
__global__ void k_export(const TileT* __restrict__ tiles, const uint32_t* __restrict__ ranks,
                         const uint32_t* __restrict__ order, const float* __restrict__ depth,
                         const int64_t* __restrict__ d_p, uint64_t* __restrict__ keys, int32_t* __restrict__ gidx) {
    const int64_t p = *d_p;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t g = order[ranks[i]];
        if (keys) keys[i] = ((uint64_t)tiles[i] << 32) | __float_as_uint(depth[g]);
        if (gidx) gidx[i] = (int32_t)g;
    }
}

int grid_stride_blocks(int64_t work, int block) {
    int64_t b = ceil_div(work > 0 ? work : 1, block);
    const int64_t cap = 148 * 16;
    return (int)(b < cap ? b : cap);
}

}  // namespace

size_t frame_binning_scratch(int64_t n, int64_t cap, int64_t n_tiles) {
    const bool wide = n_tiles > 65536;
    const size_t tile_sz = wide ? 4 : 2;
    const int64_t nlb = ceil_div(n > 0 ? n : 1, kLbTile);
    size_t s = 0;
    s += align_up(4 * (size_t)n) * 6;                       // cnt, sel_key, sel_idx, skey, order, off
    s += align_up(sizeof(Record) * (size_t)n);              // records
    s += radix_scratch_bytes<uint32_t, uint32_t>(n);
    s += 2 * (align_up(tile_sz * (size_t)cap) + align_up(4 * (size_t)cap));  // tiles, ranks (+sorted)
    s += wide ? radix_scratch_bytes<uint32_t, uint32_t>(cap) : radix_scratch_bytes<uint16_t, uint32_t>(cap);
    s += 2 * lookback_bytes(nlb);
    return s + 4096;
}

template <typename TileT>
static int32_t frame_binning_t(const FrameBinning& fb, cudaStream_t st) {
    Carver c(fb.scratch, fb.scratch_bytes);
    const int64_t n = fb.n, cap = fb.cap;
    uint32_t* cnt = fb.cnt;
    uint32_t* sel_key = c.take<uint32_t>(n);
    uint32_t* sel_idx = c.take<uint32_t>(n);
    uint32_t* skey = c.take<uint32_t>(n);
    uint32_t* order = fb.order;
    uint32_t* off = c.take<uint32_t>(n);
    Record* rec = fb.rec;
    void* rs1 = c.take<char>((int64_t)radix_scratch_bytes<uint32_t, uint32_t>(n));
    TileT* tiles = c.take<TileT>(cap);
    uint32_t* ranks = c.take<uint32_t>(cap);
    TileT* stiles = c.take<TileT>(cap);
    uint32_t* sranks = fb.sorted_ranks;
    void* rs2 = c.take<char>((int64_t)radix_scratch_bytes<TileT, uint32_t>(cap));
    const int64_t nlb = ceil_div(n, kLbTile);
    uint64_t* st1 = c.take<uint64_t>(nlb + 1);
    uint64_t* st2 = c.take<uint64_t>(nlb + 1);
    if (!c.ok()) return fail(ADR_ERR_VALUE, "render_frame: scratch too small");
    int64_t* ctr = fb.counters;  // [0]=P, [1]=culled, [2]=M, [3]=P clamped

    // (a) compaction of Gaussians with pairs, keyed by depth bits
    ADR_CUDA_TRY(cudaMemsetAsync(st1, 0, sizeof(uint64_t) * (nlb + 1), st));
    SelectOp sel{cnt, fb.proj.d_depth, sel_key, sel_idx, ctr + 2};
    k_scan_lookback<SelectOp><<<nlb, kLbBlock, 0, st>>>(sel, nullptr, n, st1, reinterpret_cast<unsigned long long*>(st1 + nlb));
    ADR_LAUNCH_CHECK();
    // (b) stable depth sort of the M survivors -> order[rank] (ties by index)
    int32_t rc = radix_sort<uint32_t, uint32_t>(sel_key, sel_idx, skey, order, ctr + 2, n, 31, rs1,
                                                radix_scratch_bytes<uint32_t, uint32_t>(n), st);
    if (rc) return rc;
    // (c) pair offsets in rank order, P
    ADR_CUDA_TRY(cudaMemsetAsync(st2, 0, sizeof(uint64_t) * (nlb + 1), st));
    OffsetsOp oo{cnt, order, off, ctr + 0, ctr + 3, cap};
    k_scan_lookback<OffsetsOp><<<nlb, kLbBlock, 0, st>>>(oo, ctr + 2, n, st2, reinterpret_cast<unsigned long long*>(st2 + nlb));
    ADR_LAUNCH_CHECK();
    if (fb.ev_after_scan) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_scan, st));
    // (d) emission + records
    k_emit<TileT><<<ceil_div(n, 128), 128, 0, st>>>(order, off, ctr + 2, fb.proj, fb.tiles_x, fb.tiles_y, cap, tiles,
                                                    ranks, rec);
    ADR_LAUNCH_CHECK();
    if (fb.ev_after_dup) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_dup, st));
    // (e) stable sort by tile id
    int tbits = 0;
    while ((int64_t(1) << tbits) < fb.n_tiles) ++tbits;
    rc = radix_sort<TileT, uint32_t>(tiles, ranks, stiles, sranks, ctr + 3, cap, tbits, rs2,
                                     radix_scratch_bytes<TileT, uint32_t>(cap), st);
    if (rc) return rc;
    if (fb.ev_after_sort) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_sort, st));
    // (f) tile ranges
    k_ranges_tiles<TileT><<<grid_stride_blocks(cap + 1, 256), 256, 0, st>>>(stiles, ctr + 3, fb.n_tiles, fb.ranges);
    ADR_LAUNCH_CHECK();
    // (g) export of the reference-layout sorted keys / Gaussian indices
    if (fb.keys || fb.gidx) {
        k_export<TileT><<<grid_stride_blocks(cap, 256), 256, 0, st>>>(stiles, sranks, order, fb.proj.d_depth, ctr + 3,
                                                                     fb.keys, fb.gidx);
        ADR_LAUNCH_CHECK();
    }
    if (fb.ev_after_ranges) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_ranges, st));
    return ADR_OK;
}

int32_t frame_binning(const FrameBinning& fb, cudaStream_t st) {
    if (fb.n <= 0) return ADR_OK;
    if (fb.n >= (int64_t(1) << 31)) return fail(ADR_ERR_CAPACITY, "more than 2^31 Gaussians");
    if (fb.cap >= (int64_t(1) << 31)) return fail(ADR_ERR_CAPACITY, "pair capacity must be < 2^31");
    return fb.n_tiles > 65536 ? frame_binning_t<uint32_t>(fb, st) : frame_binning_t<uint16_t>(fb, st);
}

}  // namespace adr
