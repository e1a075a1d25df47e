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



// Pair offsets in rank order without a separate offsets array: the stream
// is cut into chunks of 256 ranks (one emission block each); this pass sums
// each chunk's rect areas, k_chunk_scan turns the sums into chunk offsets and
// P, and the emission block scans its own 256 areas.
__global__ void __launch_bounds__(256) k_chunk_area_sums(const uint2* __restrict__ rect, const int64_t* __restrict__ d_m,
                                                         int64_t nc, uint64_t* __restrict__ csum) {
    // warp per 256-rank chunk, 8 consecutive ranks per lane (four 16-byte loads)
    const int64_t chunk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (chunk >= nc) return;
    const int64_t m = *d_m;
    const int64_t r0 = chunk * 256 + (int64_t)(threadIdx.x & 31) * 8;
    uint64_t a = 0;
    if (r0 + 8 <= m) {
        const uint4* q = reinterpret_cast<const uint4*>(rect + r0);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint4 t = q[k];
            a += (uint64_t)((t.x >> 16) - (t.x & 0xffffu)) * ((t.y >> 16) - (t.y & 0xffffu));
            a += (uint64_t)((t.z >> 16) - (t.z & 0xffffu)) * ((t.w >> 16) - (t.w & 0xffffu));
        }
    } else {
        for (int64_t r = r0; r < r0 + 8 && r < m; ++r) {
            const uint2 inf = rect[r];
            a += (uint64_t)((inf.x >> 16) - (inf.x & 0xffffu)) * ((inf.y >> 16) - (inf.y & 0xffffu));
        }
    }
    a = warp_sum(a);
    if ((threadIdx.x & 31) == 0) csum[chunk] = a;
}

// Exclusive scan of the chunk sums in place (one block); P and P clamped to
// the pair capacity go to the counters.
__global__ void __launch_bounds__(1024) k_chunk_scan(uint64_t* __restrict__ csum, int64_t nc, int64_t* __restrict__ d_p,
                                                     int64_t* __restrict__ d_pc, int64_t cap) {
    // warp w owns the contiguous segment [w*seg, (w+1)*seg), read in coalesced
    // rounds of 32: pass 1 sums it, a block scan of the 32 warp sums gives each
    // segment's start, pass 2 (L1-resident re-read) writes the prefixes
    __shared__ uint64_t sred[33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t seg = (nc + 31) / 32, s0 = (int64_t)warp * seg;
    const int64_t s1 = s0 + seg < nc ? s0 + seg : nc;
    uint64_t sum = 0;
    for (int64_t i = s0 + lane; i < s1; i += 32) sum += csum[i];
    sum = warp_sum(sum);
    uint64_t tot;
    uint64_t run = block_exclusive_sum<uint64_t, 1024>(lane == 0 ? sum : 0ull, sred, &tot);
    run = __shfl_sync(kFull, run, 0);
    for (int64_t base = s0; base < s1; base += 32) {
        const int64_t i = base + lane;
        const uint64_t v = i < s1 ? csum[i] : 0ull;
        const uint64_t inc = warp_inclusive_sum(v);
        if (i < s1) csum[i] = run + inc - v;
        run += __shfl_sync(kFull, inc, 31);
    }
    if (threadIdx.x == 0) {
        *d_p = (int64_t)tot;
        *d_pc = tot < (uint64_t)cap ? (int64_t)tot : cap;
        d_pc[3] = tot > (uint64_t)cap ? 1 : 0;   // counters[6]: frame truncated
    }
}

// ---- rank-ordered pair stream ---------------------------------------------
// Rank r owns stream positions [off[r], off[r+1]), row-major over its tile
// rectangle.  A stable sort of this stream by tile is exactly the reference's
// np.argsort(keys, kind="stable") (tiling.py:159-164) because ranks are
// ordered by (depth bits, Gaussian index).

// Balanced emission: a warp owns 32 consecutive ranks and the contiguous
// stream range [off[r0], off[r0 + 32]); lane l writes positions
// wstart + l, wstart + l + 32, ... (coalesced stores), finding each position's
// owner among the warp's ranks with a 5-step shuffle search over the lanes'
// start offsets, so lanes do equal work however uneven the rectangles are.
template <typename TileT>
__global__ void __launch_bounds__(256)
k_emit_balanced(const uint2* __restrict__ rect, const uint32_t* __restrict__ order, const uint64_t* __restrict__ coff,
                const int64_t* __restrict__ d_m,
                const int64_t* __restrict__ d_pc, int32_t tiles_x, TileT* __restrict__ tiles, uint32_t* __restrict__ gs) {
    __shared__ uint64_t sred[33];
    __shared__ uint32_t sred32[33];
    const int lane = threadIdx.x & 31;
    const uint32_t m = (uint32_t)*d_m;
    const uint32_t pc = (uint32_t)*d_pc;
    const uint32_t r = blockIdx.x * 256u + threadIdx.x;   // the block is one 256-rank chunk
    const uint32_t r0 = r - (uint32_t)lane;
    const bool valid = r < m;
    const uint2 inf = valid ? rect[r] : make_uint2(0, 0);
    const uint32_t gidx = valid ? order[r] : 0u;
    // this rank's stream offset: chunk offset + exclusive scan of the chunk's areas
    const uint64_t area = (uint64_t)((inf.x >> 16) - (inf.x & 0xffffu)) * ((inf.y >> 16) - (inf.y & 0xffffu));
    uint64_t g64;
    if constexpr (sizeof(TileT) == 2) {   // areas <= 2^16 tiles, a chunk's sum < 2^24: 32-bit scan
        uint32_t btot;
        g64 = coff[blockIdx.x] + block_exclusive_sum<uint32_t, 256>((uint32_t)area, sred32, &btot);
    } else {
        uint64_t btot;
        g64 = coff[blockIdx.x] + block_exclusive_sum<uint64_t, 256>(area, sred, &btot);
    }
    if (r0 >= m) return;
    const uint32_t o = valid ? (g64 < pc ? (uint32_t)g64 : pc) : pc;
    const uint32_t wstart = __shfl_sync(kFull, o, 0);
    const uint64_t wend64 = __shfl_sync(kFull, g64 + area, 31);   // invalid lanes have area 0
    const uint32_t wend = wend64 < pc ? (uint32_t)wend64 : pc;
    const uint32_t x0 = inf.x & 0xffffu, w = (inf.x >> 16) - x0, y0 = inf.y & 0xffffu;
    const float rw = w ? __frcp_rn((float)w) : 0.0f;
    const uint32_t xy0 = x0 | (y0 << 16);
    // u16 tile ids (<= 65536 tiles, so every rect area j < 2^16): position j
    // of a rect is tile t0 + j + row * (tiles_x - w) with row = floor(j / w)
    // = floor((j + 0.5) * RN(1/w)) exactly — (j + 0.5) / w stays >= 0.5 / w
    // from an integer, far more than the <= 2 ulp product error
    const uint32_t t0 = y0 * (uint32_t)tiles_x + x0, dw = (uint32_t)tiles_x - w;
    for (uint32_t base = wstart; base < wend; base += 32) {
        const uint32_t q = base + lane;
        // owner of position q: (ranks starting at or before q) - 1, from a
        // ballot of the ranks that start before this window and the OR of
        // the in-window start bits (starts are distinct: every rank owns >= 1)
        const uint32_t before = __popc(__ballot_sync(kFull, valid && o < base));
        const uint32_t d = o - base;
        const uint32_t starts = __reduce_or_sync(kFull, (valid && o >= base && d < 32u) ? (1u << d) : 0u);
        const int L = (int)(before + __popc(starts & ((2u << lane) - 1u))) - 1;
        const uint32_t oL = __shfl_sync(kFull, o, L);
        const float rwL = __shfl_sync(kFull, rw, L);
        const uint32_t gL = __shfl_sync(kFull, gidx, L);
        if constexpr (sizeof(TileT) == 2) {
            const uint32_t tL = __shfl_sync(kFull, t0, L);
            const uint32_t dL = __shfl_sync(kFull, dw, L);
            if (q < wend) {
                const uint32_t j = q - oL;
                const uint32_t row = (uint32_t)(__fadd_rn((float)j, 0.5f) * rwL);
                tiles[q] = (TileT)(tL + j + row * dL);
                gs[q] = gL;
            }
        } else {
            const uint32_t wL = __shfl_sync(kFull, w, L);
            const uint32_t xyL = __shfl_sync(kFull, xy0, L);
            if (q < wend) {
                const uint32_t j = q - oL;
                uint32_t row = (uint32_t)((float)j * rwL);
                int32_t col = (int32_t)j - (int32_t)(row * wL);
                if (col < 0) { --row; col += (int32_t)wL; }
                if (col >= (int32_t)wL) { ++row; col -= (int32_t)wL; }
                tiles[q] = (TileT)(((xyL >> 16) + row) * (uint32_t)tiles_x + (xyL & 0xffffu) + (uint32_t)col);
                gs[q] = gL;
            }
        }
    }
}

// Tile ranges by search instead of a scan of all P sorted tile ids: warp t
// finds lower_bound(t) with a 32-ary search (each step probes 32 evenly spaced
// positions of the current interval and keeps the one gap where the ids cross
// t), so the whole pass reads ~(T + 1) * 32 * log32(P) ids instead of P.
// ranges[t] = (lb(t), lb(t + 1)); lb(T) = P closes the last tile.
// tile id of sorted position q: the sorted tile array, or the high word of
// the exported reference key (the last sort pass then skips the tile copy)
template <typename TileT>
struct TileIds {
    const TileT* tiles;
    const uint64_t* keys;
    __device__ __forceinline__ int64_t operator[](int64_t q) const {
        return keys ? (int64_t)(keys[q] >> 32) : (int64_t)tiles[q];
    }
};

template <typename TileT>
__global__ void __launch_bounds__(256) k_ranges_search(TileIds<TileT> tiles, const int64_t* __restrict__ d_p,
                                                       int64_t n_tiles, int64_t* __restrict__ ranges,
                                                       adr_load_stats* stats) {
    const int lane = threadIdx.x & 31;
    if (stats && blockIdx.x == 0 && threadIdx.x == 0) {   // the render's load-statistics accumulators
        stats->sum = 0;
        stats->sum_sq = 0;
        stats->min = INT_MAX;
        stats->max = INT_MIN;
    }
    const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (t > n_tiles) return;
    const int64_t p = *d_p;
    int64_t lo = 0, hi = p;   // lb(t) in [lo, hi]
    while (hi - lo > 32) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t q = lo + lane * step;
        const bool below = q < hi && tiles[q] < t;
        const int c = __popc(__ballot_sync(kFull, below));
        const int64_t nlo = c > 0 ? lo + (int64_t)(c - 1) * step + 1 : lo;
        const int64_t qc = lo + (int64_t)c * step;
        hi = (c < 32 && qc < hi) ? qc : hi;
        lo = nlo;
    }
    const bool below = lo + lane < hi && tiles[lo + lane] < t;
    const int64_t lb = lo + __popc(__ballot_sync(kFull, below));
    if (lane == 0) {
        if (t < n_tiles) ranges[2 * t] = lb;
        if (t > 0) ranges[2 * (t - 1) + 1] = lb;
    }
}

}  // namespace

size_t frame_binning_scratch(int64_t n, int64_t cap, int32_t tiles_x, int32_t tiles_y) {
    const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
    if (supertile_path(n_tiles, tiles_x, tiles_y)) return supertile_scratch(n, cap, tiles_x, tiles_y);
    const int64_t nc = ceil_div(n > 0 ? n : 1, 256);
    const bool wide = n_tiles > 65536;
    const size_t tile_sz = wide ? 4 : 2;
    size_t s = 0;
    s += align_up(4 * (size_t)n);                                      // skey
    s += align_up(8 * (size_t)nc);                                     // chunk offsets
    s += align_up(8 * (size_t)n);                                      // rect by rank
    s += radix_scratch_bytes<uint32_t, uint32_t>(n);
    s += 2 * align_up(tile_sz * (size_t)cap) + align_up(4 * (size_t)cap);  // tiles, sorted tiles, gs
    s += wide ? radix_scratch_bytes<uint32_t, uint32_t>(cap) : radix_scratch_bytes<uint16_t, uint32_t>(cap);
    return s + 8192;
}

template <typename TileT>
static int32_t frame_binning_t(const FrameBinning& fb, cudaStream_t st) {
    Carver c(fb.scratch, fb.scratch_bytes);
    const int64_t n = fb.n, cap = fb.cap;
    uint32_t* skey = c.take<uint32_t>(n);
    uint64_t* coff = c.take<uint64_t>(ceil_div(n, 256));
    uint2* rect = c.take<uint2>(n);
    void* rs1 = c.take<char>((int64_t)radix_scratch_bytes<uint32_t, uint32_t>(n));
    TileT* tiles = c.take<TileT>(cap);
    TileT* stiles = c.take<TileT>(cap);
    uint32_t* gs = c.take<uint32_t>(cap);
    void* rs2 = c.take<char>((int64_t)radix_scratch_bytes<TileT, uint32_t>(cap));
    if (!c.ok()) return fail(ADR_ERR_VALUE, "render_frame: scratch too small");
    int64_t* ctr = fb.counters;  // [0]=P, [1]=culled, [2]=M, [3]=P clamped

    // (a)+(b) stable depth sort of all N Gaussians by the key stage 1 wrote
    //     (float32 depth bits, all-ones for Gaussians without pairs) with
    //     the identity as values: ranks [0, M) are the Gaussians with pairs
    //     ordered by (depth bits, index); the last pass writes, per rank,
    //     order[rank] = Gaussian index and rect[rank] = its tile rectangle
    SortExtra dx;
    dx.mode = 2;
    dx.gsrc = fb.gpack;
    dx.gdst = rect;
    int32_t rc = radix_sort<uint32_t, uint32_t>(fb.dkey, nullptr, skey, fb.order, nullptr, n, 32, rs1,
                                                radix_scratch_bytes<uint32_t, uint32_t>(n), st, dx);
    if (rc) return rc;
    // (c) pair offsets in rank order (per 256-rank chunk), and P
    const int64_t nc = ceil_div(n, 256);
    k_chunk_area_sums<<<ceil_div(nc * 32, 256), 256, 0, st>>>(rect, ctr + 2, nc, coff);
    ADR_LAUNCH_CHECK();
    k_chunk_scan<<<1, 1024, 0, st>>>(coff, nc, ctr + 0, ctr + 3, cap);
    ADR_LAUNCH_CHECK();
    if (fb.ev_after_scan) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_scan, st));
    // (d) emission of the stream as (tile, Gaussian)
    int tbits = 0;
    while ((int64_t(1) << tbits) < fb.n_tiles) ++tbits;
    if (tbits == 0) tbits = 1;
    k_emit_balanced<TileT><<<nc, 256, 0, st>>>(rect, fb.order, coff, ctr + 2, ctr + 3, fb.tiles_x, tiles, gs);
    ADR_LAUNCH_CHECK();
    if (fb.ev_after_dup) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_dup, st));
    // (e) stable radix sort by tile id; the last pass writes the sorted
    //     Gaussian indices (the render's record index and the gidx export)
    //     and the reference-layout keys (tile << 32 | depth bits)
    SortExtra tx;
    tx.mode = 1;
    tx.exp_depth = fb.proj.d_depth;
    tx.exp_keys = fb.keys;
    tx.skip_keys_out = fb.keys != nullptr;
    rc = radix_sort<TileT, uint32_t>(tiles, gs, stiles, reinterpret_cast<uint32_t*>(fb.gidx), ctr + 3, cap, tbits,
                                     rs2, radix_scratch_bytes<TileT, uint32_t>(cap), st, tx);
    if (rc) return rc;
    if (fb.ev_after_sort) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_sort, st));
    // (f) tile ranges
    k_ranges_search<TileT><<<ceil_div((fb.n_tiles + 1) * 32, 256), 256, 0, st>>>(
        TileIds<TileT>{stiles, fb.keys}, ctr + 3, fb.n_tiles, fb.ranges, fb.stats);
    ADR_LAUNCH_CHECK();
    if (fb.ev_after_ranges) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_ranges, st));
    return ADR_OK;
}

int32_t frame_binning(const FrameBinning& fb, cudaStream_t st) {
    if (fb.n <= 0) return ADR_OK;
    if (fb.n >= (int64_t(1) << 31)) return fail(ADR_ERR_CAPACITY, "more than 2^31 Gaussians");
    if (fb.cap >= (int64_t(1) << 31)) return fail(ADR_ERR_CAPACITY, "pair capacity must be < 2^31");
    if (fb.tiles_x >= 65536 || fb.tiles_y >= 65536) return fail(ADR_ERR_CAPACITY, "tile grid side >= 65536");
    if (!fb.gidx) return fail(ADR_ERR_VALUE, "render_frame needs the sorted index buffer");
    if (supertile_path(fb.n_tiles, fb.tiles_x, fb.tiles_y)) return frame_binning_supertile(fb, st);
    return fb.n_tiles > 65536 ? frame_binning_t<uint32_t>(fb, st) : frame_binning_t<uint16_t>(fb, st);
}

}  // namespace adr
