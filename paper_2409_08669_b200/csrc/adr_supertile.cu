// adr_supertile.cu — fused-frame tile binning by two-level counting placement
// (replaces pair emission + stable tile sort + range search for grids of at
// most 1024 supertiles).
//
// Reference semantics (sb/tiling.py:125-177): the pair list is every
// (tile, Gaussian) of each Gaussian's tile rectangle, keyed tile << 32 |
// float32 depth bits and stably sorted, so a tile's span lists its Gaussians
// by (depth bits, Gaussian index); ranges[t] = [lower_bound(t), lower_bound(t+1)).
//
// Input: the depth-rank order of the fused frame (adr_binning.cu, depth sort
// with MODE 3): rinfo[rank] = {Gaussian index, depth bits, packed tile rect}
// for ranks [0, M), M = Gaussians with pairs, in (depth bits, index) order.
// Since ranks are already in the reference's within-tile order, placing
// every pair at  tile_start[t] + #(earlier ranks covering t)  reproduces the
// stable sort exactly — a counting sort over tiles whose "rank among equal
// keys" is computed instead of sorted for.
//
// Two levels, so that every counter table is small:
//   L1  ranks -> supertile items.  A supertile is an 8x8 block of tiles; a
//       rank's rectangle touches a few supertiles (1.3 on average at
//       config 3).  Items (one per rank and touched supertile: Gaussian,
//       depth bits, the rectangle clipped to the supertile in local 4-bit
//       coordinates) are placed into per-supertile buckets, stably in rank
//       order: count (warp per 512 ranks, per-warp histogram) -> column scan
//       -> scatter (per-warp running offsets, in-round order from lane masks).
//       Buckets are padded to whole 256-item chunks.
//   L2  items -> pairs.  A chunk holds 256 items of ONE supertile, so the
//       tile alphabet is 64: each warp turns its 32 items' 64-bit tile masks
//       into per-tile 32-bit "cover" masks with a warp bit-matrix transpose;
//       the count pass sums cover popcounts per tile and chunk, a scan per
//       supertile + one global tile scan give every (chunk, tile) its output
//       offset (and the tile ranges), and the placement pass enumerates each
//       warp's pairs item-major (lanes balanced over the pair stream),
//       computes each pair's slot in the chunk's tile-major order from the
//       cover masks, stages the chunk in shared memory and writes it out as
//       coalesced per-tile runs (Gaussian index + reference key).
//
// No atomics decide any order; the result is deterministic and bit-identical
// to the reference's stable argsort.
#include "adr_binning.cuh"
#include "adr_sort.cuh"

namespace adr {

// adr_depthsort.cu
size_t depth_sort_scratch(int64_t n);
int32_t depth_sort_onesweep(const uint32_t* dkey, int64_t n, const DepthPlan& dp, const uint2* gpack, uint4* rinfo,
                            void* scratch, size_t scratch_bytes, cudaStream_t st);

namespace {

constexpr int kStSide = 8;            // supertile side in tiles
constexpr int kL1Ranks = 256;         // ranks per L1 warp chunk
constexpr int kL1Block = 8 * kL1Ranks; // ranks per L1 block (h1b column entry, scatter block)
#ifndef ADR_L1CAP
#define ADR_L1CAP 4096
#endif
#ifndef ADR_XLIST
#define ADR_XLIST 64
#endif
constexpr int kL1Cap = ADR_L1CAP;     // items staged per L1 scatter window
constexpr int kXList = ADR_XLIST;     // per-warp expanded-item list of the L1 scatter (one round segment)
constexpr int kChunk = 256;           // items per L2 chunk (= one 256-thread block)
constexpr int kStageCap = 3072;       // pairs staged per placement window

struct StGeom {
    int32_t tx, ty;      // tile grid
    int32_t sxn, syn;    // supertile grid
    int32_t S;           // supertiles
    float rsxn;          // 1 / sxn
    int64_t n1p;         // H1 column pitch (warp chunks, multiple of 8)
};
constexpr int kUnit = 4;              // chunks per count/scan unit

// (sx, sy) of supertile s: (s + 0.5) / sxn is >= 0.5 / sxn from an integer
// and s < 2^10, so the fp32 quotient floors exactly.
__device__ __forceinline__ void st_xy(const StGeom& g, int s, int* sx, int* sy) {
    *sy = (int)(__fadd_rn((float)s, 0.5f) * g.rsxn);
    *sx = s - *sy * g.sxn;
}

// Per-frame control arrays (in binning scratch).
struct StCtl {
    uint32_t* total;     // [S]   items per supertile
    uint32_t* pstart;    // [S+1] padded bucket starts (items); pstart[S] = padded item count
    uint32_t* iend;      // [S]   pstart[s] + total[s]
    uint16_t* cmap;      // [chunks] supertile of each L2 chunk
    uint32_t* ubase;     // [S+1] first unit of each supertile (a unit = <= 32 consecutive chunks)
    uint32_t* umap;      // [units] first chunk of each unit
    uint32_t* ttot;      // [T]   pairs per tile
    uint32_t* tstart;    // [T]   tile start in the sorted pair list (saturating)
    unsigned int* ticket;  // two self-resetting u32 tickets (counters[7])
};

// Items (SoA): {Gaussian index, depth bits} and the local rectangle.
struct StItems {
    uint2* gd;
    uint16_t* lr;
};

// 32x32 bit transpose across the warp: lane i holds row i (bit k = A[i][k])
// in, lane k holds column k (bit i = A[i][k]) out.  Two byte-permute stages
// and three masked-shift stages.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
    uint32_t y = __shfl_xor_sync(kFull, x, 16);
    x = __byte_perm(x, y, (lane & 16) ? 0x3276 : 0x5410);
    y = __shfl_xor_sync(kFull, x, 8);
    x = __byte_perm(x, y, (lane & 8) ? 0x3715 : 0x6240);
#pragma unroll
    for (int j = 4; j >= 1; j >>= 1) {
        const uint32_t m = j == 4 ? 0x0F0F0F0Fu : (j == 2 ? 0x33333333u : 0x55555555u);
        y = __shfl_xor_sync(kFull, x, j);
        const bool up = (lane & j) != 0;
        const uint32_t mm = up ? ~m : m;
        const uint32_t t = up ? (y >> j) : (y << j);
        x = (x & mm) | (t & ~mm);
    }
    return x;
}

// Local rectangle (4-bit coordinates inside the supertile, x1/y1 exclusive)
// -> 64-bit tile mask, bit ly * 8 + lx.
__device__ __forceinline__ uint64_t lrect_mask(uint32_t lr) {
    const uint32_t x0 = lr & 15u, x1 = (lr >> 4) & 15u, y0 = (lr >> 8) & 15u, y1 = (lr >> 12) & 15u;
    const uint32_t row = ((1u << x1) - 1u) & ~((1u << x0) - 1u);
    const uint64_t hi = y1 >= 8 ? ~0ull : ((1ull << (8 * y1)) - 1ull);
    const uint64_t rows = 0x0101010101010101ull & hi & ~((1ull << (8 * y0)) - 1ull);
    return (uint64_t)row * rows;
}

// ---------------------------------------------------------------- L1

// Items per (2048-rank block, supertile) into H1[s * n1p + b] (one shared
// histogram per block; each thread's 8 rectangles are loaded up front), and
// the true pair count P (sum of rectangle areas) into *d_p.
__global__ void __launch_bounds__(256) k_st_count1(const uint4* __restrict__ rinfo, const int64_t* __restrict__ d_m,
                                                   StGeom g, uint32_t* __restrict__ H1,
                                                   unsigned long long* __restrict__ d_p) {
    extern __shared__ uint32_t hist[];   // [S]
    constexpr int kR = kL1Block / 256;
    const int lane = threadIdx.x & 31;
    const int64_t m = *d_m;
    const int64_t b = blockIdx.x;
    const int64_t r0 = b * kL1Block;
    if (r0 >= m) return;
    uint2 rc[kR];
#pragma unroll
    for (int k = 0; k < kR; ++k) {
        const int64_t r = r0 + k * 256 + threadIdx.x;
        rc[k] = r < m ? __ldg(reinterpret_cast<const uint2*>(rinfo + r) + 1) : make_uint2(0u, 0u);
    }
    for (int s = threadIdx.x; s < g.S; s += 256) hist[s] = 0;
    __syncthreads();
    uint64_t area = 0;
#pragma unroll
    for (int k = 0; k < kR; ++k) {
        const uint32_t x0 = rc[k].x & 0xffffu, x1 = rc[k].x >> 16, y0 = rc[k].y & 0xffffu, y1 = rc[k].y >> 16;
        if (x1 > x0) {   // ranks < M have a non-empty rectangle; padding threads are (0, 0)
            area += (uint64_t)(x1 - x0) * (y1 - y0);
            for (uint32_t sy = y0 >> 3; sy <= (y1 - 1) >> 3; ++sy)
                for (uint32_t sx = x0 >> 3; sx <= (x1 - 1) >> 3; ++sx) atomicAdd(&hist[sy * g.sxn + sx], 1u);
        }
    }
    __syncthreads();
    for (int s = threadIdx.x; s < g.S; s += 256) H1[s * g.n1p + b] = hist[s];
    area = warp_sum(area);
    if (lane == 0 && area) atomicAdd(d_p, (unsigned long long)area);
}

// Exclusive scan of every supertile column of H1 (items per 2048-rank block,
// counted by the depth sort's last pass) over the blocks (block per
// supertile; per batch each thread holds 8 consecutive rows, loaded as two
// 16-byte vectors), the bucket totals, and (last block) the padded bucket
// starts, the bucket ends and the chunk -> supertile / unit -> chunk maps.
__global__ void __launch_bounds__(1024) k_st_scan1(uint32_t* __restrict__ H1, const int64_t* __restrict__ d_m,
                                                   StGeom g, StCtl c, int64_t items_cap,
                                                   int64_t* __restrict__ counters, adr_load_stats* stats) {
    constexpr int K = 8;
    __shared__ uint32_t sred[33];
    __shared__ bool last;
    if (stats && blockIdx.x == 0 && threadIdx.x == 0) {   // the render's load-statistics accumulators
        stats->sum = 0;
        stats->sum_sq = 0;
        stats->min = INT_MAX;
        stats->max = INT_MIN;
    }
    const int64_t n1 = (*d_m + kL1Block - 1) / kL1Block;
    uint32_t* col = H1 + blockIdx.x * g.n1p;
    uint32_t carry = 0;
    for (int64_t b0 = 0; b0 < n1; b0 += 1024 * K) {
        const int64_t a = b0 + (int64_t)threadIdx.x * K;
        uint32_t v[K], sum = 0;
        if (a + K <= n1) {
            const uint4 p = *reinterpret_cast<const uint4*>(col + a), q = *reinterpret_cast<const uint4*>(col + a + 4);
            v[0] = p.x; v[1] = p.y; v[2] = p.z; v[3] = p.w; v[4] = q.x; v[5] = q.y; v[6] = q.z; v[7] = q.w;
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k) v[k] = a + k < n1 ? col[a + k] : 0u;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) sum += v[k];
        uint32_t tot;
        uint32_t run = carry + block_exclusive_sum<uint32_t, 1024>(sum, sred, &tot);
        uint32_t o[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            o[k] = run;
            run += v[k];
        }
        if (a + K <= n1) {
            *reinterpret_cast<uint4*>(col + a) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(col + a + 4) = make_uint4(o[4], o[5], o[6], o[7]);
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (a + k < n1) col[a + k] = o[k];
        }
        carry += tot;
    }
    if (threadIdx.x == 0) c.total[blockIdx.x] = carry;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&c.ticket[0], 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // padded bucket starts (S <= 1024: one supertile per thread), bucket ends
    // and the first unit of every supertile; the chunk -> supertile and
    // unit -> chunk maps are filled by k_st_scatter1's blocks
    const int t = threadIdx.x;
    const int64_t n2cap = items_cap / kChunk;
    const uint32_t tt = t < g.S ? __ldcg(c.total + t) : 0u;
    const uint32_t padded = (tt + kChunk - 1) / kChunk * kChunk;
    uint32_t all;
    const uint32_t pre = block_exclusive_sum<uint32_t, 1024>(padded, sred, &all);
    int64_t ch0 = pre / kChunk, ch1 = (int64_t)(pre + padded) / kChunk;
    if (ch1 > n2cap) ch1 = n2cap;
    if (ch0 > ch1) ch0 = ch1;
    const uint32_t units = (uint32_t)((ch1 - ch0 + kUnit - 1) / kUnit);
    uint32_t all_units;
    const uint32_t upre = block_exclusive_sum<uint32_t, 1024>(t < g.S ? units : 0u, sred, &all_units);
    if (t < g.S) {
        c.pstart[t] = pre;
        c.iend[t] = pre + tt;
        c.ubase[t] = upre;
    }
    if (t == 0) {
        c.pstart[g.S] = all;
        c.ubase[g.S] = all_units;
        if ((int64_t)all > items_cap) counters[6] = 1;   // cannot happen unless P > capacity
        c.ticket[0] = 0;
    }
}

// Place the items, stably in rank order within each supertile bucket.  Block
// = 2048 ranks, warp = 256 ranks (held in registers: a per-warp supertile
// histogram first, then the placement).  Per round of 32 ranks a warp's items
// form a stream in (rank, supertile) order; each lane writes its own items
// into a per-warp shared list at their stream positions, then lanes take 32
// consecutive entries, peers with the same supertile come from match.any and
// the lowest peer bumps the warp's running offset.  Items are staged in shared memory in bucket order (the block's
// items of one supertile are contiguous in the output) and flushed as
// coalesced runs.
#ifndef ADR_SC1_MINB
#define ADR_SC1_MINB 4
#endif
__global__ void __launch_bounds__(256, ADR_SC1_MINB) k_st_scatter1(const uint4* __restrict__ rinfo, const int64_t* __restrict__ d_m,
                                                     StGeom g, const uint32_t* __restrict__ H1, StCtl c,
                                                     StItems items, int64_t items_cap) {
    extern __shared__ __align__(16) unsigned char sc_raw[];
    uint4* xlist = reinterpret_cast<uint4*>(sc_raw);                             // [8][kXList] expanded items
    uint2* sgd = reinterpret_cast<uint2*>(xlist + 8 * kXList);                   // [kL1Cap]
    uint16_t* slr = reinterpret_cast<uint16_t*>(sgd + kL1Cap);                   // [kL1Cap]
    uint16_t* sdig = slr + kL1Cap;                                               // [kL1Cap]
    uint32_t* wbase = reinterpret_cast<uint32_t*>(sdig + kL1Cap);                // [8][S] warp slot bases
    uint32_t* woff = wbase + 8 * g.S;                                            // [8][S] running
    uint32_t* lst = woff + 8 * g.S;                                              // [S] block-local bucket starts
    uint32_t* g0 = lst + g.S;                                                    // [S] global start of the block's run
    __shared__ uint32_t sred[33];
    constexpr int kR = kL1Ranks / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t m = *d_m;
    const int64_t b = blockIdx.x;
    const int64_t r0 = b * kL1Block + warp * kL1Ranks;
    const int64_t r1 = r0 + kL1Ranks < m ? r0 + kL1Ranks : m;
    // this warp's ranks' rectangles, and its items per supertile (shared-memory histogram)
    uint2 vb[kR];
#pragma unroll
    for (int k = 0; k < kR; ++k) {
        const int64_t r = r0 + k * 32 + lane;
        vb[k] = r < r1 ? __ldg(reinterpret_cast<const uint2*>(rinfo + r) + 1) : make_uint2(0u, 0u);
    }
    uint32_t* wh = wbase + warp * g.S;
    for (int s = lane; s < g.S; s += 32) wh[s] = 0;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kR; ++k) {
        const uint32_t x0 = vb[k].x & 0xffffu, x1 = vb[k].x >> 16, y0 = vb[k].y & 0xffffu, y1 = vb[k].y >> 16;
        if (x1 > x0)
            for (uint32_t sy = y0 >> 3; sy <= (y1 - 1) >> 3; ++sy)
                for (uint32_t sx = x0 >> 3; sx <= (x1 - 1) >> 3; ++sx) atomicAdd(&wh[sy * g.sxn + sx], 1u);
    }
    __syncthreads();
    // per supertile: per-warp exclusive prefixes (in place), block total,
    // block-local bucket start and the global start of the block's run
    uint32_t mysum = 0;
    constexpr int kPer = 4;   // supertiles per thread (S <= 1024)
    uint32_t bt[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int s = threadIdx.x * kPer + k;
        bt[k] = 0;
        if (s < g.S) {
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const uint32_t v = wbase[w * g.S + s];
                wbase[w * g.S + s] = run;
                run += v;
            }
            bt[k] = run;
            g0[s] = __ldg(c.pstart + s) + H1[s * g.n1p + b];
        }
        mysum += bt[k];
    }
    uint32_t btotal;
    uint32_t run = block_exclusive_sum<uint32_t, 256>(mysum, sred, &btotal);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int s = threadIdx.x * kPer + k;
        if (s < g.S) lst[s] = run;
        run += bt[k];
    }
    // this block's share of the chunk -> supertile and unit -> chunk maps
    {
        const int64_t n2cap = items_cap / kChunk;
        int64_t n2 = __ldg(c.pstart + g.S) / kChunk;
        n2 = n2 < n2cap ? n2 : n2cap;
        const int64_t per = (n2 + gridDim.x - 1) / gridDim.x;
        for (int64_t ch = b * per + threadIdx.x; ch < (b + 1) * per && ch < n2; ch += 256) {
            int lo = 0, hi = g.S - 1;   // last supertile whose first chunk <= ch
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if ((int64_t)(__ldg(c.pstart + mid) / kChunk) <= ch) lo = mid; else hi = mid - 1;
            }
            c.cmap[ch] = (uint16_t)lo;
        }
        const uint32_t nu = __ldg(c.ubase + g.S);
        const uint32_t uper = (nu + gridDim.x - 1) / gridDim.x;
        for (uint32_t u = (uint32_t)b * uper + threadIdx.x; u < ((uint32_t)b + 1) * uper && u < nu; u += 256) {
            int lo = 0, hi = g.S - 1;   // last supertile whose first unit <= u
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (__ldg(c.ubase + mid) <= u) lo = mid; else hi = mid - 1;
            }
            c.umap[u] = __ldg(c.pstart + lo) / kChunk + (u - __ldg(c.ubase + lo)) * kUnit;
        }
    }
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t* off = woff + warp * g.S;
    for (uint32_t win = 0; win < btotal; win += kL1Cap) {
        for (int s = lane; s < g.S; s += 32) off[s] = lst[s] + wbase[warp * g.S + s];
        __syncwarp();
        if (r0 < r1) {
            uint4* xl = xlist + warp * kXList;
            uint4 vn = rinfo[r0 + lane < r1 ? r0 + lane : r0];
#pragma unroll 1
            for (int k = 0; k < kR; ++k) {
                // the round's items in stream order (rank, then supertile): each
                // lane expands its own rank's items into the warp's list ...
                const bool in = r0 + k * 32 + lane < r1;
                const uint4 v = in ? vn : make_uint4(0u, 0u, 0u, 0u);
                if (k + 1 < kR) {   // next round's rank record (L2-hot: read by the histogram above)
                    const int64_t rn = r0 + (k + 1) * 32 + lane;
                    vn = rinfo[rn < r1 ? rn : r0];
                }
                const uint32_t x0 = v.z & 0xffffu, x1 = v.z >> 16, y0 = v.w & 0xffffu, y1 = v.w >> 16;
                const bool has = x1 > x0;
                const uint32_t sx0 = x0 >> 3, sy0 = y0 >> 3, sx1 = has ? (x1 - 1) >> 3 : 0u, sy1 = has ? (y1 - 1) >> 3 : 0u;
                const uint32_t cnt = has ? (sx1 - sx0 + 1) * (sy1 - sy0 + 1) : 0u;
                const uint32_t incl = warp_inclusive_sum(cnt);
                const uint32_t o = incl - cnt;
                const uint32_t total = __shfl_sync(kFull, incl, 31);
                for (uint32_t seg = 0; seg < total; seg += kXList) {
                    if (has && o < seg + kXList && o + cnt > seg) {
                        uint32_t q = o;
                        for (uint32_t sy = sy0; sy <= sy1; ++sy) {
                            const uint32_t ly0 = (y0 > sy * 8 ? y0 : sy * 8) - sy * 8;
                            const uint32_t ly1 = (y1 < sy * 8 + 8 ? y1 : sy * 8 + 8) - sy * 8;
                            for (uint32_t sx = sx0; sx <= sx1; ++sx, ++q) {
                                if (q - seg >= (uint32_t)kXList) continue;
                                const uint32_t lx0 = (x0 > sx * 8 ? x0 : sx * 8) - sx * 8;
                                const uint32_t lx1 = (x1 < sx * 8 + 8 ? x1 : sx * 8 + 8) - sx * 8;
                                xl[q - seg] = make_uint4(v.x, v.y, lx0 | (lx1 << 4) | (ly0 << 8) | (ly1 << 12),
                                                         sy * g.sxn + sx);
                            }
                        }
                    }
                    __syncwarp();
                    // ... then 32 consecutive entries at a time are ranked among
                    // equal supertiles (match.any; lane order = stream order) and
                    // staged at the warp's running bucket offsets
                    const uint32_t nseg = total - seg < (uint32_t)kXList ? total - seg : (uint32_t)kXList;
                    for (uint32_t base = 0; base < nseg; base += 32) {
                        const bool live = base + lane < nseg;
                        const uint4 e = live ? xl[base + lane] : make_uint4(0u, 0u, 0u, 0xffffffffu);
                        const uint32_t peers = __match_any_sync(kFull, e.w);
                        const uint32_t ob = live ? off[e.w] : 0u;
                        __syncwarp();
                        if (live) {
                            if ((peers & lt) == 0) off[e.w] = ob + __popc(peers);
                            const uint32_t slot = ob + __popc(peers & lt) - win;
                            if (slot < (uint32_t)kL1Cap) {
                                sgd[slot] = make_uint2(e.x, e.y);
                                slr[slot] = (uint16_t)e.z;
                                sdig[slot] = (uint16_t)e.w;
                            }
                        }
                        __syncwarp();
                    }
                }
            }
        }
        __syncthreads();
        const uint32_t wend = btotal - win < (uint32_t)kL1Cap ? btotal - win : (uint32_t)kL1Cap;
        for (uint32_t k = threadIdx.x; k < wend; k += 256) {
            const uint32_t s = sdig[k];
            const int64_t gpos = (int64_t)g0[s] + (int64_t)(win + k - lst[s]);
            if (gpos < items_cap) {
                items.gd[gpos] = sgd[k];
                items.lr[gpos] = slr[k];
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- L2

__device__ __forceinline__ int64_t live_chunks(const StCtl& c, int S, int64_t items_cap) {
    int64_t nitems = __ldg(c.pstart + S);
    if (nitems > items_cap) nitems = items_cap / kChunk * kChunk;
    return nitems / kChunk;
}

// Per-chunk pair counts, scanned within 32-chunk units.  Warp per unit
// (persistent): for each chunk, 8 rounds of cover popcounts per local tile;
// C2[chunk * 64 + l] = pairs of tile l in the unit's earlier chunks, U[unit *
// 64 + l] = the unit's total.
#ifndef ADR_C2_MINB
#define ADR_C2_MINB 1
#endif
__global__ void __launch_bounds__(256, ADR_C2_MINB) k_st_count2(StItems items, StGeom g, StCtl c, int64_t items_cap,
                                                   uint32_t* __restrict__ C2, uint32_t* __restrict__ U) {
    const int lane = threadIdx.x & 31;
    const int64_t n2 = live_chunks(c, g.S, items_cap);
    const uint32_t nunits = __ldg(c.ubase + g.S);
    const uint32_t nw = gridDim.x * 8;
    for (uint32_t u = blockIdx.x * 8 + (threadIdx.x >> 5); u < nunits; u += nw) {
        const uint32_t cf = __ldg(c.umap + u);
        const int s = __ldg(c.cmap + cf);
        const uint32_t iend = __ldg(c.iend + s);
        int64_t ce = (int64_t)(__ldg(c.pstart + s + 1) / kChunk);
        if (ce > (int64_t)cf + kUnit) ce = (int64_t)cf + kUnit;
        if (ce > n2) ce = n2;
        uint32_t run_lo = 0, run_hi = 0;
        for (int64_t ch = cf; ch < ce; ++ch) {
            const uint32_t item0 = (uint32_t)(ch * kChunk);
            uint32_t clo = 0, chi = 0, lr[kChunk / 32];
#pragma unroll
            for (int rd = 0; rd < kChunk / 32; ++rd) {
                const uint32_t i = item0 + rd * 32 + lane;
                lr[rd] = i < iend ? __ldg(items.lr + i) : 0u;
            }
#pragma unroll
            for (int rd = 0; rd < kChunk / 32; ++rd) {
                const uint64_t mk = lr[rd] ? lrect_mask(lr[rd]) : 0ull;
                clo += __popc(warp_transpose32((uint32_t)mk, lane));
                chi += __popc(warp_transpose32((uint32_t)(mk >> 32), lane));
            }
            C2[ch * 64 + lane] = run_lo;
            C2[ch * 64 + 32 + lane] = run_hi;
            run_lo += clo;
            run_hi += chi;
        }
        U[(int64_t)u * 64 + lane] = run_lo;
        U[(int64_t)u * 64 + 32 + lane] = run_hi;
    }
}

// Per supertile (block of 64 tiles x 16 unit slices): exclusive scan of the
// unit totals over the supertile's units (in place) and the per-tile totals;
// the last block scans the tile totals in tile order into tile starts and
// the tile ranges.
__global__ void __launch_bounds__(1024) k_st_scan2(uint32_t* __restrict__ U, StGeom g, StCtl c, int64_t cap,
                                                   int64_t n_tiles, int64_t* __restrict__ ranges,
                                                   int64_t* __restrict__ counters) {
    constexpr int kParts = 16, K = 8;
    __shared__ uint32_t part[kParts][64];
    __shared__ uint64_t sred[33];
    __shared__ bool last;
    const int s = blockIdx.x;
    const int l = threadIdx.x & 63, q = threadIdx.x >> 6;
    const int64_t u0 = __ldg(c.ubase + s), u1 = __ldg(c.ubase + s + 1);
    uint32_t carry = 0;
    for (int64_t b0 = u0; b0 < u1; b0 += kParts * K) {
        const int64_t a = b0 + q * K;
        uint32_t v[K], sum = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            v[k] = a + k < u1 ? U[(a + k) * 64 + l] : 0u;
            sum += v[k];
        }
        part[q][l] = sum;
        __syncthreads();
        uint32_t run = carry, tot = 0;
#pragma unroll
        for (int j = 0; j < kParts; ++j) {
            const uint32_t pj = part[j][l];
            run += j < q ? pj : 0u;
            tot += pj;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (a + k < u1) U[(a + k) * 64 + l] = run;
            run += v[k];
        }
        carry += tot;
    }
    int sx, sy;
    st_xy(g, s, &sx, &sy);
    const int tyy = sy * kStSide + (l >> 3), txx = sx * kStSide + (l & 7);
    if (q == 0 && txx < g.tx && tyy < g.ty) c.ttot[tyy * g.tx + txx] = carry;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&c.ticket[1], 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // tile starts in tile order, ranges, P (counted) and P clamped to capacity;
    // each thread scans a run of up to 8 consecutive tiles per batch
    uint64_t acc = 0;
    for (int64_t t0 = 0; t0 < n_tiles; t0 += 1024 * 8) {
        const int64_t a = t0 + (int64_t)threadIdx.x * 8;
        uint32_t v[8];
        uint64_t sum = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            v[k] = a + k < n_tiles ? __ldcg(c.ttot + a + k) : 0u;
            sum += v[k];
        }
        uint64_t blk;
        uint64_t pre = acc + block_exclusive_sum<uint64_t, 1024>(sum, sred, &blk);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int64_t t = a + k;
            if (t < n_tiles) {
                c.tstart[t] = pre < 0xffffffffull ? (uint32_t)pre : 0xffffffffu;
                const int64_t lo = (int64_t)pre < cap ? (int64_t)pre : cap;
                const int64_t hi = (int64_t)(pre + v[k]) < cap ? (int64_t)(pre + v[k]) : cap;
                ranges[2 * t] = lo;
                ranges[2 * t + 1] = hi;
            }
            pre += v[k];
        }
        acc += blk;
    }
    if (threadIdx.x == 0) {
        const int64_t p_true = counters[0];
        counters[3] = (int64_t)acc < cap ? (int64_t)acc : cap;
        if (p_true > cap || (int64_t)acc != p_true) counters[6] = 1;
        c.ticket[1] = 0;
    }
}

// Placement: block per chunk (warp w owns items w*32 .. w*32+31), persistent
// over chunks with the next chunk's items prefetched.
//   A  tile masks -> per-warp cover masks (transpose) and per-warp tile counts;
//   B  (after one barrier) each warp derives its own slot bases in the chunk's
//      tile-major order from the 8 x 64 counts; warp 0 the tile runs' global
//      offsets;
//   C  lane = tile (two per lane): walk the set bits of the tile's cover mask
//      (the warp's items on that tile, in rank order) and stage each item's
//      {index, depth bits} at consecutive slots of the tile's run;
//   D  (barrier) thread per slot: coalesced per-tile runs out; (barrier).
#ifndef ADR_PLACE_MINB
#define ADR_PLACE_MINB 6
#endif
__global__ void __launch_bounds__(256, ADR_PLACE_MINB) k_st_place(StItems items, StGeom g, StCtl c, int64_t items_cap,
                                                  const uint32_t* __restrict__ C2, const uint32_t* __restrict__ U,
                                                  const int64_t* __restrict__ d_pc, uint32_t* __restrict__ gidx_out,
                                                  uint64_t* __restrict__ keys_out) {
    __shared__ uint2 stage[kStageCap];
    __shared__ uint8_t stile[kStageCap];
    __shared__ uint2 scnt[64];          // per tile: the 8 warps' counts, one byte each
    __shared__ uint2 sitem[8][32];
    __shared__ uint2 gtile[64];        // (global position - local slot of the run, tile id)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n2 = live_chunks(c, g.S, items_cap);
    const uint32_t pc = (uint32_t)*d_pc;
    int64_t ch = blockIdx.x;
    uint2 nx_gd = make_uint2(0u, 0u);
    uint32_t nx_lr = 0u;
    if (ch < n2) {
        const uint32_t i = (uint32_t)(ch * kChunk) + threadIdx.x;
        if (i < __ldg(c.iend + __ldg(c.cmap + ch))) {
            nx_gd = items.gd[i];
            nx_lr = items.lr[i];
        }
    }
    for (; ch < n2; ch += gridDim.x) {
        const int s = __ldg(c.cmap + ch);
        // A: this chunk's item (prefetched), then prefetch the next chunk's
        const uint32_t lr = nx_lr;
        sitem[warp][lane] = nx_gd;
        {
            const int64_t cn = ch + gridDim.x;
            nx_lr = 0u;
            if (cn < n2) {
                const uint32_t i = (uint32_t)(cn * kChunk) + threadIdx.x;
                if (i < __ldg(c.iend + __ldg(c.cmap + cn))) {
                    nx_gd = items.gd[i];
                    nx_lr = items.lr[i];
                }
            }
        }
        const uint64_t mk = lr ? lrect_mask(lr) : 0ull;
        const uint32_t clo = warp_transpose32((uint32_t)mk, lane);
        const uint32_t chi = warp_transpose32((uint32_t)(mk >> 32), lane);
        reinterpret_cast<uint8_t*>(&scnt[lane])[warp] = (uint8_t)__popc(clo);
        reinterpret_cast<uint8_t*>(&scnt[lane + 32])[warp] = (uint8_t)__popc(chi);
        __syncthreads();
        // B: tile-major slots.  Lane owns tiles lane and lane + 32; per tile the
        // 8 warp counts (<= 32 each) are bytes, prefix-summed in-register
        // (x * 0x01010101: byte k = c0 + ... + ck, no carries below 256)
        uint32_t wpre_lo, wpre_hi, tot_lo, tot_hi;
        {
            const uint2 a = scnt[lane], b = scnt[lane + 32];
            const uint32_t pa0 = a.x * 0x01010101u, pa1 = a.y * 0x01010101u;
            const uint32_t pb0 = b.x * 0x01010101u, pb1 = b.y * 0x01010101u;
            const uint32_t ta0 = pa0 >> 24, tb0 = pb0 >> 24;
            tot_lo = ta0 + (pa1 >> 24);
            tot_hi = tb0 + (pb1 >> 24);
            // exclusive prefix of warp `warp` (warp-uniform shifts)
            wpre_lo = warp == 0 ? 0u : (warp <= 4 ? (pa0 >> (8 * (warp - 1))) & 0xffu : ta0 + ((pa1 >> (8 * (warp - 5))) & 0xffu));
            wpre_hi = warp == 0 ? 0u : (warp <= 4 ? (pb0 >> (8 * (warp - 1))) & 0xffu : tb0 + ((pb1 >> (8 * (warp - 5))) & 0xffu));
        }
        // both tile halves in one scan (each half sums to < 2^16)
        const uint32_t inc = warp_inclusive_sum(tot_lo | (tot_hi << 16));
        const uint32_t sums = __shfl_sync(kFull, inc, 31);
        const uint32_t sum_lo = sums & 0xffffu;
        const uint32_t ls_lo = (inc & 0xffffu) - tot_lo, ls_hi = sum_lo + (inc >> 16) - tot_hi;   // local run starts
        const uint32_t ctotal = sum_lo + (sums >> 16);
        if (warp == 0) {
            int sx, sy;
            st_xy(g, s, &sx, &sy);
            const uint32_t unit = __ldg(c.ubase + s) + (uint32_t)(ch - (int64_t)(__ldg(c.pstart + s) / kChunk)) / kUnit;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int l = lane + 32 * h;
                const int tyy = sy * kStSide + (l >> 3), txx = sx * kStSide + (l & 7);
                const bool in = txx < g.tx && tyy < g.ty;
                const uint32_t t = in ? (uint32_t)(tyy * g.tx + txx) : 0u;
                const uint64_t gb = in ? (uint64_t)__ldg(c.tstart + t) + __ldg(U + (int64_t)unit * 64 + l) +
                                             __ldg(C2 + ch * 64 + l)
                                       : 0xffffffffull;
                // gpos = gb + (slot - run start); runs starting at or past the
                // capacity are flagged so every gpos lands >= pc (pc < 2^31)
                gtile[l] = make_uint2(gb < pc ? (uint32_t)gb - (h ? ls_hi : ls_lo) : 0x80000000u, t);
            }
        }
        __syncwarp();
        // C + D, window by window (one window unless the chunk has > kStageCap pairs)
        for (uint32_t win = 0; win < ctotal; win += kStageCap) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t m = h ? chi : clo;
                uint32_t slot = (h ? ls_hi + wpre_hi : ls_lo + wpre_lo) - win;
                const uint8_t l = (uint8_t)(lane + 32 * h);
                if (slot <= (uint32_t)kStageCap - __popc(m)) {   // the whole run of this warp's items is in the window
                    uint2* dst = stage + slot;
                    uint8_t* dtl = stile + slot;
                    while (m) {
                        const int L = __ffs(m) - 1;
                        m &= m - 1u;
                        *dst++ = sitem[warp][L];
                        *dtl++ = l;
                    }
                } else {
                    while (m) {
                        const int L = __ffs(m) - 1;
                        m &= m - 1u;
                        if (slot < (uint32_t)kStageCap) {
                            stage[slot] = sitem[warp][L];
                            stile[slot] = l;
                        }
                        ++slot;
                    }
                }
            }
            __syncthreads();
            const uint32_t wend = ctotal - win < (uint32_t)kStageCap ? ctotal - win : (uint32_t)kStageCap;
            for (uint32_t k = threadIdx.x; k < wend; k += 256) {
                const uint2 gt = gtile[stile[k]];
                const uint32_t gpos = gt.x + win + k;
                if (gpos < pc) {
                    const uint2 v = stage[k];
                    gidx_out[gpos] = v.x;
                    if (keys_out) keys_out[gpos] = ((uint64_t)gt.y << 32) | v.y;
                }
            }
            __syncthreads();
        }
        if (ctotal == 0) __syncthreads();   // (never taken: every live chunk holds pairs)
    }
}

}  // namespace

int64_t supertile_count(int32_t tx, int32_t ty) {
    return ceil_div(tx, kStSide) * ceil_div(ty, kStSide);
}

bool supertile_path(int64_t n_tiles, int32_t tx, int32_t ty) {
    return n_tiles <= 65536 && supertile_count(tx, ty) <= 1024;
}

static int64_t st_items_cap(int64_t cap, int64_t S) { return cap + (int64_t)kChunk * (S + 1); }

size_t supertile_scratch(int64_t n, int64_t cap, int32_t tx, int32_t ty) {
    const int64_t S = supertile_count(tx, ty), T = (int64_t)tx * ty;
    const int64_t n1p = align_up(ceil_div(n > 0 ? n : 1, kL1Block) + 8, 8);
    const int64_t icap = st_items_cap(cap, S);
    size_t s = 0;
    s += align_up(16 * (size_t)n);               // rinfo
    s += depth_sort_scratch(n);
    s += align_up(4 * (size_t)(n1p * S));        // H1
    s += 3 * align_up(4 * (size_t)(S + 1));      // total, pstart, iend
    s += align_up(2 * (size_t)(icap / kChunk + 1));  // cmap
    s += align_up(4 * (size_t)(S + 1)) + align_up(4 * (size_t)(icap / kChunk / kUnit + S + 1));  // ubase, umap
    s += align_up(256 * (size_t)(icap / kChunk / kUnit + S + 1));  // U
    s += 2 * align_up(4 * (size_t)T);            // ttot, tstart
    s += align_up(8 * (size_t)icap) + align_up(2 * (size_t)icap);  // items
    s += align_up(256 * (size_t)(icap / kChunk + 1));  // C2
    return s + 8192;
}

static int blocks_per_sm(const void* fn, int threads, size_t smem) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, threads, smem) != cudaSuccess || b < 1) b = 1;
    return b;
}

int32_t frame_binning_supertile(const FrameBinning& fb, cudaStream_t st) {
    const int64_t n = fb.n, cap = fb.cap;
    StGeom g;
    g.tx = fb.tiles_x;
    g.ty = fb.tiles_y;
    g.sxn = (int32_t)ceil_div(g.tx, kStSide);
    g.syn = (int32_t)ceil_div(g.ty, kStSide);
    g.S = g.sxn * g.syn;
    g.rsxn = 1.0f / (float)g.sxn;
    g.n1p = (int64_t)align_up(ceil_div(n, kL1Block) + 8, 8);
    const int64_t T = fb.n_tiles;
    const int64_t icap = st_items_cap(cap, g.S);
    const int64_t n2max = icap / kChunk;
    Carver cv(fb.scratch, fb.scratch_bytes);
    uint4* rinfo = cv.take<uint4>(n);
    const size_t ds_bytes = depth_sort_scratch(n);
    void* ds_scratch = cv.take<char>((int64_t)ds_bytes);
    uint32_t* H1 = cv.take<uint32_t>(g.n1p * g.S);
    StCtl c;
    c.total = cv.take<uint32_t>(g.S + 1);
    c.pstart = cv.take<uint32_t>(g.S + 1);
    c.iend = cv.take<uint32_t>(g.S + 1);
    c.cmap = cv.take<uint16_t>(n2max + 1);
    const int64_t umax = n2max / kUnit + g.S + 1;
    c.ubase = cv.take<uint32_t>(g.S + 1);
    c.umap = cv.take<uint32_t>(umax);
    uint32_t* Ut = cv.take<uint32_t>(umax * 64);
    c.ttot = cv.take<uint32_t>(T);
    c.tstart = cv.take<uint32_t>(T);
    StItems items;
    items.gd = cv.take<uint2>(icap);
    items.lr = cv.take<uint16_t>(icap);
    uint32_t* C2 = cv.take<uint32_t>((n2max + 1) * 64);
    if (!cv.ok()) return fail(ADR_ERR_VALUE, "render_frame: scratch too small");
    int64_t* ctr = fb.counters;   // [0]=P, [1]=culled, [2]=M, [3]=P clamped, [6]=truncated, [7]=tickets
    c.ticket = reinterpret_cast<unsigned int*>(ctr + 7);

    // depth-rank order (onesweep, adr_depthsort.cu); the last pass writes
    // rinfo[rank] = {index, depth bits, rect}
    DepthPlan dp;
    if (fb.kminmax && fb.plan_mm) {   // key-range plan from the preprocess's per-block extrema
        dp.plan = fb.plan_mm;
        dp.plan_out = fb.plan_mm;
        dp.kminmax = fb.kminmax;
        dp.nkb = 4 * ceil_div(n, 128);   // one (min, max) per preprocess warp
    }
    int32_t rc = depth_sort_onesweep(fb.dkey, n, dp, fb.gpack, rinfo, ds_scratch, ds_bytes, st);
    if (rc) return rc;
    if (fb.ev_after_scan) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_scan, st));   // stage "depth sort"
    // L1: ranks -> supertile items
    const unsigned nb1 = (unsigned)ceil_div(n, kL1Block);
    k_st_count1<<<nb1, 256, g.S * sizeof(uint32_t), st>>>(rinfo, ctr + 2, g, H1,
                                                         reinterpret_cast<unsigned long long*>(ctr));
    ADR_LAUNCH_CHECK();
    k_st_scan1<<<(unsigned)g.S, 1024, 0, st>>>(H1, ctr + 2, g, c, icap, ctr, fb.stats);
    ADR_LAUNCH_CHECK();
    const size_t sm_sc = 16 * 8 * (size_t)kXList + 12 * (size_t)kL1Cap + (18 * (size_t)g.S + 2) * sizeof(uint32_t);  // see k_st_scatter1
    ADR_CUDA_TRY(cudaFuncSetAttribute(k_st_scatter1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_sc));
    k_st_scatter1<<<nb1, 256, sm_sc, st>>>(rinfo, ctr + 2, g, H1, c, items, icap);
    ADR_LAUNCH_CHECK();
    if (fb.ev_after_dup) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_dup, st));   // stage "L1 items"
    // L2: items -> pairs
    static int sms = 0, bps_c2 = 0, bps_pl = 0;
    if (!sms) {
        int dev = 0;
        ADR_CUDA_TRY(cudaGetDevice(&dev));
        ADR_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        bps_c2 = blocks_per_sm((const void*)k_st_count2, 256, 0);
        bps_pl = blocks_per_sm((const void*)k_st_place, 256, 0);
    }
    int64_t grid_c2 = (int64_t)sms * bps_c2;
    if (grid_c2 > ceil_div(umax, 8)) grid_c2 = ceil_div(umax, 8);
    k_st_count2<<<(unsigned)grid_c2, 256, 0, st>>>(items, g, c, icap, C2, Ut);
    ADR_LAUNCH_CHECK();
    k_st_scan2<<<(unsigned)g.S, 1024, 0, st>>>(Ut, g, c, cap, T, fb.ranges, ctr);
    ADR_LAUNCH_CHECK();
    int64_t grid_pl = (int64_t)sms * bps_pl;
    if (grid_pl > n2max) grid_pl = n2max > 0 ? n2max : 1;
    k_st_place<<<(unsigned)grid_pl, 256, 0, st>>>(
        items, g, c, icap, C2, Ut, ctr + 3, reinterpret_cast<uint32_t*>(fb.gidx), fb.keys);
    ADR_LAUNCH_CHECK();
    if (fb.ev_after_sort) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_sort, st));
    if (fb.ev_after_ranges) ADR_CUDA_TRY(cudaEventRecord(fb.ev_after_ranges, st));
    return ADR_OK;
}

}  // namespace adr
