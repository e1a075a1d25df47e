// adr_binning.cuh — stages 2-5 launchers (stage API + fused frame).
#pragma once

#include "adr_kernels.cuh"

namespace adr {

int32_t stage_touched_counts(const adr_projection& p, int64_t n, int32_t tx, int32_t ty, int64_t* counts,
                             cudaStream_t st);
size_t stage_inclusive_sum_scratch(int64_t n);
int32_t stage_inclusive_sum(const int64_t* in, int64_t n, int64_t* out, int32_t* overflow, void* scratch,
                            size_t bytes, cudaStream_t st);
int32_t stage_duplicate(const adr_projection& p, int64_t n, const int64_t* offsets, int32_t tx, int32_t ty,
                        uint64_t* keys, int64_t* gidx, cudaStream_t st);
size_t stage_sort_scratch(int64_t p);
int32_t stage_sort(const uint64_t* k, const int64_t* v, int64_t p, int32_t end_bit, uint64_t* ko, int64_t* vo,
                   void* scratch, size_t bytes, cudaStream_t st);
int32_t stage_ranges(const uint64_t* keys, int64_t p, int64_t n_tiles, int64_t* ranges, int32_t* error,
                     cudaStream_t st);

// Fused-frame binning: compaction → depth-rank sort of Gaussians → rank-ordered
// pair emission → stable onesweep tile sort (with the reference-layout export)
// → tile ranges.
struct FrameBinning {
    adr_projection proj;
    int64_t n = 0;
    int64_t cap = 0;            // pair capacity
    int64_t n_tiles = 0;
    int32_t tiles_x = 0, tiles_y = 0;
    const uint32_t* dkey = nullptr;  // stage 1 depth-sort key (all-ones: no pairs)
    const uint2* gpack = nullptr;  // per-Gaussian packed tile rect (stage 1)
    const uint32_t* kminmax = nullptr;  // per preprocess block: min / max selected depth key (optional)
    uint32_t* plan_mm = nullptr;        // depth plan (min, max), reset by the preprocess
    uint32_t* order = nullptr;  // scratch: order[rank] = Gaussian index
    int64_t* ranges = nullptr;  // out: (n_tiles, 2)
    uint64_t* keys = nullptr;   // optional out: sorted keys (tile << 32 | depth bits)
    int32_t* gidx = nullptr;    // out: sorted Gaussian indices (render record index)
    int64_t* counters = nullptr;
    adr_load_stats* stats = nullptr;  // optional: reset by the ranges pass (saves the render's init launch)
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    cudaEvent_t ev_after_scan = nullptr, ev_after_dup = nullptr, ev_after_sort = nullptr,
                ev_after_ranges = nullptr;
};

size_t frame_binning_scratch(int64_t n, int64_t cap, int32_t tiles_x, int32_t tiles_y);
int32_t frame_binning(const FrameBinning& fb, cudaStream_t st);

// Supertile counting placement (adr_supertile.cu), used when the grid has at
// most 1024 supertiles of 8x8 tiles (<= 65536 tiles).
bool supertile_path(int64_t n_tiles, int32_t tiles_x, int32_t tiles_y);
size_t supertile_scratch(int64_t n, int64_t cap, int32_t tiles_x, int32_t tiles_y);
int32_t frame_binning_supertile(const FrameBinning& fb, cudaStream_t st);

}  // namespace adr
