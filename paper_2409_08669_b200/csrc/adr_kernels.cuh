// adr_kernels.cuh — host-side launchers shared between translation units.
#pragma once

#include "adr_common.cuh"

namespace adr {

// Render-side per-Gaussian record (indexed by Gaussian), 48 bytes.
//   a = (mx, my, conic_a, conic_b)
//   b = (conic_c, opacity, r, g)
//   c = (b, unused, unused, unused)
struct __align__(16) Record {
    float4 a, b, c;
};

// Extra per-Gaussian outputs the fused frame needs from stage 1.
struct FusedPre {
    Record* rec = nullptr;                    // render record (valid rows)
    uint4* gpack = nullptr;                   // (x0 | x1 << 16, y0 | y1 << 16, 0, depth bits)
    unsigned long long* culled = nullptr;     // += number of !valid rows
    uint32_t* dkey = nullptr;                 // depth-sort key (all-ones: no pairs)
    int64_t* d_m = nullptr;                   // += number of Gaussians with pairs (zeroed)
    int32_t tiles_x = 0, tiles_y = 0;
};

int32_t launch_preprocess(const adr_scene& scene, const adr_camera& cam, int32_t mode,
                          double alpha_low, double dilation, const adr_projection& out,
                          const FusedPre* fused, cudaStream_t st);

struct RenderArgs {
    const Record* rec;        // records
    const uint32_t* idx;      // per sorted pair: record index
    const int64_t* ranges;    // (n_tiles, 2) int64 spans
    int32_t width, height, tiles_x, tiles_y;
    float bg[3];
    float alpha_low;
    float term;
    float* pixels;
    int32_t* load;
    adr_load_stats* stats;    // may be null
    int32_t* hist;            // may be null
    int32_t hist_bins;
};

int32_t launch_render(const RenderArgs& a, cudaStream_t st);
int32_t launch_render_proj(const adr_projection& p, const int64_t* gidx, const int64_t* ranges, int32_t width,
                           int32_t height, const float* bg, float alpha_low, float term, float* pixels,
                           int32_t* load, adr_load_stats* stats, int32_t* hist, int32_t bins, cudaStream_t st);
int32_t launch_init_stats(adr_load_stats* stats, int32_t* hist, int32_t bins, cudaStream_t st);

}  // namespace adr
