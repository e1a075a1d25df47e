// adr_metrics.cu — image-quality terms of the load-balancing objective
// (sb/metrics.py:94-143): L1 and SSIM of a rendered image against a
// reference, in fp64, for the GPU toy optimizer.
//
// SSIM follows sb/metrics.py:120-140: per channel, windowed means with an
// 11-tap Gaussian (sigma 1.5, computed on the host with numpy's own
// expression) applied as scipy.ndimage.correlate1d along axis 0 then axis 1
// with zero padding; the symmetric-kernel summation order of scipy's
// NI_Correlate1D (centre tap first, then (in[-j] + in[+j]) * w[j] from the
// outermost pair inwards) and the reference's expression order for the SSIM
// map are kept, so per-pixel values agree to the last bit or so; the image
// mean is a fixed-order (deterministic) reduction.
#include "adr_common.cuh"

namespace adr {
namespace {

constexpr int kT = 32;               // output tile side
constexpr int kHalo = 5;             // (11 - 1) / 2
constexpr int kIn = kT + 2 * kHalo;  // 42
constexpr int kThreads = 256;

struct Win {
    double w[11];
    double c1, c2;
};

__global__ void __launch_bounds__(kThreads)
k_ssim_l1(const float* __restrict__ a, const float* __restrict__ b, int32_t width, int32_t height, Win win,
          double* __restrict__ part) {
    extern __shared__ __align__(16) unsigned char m_smem[];
    float* sx = reinterpret_cast<float*>(m_smem);                 // kIn x kIn
    float* sy = sx + kIn * kIn;
    double* v = reinterpret_cast<double*>(sy + kIn * kIn);        // 5 x kT x kIn (vertical sums)
    __shared__ double red[2][kThreads / 32];
    const int ch = blockIdx.z;
    const int x0 = blockIdx.x * kT - kHalo, y0 = blockIdx.y * kT - kHalo;
    for (int i = threadIdx.x; i < kIn * kIn; i += kThreads) {
        const int r = i / kIn, c = i - r * kIn;
        const int gy = y0 + r, gx = x0 + c;
        const bool in = gx >= 0 && gx < width && gy >= 0 && gy < height;
        const int64_t o = ((int64_t)gy * width + gx) * 3 + ch;
        sx[i] = in ? a[o] : 0.0f;
        sy[i] = in ? b[o] : 0.0f;
    }
    __syncthreads();
    // axis 0 (rows): output row r of the tile, every input column c
    for (int i = threadIdx.x; i < kT * kIn; i += kThreads) {
        const int r = i / kIn, c = i - r * kIn;
        const int rc = r + kHalo;
        double q[5];
        {
            const double x = sx[rc * kIn + c], y = sy[rc * kIn + c];
            q[0] = __dmul_rn(x, win.w[5]);
            q[1] = __dmul_rn(y, win.w[5]);
            q[2] = __dmul_rn(__dmul_rn(x, x), win.w[5]);
            q[3] = __dmul_rn(__dmul_rn(y, y), win.w[5]);
            q[4] = __dmul_rn(__dmul_rn(x, y), win.w[5]);
        }
#pragma unroll
        for (int j = kHalo; j >= 1; --j) {
            const double xm = sx[(rc - j) * kIn + c], xp = sx[(rc + j) * kIn + c];
            const double ym = sy[(rc - j) * kIn + c], yp = sy[(rc + j) * kIn + c];
            const double wj = win.w[5 - j];
            q[0] = __dadd_rn(q[0], __dmul_rn(__dadd_rn(xm, xp), wj));
            q[1] = __dadd_rn(q[1], __dmul_rn(__dadd_rn(ym, yp), wj));
            q[2] = __dadd_rn(q[2], __dmul_rn(__dadd_rn(__dmul_rn(xm, xm), __dmul_rn(xp, xp)), wj));
            q[3] = __dadd_rn(q[3], __dmul_rn(__dadd_rn(__dmul_rn(ym, ym), __dmul_rn(yp, yp)), wj));
            q[4] = __dadd_rn(q[4], __dmul_rn(__dadd_rn(__dmul_rn(xm, ym), __dmul_rn(xp, yp)), wj));
        }
        // columns outside the image: the axis-0 result is zero there (the
        // second pass pads with zeros, sb/metrics.py:114-117)
        const int gx = x0 + c;
        const bool colin = gx >= 0 && gx < width;
#pragma unroll
        for (int k = 0; k < 5; ++k) v[(k * kT + r) * kIn + c] = colin ? q[k] : 0.0;
    }
    __syncthreads();
    // axis 1 (columns) + SSIM map + L1, for the kT x kT outputs
    double s_ssim = 0.0, s_l1 = 0.0;
    for (int i = threadIdx.x; i < kT * kT; i += kThreads) {
        const int r = i / kT, c = i - r * kT;
        const int gy = blockIdx.y * kT + r, gx = blockIdx.x * kT + c;
        if (gx >= width || gy >= height) continue;
        const int cc = c + kHalo;
        double m[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const double* row = v + (k * kT + r) * kIn;
            double acc = __dmul_rn(row[cc], win.w[5]);
#pragma unroll
            for (int j = kHalo; j >= 1; --j) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(row[cc - j], row[cc + j]), win.w[5 - j]));
            m[k] = acc;
        }
        const double mu_x = m[0], mu_y = m[1];
        const double var_x = __dsub_rn(m[2], __dmul_rn(mu_x, mu_x));
        const double var_y = __dsub_rn(m[3], __dmul_rn(mu_y, mu_y));
        const double cov = __dsub_rn(m[4], __dmul_rn(mu_x, mu_y));
        const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mu_x), mu_y), win.c1),
                                     __dadd_rn(__dmul_rn(2.0, cov), win.c2));
        const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mu_x, mu_x), __dmul_rn(mu_y, mu_y)), win.c1),
                                     __dadd_rn(__dadd_rn(var_x, var_y), win.c2));
        s_ssim = __dadd_rn(s_ssim, __ddiv_rn(num, den));
        const double x = sx[(r + kHalo) * kIn + cc], y = sy[(r + kHalo) * kIn + cc];
        s_l1 = __dadd_rn(s_l1, fabs(__dsub_rn(x, y)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s_ssim += __shfl_xor_sync(0xffffffffu, s_ssim, o);
        s_l1 += __shfl_xor_sync(0xffffffffu, s_l1, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = s_ssim;
        red[1][threadIdx.x >> 5] = s_l1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) {
            t0 += red[0][w];
            t1 += red[1][w];
        }
        const int64_t blk = ((int64_t)ch * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        part[2 * blk] = t0;
        part[2 * blk + 1] = t1;
    }
}

// Fixed-order reduction of the per-tile partials: out[0] = mean |a - b| over
// all H*W*3 values, out[1] = mean over channels of the per-channel mean SSIM
// (sb/metrics.py:94-97, :135-140).  96 threads: warp c sums channel c.
__global__ void k_loss_finalize(const double* __restrict__ part, int64_t tiles_per_ch, int32_t width,
                                int32_t height, double* __restrict__ out) {
    __shared__ double s[2][3][32];
    const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
    double ss = 0.0, ll = 0.0;
    for (int64_t t = lane; t < tiles_per_ch; t += 32) {
        ss += part[2 * (c * tiles_per_ch + t)];
        ll += part[2 * (c * tiles_per_ch + t) + 1];
    }
    s[0][c][lane] = ss;
    s[1][c][lane] = ll;
    __syncthreads();
    if (threadIdx.x == 0) {
        const double npix = (double)width * (double)height;
        double tot_ssim = 0.0, l1 = 0.0;
        for (int ch = 0; ch < 3; ++ch) {
            double t = 0.0;
            for (int k = 0; k < 32; ++k) t += s[0][ch][k];
            tot_ssim += t / npix;
            for (int k = 0; k < 32; ++k) l1 += s[1][ch][k];
        }
        out[0] = l1 / (npix * 3.0);
        out[1] = tot_ssim / 3.0;
    }
}

inline int64_t tiles_of32(int32_t v) { return (v + kT - 1) / kT; }

}  // namespace
}  // namespace adr

using namespace adr;

extern "C" {

size_t adr_image_loss_scratch_bytes(int32_t width, int32_t height) {
    return align_up(sizeof(double) * 2 * 3 * (size_t)(tiles_of32(width) * tiles_of32(height)));
}

int32_t adr_image_losses(const float* d_a, const float* d_b, int32_t width, int32_t height, const double* h_window,
                         double c1, double c2, double* d_out, void* d_scratch, size_t scratch_bytes, void* stream) {
    if (!d_a || !d_b || !h_window || !d_out) return fail(ADR_ERR_VALUE, "null argument");
    if (width < 1 || height < 1) return fail(ADR_ERR_VALUE, "image dimensions must be positive");
    if (scratch_bytes < adr_image_loss_scratch_bytes(width, height)) return fail(ADR_ERR_VALUE, "scratch too small");
    cudaStream_t st = as_stream(stream);
    Win win;
    for (int i = 0; i < 11; ++i) win.w[i] = h_window[i];
    win.c1 = c1;
    win.c2 = c2;
    const dim3 grid((unsigned)tiles_of32(width), (unsigned)tiles_of32(height), 3);
    const size_t smem = 2 * sizeof(float) * kIn * kIn + 5 * sizeof(double) * kT * kIn;
    ADR_CUDA_TRY(cudaFuncSetAttribute(k_ssim_l1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_ssim_l1<<<grid, kThreads, smem, st>>>(d_a, d_b, width, height, win, static_cast<double*>(d_scratch));
    ADR_LAUNCH_CHECK();
    k_loss_finalize<<<1, 96, 0, st>>>(static_cast<const double*>(d_scratch), (int64_t)grid.x * grid.y, width,
                                      height, d_out);
    ADR_LAUNCH_CHECK();
    return ADR_OK;
}

}  // extern "C"
