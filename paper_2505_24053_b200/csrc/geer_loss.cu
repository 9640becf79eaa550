// geer_loss.cu — the training loss of the multi-view step on the GPU:
// masked (1 - w) L1 + w (1 - SSIM) and its analytic image gradient, restating raygauss
// trainer.loss (trainer.py:114-155) with _ssim_channel / _ssim_channel_backward (:39-69).
//
// SSIM uses scipy's gaussian_filter(sigma 1.5, truncate 3.5, mode="constant"): an 11-tap separable
// zero-padded Gaussian (trainer.py:26-36), which is self-adjoint, so the backward blurs with the
// same filter.  Two tiled kernels (32 x 32 outputs + a 5-pixel halo in shared memory):
//   k_ssim_fwd : per channel the five blurred moments, the SSIM map summed over the cropped region,
//                and the three per-pixel adjoint inputs (d ux, d uxx, d uxy) -> 9 planes
//   k_ssim_bwd : blur of those planes, combined with x, y and the L1 sign term -> dL/dimage
// Sums (L1, SSIM, pixel counts) are accumulated in fp64 on the device.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "geer.h"

namespace {

constexpr int kR = 5;             // int(3.5 * 1.5 + 0.5), trainer.py:28
constexpr int kT = 32;            // output tile
constexpr int kH = kT + 2 * kR;   // tile + halo
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;  // trainer.py:29-30

__constant__ float c_w[2 * kR + 1];  // normalised Gaussian taps (scipy _gaussian_kernel1d)

struct LossSums {
    double l1, ssim[3];
    unsigned long long n_valid, n_region;
};

__device__ __forceinline__ bool in_region(const uint8_t *mask, int y, int x, int H, int W) {
    // trainer.py:72-76 _crop_mask: the window-radius border is never averaged
    if (H <= 2 * kR || W <= 2 * kR) return false;
    if (y < kR || y >= H - kR || x < kR || x >= W - kR) return false;
    return mask == nullptr || mask[(int64_t)y * W + x] != 0;
}

constexpr int kRun = 4;  // consecutive outputs per thread in the sliding 11-tap window

// Horizontal pass for M planes at once: tmp[m][r][c] = sum_k w_k src_m[r][c + k] over the haloed rows.
// src_m(i) is evaluated from the staged x / y planes (moments) or read directly.
template <int M, class Src>
__device__ __forceinline__ void hblur(Src src, float (*tmp)[kH * kT]) {
    for (int i = threadIdx.x; i < kH * (kT / kRun); i += blockDim.x) {
        const int r = i / (kT / kRun), c0 = (i % (kT / kRun)) * kRun;
        float acc[M][kRun];
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
            for (int o = 0; o < kRun; ++o) acc[m][o] = 0.f;
#pragma unroll
        for (int k = 0; k < kRun + 2 * kR; ++k) {
            float v[M];
            src(r * kH + c0 + k, v);
#pragma unroll
            for (int o = 0; o < kRun; ++o) {
                const int t = k - o;  // tap index of this input for output o
                if (t >= 0 && t <= 2 * kR)
#pragma unroll
                    for (int m = 0; m < M; ++m) acc[m][o] = fmaf(c_w[t], v[m], acc[m][o]);
            }
        }
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
            for (int o = 0; o < kRun; ++o) tmp[m][r * kT + c0 + o] = acc[m][o];
    }
}

// Vertical pass for M planes: out[m][o] = blurred value at (r0 + o, c) of this thread's run.
template <int M>
__device__ __forceinline__ void vblur(const float (*tmp)[kH * kT], int r0, int c, float (&out)[M][kRun]) {
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
        for (int o = 0; o < kRun; ++o) out[m][o] = 0.f;
#pragma unroll
    for (int k = 0; k < kRun + 2 * kR; ++k) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const float v = tmp[m][(r0 + k) * kT + c];
#pragma unroll
            for (int o = 0; o < kRun; ++o) {
                const int t = k - o;
                if (t >= 0 && t <= 2 * kR) out[m][o] = fmaf(c_w[t], v, out[m][o]);
            }
        }
    }
}

// trainer.py:123: invalid target pixels take the target value (r_eff); zero outside the image
__device__ __forceinline__ void load_xy(const float *color, const float *target, const uint8_t *mask, int H, int W,
                                        int y, int x, int c, float &xv, float &yv) {
    xv = yv = 0.f;
    if (y >= 0 && y < H && x >= 0 && x < W) {
        const int64_t p = (int64_t)y * W + x;
        yv = target[p * 3 + c];
        xv = (mask == nullptr || mask[p]) ? color[p * 3 + c] : yv;
    }
}

__global__ void __launch_bounds__(256, 3) k_ssim_fwd(const float *__restrict__ color, const float *__restrict__ target,
                                                  const uint8_t *__restrict__ mask, int H, int W,
                                                  float *__restrict__ adj, double *__restrict__ partial) {
    __shared__ float xs[kH * kH], ys[kH * kH];  // x and y over the haloed tile
    __shared__ double red[8][6];
    __shared__ float tmp[5][kH * kT];           // horizontally blurred x, y, xx, yy, xy
    const int y0 = blockIdx.y * kT - kR, x0 = blockIdx.x * kT - kR;
    const int64_t plane = (int64_t)H * W;
    double l1 = 0.0, ss[3] = {0.0, 0.0, 0.0};
    unsigned long long nv = 0, nr = 0;
    const int c = threadIdx.x % kT, r0 = (threadIdx.x / kT) * kRun;  // this thread's output run
    for (int ch = 0; ch < 3; ++ch) {
        for (int i = threadIdx.x; i < kH * kH; i += blockDim.x) {
            float xv, yv;
            load_xy(color, target, mask, H, W, y0 + i / kH, x0 + i % kH, ch, xv, yv);
            xs[i] = xv;
            ys[i] = yv;
        }
        __syncthreads();
        hblur<5>([&](int i, float (&v)[5]) {
            const float xv = xs[i], yv = ys[i];
            v[0] = xv; v[1] = yv; v[2] = xv * xv; v[3] = yv * yv; v[4] = xv * yv;
        }, tmp);
        __syncthreads();
        float bm[5][kRun];
        vblur<5>(tmp, r0, c, bm);
#pragma unroll
        for (int o = 0; o < kRun; ++o) {
            const int y = blockIdx.y * kT + r0 + o, x = blockIdx.x * kT + c;
            if (y >= H || x >= W) continue;
            const int64_t p = (int64_t)y * W + x;
            // trainer.py:39-52 (_ssim_channel) and :55-69 (_ssim_channel_backward, before the blurs)
            const double ux = bm[0][o], uy = bm[1][o];
            const double vx = bm[2][o] - ux * ux, vy = bm[3][o] - uy * uy, vxy = bm[4][o] - ux * uy;
            const double a1 = 2.0 * ux * uy + kC1, a2 = 2.0 * vxy + kC2;
            const double b1 = ux * ux + uy * uy + kC1, b2 = vx + vy + kC2;
            // 1 / (b1 b2) from the fp32 reciprocal and two Newton steps (relative error ~1e-15; b1, b2 > 0)
            const double den = b1 * b2;
            double inv = (double)__frcp_rn((float)den);
            inv = fma(inv, fma(-den, inv, 1.0), inv);
            inv = fma(inv, fma(-den, inv, 1.0), inv);
            const double s = a1 * a2 * inv;
            const bool reg = in_region(mask, y, x, H, W);
            float d_ux = 0.f, d_uxx = 0.f, d_uxy = 0.f;
            if (reg) {
                ss[ch] += s;
                // ds = 1 here; the -1 / (n_region * 3) factor is applied in k_ssim_bwd
                const double da1 = a2 * inv, da2 = a1 * inv;
                const double db1 = -s * b2 * inv, db2 = -s * b1 * inv;
                double dux = 2.0 * uy * da1 + 2.0 * ux * db1;
                const double dvx = db2, dvxy = 2.0 * da2;
                dux = dux - 2.0 * ux * dvx - uy * dvxy;
                d_ux = (float)dux;
                d_uxx = (float)dvx;
                d_uxy = (float)dvxy;
            }
            adj[(0 * 3 + ch) * plane + p] = d_ux;
            adj[(1 * 3 + ch) * plane + p] = d_uxx;
            adj[(2 * 3 + ch) * plane + p] = d_uxy;
            const bool valid = mask == nullptr || mask[p] != 0;
            if (ch == 0) {
                nv += valid;
                nr += reg;
            }
            // (staged: x = colour where the mask is set)
            if (valid) l1 += fabs((double)xs[(r0 + o + kR) * kH + c + kR] - (double)ys[(r0 + o + kR) * kH + c + kR]);
        }
        __syncthreads();
    }
    // block partials (no same-address atomics: k_loss_reduce sums the blocks)
    double v[6] = {l1, ss[0], ss[1], ss[2], (double)nv, (double)nr};
#pragma unroll
    for (int k = 0; k < 6; ++k)
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 6; ++k) red[threadIdx.x >> 5][k] = v[k];
    __syncthreads();
    if (threadIdx.x < 6) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w][threadIdx.x];
        partial[(int64_t)(blockIdx.y * gridDim.x + blockIdx.x) * 6 + threadIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) k_loss_reduce(const double *__restrict__ partial, int n_blocks,
                                                      LossSums *__restrict__ sums) {
    __shared__ double red[32][6];
    double v[6] = {0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < n_blocks; b += blockDim.x)
        for (int k = 0; k < 6; ++k) v[k] += partial[(int64_t)b * 6 + k];
    for (int k = 0; k < 6; ++k)
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 6; ++k) red[threadIdx.x >> 5][k] = v[k];
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[6] = {0, 0, 0, 0, 0, 0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            for (int k = 0; k < 6; ++k) t[k] += red[w][k];
        sums->l1 = t[0];
        sums->ssim[0] = t[1];
        sums->ssim[1] = t[2];
        sums->ssim[2] = t[3];
        sums->n_valid = (unsigned long long)t[4];
        sums->n_region = (unsigned long long)t[5];
    }
}

__global__ void __launch_bounds__(256) k_ssim_bwd(const float *__restrict__ color, const float *__restrict__ target,
                                                  const uint8_t *__restrict__ mask, int H, int W, float ssim_weight,
                                                  const float *__restrict__ adj, const LossSums *__restrict__ sums,
                                                  float *__restrict__ grad) {
    __shared__ float q[3][kH * kH];
    __shared__ float tmp[3][kH * kT];
    const int y0 = blockIdx.y * kT - kR, x0 = blockIdx.x * kT - kR;
    const int64_t plane = (int64_t)H * W;
    const double nv = (double)sums->n_valid, nr = (double)sums->n_region;
    const float s_l1 = nv > 0 ? (float)((1.0 - ssim_weight) / (nv * 3.0)) : 0.f;  // trainer.py:131
    const float s_ss = nr > 0 ? (float)(-ssim_weight / (nr * 3.0)) : 0.f;         // trainer.py:145
    const int c = threadIdx.x % kT, r0 = (threadIdx.x / kT) * kRun;
    for (int ch = 0; ch < 3; ++ch) {
        for (int i = threadIdx.x; i < kH * kH; i += blockDim.x) {
            const int y = y0 + i / kH, x = x0 + i % kH;
            const bool in = y >= 0 && y < H && x >= 0 && x < W;
            const int64_t p = (int64_t)y * W + x;
#pragma unroll
            for (int m = 0; m < 3; ++m) q[m][i] = in ? adj[(m * 3 + ch) * plane + p] : 0.f;
        }
        __syncthreads();
        hblur<3>([&](int i, float (&v)[3]) {
            v[0] = q[0][i]; v[1] = q[1][i]; v[2] = q[2][i];
        }, tmp);
        __syncthreads();
        float bm[3][kRun];
        vblur<3>(tmp, r0, c, bm);
#pragma unroll
        for (int o = 0; o < kRun; ++o) {
            const int y = blockIdx.y * kT + r0 + o, x = blockIdx.x * kT + c;
            if (y >= H || x >= W) continue;
            const int64_t p = (int64_t)y * W + x;
            float g = 0.f;
            if (mask == nullptr || mask[p] != 0) {  // trainer.py:147 dssim[~mask] = 0; :130-131 L1 on the mask
                const float xv = color[p * 3 + ch], yv = target[p * 3 + ch];
                const float d = xv - yv;
                const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
                // trainer.py:69: blur(dux) + 2 x blur(duxx) + y blur(duxy)
                const float dss = bm[0][o] + 2.f * xv * bm[1][o] + yv * bm[2][o];
                g = s_l1 * sgn + s_ss * dss;
            }
            grad[p * 3 + ch] = g;
        }
        __syncthreads();
    }
}

__global__ void k_loss_total(const LossSums *__restrict__ sums, float ssim_weight, double *__restrict__ out) {
    const double nv = (double)sums->n_valid, nr = (double)sums->n_region;
    const double l1 = nv > 0 ? sums->l1 / (nv * 3.0) : 0.0;
    double s_mean = 0.0;
    for (int c = 0; c < 3; ++c) s_mean += (nr > 0 ? sums->ssim[c] / nr : 0.0) / 3.0;
    const double ssim_loss = (ssim_weight > 0.f && nr > 0) ? 1.0 - s_mean : 0.0;
    out[0] = nv > 0 ? (1.0 - ssim_weight) * l1 + ssim_weight * ssim_loss : 0.0;  // trainer.py:152
    out[1] = l1;
    out[2] = ssim_loss;
}

void gaussian_taps(float w[2 * kR + 1]) {  // scipy.ndimage _gaussian_kernel1d(sigma=1.5, order=0, radius=5)
    const double s2 = 1.5 * 1.5;
    double t[2 * kR + 1], sum = 0.0;
    for (int k = -kR; k <= kR; ++k) sum += (t[k + kR] = exp(-0.5 / s2 * k * k));
    for (int k = 0; k <= 2 * kR; ++k) w[k] = (float)(t[k] / sum);
}

}  // namespace

extern "C" {

size_t geer_loss_workspace_bytes(int height, int width) {
    const size_t blocks = (size_t)((width + kT - 1) / kT) * ((height + kT - 1) / kT);
    return 256 + ((blocks * 6 * sizeof(double) + 255) / 256) * 256 + sizeof(float) * 9 * (size_t)height * width;
}

int geer_loss(const float *color, const float *target, const uint8_t *mask, int height, int width, float ssim_weight,
              void *workspace, double *out, float *dl_dimage, void *stream) {
    if (!color || !target || !workspace || !out || !dl_dimage || height <= 0 || width <= 0) return GEER_ERR_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    static bool taps_ready[64] = {};  // __constant__ taps are per device
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return GEER_ERR_CUDA;
    if (!taps_ready[dev]) {
        float w[2 * kR + 1];
        gaussian_taps(w);
        if (cudaMemcpyToSymbol(c_w, w, sizeof(w)) != cudaSuccess) return GEER_ERR_CUDA;
        taps_ready[dev] = true;
    }
    static_assert(sizeof(LossSums) <= 256, "workspace header");
    const dim3 grid((width + kT - 1) / kT, (height + kT - 1) / kT);
    const int n_blocks = (int)(grid.x * grid.y);
    LossSums *sums = reinterpret_cast<LossSums *>(workspace);
    double *partial = reinterpret_cast<double *>(reinterpret_cast<char *>(workspace) + 256);
    float *adj = reinterpret_cast<float *>(reinterpret_cast<char *>(workspace) + 256 +
                                           ((n_blocks * 6 * sizeof(double) + 255) / 256) * 256);
    k_ssim_fwd<<<grid, 256, 0, st>>>(color, target, mask, height, width, adj, partial);
    k_loss_reduce<<<1, 1024, 0, st>>>(partial, n_blocks, sums);
    k_ssim_bwd<<<grid, 256, 0, st>>>(color, target, mask, height, width, ssim_weight, adj, sums, dl_dimage);
    k_loss_total<<<1, 1, 0, st>>>(sums, ssim_weight, out);
    return cudaGetLastError() == cudaSuccess ? GEER_OK : GEER_ERR_CUDA;
}

}  // extern "C"
