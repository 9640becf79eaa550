// geer_common.cuh — shared device-side definitions of the B200 3DGEER path.
//
// Reference: raygauss 0.1.0 (/root/reference/pkg/src/raygauss).  Constants are
// core.py:27-51 and association.py:36-41.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "geer.h"

namespace geer {

constexpr double kMaxBlendT = 0.999;        // core.py:30
constexpr double kMinRemaining = 1e-4;      // core.py:31
constexpr double kNearLimit = 0.01;         // association.py:36
constexpr double kMinClampedOpacity = 0.05; // association.py:39
// smallest float >= 1e-4: (float)rem >= 1e-4 in fp64 <=> rem >= kMinRemainingF
constexpr float kMinRemainingF = 1.00000005e-04f;
constexpr float kMaxBlendTF = 0.999f;

constexpr int kRasterThreads = 256;  // pixels per raster work item (one CTA)
constexpr int kFwdBatch = 128;       // entries staged per forward batch
constexpr int kBwdBatch = 32;        // entries per backward reduction batch

// Per-frame camera / config constants, passed by value to every kernel.
struct FrameConst {
    int width, height, model, tile_px;
    int n_x, n_y, n_tiles, n_bands;
    int cutoff, pad_;
    double R[9], t[3], origin[3];
    double fov_x, fov_y, fx, fy, cx, cy, k[4];
    double lam, lam2;
    float bg[3];
    float lam2f;
};

// fp32 raster payload, one per Gaussian (80 B, 16-B aligned):
//   r0..r2 = (W_i0, W_i1, W_i2, o_u_i)  rows of W = S^-1 R^T with o_u = W (o - mu)
//   col    = (r, g, b, sigma)
//   ext    = (kappa band, 0, 0, 0)   half-width of the fp64 re-check band around lam^2
struct __align__(16) Payload {
    float4 r0, r1, r2, col, ext;
};

// Per-axis tile ranges: up to 3 disjoint [lo, hi) pairs packed lo | hi << 16.
struct AxisRanges {
    uint32_t x[3];
    uint32_t y[3];
};

__host__ __device__ inline int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

__host__ __device__ inline int ceil_log2(int64_t v) {
    int b = 0;
    while ((int64_t(1) << b) < v) ++b;
    return b;
}

}  // namespace geer
