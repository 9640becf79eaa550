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

// Per-frame camera / config constants, passed by value to every kernel.
struct FrameConst {
    int width, height, model, tile_px;
    int n_x, n_y, n_tiles, n_bands;
    int cutoff;
    int cull;  // per-warp PBF culling of raster entries (support cutoff on and not disabled)
    int exhaustive;  // GEER_CFG_EXHAUSTIVE: every tile's list = all kept Gaussians in depth order
    double R[9], t[3], origin[3];
    double fov_x, fov_y, fx, fy, cx, cy, k[4];
    double lam, lam2;
    float bg[3];
    float lam2f;
    float cutoff_tol;  // |kappa_fp32 - lam^2| below which the cutoff is re-decided in fp64 (generic path)
    float thrk;        // kHalfLog2e * lam^2: the cutoff in the raster's scaled units k = kHalfLog2e * kappa
    float thrkc;       // thrk under the support cutoff, +inf without it (renderer.py:103-105)
};

// exp(-kappa / 2) = 2^(-kHalfLog2e kappa): the raster works with k = kHalfLog2e kappa (ex2 argument).
constexpr double kHalfLog2e = 0.72134752044448170;
constexpr double kSqrtHalfLog2e = 0.84932180028801907;  // m is stored scaled by this, so |m|^2 / dd = k

// Per raster work item (cached with the camera): an orthonormal fp64 frame (dc = normalised sum of the
// item's world rays, e1, e2) in which every pixel ray of the item is d' = dc + x e1 + y e2 (d' = d /
// (d . dc); kappa is scale-invariant in d).  rx, ry bound |x|, |y| over the item's pixels; rx < 0
// marks an item too wide for the offset evaluation (cone > 60 deg), which takes the fp64 path.
struct __align__(16) ItemFrame {
    double dc[3], e1[3], e2[3];
    float rx, ry, pad0, pad1;
};

// Raster culling record of one Gaussian (48 B, written by K1, streamed with the payload):
//   box  = PBF hull in camera-frame mirror space (x_lo, x_hi, y_lo, y_hi), outward-rounded
//   k0, k1 = visual-cone matrix K (K00, K11, K22, K01 | K02, K12, lambda_max bound, 0), see cone_misses
struct __align__(16) Cull {
    float4 box;
    float4 k0, k1;
};

// Raster payload, one per Gaussian (176 B, see make_payload in geer_geometry.cu; one TMA row):
//   q[12]  W (row-major, W = S^-1 R^T) and o_u = W (o - mu) in fp64 (renderer.py:78-79)
//   col  = (r, g, b, sigma)
//   ext  = (absolute kappa error bound of the fp64 cross-product evaluation, the fp64 opacity as two
//           32-bit halves (lo, hi), 0)
//   cull = the culling record (written by the association half of K1)
struct __align__(16) Payload {
    double q[12];
    float4 col;
    float4 ext;
    Cull cull;
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
