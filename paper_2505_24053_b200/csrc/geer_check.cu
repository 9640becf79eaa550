// geer_check.cu — GPU oracle for the association at scale: a restatement of
// oracle.association_bruteforce (oracle.py:235-281) checked against the context's render graph.
//
// The reference's brute force samples side x side rays per tile (side = max(8, ceil(sqrt(rays)))),
// at the centres of a regular grid in bipolar angle between the tile's mirror edges
// (theta = 2 atan(edge)), and puts Gaussian g in the tile iff the minimum full-line distance
// kappa = |o_u x d_u|^2 / |d_u|^2 over those rays is <= lambda^2.  This file evaluates that for
// every (tile, kept Gaussian) pair in fp64 — O(tiles x N x rays), about 1e13 fp64 flops for the
// 1M-Gaussian 1080p config, i.e. a fraction of a second — and reports the pairs the brute force
// finds that the tile lists (K1 PBF ranges -> emit -> tile sort) lack.  A sound association has none.
// Validation only: nothing on the render path calls it.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "geer_common.cuh"
#include "geer_kernels.h"

namespace geer {
namespace {

constexpr int kMaxSide = 16;

// W = S^-1 R^T (scene.whitening_matrices, scene.py:72-75; R from the quaternion, scene.py:17-32)
// and o_u = W (o - mu) (oracle.py:253-254), one row of 12 doubles per Gaussian.
__global__ void k_whiten(geer_scene sc, const double *__restrict__ origin3, double *__restrict__ wo) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < sc.n; g += (int64_t)gridDim.x * blockDim.x) {
        double q0 = sc.quats[g * 4 + 0], q1 = sc.quats[g * 4 + 1], q2 = sc.quats[g * 4 + 2], q3 = sc.quats[g * 4 + 3];
        const double nq = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
        const double r = q0 / nq, i = q1 / nq, j = q2 / nq, k = q3 / nq;
        const double rot[9] = {1 - 2 * (j * j + k * k), 2 * (i * j - r * k),     2 * (i * k + r * j),
                               2 * (i * j + r * k),     1 - 2 * (i * i + k * k), 2 * (j * k - r * i),
                               2 * (i * k - r * j),     2 * (j * k + r * i),     1 - 2 * (i * i + j * j)};
        double w[9];
        for (int a = 0; a < 3; ++a) {
            const double s = exp((double)sc.log_scales[g * 3 + a]);
            for (int b = 0; b < 3; ++b) w[a * 3 + b] = rot[b * 3 + a] / s;
        }
        const double d[3] = {origin3[0] - sc.means[g * 3 + 0], origin3[1] - sc.means[g * 3 + 1],
                             origin3[2] - sc.means[g * 3 + 2]};
        double *o = wo + g * 12;
        for (int a = 0; a < 9; ++a) o[a] = w[a];
        for (int a = 0; a < 3; ++a) o[9 + a] = w[a * 3 + 0] * d[0] + w[a * 3 + 1] * d[1] + w[a * 3 + 2] * d[2];
    }
}

// Membership bitmap of the graph: bit (tile, gid) for every entry of the tile lists.
__global__ void k_graph_bits(const int32_t *__restrict__ ranges, const uint32_t *__restrict__ order, int n_tiles,
                             int64_t words, uint32_t *__restrict__ bits) {
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        uint32_t *row = bits + (int64_t)t * words;
        for (int e = ranges[t] + threadIdx.x; e < ranges[t + 1]; e += blockDim.x) {
            const uint32_t g = order[e];
            atomicOr(&row[g >> 5], 1u << (g & 31));
        }
    }
}

// One block per (Gaussian chunk, tile): the tile's sampled rays (world frame) in shared memory,
// one thread per Gaussian.
__global__ void __launch_bounds__(256) k_brute(FrameConst fc, int64_t n, const double *__restrict__ medges_x,
                                               const double *__restrict__ medges_y, const uint8_t *__restrict__ flags,
                                               const double *__restrict__ wo, int side, int64_t words,
                                               const uint32_t *__restrict__ graph_bits, uint32_t *__restrict__ hit_bits,
                                               unsigned long long *__restrict__ counters, int32_t *__restrict__ missing,
                                               int max_missing) {
    __shared__ double dirs[kMaxSide * kMaxSide][3];
    const int nr = side * side;
    for (int t = blockIdx.y; t < fc.n_tiles; t += gridDim.y) {
        const int iy = t / fc.n_x, ix = t - iy * fc.n_x;
        __syncthreads();
        for (int r = threadIdx.x; r < nr; r += blockDim.x) {
            const int ry = r / side, rx = r - ry * side;  // np.meshgrid(thetas, phis): row = phi
            const double t0 = 2.0 * atan(medges_x[ix]), t1 = 2.0 * atan(medges_x[ix + 1]);
            const double p0 = 2.0 * atan(medges_y[iy]), p1 = 2.0 * atan(medges_y[iy + 1]);
            const double th = t0 + (t1 - t0) * ((rx + 0.5) / side);
            const double ph = p0 + (p1 - p0) * ((ry + 0.5) / side);
            // camera.angles_to_dir (camera.py:141-155), then @ camera.rotation (oracle.py:268)
            const double st = sin(th), ct = cos(th), sp = sin(ph), cp = cos(ph);
            const double x = st * cp, y = ct * sp, z = ct * cp;
            const double nn = sqrt(x * x + y * y + z * z);
            const double dc[3] = {x / nn, y / nn, z / nn};
            for (int a = 0; a < 3; ++a) dirs[r][a] = dc[0] * fc.R[0 * 3 + a] + dc[1] * fc.R[1 * 3 + a] + dc[2] * fc.R[2 * 3 + a];
        }
        __syncthreads();
        const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        bool hit = false;
        if (g < n && (flags[g] & 1)) {
            double w[12];
            for (int a = 0; a < 12; ++a) w[a] = wo[g * 12 + a];
            for (int r = 0; r < nr && !hit; ++r) {
                const double d0 = dirs[r][0], d1 = dirs[r][1], d2 = dirs[r][2];
                const double u0 = w[0] * d0 + w[1] * d1 + w[2] * d2;
                const double u1 = w[3] * d0 + w[4] * d1 + w[5] * d2;
                const double u2 = w[6] * d0 + w[7] * d1 + w[8] * d2;
                const double m0 = w[10] * u2 - w[11] * u1, m1 = w[11] * u0 - w[9] * u2, m2 = w[9] * u1 - w[10] * u0;
                const double kappa = (m0 * m0 + m1 * m1 + m2 * m2) / (u0 * u0 + u1 * u1 + u2 * u2);
                hit = kappa <= fc.lam2;
            }
        }
        const unsigned hb = __ballot_sync(0xffffffffu, hit);
        if (hb && (threadIdx.x & 31) == 0) atomicAdd(&counters[0], (unsigned long long)__popc(hb));
        if (hit) {
            const int64_t wi = (int64_t)t * words + (g >> 5);
            if (hit_bits) atomicOr(&hit_bits[wi], 1u << (g & 31));
            if (!((graph_bits[wi] >> (g & 31)) & 1)) {
                const unsigned long long k = atomicAdd(&counters[1], 1ull);
                if ((int64_t)k < max_missing && missing) {
                    missing[2 * k] = t;
                    missing[2 * k + 1] = (int32_t)g;
                }
            }
        }
    }
}

__global__ void k_count_kept(const uint8_t *__restrict__ flags, int64_t n, unsigned long long *__restrict__ out) {
    int c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += flags[i] & 1;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

}  // namespace

int launch_assoc_check(const FrameConst &fc, const geer_scene &sc, const double *medges_x, const double *medges_y,
                       const uint8_t *flags, const int32_t *ranges, const uint32_t *order, int side, double *wo,
                       double *origin3, uint32_t *graph_bits, uint32_t *hit_bits, unsigned long long *counters,
                       int32_t *missing, int max_missing, cudaStream_t st) {
    if (side < 1 || side > kMaxSide) return GEER_ERR_INVALID;
    const int64_t n = sc.n, words = (n + 31) / 32;
    cudaMemsetAsync(counters, 0, 3 * sizeof(unsigned long long), st);
    cudaMemcpyAsync(origin3, fc.origin, 3 * sizeof(double), cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(graph_bits, 0, (size_t)fc.n_tiles * words * 4, st);
    if (hit_bits) cudaMemsetAsync(hit_bits, 0, (size_t)fc.n_tiles * words * 4, st);
    if (n == 0) return cudaGetLastError() == cudaSuccess ? GEER_OK : GEER_ERR_CUDA;
    const int gb = (int)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
    k_whiten<<<gb, 256, 0, st>>>(sc, origin3, wo);
    k_count_kept<<<gb, 256, 0, st>>>(flags, n, counters + 2);
    k_graph_bits<<<fc.n_tiles < 148 * 16 ? fc.n_tiles : 148 * 16, 256, 0, st>>>(ranges, order, fc.n_tiles, words,
                                                                                 graph_bits);
    const dim3 grid((unsigned)((n + 255) / 256), (unsigned)(fc.n_tiles < 65535 ? fc.n_tiles : 65535));
    k_brute<<<grid, 256, 0, st>>>(fc, n, medges_x, medges_y, flags, wo, side, words, graph_bits, hit_bits, counters,
                                  missing, max_missing);
    return cudaGetLastError() == cudaSuccess ? GEER_OK : GEER_ERR_CUDA;
}

}  // namespace geer
