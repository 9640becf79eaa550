// geer_geometry.cu — fp64 per-camera and per-Gaussian stages.
//
//   K0  camera setup: BEAP trig tables / pinhole+KB per-pixel rays, CSF tile
//       edges in mirror space, pixel -> tile CSR, raster work items
//       (camera.py:119-190,213-282; association.py:91-105,301-332)
//   K1  per-Gaussian preprocess: view transform, PD check, PBF roots, mirror
//       arcs, tile ranges, depth key, fp32 raster payload, SH colour
//       (scene.py:17-80; association.py:82-88,129-224,343-350,373-451;
//        renderer.py:57-81)
//   K7  per-Gaussian backward finalisation (renderer.py:204-231,320-332)
//
// This translation unit is compiled with -fmad=false: every fp64 expression
// rounds exactly like the numpy statement it restates (no contraction), so
// the association decisions (tile sets, clamps, depth keys) are the
// reference's bit for bit except at enumerated ulp ties.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "geer_common.cuh"
#include "geer_kernels.h"

namespace geer {

// ---------------------------------------------------------------- shared math

__device__ __forceinline__ double beap_center_angle(int idx, int n, double fov) {
    return ((idx + 0.5) - (n + 1) / 2.0) * fov / n;  // camera.py:126-127
}
__device__ __forceinline__ double beap_edge_angle(int idx, int n, double fov) {
    return (idx - (n + 1) / 2.0) * fov / n;  // camera.py:136-137
}
__device__ __forceinline__ double mirror_from_angle(double theta) {  // association.py:91-105
    double denom = cos(theta) + 1.0;
    if (fabs(denom) < 1e-300) return theta >= 0 ? INFINITY : -INFINITY;
    return sin(theta) / denom;
}

// camera.py:213-219 / 249-269: camera-space unit ray of a pinhole or KB pixel
__device__ void unproject(const FrameConst &fc, int x, int y, double out[3]) {
    double u = ((double)x - fc.cx) / fc.fx;
    double v = ((double)y - fc.cy) / fc.fy;
    if (fc.model == GEER_PINHOLE) {
        double n = sqrt(u * u + v * v + 1.0 * 1.0);
        out[0] = u / n;
        out[1] = v / n;
        out[2] = 1.0 / n;
        return;
    }
    const double *k = fc.k;
    double alpha_d = sqrt(u * u + v * v);
    double alpha = alpha_d;
    for (int it = 0; it < 20; ++it) {
        double a2 = alpha * alpha;
        double f = alpha * (1.0 + a2 * (k[0] + a2 * (k[1] + a2 * (k[2] + a2 * k[3])))) - alpha_d;
        double df = 1.0 + a2 * (3 * k[0] + a2 * (5 * k[1] + a2 * (7 * k[2] + a2 * 9 * k[3])));
        alpha = alpha - f / df;
    }
    double scale = alpha_d > 1e-12 ? sin(alpha) / fmax(alpha_d, 1e-300) : 1.0;
    double dx = u * scale, dy = v * scale, dz = cos(alpha);
    double n = sqrt(dx * dx + dy * dy + dz * dz);
    out[0] = dx / n;
    out[1] = dy / n;
    out[2] = dz / n;
}

// numpy matmul's length-3 dot product: fma(a2, b2, fma(a1, b1, a0 * b0)) (see oracle/geer_oracle.c mm3)
__device__ __forceinline__ double mm3(double a0, double b0, double a1, double b1, double a2, double b2) {
    return __fma_rn(a2, b2, __fma_rn(a1, b1, a0 * b0));
}

__device__ __forceinline__ long long ordered_bits(double x) {
    long long i = __double_as_longlong(x);
    return i >= 0 ? i : i ^ 0x7FFFFFFFFFFFFFFFLL;
}
__device__ __forceinline__ double from_ordered_bits(long long i) {
    return __longlong_as_double(i >= 0 ? i : i ^ 0x7FFFFFFFFFFFFFFFLL);
}

// ---------------------------------------------------------------- K0: BEAP

// Per-column (sin, cos) of theta and per-row (sin, cos) of phi, plus mirror edges.
__global__ void k_beap_tables(FrameConst fc, double2 *col_sc, double2 *row_sc, double *medges_x, double *medges_y) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < fc.width) {
        double th = beap_center_angle(i, fc.width, fc.fov_x);
        col_sc[i] = make_double2(sin(th), cos(th));
    }
    if (i < fc.height) {
        double ph = beap_center_angle(i, fc.height, fc.fov_y);
        row_sc[i] = make_double2(sin(ph), cos(ph));
    }
    if (i <= fc.n_x) {
        int idx = min(i * fc.tile_px, fc.width);
        medges_x[i] = mirror_from_angle(beap_edge_angle(idx, fc.width, fc.fov_x));
    }
    if (i <= fc.n_y) {
        int idx = min(i * fc.tile_px, fc.height);
        medges_y[i] = mirror_from_angle(beap_edge_angle(idx, fc.height, fc.fov_y));
    }
}

// BEAP tiles are tile_px x tile_px pixel blocks (association.py:310-316).  Pixel
// list of a 16x16 tile: pixel q = half * 128 + w * 32 + lane lies in the 8x8 patch w (2 x 2 patches)
// at row 4 * half + lane / 8, column lane % 8 — so a raster thread owning pixels q and q + 128 keeps
// both in its warp's 8x8 patch, and a warp of 32 consecutive q covers an 8x4 half-patch (coherent
// early stop either way); other tile sizes row-major.
__global__ void k_beap_csr(FrameConst fc, int32_t *tile_off, int32_t *pix_list, int32_t *pixel_tile) {
    int t = blockIdx.x;
    int tx = t % fc.n_x, ty = t / fc.n_x;
    int tp = fc.tile_px;
    int x0 = tx * tp, y0 = ty * tp;
    // association.py:314-315: the last tile absorbs nothing extra (n = ceil), so sizes are clipped
    int w = min(tp, fc.width - x0), h = min(tp, fc.height - y0);
    int64_t base = (int64_t)y0 * fc.width + (int64_t)h * x0;
    if (threadIdx.x == 0) {
        tile_off[t] = (int32_t)base;
        if (t == fc.n_tiles - 1) tile_off[fc.n_tiles] = fc.width * fc.height;
    }
    int cnt = w * h;
    bool swz = (tp == 16 && w == 16 && h == 16);
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
        int lx, ly;
        if (swz) {
            const int half = q >> 7, w = (q >> 5) & 3, lane = q & 31;
            lx = (w & 1) * 8 + (lane & 7);
            ly = (w >> 1) * 8 + half * 4 + (lane >> 3);
        } else {
            lx = q % w;
            ly = q / w;
        }
        int p = (y0 + ly) * fc.width + (x0 + lx);
        pix_list[base + q] = p;
        if (pixel_tile) pixel_tile[p] = t;
    }
}

// ---------------------------------------------------------------- K0: pinhole / KB

// Per-pixel world ray (fp64), principal angles (camera.py:158-172) and their min/max.
__global__ void k_cam_pixels(FrameConst fc, double *dir64, double *theta, double *phi, long long *minmax) {
    int64_t npx = (int64_t)fc.width * fc.height;
    double tmin = INFINITY, tmax = -INFINITY, pmin = INFINITY, pmax = -INFINITY;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npx; p += (int64_t)gridDim.x * blockDim.x) {
        int x = (int)(p % fc.width), y = (int)(p / fc.width);
        double dc[3];
        unproject(fc, x, y, dc);
        for (int j = 0; j < 3; ++j)
            dir64[p * 3 + j] = mm3(dc[0], fc.R[0 * 3 + j], dc[1], fc.R[1 * 3 + j], dc[2], fc.R[2 * 3 + j]);
        double th = atan2(dc[0], dc[2]), ph;
        if (dc[2] == 0.0)
            ph = dc[1] == 0.0 ? 0.0 : (dc[1] > 0 ? M_PI / 2 : -M_PI / 2);
        else if (dc[2] > 0)
            ph = atan2(dc[1], dc[2]);
        else
            ph = atan(dc[1] / dc[2]);
        theta[p] = th;
        phi[p] = ph;
        tmin = fmin(tmin, th);
        tmax = fmax(tmax, th);
        pmin = fmin(pmin, ph);
        pmax = fmax(pmax, ph);
    }
    for (int o = 16; o > 0; o >>= 1) {
        tmin = fmin(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
        tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        pmin = fmin(pmin, __shfl_xor_sync(0xffffffffu, pmin, o));
        pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&minmax[0], ordered_bits(tmin));
        atomicMax(&minmax[1], ordered_bits(tmax));
        atomicMin(&minmax[2], ordered_bits(pmin));
        atomicMax(&minmax[3], ordered_bits(pmax));
    }
}

// numpy.linspace(min - 1e-9, max + 1e-9, n + 1) (association.py:320-322) + mirror edges.
__global__ void k_cam_edges(FrameConst fc, const long long *minmax, double *edges_x, double *edges_y,
                            double *medges_x, double *medges_y) {
    const double pad = 1e-9;
    for (int axis = 0; axis < 2; ++axis) {
        double lo = from_ordered_bits(minmax[axis * 2 + 0]) - pad;
        double hi = from_ordered_bits(minmax[axis * 2 + 1]) + pad;
        int num = (axis == 0 ? fc.n_x : fc.n_y) + 1;
        double *e = axis == 0 ? edges_x : edges_y;
        double *m = axis == 0 ? medges_x : medges_y;
        int div = num - 1;
        double delta = hi - lo;
        double step = delta / div;
        for (int i = threadIdx.x; i < num; i += blockDim.x) {
            double y = (double)i;
            if (step == 0.0) {
                y = y / div;
                y = y * delta;
            } else {
                y = y * step;
            }
            double v = y + lo;
            if (i == num - 1) v = hi;
            e[i] = v;
            m[i] = mirror_from_angle(v);
        }
    }
}

__device__ __forceinline__ int ss_right(const double *a, int n, double v) {  // #(a <= v)
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int ss_left(const double *a, int n, double v) {  // #(a < v)
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// association.py:323-325: pixel -> tile by centre angle
__global__ void k_cam_bin(FrameConst fc, const double *theta, const double *phi, const double *edges_x,
                          const double *edges_y, int32_t *pixel_tile, int32_t *tile_count) {
    int64_t npx = (int64_t)fc.width * fc.height;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npx; p += (int64_t)gridDim.x * blockDim.x) {
        int c = ss_right(edges_x, fc.n_x + 1, theta[p]) - 1;
        int r = ss_right(edges_y, fc.n_y + 1, phi[p]) - 1;
        c = min(max(c, 0), fc.n_x - 1);
        r = min(max(r, 0), fc.n_y - 1);
        int t = r * fc.n_x + c;
        pixel_tile[p] = t;
        atomicAdd(&tile_count[t], 1);
    }
}

__global__ void k_iota(int32_t *v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (int32_t)i;
}

// ---------------------------------------------------------------- work items

// items per tile = ceil(pixels / 256) (0 for pixel-less tiles)
__global__ void k_item_counts(int n_tiles, const int32_t *tile_off, int32_t *item_count) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_tiles) {
        int c = tile_off[t + 1] - tile_off[t];
        item_count[t] = (c + kRasterThreads - 1) / kRasterThreads;
    }
}
__global__ void k_item_fill(int n_tiles, const int32_t *tile_off, const int32_t *item_off, int4 *items,
                            int32_t *n_items) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_tiles) {
        int c = tile_off[t + 1] - tile_off[t];
        int k0 = item_off[t];
        for (int k = 0; k * kRasterThreads < c; ++k)
            items[k0 + k] = make_int4(t, tile_off[t] + k * kRasterThreads, min(kRasterThreads, c - k * kRasterThreads), k0 + k);
        if (t == n_tiles - 1) *n_items = item_off[t] + (c + kRasterThreads - 1) / kRasterThreads;
    }
}

// ---------------------------------------------------------------- K1

__device__ __forceinline__ void quat_rot(const float *q4, double rot[9]) {  // scene.py:17-32
    double q0 = q4[0], q1 = q4[1], q2 = q4[2], q3 = q4[3];
    double n = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    double r = q0 / n, i = q1 / n, j = q2 / n, k = q3 / n;
    rot[0] = 1 - 2 * (j * j + k * k);
    rot[1] = 2 * (i * j - r * k);
    rot[2] = 2 * (i * k + r * j);
    rot[3] = 2 * (i * j + r * k);
    rot[4] = 1 - 2 * (i * i + k * k);
    rot[5] = 2 * (j * k - r * i);
    rot[6] = 2 * (i * k - r * j);
    rot[7] = 2 * (j * k + r * i);
    rot[8] = 1 - 2 * (i * i + j * j);
}

__device__ __forceinline__ double sigmoid(double x) {  // core.py:58-67
    if (x >= 0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}

// core.py:289-313
// One term of the basis (b a compile-time constant after unrolling), same expressions as sh_basis.
__device__ __forceinline__ double sh_term(int b, double x, double y, double z) {
    const double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    switch (b) {
        case 0: return 0.28209479177387814;
        case 1: return -0.4886025119029199 * y;
        case 2: return 0.4886025119029199 * z;
        case 3: return -0.4886025119029199 * x;
        case 4: return 1.0925484305920792 * xy;
        case 5: return -1.0925484305920792 * yz;
        case 6: return 0.31539156525252005 * (2.0 * zz - xx - yy);
        case 7: return -1.0925484305920792 * xz;
        case 8: return 0.5462742152960396 * (xx - yy);
        case 9: return -0.5900435899266435 * y * (3.0 * xx - yy);
        case 10: return 2.890611442640554 * xy * z;
        case 11: return -0.4570457994644658 * y * (4.0 * zz - xx - yy);
        case 12: return 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
        case 13: return -0.4570457994644658 * x * (4.0 * zz - xx - yy);
        case 14: return 1.445305721320277 * z * (xx - yy);
        default: return -0.5900435899266435 * x * (xx - 3.0 * yy);
    }
}

__device__ __forceinline__ void sh_basis(double x, double y, double z, double b[16]) {
#pragma unroll
    for (int k = 0; k < 16; ++k) b[k] = sh_term(k, x, y, z);
}

// association.py:129-145
__device__ __forceinline__ bool quadratic_roots(double a, double b_half, double c, double &r0, double &r1) {
    double disc = b_half * b_half - a * c;
    if (disc < 0) return false;
    double sq = sqrt(disc);
    double q = b_half >= 0 ? b_half + sq : b_half - sq;
    if (q == 0.0) {
        if (a == 0.0) return false;
        double r = fabs(sq / a);
        r0 = -r;
        r1 = r;
        return true;
    }
    double x0 = q / a, x1 = c / q;
    r0 = x1 < x0 ? x1 : x0;
    r1 = x1 < x0 ? x0 : x1;
    return true;
}

// association.py:108-126
__device__ __forceinline__ void mirror_candidates(double t, double &a, double &b) {
    double denom = 1.0 + 1.0 * 1.0 * sqrt(1.0 + t * t);
    double m = t / denom;
    if (fabs(denom) < 1e-300) m = t >= 0 ? INFINITY : -INFINITY;
    if (m == 0.0) {
        a = 0.0;
        b = INFINITY;
    } else {
        a = m;
        b = -1.0 / m;
    }
}

__device__ __forceinline__ void cswap(double &a, double &b) {
    if (b < a) {
        double t = a;
        a = b;
        b = t;
    }
}

// Absolute mirror-space margin of the raster's per-warp PBF culling bounds: far above the fp64
// rounding of the interval endpoints, far below a pixel (1920 px over 180 deg: ~8e-4 per pixel).
constexpr double kCullMargin = 1e-6;

// association.py:189-217 + :373-388 + union (:435-446): merged disjoint tile-index ranges of one axis.
// Returns the tile count; ranges packed lo | hi << 16 (empty slots = 0).  hull_lo/hull_hi: fp32
// bounds (rounded outward, widened by kCullMargin) of the arcs' union restricted to the open front
// half |m| < 1, where every camera-frame ray with z > 0 has its mirror coordinate; empty -> (+inf, -inf).
__device__ int axis_tiles(double t_aa, double t_a2, double t22, double r0, double r1, const double *edges, int n_edges,
                          uint32_t out[3], float &hull_lo, float &hull_hi) {
    double c[4];
    mirror_candidates(r0, c[0], c[1]);
    mirror_candidates(r1, c[2], c[3]);
    // sorting network (np.sort; +inf sorts last)
    cswap(c[0], c[1]);
    cswap(c[2], c[3]);
    cswap(c[0], c[2]);
    cswap(c[1], c[3]);
    cswap(c[1], c[2]);
    double lo_mid = isfinite(c[1]) ? c[1] : -1e12;
    double hi_mid = isfinite(c[2]) ? c[2] : 1e12;
    double probe = 0.5 * (lo_mid + hi_mid);
    double q;
    if (!isfinite(probe) || fabs(1.0 - probe * probe) < 1e-12) {
        q = t22;
    } else {
        double cc = 2.0 * probe / (1.0 - probe * probe);
        q = t22 * cc * cc - 2.0 * t_a2 * cc + t_aa;
    }
    double ilo[3], ihi[3];
    int ni;
    if (q >= 0) {
        ilo[0] = c[1]; ihi[0] = c[2];
        ilo[1] = c[3]; ihi[1] = INFINITY;
        ilo[2] = -INFINITY; ihi[2] = c[0];
        ni = 3;
    } else {
        ilo[0] = c[0]; ihi[0] = c[1];
        ilo[1] = c[2]; ihi[1] = c[3];
        ni = 2;
    }
    {
        double hl = INFINITY, hh = -INFINITY;
        for (int k = 0; k < ni; ++k) {
            const double lo = ilo[k] > -1.0 ? ilo[k] : -1.0, hi = ihi[k] < 1.0 ? ihi[k] : 1.0;
            if (lo <= hi) {
                hl = lo < hl ? lo : hl;
                hh = hi > hh ? hi : hh;
            }
        }
        hull_lo = hl <= hh ? __double2float_rd(hl - kCullMargin) : INFINITY;
        hull_hi = hl <= hh ? __double2float_ru(hh + kCullMargin) : -INFINITY;
    }
    const double wlo = edges[0], whi = edges[n_edges - 1];
    // tile-index range of each interval after window clipping (association.py:373-388); empty -> [BIG, BIG)
    const int BIG = 1 << 20;
    int a0[3], a1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a0[k] = BIG;
        a1[k] = BIG;
        if (k < ni) {
            const double lo2 = wlo > ilo[k] ? wlo : ilo[k];
            const double hi2 = whi < ihi[k] ? whi : ihi[k];
            if (!(lo2 > hi2)) {
                const int i0 = max(ss_right(edges, n_edges, lo2) - 1, 0);
                const int i1 = min(ss_left(edges, n_edges, hi2), n_edges - 1);
                if (i0 < i1) {
                    a0[k] = i0;
                    a1[k] = i1;
                }
            }
        }
    }
    // sort the three ranges by start (network), then merge overlapping/adjacent ones (set union)
    auto cs = [&](int i, int j) {
        if (a0[j] < a0[i]) {
            int t = a0[i]; a0[i] = a0[j]; a0[j] = t;
            t = a1[i]; a1[i] = a1[j]; a1[j] = t;
        }
    };
    cs(0, 1);
    cs(1, 2);
    cs(0, 1);
    // merge 1 into 0, then 2 into the last kept
    int m0 = a0[0], m1 = a1[0], n0 = BIG, n1 = BIG, p0 = BIG, p1 = BIG;
    if (a0[1] < BIG) {
        if (a0[1] <= m1) m1 = max(m1, a1[1]);
        else { n0 = a0[1]; n1 = a1[1]; }
    }
    if (a0[2] < BIG) {
        if (n0 < BIG) {
            if (a0[2] <= n1) n1 = max(n1, a1[2]);
            else { p0 = a0[2]; p1 = a1[2]; }
        } else if (a0[2] <= m1) {
            m1 = max(m1, a1[2]);
        } else {
            n0 = a0[2]; n1 = a1[2];
        }
    }
    int cnt = 0;
    out[0] = out[1] = out[2] = 0;
    if (m0 < BIG) { out[0] = (uint32_t)m0 | ((uint32_t)m1 << 16); cnt += m1 - m0; }
    if (n0 < BIG) { out[1] = (uint32_t)n0 | ((uint32_t)n1 << 16); cnt += n1 - n0; }
    if (p0 < BIG) { out[2] = (uint32_t)p0 | ((uint32_t)p1 << 16); cnt += p1 - p0; }
    return cnt;
}

// Raster payload of one Gaussian (renderer.py:78-80 quantities, precomputed per view): W and o_u in
// fp64 for the raster's per-item offset records and its fp64 re-checks (the cross product
// m = o_u x W d, the reference's formulation, core.py:184-199), whose kappa error grows only like
// |o_u| cond(W); the absolute bound goes to ext.x.
__device__ void make_payload(const double W[9], const double ou[3], const double rgb[3], double sigma, double cond,
                             double lam, Payload &pl) {
    const double u64 = 1.1102230246251565e-16;
    const double on = sqrt(ou[0] * ou[0] + ou[1] * ou[1] + ou[2] * ou[2]);
    for (int i = 0; i < 9; ++i) pl.q[i] = W[i];
    for (int i = 0; i < 3; ++i) pl.q[9 + i] = ou[i];
    const double band1 = 64.0 * u64 * (on + 1.0) * (cond + 1.0) * (2.0 * lam + 1.0);
    pl.col = make_float4((float)rgb[0], (float)rgb[1], (float)rgb[2], (float)sigma);
    // ext.y / ext.z: the bits of the fp64 opacity (core.py:58-67), for the fix-up's fp64 t
    pl.ext = make_float4((float)band1, __int_as_float(__double2loint(sigma)), __int_as_float(__double2hiint(sigma)), 0.f);
}

__device__ __forceinline__ void named_barrier(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// K1a: exact fp64 association of one Gaussian (association.py:82-88, 148-224, 343-350, 373-451).
// sex / sey: the mirror tile edges in shared memory.  Returns the keep / clamped flag bits.
__device__ uint8_t associate_one(const FrameConst &fc, const geer_scene &sc, const double *sex, const double *sey,
                                 int64_t g, uint32_t *__restrict__ depth_key, int64_t &count,
                                 AxisRanges *__restrict__ ranges, Cull &cr,
                                 double *__restrict__ mu_out, double *__restrict__ depth_out, int *__restrict__ err) {

    const double *R = fc.R;
    const double mean[3] = {sc.means[g * 3 + 0], sc.means[g * 3 + 1], sc.means[g * 3 + 2]};
    const float4 q4v = *reinterpret_cast<const float4 *>(sc.quats + g * 4);
    const float q4[4] = {q4v.x, q4v.y, q4v.z, q4v.w};
    double rot[9], s[3];
    quat_rot(q4, rot);
    for (int i = 0; i < 3; ++i) s[i] = exp((double)sc.log_scales[g * 3 + i]);
    // association.py:84-87
    double mu[3];
    for (int i = 0; i < 3; ++i) mu[i] = mm3(mean[0], R[i * 3 + 0], mean[1], R[i * 3 + 1], mean[2], R[i * 3 + 2]) + fc.t[i];
    double m[9], cov[9], covc[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[i * 3 + j] = rot[i * 3 + j] * s[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            cov[i * 3 + j] = mm3(m[i * 3 + 0], m[j * 3 + 0], m[i * 3 + 1], m[j * 3 + 1], m[i * 3 + 2], m[j * 3 + 2]);
    for (int i = 0; i < 3; ++i)
        for (int l = 0; l < 3; ++l) {
            double acc = 0.0;
            for (int j = 0; j < 3; ++j)
                for (int k = 0; k < 3; ++k) acc += R[i * 3 + j] * cov[j * 3 + k] * R[l * 3 + k];
            covc[i * 3 + l] = acc;
        }
    const double depth = sqrt(mu[0] * mu[0] + mu[1] * mu[1] + mu[2] * mu[2]);
    if (mu_out) {
        for (int i = 0; i < 3; ++i) mu_out[g * 3 + i] = mu[i];
        depth_out[g] = depth;
    }
    uint8_t fl = 0;
    int64_t n_ent = 0;
    AxisRanges ar;
    for (int i = 0; i < 3; ++i) ar.x[i] = ar.y[i] = 0;
    // raster culling bounds in mirror space (x_lo, x_hi, y_lo, y_hi); clamped: everything
    float4 bx = make_float4(-INFINITY, INFINITY, -INFINITY, INFINITY);
    // association.py:417-419 near cull
    if (depth >= kNearLimit) {
        // association.py:154-160 symmetric + positive-definite (Cholesky pivots)
        double amax = 0.0, dmax = 0.0;
        for (int i = 0; i < 9; ++i) amax = fmax(amax, fabs(covc[i]));
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) dmax = fmax(dmax, fabs(covc[i * 3 + j] - covc[j * 3 + i]));
        bool ok = true;
        if (dmax > 1e-9 * fmax(amax, 1e-300)) {
            atomicMax(err, (int)GEER_ERR_NOT_SYMMETRIC);
            ok = false;
        } else {
            // np.linalg.cholesky (LAPACK potf2, lower) operation sequence: reciprocal-pivot column
            // scaling and fma dot products (see oracle/geer_oracle.c)
            const double a00 = covc[0];
            bool pd = a00 > 0.0;
            if (pd) {
                const double l00 = sqrt(a00), r0 = 1.0 / l00;
                const double l10 = covc[3] * r0, l20 = covc[6] * r0;
                const double a11 = covc[4] - l10 * l10;
                pd = a11 > 0.0;
                if (pd) {
                    const double l11 = sqrt(a11);
                    const double l21 = (covc[7] - l20 * l10) * (1.0 / l11);
                    const double a22 = covc[8] - __fma_rn(l21, l21, l20 * l20);
                    pd = a22 > 0.0;
                }
            }
            if (!pd) {
                atomicMax(err, (int)GEER_ERR_NOT_PD);
                ok = false;
            }
        }
        if (ok) {
            const double lam2 = fc.lam * fc.lam;
            const double t00 = lam2 * covc[0] - mu[0] * mu[0];
            const double t02 = lam2 * covc[2] - mu[0] * mu[2];
            const double t11 = lam2 * covc[4] - mu[1] * mu[1];
            const double t12 = lam2 * covc[5] - mu[1] * mu[2];
            const double t22 = lam2 * covc[8] - mu[2] * mu[2];
            const double scale =
                fmax(fmax(fmax(fabs(t00), fabs(t02)), fmax(fabs(t11), fabs(t12))), fmax(fabs(t22), 1e-300));
            bool clamped = false;
            double rt0 = 0, rt1 = 0, rp0 = 0, rp1 = 0;
            if (fabs(t22) < 1e-12 * scale) {
                clamped = true;
            } else {
                const bool okt = quadratic_roots(t22, t02, t00, rt0, rt1);
                const bool okp = quadratic_roots(t22, t12, t11, rp0, rp1);
                clamped = !okt || !okp;
            }
            // association.py:343-350 (sigma is only needed for a clamped particle)
            const bool keep = !(clamped && sigmoid((double)sc.opacity_logits[g]) < kMinClampedOpacity);
            if (clamped) fl |= 2;
            if (keep) {
                fl |= 1;
                if (clamped) {  // association.py:430-433: every tile
                    ar.x[0] = (uint32_t)fc.n_x << 16;
                    ar.y[0] = (uint32_t)fc.n_y << 16;
                    n_ent = (int64_t)fc.n_x * fc.n_y;
                } else {
                    const int cx = axis_tiles(t00, t02, t22, rt0, rt1, sex, fc.n_x + 1, ar.x, bx.x, bx.y);
                    const int cy = axis_tiles(t11, t12, t22, rp0, rp1, sey, fc.n_y + 1, ar.y, bx.z, bx.w);
                    n_ent = (int64_t)cx * cy;
                }
            }
        }
    }
    count = n_ent;
    ranges[g] = ar;
    cr.box = bx;  // (the visual-cone part of the record is written by the payload half)
    // association.py:335-340 key bits (depth > 0): f32 bits | 0x80000000; non-emitting last
    const uint32_t kb = __float_as_uint((float)depth) | 0x80000000u;
    // (exhaustive mode: every kept Gaussian takes part, whatever its tile set)
    depth_key[g] = (fc.exhaustive ? (fl & 1) != 0 : n_ent > 0) ? kb : 0xFFFFFFFFu;
    return fl;
}

// K1b: raster payload of one Gaussian (renderer.py:57-81): W, o_u, the fp64 quadratic forms, SH colour.
// Only the pixel-side arithmetic of the raster depends on these values (not the association), so
// reciprocals replace divisions here.  NB = SH band count (compile-time: static register arrays).
// Runs on a group of 128 threads (lt = 0..127) that synchronises with named barrier 2; ssh: SH
// staging, then payload staging (9 float4 = 36 floats per Gaussian, padded rows).  Returns the
// SH clamp gate flag bits (3-5) of Gaussian g0 + lt.
constexpr int kPayHead = offsetof(Payload, cull) / 16;    // float4s of a payload before its culling record
constexpr int kPayRow = sizeof(Payload) / 16;             // float4s of a payload
constexpr int kStageRow = kPayHead + 1;                   // padded staging row

template <int NB>
__device__ uint8_t payload_block(const FrameConst &fc, const geer_scene &sc, float *ssh, Cull *scull, int64_t g0,
                                 int cnt_b, int lt) {
    const int nthr = 128;
    {
        // stage this block's SH coefficients (contiguous) with coalesced loads
        const float *src = sc.sh + g0 * NB * 3;
        const int total = cnt_b * NB * 3;
        if ((((uintptr_t)src) & 15) == 0 && (total & 3) == 0) {
            const float4 *s4 = reinterpret_cast<const float4 *>(src);
            float4 *d4 = reinterpret_cast<float4 *>(ssh);
            for (int i = lt; i < total / 4; i += nthr) d4[i] = __ldg(s4 + i);
        } else {
            for (int i = lt; i < total; i += nthr) ssh[i] = __ldg(src + i);
        }
    }
    named_barrier(2, 128);
    const bool live = lt < cnt_b;  // threads past the end compute a copy of row 0 (not stored)
    const int64_t g = g0 + (live ? lt : 0);
    const double mean[3] = {sc.means[g * 3 + 0], sc.means[g * 3 + 1], sc.means[g * 3 + 2]};
    const float4 q4v = *reinterpret_cast<const float4 *>(sc.quats + g * 4);
    const float q4[4] = {q4v.x, q4v.y, q4v.z, q4v.w};
    double rot[9], s[3], is[3];
    quat_rot(q4, rot);
    for (int i = 0; i < 3; ++i) {
        s[i] = exp((double)sc.log_scales[g * 3 + i]);
        is[i] = exp(-(double)sc.log_scales[g * 3 + i]);
    }
    // renderer.py:78-79: W = S^-1 R^T, o_u = W (o - mean)
    double W[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) W[i * 3 + j] = rot[j * 3 + i] * is[i];
    const double rel[3] = {fc.origin[0] - mean[0], fc.origin[1] - mean[1], fc.origin[2] - mean[2]};
    double ou[3];
    for (int i = 0; i < 3; ++i) ou[i] = W[i * 3 + 0] * rel[0] + W[i * 3 + 1] * rel[1] + W[i * 3 + 2] * rel[2];
    const double sigma = sigmoid((double)sc.opacity_logits[g]);
    // renderer.py:57-70 sh_colors (view direction from the optical centre, stop-gradient)
    const double vd[3] = {-rel[0], -rel[1], -rel[2]};
    double vn = sqrt(vd[0] * vd[0] + vd[1] * vd[1] + vd[2] * vd[2]);
    const double ivn = 1.0 / (vn > 1e-12 ? vn : 1e-12);
    const double ux = vd[0] * ivn, uy = vd[1] * ivn, uz = vd[2] * ivn;
    const float *shg = ssh + (live ? lt : 0) * NB * 3;
    double rgb[3];
    uint8_t gate = 0;
    // (band-outer order: each basis value dies after use; per channel the sum is still sequential in b)
    double pre[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const double basis_b = sh_term(b, ux, uy, uz);
#pragma unroll
        for (int c = 0; c < 3; ++c) pre[c] += basis_b * (double)shg[b * 3 + c];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        pre[c] += 0.5;
        if (pre[c] > 0) gate |= (uint8_t)(1u << c);
        rgb[c] = pre[c] > 0.0 ? pre[c] : 0.0;
    }
    // raster culling: the visual cone of the lam-ellipsoid (camera frame, full line).  With
    // P = Sigma_c^-1 = (W R_c^T)^T (W R_c^T), nu = P mu_c, a = mu_c^T nu - lam^2 > 0 (camera outside):
    // kappa(d) <= lam^2 <=> d^T K d >= 0, K = nu nu^T - a P, stored divided by nu^T nu (then
    // lambda_max(K) <= 1).  k1.z is the lambda_max bound (inf: never culled, e.g. camera inside).
    {
        double Wc[9], P[9], mc[3], nu[3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                Wc[i * 3 + j] = W[i * 3 + 0] * fc.R[j * 3 + 0] + W[i * 3 + 1] * fc.R[j * 3 + 1] + W[i * 3 + 2] * fc.R[j * 3 + 2];
        for (int i = 0; i < 3; ++i)
            for (int j = i; j < 3; ++j)
                P[i * 3 + j] = P[j * 3 + i] = Wc[0 * 3 + i] * Wc[0 * 3 + j] + Wc[1 * 3 + i] * Wc[1 * 3 + j] + Wc[2 * 3 + i] * Wc[2 * 3 + j];
        for (int i = 0; i < 3; ++i)
            mc[i] = fc.R[i * 3 + 0] * mean[0] + fc.R[i * 3 + 1] * mean[1] + fc.R[i * 3 + 2] * mean[2] + fc.t[i];
        for (int i = 0; i < 3; ++i) nu[i] = P[i * 3 + 0] * mc[0] + P[i * 3 + 1] * mc[1] + P[i * 3 + 2] * mc[2];
        const double a = mc[0] * nu[0] + mc[1] * nu[1] + mc[2] * nu[2] - fc.lam * fc.lam;
        const double nn = nu[0] * nu[0] + nu[1] * nu[1] + nu[2] * nu[2];
        Cull &cr = scull[lt];
        cr.k0 = make_float4(0.f, 0.f, 0.f, 0.f);
        cr.k1 = make_float4(0.f, 0.f, INFINITY, 0.f);
        if (a > 0.0 && nn > 0.0) {
            const double in = 1.0 / nn;
            auto K = [&](int i, int j) { return (float)((nu[i] * nu[j] - a * P[i * 3 + j]) * in); };
            cr.k0 = make_float4(K(0, 0), K(1, 1), K(2, 2), K(0, 1));
            cr.k1 = make_float4(K(0, 2), K(1, 2), 1.0f, 0.f);
        }
    }
    const double smax = fmax(s[0], fmax(s[1], s[2])), smin = fmin(s[0], fmin(s[1], s[2]));
    Payload pl;
    make_payload(W, ou, rgb, sigma, smax / smin, fc.lam, pl);
    // flags: bit0 keep, bit1 clamped (K1a), bits3-5 SH clamp gate per channel
    const uint8_t bits = (uint8_t)(gate << 3);
    // stage the block's payloads (first 8 float4; the culling record comes from the association
    // half) in shared memory, reusing the SH buffer: k_preprocess writes them out as contiguous
    // float4 runs.  Rows padded to 9 float4: conflict-free 16-B stores.
    float4 *sp = reinterpret_cast<float4 *>(ssh);
    named_barrier(2, 128);  // every thread is done reading its SH coefficients
    const float4 *plv = reinterpret_cast<const float4 *>(&pl);
#pragma unroll
    for (int k = 0; k < kPayHead; ++k) sp[lt * kStageRow + k] = plv[k];
    return bits;
}

// K1: one block = 128 Gaussians; threads 0-127 run the exact fp64 association, threads 128-255 the
// raster payload of the same Gaussians (the first is fp64-issue-bound, the second latency-bound,
// so co-resident they overlap), then the flag bits of both are merged.
#ifndef K1_MIN_BLOCKS
#define K1_MIN_BLOCKS 4
#endif
template <int NB>
__global__ void __launch_bounds__(256, K1_MIN_BLOCKS)
    k_preprocess(FrameConst fc, geer_scene sc, const double *__restrict__ medges_x, const double *__restrict__ medges_y,
                 Payload *__restrict__ payload, uint32_t *__restrict__ depth_key,
                 AxisRanges *__restrict__ ranges, uint8_t *__restrict__ flags,
                 double *__restrict__ mu_out, double *__restrict__ depth_out, int *__restrict__ err,
                 unsigned long long *__restrict__ total_entries) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int kStageFloats = kStageRow * 4;  // payload-head staging
    __shared__ __align__(16) float ssh[128 * (NB * 3 > kStageFloats ? NB * 3 : kStageFloats)];
    __shared__ Cull scull[128];
    const int64_t g0 = (int64_t)blockIdx.x * 128;
    const int cnt_b = (int)lmin(128, sc.n - g0);
    const int lt = threadIdx.x & 127;
    // The two halves never meet at a block barrier (their run times differ per Gaussian, and the
    // faster half would idle): each writes its own flag byte and its own part of the payload rows.
    if (threadIdx.x < 128) {
        double *sex = reinterpret_cast<double *>(smem_raw);
        double *sey = sex + (fc.n_x + 1);
        for (int i = lt; i <= fc.n_x; i += 128) sex[i] = medges_x[i];
        for (int i = lt; i <= fc.n_y; i += 128) sey[i] = medges_y[i];
        named_barrier(1, 128);
        int64_t ne = 0;
        unsigned long long rows = 0;
        if (lt < cnt_b) {
            const int64_t g = g0 + lt;
            Cull cl;
            cl.box = make_float4(0.f, 0.f, 0.f, 0.f);
            flags[g] = associate_one(fc, sc, sex, sey, g, depth_key, ne, ranges, cl, mu_out, depth_out, err);
            payload[g].cull.box = cl.box;  // (the visual-cone part is the payload half's)
            if (ne > 0) {
                const AxisRanges &a = ranges[g];
                for (int k = 0; k < 3; ++k) rows += (a.y[k] >> 16) - (a.y[k] & 0xFFFFu);
            }
        }
        // the warp's entries and (Gaussian, tile row) pairs, for the frame totals
        unsigned long long t = (unsigned long long)ne;
        for (int o = 16; o > 0; o >>= 1) {
            t += __shfl_xor_sync(0xffffffffu, t, o);
            rows += __shfl_xor_sync(0xffffffffu, rows, o);
        }
        if ((lt & 31) == 0 && t) atomicAdd(total_entries, t);
        if ((lt & 31) == 0 && rows) atomicAdd(total_entries + 1, rows);  // (the next counter)
    } else {
        const uint8_t bits = payload_block<NB>(fc, sc, ssh, scull, g0, cnt_b, lt);
        if (lt < cnt_b) flags[sc.n + g0 + lt] = bits;
        named_barrier(2, 128);  // the half's staged rows are complete
        // coalesced write-out of the block's payload heads and visual-cone records
        const float4 *sp = reinterpret_cast<const float4 *>(ssh);
        const float4 *scv = reinterpret_cast<const float4 *>(scull);
        float4 *dp = reinterpret_cast<float4 *>(payload + g0);
        constexpr int kBox = kPayHead + (int)(offsetof(Cull, box) / 16);
        for (int i = lt; i < cnt_b * kPayRow; i += 128) {
            const int r = i / kPayRow, k = i - r * kPayRow;
            if (k == kBox) continue;  // the association half's
            dp[i] = k < kPayHead ? sp[r * kStageRow + k] : scv[r * (sizeof(Cull) / 16) + (k - kPayHead)];
        }
    }
}

// ---------------------------------------------------------------- K7

// Coalesced block store of per-Gaussian rows: thread i holds row i (width values) of this block's
// cnt rows; rows go through shared memory so the global stores are contiguous (the SoA gradient
// arrays have 1..48 values per Gaussian, which would otherwise be strided partial-sector writes).
template <typename T, int W>
__device__ __forceinline__ void store_rows(float *sm, const float (&v)[W], int cnt, T *dst, bool acc) {
    __syncthreads();  // previous round's readers are done
#pragma unroll
    for (int k = 0; k < W; ++k) sm[threadIdx.x * (W | 1) + k] = v[k];  // odd stride: no bank conflicts
    __syncthreads();
    for (int i = threadIdx.x; i < cnt * W; i += blockDim.x) {
        const float x = sm[(i / W) * (W | 1) + i % W];
        dst[i] = acc ? (T)((double)dst[i] + (double)x) : (T)x;
    }
}

// accum layout per Gaussian (16 f32): dW_rc (9, row-major), sum dl/do_u (3), sum dsigma, sum dcol (3).
// fp32 arithmetic (the accumulators are fp32 already); renderer.py:304-307, 204-231, 332.
template <typename T, int NB>
__global__ void __launch_bounds__(128) k_finalize(FrameConst fc, geer_scene sc, const float4 *__restrict__ accum,
                                                  const uint8_t *__restrict__ flags, T *dmeans, T *dlog_scales,
                                                  T *dquats, T *dopac, T *dsh, int accumulate) {
    __shared__ float sm[128 * ((NB * 3 | 1) > 5 ? (NB * 3 | 1) : 5)];  // widest row: max(NB * 3, 4), odd stride
    const int64_t g0 = (int64_t)blockIdx.x * blockDim.x;
    const int cnt = (int)lmin((int64_t)blockDim.x, sc.n - g0);
    const int64_t g = g0 + (threadIdx.x < cnt ? threadIdx.x : 0);
    float a[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float4 v = accum[g * 4 + i];
        a[i * 4 + 0] = v.x;
        a[i * 4 + 1] = v.y;
        a[i * 4 + 2] = v.z;
        a[i * 4 + 3] = v.w;
    }
    const float mean[3] = {sc.means[g * 3 + 0], sc.means[g * 3 + 1], sc.means[g * 3 + 2]};
    const float4 q4v = *reinterpret_cast<const float4 *>(sc.quats + g * 4);
    const float q0 = q4v.x, q1 = q4v.y, q2 = q4v.z, q3 = q4v.w;
    const float qn = sqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    const float iqn = 1.0f / qn;
    const float r = q0 * iqn, i = q1 * iqn, j = q2 * iqn, k = q3 * iqn;
    const float rot[9] = {1 - 2 * (j * j + k * k), 2 * (i * j - r * k), 2 * (i * k + r * j),
                          2 * (i * j + r * k), 1 - 2 * (i * i + k * k), 2 * (j * k - r * i),
                          2 * (i * k - r * j), 2 * (j * k + r * i), 1 - 2 * (i * i + j * j)};
    float is[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) is[c] = __expf(-sc.log_scales[g * 3 + c]);
    const float rel[3] = {(float)fc.origin[0] - mean[0], (float)fc.origin[1] - mean[1], (float)fc.origin[2] - mean[2]};
    const float dos[3] = {a[9], a[10], a[11]};
    // renderer.py:304-307: dW = dW_rc + (sum dl/do) (o - mu)^T ; dmu = -W^T sum dl/do, W[i][j] = rot[j][i] / s_i
    float dw[9];
#pragma unroll
    for (int x = 0; x < 3; ++x)
#pragma unroll
        for (int y = 0; y < 3; ++y) dw[x * 3 + y] = fmaf(dos[x], rel[y], a[x * 3 + y]);
    float dmu[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
        dmu[c] = -(rot[c * 3 + 0] * is[0] * dos[0] + rot[c * 3 + 1] * is[1] * dos[1] + rot[c * 3 + 2] * is[2] * dos[2]);
    // renderer.py:208-209: dlog_s_k = -(sum_j dW[k][j] R[j][k]) / s_k
    float dls[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
        dls[c] = -(dw[c * 3 + 0] * rot[0 * 3 + c] + dw[c * 3 + 1] * rot[1 * 3 + c] + dw[c * 3 + 2] * rot[2 * 3 + c]) * is[c];
    // renderer.py:211-230: dq_raw_m = sum_ab dW[a][b] 2 D_m[a][b] / s_a, then the normalisation Jacobian
    float e[9];
#pragma unroll
    for (int x = 0; x < 3; ++x)
#pragma unroll
        for (int y = 0; y < 3; ++y) e[x * 3 + y] = 2.0f * dw[x * 3 + y] * is[x];
    const float dqr0 = e[1] * k - e[2] * j - e[3] * k + e[5] * i + e[6] * j - e[7] * i;
    const float dqr1 = e[1] * j + e[2] * k + e[3] * j - 2 * i * e[4] + e[5] * r + e[6] * k - e[7] * r - 2 * i * e[8];
    const float dqr2 = -2 * j * e[0] + e[1] * i - e[2] * r + e[3] * i + e[5] * k + e[6] * r + e[7] * k - 2 * j * e[8];
    const float dqr3 = -2 * k * e[0] + e[1] * r + e[2] * i - e[3] * r - 2 * k * e[4] + e[5] * j + e[6] * i + e[7] * j;
    const float dot = dqr0 * r + dqr1 * i + dqr2 * j + dqr3 * k;
    // renderer.py:332 dsh = basis (x) (dcol * gate), view direction stop-gradient
    const float vx = -rel[0], vy = -rel[1], vz = -rel[2];
    const float ivn = 1.0f / fmaxf(sqrtf(vx * vx + vy * vy + vz * vz), 1e-12f);
    double basis[16];
    sh_basis((double)(vx * ivn), (double)(vy * ivn), (double)(vz * ivn), basis);
    const uint8_t gate = flags[g] >> 3;
    float dcol[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) dcol[c] = ((gate >> c) & 1) ? a[13 + c] : 0.0f;
    float dsig = a[12];
    if (accumulate & GEER_OPACITY_LOGIT) {  // trainer.py:208-217 stored_grads: chain through the logit
        const float sg = 1.0f / (1.0f + __expf(-sc.opacity_logits[g]));
        dsig = dsig * sg * (1.0f - sg);
    }
    const bool acc = accumulate & GEER_ACCUMULATE;
    const float dq[4] = {(dqr0 - dot * r) * iqn, (dqr1 - dot * i) * iqn, (dqr2 - dot * j) * iqn, (dqr3 - dot * k) * iqn};
    const float dop[1] = {dsig};
    float dshv[NB * 3];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) dshv[b * 3 + c] = (float)basis[b] * dcol[c];
    store_rows<T, 3>(sm, dmu, cnt, dmeans + g0 * 3, acc);
    store_rows<T, 3>(sm, dls, cnt, dlog_scales + g0 * 3, acc);
    store_rows<T, 4>(sm, dq, cnt, dquats + g0 * 4, acc);
    store_rows<T, 1>(sm, dop, cnt, dopac + g0, acc);
    store_rows<T, NB * 3>(sm, dshv, cnt, dsh + g0 * NB * 3, acc);
}

// ---------------------------------------------------------------- launchers

void launch_beap_setup(const FrameConst &fc, double2 *col_sc, double2 *row_sc, double *medges_x, double *medges_y,
                       int32_t *tile_off, int32_t *pix_list, int32_t *pixel_tile, cudaStream_t st) {
    int n = max(max(fc.width, fc.height), max(fc.n_x, fc.n_y) + 1);
    k_beap_tables<<<(n + 255) / 256, 256, 0, st>>>(fc, col_sc, row_sc, medges_x, medges_y);
    k_beap_csr<<<fc.n_tiles, 256, 0, st>>>(fc, tile_off, pix_list, pixel_tile);
}

void launch_cam_pixels(const FrameConst &fc, double *dir64, double *theta, double *phi, long long *minmax,
                       cudaStream_t st) {
    int64_t npx = (int64_t)fc.width * fc.height;
    int blocks = (int)lmin((npx + 255) / 256, 148 * 16);
    k_cam_pixels<<<blocks, 256, 0, st>>>(fc, dir64, theta, phi, minmax);
}

void launch_cam_edges(const FrameConst &fc, const long long *minmax, double *edges_x, double *edges_y,
                      double *medges_x, double *medges_y, cudaStream_t st) {
    k_cam_edges<<<1, 256, 0, st>>>(fc, minmax, edges_x, edges_y, medges_x, medges_y);
}

void launch_cam_bin(const FrameConst &fc, const double *theta, const double *phi, const double *edges_x,
                    const double *edges_y, int32_t *pixel_tile, int32_t *tile_count, cudaStream_t st) {
    int64_t npx = (int64_t)fc.width * fc.height;
    int blocks = (int)lmin((npx + 255) / 256, 148 * 16);
    k_cam_bin<<<blocks, 256, 0, st>>>(fc, theta, phi, edges_x, edges_y, pixel_tile, tile_count);
}

void launch_iota(int32_t *v, int64_t n, cudaStream_t st) {
    int blocks = (int)lmin((n + 255) / 256, 148 * 16);
    if (blocks > 0) k_iota<<<blocks, 256, 0, st>>>(v, n);
}

void launch_items(int n_tiles, const int32_t *tile_off, int32_t *item_count, cudaStream_t st) {
    k_item_counts<<<(n_tiles + 255) / 256, 256, 0, st>>>(n_tiles, tile_off, item_count);
}
void launch_item_fill(int n_tiles, const int32_t *tile_off, const int32_t *item_off, int4 *items, int32_t *n_items,
                      cudaStream_t st) {
    k_item_fill<<<(n_tiles + 255) / 256, 256, 0, st>>>(n_tiles, tile_off, item_off, items, n_items);
}

size_t preprocess_smem(const FrameConst &fc) { return sizeof(double) * (fc.n_x + fc.n_y + 2); }

void launch_preprocess(const FrameConst &fc, const geer_scene &sc, const double *medges_x, const double *medges_y,
                       Payload *payload, uint32_t *depth_key, AxisRanges *ranges,
                       uint8_t *flags, double *mu_out, double *depth_out, int *err,
                       unsigned long long *total_entries, cudaStream_t st) {
    if (sc.n == 0) return;
    const int blocks = (int)((sc.n + 127) / 128);
    switch (sc.n_bands) {
#define GEER_NB_CASE(NB)                                                                                            \
    case NB:                                                                                                        \
        k_preprocess<NB><<<blocks, 256, preprocess_smem(fc), st>>>(fc, sc, medges_x, medges_y, payload,             \
                                                                   depth_key, ranges, flags,                       \
                                                                   mu_out, depth_out, err, total_entries);         \
        break;
        GEER_NB_CASE(1) GEER_NB_CASE(2) GEER_NB_CASE(3) GEER_NB_CASE(4) GEER_NB_CASE(5) GEER_NB_CASE(6)
        GEER_NB_CASE(7) GEER_NB_CASE(8) GEER_NB_CASE(9) GEER_NB_CASE(10) GEER_NB_CASE(11) GEER_NB_CASE(12)
        GEER_NB_CASE(13) GEER_NB_CASE(14) GEER_NB_CASE(15) GEER_NB_CASE(16)
#undef GEER_NB_CASE
        default: break;
    }
}

template <typename T>
void launch_finalize(const FrameConst &fc, const geer_scene &sc, const float4 *accum, const uint8_t *flags, T *dmeans,
                     T *dlog_scales, T *dquats, T *dopac, T *dsh, int accumulate, cudaStream_t st) {
    if (sc.n == 0) return;
    const int blocks = (int)((sc.n + 127) / 128);
    switch (sc.n_bands) {
#define GEER_NB_CASE(NB)                                                                                           \
    case NB:                                                                                                       \
        k_finalize<T, NB><<<blocks, 128, 0, st>>>(fc, sc, accum, flags, dmeans, dlog_scales, dquats, dopac, dsh, \
                                                  accumulate);                                                     \
        break;
        GEER_NB_CASE(1) GEER_NB_CASE(2) GEER_NB_CASE(3) GEER_NB_CASE(4) GEER_NB_CASE(5) GEER_NB_CASE(6)
        GEER_NB_CASE(7) GEER_NB_CASE(8) GEER_NB_CASE(9) GEER_NB_CASE(10) GEER_NB_CASE(11) GEER_NB_CASE(12)
        GEER_NB_CASE(13) GEER_NB_CASE(14) GEER_NB_CASE(15) GEER_NB_CASE(16)
#undef GEER_NB_CASE
        default: break;
    }
}
template void launch_finalize<float>(const FrameConst &, const geer_scene &, const float4 *, const uint8_t *, float *,
                                     float *, float *, float *, float *, int, cudaStream_t);
template void launch_finalize<double>(const FrameConst &, const geer_scene &, const float4 *, const uint8_t *,
                                      double *, double *, double *, double *, double *, int, cudaStream_t);

}  // namespace geer
