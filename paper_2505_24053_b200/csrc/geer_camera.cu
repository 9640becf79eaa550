// geer_camera.cu — ground-truth resampling onto the equiangular (BEAP) grid:
// restates raygauss camera.resample_to_beap (camera.py:302-339) with project_pinhole (:197-210),
// project_kb (:227-246), beap_ray_grid / angles_to_dir (:119-155,183-190) and _bilinear (:289-299).
//
// One thread per target pixel: the BEAP ray (fp64, the reference's operation order), its projection
// into the source camera (fp64: the inside/mask decision is a comparison against the image border),
// then the bilinear tap of the fp32 source image.  HBM-bound: 12 B read (x4 taps, mostly cached) and
// 13 B written per pixel.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "geer.h"

namespace {

struct ResampleParams {
    int tw, th, sw, sh, model;
    double fov_x, fov_y;        // target (beap)
    double fx, fy, cx, cy, k[4];  // source (pinhole / kb)
};

__global__ void k_resample(ResampleParams P, const float *__restrict__ src, float *__restrict__ color,
                           uint8_t *__restrict__ mask) {
    const int64_t n = (int64_t)P.tw * P.th;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(i % P.tw), y = (int)(i / P.tw);
        // camera.py:126-127 beap_angles, :141-155 angles_to_dir
        const double theta = ((x + 0.5) - (P.tw + 1) / 2.0) * P.fov_x / P.tw;
        const double phi = ((y + 0.5) - (P.th + 1) / 2.0) * P.fov_y / P.th;
        const double st = sin(theta), ct = cos(theta), sp = sin(phi), cp = cos(phi);
        const double dx0 = st * cp, dy0 = ct * sp, dz0 = ct * cp;
        const double nn = sqrt(dx0 * dx0 + dy0 * dy0 + dz0 * dz0);
        const double dx = dx0 / nn, dy = dy0 / nn, dz = dz0 / nn;
        double xp, yp;
        bool valid;
        if (P.model == GEER_PINHOLE) {  // camera.py:197-210
            valid = dz > 0;
            xp = P.fx * dx / dz + P.cx;
            yp = P.fy * dy / dz + P.cy;
        } else {  // camera.py:227-246
            const double r = sqrt(dx * dx + dy * dy);
            const double alpha = atan2(r, dz);
            const double a2 = alpha * alpha;
            const double ad = alpha * (1.0 + a2 * (P.k[0] + a2 * (P.k[1] + a2 * (P.k[2] + a2 * P.k[3]))));
            const double factor = r > 1e-12 ? ad / fmax(r, 1e-300) : 1.0;
            xp = P.fx * factor * dx + P.cx;
            yp = P.fy * factor * dy + P.cy;
            valid = alpha < M_PI;
        }
        // camera.py:331-338: inside the source image, else masked and zero
        const bool inside = valid && xp >= 0.0 && xp <= P.sw - 1 && yp >= 0.0 && yp <= P.sh - 1;
        float c[3] = {0.f, 0.f, 0.f};
        if (inside) {  // camera.py:289-299 _bilinear (x0, y0 clipped to w - 2, h - 2)
            int x0 = (int)floor(xp), y0 = (int)floor(yp);
            x0 = min(max(x0, 0), P.sw - 2);
            y0 = min(max(y0, 0), P.sh - 2);
            const double fx = xp - x0, fy = yp - y0;
            const float *r0 = src + ((int64_t)y0 * P.sw + x0) * 3, *r1 = r0 + (int64_t)P.sw * 3;
            for (int ch = 0; ch < 3; ++ch)
                c[ch] = (float)(r0[ch] * (1 - fx) * (1 - fy) + r0[3 + ch] * fx * (1 - fy) + r1[ch] * (1 - fx) * fy +
                                r1[3 + ch] * fx * fy);
        }
        color[i * 3 + 0] = c[0];
        color[i * 3 + 1] = c[1];
        color[i * 3 + 2] = c[2];
        mask[i] = inside ? 1 : 0;
    }
}

}  // namespace

extern "C" int geer_resample_to_beap(const float *source, int source_height, int source_width,
                                     const geer_camera *source_camera, const geer_camera *target_camera,
                                     float *color, uint8_t *mask, void *stream) {
    if (!source || !source_camera || !target_camera || !color || !mask) return GEER_ERR_INVALID;
    if (target_camera->model != GEER_BEAP) return GEER_ERR_INVALID;
    if (source_camera->model != GEER_PINHOLE && source_camera->model != GEER_KB) return GEER_ERR_INVALID;
    if (source_height < 2 || source_width < 2 || target_camera->width <= 0 || target_camera->height <= 0)
        return GEER_ERR_INVALID;
    ResampleParams P;
    P.tw = target_camera->width;
    P.th = target_camera->height;
    P.sw = source_width;
    P.sh = source_height;
    P.model = source_camera->model;
    P.fov_x = target_camera->fov_x;
    P.fov_y = target_camera->fov_y;
    P.fx = source_camera->fx;
    P.fy = source_camera->fy;
    P.cx = source_camera->cx;
    P.cy = source_camera->cy;
    for (int i = 0; i < 4; ++i) P.k[i] = source_camera->k[i];
    const int64_t n = (int64_t)P.tw * P.th;
    int blocks = (int)((n + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_resample<<<blocks, 256, 0, (cudaStream_t)stream>>>(P, source, color, mask);
    return cudaGetLastError() == cudaSuccess ? GEER_OK : GEER_ERR_CUDA;
}

// ---------------------------------------------------------------- PLY vertex block -> device SoA
// (ply.py:94-137 without the float64 detour): record v holds n_props float32; column cols[k] of it
// goes to SoA value k (means 3, log_scales 3, quats 4, opacity 1, sh band-major).  One thread per value.
namespace {
struct ColMap {
    int c[64];
};
__global__ void k_ply_to_soa(const float *__restrict__ block, int64_t n, int n_props, ColMap cm, int n_vals,
                             float *__restrict__ soa) {
    const int64_t total = n * n_vals;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / n_vals;
        const int k = (int)(i - v * n_vals);
        const float x = block[v * n_props + cm.c[k]];
        // SoA groups: [0,3) means, [3,6) log_scales, [6,10) quats, [10,11) opacity, [11, n_vals) sh
        int64_t dst;
        if (k < 3) dst = v * 3 + k;
        else if (k < 6) dst = 3 * n + v * 3 + (k - 3);
        else if (k < 10) dst = 6 * n + v * 4 + (k - 6);
        else if (k < 11) dst = 10 * n + v;
        else dst = 11 * n + v * (n_vals - 11) + (k - 11);
        soa[dst] = x;
    }
}
}  // namespace

extern "C" int geer_ply_to_soa(const float *block, int64_t n, int n_props, const int32_t *cols, int n_vals, float *soa,
                               void *stream) {
    if (!block || !cols || !soa || n < 0 || n_vals < 11 || n_vals > 64 || n_props <= 0) return GEER_ERR_INVALID;
    ColMap cm;
    for (int k = 0; k < n_vals; ++k) {
        if (cols[k] < 0 || cols[k] >= n_props) return GEER_ERR_INVALID;
        cm.c[k] = cols[k];
    }
    if (n == 0) return GEER_OK;
    const int64_t total = n * n_vals;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 32) blocks = 148 * 32;
    k_ply_to_soa<<<blocks, 256, 0, (cudaStream_t)stream>>>(block, n, n_props, cm, n_vals, soa);
    return cudaGetLastError() == cudaSuccess ? GEER_OK : GEER_ERR_CUDA;
}
