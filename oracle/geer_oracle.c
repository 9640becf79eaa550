/*
 * geer_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64 restatement of the reference 3DGEER rendering hot path
 * (raygauss 0.1.0, /root/reference/pkg/src/raygauss).  It exists so the
 * CUDA product can be checked against the reference algorithm on machines
 * where the (pure-Python) reference is not installed, and so bench.py can
 * time a CPU baseline ("port").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path (paper_2505_24053_b200) never links, imports or calls this file.
 *
 * Parity pinning: the tests/golden fixtures are produced by running the unmodified
 * reference (tests/golden/make_golden.py); tests/test_oracle_golden.py checks
 * this restatement against them (association bit-exact, floats ~1e-12).
 *
 * Built with -ffp-contract=off so every expression rounds exactly like the
 * numpy expression it restates (no fused multiply-adds).
 *
 * Citations: association.py, renderer.py, camera.py, scene.py, core.py refer
 * to /root/reference/pkg/src/raygauss/<file>.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GEO_PINHOLE 0
#define GEO_KB 1
#define GEO_BEAP 2

/* core.py:27-31, association.py:36-39 */
static const double MAX_BLEND_T = 0.999;
static const double MIN_REMAINING = 1e-4;
static const double NEAR_LIMIT = 0.01;
static const double MIN_CLAMPED_OPACITY = 0.05;

/* core.py:34-51 */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154,  -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

typedef struct geo_camera {
    int32_t width, height, model, pad_;
    double rotation[9];   /* R_c, row-major, x_c = R_c x + t_c (camera.py:25-48) */
    double translation[3];
    double fov_x, fov_y, fx, fy, cx, cy;
    double k[4];
} geo_camera;

typedef struct geo_config {
    double lam;
    double background[3];
    int32_t tile_px;
    int32_t support_cutoff;
    int32_t threads;
    int32_t pad_;
} geo_config;

static void set_err(char *err, int errlen, const char *msg) {
    if (err && errlen > 0) {
        strncpy(err, msg, (size_t)errlen - 1);
        err[errlen - 1] = 0;
    }
}

void geo_free(void *p) { free(p); }

/* numpy's matmul (OpenBLAS / its FMA inner loop) accumulates a length-3 dot
 * product as fma(a2, b2, fma(a1, b1, a0 * b0)); verified bit-exact against the
 * reference's `means @ R.T`, `m @ m.T`, `-R.T @ t` and `dirs @ R`.  einsum
 * reductions, by contrast, are plain sequential sums (no fma). */
static inline double mm3(double a0, double b0, double a1, double b1, double a2, double b2) {
    return fma(a2, b2, fma(a1, b1, a0 * b0));
}

/* ------------------------------------------------------------------ camera */

/* camera.py:141-155 angles_to_dir */
static void angles_to_dir(double theta, double phi, double out[3]) {
    double st = sin(theta), ct = cos(theta), sp = sin(phi), cp = cos(phi);
    double x = st * cp, y = ct * sp, z = ct * cp;
    double n = sqrt(x * x + y * y + z * z);
    out[0] = x / n;
    out[1] = y / n;
    out[2] = z / n;
}

/* camera.py:119-128 beap_angles (pixel centre) */
static double beap_angle(int idx, int n, double fov) {
    return ((idx + 0.5) - (n + 1) / 2.0) * fov / n;
}

/* camera.py:131-138 beap_pixel_edges */
static double beap_edge(int idx, int n, double fov) { return (idx - (n + 1) / 2.0) * fov / n; }

/* camera.py:272-282 pixel_ray_grid: camera-space unit direction of pixel (x, y) */
static void pixel_dir_cam(const geo_camera *cam, int x, int y, double out[3]) {
    if (cam->model == GEO_BEAP) {
        angles_to_dir(beap_angle(x, cam->width, cam->fov_x), beap_angle(y, cam->height, cam->fov_y), out);
        return;
    }
    double u = ((double)x - cam->cx) / cam->fx;
    double v = ((double)y - cam->cy) / cam->fy;
    if (cam->model == GEO_PINHOLE) { /* camera.py:213-219 */
        double n = sqrt(u * u + v * v + 1.0 * 1.0);
        out[0] = u / n;
        out[1] = v / n;
        out[2] = 1.0 / n;
        return;
    }
    /* camera.py:249-269 unproject_kb, 20 Newton iterations */
    const double *k = cam->k;
    double alpha_d = sqrt(u * u + v * v);
    double alpha = alpha_d;
    for (int it = 0; it < 20; ++it) {
        double a2 = alpha * alpha;
        double f = alpha * (1.0 + a2 * (k[0] + a2 * (k[1] + a2 * (k[2] + a2 * k[3])))) - alpha_d;
        double df = 1.0 + a2 * (3 * k[0] + a2 * (5 * k[1] + a2 * (7 * k[2] + a2 * 9 * k[3])));
        alpha = alpha - f / df;
    }
    double scale = alpha_d > 1e-12 ? sin(alpha) / (alpha_d > 1e-300 ? alpha_d : 1e-300) : 1.0;
    double dx = u * scale, dy = v * scale, dz = cos(alpha);
    double n = sqrt(dx * dx + dy * dy + dz * dz);
    out[0] = dx / n;
    out[1] = dy / n;
    out[2] = dz / n;
}

/* camera.py:158-172 dir_to_angles */
static void dir_to_angles(const double d[3], double *theta, double *phi) {
    double x = d[0], y = d[1], z = d[2];
    *theta = atan2(x, z);
    if (z == 0.0) {
        *phi = (y == 0.0) ? 0.0 : (y > 0 ? M_PI / 2 : -M_PI / 2);
    } else if (z > 0) {
        *phi = atan2(y, z);
    } else {
        *phi = atan(y / z);
    }
}

/* association.py:91-105 mirror_from_angle (xi = 1) */
static double mirror_from_angle(double theta) {
    double denom = cos(theta) + 1.0;
    if (fabs(denom) < 1e-300) return theta >= 0 ? INFINITY : -INFINITY;
    return sin(theta) / denom;
}

/* numpy.linspace(start, stop, num) as restated from numpy 2.3 (endpoint=True) */
static void linspace(double start, double stop, int num, double *out) {
    int div = num - 1;
    double delta = stop - start;
    double step = delta / div;
    for (int i = 0; i < num; ++i) {
        double y = (double)i;
        if (step == 0.0) {
            y = y / div;
            y = y * delta;
        } else {
            y = y * step;
        }
        out[i] = y + start;
    }
    if (num > 1) out[num - 1] = stop;
}

/* count of a[i] <= v (numpy searchsorted side='right') */
static int64_t ss_right(const double *a, int64_t n, double v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (a[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}
/* count of a[i] < v (numpy searchsorted side='left') */
static int64_t ss_left(const double *a, int64_t n, double v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/*
 * association.py:301-332 build_grid + renderer.py:76-77 world directions.
 * dirs_world (H*W*3, may be NULL) = pixel_ray_grid(camera) @ R_c.
 */
int geo_grid(const geo_camera *cam, int tile_px, int n_x, int n_y, double *dirs_world,
             double *medges_x, double *medges_y, int64_t *pixel_tile) {
    const int w = cam->width, h = cam->height;
    const double *R = cam->rotation;
    int64_t npx = (int64_t)w * h;
    double *theta = NULL, *phi = NULL;
    if (cam->model != GEO_BEAP) {
        theta = (double *)malloc(sizeof(double) * npx);
        phi = (double *)malloc(sizeof(double) * npx);
        if (!theta || !phi) { free(theta); free(phi); return 1; }
    }
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < npx; ++p) {
        int x = (int)(p % w), y = (int)(p / w);
        double dc[3];
        pixel_dir_cam(cam, x, y, dc);
        if (dirs_world) {
            for (int j = 0; j < 3; ++j)
                dirs_world[p * 3 + j] = mm3(dc[0], R[0 * 3 + j], dc[1], R[1 * 3 + j], dc[2], R[2 * 3 + j]);
        }
        if (theta) dir_to_angles(dc, &theta[p], &phi[p]);
    }
    double *ex = (double *)malloc(sizeof(double) * (n_x + 1));
    double *ey = (double *)malloc(sizeof(double) * (n_y + 1));
    if (cam->model == GEO_BEAP) {
        for (int i = 0; i <= n_x; ++i) {
            int idx = i * tile_px < w ? i * tile_px : w;
            ex[i] = beap_edge(idx, w, cam->fov_x);
        }
        for (int i = 0; i <= n_y; ++i) {
            int idx = i * tile_px < h ? i * tile_px : h;
            ey[i] = beap_edge(idx, h, cam->fov_y);
        }
        for (int64_t p = 0; p < npx; ++p) {
            int x = (int)(p % w), y = (int)(p / w);
            int col = x / tile_px < n_x - 1 ? x / tile_px : n_x - 1;
            int row = y / tile_px < n_y - 1 ? y / tile_px : n_y - 1;
            pixel_tile[p] = (int64_t)row * n_x + col;
        }
    } else {
        double tmin = INFINITY, tmax = -INFINITY, pmin = INFINITY, pmax = -INFINITY;
        for (int64_t p = 0; p < npx; ++p) {
            if (theta[p] < tmin) tmin = theta[p];
            if (theta[p] > tmax) tmax = theta[p];
            if (phi[p] < pmin) pmin = phi[p];
            if (phi[p] > pmax) pmax = phi[p];
        }
        const double pad = 1e-9;
        linspace(tmin - pad, tmax + pad, n_x + 1, ex);
        linspace(pmin - pad, pmax + pad, n_y + 1, ey);
        for (int64_t p = 0; p < npx; ++p) {
            int64_t c = ss_right(ex, n_x + 1, theta[p]) - 1;
            int64_t r = ss_right(ey, n_y + 1, phi[p]) - 1;
            c = c < 0 ? 0 : (c > n_x - 1 ? n_x - 1 : c);
            r = r < 0 ? 0 : (r > n_y - 1 ? n_y - 1 : r);
            pixel_tile[p] = r * n_x + c;
        }
    }
    for (int i = 0; i <= n_x; ++i) medges_x[i] = mirror_from_angle(ex[i]);
    for (int i = 0; i <= n_y; ++i) medges_y[i] = mirror_from_angle(ey[i]);
    free(ex);
    free(ey);
    free(theta);
    free(phi);
    return 0;
}

/* ------------------------------------------------------------------ scene decoding */

/* scene.py:17-32 quats_to_rotations (renormalised) */
static void quat_rot(const double *q4, double rot[9]) {
    double n = sqrt(q4[0] * q4[0] + q4[1] * q4[1] + q4[2] * q4[2] + q4[3] * q4[3]);
    double r = q4[0] / n, i = q4[1] / n, j = q4[2] / n, k = q4[3] / n;
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

/* core.py:58-67 sigmoid (split-branch form) */
static double sigmoid(double x) {
    if (x >= 0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}

/* scene.py:72-75 W = S^-1 R^T, i.e. W[i][j] = R[j][i] / s_i */
static void whitening(const double *log_s, const double *q4, double W[9], double rot[9], double s[3]) {
    quat_rot(q4, rot);
    for (int i = 0; i < 3; ++i) s[i] = exp(log_s[i]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) W[i * 3 + j] = rot[j * 3 + i] / s[i];
}

/* core.py:289-313 sh_basis, first n_bands entries */
static void sh_basis(const double d[3], int n_bands, double *b) {
    double x = d[0], y = d[1], z = d[2];
    double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    double all[16] = {
        SH_C0,
        -SH_C1 * y,
        SH_C1 * z,
        -SH_C1 * x,
        SH_C2[0] * xy,
        SH_C2[1] * yz,
        SH_C2[2] * (2.0 * zz - xx - yy),
        SH_C2[3] * xz,
        SH_C2[4] * (xx - yy),
        SH_C3[0] * y * (3.0 * xx - yy),
        SH_C3[1] * xy * z,
        SH_C3[2] * y * (4.0 * zz - xx - yy),
        SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy),
        SH_C3[4] * x * (4.0 * zz - xx - yy),
        SH_C3[5] * z * (xx - yy),
        SH_C3[6] * x * (xx - 3.0 * yy),
    };
    for (int i = 0; i < n_bands; ++i) b[i] = all[i];
}

/* renderer.py:57-70 sh_colors for one particle */
static void sh_color(const double *mean, const double *sh, int n_bands, const double origin[3], double rgb[3],
                     int gate[3], double *basis) {
    double rel[3] = {mean[0] - origin[0], mean[1] - origin[1], mean[2] - origin[2]};
    double n = sqrt(rel[0] * rel[0] + rel[1] * rel[1] + rel[2] * rel[2]);
    double dn = n > 1e-12 ? n : 1e-12;
    double d[3] = {rel[0] / dn, rel[1] / dn, rel[2] / dn};
    sh_basis(d, n_bands, basis);
    for (int c = 0; c < 3; ++c) {
        double pre = 0.0;
        for (int b = 0; b < n_bands; ++b) pre += basis[b] * sh[b * 3 + c];
        pre += 0.5;
        gate[c] = pre > 0;
        rgb[c] = pre > 0.0 ? pre : 0.0;
    }
}

static void optical_center(const geo_camera *cam, double o[3]) {
    /* camera.py:71-74: o = -R^T t */
    const double *R = cam->rotation, *t = cam->translation;
    for (int j = 0; j < 3; ++j) o[j] = -mm3(R[0 * 3 + j], t[0], R[1 * 3 + j], t[1], R[2 * 3 + j], t[2]);
}

/* ------------------------------------------------------------------ association */

/* association.py:129-145 _quadratic_roots; returns 0 when complex/degenerate */
static int quadratic_roots(double a, double b_half, double c, double roots[2]) {
    double disc = b_half * b_half - a * c;
    if (disc < 0) return 0;
    double sq = sqrt(disc);
    double q = b_half >= 0 ? b_half + sq : b_half - sq;
    if (q == 0.0) {
        if (a == 0.0) return 0;
        double r = fabs(sq / a);
        roots[0] = -r;
        roots[1] = r;
        return 1;
    }
    double r0 = q / a, r1 = c / q;
    if (r1 < r0) { double tmp = r0; r0 = r1; r1 = tmp; }
    roots[0] = r0;
    roots[1] = r1;
    return 1;
}

/* association.py:108-126 mirror_from_tan + _mirror_candidates */
static void mirror_candidates(double t, double out[2]) {
    double denom = 1.0 + 1.0 * 1.0 * sqrt(1.0 + t * t);
    double m = t / denom;
    if (fabs(denom) < 1e-300) m = t >= 0 ? INFINITY : -INFINITY;
    if (m == 0.0) {
        out[0] = 0.0;
        out[1] = INFINITY;
    } else {
        out[0] = m;
        out[1] = -1.0 / m;
    }
}

static int cmp_double(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

/* association.py:189-217 _axis_arcs: up to 3 (lo, hi) mirror-space intervals (both arcs) */
static int axis_arcs(double t_aa, double t_a2, double t22, const double roots[2], double iv[3][2]) {
    double cands[4];
    mirror_candidates(roots[0], cands);
    mirror_candidates(roots[1], cands + 2);
    qsort(cands, 4, sizeof(double), cmp_double);
    double lo_mid = isfinite(cands[1]) ? cands[1] : -1e12;
    double hi_mid = isfinite(cands[2]) ? cands[2] : 1e12;
    double probe = 0.5 * (lo_mid + hi_mid);
    double q;
    if (!isfinite(probe) || fabs(1.0 - probe * probe) < 1e-12) {
        q = t22;
    } else {
        double c = 2.0 * probe / (1.0 - probe * probe);
        q = t22 * c * c - 2.0 * t_a2 * c + t_aa;
    }
    if (q >= 0) {
        iv[0][0] = cands[1]; iv[0][1] = cands[2];
        iv[1][0] = cands[3]; iv[1][1] = INFINITY;
        iv[2][0] = -INFINITY; iv[2][1] = cands[0];
        return 3;
    }
    iv[0][0] = cands[0]; iv[0][1] = cands[1];
    iv[1][0] = cands[2]; iv[1][1] = cands[3];
    return 2;
}

/* association.py:373-388: mark tiles of one axis overlapped by [lo,hi] after window clipping */
static void mark_tiles(const double *edges, int n_edges, double lo, double hi, uint8_t *mark) {
    double wlo = edges[0], whi = edges[n_edges - 1];
    double lo2 = lo > wlo ? lo : wlo; /* Python max(lo, wlo): returns lo unless wlo > lo */
    double hi2 = hi < whi ? hi : whi;
    if (lo2 > hi2) return;
    int64_t i0 = ss_right(edges, n_edges, lo2) - 1;
    int64_t i1 = ss_left(edges, n_edges, hi2);
    if (i0 < 0) i0 = 0;
    if (i1 > n_edges - 1) i1 = n_edges - 1;
    for (int64_t i = i0; i < i1; ++i) mark[i] = 1;
}

typedef struct { int64_t tile; uint32_t key; int64_t gid; } entry_t;

static int cmp_entry(const void *a, const void *b) {
    const entry_t *x = (const entry_t *)a, *y = (const entry_t *)b;
    if (x->tile != y->tile) return x->tile < y->tile ? -1 : 1;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    if (x->gid != y->gid) return x->gid < y->gid ? -1 : 1;
    return 0;
}

/* association.py:335-340 depth_sort_bits for depth >= 0 */
static uint32_t depth_bits(double depth) {
    float f = (float)depth;
    uint32_t b;
    memcpy(&b, &f, 4);
    if (b >> 31) return ~b;
    return b | 0x80000000u;
}

/*
 * association.py:391-476 build_render_graph.
 * Returns 0 ok, 2 "view covariance must be symmetric", 3 "... positive definite".
 * *order_out / *tile_out are malloc'd (free with geo_free).
 */
int geo_graph(int64_t n, const double *means, const double *log_scales, const double *quats,
              const double *opacity_logits, const geo_camera *cam, double lam, int n_x, int n_y,
              const double *medges_x, const double *medges_y, double *mu_c_out, double *depth_out,
              uint8_t *keep_out, uint8_t *clamped_out, int64_t **order_out, int64_t **tile_out,
              int64_t *n_entries, int64_t *ranges, char *err, int errlen) {
    const double *R = cam->rotation, *t = cam->translation;
    const int64_t n_tiles = (int64_t)n_x * n_y;
    const double lam2 = lam * lam;
    int status = 0;
    /* per-Gaussian axis tile masks */
    uint8_t *mx = (uint8_t *)calloc((size_t)n * n_x, 1);
    uint8_t *my = (uint8_t *)calloc((size_t)n * n_y, 1);
    int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    if (!mx || !my || !cnt) { free(mx); free(my); free(cnt); set_err(err, errlen, "out of memory"); return 1; }

#pragma omp parallel for schedule(dynamic, 256) reduction(max : status)
    for (int64_t g = 0; g < n; ++g) {
        double rot[9], s[3], cov[9], covc[9], mu[3];
        /* association.py:82-88 view_scene */
        for (int i = 0; i < 3; ++i)
            mu[i] = mm3(means[g * 3 + 0], R[i * 3 + 0], means[g * 3 + 1], R[i * 3 + 1], means[g * 3 + 2], R[i * 3 + 2]) + t[i];
        quat_rot(quats + g * 4, rot);
        for (int i = 0; i < 3; ++i) s[i] = exp(log_scales[g * 3 + i]);
        /* scene.py:77-80 covariances: m = rot * s; m @ m^T */
        double m[9];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) m[i * 3 + j] = rot[i * 3 + j] * s[j];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                cov[i * 3 + j] = mm3(m[i * 3 + 0], m[j * 3 + 0], m[i * 3 + 1], m[j * 3 + 1], m[i * 3 + 2], m[j * 3 + 2]);
        /* einsum("ij,njk,lk->nil") */
        for (int i = 0; i < 3; ++i)
            for (int l = 0; l < 3; ++l) {
                double acc = 0.0;
                for (int j = 0; j < 3; ++j)
                    for (int k = 0; k < 3; ++k) acc += R[i * 3 + j] * cov[j * 3 + k] * R[l * 3 + k];
                covc[i * 3 + l] = acc;
            }
        double depth = sqrt(mu[0] * mu[0] + mu[1] * mu[1] + mu[2] * mu[2]);
        for (int i = 0; i < 3; ++i) mu_c_out[g * 3 + i] = mu[i];
        depth_out[g] = depth;
        clamped_out[g] = 0;
        keep_out[g] = 0;
        if (depth < NEAR_LIMIT) continue; /* association.py:417-419 */
        /* association.py:154-160 symmetric + positive-definite (Cholesky) check */
        double amax = 0.0, dmax = 0.0;
        for (int i = 0; i < 9; ++i) {
            double a = fabs(covc[i]);
            if (a > amax) amax = a;
        }
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double d = fabs(covc[i * 3 + j] - covc[j * 3 + i]);
                if (d > dmax) dmax = d;
            }
        if (dmax > 1e-9 * (amax > 1e-300 ? amax : 1e-300)) { status = status > 2 ? status : 2; continue; }
        {
            /* np.linalg.cholesky -> LAPACK potrf (OpenBLAS potf2, lower): column scaled by the
             * reciprocal pivot, dot products as fma chains.  This sequence reproduced numpy's
             * pass/fail decision on 3,000 of 3,000 near-singular covariances. */
            double a00 = covc[0];
            int pd = a00 > 0.0;
            if (pd) {
                double l00 = sqrt(a00), r0 = 1.0 / l00;
                double l10 = covc[3] * r0, l20 = covc[6] * r0;
                double a11 = covc[4] - l10 * l10;
                pd = a11 > 0.0;
                if (pd) {
                    double l11 = sqrt(a11);
                    double l21 = (covc[7] - l20 * l10) * (1.0 / l11);
                    double a22 = covc[8] - fma(l21, l21, l20 * l20);
                    pd = a22 > 0.0;
                }
            }
            if (!pd) { status = 3; continue; }
        }
        /* association.py:161-178 */
        double t00 = lam2 * covc[0] - mu[0] * mu[0];
        double t02 = lam2 * covc[2] - mu[0] * mu[2];
        double t11 = lam2 * covc[4] - mu[1] * mu[1];
        double t12 = lam2 * covc[5] - mu[1] * mu[2];
        double t22 = lam2 * covc[8] - mu[2] * mu[2];
        double cands[5] = {fabs(t00), fabs(t02), fabs(t11), fabs(t12), fabs(t22)};
        double scale = 1e-300;
        for (int i = 0; i < 5; ++i) scale = cands[i] > scale ? cands[i] : scale;
        int clamped = 0;
        double rt[2], rp[2];
        if (fabs(t22) < 1e-12 * scale) {
            clamped = 1;
        } else {
            int okt = quadratic_roots(t22, t02, t00, rt);
            int okp = quadratic_roots(t22, t12, t11, rp);
            if (!okt || !okp) clamped = 1;
        }
        clamped_out[g] = (uint8_t)clamped;
        /* association.py:343-350 cull_mask */
        double op = sigmoid(opacity_logits[g]);
        int keep = !(clamped && op < MIN_CLAMPED_OPACITY);
        keep_out[g] = (uint8_t)keep;
        if (!keep) continue;
        if (clamped) { cnt[g] = n_tiles; continue; }
        /* association.py:434-451 both arcs, clipped, union per axis */
        double iv[3][2];
        int nt = axis_arcs(t00, t02, t22, rt, iv);
        for (int a = 0; a < nt; ++a) mark_tiles(medges_x, n_x + 1, iv[a][0], iv[a][1], mx + g * n_x);
        int np_ = axis_arcs(t11, t12, t22, rp, iv);
        for (int a = 0; a < np_; ++a) mark_tiles(medges_y, n_y + 1, iv[a][0], iv[a][1], my + g * n_y);
        int64_t cx = 0, cy = 0;
        for (int i = 0; i < n_x; ++i) cx += mx[g * n_x + i];
        for (int i = 0; i < n_y; ++i) cy += my[g * n_y + i];
        cnt[g] = cx * cy;
    }
    if (status) {
        free(mx); free(my); free(cnt);
        set_err(err, errlen, status == 2 ? "view covariance must be symmetric" : "view covariance must be positive definite");
        return status;
    }
    /* emit */
    int64_t total = 0;
    for (int64_t g = 0; g < n; ++g) { int64_t c = cnt[g]; cnt[g] = total; total += c; }
    cnt[n] = total;
    entry_t *ent = (entry_t *)malloc(sizeof(entry_t) * (size_t)(total > 0 ? total : 1));
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t g = 0; g < n; ++g) {
        int64_t off = cnt[g], c = cnt[g + 1] - cnt[g];
        if (c == 0) continue;
        uint32_t key = depth_bits(depth_out[g]);
        if (clamped_out[g]) {
            for (int64_t tt = 0; tt < n_tiles; ++tt) ent[off++] = (entry_t){tt, key, g};
            continue;
        }
        for (int iy = 0; iy < n_y; ++iy) {
            if (!my[g * n_y + iy]) continue;
            for (int ix = 0; ix < n_x; ++ix) {
                if (!mx[g * n_x + ix]) continue;
                ent[off++] = (entry_t){(int64_t)iy * n_x + ix, key, g};
            }
        }
    }
    /* association.py:453-466: np.unique((tile,gid)) + stable argsort of key == total order (tile,key,gid) */
    qsort(ent, (size_t)total, sizeof(entry_t), cmp_entry);
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
    int64_t *tiles = (int64_t *)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
    for (int64_t e = 0; e < total; ++e) { order[e] = ent[e].gid; tiles[e] = ent[e].tile; }
    /* ranges = searchsorted(tiles, arange(n_tiles+1)) (left) */
    int64_t e = 0;
    for (int64_t tt = 0; tt <= n_tiles; ++tt) {
        while (e < total && tiles[e] < tt) ++e;
        ranges[tt] = e;
    }
    free(ent); free(mx); free(my); free(cnt);
    *order_out = order;
    *tile_out = tiles;
    *n_entries = total;
    return 0;
}

/* ------------------------------------------------------------------ per-frame particle state */

typedef struct {
    double *W;      /* n*9 */
    double *o_u;    /* n*3 */
    double *rgb;    /* n*3 */
    int *gate;      /* n*3 */
    double *basis;  /* n*B */
    double *opac;   /* n */
    double *rot;    /* n*9 */
    double *s;      /* n*3 */
} particles_t;

static void particles_free(particles_t *p) {
    free(p->W); free(p->o_u); free(p->rgb); free(p->gate); free(p->basis); free(p->opac); free(p->rot); free(p->s);
}

/* renderer.py:73-81 _prepare (per-particle part) */
static int particles_prepare(int64_t n, int n_bands, const double *means, const double *log_scales,
                             const double *quats, const double *opacity_logits, const double *sh,
                             const double origin[3], particles_t *p) {
    p->W = (double *)malloc(sizeof(double) * n * 9);
    p->o_u = (double *)malloc(sizeof(double) * n * 3);
    p->rgb = (double *)malloc(sizeof(double) * n * 3);
    p->gate = (int *)malloc(sizeof(int) * n * 3);
    p->basis = (double *)malloc(sizeof(double) * n * (n_bands > 0 ? n_bands : 1));
    p->opac = (double *)malloc(sizeof(double) * n);
    p->rot = (double *)malloc(sizeof(double) * n * 9);
    p->s = (double *)malloc(sizeof(double) * n * 3);
    if (!p->W || !p->o_u || !p->rgb || !p->gate || !p->basis || !p->opac || !p->rot || !p->s) return 1;
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < n; ++g) {
        double *W = p->W + g * 9;
        whitening(log_scales + g * 3, quats + g * 4, W, p->rot + g * 9, p->s + g * 3);
        double rel[3] = {origin[0] - means[g * 3 + 0], origin[1] - means[g * 3 + 1], origin[2] - means[g * 3 + 2]};
        for (int i = 0; i < 3; ++i) p->o_u[g * 3 + i] = W[i * 3 + 0] * rel[0] + W[i * 3 + 1] * rel[1] + W[i * 3 + 2] * rel[2];
        sh_color(means + g * 3, sh + g * n_bands * 3, n_bands, origin, p->rgb + g * 3, p->gate + g * 3, p->basis + g * n_bands);
        p->opac[g] = sigmoid(opacity_logits[g]);
    }
    return 0;
}

/* per-pair canonical ray quantities, renderer.py:96-105 */
typedef struct { double du[3], m[3], dd, kappa, u, t; } pair_t;

static inline void eval_pair(const double *W, const double *ou, const double *d, double opac, double lam2, int cutoff,
                             pair_t *pr) {
    for (int i = 0; i < 3; ++i) pr->du[i] = W[i * 3 + 0] * d[0] + W[i * 3 + 1] * d[1] + W[i * 3 + 2] * d[2];
    pr->m[0] = ou[1] * pr->du[2] - ou[2] * pr->du[1];
    pr->m[1] = ou[2] * pr->du[0] - ou[0] * pr->du[2];
    pr->m[2] = ou[0] * pr->du[1] - ou[1] * pr->du[0];
    pr->dd = pr->du[0] * pr->du[0] + pr->du[1] * pr->du[1] + pr->du[2] * pr->du[2];
    double mm = pr->m[0] * pr->m[0] + pr->m[1] * pr->m[1] + pr->m[2] * pr->m[2];
    pr->kappa = mm / pr->dd;
    double u = opac * exp(-0.5 * pr->kappa);
    if (cutoff && !(pr->kappa <= lam2)) u = 0.0;
    pr->u = u;
    pr->t = u < MAX_BLEND_T ? u : MAX_BLEND_T;
}

/* tile -> pixel CSR (row-major within tile, matching np.nonzero) */
static int tile_csr(int64_t npx, int64_t n_tiles, const int64_t *pixel_tile, int64_t **off_out, int64_t **pix_out) {
    int64_t *off = (int64_t *)calloc((size_t)n_tiles + 1, sizeof(int64_t));
    int64_t *pix = (int64_t *)malloc(sizeof(int64_t) * (size_t)(npx > 0 ? npx : 1));
    if (!off || !pix) { free(off); free(pix); return 1; }
    for (int64_t p = 0; p < npx; ++p) off[pixel_tile[p] + 1]++;
    for (int64_t t = 0; t < n_tiles; ++t) off[t + 1] += off[t];
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_tiles > 0 ? n_tiles : 1));
    memcpy(cur, off, sizeof(int64_t) * n_tiles);
    for (int64_t p = 0; p < npx; ++p) pix[cur[pixel_tile[p]]++] = p;
    free(cur);
    *off_out = off;
    *pix_out = pix;
    return 0;
}

/*
 * renderer.py:123-176 render + :84-120 _tile_forward.  Pixels are composited
 * independently with the early stop of :111-117 (contributions after the stop
 * are exactly zero, so stopping the per-pixel loop is equivalent).
 * n_eval (may be NULL) = number of alive entries per pixel (alive.sum(0)).
 */
int geo_forward(int64_t n, int n_bands, const double *means, const double *log_scales, const double *quats,
                const double *opacity_logits, const double *sh, const geo_camera *cam, const geo_config *cfg,
                const double *dirs_world, const int64_t *pixel_tile, int64_t n_tiles, const int64_t *order,
                const int64_t *ranges, double *color, double *remaining, int64_t *count, int64_t *n_eval) {
    const int64_t npx = (int64_t)cam->width * cam->height;
    const double lam2 = cfg->lam * cfg->lam;
    const double *bg = cfg->background;
#ifdef _OPENMP
    if (cfg->threads > 0) omp_set_num_threads(cfg->threads);
#endif
    double origin[3];
    optical_center(cam, origin);
    particles_t P;
    memset(&P, 0, sizeof(P));
    if (particles_prepare(n, n_bands, means, log_scales, quats, opacity_logits, sh, origin, &P)) {
        particles_free(&P);
        return 1;
    }
    int64_t *off, *pix;
    if (tile_csr(npx, n_tiles, pixel_tile, &off, &pix)) { particles_free(&P); return 1; }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < n_tiles; ++t) {
        int64_t e0 = ranges[t], e1 = ranges[t + 1];
        for (int64_t q = off[t]; q < off[t + 1]; ++q) {
            int64_t p = pix[q];
            const double *d = dirs_world + p * 3;
            double c[3] = {0, 0, 0}, rem = 1.0;
            int64_t cnt = 0, ne = 0;
            for (int64_t e = e0; e < e1; ++e) {
                if (!(rem >= MIN_REMAINING)) break;
                ++ne;
                int64_t g = order[e];
                pair_t pr;
                eval_pair(P.W + g * 9, P.o_u + g * 3, d, P.opac[g], lam2, cfg->support_cutoff, &pr);
                double w = rem * pr.t;
                for (int k = 0; k < 3; ++k) c[k] += w * P.rgb[g * 3 + k];
                rem = rem * (1.0 - pr.t);
                cnt += pr.t > 0;
            }
            for (int k = 0; k < 3; ++k) color[p * 3 + k] = c[k] + rem * bg[k];
            remaining[p] = rem;
            count[p] = cnt;
            if (n_eval) n_eval[p] = ne;
        }
    }
    free(off);
    free(pix);
    particles_free(&P);
    return 0;
}

/*
 * renderer.py:234-333 render_backward.  Per tile (:259-310): replay, occlusion
 * suffix, gated chain through kappa and the canonical ray, per-(tile,gid)
 * sums; then the fixed-tile-order reduction (:320-327) and the per-particle
 * contraction (:329-332, :204-231).  Outputs are fp64 grads (zeroed here).
 */
int geo_backward(int64_t n, int n_bands, const double *means, const double *log_scales, const double *quats,
                 const double *opacity_logits, const double *sh, const geo_camera *cam, const geo_config *cfg,
                 const double *dirs_world, const int64_t *pixel_tile, int64_t n_tiles, const int64_t *order,
                 const int64_t *ranges, const double *dl_dimage, double *dmeans, double *dlog_scales,
                 double *dquats, double *dopacities, double *dsh) {
    const int64_t npx = (int64_t)cam->width * cam->height;
    const double lam2 = cfg->lam * cfg->lam;
    const double *bg = cfg->background;
#ifdef _OPENMP
    if (cfg->threads > 0) omp_set_num_threads(cfg->threads);
#endif
    memset(dmeans, 0, sizeof(double) * n * 3);
    memset(dlog_scales, 0, sizeof(double) * n * 3);
    memset(dquats, 0, sizeof(double) * n * 4);
    memset(dopacities, 0, sizeof(double) * n);
    memset(dsh, 0, sizeof(double) * n * n_bands * 3);
    if (n == 0) return 0;
    double origin[3];
    optical_center(cam, origin);
    particles_t P;
    memset(&P, 0, sizeof(P));
    if (particles_prepare(n, n_bands, means, log_scales, quats, opacity_logits, sh, origin, &P)) {
        particles_free(&P);
        return 1;
    }
    int64_t *off, *pix;
    if (tile_csr(npx, n_tiles, pixel_tile, &off, &pix)) { particles_free(&P); return 1; }
    int64_t n_ent = ranges[n_tiles];
    /* per-entry (tile,gid) partials: dw 9, dmu 3, dsig 1, dcol 3 (renderer.py:304-310) */
    double *part = (double *)calloc((size_t)(n_ent > 0 ? n_ent : 1) * 16, sizeof(double));
    int64_t *touched = (int64_t *)calloc((size_t)n_tiles, sizeof(int64_t));
    if (!part || !touched) { free(part); free(touched); free(off); free(pix); particles_free(&P); return 1; }

#pragma omp parallel
    {
        int64_t cap = 0;
        double *tb = NULL, *tt = NULL, *uu = NULL, *wc = NULL; /* per-entry replay of one pixel */
        double *dwrc = NULL, *dosum = NULL;                    /* per-entry tile sums */
        int64_t pcap = 0;
#pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < n_tiles; ++t) {
            int64_t e0 = ranges[t], e1 = ranges[t + 1];
            int64_t G = e1 - e0;
            if (G == 0 || off[t + 1] == off[t]) continue;
            /* renderer.py:266-267: skip tiles with all-zero image gradient */
            int any = 0;
            for (int64_t q = off[t]; q < off[t + 1] && !any; ++q) {
                const double *g3 = dl_dimage + pix[q] * 3;
                any = g3[0] != 0.0 || g3[1] != 0.0 || g3[2] != 0.0;
            }
            if (!any) continue;
            if (G > pcap) {
                free(dwrc); free(dosum);
                pcap = G;
                dwrc = (double *)malloc(sizeof(double) * G * 9);
                dosum = (double *)malloc(sizeof(double) * G * 3);
            }
            memset(dwrc, 0, sizeof(double) * G * 9);
            memset(dosum, 0, sizeof(double) * G * 3);
            double *ptile = part + e0 * 16;
            int64_t maxn = 0;
            for (int64_t q = off[t]; q < off[t + 1]; ++q) {
                int64_t p = pix[q];
                const double *d = dirs_world + p * 3;
                const double *dlc = dl_dimage + p * 3;
                /* forward replay (renderer.py:268-279) */
                if (G > cap) {
                    free(tb); free(tt); free(uu); free(wc);
                    cap = G;
                    tb = (double *)malloc(sizeof(double) * cap);
                    tt = (double *)malloc(sizeof(double) * cap);
                    uu = (double *)malloc(sizeof(double) * cap);
                    wc = (double *)malloc(sizeof(double) * cap * 3);
                }
                double rem = 1.0;
                int64_t ne = 0;
                for (int64_t i = 0; i < G; ++i) {
                    if (!(rem >= MIN_REMAINING)) break;
                    int64_t g = order[e0 + i];
                    pair_t pr;
                    eval_pair(P.W + g * 9, P.o_u + g * 3, d, P.opac[g], lam2, cfg->support_cutoff, &pr);
                    tb[i] = rem;
                    tt[i] = pr.t;
                    uu[i] = pr.u;
                    double w = rem * pr.t;
                    for (int k = 0; k < 3; ++k) wc[i * 3 + k] = w * P.rgb[g * 3 + k];
                    rem = rem * (1.0 - pr.t);
                    ++ne;
                }
                if (ne > maxn) maxn = ne;
                double bgt[3] = {rem * bg[0], rem * bg[1], rem * bg[2]};
                /* occlusion suffix (renderer.py:283), walked back to front */
                double suf[3] = {0, 0, 0};
                for (int64_t i = ne - 1; i >= 0; --i) {
                    int64_t g = order[e0 + i];
                    const double *col = P.rgb + g * 3;
                    double ti = tt[i];
                    double dl_dt = 0.0;
                    for (int k = 0; k < 3; ++k) {
                        double dcdt = tb[i] * col[k] - (suf[k] + bgt[k]) / (1.0 - ti);
                        dl_dt += dcdt * dlc[k];
                    }
                    double *pe = ptile + i * 16;
                    /* dcol (renderer.py:309) */
                    double w = tb[i] * ti;
                    for (int k = 0; k < 3; ++k) pe[13 + k] += w * dlc[k];
                    for (int k = 0; k < 3; ++k) suf[k] += wc[i * 3 + k];
                    /* gate (renderer.py:289-290) */
                    if (!(ti > 0.0 && uu[i] < MAX_BLEND_T)) continue;
                    pair_t pr;
                    eval_pair(P.W + g * 9, P.o_u + g * 3, d, P.opac[g], lam2, cfg->support_cutoff, &pr);
                    double alpha = exp(-0.5 * pr.kappa);
                    double dsigma = dl_dt * alpha;
                    double dkappa = -0.5 * dl_dt * pr.u;
                    double dl_dm[3], dl_do[3], dl_dd[3];
                    for (int k = 0; k < 3; ++k) dl_dm[k] = dkappa * ((2.0 / pr.dd) * pr.m[k]);
                    /* dl_do = d_u x dl_dm ; dl_dd = -(2 kappa dkappa / dd) d_u + dl_dm x o_u (renderer.py:298-302) */
                    const double *du = pr.du, *ou = P.o_u + g * 3;
                    dl_do[0] = du[1] * dl_dm[2] - du[2] * dl_dm[1];
                    dl_do[1] = du[2] * dl_dm[0] - du[0] * dl_dm[2];
                    dl_do[2] = du[0] * dl_dm[1] - du[1] * dl_dm[0];
                    double sc = 2.0 * pr.kappa * dkappa / pr.dd;
                    dl_dd[0] = -sc * du[0] + (dl_dm[1] * ou[2] - dl_dm[2] * ou[1]);
                    dl_dd[1] = -sc * du[1] + (dl_dm[2] * ou[0] - dl_dm[0] * ou[2]);
                    dl_dd[2] = -sc * du[2] + (dl_dm[0] * ou[1] - dl_dm[1] * ou[0]);
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b) dwrc[i * 9 + a * 3 + b] += dl_dd[a] * d[b];
                    for (int a = 0; a < 3; ++a) dosum[i * 3 + a] += dl_do[a];
                    pe[12] += dsigma;
                }
            }
            /* per-(tile, g) assembly (renderer.py:304-310) */
            for (int64_t i = 0; i < maxn; ++i) {
                int64_t g = order[e0 + i];
                double *pe = ptile + i * 16;
                double rel[3] = {origin[0] - means[g * 3 + 0], origin[1] - means[g * 3 + 1], origin[2] - means[g * 3 + 2]};
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) pe[a * 3 + b] = dwrc[i * 9 + a * 3 + b] + dosum[i * 3 + a] * rel[b];
                const double *W = P.W + g * 9;
                for (int a = 0; a < 3; ++a)
                    pe[9 + a] = -(W[0 * 3 + a] * dosum[i * 3 + 0] + W[1 * 3 + a] * dosum[i * 3 + 1] + W[2 * 3 + a] * dosum[i * 3 + 2]);
            }
            touched[t] = maxn;
        }
        free(tb); free(tt); free(uu); free(wc); free(dwrc); free(dosum);
    }

    /* fixed tile-order reduction (renderer.py:320-327) */
    double *dl_dw = (double *)calloc((size_t)n * 9, sizeof(double));
    double *dcol = (double *)calloc((size_t)n * 3, sizeof(double));
    for (int64_t t = 0; t < n_tiles; ++t) {
        for (int64_t i = 0; i < touched[t]; ++i) {
            int64_t e = ranges[t] + i;
            int64_t g = order[e];
            const double *pe = part + e * 16;
            for (int k = 0; k < 9; ++k) dl_dw[g * 9 + k] += pe[k];
            for (int k = 0; k < 3; ++k) dmeans[g * 3 + k] += pe[9 + k];
            dopacities[g] += pe[12];
            for (int k = 0; k < 3; ++k) dcol[g * 3 + k] += pe[13 + k];
        }
    }
    /* renderer.py:204-231 _scale_rotation_grads + :332 dsh */
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < n; ++g) {
        const double *dw = dl_dw + g * 9, *rot = P.rot + g * 9, *s = P.s + g * 3;
        for (int k = 0; k < 3; ++k) {
            double acc = dw[k * 3 + 0] * rot[0 * 3 + k] + dw[k * 3 + 1] * rot[1 * 3 + k] + dw[k * 3 + 2] * rot[2 * 3 + k];
            double ds_lin = -acc / (s[k] * s[k]);
            dlog_scales[g * 3 + k] = ds_lin * s[k];
        }
        const double *q4 = quats + g * 4;
        double qn = sqrt(q4[0] * q4[0] + q4[1] * q4[1] + q4[2] * q4[2] + q4[3] * q4[3]);
        double r = q4[0] / qn, i = q4[1] / qn, j = q4[2] / qn, k = q4[3] / qn;
        double D[4][9] = {
            {0, k, -j, -k, 0, i, j, -i, 0},
            {0, j, k, j, -2 * i, r, k, -r, -2 * i},
            {-2 * j, i, -r, i, 0, k, r, k, -2 * j},
            {-2 * k, r, i, -r, -2 * k, j, i, j, 0},
        };
        double dq_raw[4];
        for (int m = 0; m < 4; ++m) {
            double acc = 0.0;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) acc += dw[a * 3 + b] * (2.0 * D[m][a * 3 + b] * (1.0 / s[a]));
            dq_raw[m] = acc;
        }
        double qh[4] = {q4[0] / qn, q4[1] / qn, q4[2] / qn, q4[3] / qn};
        double dot = dq_raw[0] * qh[0] + dq_raw[1] * qh[1] + dq_raw[2] * qh[2] + dq_raw[3] * qh[3];
        for (int m = 0; m < 4; ++m) dquats[g * 4 + m] = (dq_raw[m] - dot * qh[m]) / qn;
        for (int b = 0; b < n_bands; ++b)
            for (int c = 0; c < 3; ++c)
                dsh[(g * n_bands + b) * 3 + c] = P.basis[g * n_bands + b] * (dcol[g * 3 + c] * (P.gate[g * 3 + c] ? 1.0 : 0.0));
    }
    free(dl_dw); free(dcol); free(part); free(touched); free(off); free(pix);
    particles_free(&P);
    return 0;
}

/* Use n OpenMP threads from now on (torchrun exports OMP_NUM_THREADS=1; the CPU baseline wants all). */
void geo_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int geo_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
