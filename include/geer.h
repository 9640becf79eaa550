/*
 * geer.h — C ABI of the B200-native 3DGEER rendering hot path (libgeer_b200.so).
 *
 * The reference (raygauss 0.1.0, pure Python) exposes this path as three
 * functions; each host-level entry point below replaces one of them 1:1 and
 * takes the same data the Python call receives, as plain pointers + sizes:
 *
 *   geer_render_host           <- raygauss.renderer.render
 *                                 (pkg/src/raygauss/renderer.py:123-176)
 *   geer_render_backward_host  <- raygauss.renderer.render_backward
 *                                 (pkg/src/raygauss/renderer.py:234-333)
 *   geer_build_graph_host      <- raygauss.association.build_render_graph
 *   + geer_graph_info/export      (pkg/src/raygauss/association.py:391-476,
 *                                  RenderGraph :353-370, CSFGrid :272-298)
 *
 * Host-level calls take HOST float64 arrays in the reference's layouts
 * (GaussianScene scene.py:35-51, dl_dimage (H,W,3), FrameOutput
 * renderer.py:39-44, SceneGrads renderer.py:179-201) and do the
 * host<->device copies themselves.  The device-level calls (geer_forward /
 * geer_backward) take DEVICE fp32 pointers and a cudaStream_t and never copy
 * to the host except the 12-byte frame header (entry count + error flag).
 *
 * Errors: every call returns a geer_status; geer_last_error() gives the
 * thread-local message.  GEER_ERR_NOT_PD / GEER_ERR_NOT_SYMMETRIC carry the
 * reference's ValueError messages (association.py:155-160) verbatim.
 * Camera validation (camera.py:54-69) is done by the caller-side wrapper
 * before the call; geer_* re-checks only what would crash a kernel.
 */
#ifndef GEER_H_
#define GEER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GEER_ABI_VERSION 1

typedef enum geer_status {
    GEER_OK = 0,
    GEER_ERR_INVALID = 1,        /* bad argument (ValueError in the wrapper) */
    GEER_ERR_NOT_SYMMETRIC = 2,  /* "view covariance must be symmetric" */
    GEER_ERR_NOT_PD = 3,         /* "view covariance must be positive definite" */
    GEER_ERR_CUDA = 4,           /* CUDA runtime error */
    GEER_ERR_NOMEM = 5,          /* device allocation failed */
    GEER_ERR_STATE = 6,          /* backward without a matching forward */
    GEER_ERR_OVERFLOW = 7        /* geer_sync: a frame since the last sync outgrew the context's graph
                                    capacity; the capacity has grown and the LAST frame has been rendered
                                    again (its outputs are valid), work that consumed an earlier one
                                    must be redone */
} geer_status;

typedef enum geer_model { GEER_PINHOLE = 0, GEER_KB = 1, GEER_BEAP = 2 } geer_model;

/* raygauss.camera.Camera (camera.py:25-48); unused intrinsics may be NaN. */
typedef struct geer_camera {
    int32_t width, height, model, pad_;
    double rotation[9];    /* R_c row-major: x_c = R_c x + t_c */
    double translation[3]; /* t_c */
    double fov_x, fov_y;   /* radians (beap) */
    double fx, fy, cx, cy; /* pinhole / kb */
    double k[4];           /* kb distortion */
} geer_camera;

/* raygauss.renderer.RenderConfig (renderer.py:24-37); threads is ignored. */
typedef struct geer_config {
    double lam;
    double background[3];
    int32_t tile_px;
    int32_t support_cutoff;
    int32_t threads;
    int32_t flags; /* GEER_CFG_* debug switches (0 = default behaviour) */
} geer_config;

/* Disable the per-warp PBF culling of the raster (results are identical; for tests). */
#define GEER_CFG_NO_CULL 1
/* Exhaustive forward (an oracle of the association at scale, oracle.py:172-228 exhaustive_render):
 * every tile composites ALL kept Gaussians in global (depth, gid) order instead of its association
 * list.  Forward only (a following geer_backward fails with GEER_ERR_STATE). */
#define GEER_CFG_EXHAUSTIVE 2

/* Device scene: fp32 SoA in the reference's stored spaces (scene.py:35-51). */
typedef struct geer_scene {
    int64_t n;
    int32_t n_bands; /* 1, 4, 9 or 16 */
    int32_t pad_;
    const float *means;          /* (n,3) */
    const float *log_scales;     /* (n,3) */
    const float *quats;          /* (n,4) raw (r,i,j,k) */
    const float *opacity_logits; /* (n,) */
    const float *sh;             /* (n,n_bands,3) */
} geer_scene;

/* Device gradients in the same SoA layout (renderer.py:179-201 conventions:
 * dopacities w.r.t. LINEAR opacity, dquats with the normalisation Jacobian). */
typedef struct geer_grads {
    float *dmeans, *dlog_scales, *dquats, *dopacities, *dsh;
} geer_grads;

/* Host scene: float64 arrays exactly as GaussianScene holds them. */
typedef struct geer_host_scene {
    int64_t n;
    int32_t n_bands;
    int32_t pad_;
    const double *means, *log_scales, *quats, *opacity_logits, *sh;
} geer_host_scene;

typedef struct geer_host_grads {
    double *dmeans, *dlog_scales, *dquats, *dopacities, *dsh;
} geer_host_grads;

/* Per-frame statistics of the last forward (filled by geer_frame_stats). */
typedef struct geer_stats {
    int64_t n_gaussians;
    int64_t n_entries;        /* |RenderGraph.order| */
    int64_t n_tiles;
    int64_t n_work_items;     /* raster CTAs launched with work */
    int64_t evaluated_pairs;  /* sum over pixels of alive entries (n_eval) */
    int64_t kappa_rechecks;   /* fp64 re-evaluations of the kappa cutoff */
    int64_t fixup_pixels;     /* pixels recomposited in fp64 (early stop too close to call in fp32) */
    int64_t clamped;          /* clamped & kept particles */
    int64_t warp_entries;     /* forward (warp, entry) evaluations after PBF culling */
    int64_t streamed_entries; /* forward entries streamed into shared memory (all raster CTAs) */
    float ms_prep, ms_dup, ms_sort, ms_render, ms_total; /* CUDA-event stage times (if timing on) */
    float ms_backward;
} geer_stats;

typedef struct geer_ctx geer_ctx;

int geer_abi_version(void);
const char *geer_last_error(void);

/* One context per (device, stream) user; owns grow-only device workspaces and the
 * state of its last forward (used by the next geer_backward). Not thread-safe. */
geer_ctx *geer_create(int device);
void geer_destroy(geer_ctx *ctx);
int geer_set_timing(geer_ctx *ctx, int enable);

/* ---- device level (fast path) -------------------------------------------------
 * color (H,W,3) f32, remaining (H,W) f32, count (H,W) i32: device buffers.
 * The scene buffers must stay valid until the matching geer_backward.
 * geer_forward is asynchronous on `stream` once the context knows the graph's size (from its first
 * frame, which still reads the entry total back): nothing blocks the host, and a frame issues the
 * same kernels with the same arguments each time (CUDA-graph capturable once the camera is cached).
 * Conditions the reference raises on (non-PD / non-symmetric view covariance, renderer.py ->
 * association.py:155-160) and a graph larger than the context's capacity are recorded on the device;
 * geer_sync synchronises the stream and returns the error (GEER_ERR_NOT_PD / NOT_SYMMETRIC), or
 * GEER_ERR_OVERFLOW after growing the capacity and re-rendering the last frame, else GEER_OK.  An
 * overflowing frame renders background only (no out-of-bounds work).  Read the outputs after
 * geer_sync (or after your own synchronisation, if you accept an unchecked frame). */
int geer_forward(geer_ctx *ctx, const geer_scene *scene, const geer_camera *camera, const geer_config *config,
                 float *color, float *remaining, int32_t *count, void *stream);
int geer_sync(geer_ctx *ctx, void *stream);
/* Frees the context's cached camera setups (K0 outputs of up to 16 other cameras, <= 1 GiB). */
int geer_clear_camera_cache(geer_ctx *ctx);

/* ---- caller-owned workspace (SURVEY 8b ownership) -------------------------------
 * geer_workspace_bytes: device bytes the device-level path (geer_forward + geer_backward) needs for
 * n Gaussians and one camera/config, for a graph of up to max_entries entries (<= 0: the context's
 * learned capacity, or 24 per Gaussian if it has none; ctx may be NULL).  Returns 0 on bad input.
 * geer_set_workspace: the context carves every buffer from [ptr, ptr + bytes) (caller-owned, e.g. a
 * torch tensor) instead of cudaMalloc; synchronises the device and drops the buffers it held.  With a
 * workspace the camera-setup cache is off (one camera's setup at a time), an undersized workspace
 * fails with GEER_ERR_NOMEM naming the bytes needed, ptr = NULL returns to library-owned memory.
 * Host-level calls and geer_association_check still allocate their own staging. */
size_t geer_workspace_bytes(geer_ctx *ctx, int64_t n, int32_t n_bands, const geer_camera *camera,
                            const geer_config *config, int64_t max_entries);
int geer_set_workspace(geer_ctx *ctx, void *ptr, size_t bytes);
int geer_workspace_used(geer_ctx *ctx, size_t *used);

/* dl_dimage (H,W,3) f32 device.  flags: GEER_ACCUMULATE adds into grads (multi-view);
 * GEER_OPACITY_LOGIT returns dopacities w.r.t. the stored logit (trainer.py:208-217)
 * instead of the reference's linear-opacity convention. */
#define GEER_ACCUMULATE 1
#define GEER_OPACITY_LOGIT 2
int geer_backward(geer_ctx *ctx, const float *dl_dimage, const geer_grads *grads, int flags, void *stream);

int geer_frame_stats(geer_ctx *ctx, geer_stats *out);

/* ---- association export (parity with RenderGraph) ------------------------------ */
int geer_graph_info(geer_ctx *ctx, int64_t *n_entries, int32_t *n_x, int32_t *n_y);
/* host pointers; any may be NULL.  order/entry_tile (n_entries), ranges (n_tiles+1),
 * mu_c (n,3), depth (n), keep/clamped (n), pixel_tile (H,W), medges_x (n_x+1), medges_y (n_y+1) */
int geer_graph_export(geer_ctx *ctx, int64_t *order, int64_t *entry_tile, int64_t *ranges, double *mu_c,
                      double *depth, uint8_t *keep, uint8_t *clamped, int64_t *pixel_tile, double *medges_x,
                      double *medges_y);

/* ---- GPU oracle of the association (validation only) --------- */
/* oracle.association_bruteforce (oracle.py:235-281) on the GPU for the context's last graph (after
 * geer_forward / geer_build_graph_host): side x side rays per tile (side = max(8, ceil(sqrt(rays_per_tile))),
 * at most 16), Gaussian g in tile t iff min kappa <= lam^2 over the rays.  out[0] = brute-force
 * (tile, Gaussian) pairs, out[1] = those missing from the tile lists (0 for a sound association),
 * out[2] = kept Gaussians, out[3] = graph entries.  missing (host, may be NULL): the first
 * max_missing missing pairs as (tile, gid).  hit_bits (device, may be NULL): the brute-force sets
 * as an (n_tiles, ceil(n/32)) u32 bitmap, bit g%32 of word g/32.  Synchronous. */
int geer_association_check(geer_ctx *ctx, int32_t rays_per_tile, int64_t *out, int32_t *missing,
                           int32_t max_missing, uint32_t *hit_bits);

/* ---- host level (drop-in replacements of the reference's Python calls) -------- */
int geer_build_graph_host(geer_ctx *ctx, const geer_host_scene *scene, const geer_camera *camera, double lam,
                          int32_t tile_px);
int geer_render_host(geer_ctx *ctx, const geer_host_scene *scene, const geer_camera *camera,
                     const geer_config *config, double *color, double *remaining, int64_t *count);
int geer_render_backward_host(geer_ctx *ctx, const geer_host_scene *scene, const geer_camera *camera,
                              const double *dl_dimage, const geer_config *config, const geer_host_grads *grads);

/* ---- multi-view training glue (BASELINE config 4) ----------------------------- */
/* g = sign(color - target) * scale per element, 0 where mask == 0 (trainer.py:129-132 L1 term). */
int geer_l1_grad(const float *color, const float *target, const uint8_t *mask, float *dl_dimage, int64_t n_pixels,
                 float scale, void *stream);
/* Adam step over a flat fp32 buffer (trainer.py:181-197), per-element lr.  nonfinite (device int32,
 * nullable): when given, the gradients are scanned first; any NaN/Inf sets *nonfinite = 1 and the
 * update is skipped on the device (the non-finite guard of trainer.py:200-205,270-282; the caller
 * zeroes the flag, reads it when it next synchronises and raises NaNLossError). */
int geer_adam(float *param, const float *grad, float *m, float *v, const float *lr, int64_t n, float beta1,
              float beta2, float eps, int32_t step, int32_t *nonfinite, void *stream);

/* Masked (1 - w) L1 + w (1 - SSIM) loss and its image gradient (trainer.py:114-155, SSIM window
 * trainer.py:26-69) for an (H,W,3) f32 device image against an (H,W,3) f32 target; mask (H,W) u8
 * (NULL = all valid).  out (device, 3 doubles): total, L1, 1 - SSIM.  workspace: device buffer of
 * geer_loss_workspace_bytes(H, W). */
size_t geer_loss_workspace_bytes(int height, int width);
int geer_loss(const float *color, const float *target, const uint8_t *mask, int height, int width, float ssim_weight,
              void *workspace, double *out, float *dl_dimage, void *stream);

/* Ground-truth resampling onto the equiangular grid (camera.py:302-339): source (H_s,W_s,3) f32 device
 * image of a pinhole / kb camera -> color (H,W,3) f32 and mask (H,W) u8 on the grid of a beap target
 * camera sharing its extrinsics (checked by the caller). */
int geer_resample_to_beap(const float *source, int source_height, int source_width, const geer_camera *source_camera,
                          const geer_camera *target_camera, float *color, uint8_t *mask, void *stream);

/* 3DGS-compatible PLY vertex block (n records of n_props float32, already on the device) into the fp32
 * SoA of geer_scene, laid out contiguously: means (n,3), log_scales (n,3), quats (n,4), opacity (n),
 * sh (n, (n_vals - 11) / 3, 3); cols[k] = record column of SoA value k (ply.py:94-137). */
int geer_ply_to_soa(const float *block, int64_t n, int n_props, const int32_t *cols, int n_vals, float *soa,
                    void *stream);

/* ---- diagnostics ------------------------------------------------------------- */
/* PCIe bytes the last host-buffer call (geer_render_host / _backward_host / geer_build_graph_host)
 * sent host->device for its inputs: the float64 scene is narrowed to fp32 on host cores, except a raw
 * float64 tail narrowed on the device (GEER_HOST_RAW_FRACTION, when the arrays are pinned). */
int64_t geer_last_h2d_bytes(const geer_ctx *ctx);
/* The last forward's per-pixel alive counts n_eval (H,W) i32 to host memory (renderer.py:113). */
int geer_debug_n_eval(geer_ctx *ctx, int32_t *host_n_eval);
/* Measured FP32 FMA throughput of the device (scalar FFMA and packed FFMA2 chains), TFLOP/s: the
 * roofline denominator of the FP32-bound raster kernels (bench.py). */
int geer_measure_fp32_peak(int device, double *tflops_scalar, double *tflops_packed);

#ifdef __cplusplus
}
#endif
#endif /* GEER_H_ */
