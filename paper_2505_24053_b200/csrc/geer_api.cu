// geer_api.cu — the extern "C" boundary (include/geer.h) and the per-frame driver.
//
// Frame pipeline on one stream (stage names follow SPEC.md:575,602):
//   prep : K0 camera setup (cached per camera: ray tables, tile CSR, work items, per-warp culling
//          regions) + K1 per-Gaussian preprocess (exact fp64 association half + raster payload half)
//   dup  : depth-order sort of the Gaussians (a context's first frame reads the 24-byte header -
//          entry total, (Gaussian, tile row) pairs, error flag - with the sort queued first; later
//          frames run without the host, sized by the learned capacity, see run_forward)
//   sort : per-tile lists by two-level stable bucketing (geer_bin.cu) + the raster work order
//   render: K5 raster + fp64 fix-up of borderline pixels
// The backward (K6 + K7) reuses the forward's graph, payload and per-pixel
// (n_eval, remaining) state held in the context.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <cmath>
#include <string>
#include <utility>

#include "geer_common.cuh"
#include "geer_host.h"
#include "geer_kernels.h"

using namespace geer;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define GEER_CUDA(call)                                                                          \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return fail(GEER_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));          \
    } while (0)

struct Buf {
    void *p = nullptr;
    size_t cap = 0;
    bool owned = true;  // cudaMalloc'ed by the library (else: a slice of the caller's workspace)
};

// A caller-owned device workspace (geer_set_workspace): buffers are carved from it by a bump
// pointer instead of cudaMalloc, so the caller's allocator (torch) owns every byte of the path.
struct Arena {
    char *base = nullptr;
    size_t size = 0, used = 0;
};
thread_local Arena *t_arena = nullptr;  // the arena of the context of the current API call

// TMA tensor map over an array of fixed-size rows (payloads), for the raster's gather4 copies.
int make_row_map(CUtensorMap *map, const void *base, int64_t rows, int row_bytes) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return fail(GEER_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
        encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    const cuuint64_t dims[2] = {(cuuint64_t)(row_bytes / 4), (cuuint64_t)(rows > 0 ? rows : 1)};
    const cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
    const cuuint32_t box[2] = {(cuuint32_t)(row_bytes / 4), 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(GEER_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return GEER_OK;
}

}  // namespace

// One cached camera setup (K0 outputs): the context swaps its camera buffers with a slot, so a
// context rendering a recurring set of views (the multi-view training step) sets each camera up once.
// Only what a frame reads after the setup is cached (ray tables, mirror tile edges, pixel lists,
// work items, per-warp culling regions + item frames, the pixel->tile map); the setup's scratch
// (angles, bin counts, sort buffers) stays with the context.  A context holds at most kCamSlots
// setups besides the current one and at most kCamCacheBytes of slot memory; when the slots are
// full a new camera is set up in the current camera's buffers (the most recently used setup is the
// one dropped: a cyclic set of more views than slots keeps kCamSlots of them cached instead of
// none).  geer_clear_camera_cache frees the slots; a failed allocation frees them and retries.
constexpr int kCamSlots = 16;
constexpr int64_t kCamSlotMaxPixels = 4 << 20;  // larger cameras are not kept (memory)
constexpr size_t kCamCacheBytes = (size_t)1 << 30;
#define GEER_CAM_BUFS(X) \
    X(col_sc) X(row_sc) X(medges_x) X(medges_y) X(dir64) X(pixel_tile) X(pix_list) X(items) X(n_items) X(wcull)
struct CamSlot {
#define GEER_DECL(b) Buf b;
    GEER_CAM_BUFS(GEER_DECL)
#undef GEER_DECL
    bool valid = false, pixel_tile_ok = false;
    FrameConst fc{};
    int max_items = 0;
    uint64_t last_use = 0;
};

struct geer_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    bool timing = false;
    cudaEvent_t ev[6] = {};
    cudaEvent_t ev_hdr = nullptr;  // the 12-byte frame header has reached the host
    // frame state
    FrameConst fc{};
    geer_scene scene{};
    bool have_frame = false;
    bool have_raster = false;
    bool have_stats = false;
    const void *iota_ptr = nullptr;  // gid_iota holds 0..iota_len-1 (buffer pointer / capacity it was written at)
    size_t iota_cap = 0;
    int64_t iota_len = 0;  // a raster ran (also exhaustive forwards, which have no backward)
    int64_t n_entries = 0;  // of the last frame; -1: on the device only (asynchronous frame)
    int64_t cap_entries = 0, cap_rows = 0;  // graph capacity of the asynchronous path (0: not known yet)
    // the last device-level forward, for geer_sync's re-run after an overflow
    float *last_color = nullptr, *last_remaining = nullptr;
    int32_t *last_count = nullptr;
    int max_items = 0;
    CUtensorMap pay_map;  // gather4 map over the payload array
    // K0 cache: the camera setup depends only on the camera and the tile size
    bool cam_valid = false, cam_pixel_tile = false;
    FrameConst cam_fc{};
    CamSlot cam_slots[kCamSlots];
    uint64_t cam_clock = 0;
    bool have_export = false;  // mu_c / depth were recorded by the last forward (graph export)
    const float *fwd_remaining = nullptr;  // remaining written by the last forward (backward input)
    float ms[6] = {};
    unsigned long long *d_counters = nullptr;  // [0] rechecks, [1] evaluated pairs, [2] fix-up pixels, [3] warp-entries, [4] streamed entries, [5] graph entries (K1)
    int *d_err = nullptr;
    int64_t *h_hdr = nullptr;  // pinned: [0] total entries, [1] error code, [2] (Gaussian, tile row) pairs
    // camera buffers
    Buf col_sc, row_sc, medges_x, medges_y, edges_x, edges_y, dir64, theta, phi, minmax, pixel_tile, pixel_tile_sorted,
        pix_iota, pix_list, tile_count, tile_off, item_count, item_off, items, n_items, work, n_work;
    // per-Gaussian buffers
    Buf payload, depth_key, depth_key_sorted, gid_iota, gid_sorted, ranges_ax, flags, mu_c,
        depth;
    // per-entry buffers
    Buf order, tile_ranges, wcull;
    Buf bin_m1, bin_p1, bin_rows, bin_rowstart, bin_segoff, bin_m2, bin_p2;
    // per-pixel buffers
    Buf color, remaining, count_px, n_eval, dl32, fixup;
    // backward
    Buf accum;
    // temp
    Buf temp;
    // host-path staging
    int64_t last_h2d = 0;     // PCIe bytes of the last host-buffer call's inputs
    void *h_stage = nullptr;  // pinned write-combined host staging of the host-buffer entry points' inputs
    size_t h_stage_cap = 0;
    void *h_down = nullptr;   // pinned (cached) host staging of their fp32 outputs
    size_t h_down_cap = 0;
    std::vector<cudaEvent_t> down_evs;
    Buf h64_raw, s32_means, s32_log, s32_quats, s32_op, s32_sh, out64, g64;
    Arena arena;  // caller-owned workspace (geer_set_workspace), if attached
};

namespace {

template <typename T>
T *ensure(Buf &b, size_t count, int *rc) {
    size_t bytes = count * sizeof(T);
    if (bytes == 0) bytes = 16;
    if (bytes > b.cap) {
        if (b.p && b.owned) cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
        b.owned = true;
        if (t_arena && t_arena->base) {  // caller-owned workspace: exact size, 256-B aligned slices
            const size_t off = (t_arena->used + 255) & ~(size_t)255;
            if (off + bytes > t_arena->size) {
                *rc = fail(GEER_ERR_NOMEM, "caller workspace too small: %zu of %zu bytes used, %zu more needed "
                           "(size it with geer_workspace_bytes)", t_arena->used, t_arena->size, bytes);
                return nullptr;
            }
            b.p = t_arena->base + off;
            b.cap = bytes;
            b.owned = false;
            t_arena->used = off + bytes;
            return reinterpret_cast<T *>(b.p);
        }
        size_t want = bytes + bytes / 4;
        cudaError_t e = cudaMalloc(&b.p, want);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            want = bytes;
            e = cudaMalloc(&b.p, want);
        }
        if (e != cudaSuccess) {
            b.p = nullptr;
            *rc = e == cudaErrorMemoryAllocation
                      ? fail(GEER_ERR_NOMEM, "cudaMalloc of %zu bytes failed", bytes)
                      : fail(GEER_ERR_CUDA, "cudaMalloc of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
            return nullptr;
        }
        b.cap = want;
    }
    return reinterpret_cast<T *>(b.p);
}

#define ENSURE(T, buf, n)                       \
    ensure<T>((buf), (size_t)(n), &rc);         \
    if (rc) return rc

void free_buf(Buf &b) {
    if (b.p && b.owned) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    b.owned = true;
}

// Sets the thread's current arena to the context's for the duration of an API call.
struct ArenaScope {
    Arena *prev;
    explicit ArenaScope(Arena *a) : prev(t_arena) { t_arena = a; }
    ~ArenaScope() { t_arena = prev; }
};

int make_frame_const(const geer_camera *cam, const geer_config *cfg, int n_bands, FrameConst *fc) {
    if (!cam || !cfg) return fail(GEER_ERR_INVALID, "camera and config are required");
    if (cam->width <= 0 || cam->height <= 0) return fail(GEER_ERR_INVALID, "image size must be positive");
    if (cam->model < 0 || cam->model > 2) return fail(GEER_ERR_INVALID, "unknown camera model %d", cam->model);
    if (cfg->tile_px <= 0) return fail(GEER_ERR_INVALID, "tile_px must be positive");
    if ((int64_t)cam->width * cam->height >= (int64_t)1 << 31) return fail(GEER_ERR_INVALID, "image too large");
    memset(fc, 0, sizeof(*fc));
    fc->width = cam->width;
    fc->height = cam->height;
    fc->model = cam->model;
    fc->tile_px = cfg->tile_px;
    fc->n_x = (cam->width + cfg->tile_px - 1) / cfg->tile_px;   // association.py:308
    fc->n_y = (cam->height + cfg->tile_px - 1) / cfg->tile_px;  // association.py:309
    if (fc->n_x < 1) fc->n_x = 1;
    if (fc->n_y < 1) fc->n_y = 1;
    if (fc->n_x >= 65535 || fc->n_y >= 65535) return fail(GEER_ERR_INVALID, "too many tiles per axis");
    fc->n_tiles = fc->n_x * fc->n_y;
    fc->n_bands = n_bands;
    fc->cutoff = cfg->support_cutoff ? 1 : 0;
    // per-warp PBF culling is exact only under the support cutoff (renderer.py:103-105)
    fc->cull = (cfg->support_cutoff && !(cfg->flags & GEER_CFG_NO_CULL)) ? 1 : 0;
    fc->exhaustive = (cfg->flags & GEER_CFG_EXHAUSTIVE) ? 1 : 0;
    for (int i = 0; i < 9; ++i) fc->R[i] = cam->rotation[i];
    for (int i = 0; i < 3; ++i) fc->t[i] = cam->translation[i];
    // camera.py:71-74: o = -R^T t
    for (int j = 0; j < 3; ++j)
        fc->origin[j] = -std::fma(cam->rotation[2 * 3 + j], cam->translation[2],
                                  std::fma(cam->rotation[1 * 3 + j], cam->translation[1],
                                           cam->rotation[0 * 3 + j] * cam->translation[0]));  // numpy matmul rounding
    fc->fov_x = cam->fov_x;
    fc->fov_y = cam->fov_y;
    fc->fx = cam->fx;
    fc->fy = cam->fy;
    fc->cx = cam->cx;
    fc->cy = cam->cy;
    for (int i = 0; i < 4; ++i) fc->k[i] = cam->k[i];
    fc->lam = cfg->lam;
    fc->lam2 = cfg->lam * cfg->lam;
    fc->lam2f = (float)fc->lam2;
    fc->cutoff_tol = (float)(1e-6 * fc->lam2 + 1e-7);
    fc->thrk = (float)(kHalfLog2e * fc->lam2);
    fc->thrkc = fc->cutoff ? fc->thrk : INFINITY;
    for (int i = 0; i < 3; ++i) fc->bg[i] = (float)cfg->background[i];
    return GEER_OK;
}

// The entry total of the last frame on the host (an asynchronous frame left it on the device).
int resolve_entries(geer_ctx *c) {
    if (c->n_entries >= 0) return GEER_OK;
    GEER_CUDA(cudaDeviceSynchronize());
    GEER_CUDA(cudaMemcpy(&c->n_entries, c->d_counters + 5, sizeof(int64_t), cudaMemcpyDeviceToHost));
    return GEER_OK;
}

// The item frames follow the per-warp culling regions in the wcull buffer.
ItemFrame *item_frames(geer_ctx *c) {
    return reinterpret_cast<ItemFrame *>(reinterpret_cast<float4 *>(c->wcull.p) + (size_t)c->max_items * 16);
}

// K0: camera setup into ctx buffers (tile CSR + work items).
int camera_setup(geer_ctx *c, bool want_pixel_tile, cudaStream_t st) {
    int rc = 0;
    FrameConst &fc = c->fc;
    const int64_t npx = (int64_t)fc.width * fc.height;
    int32_t *tile_off = ENSURE(int32_t, c->tile_off, fc.n_tiles + 1);
    int32_t *pix_list = ENSURE(int32_t, c->pix_list, npx);
    double *mex = ENSURE(double, c->medges_x, fc.n_x + 1);
    double *mey = ENSURE(double, c->medges_y, fc.n_y + 1);
    if (fc.model == GEER_BEAP) {
        double2 *col = ENSURE(double2, c->col_sc, fc.width);
        double2 *row = ENSURE(double2, c->row_sc, fc.height);
        int32_t *pt = nullptr;
        if (want_pixel_tile) {
            pt = ENSURE(int32_t, c->pixel_tile, npx);
        }
        launch_beap_setup(fc, col, row, mex, mey, tile_off, pix_list, pt, st);
    } else {
        double *dir = ENSURE(double, c->dir64, npx * 3);
        double *th = ENSURE(double, c->theta, npx);
        double *ph = ENSURE(double, c->phi, npx);
        long long *mm = ENSURE(long long, c->minmax, 4);
        double *ex = ENSURE(double, c->edges_x, fc.n_x + 1);
        double *ey = ENSURE(double, c->edges_y, fc.n_y + 1);
        int32_t *pt = ENSURE(int32_t, c->pixel_tile, npx);
        int32_t *pts = ENSURE(int32_t, c->pixel_tile_sorted, npx);
        int32_t *iota = ENSURE(int32_t, c->pix_iota, npx);
        int32_t *tcnt = ENSURE(int32_t, c->tile_count, fc.n_tiles + 1);
        const long long init[4] = {0x7FFFFFFFFFFFFFFFLL, (long long)0x8000000000000000ULL, 0x7FFFFFFFFFFFFFFFLL,
                                   (long long)0x8000000000000000ULL};
        GEER_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, st));
        GEER_CUDA(cudaMemsetAsync(tcnt, 0, sizeof(int32_t) * (fc.n_tiles + 1), st));
        launch_cam_pixels(fc, dir, th, ph, mm, st);
        launch_cam_edges(fc, mm, ex, ey, mex, mey, st);
        launch_cam_bin(fc, th, ph, ex, ey, pt, tcnt, st);
        launch_iota(iota, npx, st);
        int bits = ceil_log2(fc.n_tiles);
        size_t tb = sort_pixels_temp_bytes(npx, bits);
        size_t sb = scan_i32_temp_bytes(fc.n_tiles + 1);
        void *tmp = ENSURE(char, c->temp, tb > sb ? tb : sb);
        sort_pixels(tmp, tb, pt, pts, iota, pix_list, npx, bits, st);
        exclusive_scan_i32(tmp, sb, tcnt, tile_off, fc.n_tiles + 1, st);
    }
    int32_t *icnt = ENSURE(int32_t, c->item_count, fc.n_tiles);
    int32_t *ioff = ENSURE(int32_t, c->item_off, fc.n_tiles);
    c->max_items = (int)(fc.n_tiles + (npx + kRasterThreads - 1) / kRasterThreads);
    int4 *items = ENSURE(int4, c->items, c->max_items);
    int32_t *nit = ENSURE(int32_t, c->n_items, 1);
    launch_items(fc.n_tiles, tile_off, icnt, st);
    size_t sb = scan_i32_temp_bytes(fc.n_tiles);
    void *tmp = ENSURE(char, c->temp, sb);
    exclusive_scan_i32(tmp, sb, icnt, ioff, fc.n_tiles, st);
    launch_item_fill(fc.n_tiles, tile_off, ioff, items, nit, st);
    // per item: 8 warps x (patch, cone), then the item frames
    float4 *wc = ENSURE(float4, c->wcull, (size_t)c->max_items * (16 + sizeof(ItemFrame) / 16));
    launch_warp_cull(fc, c->max_items, items, nit, (const int32_t *)c->pix_list.p, (const double2 *)c->col_sc.p,
                     (const double2 *)c->row_sc.p, (const double *)c->dir64.p, wc, item_frames(c), st);
    return GEER_OK;
}

// Whether the K0 outputs in the context are those of this frame's camera (same model, size, tiling,
// pose and intrinsics, compared bit for bit).
bool same_camera(const FrameConst &a, const FrameConst &b) {
    return a.width == b.width && a.height == b.height && a.model == b.model && a.tile_px == b.tile_px &&
           memcmp(a.R, b.R, sizeof(a.R)) == 0 && memcmp(&a.fov_x, &b.fov_x, sizeof(double) * 10) == 0;
}
bool camera_cached(const geer_ctx *c, bool want_pixel_tile) {
    if (!c->cam_valid || (want_pixel_tile && !c->cam_pixel_tile)) return false;
    return same_camera(c->cam_fc, c->fc);
}
// Exchange the context's camera setup with slot s (buffers by pointer, no copies).
void swap_camera(geer_ctx *c, CamSlot &s) {
#define GEER_SWAP(b) std::swap(c->b, s.b);
    GEER_CAM_BUFS(GEER_SWAP)
#undef GEER_SWAP
    std::swap(c->cam_valid, s.valid);
    std::swap(c->cam_pixel_tile, s.pixel_tile_ok);
    std::swap(c->cam_fc, s.fc);
    std::swap(c->max_items, s.max_items);
}
size_t slot_bytes(const CamSlot &sl) {
    size_t t = 0;
#define GEER_SUM(b) t += sl.b.cap;
    GEER_CAM_BUFS(GEER_SUM)
#undef GEER_SUM
    return t;
}
size_t current_camera_bytes(const geer_ctx *c) {
    size_t t = 0;
#define GEER_SUM(b) t += c->b.cap;
    GEER_CAM_BUFS(GEER_SUM)
#undef GEER_SUM
    return t;
}
void clear_camera_cache(geer_ctx *c) {
    for (CamSlot &sl : c->cam_slots) {
#define GEER_FREE(b) free_buf(sl.b);
        GEER_CAM_BUFS(GEER_FREE)
#undef GEER_FREE
        sl.valid = sl.pixel_tile_ok = false;
        sl.max_items = 0;
    }
}

// Every workspace buffer of a context (and its cached camera setups) released; state that points
// into them reset.
void free_all_buffers(geer_ctx *c) {
    Buf *bufs[] = {&c->col_sc, &c->row_sc, &c->medges_x, &c->medges_y, &c->edges_x, &c->edges_y, &c->dir64,
                   &c->theta, &c->phi, &c->minmax, &c->pixel_tile, &c->pixel_tile_sorted, &c->pix_iota, &c->pix_list,
                   &c->tile_count, &c->tile_off, &c->item_count, &c->item_off, &c->items, &c->n_items, &c->work, &c->n_work, &c->payload,
                   &c->depth_key, &c->depth_key_sorted, &c->gid_iota, &c->gid_sorted,
                   &c->ranges_ax, &c->flags, &c->mu_c, &c->depth,
                   &c->order, &c->tile_ranges, &c->wcull,
                   &c->bin_m1, &c->bin_p1, &c->bin_rows, &c->bin_rowstart, &c->bin_segoff, &c->bin_m2, &c->bin_p2, &c->color, &c->remaining, &c->count_px, &c->n_eval, &c->dl32, &c->fixup,
                   &c->accum, &c->temp, &c->h64_raw,
                   &c->s32_means, &c->s32_log, &c->s32_quats, &c->s32_op, &c->s32_sh, &c->out64, &c->g64};
    for (Buf *b : bufs) free_buf(*b);
    clear_camera_cache(c);
    c->cam_valid = c->cam_pixel_tile = false;
    c->have_frame = c->have_raster = c->have_stats = c->have_export = false;
    c->iota_ptr = nullptr;
    c->iota_cap = 0;
    c->iota_len = 0;
    c->cap_entries = c->cap_rows = 0;
    c->fwd_remaining = nullptr;
}

// Make the context's camera setup the one of c->fc: from a slot if it is cached there (the current
// setup moves into that slot), else rebuilt by camera_setup - after parking the current setup in a
// free slot when there is one and the byte budget allows, otherwise over the current setup.
int select_camera(geer_ctx *c, bool want_pixel_tile, cudaStream_t st) {
    if (camera_cached(c, want_pixel_tile)) return GEER_OK;
    const FrameConst &fc = c->fc;
    const bool small = (int64_t)fc.width * fc.height <= kCamSlotMaxPixels;
    int hit = -1, free_slot = -1;
    size_t used = 0;
    for (int i = 0; i < kCamSlots; ++i) {
        const CamSlot &sl = c->cam_slots[i];
        if (sl.valid && (!want_pixel_tile || sl.pixel_tile_ok) && same_camera(sl.fc, fc)) hit = i;
        if (!sl.valid && free_slot < 0) free_slot = i;
        used += slot_bytes(sl);
    }
    if (hit >= 0) {
        swap_camera(c, c->cam_slots[hit]);  // the previous camera stays cached in that slot
        c->cam_slots[hit].last_use = ++c->cam_clock;
        return GEER_OK;
    }
    const bool park = small && c->cam_valid && free_slot >= 0 && !c->arena.base &&
                      (int64_t)c->cam_fc.width * c->cam_fc.height <= kCamSlotMaxPixels &&
                      used + current_camera_bytes(c) <= kCamCacheBytes;
    if (park) {
        CamSlot &sl = c->cam_slots[free_slot];
        swap_camera(c, sl);  // sl takes the current setup; the context gets the slot's (empty) buffers
        sl.last_use = ++c->cam_clock;
    }
    c->cam_valid = false;
    int rc = camera_setup(c, want_pixel_tile, st);
    if (rc == GEER_ERR_NOMEM) {  // give the cached setups' memory back and try once more
        cudaGetLastError();
        clear_camera_cache(c);
        rc = camera_setup(c, want_pixel_tile, st);
    }
    if (rc) return rc;
    c->cam_valid = true;
    c->cam_pixel_tile = want_pixel_tile || fc.model != GEER_BEAP;
    c->cam_fc = fc;
    return GEER_OK;
}

// Largest CUB temporary of a frame (depth sort, the two binning scans, the camera setup's scans and
// pixel sort).
size_t frame_temp_bytes(const FrameConst &fc, int64_t n, int64_t cap_e, int64_t cap_r) {
    const int64_t npx = (int64_t)fc.width * fc.height;
    size_t t = sort_depth_temp_bytes(lmax(n, 1));
    const BinPlan bp = bin_plan(lmax(n, 1), fc.n_x, fc.n_y, lmax(cap_e, 1), lmax(cap_r, 1));
    t = t > bp.temp_bytes ? t : bp.temp_bytes;
    const size_t sc = scan_i32_temp_bytes(fc.n_tiles + 1);
    t = t > sc ? t : sc;
    if (fc.model != GEER_BEAP) {
        const size_t sp = sort_pixels_temp_bytes(npx, ceil_log2(fc.n_tiles));
        t = t > sp ? t : sp;
    }
    return t;
}

// Device bytes of the device-level path (geer_forward + geer_backward) for one camera: the same
// buffers camera_setup / run_forward / run_backward ensure, each a 256-B aligned slice.
size_t workspace_estimate(const FrameConst &fc, int64_t n, int64_t cap_e, int64_t cap_r) {
    const int64_t npx = (int64_t)fc.width * fc.height, nt = fc.n_tiles;
    const int64_t max_items = nt + (npx + kRasterThreads - 1) / kRasterThreads;
    size_t total = 0;
    auto add = [&](int64_t bytes) { total += (size_t)((lmax(bytes, 16) + 255) & ~(int64_t)255); };
    // camera setup
    add((nt + 1) * 4);                                   // tile_off
    add(npx * 4);                                        // pix_list
    add((fc.n_x + 1) * 8);                               // medges_x
    add((fc.n_y + 1) * 8);                               // medges_y
    if (fc.model == GEER_BEAP) {
        add(fc.width * 16);                              // col_sc
        add(fc.height * 16);                             // row_sc
    } else {
        add(npx * 24);                                   // dir64
        add(npx * 8);                                    // theta
        add(npx * 8);                                    // phi
        add(32);                                         // minmax
        add((fc.n_x + 1) * 8);                           // edges_x
        add((fc.n_y + 1) * 8);                           // edges_y
        add(npx * 4);                                    // pixel_tile
        add(npx * 4);                                    // pixel_tile_sorted
        add(npx * 4);                                    // pix_iota
        add((nt + 1) * 4);                               // tile_count
    }
    add(nt * 4);                                         // item_count
    add(nt * 4);                                         // item_off
    add(max_items * 16);                                 // items
    add(4);                                              // n_items
    add(max_items * (16 + (int64_t)sizeof(ItemFrame) / 16) * 16);  // wcull + item frames
    // per Gaussian
    add(n * (int64_t)sizeof(Payload));
    add(n * 4);                                          // depth keys
    add(n * 4);                                          // sorted depth keys
    add(n * 4);                                          // gid iota
    add(n * 4);                                          // sorted gids
    add(n * (int64_t)sizeof(AxisRanges));
    add(2 * n);                                          // flags
    add((nt + 1) * 4);                                   // tile ranges
    // per entry (the capacity) and the binning matrices
    const BinPlan bp = bin_plan(lmax(n, 1), fc.n_x, fc.n_y, lmax(cap_e, 1), lmax(cap_r, 1));
    add((bp.m1_len + 1) * 4);
    add((bp.m1_len + 1) * 4);
    add((bp.rows_cap + 1) * 8);
    add((fc.n_y + 1) * 4);
    add((fc.n_y + 1) * 4);
    add((bp.m2_len + 1) * 4);
    add((bp.m2_len + 1) * 4);
    add((lmax(cap_e, 1) + 1) * 4);                       // order
    add(max_items * 16);                                 // work
    add(4 * order_items_ints());                         // n_work (+ work-order scratch)
    // per pixel
    add(npx * 4);                                        // n_eval
    add(npx * 4);                                        // fix-up list
    // backward
    add(n * 64);                                         // accumulators
    add((int64_t)frame_temp_bytes(fc, n, cap_e, cap_r)); // CUB temp
    return total;
}

// Full association (+ raster when color != null) for the scene in c->scene.
int run_forward(geer_ctx *c, float *color, float *remaining, int32_t *count, bool want_export, cudaStream_t st,
                bool allow_async = false) {
    int rc = 0;
    FrameConst &fc = c->fc;
    const geer_scene &sc = c->scene;
    const int64_t n = sc.n;
    const int64_t npx = (int64_t)fc.width * fc.height;
    c->have_frame = false;
    c->have_raster = false;
    c->have_stats = false;
    c->have_export = false;
    if (c->timing) GEER_CUDA(cudaEventRecord(c->ev[0], st));
    GEER_CUDA(cudaMemsetAsync(c->d_counters, 0, 7 * sizeof(unsigned long long), st));
    GEER_CUDA(cudaMemsetAsync(c->d_err, 0, sizeof(int), st));
    rc = select_camera(c, want_export, st);
    if (rc) return rc;

    // ---- K1 preprocess
    Payload *payload = ENSURE(Payload, c->payload, n);
    uint32_t *dkey = ENSURE(uint32_t, c->depth_key, n);
    uint32_t *dkey_s = ENSURE(uint32_t, c->depth_key_sorted, n);
    int32_t *giota = ENSURE(int32_t, c->gid_iota, n);
    int32_t *gsorted = ENSURE(int32_t, c->gid_sorted, n);
    AxisRanges *ar = ENSURE(AxisRanges, c->ranges_ax, n);
    uint8_t *flags = ENSURE(uint8_t, c->flags, 2 * n);  // [0, n): association bits, [n, 2n): payload bits
    double *mu = nullptr, *dep = nullptr;
    if (want_export) {
        mu = ENSURE(double, c->mu_c, n * 3);
        dep = ENSURE(double, c->depth, n);
    }
    int32_t *ranges = ENSURE(int32_t, c->tile_ranges, fc.n_tiles + 1);
    rc = make_row_map(&c->pay_map, payload, n, (int)sizeof(Payload));
    if (rc) return rc;
    launch_preprocess(fc, sc, (const double *)c->medges_x.p, (const double *)c->medges_y.p, payload, dkey, ar,
                      flags, mu, dep, c->d_err, c->d_counters + 5, st);
    if (c->timing) GEER_CUDA(cudaEventRecord(c->ev[1], st));

    // ---- dup: depth order
    // Asynchronous frame: the graph buffers are sized by the context's capacity (learned from earlier
    // frames) and the frame runs to the end without the host; a total above capacity is flagged on
    // the device (k_check_capacity) and turns the rest of the association into no-ops (geer_sync
    // re-runs such a frame).  First frame / export / exhaustive: the 24-byte header (entry total,
    // (Gaussian, tile row) pairs, error flag) is read back right after K1, with the depth sort queued
    // before the host waits, so the GPU never idles on the round trip.
    const bool async = allow_async && c->cap_entries > 0 && !want_export && !fc.exhaustive;
    int64_t total = 0, rows = 0;
    if (!async) {
        GEER_CUDA(cudaMemcpyAsync(&c->h_hdr[0], c->d_counters + 5, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        GEER_CUDA(cudaMemcpyAsync(&c->h_hdr[1], c->d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
        GEER_CUDA(cudaMemcpyAsync(&c->h_hdr[2], c->d_counters + 6, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        GEER_CUDA(cudaEventRecord(c->ev_hdr, st));
    }
    if (n > 0) {
        // gid values 0..n-1 stay valid while the buffer is not reallocated (a growth changes its capacity)
        if (c->iota_ptr != giota || c->iota_cap != c->gid_iota.cap || c->iota_len < n) {
            launch_iota(giota, n, st);
            c->iota_ptr = giota;
            c->iota_cap = c->gid_iota.cap;
            c->iota_len = n;
        }
        size_t b1 = sort_depth_temp_bytes(n);
        // (the temp buffer is sized once for every user of the frame: a caller workspace is not regrown)
        void *tmp = ENSURE(char, c->temp, lmax((int64_t)b1, (int64_t)frame_temp_bytes(fc, n, c->cap_entries, c->cap_rows)));
        sort_depth(tmp, b1, dkey, dkey_s, giota, gsorted, n, st);
    }
    if (!async) {
        GEER_CUDA(cudaEventSynchronize(c->ev_hdr));
        int err = (int)(c->h_hdr[1] & 0xFFFFFFFF);
        if (err == GEER_ERR_NOT_PD) return fail(GEER_ERR_NOT_PD, "view covariance must be positive definite");
        if (err == GEER_ERR_NOT_SYMMETRIC) return fail(GEER_ERR_NOT_SYMMETRIC, "view covariance must be symmetric");
        if (err) return fail(GEER_ERR_INVALID, "preprocess error %d", err);
    }
    if (fc.exhaustive) {  // every tile composites all kept Gaussians: no emit, no tile sort
        int32_t *r2 = ENSURE(int32_t, c->tile_ranges, fc.n_tiles + 1);
        launch_exhaustive_ranges((const uint8_t *)c->flags.p, n, r2, st);
        int32_t *nwork = ENSURE(int32_t, c->n_work, order_items_ints());
        GEER_CUDA(cudaMemcpyAsync(nwork, c->n_items.p, sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        GEER_CUDA(cudaMemsetAsync(nwork + 1, 0, sizeof(int32_t), st));
        if (c->timing) {
            GEER_CUDA(cudaEventRecord(c->ev[2], st));
            GEER_CUDA(cudaEventRecord(c->ev[3], st));
        }
        c->n_entries = 0;
        if (color) {
            int32_t *ne = ENSURE(int32_t, c->n_eval, npx);
            int32_t *fix = ENSURE(int32_t, c->fixup, npx);
            launch_forward(fc, sc, c->max_items, (const int4 *)c->items.p, nwork, (const int32_t *)c->pix_list.p,
                           (const double2 *)c->col_sc.p, (const double2 *)c->row_sc.p, (const double *)c->dir64.p,
                           r2, (const uint32_t *)gsorted, payload, c->pay_map, (const float4 *)c->wcull.p, item_frames(c), color, remaining, count, ne,
                           c->d_counters, fix, st);
            c->have_stats = true;
        }
        GEER_CUDA(cudaGetLastError());
        return GEER_OK;  // forward only: have_frame / have_raster stay false
    }
    if (async) {
        total = c->cap_entries;
        rows = c->cap_rows;
        c->n_entries = -1;
        launch_check_capacity(c->d_counters + 5, c->cap_entries, c->cap_rows, c->d_err, st);
    } else {
        total = c->h_hdr[0];
        rows = c->h_hdr[2];
        if (total >= ((int64_t)1 << 31) - 1)
            return fail(GEER_ERR_NOMEM, "render graph has %lld entries (limit 2^31)", (long long)total);
        c->n_entries = total;
        // capacity of the following asynchronous frames (grow-only, 25 % headroom); the buffers are
        // sized by it from this frame on, so the asynchronous frames never regrow them
        c->cap_entries = lmax(c->cap_entries, lmin(total + total / 4 + 4096, ((int64_t)1 << 31) - 2));
        c->cap_rows = lmax(c->cap_rows, rows + rows / 4 + 1024);
        total = c->cap_entries;
        rows = c->cap_rows;
    }
    // ---- sort: per-tile lists (stable in depth order) and their ranges, then the raster work order
    {
        const BinPlan bp = bin_plan(n, fc.n_x, fc.n_y, total, rows);
        uint32_t *m1 = ENSURE(uint32_t, c->bin_m1, bp.m1_len + 1);
        uint32_t *p1 = ENSURE(uint32_t, c->bin_p1, bp.m1_len + 1);
        uint2 *brows = ENSURE(uint2, c->bin_rows, bp.rows_cap + 1);
        int32_t *rst = ENSURE(int32_t, c->bin_rowstart, fc.n_y + 1);
        int32_t *sof = ENSURE(int32_t, c->bin_segoff, fc.n_y + 1);
        uint32_t *m2 = ENSURE(uint32_t, c->bin_m2, bp.m2_len + 1);
        uint32_t *p2 = ENSURE(uint32_t, c->bin_p2, bp.m2_len + 1);
        void *tmp = ENSURE(char, c->temp, bp.temp_bytes);
        uint32_t *order = ENSURE(uint32_t, c->order, total + 1);
        if (c->timing) GEER_CUDA(cudaEventRecord(c->ev[2], st));
        rc = bin_tiles(bp, gsorted, ar, n, fc.n_x, fc.n_y, c->d_counters + 5, c->d_err, m1, p1, brows, rst, sof, m2, p2,
                       tmp, order, ranges, st);
        if (rc) return fail(rc, "tile binning failed: %s", cudaGetErrorString(cudaGetLastError()));
        int4 *work = ENSURE(int4, c->work, c->max_items);
        int32_t *nwork = ENSURE(int32_t, c->n_work, order_items_ints());
        order_items((const int4 *)c->items.p, (const int32_t *)c->n_items.p, ranges, c->max_items, work, nwork, st);
        if (c->timing) GEER_CUDA(cudaEventRecord(c->ev[3], st));
    }
    c->have_frame = true;
    c->have_export = want_export;

    // ---- render
    if (color) {
        int32_t *ne = ENSURE(int32_t, c->n_eval, npx);
        int32_t *fix = ENSURE(int32_t, c->fixup, npx);
        launch_forward(fc, sc, c->max_items, (const int4 *)c->work.p, (const int32_t *)c->n_work.p,
                       (const int32_t *)c->pix_list.p, (const double2 *)c->col_sc.p, (const double2 *)c->row_sc.p,
                       (const double *)c->dir64.p, ranges, (const uint32_t *)c->order.p, payload, c->pay_map, (const float4 *)c->wcull.p, item_frames(c), color, remaining, count, ne,
                       c->d_counters, fix, st);
        c->fwd_remaining = remaining;
        c->have_raster = c->have_stats = true;
    }
    if (c->timing) {
        GEER_CUDA(cudaEventRecord(c->ev[4], st));
        GEER_CUDA(cudaEventSynchronize(c->ev[4]));
        cudaEventElapsedTime(&c->ms[0], c->ev[0], c->ev[1]);
        cudaEventElapsedTime(&c->ms[1], c->ev[1], c->ev[2]);
        cudaEventElapsedTime(&c->ms[2], c->ev[2], c->ev[3]);
        cudaEventElapsedTime(&c->ms[3], c->ev[3], c->ev[4]);
        cudaEventElapsedTime(&c->ms[4], c->ev[0], c->ev[4]);
    }
    GEER_CUDA(cudaGetLastError());
    return GEER_OK;
}

int run_backward(geer_ctx *c, const float *dl_dimage, bool f64_out, void *const *gout, int accumulate, cudaStream_t st) {
    int rc = 0;
    if (!c->have_raster) return fail(GEER_ERR_STATE, "geer_backward needs a preceding geer_forward with a raster");
    FrameConst &fc = c->fc;
    const geer_scene &sc = c->scene;
    if (c->timing) GEER_CUDA(cudaEventRecord(c->ev[0], st));
    float *accum = ENSURE(float, c->accum, sc.n * 16);
    if (sc.n > 0) GEER_CUDA(cudaMemsetAsync(accum, 0, sizeof(float) * 16 * sc.n, st));
    launch_backward(fc, sc, c->max_items, (const int4 *)c->work.p, (const int32_t *)c->n_work.p,
                    (const int32_t *)c->pix_list.p, (const double2 *)c->col_sc.p, (const double2 *)c->row_sc.p,
                    (const double *)c->dir64.p, (const int32_t *)c->tile_ranges.p, (const uint32_t *)c->order.p,
                    c->pay_map, (const float4 *)c->wcull.p, item_frames(c),
                    c->fwd_remaining, (const int32_t *)c->n_eval.p,
                    dl_dimage, accum, st);
    if (f64_out)
        launch_finalize<double>(fc, sc, (const float4 *)accum, (const uint8_t *)c->flags.p + sc.n, (double *)gout[0], (double *)gout[1],
                                (double *)gout[2], (double *)gout[3], (double *)gout[4], accumulate, st);
    else
        launch_finalize<float>(fc, sc, (const float4 *)accum, (const uint8_t *)c->flags.p + sc.n, (float *)gout[0], (float *)gout[1],
                               (float *)gout[2], (float *)gout[3], (float *)gout[4], accumulate, st);
    if (c->timing) {
        GEER_CUDA(cudaEventRecord(c->ev[1], st));
        GEER_CUDA(cudaEventSynchronize(c->ev[1]));
        cudaEventElapsedTime(&c->ms[5], c->ev[0], c->ev[1]);
    }
    GEER_CUDA(cudaGetLastError());
    return GEER_OK;
}

int check_scene_dev(const geer_scene *s) {
    if (!s) return fail(GEER_ERR_INVALID, "scene is required");
    if (s->n < 0) return fail(GEER_ERR_INVALID, "negative Gaussian count");
    if (s->n >= ((int64_t)1 << 31)) return fail(GEER_ERR_INVALID, "too many Gaussians");
    // renderer.py:66-68 uses sh_basis(d)[:n_bands]: any 1..16 bands evaluate, more cannot
    if (s->n_bands < 1 || s->n_bands > 16)
        return fail(GEER_ERR_INVALID, "unsupported SH band count %d; at most 16 bands (degree 3)", s->n_bands);
    if (s->n > 0 && (!s->means || !s->log_scales || !s->quats || !s->opacity_logits || !s->sh))
        return fail(GEER_ERR_INVALID, "scene pointers must be non-null");
    return GEER_OK;
}

// Copy a host f64 scene into device fp32 buffers held by the context.
// A grow-only pinned host buffer (write-combined: written by the host, read only by DMA).
int ensure_pinned(void *&p, size_t &cap, size_t need, bool write_combined, cudaStream_t st) {
    if (cap >= need) return GEER_OK;
    GEER_CUDA(cudaStreamSynchronize(st));  // (copies from the old buffer may be in flight)
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t bytes = need + need / 8;
    if (cudaHostAlloc(&p, bytes, write_combined ? cudaHostAllocWriteCombined : cudaHostAllocDefault) != cudaSuccess) {
        p = nullptr;
        cudaGetLastError();
        return fail(GEER_ERR_NOMEM, "pinned staging allocation of %zu bytes failed", bytes);
    }
    cap = bytes;
    return GEER_OK;
}

int upload_host_scene(geer_ctx *c, const geer_host_scene *hs, cudaStream_t st) {
    int rc = 0;
    if (!hs) return fail(GEER_ERR_INVALID, "scene is required");
    const int64_t n = hs->n;
    if (n < 0 || n >= ((int64_t)1 << 31)) return fail(GEER_ERR_INVALID, "bad Gaussian count");
    c->last_h2d = 0;
    const int64_t nsh = n * hs->n_bands * 3;
    float *m = ENSURE(float, c->s32_means, n * 3);
    float *l = ENSURE(float, c->s32_log, n * 3);
    float *q = ENSURE(float, c->s32_quats, n * 4);
    float *op = ENSURE(float, c->s32_op, n);
    float *sh = ENSURE(float, c->s32_sh, nsh);
    if (n > 0) {
        // fp64 -> fp32 on the host cores, overlapped with the DMA of the finished chunks (geer_host.cu)
        const HostSeg segs[5] = {{hs->means, n * 3, m},
                                 {hs->log_scales, n * 3, l},
                                 {hs->quats, n * 4, q},
                                 {hs->opacity_logits, n, op},
                                 {hs->sh, nsh, sh}};
        rc = ensure_pinned(c->h_stage, c->h_stage_cap, sizeof(float) * (size_t)(n * 11 + nsh), true, st);
        if (rc) return rc;
        const int64_t raw = raw_upload_elems(n * 11 + nsh);
        double *raw_dev = nullptr;
        if (raw > 0) raw_dev = ENSURE(double, c->h64_raw, raw);
        GEER_CUDA(upload_narrowed(segs, 5, (float *)c->h_stage, raw_dev, raw, st, &c->last_h2d));
    }
    geer_scene s;
    s.n = n;
    s.n_bands = hs->n_bands;
    s.pad_ = 0;
    s.means = m;
    s.log_scales = l;
    s.quats = q;
    s.opacity_logits = op;
    s.sh = sh;
    rc = check_scene_dev(&s);
    if (rc) return rc;
    c->scene = s;
    return GEER_OK;
}

}  // namespace

// =============================================================================== C ABI

extern "C" {

int geer_abi_version(void) { return GEER_ABI_VERSION; }

const char *geer_last_error(void) { return g_last_error.c_str(); }

geer_ctx *geer_create(int device) {
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        fail(GEER_ERR_CUDA, "cudaSetDevice(%d) failed", device);
        return nullptr;
    }
    geer_ctx *c = new geer_ctx();
    c->device = device;
    bool ok = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) == cudaSuccess;
    for (int i = 0; i < 6 && ok; ++i) ok = cudaEventCreate(&c->ev[i]) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&c->ev_hdr, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaMalloc(&c->d_counters, 7 * sizeof(unsigned long long)) == cudaSuccess;
    ok = ok && cudaMalloc(&c->d_err, 8 * sizeof(int)) == cudaSuccess;  // frame error, sticky overflow, maxima
    ok = ok && cudaMemset(c->d_err, 0, 8 * sizeof(int)) == cudaSuccess;
    ok = ok && cudaMallocHost(&c->h_hdr, 3 * sizeof(int64_t)) == cudaSuccess;
    if (!ok) {
        fail(GEER_ERR_CUDA, "context creation failed: %s", cudaGetErrorString(cudaGetLastError()));
        geer_destroy(c);
        return nullptr;
    }
    return c;
}

void geer_destroy(geer_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->own_stream) cudaStreamSynchronize(c->own_stream);
    free_all_buffers(c);
    for (int i = 0; i < 6; ++i)
        if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    if (c->ev_hdr) cudaEventDestroy(c->ev_hdr);
    if (c->d_counters) cudaFree(c->d_counters);
    if (c->d_err) cudaFree(c->d_err);
    if (c->h_hdr) cudaFreeHost(c->h_hdr);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->h_down) cudaFreeHost(c->h_down);
    for (cudaEvent_t e : c->down_evs) cudaEventDestroy(e);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
}

size_t geer_workspace_bytes(geer_ctx *c, int64_t n, int32_t n_bands, const geer_camera *camera,
                            const geer_config *config, int64_t max_entries) {
    FrameConst fc;
    if (make_frame_const(camera, config, n_bands, &fc)) return 0;
    if (n < 0) {
        fail(GEER_ERR_INVALID, "negative Gaussian count");
        return 0;
    }
    int64_t cap_e = max_entries, cap_r = max_entries;
    if (cap_e <= 0) {  // the context's learned capacity, else a generous default (24 entries per Gaussian)
        cap_e = c && c->cap_entries > 0 ? c->cap_entries : 24 * n + 4096;
        cap_r = c && c->cap_rows > 0 ? c->cap_rows : cap_e;
    } else {
        cap_e = lmin(cap_e + cap_e / 4 + 4096, ((int64_t)1 << 31) - 2);  // (the capacity the frame will keep)
        cap_r = cap_e;
    }
    return workspace_estimate(fc, n, cap_e, cap_r);
}

int geer_set_workspace(geer_ctx *c, void *ptr, size_t bytes) {
    if (!c) return fail(GEER_ERR_INVALID, "null context");
    cudaSetDevice(c->device);
    GEER_CUDA(cudaDeviceSynchronize());  // (queued frames may still use the current buffers)
    free_all_buffers(c);                 // library-owned memory back; slices of a previous workspace dropped
    c->arena = Arena{};
    if (ptr) {
        if (bytes < 4096) return fail(GEER_ERR_INVALID, "workspace of %zu bytes is too small", bytes);
        c->arena.base = reinterpret_cast<char *>(ptr);
        c->arena.size = bytes;
    }
    return GEER_OK;
}

int geer_workspace_used(geer_ctx *c, size_t *used) {
    if (!c || !used) return fail(GEER_ERR_INVALID, "null argument");
    *used = c->arena.used;
    return GEER_OK;
}

int geer_clear_camera_cache(geer_ctx *c) {
    if (!c) return fail(GEER_ERR_INVALID, "null context");
    cudaSetDevice(c->device);
    GEER_CUDA(cudaDeviceSynchronize());  // (slot buffers may still be read by queued frames)
    clear_camera_cache(c);
    return GEER_OK;
}

int geer_set_timing(geer_ctx *c, int enable) {
    if (!c) return fail(GEER_ERR_INVALID, "null context");
    c->timing = enable != 0;
    return GEER_OK;
}

int geer_forward(geer_ctx *c, const geer_scene *scene, const geer_camera *camera, const geer_config *config,
                 float *color, float *remaining, int32_t *count, void *stream) {
    if (!c) return fail(GEER_ERR_INVALID, "null context");
    ArenaScope arena_scope(&c->arena);
    int rc = check_scene_dev(scene);
    if (rc) return rc;
    if (!color || !remaining || !count) return fail(GEER_ERR_INVALID, "output buffers must be non-null");
    rc = make_frame_const(camera, config, scene->n_bands, &c->fc);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    c->scene = *scene;
    if (scene->n == 0) {
        // renderer.py:131-138: empty scene renders the background
        int32_t *ne = ensure<int32_t>(c->n_eval, (size_t)c->fc.width * c->fc.height, &rc);
        if (rc) return rc;
        launch_fill_background(c->fc, color, remaining, count, ne, st);
        c->have_frame = false;
        c->have_raster = false;
        c->have_stats = false;
        c->n_entries = 0;
        GEER_CUDA(cudaGetLastError());
        return GEER_OK;
    }
    c->last_color = color;
    c->last_remaining = remaining;
    c->last_count = count;
    return run_forward(c, color, remaining, count, false, st, true);
}

int geer_sync(geer_ctx *c, void *stream) {
    if (!c) return fail(GEER_ERR_INVALID, "null context");
    ArenaScope arena_scope(&c->arena);
    cudaStream_t st = (cudaStream_t)stream;
    GEER_CUDA(cudaStreamSynchronize(st));
    int status[8];
    GEER_CUDA(cudaMemcpy(status, c->d_err, sizeof(status), cudaMemcpyDeviceToHost));
    const int err = status[0];
    if (err == GEER_ERR_NOT_PD) return fail(GEER_ERR_NOT_PD, "view covariance must be positive definite");
    if (err == GEER_ERR_NOT_SYMMETRIC) return fail(GEER_ERR_NOT_SYMMETRIC, "view covariance must be symmetric");
    if (err && err != GEER_ERR_OVERFLOW) return fail(GEER_ERR_INVALID, "preprocess error %d", err);
    if (status[1]) {  // a frame since the last sync outgrew the capacity: grow it (25 % headroom)
        int64_t mx[2];
        memcpy(mx, status + 2, sizeof(mx));
        c->cap_entries = lmax(c->cap_entries, lmin(mx[0] + mx[0] / 4 + 4096, ((int64_t)1 << 31) - 2));
        c->cap_rows = lmax(c->cap_rows, mx[1] + mx[1] / 4 + 1024);
        GEER_CUDA(cudaMemset(c->d_err + 1, 0, 7 * sizeof(int)));
        if (err == GEER_ERR_OVERFLOW) {  // the last frame itself: render it again
            int rc = run_forward(c, c->last_color, c->last_remaining, c->last_count, false, st);
            if (rc) return rc;
            GEER_CUDA(cudaStreamSynchronize(st));
            GEER_CUDA(cudaMemcpy(status, c->d_err, sizeof(int), cudaMemcpyDeviceToHost));
            if (status[0]) return fail(GEER_ERR_INVALID, "frame error %d after the re-run", status[0]);
        }
        if (c->n_entries < 0 && c->have_frame)
            GEER_CUDA(cudaMemcpy(&c->n_entries, c->d_counters + 5, sizeof(int64_t), cudaMemcpyDeviceToHost));
        return fail(GEER_ERR_OVERFLOW, "a frame outgrew the graph capacity (the last frame has been re-rendered)");
    }
    if (c->n_entries < 0 && c->have_frame)
        GEER_CUDA(cudaMemcpy(&c->n_entries, c->d_counters + 5, sizeof(int64_t), cudaMemcpyDeviceToHost));
    return GEER_OK;
}

int geer_backward(geer_ctx *c, const float *dl_dimage, const geer_grads *grads, int accumulate, void *stream) {
    if (!c) return fail(GEER_ERR_INVALID, "null context");
    ArenaScope arena_scope(&c->arena);
    if (!grads || !dl_dimage) return fail(GEER_ERR_INVALID, "dl_dimage and grads are required");
    cudaStream_t st = (cudaStream_t)stream;
    if (c->scene.n == 0) return GEER_OK;  // renderer.py:248-249
    void *g[5] = {grads->dmeans, grads->dlog_scales, grads->dquats, grads->dopacities, grads->dsh};
    for (int i = 0; i < 5; ++i)
        if (!g[i]) return fail(GEER_ERR_INVALID, "gradient pointers must be non-null");
    return run_backward(c, dl_dimage, false, g, accumulate & (GEER_ACCUMULATE | GEER_OPACITY_LOGIT), st);
}

int geer_frame_stats(geer_ctx *c, geer_stats *out) {
    if (!c || !out) return fail(GEER_ERR_INVALID, "null argument");
    memset(out, 0, sizeof(*out));
    int rc0 = resolve_entries(c);
    if (rc0) return rc0;
    out->n_gaussians = c->scene.n;
    out->n_entries = c->n_entries;
    out->n_tiles = c->fc.n_tiles;
    if (c->have_stats) {
        cudaStream_t st = c->own_stream;
        GEER_CUDA(cudaDeviceSynchronize());
        GEER_CUDA(cudaMemsetAsync(c->d_counters + 1, 0, sizeof(unsigned long long), st));
        launch_sum_i32((const int32_t *)c->n_eval.p, (int64_t)c->fc.width * c->fc.height, c->d_counters + 1, st);
        unsigned long long h[5];
        int32_t nit = 0;
        GEER_CUDA(cudaMemcpyAsync(h, c->d_counters, sizeof(h), cudaMemcpyDeviceToHost, st));
        GEER_CUDA(cudaMemcpyAsync(&nit, c->n_work.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));  // items with entries
        GEER_CUDA(cudaStreamSynchronize(st));
        out->kappa_rechecks = (int64_t)h[0];
        out->evaluated_pairs = (int64_t)h[1];
        out->fixup_pixels = (int64_t)h[2];
        out->warp_entries = (int64_t)h[3];
        out->streamed_entries = (int64_t)h[4];
        out->n_work_items = nit;
    }
    if (c->have_frame && c->scene.n > 0) {
        // clamped & kept count from the flags
        int64_t n = c->scene.n;
        uint8_t *hf = (uint8_t *)malloc((size_t)n);
        if (hf) {
            if (cudaMemcpy(hf, c->flags.p, (size_t)n, cudaMemcpyDeviceToHost) == cudaSuccess) {
                int64_t k = 0;
                for (int64_t i = 0; i < n; ++i) k += (hf[i] & 3) == 3;
                out->clamped = k;
            }
            free(hf);
        }
    }
    out->ms_prep = c->ms[0];
    out->ms_dup = c->ms[1];
    out->ms_sort = c->ms[2];
    out->ms_render = c->ms[3];
    out->ms_total = c->ms[4];
    out->ms_backward = c->ms[5];
    return GEER_OK;
}

int geer_association_check(geer_ctx *c, int32_t rays_per_tile, int64_t *out, int32_t *missing, int32_t max_missing,
                           uint32_t *hit_bits) {
    if (!c || !out) return fail(GEER_ERR_INVALID, "null argument");
    if (!c->have_frame) return fail(GEER_ERR_STATE, "association check needs a preceding forward or graph build");
    int side = 8;
    while (side * side < rays_per_tile) ++side;  // oracle.py:247 max(8, ceil(sqrt(rays_per_tile)))
    if (side > 16) return fail(GEER_ERR_INVALID, "rays_per_tile must be at most 256");
    if (max_missing < 0 || (max_missing > 0 && !missing)) return fail(GEER_ERR_INVALID, "bad missing buffer");
    const FrameConst &fc = c->fc;
    const int64_t n = c->scene.n, words = (n + 31) / 32;
    cudaStream_t st = c->own_stream;
    GEER_CUDA(cudaDeviceSynchronize());
    int rc = resolve_entries(c);
    if (rc) return rc;
    ArenaScope no_arena(nullptr);  // (transient buffers: cudaMalloc, freed below)
    Buf wo, bits, misc;  // transient (the bitmap is n_tiles * n / 8 bytes: 1 GB at 1M Gaussians, 1080p)
    struct Free {
        Buf *b[3];
        ~Free() {
            for (Buf *x : b) free_buf(*x);
        }
    } guard{{&wo, &bits, &misc}};
    double *w = ENSURE(double, wo, n * 12 + 1);
    uint32_t *gb = ENSURE(uint32_t, bits, (size_t)fc.n_tiles * words + 1);
    char *m = ENSURE(char, misc, 64 + 8 * (size_t)max_missing + 8);
    unsigned long long *cnt = (unsigned long long *)m;
    double *origin3 = (double *)(m + 24);
    int32_t *dmiss = max_missing ? (int32_t *)(m + 64) : nullptr;
    if (dmiss) GEER_CUDA(cudaMemsetAsync(dmiss, 0, 8 * (size_t)max_missing, st));
    rc = launch_assoc_check(fc, c->scene, (const double *)c->medges_x.p, (const double *)c->medges_y.p,
                            (const uint8_t *)c->flags.p, (const int32_t *)c->tile_ranges.p, (const uint32_t *)c->order.p,
                            side, w, origin3, gb, hit_bits, cnt, dmiss, max_missing, st);
    if (rc) return fail(rc, "association check launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    unsigned long long h[3];
    GEER_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
    if (max_missing) GEER_CUDA(cudaMemcpyAsync(missing, dmiss, 8 * (size_t)max_missing, cudaMemcpyDeviceToHost, st));
    GEER_CUDA(cudaStreamSynchronize(st));
    out[0] = (int64_t)h[0];
    out[1] = (int64_t)h[1];
    out[2] = (int64_t)h[2];
    out[3] = c->n_entries;
    return GEER_OK;
}

int64_t geer_last_h2d_bytes(const geer_ctx *c) { return c ? c->last_h2d : 0; }

// Diagnostics: the last forward's per-pixel alive counts (n_eval, renderer.py:113) to the host.
extern "C" int geer_debug_n_eval(geer_ctx *c, int32_t *host) {
    if (!c || !host) return fail(GEER_ERR_INVALID, "null argument");
    if (!c->have_stats) return fail(GEER_ERR_STATE, "no forward raster");
    GEER_CUDA(cudaDeviceSynchronize());
    GEER_CUDA(cudaMemcpy(host, c->n_eval.p, sizeof(int32_t) * (size_t)c->fc.width * c->fc.height, cudaMemcpyDeviceToHost));
    return GEER_OK;
}

int geer_graph_info(geer_ctx *c, int64_t *n_entries, int32_t *n_x, int32_t *n_y) {
    if (!c) return fail(GEER_ERR_INVALID, "null context");
    int rc0 = resolve_entries(c);
    if (rc0) return rc0;
    if (n_entries) *n_entries = c->n_entries;
    if (n_x) *n_x = c->fc.n_x;
    if (n_y) *n_y = c->fc.n_y;
    return GEER_OK;
}

static int d2h_u32_as_i64(const void *dev, int64_t *host, int64_t n) {
    if (!host || n <= 0) return GEER_OK;
    uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
    if (!tmp) return fail(GEER_ERR_NOMEM, "host allocation failed");
    cudaError_t e = cudaMemcpy(tmp, dev, sizeof(uint32_t) * (size_t)n, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        free(tmp);
        return fail(GEER_ERR_CUDA, "graph export copy failed: %s", cudaGetErrorString(e));
    }
    for (int64_t i = 0; i < n; ++i) host[i] = (int64_t)tmp[i];
    free(tmp);
    return GEER_OK;
}

int geer_graph_export(geer_ctx *c, int64_t *order, int64_t *entry_tile, int64_t *ranges, double *mu_c, double *depth,
                      uint8_t *keep, uint8_t *clamped, int64_t *pixel_tile, double *medges_x, double *medges_y) {
    if (!c) return fail(GEER_ERR_INVALID, "null context");
    if (!c->have_frame) return fail(GEER_ERR_STATE, "no render graph: run a forward or geer_build_graph_host first");
    GEER_CUDA(cudaDeviceSynchronize());
    int rc0 = resolve_entries(c);
    if (rc0) return rc0;
    const FrameConst &fc = c->fc;
    const int64_t n = c->scene.n, E = c->n_entries, npx = (int64_t)fc.width * fc.height;
    int rc = d2h_u32_as_i64(c->order.p, order, E);
    if (rc) return rc;
    if (entry_tile || ranges) {  // entry tiles from the tile ranges (the lists are tile-major)
        const int nt = fc.n_tiles;
        int64_t *rg = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nt + 1));
        if (!rg) return fail(GEER_ERR_NOMEM, "host allocation failed");
        rc = d2h_u32_as_i64(c->tile_ranges.p, rg, nt + 1);
        if (rc) {
            free(rg);
            return rc;
        }
        if (entry_tile)
            for (int t = 0; t < nt; ++t)
                for (int64_t e = rg[t]; e < rg[t + 1] && e < E; ++e) entry_tile[e] = t;
        if (ranges) memcpy(ranges, rg, sizeof(int64_t) * (size_t)(nt + 1));
        free(rg);
    }
    if (pixel_tile) {
        if (!c->cam_valid || !c->cam_pixel_tile)
            return fail(GEER_ERR_STATE, "pixel tiles were not recorded (use the host graph build)");
        rc = d2h_u32_as_i64(c->pixel_tile.p, pixel_tile, npx);
        if (rc) return rc;
    }
    if (mu_c) {
        if (!c->have_export) return fail(GEER_ERR_STATE, "camera-frame means were not recorded");
        GEER_CUDA(cudaMemcpy(mu_c, c->mu_c.p, sizeof(double) * n * 3, cudaMemcpyDeviceToHost));
    }
    if (depth) {
        if (!c->have_export) return fail(GEER_ERR_STATE, "depths were not recorded");
        GEER_CUDA(cudaMemcpy(depth, c->depth.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    }
    if ((keep || clamped) && n > 0) {
        uint8_t *hf = (uint8_t *)malloc((size_t)n);
        if (!hf) return fail(GEER_ERR_NOMEM, "host allocation failed");
        cudaError_t e = cudaMemcpy(hf, c->flags.p, (size_t)n, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            free(hf);
            return fail(GEER_ERR_CUDA, "flag export failed: %s", cudaGetErrorString(e));
        }
        for (int64_t i = 0; i < n; ++i) {
            if (keep) keep[i] = hf[i] & 1;
            if (clamped) clamped[i] = (hf[i] >> 1) & 1;
        }
        free(hf);
    }
    if (medges_x) GEER_CUDA(cudaMemcpy(medges_x, c->medges_x.p, sizeof(double) * (fc.n_x + 1), cudaMemcpyDeviceToHost));
    if (medges_y) GEER_CUDA(cudaMemcpy(medges_y, c->medges_y.p, sizeof(double) * (fc.n_y + 1), cudaMemcpyDeviceToHost));
    return GEER_OK;
}

int geer_build_graph_host(geer_ctx *c, const geer_host_scene *scene, const geer_camera *camera, double lam,
                          int32_t tile_px) {
    if (!c) return fail(GEER_ERR_INVALID, "null context");
    cudaStream_t st = c->own_stream;
    int rc = upload_host_scene(c, scene, st);
    if (rc) return rc;
    geer_config cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.lam = lam;
    cfg.tile_px = tile_px;
    cfg.support_cutoff = 1;
    rc = make_frame_const(camera, &cfg, scene->n_bands, &c->fc);
    if (rc) return rc;
    rc = run_forward(c, nullptr, nullptr, nullptr, true, st);
    if (rc) return rc;
    GEER_CUDA(cudaStreamSynchronize(st));
    return GEER_OK;
}

// Forward into context-owned fp32 buffers (host paths).
static int host_forward(geer_ctx *c, const geer_host_scene *scene, const geer_camera *camera,
                        const geer_config *config, cudaStream_t st) {
    int rc = upload_host_scene(c, scene, st);
    if (rc) return rc;
    rc = make_frame_const(camera, config, scene->n_bands, &c->fc);
    if (rc) return rc;
    const int64_t npx = (int64_t)c->fc.width * c->fc.height;
    float *col = ensure<float>(c->color, (size_t)npx * 3, &rc);
    if (rc) return rc;
    float *rem = ensure<float>(c->remaining, (size_t)npx, &rc);
    if (rc) return rc;
    int32_t *cnt = ensure<int32_t>(c->count_px, (size_t)npx, &rc);
    if (rc) return rc;
    if (scene->n == 0) {
        int32_t *ne = ensure<int32_t>(c->n_eval, (size_t)npx, &rc);
        if (rc) return rc;
        launch_fill_background(c->fc, col, rem, cnt, ne, st);
        c->have_frame = c->have_raster = c->have_stats = false;
        c->n_entries = 0;
        GEER_CUDA(cudaGetLastError());
        return GEER_OK;
    }
    return run_forward(c, col, rem, cnt, false, st);
}

int geer_render_host(geer_ctx *c, const geer_host_scene *scene, const geer_camera *camera, const geer_config *config,
                     double *color, double *remaining, int64_t *count) {
    if (!c) return fail(GEER_ERR_INVALID, "null context");
    if (!color || !remaining || !count) return fail(GEER_ERR_INVALID, "output buffers must be non-null");
    cudaStream_t st = c->own_stream;
    int rc = host_forward(c, scene, camera, config, st);
    if (rc) return rc;
    const int64_t npx = (int64_t)c->fc.width * c->fc.height;
    // convert on device, then one D2H per output (renderer.py:39-44 dtypes: f64, f64, i64)
    char *o = ensure<char>(c->out64, (size_t)npx * (3 * 8 + 8 + 8), &rc);
    if (rc) return rc;
    double *c64 = (double *)o;
    double *r64 = c64 + npx * 3;
    int64_t *n64 = (int64_t *)(r64 + npx);
    launch_convert_f32_f64((const float *)c->color.p, c64, npx * 3, st);
    launch_convert_f32_f64((const float *)c->remaining.p, r64, npx, st);
    launch_convert_i32_i64((const int32_t *)c->count_px.p, n64, npx, st);
    GEER_CUDA(cudaMemcpyAsync(color, c64, sizeof(double) * npx * 3, cudaMemcpyDeviceToHost, st));
    GEER_CUDA(cudaMemcpyAsync(remaining, r64, sizeof(double) * npx, cudaMemcpyDeviceToHost, st));
    GEER_CUDA(cudaMemcpyAsync(count, n64, sizeof(int64_t) * npx, cudaMemcpyDeviceToHost, st));
    GEER_CUDA(cudaStreamSynchronize(st));
    return GEER_OK;
}

int geer_render_backward_host(geer_ctx *c, const geer_host_scene *scene, const geer_camera *camera,
                              const double *dl_dimage, const geer_config *config, const geer_host_grads *grads) {
    if (!c) return fail(GEER_ERR_INVALID, "null context");
    if (!dl_dimage || !grads) return fail(GEER_ERR_INVALID, "dl_dimage and grads are required");
    cudaStream_t st = c->own_stream;
    int rc = host_forward(c, scene, camera, config, st);
    if (rc) return rc;
    const int64_t n = scene->n, nb = scene->n_bands, npx = (int64_t)c->fc.width * c->fc.height;
    const int64_t sizes[5] = {n * 3, n * 3, n * 4, n, n * nb * 3};
    double *hout[5] = {grads->dmeans, grads->dlog_scales, grads->dquats, grads->dopacities, grads->dsh};
    if (n == 0) return GEER_OK;
    for (int i = 0; i < 5; ++i)
        if (!hout[i]) return fail(GEER_ERR_INVALID, "gradient pointers must be non-null");
    // dl_dimage f64 host -> f32 device: narrowed on the host like the scene, into the staging region
    // after the scene's (whose copies may still be in flight)
    float *dl32 = ensure<float>(c->dl32, (size_t)npx * 3, &rc);
    if (rc) return rc;
    const int64_t scene_floats = n * 11 + n * nb * 3;
    rc = ensure_pinned(c->h_stage, c->h_stage_cap, sizeof(float) * (size_t)(scene_floats + npx * 3), true, st);
    if (rc) return rc;
    {
        const HostSeg seg = {dl_dimage, npx * 3, dl32};
        const int64_t raw = raw_upload_elems(npx * 3);
        double *raw_dev = nullptr;
        if (raw > 0) raw_dev = ensure<double>(c->out64, (size_t)raw, &rc);
        if (rc) return rc;
        int64_t sent = 0;
        GEER_CUDA(upload_narrowed(&seg, 1, (float *)c->h_stage + scene_floats, raw_dev, raw, st, &sent));
        c->last_h2d += sent;
    }
    // fp32 gradients (k_finalize's arithmetic is fp32; its f64 output would be the exact widening),
    // downloaded chunk by chunk and widened on the host pool
    int64_t tot = 0;
    for (int i = 0; i < 5; ++i) tot += sizes[i];
    float *g = ensure<float>(c->g64, (size_t)tot, &rc);
    if (rc) return rc;
    void *gp[5];
    HostOut outs[5];
    int64_t off = 0;
    for (int i = 0; i < 5; ++i) {
        gp[i] = g + off;
        outs[i] = HostOut{g + off, sizes[i], hout[i]};
        off += sizes[i];
    }
    rc = run_backward(c, dl32, false, gp, 0, st);
    if (rc) return rc;
    rc = ensure_pinned(c->h_down, c->h_down_cap, sizeof(float) * (size_t)tot, false, st);
    if (rc) return rc;
    GEER_CUDA(download_widened(outs, 5, (float *)c->h_down, c->down_evs, st));
    GEER_CUDA(cudaStreamSynchronize(st));
    return GEER_OK;
}

}  // extern "C"
