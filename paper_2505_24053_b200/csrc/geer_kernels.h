// geer_kernels.h — host-side launchers shared between the translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "geer_common.cuh"

namespace geer {

// geer_geometry.cu (fp64, -fmad=false)
void launch_beap_setup(const FrameConst &fc, double2 *col_sc, double2 *row_sc, double *medges_x, double *medges_y,
                       int32_t *tile_off, int32_t *pix_list, int32_t *pixel_tile, cudaStream_t st);
void launch_cam_pixels(const FrameConst &fc, double *dir64, double *theta, double *phi, long long *minmax,
                       cudaStream_t st);
void launch_cam_edges(const FrameConst &fc, const long long *minmax, double *edges_x, double *edges_y,
                      double *medges_x, double *medges_y, cudaStream_t st);
void launch_cam_bin(const FrameConst &fc, const double *theta, const double *phi, const double *edges_x,
                    const double *edges_y, int32_t *pixel_tile, int32_t *tile_count, cudaStream_t st);
void launch_iota(int32_t *v, int64_t n, cudaStream_t st);
void launch_items(int n_tiles, const int32_t *tile_off, int32_t *item_count, cudaStream_t st);
void launch_item_fill(int n_tiles, const int32_t *tile_off, const int32_t *item_off, int4 *items, int32_t *n_items,
                      cudaStream_t st);
size_t preprocess_smem(const FrameConst &fc);
void launch_preprocess(const FrameConst &fc, const geer_scene &sc, const double *medges_x, const double *medges_y,
                       Payload *payload, uint32_t *depth_key, AxisRanges *ranges, uint8_t *flags,
                       double *mu_out, double *depth_out, int *err, unsigned long long *total_entries,
                       cudaStream_t st);
template <typename T>
void launch_finalize(const FrameConst &fc, const geer_scene &sc, const float4 *accum, const uint8_t *flags, T *dmeans,
                     T *dlog_scales, T *dquats, T *dopac, T *dsh, int accumulate, cudaStream_t st);

// geer_sort.cu (association: depth order, scan, emit, tile sort, ranges)
struct SortTemp {
    void *p = nullptr;
    size_t bytes = 0;
};
size_t sort_depth_temp_bytes(int64_t n);
size_t scan_i32_temp_bytes(int64_t n);
void sort_depth(void *temp, size_t temp_bytes, const uint32_t *keys_in, uint32_t *keys_out, const int32_t *vals_in,
                int32_t *vals_out, int64_t n, cudaStream_t st);
void exclusive_scan_i32(void *temp, size_t temp_bytes, const int32_t *in, int32_t *out, int64_t n, cudaStream_t st);
// Per-tile lists by two-level stable bucketing (geer_bin.cu): order / ranges equal the stable tile
// sort of the depth-ordered entries.
struct BinPlan {
    int nch;                                    // level-1 chunks
    int64_t m1_len, rows_cap, seg_cap, m2_len;  // [row][chunk] counts, row-bin capacity, segments, [row][tile][seg]
    size_t temp_bytes;                          // CUB scan workspace
};
BinPlan bin_plan(int64_t n, int n_x, int n_y, int64_t n_entries, int64_t n_rows);
// d_total: the device entry total (K1's counter); err: the frame's device status (an overflow turns
// the binning into no-ops and leaves every tile empty).
int bin_tiles(const BinPlan &p, const int32_t *gsorted, const AxisRanges *ar, int64_t n, int n_x, int n_y,
              const unsigned long long *d_total, const int *err, uint32_t *m1, uint32_t *p1, uint2 *rowbin,
              int32_t *rowstart, int32_t *seg_off, uint32_t *m2, uint32_t *p2, void *temp, uint32_t *order,
              int32_t *ranges, cudaStream_t st);
// err = GEER_ERR_OVERFLOW when totals[0] (entries) > cap_entries or totals[1] ((Gaussian, row) pairs) > cap_rows
void launch_check_capacity(const unsigned long long *totals, int64_t cap_entries, int64_t cap_rows, int *err,
                           cudaStream_t st);
void sort_pixels(void *temp, size_t temp_bytes, const int32_t *keys_in, int32_t *keys_out, const int32_t *vals_in,
                 int32_t *vals_out, int64_t n, int n_bits, cudaStream_t st);
size_t sort_pixels_temp_bytes(int64_t n, int n_bits);
void order_items(const int4 *items, const int32_t *n_items, const int32_t *ranges, int max_items, int4 *work,
                 int32_t *n_work, cudaStream_t st);
int order_items_ints();  // ints order_items needs at n_work (counts + its scratch)

// geer_raster.cu (fp32 raster forward / backward)
// per-warp culling regions (wcull: 2 float4 per warp) and the frame of every work item, cached with the camera
void launch_warp_cull(const FrameConst &fc, int max_items, const int4 *items, const int32_t *n_items,
                      const int32_t *pix_list, const double2 *col_sc, const double2 *row_sc, const double *dir64,
                      float4 *wcull, ItemFrame *iframe, cudaStream_t st);
void launch_forward(const FrameConst &fc, const geer_scene &sc, int max_items, const int4 *items,
                    const int32_t *n_items, const int32_t *pix_list, const double2 *col_sc, const double2 *row_sc,
                    const double *dir64, const int32_t *ranges, const uint32_t *order, const Payload *payload,
                    const CUtensorMap &pay_map, const float4 *wcull, const ItemFrame *iframe, float *color,
                    float *remaining, int32_t *count, int32_t *n_eval, unsigned long long *counters,
                    int32_t *fixup_list, cudaStream_t st);
void launch_backward(const FrameConst &fc, const geer_scene &sc, int max_items, const int4 *items,
                     const int32_t *n_items, const int32_t *pix_list, const double2 *col_sc, const double2 *row_sc,
                     const double *dir64, const int32_t *ranges, const uint32_t *order, const CUtensorMap &pay_map,
                     const float4 *wcull, const ItemFrame *iframe, const float *remaining, const int32_t *n_eval,
                     const float *dl_dimage, float *accum, cudaStream_t st);
int launch_assoc_check(const FrameConst &fc, const geer_scene &sc, const double *medges_x, const double *medges_y,
                       const uint8_t *flags, const int32_t *ranges, const uint32_t *order, int side, double *wo,
                       double *origin3, uint32_t *graph_bits, uint32_t *hit_bits, unsigned long long *counters,
                       int32_t *missing, int max_missing, cudaStream_t st);
void launch_exhaustive_ranges(const uint8_t *flags, int64_t n, int32_t *ranges2, cudaStream_t st);
void launch_sum_i32(const int32_t *v, int64_t n, unsigned long long *out, cudaStream_t st);
void launch_convert_f64_f32(const double *in, float *out, int64_t n, cudaStream_t st);
void launch_convert_f32_f64(const float *in, double *out, int64_t n, cudaStream_t st);
void launch_convert_i32_i64(const int32_t *in, int64_t *out, int64_t n, cudaStream_t st);
void launch_fill_background(const FrameConst &fc, float *color, float *remaining, int32_t *count, int32_t *n_eval,
                            cudaStream_t st);

}  // namespace geer
