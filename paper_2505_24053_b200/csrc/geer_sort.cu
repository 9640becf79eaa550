// geer_sort.cu — association back half, part 1: depth order (and the CUB sorts/scans of the
// camera setup), plus the raster work order.
//
// The reference orders entries by (tile, f32 depth bits, gid) (association.py:453-461: np.unique on
// (tile, gid) then a stable argsort of key = tile << 32 | depth_sort_bits).  We get the same total
// order from a stable radix sort of the N per-Gaussian depth keys (values = gid, so equal depths
// stay in gid order) followed by the stable per-tile bucketing of geer_bin.cu.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "geer_common.cuh"
#include "geer_kernels.h"

namespace geer {

size_t sort_depth_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, 32);
    return bytes;
}

size_t scan_i32_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int32_t *)nullptr, (int32_t *)nullptr, (int)n);
    return bytes;
}

size_t sort_pixels_temp_bytes(int64_t n, int n_bits) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t *)nullptr, (int32_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, n_bits > 0 ? n_bits : 1);
    return bytes;
}

void sort_depth(void *temp, size_t temp_bytes, const uint32_t *keys_in, uint32_t *keys_out, const int32_t *vals_in,
                int32_t *vals_out, int64_t n, cudaStream_t st) {
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, (int)n, 0, 32, st);
}

void sort_pixels(void *temp, size_t temp_bytes, const int32_t *keys_in, int32_t *keys_out, const int32_t *vals_in,
                 int32_t *vals_out, int64_t n, int n_bits, cudaStream_t st) {
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, (int)n, 0,
                                    n_bits > 0 ? n_bits : 1, st);
}

void exclusive_scan_i32(void *temp, size_t temp_bytes, const int32_t *in, int32_t *out, int64_t n, cudaStream_t st) {
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, (int)n, st);
}

// Raster work order: items of tiles with entries fill work[] from the front, the empty ones (which
// only write the background) from the back.  n_work[0] = items with entries, n_work[1] = empty
// items (both zeroed before the launch).  The order among full items does not affect results.
__global__ void k_order_items(const int4 *__restrict__ items, const int32_t *__restrict__ n_items,
                              const int32_t *__restrict__ ranges, int max_items, int4 *__restrict__ work,
                              int32_t *__restrict__ n_work) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = i < *n_items;
    int4 it = make_int4(0, 0, 0, 0);
    bool full = false;
    if (in) {
        it = items[i];
        full = ranges[it.x + 1] > ranges[it.x];
    }
    // warp-aggregated slots
    const unsigned mf = __ballot_sync(0xffffffffu, in && full), me = __ballot_sync(0xffffffffu, in && !full);
    const int lane = threadIdx.x & 31;
    int bf = 0, be = 0;
    if (lane == 0) {
        if (mf) bf = atomicAdd(&n_work[0], __popc(mf));
        if (me) be = atomicAdd(&n_work[1], __popc(me));
    }
    bf = __shfl_sync(0xffffffffu, bf, 0);
    be = __shfl_sync(0xffffffffu, be, 0);
    const unsigned lt = (1u << lane) - 1u;
    if (in && full) work[bf + __popc(mf & lt)] = it;
    if (in && !full) work[*n_items - 1 - (be + __popc(me & lt))] = it;  // empty items: the tail of [0, n_items)
}

// Longest-first work order (the raster's CTAs start in grid order, so the longest tile lists go
// first and the short ones fill the tail): items bucketed by floor(log2(list length)) + 1, buckets
// in descending order, empty items (bucket 0) last.  hist[0..33): bucket counts, then cursors.
constexpr int kLenBuckets = 33;
__device__ __forceinline__ int len_bucket(int len) { return len > 0 ? 32 - __clz(len) : 0; }

__global__ void k_item_hist(const int4 *__restrict__ items, const int32_t *__restrict__ n_items,
                            const int32_t *__restrict__ ranges, int32_t *__restrict__ hist) {
    __shared__ int h[kLenBuckets];
    if (threadIdx.x < kLenBuckets) h[threadIdx.x] = 0;
    __syncthreads();
    const int n = *n_items;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int t = items[i].x;
        atomicAdd(&h[len_bucket(ranges[t + 1] - ranges[t])], 1);
    }
    __syncthreads();
    if (threadIdx.x < kLenBuckets && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void k_item_place(const int4 *__restrict__ items, const int32_t *__restrict__ n_items,
                             const int32_t *__restrict__ ranges, const int32_t *__restrict__ hist,
                             int32_t *__restrict__ cursor, int4 *__restrict__ work, int32_t *__restrict__ n_work) {
    __shared__ int start[kLenBuckets];
    if (threadIdx.x == 0) {  // bucket starts: 32, 31, ..., 1, then 0 (empty)
        int run = 0;
        for (int b = kLenBuckets - 1; b >= 1; --b) {
            start[b] = run;
            run += hist[b];
        }
        start[0] = run;
        if (blockIdx.x == 0) {
            n_work[0] = run;      // items with entries
            n_work[1] = hist[0];  // empty items
        }
    }
    __syncthreads();
    const int n = *n_items;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int4 it = items[i];
        const int b = len_bucket(ranges[it.x + 1] - ranges[it.x]);
        work[start[b] + atomicAdd(&cursor[b], 1)] = it;
    }
}

void order_items(const int4 *items, const int32_t *n_items, const int32_t *ranges, int max_items, int4 *work,
                 int32_t *n_work, cudaStream_t st) {
#ifdef GEER_ORDER_ARBITRARY
    cudaMemsetAsync(n_work, 0, 2 * sizeof(int32_t), st);
    k_order_items<<<(max_items + 255) / 256, 256, 0, st>>>(items, n_items, ranges, max_items, work, n_work);
#else
    // n_work holds 2 + 2 * kLenBuckets ints: the counts, then the histogram and the cursors
    int32_t *hist = n_work + 2, *cursor = hist + kLenBuckets;
    cudaMemsetAsync(hist, 0, 2 * kLenBuckets * sizeof(int32_t), st);
    const int blocks = (max_items + 255) / 256 < 148 ? (max_items + 255) / 256 : 148;
    k_item_hist<<<blocks, 256, 0, st>>>(items, n_items, ranges, hist);
    k_item_place<<<blocks, 256, 0, st>>>(items, n_items, ranges, hist, cursor, work, n_work);
#endif
}

int order_items_ints() { return 2 + 2 * kLenBuckets; }

}  // namespace geer
