// geer_sort.cu — association back half: depth order, scan, emit, tile sort, ranges.
//
// The reference orders entries by (tile, f32 depth bits, gid) (association.py:
// 453-461: np.unique on (tile, gid) then a stable argsort of
// key = tile << 32 | depth_sort_bits).  We get the same total order with far
// less sort traffic:
//   1. stable radix sort of the N per-Gaussian depth keys (values = gid, so
//      equal depths stay in gid order);
//   2. scan of the per-Gaussian entry counts in that depth order;
//   3. load-balanced emit: one thread per entry writes (tile, gid), entries of
//      each Gaussian contiguous, Gaussians in (depth, gid) order;
//   4. stable radix sort on the tile id only (ceil(log2 n_tiles) bits,
//      2 passes at 8,160 tiles instead of 6 passes over 45-bit keys);
//   5. per-tile [start, end) ranges (association.py:466).
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

size_t scan_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, (const int64_t *)nullptr, (int64_t *)nullptr, (int)n);
    return bytes;
}

size_t scan_i32_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int32_t *)nullptr, (int32_t *)nullptr, (int)n);
    return bytes;
}

template <typename K>
size_t sort_tiles_temp_bytes(int64_t n_entries, int n_bits) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const K *)nullptr, (K *)nullptr, (const uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (int)n_entries, 0, n_bits > 0 ? n_bits : 1);
    return bytes;
}
template size_t sort_tiles_temp_bytes<uint16_t>(int64_t, int);
template size_t sort_tiles_temp_bytes<uint32_t>(int64_t, int);

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

template <typename K>
void sort_tiles(void *temp, size_t temp_bytes, const K *keys_in, K *keys_out, const uint32_t *vals_in,
                uint32_t *vals_out, int64_t n, int n_bits, cudaStream_t st) {
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, (int)n, 0,
                                    n_bits > 0 ? n_bits : 1, st);
}
template void sort_tiles<uint16_t>(void *, size_t, const uint16_t *, uint16_t *, const uint32_t *, uint32_t *, int64_t,
                                   int, cudaStream_t);
template void sort_tiles<uint32_t>(void *, size_t, const uint32_t *, uint32_t *, const uint32_t *, uint32_t *, int64_t,
                                   int, cudaStream_t);

void sort_pixels(void *temp, size_t temp_bytes, const int32_t *keys_in, int32_t *keys_out, const int32_t *vals_in,
                 int32_t *vals_out, int64_t n, int n_bits, cudaStream_t st) {
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, (int)n, 0,
                                    n_bits > 0 ? n_bits : 1, st);
}

__global__ void k_gather_counts(const int32_t *sorted_gid, const int64_t *count, int64_t *cnt_sorted, int64_t n) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        cnt_sorted[r] = count[sorted_gid[r]];
}

void gather_counts(const int32_t *sorted_gid, const int64_t *count, int64_t *cnt_sorted, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    int blocks = (int)lmin((n + 255) / 256, 148 * 16);
    k_gather_counts<<<blocks, 256, 0, st>>>(sorted_gid, count, cnt_sorted, n);
}

void inclusive_scan_i64(void *temp, size_t temp_bytes, const int64_t *in, int64_t *out, int64_t n, cudaStream_t st) {
    cub::DeviceScan::InclusiveSum(temp, temp_bytes, in, out, (int)n, st);
}

void exclusive_scan_i32(void *temp, size_t temp_bytes, const int32_t *in, int32_t *out, int64_t n, cudaStream_t st) {
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, (int)n, st);
}

// Decode the k-th index of a merged range list (ranges packed lo | hi << 16).
__device__ __forceinline__ int range_index(const uint32_t r[3], int k) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        int lo = (int)(r[i] & 0xFFFFu), hi = (int)(r[i] >> 16);
        int len = hi - lo;
        if (k < len) return lo + k;
        k -= len;
    }
    return -1;
}
__device__ __forceinline__ int range_len(const uint32_t r[3]) {
    int s = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) s += (int)(r[i] >> 16) - (int)(r[i] & 0xFFFFu);
    return s;
}

// offs[r] = entries before depth-rank r (offs[0] = 0, offs[n] = total).
// Each block covers kEmitPerBlock consecutive entries.  Every Gaussian of rank
// < n_emitting owns >= 1 entry, so a block spans <= kEmitPerBlock + 1 ranks:
// their offsets are staged in shared memory and each thread binary-searches
// its entry's rank there (coalesced writes, no per-Gaussian load imbalance).
constexpr int kEmitPerBlock = 1024;

// block_rank[b] = depth rank owning entry b * kEmitPerBlock; block_rank[n_blocks] = rank of the last
// entry.  One thread per rank: a rank owns the block starts inside its [offs[r], offs[r+1]).
__global__ void k_block_ranks(const int64_t *__restrict__ offs, int64_t n, int64_t n_entries, int n_blocks,
                              int32_t *__restrict__ block_rank) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t lo = offs[r], hi = offs[r + 1];
        if (lo == hi) continue;
        for (int64_t b = (lo + kEmitPerBlock - 1) / kEmitPerBlock; b * kEmitPerBlock < hi; ++b) block_rank[b] = (int32_t)r;
        if (lo <= n_entries - 1 && n_entries - 1 < hi) block_rank[n_blocks] = (int32_t)r;
    }
}
// One block = kEmitPerBlock consecutive entries (4 per thread).  The block's ranks are staged
// once (gid, axis ranges, local start), each rank marks the position of its first entry, and an
// inclusive max-scan over the positions gives every entry its rank; entries are then decoded from
// shared memory and written with coalesced stores.
template <typename K>
__global__ void __launch_bounds__(256) k_emit(const int64_t *__restrict__ offs, const int32_t *__restrict__ block_rank,
                                              const int32_t *__restrict__ sorted_gid,
                                              const AxisRanges *__restrict__ ranges, int n_x, int64_t n_entries,
                                              int64_t n, K *__restrict__ tile_keys, uint32_t *__restrict__ gids) {
    __shared__ int s_pos[kEmitPerBlock];
    __shared__ int s_start[kEmitPerBlock + 1];
    __shared__ uint32_t s_g[kEmitPerBlock + 1];
    __shared__ AxisRanges s_ar[kEmitPerBlock + 1];
    __shared__ int s_wmax[8];
    const int64_t e_begin = (int64_t)blockIdx.x * kEmitPerBlock;
    const int n_here = (int)lmin(kEmitPerBlock, n_entries - e_begin);
    // ranks owning this block's first entry and (at most) the next block's first entry
    const int64_t r0 = block_rank[blockIdx.x], r1 = block_rank[blockIdx.x + 1];
    const int span = (int)(r1 - r0 + 1);  // <= kEmitPerBlock + 1
    for (int j = threadIdx.x; j < kEmitPerBlock; j += blockDim.x) s_pos[j] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < span; i += blockDim.x) {
        const int st = (int)(offs[r0 + i] - e_begin);  // < 0 only for rank r0
        const uint32_t g = (uint32_t)sorted_gid[r0 + i];
        s_start[i] = st;
        s_g[i] = g;
        s_ar[i] = ranges[g];
        if (st >= 0 && st < kEmitPerBlock) s_pos[st] = i;
    }
    __syncthreads();
    // inclusive max-scan of s_pos (local ranks increase with position)
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = s_pos[4 * t + u];
#pragma unroll
    for (int u = 1; u < 4; ++u) v[u] = max(v[u], v[u - 1]);
    int run = v[3];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, run, o);
        if (lane >= o) run = max(run, y);
    }
    if (lane == 31) s_wmax[warp] = run;
    __syncthreads();
    int carry = 0;
    for (int w = 0; w < warp; ++w) carry = max(carry, s_wmax[w]);
    int prev = __shfl_up_sync(0xffffffffu, run, 1);
    prev = max(lane > 0 ? prev : 0, carry);
#pragma unroll
    for (int u = 0; u < 4; ++u) s_pos[4 * t + u] = max(v[u], prev);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int j = u * 256 + t;
        if (j >= n_here) break;
        const int rl = s_pos[j];
        const AxisRanges ar = s_ar[rl];
        const int cx = range_len(ar.x);
        const int k = j - s_start[rl];
        const int ky = k / cx;
        const int iy = range_index(ar.y, ky);
        const int ix = range_index(ar.x, k - ky * cx);
        tile_keys[e_begin + j] = (K)(iy * n_x + ix);
        gids[e_begin + j] = s_g[rl];
    }
}

int64_t emit_blocks(int64_t n_entries) { return (n_entries + kEmitPerBlock - 1) / kEmitPerBlock; }

template <typename K>
void emit_entries(const int64_t *offs, const int32_t *sorted_gid, const AxisRanges *ranges, int n_x,
                  int64_t n_entries, int64_t n, int32_t *block_rank, K *tile_keys, uint32_t *gids,
                  cudaStream_t st) {
    if (n_entries <= 0) return;
    const int64_t blocks = emit_blocks(n_entries);
    k_block_ranks<<<(unsigned)lmin((n + 255) / 256, 148 * 16), 256, 0, st>>>(offs, n, n_entries, (int)blocks, block_rank);
    k_emit<K><<<(unsigned)blocks, 256, 0, st>>>(offs, block_rank, sorted_gid, ranges, n_x, n_entries, n, tile_keys, gids);
}
template void emit_entries<uint16_t>(const int64_t *, const int32_t *, const AxisRanges *, int, int64_t, int64_t,
                                     int32_t *, uint16_t *, uint32_t *, cudaStream_t);
template void emit_entries<uint32_t>(const int64_t *, const int32_t *, const AxisRanges *, int, int64_t, int64_t,
                                     int32_t *, uint32_t *, uint32_t *, cudaStream_t);

// ranges[t] = first entry with tile >= t (np.searchsorted(tiles, arange(n_tiles + 1)))
template <typename K>
__global__ void k_ranges(const K *__restrict__ tiles, int64_t n_entries, int n_tiles, int32_t *__restrict__ ranges) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= n_entries; e += (int64_t)gridDim.x * blockDim.x) {
        int prev = e == 0 ? -1 : (int)tiles[e - 1];
        int cur = e == n_entries ? n_tiles : (int)tiles[e];
        for (int t = prev + 1; t <= cur; ++t) ranges[t] = (int32_t)e;
    }
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
    if (in && !full) work[max_items - 1 - (be + __popc(me & lt))] = it;
}

void order_items(const int4 *items, const int32_t *n_items, const int32_t *ranges, int max_items, int4 *work,
                 int32_t *n_work, cudaStream_t st) {
    cudaMemsetAsync(n_work, 0, 2 * sizeof(int32_t), st);
    k_order_items<<<(max_items + 255) / 256, 256, 0, st>>>(items, n_items, ranges, max_items, work, n_work);
}

template <typename K>
void tile_ranges(const K *sorted_tiles, int64_t n_entries, int n_tiles, int32_t *ranges, cudaStream_t st) {
    int blocks = (int)lmin((n_entries + 1 + 255) / 256, 148 * 16);
    k_ranges<K><<<blocks, 256, 0, st>>>(sorted_tiles, n_entries, n_tiles, ranges);
}
template void tile_ranges<uint16_t>(const uint16_t *, int64_t, int, int32_t *, cudaStream_t);
template void tile_ranges<uint32_t>(const uint32_t *, int64_t, int, int32_t *, cudaStream_t);

}  // namespace geer
