// geer_bin.cu — per-tile Gaussian lists without a tile sort (association.py:452-466: entries
// ordered by tile, then by depth rank, i.e. a stable sort of the depth-ordered (tile, gid) pairs).
//
// The lists are built by a two-level stable bucketing of the depth-ordered Gaussians, each level a
// count / exclusive-scan / ordered-scatter triple:
//   level 1 (rows):  chunk c of kBinChunk consecutive depth ranks counts its Gaussians per tile
//                    row; one flat exclusive scan of the [row][chunk] count matrix gives every
//                    (row, chunk) its start in the row bins; a block per chunk then places each
//                    (Gaussian, row) pair, (gid, x-range), in depth order.
//   level 2 (tiles): the row bins are cut into segments of kSegLen entries; the [row][tile][segment]
//                    count matrix, scanned flat in that order, is exactly the final entry position
//                    of every (tile, segment) (tile-major order, segments of a row in depth order);
//                    a block per segment places each (entry, tile) pair.
// The scatters are order-exact without atomics on positions: each pair sets its item's bit in a
// per-bucket membership mask (one bit per item of the chunk / segment, shared memory), and its slot is
// the bucket's start plus the number of earlier items in the bucket, popc of the mask below its bit.
// The output equals the stable tile sort bit for bit.  Traffic is a few bytes per entry (vs. two
// radix passes over 6-byte pairs plus the emitted pairs themselves).
#include <cub/cub.cuh>
#include <stdint.h>

#include "geer_common.cuh"
#include "geer_kernels.h"

namespace geer {
namespace {

#ifndef GEER_BIN_CHUNK
#define GEER_BIN_CHUNK 256
#endif
#ifndef GEER_SEG_LEN
#define GEER_SEG_LEN 512
#endif
constexpr int kBinChunk = GEER_BIN_CHUNK;  // depth-ordered Gaussians per level-1 chunk (= threads of a count block)
constexpr int kSegLen = GEER_SEG_LEN;      // row-bin entries per level-2 segment (= threads of a count block)
constexpr uint32_t kMultiX = 0xFFFFFFFFu;  // row-bin x info: several x ranges, read them from AxisRanges

__device__ __forceinline__ int rlen(uint32_t r) { return (int)(r >> 16) - (int)(r & 0xFFFFu); }

// Row-bin x info of a Gaussian: its single packed x range, or kMultiX.
__device__ __forceinline__ uint32_t x_info(const AxisRanges &a) {
    return (rlen(a.x[1]) > 0 || rlen(a.x[2]) > 0) ? kMultiX : a.x[0];
}
__device__ __forceinline__ bool has_entries(const AxisRanges &a) {
    return (rlen(a.x[0]) + rlen(a.x[1]) + rlen(a.x[2])) > 0 && (rlen(a.y[0]) + rlen(a.y[1]) + rlen(a.y[2])) > 0;
}

__global__ void __launch_bounds__(kBinChunk) k_rows_count(const int32_t *__restrict__ gsorted,
                                                          const AxisRanges *__restrict__ ar, int64_t n, int n_y,
                                                          int nch, uint32_t *__restrict__ m1,
                                                          const int *__restrict__ err) {
    extern __shared__ uint32_t cnt[];
    if (*err == GEER_ERR_OVERFLOW) return;  // (the graph exceeds the capacity: the frame is re-run)
    for (int r = threadIdx.x; r < n_y; r += blockDim.x) cnt[r] = 0;
    __syncthreads();
    const int64_t p = (int64_t)blockIdx.x * kBinChunk + threadIdx.x;
    if (p < n) {
        const AxisRanges a = ar[gsorted[p]];
        if (has_entries(a)) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                for (int r = (int)(a.y[k] & 0xFFFFu); r < (int)(a.y[k] >> 16); ++r) atomicAdd(&cnt[r], 1u);
        }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < n_y; r += blockDim.x) m1[(int64_t)r * nch + blockIdx.x] = cnt[r];
}

// Level-1 scatter, one thread per Gaussian of the chunk (a block per chunk): each (Gaussian, row)
// pair sets the Gaussian's bit in the row's kBinChunk-bit membership mask (shared memory,
// word-major), and its slot is the (row, chunk) start plus popc of the mask below it: the rows'
// entries stay in depth order.
constexpr int kRW = kBinChunk / 32;  // mask words per row
static_assert(kRW % 4 == 0, "the mask is zeroed in 16-byte stores");
__global__ void __launch_bounds__(kBinChunk) k_rows_scatter_mask(const int32_t *__restrict__ gsorted,
                                                                 const AxisRanges *__restrict__ ar, int64_t n,
                                                                 int n_y, int nch, const uint32_t *__restrict__ p1,
                                                                 uint2 *__restrict__ rowbin,
                                                                 const int *__restrict__ err) {
    extern __shared__ uint32_t smem[];
    if (*err == GEER_ERR_OVERFLOW) return;
    uint32_t *mask = smem;            // [kRW][n_y]
    uint32_t *pre = smem + n_y * kRW; // [kRW][n_y]
    const int c = blockIdx.x, tid = threadIdx.x;
    for (int i = tid; i < n_y * kRW / 4; i += kBinChunk) reinterpret_cast<uint4 *>(mask)[i] = make_uint4(0u, 0u, 0u, 0u);
    uint32_t start0 = 0;
    if (tid < n_y) start0 = p1[(int64_t)tid * nch + c];
    const int64_t p = (int64_t)c * kBinChunk + tid;
    uint32_t g = 0, xi = 0, yr[3] = {0u, 0u, 0u};
    if (p < n) {
        g = (uint32_t)gsorted[p];
        const AxisRanges a = ar[g];
        if (has_entries(a)) {
            xi = x_info(a);
            yr[0] = a.y[0];
            yr[1] = a.y[1];
            yr[2] = a.y[2];
        }
    }
    __syncthreads();
    const int w = tid >> 5;
    const uint32_t bit = 1u << (tid & 31);
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int r = (int)(yr[k] & 0xFFFFu); r < (int)(yr[k] >> 16); ++r) atomicOr(&mask[w * n_y + r], bit);
    __syncthreads();
    for (int r = tid; r < n_y; r += kBinChunk) {
        uint32_t run = r == tid ? start0 : p1[(int64_t)r * nch + c];
#pragma unroll
        for (int j = 0; j < kRW; ++j) {
            pre[j * n_y + r] = run;
            run += __popc(mask[j * n_y + r]);
        }
    }
    __syncthreads();
    const uint32_t below = bit - 1u;
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int r = (int)(yr[k] & 0xFFFFu); r < (int)(yr[k] >> 16); ++r)
            rowbin[pre[w * n_y + r] + __popc(mask[w * n_y + r] & below)] = make_uint2(g, xi);
}

// Row starts, segments per row (>= 1, so every tile has a (tile, segment 0) slot) and their
// exclusive prefix; also the list end ranges[n_tiles] = total.  One block.
__global__ void k_segments(const uint32_t *__restrict__ m1, const uint32_t *__restrict__ p1, int n_y, int nch,
                           int32_t *__restrict__ rowstart, int32_t *__restrict__ seg_off, int n_tiles,
                           const unsigned long long *__restrict__ d_total, int32_t *__restrict__ ranges,
                           const int *__restrict__ err) {
    __shared__ int carry;
    if (*err == GEER_ERR_OVERFLOW) {  // every tile empty (the raster renders background; the frame is re-run)
        for (int t = threadIdx.x; t <= n_tiles; t += blockDim.x) ranges[t] = 0;
        if (threadIdx.x == 0) seg_off[n_y] = 0;
        return;
    }
    const int32_t total = (int32_t)*d_total;
    const int64_t last = (int64_t)n_y * nch - 1;
    const uint32_t R = last >= 0 ? p1[last] + m1[last] : 0u;
    if (threadIdx.x == 0) {
        carry = 0;
        rowstart[n_y] = (int32_t)R;
        ranges[n_tiles] = total;
    }
    __syncthreads();
    for (int r0 = 0; r0 < n_y; r0 += blockDim.x) {
        const int r = r0 + threadIdx.x;
        int ns = 0;
        if (r < n_y) {
            const uint32_t a = p1[(int64_t)r * nch], b = r + 1 < n_y ? p1[(int64_t)(r + 1) * nch] : R;
            rowstart[r] = (int32_t)a;
            ns = max(1, (int)((b - a + kSegLen - 1) / kSegLen));
        }
        int incl;
        {
            typedef cub::BlockScan<int, 1024> Scan;
            __shared__ typename Scan::TempStorage tmp;
            Scan(tmp).InclusiveSum(ns, incl);
        }
        if (r < n_y) seg_off[r] = carry + incl - ns;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) seg_off[n_y] = carry;
}

__device__ __forceinline__ int seg_row(const int32_t *seg_off, int n_y, int sgl) {
    int lo = 0, hi = n_y;  // largest r with seg_off[r] <= sgl
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (seg_off[mid] <= sgl) lo = mid;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kSegLen) k_tiles_count(const uint2 *__restrict__ rowbin,
                                                         const AxisRanges *__restrict__ ar,
                                                         const int32_t *__restrict__ rowstart,
                                                         const int32_t *__restrict__ seg_off, int n_y, int n_x,
                                                         uint32_t *__restrict__ m2) {
    extern __shared__ uint32_t cnt[];
    const int sgl = blockIdx.x;  // (after an overflow seg_off[n_y] = 0: every block zeroes its slice)
    if (sgl >= seg_off[n_y]) {  // past the real segments: zero one n_x slice of the matrix tail (it is scanned)
        for (int t = threadIdx.x; t < n_x; t += blockDim.x) m2[(int64_t)n_x * sgl + t] = 0u;
        return;
    }
    const int r = seg_row(seg_off, n_y, sgl);
    const int s = sgl - seg_off[r], ns = seg_off[r + 1] - seg_off[r];
    for (int t = threadIdx.x; t < n_x; t += blockDim.x) cnt[t] = 0;
    __syncthreads();
    const int e = rowstart[r] + s * kSegLen + threadIdx.x;
    if (e < rowstart[r + 1] && threadIdx.x < kSegLen) {
        const uint2 v = rowbin[e];
        if (v.y != kMultiX) {
            for (int t = (int)(v.y & 0xFFFFu); t < (int)(v.y >> 16); ++t) atomicAdd(&cnt[t], 1u);
        } else {
            const AxisRanges a = ar[v.x];
#pragma unroll
            for (int k = 0; k < 3; ++k)
                for (int t = (int)(a.x[k] & 0xFFFFu); t < (int)(a.x[k] >> 16); ++t) atomicAdd(&cnt[t], 1u);
        }
    }
    __syncthreads();
    const int64_t base = (int64_t)n_x * seg_off[r] + s;
    for (int t = threadIdx.x; t < n_x; t += blockDim.x) m2[base + (int64_t)t * ns] = cnt[t];
}

// Level-2 scatter, one thread per row-bin entry (a block per segment): every (entry, tile) pair sets entry e's bit in its tile's
// kSegLen-bit membership mask (kW words, shared memory), then its slot is the (tile, segment) start
// plus the number of earlier entries of the segment in that tile, popc of the mask below e (the
// order within a tile is the entries' order in the segment).
constexpr int kW = kSegLen / 32;  // mask words per tile
static_assert(kW % 4 == 0, "the mask is zeroed in 16-byte stores");
__global__ void __launch_bounds__(kSegLen) k_tiles_scatter_mask(const uint2 *__restrict__ rowbin,
                                                                const AxisRanges *__restrict__ ar,
                                                                const int32_t *__restrict__ rowstart,
                                                                const int32_t *__restrict__ seg_off, int n_y, int n_x,
                                                                const uint32_t *__restrict__ p2,
                                                                uint32_t *__restrict__ order,
                                                                int32_t *__restrict__ ranges) {
    extern __shared__ uint32_t smem[];
    uint32_t *mask = smem;             // [kW][n_x] (word-major: the prefix pass reads it conflict-free)
    uint32_t *pre = smem + n_x * kW;   // [kW][n_x]: slot of the first entry of word w in tile t
    const int sgl = blockIdx.x;
    if (sgl >= seg_off[n_y]) return;
    const int tid = threadIdx.x;
    const int r = seg_row(seg_off, n_y, sgl);
    const int s = sgl - seg_off[r], ns = seg_off[r + 1] - seg_off[r];
    const int64_t base = (int64_t)n_x * seg_off[r] + s;
    const int e0 = rowstart[r] + s * kSegLen, m = min(kSegLen, rowstart[r + 1] - e0);
    for (int i = tid; i < n_x * kW / 4; i += kSegLen) reinterpret_cast<uint4 *>(mask)[i] = make_uint4(0u, 0u, 0u, 0u);
    // (tile, segment) starts, loaded up front so their latency overlaps the mask phase
    uint32_t start0 = 0;
    if (tid < n_x) start0 = p2[base + (int64_t)tid * ns];
    uint32_t gid = 0, xr[3] = {0u, 0u, 0u};  // this entry's x ranges (lo | hi << 16)
    if (tid < m) {
        const uint2 v = rowbin[e0 + tid];
        gid = v.x;
        if (v.y != kMultiX) {
            xr[0] = v.y;
        } else {
            const AxisRanges a = ar[v.x];
            xr[0] = a.x[0];
            xr[1] = a.x[1];
            xr[2] = a.x[2];
        }
    }
    __syncthreads();
    const int w = tid >> 5;
    const uint32_t bit = 1u << (tid & 31);
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int t = (int)(xr[k] & 0xFFFFu); t < (int)(xr[k] >> 16); ++t) atomicOr(&mask[w * n_x + t], bit);
    __syncthreads();
    for (int t = tid; t < n_x; t += kSegLen) {
        uint32_t run = t == tid ? start0 : p2[base + (int64_t)t * ns];
        if (s == 0) ranges[r * n_x + t] = (int32_t)run;  // first entry of tile (r, t)
#pragma unroll
        for (int j = 0; j < kW; ++j) {
            pre[j * n_x + t] = run;
            run += __popc(mask[j * n_x + t]);
        }
    }
    __syncthreads();
    const uint32_t below = bit - 1u;
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int t = (int)(xr[k] & 0xFFFFu); t < (int)(xr[k] >> 16); ++t)
            order[pre[w * n_x + t] + __popc(mask[w * n_x + t] & below)] = gid;
}

// status: [0] the frame's error code, [1] sticky overflow flag (cleared by geer_sync), [2..3] the largest
// (entries, rows) of an overflowing frame since (u64 at byte 8).
__global__ void k_check_capacity(const unsigned long long *__restrict__ totals, int64_t cap_entries, int64_t cap_rows,
                                 int *__restrict__ status) {
    if ((int64_t)totals[0] > cap_entries || (int64_t)totals[1] > cap_rows) {
        atomicMax(status, (int)GEER_ERR_OVERFLOW);
        status[1] = 1;
        unsigned long long *mx = reinterpret_cast<unsigned long long *>(status + 2);
        atomicMax(mx + 0, totals[0]);
        atomicMax(mx + 1, totals[1]);
    }
}

}  // namespace

void launch_check_capacity(const unsigned long long *totals, int64_t cap_entries, int64_t cap_rows, int *err,
                           cudaStream_t st) {
    k_check_capacity<<<1, 1, 0, st>>>(totals, cap_entries, cap_rows, err);
}

BinPlan bin_plan(int64_t n, int n_x, int n_y, int64_t n_entries, int64_t n_rows) {
    BinPlan p;
    p.nch = (int)((n + kBinChunk - 1) / kBinChunk);
    p.m1_len = (int64_t)n_y * p.nch;
    // (Gaussian, tile row) pairs, summed by K1 (each holds >= 1 entry, so n_entries bounds it too)
    p.rows_cap = n_rows > 0 && n_rows <= n_entries ? n_rows : n_entries;
    p.seg_cap = (p.rows_cap + kSegLen - 1) / kSegLen + n_y;
    p.m2_len = (int64_t)n_x * p.seg_cap;
    size_t b1 = 0, b2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b1, (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)lmax(p.m1_len, 1));
    cub::DeviceScan::ExclusiveSum(nullptr, b2, (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)lmax(p.m2_len, 1));
    p.temp_bytes = b1 > b2 ? b1 : b2;
    return p;
}

int bin_tiles(const BinPlan &p, const int32_t *gsorted, const AxisRanges *ar, int64_t n, int n_x, int n_y,
              const unsigned long long *d_total, const int *err, uint32_t *m1, uint32_t *p1, uint2 *rowbin,
              int32_t *rowstart, int32_t *seg_off, uint32_t *m2, uint32_t *p2, void *temp, uint32_t *order,
              int32_t *ranges, cudaStream_t st) {
    const int n_tiles = n_x * n_y;
    if (n <= 0) {  // every tile empty
        cudaMemsetAsync(ranges, 0, sizeof(int32_t) * (n_tiles + 1), st);
        return cudaGetLastError() == cudaSuccess ? GEER_OK : GEER_ERR_CUDA;
    }
    if ((size_t)n_y * kRW * 8 > 200 * 1024 || (size_t)n_x * kW * 8 > 200 * 1024) return GEER_ERR_INVALID;
    k_rows_count<<<p.nch, kBinChunk, n_y * 4, st>>>(gsorted, ar, n, n_y, p.nch, m1, err);
    size_t tb = p.temp_bytes;
    cub::DeviceScan::ExclusiveSum(temp, tb, m1, p1, (int)p.m1_len, st);
    const int wsm_rows = n_y * kRW * 2 * 4;
    if (wsm_rows > 48 * 1024)
        cudaFuncSetAttribute(k_rows_scatter_mask, cudaFuncAttributeMaxDynamicSharedMemorySize, wsm_rows);
    k_rows_scatter_mask<<<p.nch, kBinChunk, wsm_rows, st>>>(gsorted, ar, n, n_y, p.nch, p1, rowbin, err);
    k_segments<<<1, 1024, 0, st>>>(m1, p1, n_y, p.nch, rowstart, seg_off, n_tiles, d_total, ranges, err);
    k_tiles_count<<<(unsigned)p.seg_cap, kSegLen, n_x * 4, st>>>(rowbin, ar, rowstart, seg_off, n_y, n_x, m2);
    tb = p.temp_bytes;
    cub::DeviceScan::ExclusiveSum(temp, tb, m2, p2, (int)p.m2_len, st);
    const int wsm_tiles = n_x * kW * 2 * 4;
    if (wsm_tiles > 48 * 1024)
        cudaFuncSetAttribute(k_tiles_scatter_mask, cudaFuncAttributeMaxDynamicSharedMemorySize, wsm_tiles);
    k_tiles_scatter_mask<<<(unsigned)p.seg_cap, kSegLen, wsm_tiles, st>>>(rowbin, ar, rowstart, seg_off, n_y, n_x, p2,
                                                                         order, ranges);
    return cudaGetLastError() == cudaSuccess ? GEER_OK : GEER_ERR_CUDA;
}

}  // namespace geer
