// geer_host.h — host-core staging of the host-buffer entry points (see geer_host.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace geer {

constexpr int64_t kHostChunk = 1 << 19;  // elements per narrowing chunk (2 MB of fp32)

struct HostSeg {
    const double *src;  // host float64 array
    int64_t n;          // elements
    float *dev;         // its fp32 device destination
};

// Narrow the segments to fp32 on the host worker pool into `staging` (pinned, >= sum of n floats,
// concatenated layout) and copy each finished run to its device destination on `st`.  The last
// ~raw_elems elements (whole chunks; only when their source arrays are pinned) instead go over PCIe as
// float64 into `raw_dev` and are narrowed on the device, which balances host memory bandwidth against
// PCIe bytes.  Returns with every copy enqueued; the caller synchronises `st` before reusing `staging`.
cudaError_t upload_narrowed(const HostSeg *segs, int nseg, float *staging, double *raw_dev, int64_t raw_elems,
                            cudaStream_t st, int64_t *pcie_bytes);

// Elements of a scene upload sent raw (float64): GEER_HOST_RAW_FRACTION of them (default 0.1,
// the measured optimum on the B200 box: profiles/r02_e2e_host_staging.md),
// rounded to whole chunks by upload_narrowed; raw_dev must hold raw_upload_elems(all) doubles.
int64_t raw_upload_elems(int64_t all);

int host_threads();

struct HostOut {
    const float *dev;  // fp32 device array
    int64_t n;         // elements
    double *dst;       // its host float64 destination
};

// Copy the device arrays into `staging` (pinned, cached, >= sum of n floats) chunk by chunk on `st`
// and widen each chunk into its float64 destination (exact) on the host pool as soon as it lands.
// Returns when every destination is written.  `evs` grows to one event per chunk (owned by the caller).
cudaError_t download_widened(const HostOut *outs, int nout, float *staging, std::vector<cudaEvent_t> &evs,
                             cudaStream_t st);

}  // namespace geer
