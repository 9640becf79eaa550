// geer_host.cu — host side of the host-buffer entry points (geer_render_host / _backward_host).
//
// The reference API hands over float64 numpy arrays (scene.py:18-30, renderer.py:24-54) and the device
// path computes from their fp32 rounding.  Shipping the float64 arrays over PCIe and narrowing them on
// the device moved 2x the bytes the device needs (472 MB per 1M-Gaussian frame, PCIe-bound).  Here the
// narrowing runs on the host cores instead, chunk by chunk on a process-wide worker pool, into a pinned
// write-combined staging buffer, and every finished run of chunks is DMA'd while later chunks are still
// being narrowed.  (float)x on the host rounds to nearest-even exactly like the device's cvt.rn.f32.f64
// (no FTZ in either), so the device sees bit-identical fp32 inputs.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <sched.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "geer_host.h"
#include "geer_kernels.h"

namespace geer {
namespace {

// Process-wide pool of host workers (GEER_HOST_THREADS, default: the cores in our affinity mask).  Never torn
// down: worker threads outlive every context and exit with the process.
class Pool {
  public:
    static Pool &get() {
        static Pool *p = new Pool();
        return *p;
    }
    int size() const { return (int)n_; }
    void submit(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> g(m_);
            q_.push_back(std::move(f));
        }
        cv_.notify_one();
    }

  private:
    Pool() {
        int n = (int)std::thread::hardware_concurrency();
        cpu_set_t set;
        if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);  // the cores we may run on
        if (const char *e = getenv("GEER_HOST_THREADS")) n = atoi(e);
        n_ = std::max(1, std::min(n, 128));
        for (int i = 0; i < n_; ++i) std::thread([this] { loop(); }).detach();
    }
    void loop() {
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [this] { return !q_.empty(); });
                f = std::move(q_.front());
                q_.pop_front();
            }
            f();
        }
    }
    int n_ = 1;
    std::mutex m_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
};

constexpr int64_t kChunk = kHostChunk;

// dst[i] = (float)src[i] (round to nearest even, like cvt.rn.f32.f64).  The AVX2 body converts 8
// doubles per step and streams the floats (non-temporal: the staging buffer is write-combined and
// never read back by the host); chosen at run time.
__attribute__((target("avx2"))) void narrow_avx2(const double *src, float *dst, int64_t n) {
    int64_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31); ++i) dst[i] = (float)src[i];
    for (; i + 8 <= n; i += 8) {
        const __m128 a = _mm256_cvtpd_ps(_mm256_loadu_pd(src + i));
        const __m128 b = _mm256_cvtpd_ps(_mm256_loadu_pd(src + i + 4));
        _mm256_stream_ps(dst + i, _mm256_set_m128(b, a));
    }
    for (; i < n; ++i) dst[i] = (float)src[i];
    _mm_sfence();  // the streamed stores are visible before the chunk's done flag
}

// (float64 results streamed past the cache: no read-for-ownership of the caller's output lines)
__attribute__((target("avx2"))) void widen_avx2(const float *src, double *dst, int64_t n) {
    int64_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31); ++i) dst[i] = (double)src[i];
    for (; i + 8 <= n; i += 8) {
        _mm256_stream_pd(dst + i, _mm256_cvtps_pd(_mm_loadu_ps(src + i)));
        _mm256_stream_pd(dst + i + 4, _mm256_cvtps_pd(_mm_loadu_ps(src + i + 4)));
    }
    for (; i < n; ++i) dst[i] = (double)src[i];
    _mm_sfence();
}

void widen_run(const float *src, double *dst, int64_t n) {
    static const bool avx2 = __builtin_cpu_supports("avx2") && !getenv("GEER_HOST_SCALAR");
    if (avx2) {
        widen_avx2(src, dst, n);
    } else {
        for (int64_t i = 0; i < n; ++i) dst[i] = (double)src[i];
    }
}

void narrow_scalar(const double *src, float *dst, int64_t n) {
    for (int64_t i = 0; i < n; ++i) dst[i] = (float)src[i];
}

void narrow_run(const double *src, float *dst, int64_t n) {
    static const bool avx2 = __builtin_cpu_supports("avx2") && !getenv("GEER_HOST_SCALAR");
    if (avx2)
        narrow_avx2(src, dst, n);
    else
        narrow_scalar(src, dst, n);
}

// One host->device upload: the segments concatenated into one index space, cut into chunks that any
// worker (or the calling thread) narrows; shared with the workers so a late one never touches freed state.
struct Job {
    std::vector<HostSeg> segs;
    std::vector<int64_t> off;  // prefix offsets of segs in the concatenated space (size nseg + 1)
    float *staging = nullptr;
    int64_t total = 0;
    int nch = 0;
    std::atomic<int> next{0};
    std::unique_ptr<std::atomic<uint8_t>[]> done;

    void narrow(int c) {
        const int64_t a = (int64_t)c * kChunk, b = std::min(total, a + kChunk);
        for (size_t s = 0; s < segs.size(); ++s) {
            const int64_t lo = std::max(a, off[s]), hi = std::min(b, off[s + 1]);
            if (lo >= hi) continue;
            narrow_run(segs[s].src + (lo - off[s]), staging + lo, hi - lo);
        }
        done[c].store(1, std::memory_order_release);
    }
    // a worker: take chunks in order until none are left
    void drain() {
        for (;;) {
            const int c = next.fetch_add(1, std::memory_order_relaxed);
            if (c >= nch) return;
            narrow(c);
        }
    }
};

}  // namespace

int host_threads() { return Pool::get().size(); }

int64_t raw_upload_elems(int64_t all) {
    static const double frac = [] {
        const char *e = getenv("GEER_HOST_RAW_FRACTION");
        const double f = e ? atof(e) : 0.1;
        return f < 0 ? 0.0 : (f > 1 ? 1.0 : f);
    }();
    const int64_t r = (int64_t)(frac * (double)all);
    return r > 0 ? std::min(all, r + kChunk) : 0;
}

bool is_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

cudaError_t upload_narrowed(const HostSeg *segs, int nseg, float *staging, double *raw_dev, int64_t raw_elems,
                            cudaStream_t st, int64_t *pcie_bytes) {
    auto job = std::make_shared<Job>();
    job->segs.assign(segs, segs + nseg);
    job->off.resize(nseg + 1);
    job->off[0] = 0;
    for (int s = 0; s < nseg; ++s) job->off[s + 1] = job->off[s] + segs[s].n;
    const int64_t all = job->off[nseg];
    // the raw tail [split, all) goes over PCIe as float64 from the caller's (pinned) arrays
    int64_t split = all;
    if (raw_dev && raw_elems > 0) {
        split = (std::max<int64_t>(0, all - raw_elems) + kChunk - 1) / kChunk * kChunk;  // <= raw_elems raw
        split = std::min(split, all);
        for (int s = 0; s < nseg; ++s)
            if (job->off[s + 1] > split && segs[s].n > 0 && !is_pinned(segs[s].src)) split = all;
    }
    job->total = split;
    if (pcie_bytes) *pcie_bytes = (int64_t)sizeof(float) * split + (int64_t)sizeof(double) * (all - split);
    job->staging = staging;
    job->nch = (int)((job->total + kChunk - 1) / kChunk);
    if (job->nch > 0) {
        job->done.reset(new std::atomic<uint8_t>[job->nch]);
        for (int c = 0; c < job->nch; ++c) job->done[c].store(0, std::memory_order_relaxed);
        Pool &pool = Pool::get();
        const int helpers = std::min(pool.size(), job->nch - 1);
        for (int i = 0; i < helpers; ++i) pool.submit([job] { job->drain(); });
    }
    // the raw tail first: its DMA runs while the host narrows the rest
    cudaError_t first_err = cudaSuccess;
    for (int s = 0; s < nseg && first_err == cudaSuccess; ++s) {
        const int64_t lo = std::max(split, job->off[s]), hi = job->off[s + 1];
        if (lo >= hi) continue;
        double *d64 = raw_dev + (lo - split);
        cudaError_t err = cudaMemcpyAsync(d64, segs[s].src + (lo - job->off[s]), sizeof(double) * (size_t)(hi - lo),
                                          cudaMemcpyHostToDevice, st);
        if (err == cudaSuccess) {
            launch_convert_f64_f32(d64, segs[s].dev + (lo - job->off[s]), hi - lo, st);
            err = cudaGetLastError();
        }
        first_err = err;
    }

    // the calling thread copies every finished run of chunks (in order) and narrows when none is ready
    // (after a failed copy the remaining chunks are still narrowed, so no worker writes `staging` late)
    int sent = 0;
    while (sent < job->nch) {
        int e = sent;
        while (e < job->nch && job->done[e].load(std::memory_order_acquire)) ++e;
        if (e > sent) {
            const int64_t a = (int64_t)sent * kChunk, b = std::min(job->total, (int64_t)e * kChunk);
            for (int s = 0; s < nseg; ++s) {
                const int64_t lo = std::max(a, job->off[s]), hi = std::min(b, job->off[s + 1]);
                if (lo >= hi) continue;
                if (first_err != cudaSuccess) continue;
                cudaError_t err = cudaMemcpyAsync(segs[s].dev + (lo - job->off[s]), staging + lo,
                                                  sizeof(float) * (size_t)(hi - lo), cudaMemcpyHostToDevice, st);
                if (err != cudaSuccess && first_err == cudaSuccess) first_err = err;
            }
            sent = e;
            continue;
        }
        const int c = job->next.fetch_add(1, std::memory_order_relaxed);
        if (c < job->nch)
            job->narrow(c);
        else
            std::this_thread::yield();
    }
    return first_err;
}

constexpr int64_t kDownChunk = 1 << 21;  // elements per download chunk (8 MB of fp32)

// One device->host download: chunk c is copied into the staging buffer and recorded on event c;
// whoever takes chunk c (a worker or the caller) waits for that event and widens it.
struct DownJob {
    std::vector<HostOut> outs;
    std::vector<int64_t> off;
    const float *staging = nullptr;
    const cudaEvent_t *evs = nullptr;
    int64_t total = 0;
    int nch = 0;
    std::atomic<int> next{0}, done{0};
    std::atomic<int> err{0};

    void widen(int c) {
        cudaError_t e;
        while ((e = cudaEventQuery(evs[c])) == cudaErrorNotReady) std::this_thread::yield();
        if (e != cudaSuccess) err.store((int)e);
        const int64_t a = (int64_t)c * kDownChunk, b = std::min(total, a + kDownChunk);
        for (size_t s = 0; s < outs.size(); ++s) {
            const int64_t lo = std::max(a, off[s]), hi = std::min(b, off[s + 1]);
            if (lo < hi && e == cudaSuccess) widen_run(staging + lo, outs[s].dst + (lo - off[s]), hi - lo);
        }
        done.fetch_add(1, std::memory_order_release);
    }
    void drain() {
        for (;;) {
            const int c = next.fetch_add(1, std::memory_order_relaxed);
            if (c >= nch) return;
            widen(c);
        }
    }
};

cudaError_t download_widened(const HostOut *outs, int nout, float *staging, std::vector<cudaEvent_t> &evs,
                             cudaStream_t st) {
    auto job = std::make_shared<DownJob>();
    job->outs.assign(outs, outs + nout);
    job->off.resize(nout + 1);
    job->off[0] = 0;
    for (int s = 0; s < nout; ++s) job->off[s + 1] = job->off[s] + outs[s].n;
    job->total = job->off[nout];
    job->staging = staging;
    job->nch = (int)((job->total + kDownChunk - 1) / kDownChunk);
    if (job->nch == 0) return cudaSuccess;
    while ((int)evs.size() < job->nch) {
        cudaEvent_t e;
        cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        if (r != cudaSuccess) return r;
        evs.push_back(e);
    }
    job->evs = evs.data();
    // every chunk's copies, each followed by its event (enqueued before any widening starts)
    for (int c = 0; c < job->nch; ++c) {
        const int64_t a = (int64_t)c * kDownChunk, b = std::min(job->total, a + kDownChunk);
        for (int s = 0; s < nout; ++s) {
            const int64_t lo = std::max(a, job->off[s]), hi = std::min(b, job->off[s + 1]);
            if (lo >= hi) continue;
            cudaError_t r = cudaMemcpyAsync(staging + lo, outs[s].dev + (lo - job->off[s]), sizeof(float) * (size_t)(hi - lo),
                                            cudaMemcpyDeviceToHost, st);
            if (r != cudaSuccess) return r;  // (nothing handed to the workers yet)
        }
        cudaError_t r = cudaEventRecord(evs[c], st);
        if (r != cudaSuccess) return r;
    }
    Pool &pool = Pool::get();
    const int helpers = std::min(pool.size(), job->nch - 1);
    for (int i = 0; i < helpers; ++i) pool.submit([job] { job->drain(); });
    job->drain();
    while (job->done.load(std::memory_order_acquire) < job->nch) std::this_thread::yield();
    return (cudaError_t)job->err.load();
}

}  // namespace geer
