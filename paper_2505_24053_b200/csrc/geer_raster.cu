// geer_raster.cu — K5 forward raster and K6 reverse-order backward raster.
//
// One CTA of 256 threads per raster work item (a tile, or a <=256-pixel chunk
// of an oversized non-BEAP tile); one pixel per thread.  The tile's depth-
// sorted entries are staged into shared memory in batches with cp.async
// (double-buffered in the forward) and every thread walks them front to back:
//
//   d_u = W d, m = o_u x d_u, kappa = |m|^2/|d_u|^2          (core.py:184-199)
//   u = sigma exp(-kappa/2) [kappa <= lam^2], t = min(u, 0.999) (renderer.py:96-105)
//   C += rem t c; rem *= 1 - t; count += t > 0; stop when rem < 1e-4 (renderer.py:107-118)
//
// The per-pair math is written with explicit __f*_rn intrinsics so the
// forward and backward kernels evaluate bit-identical t values (the backward
// recovers T_i = T_{i+1} / (1 - t_i) exactly as the forward multiplied).
// Pairs whose fp32 kappa lies within the per-Gaussian error band of lam^2 are
// re-decided in fp64, so the support cutoff matches the fp64
// reference.  The backward (renderer.py:259-310) walks each pixel's alive
// entries back to front, forms the 16 per-(pixel, Gaussian) partials,
// warp-reduces them with a shuffle transpose, CTA-reduces them in shared
// memory and issues one vector atomic per 4 partials per entry.
#include <cuda_runtime.h>
#include <stdint.h>

#include "geer_common.cuh"
#include "geer_kernels.h"

namespace geer {

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Pixel ray (world frame): fp64 for the cutoff re-check, fp32 for the raster.
template <bool kBEAP>
__device__ __forceinline__ void pixel_ray(const FrameConst &fc, int p, const double2 *col_sc, const double2 *row_sc,
                                          const double *dir64, double d[3]) {
    if (kBEAP) {
        // camera.py:141-155 + renderer.py:77 (dirs_cam @ R_c)
        double2 cs = col_sc[p % fc.width], rs = row_sc[p / fc.width];
        double x = __dmul_rn(cs.x, rs.y), y = __dmul_rn(cs.y, rs.x), z = __dmul_rn(cs.y, rs.y);
        double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
        double dc[3] = {__ddiv_rn(x, n), __ddiv_rn(y, n), __ddiv_rn(z, n)};
        for (int j = 0; j < 3; ++j)  // numpy matmul rounding: fma(a2,b2, fma(a1,b1, a0*b0))
            d[j] = __fma_rn(dc[2], fc.R[2 * 3 + j], __fma_rn(dc[1], fc.R[1 * 3 + j], __dmul_rn(dc[0], fc.R[0 * 3 + j])));
    } else {
        d[0] = dir64[(int64_t)p * 3 + 0];
        d[1] = dir64[(int64_t)p * 3 + 1];
        d[2] = dir64[(int64_t)p * 3 + 2];
    }
}

// fp64 kappa of (Gaussian g, ray d) from the stored parameters, in the
// reference's operation order (renderer.py:78-79,96-101; no contraction).
__device__ __noinline__ double kappa_fp64(const FrameConst &fc, const geer_scene &sc, int64_t g, const double d[3]) {
    double q0 = sc.quats[g * 4 + 0], q1 = sc.quats[g * 4 + 1], q2 = sc.quats[g * 4 + 2], q3 = sc.quats[g * 4 + 3];
    double qn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(q0, q0), __dmul_rn(q1, q1)), __dmul_rn(q2, q2)),
                                     __dmul_rn(q3, q3)));
    double r = __ddiv_rn(q0, qn), i = __ddiv_rn(q1, qn), j = __ddiv_rn(q2, qn), k = __ddiv_rn(q3, qn);
    double rot[9];
    rot[0] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(j, j), __dmul_rn(k, k))));
    rot[1] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(i, j), __dmul_rn(r, k)));
    rot[2] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(i, k), __dmul_rn(r, j)));
    rot[3] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(i, j), __dmul_rn(r, k)));
    rot[4] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(i, i), __dmul_rn(k, k))));
    rot[5] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(j, k), __dmul_rn(r, i)));
    rot[6] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(i, k), __dmul_rn(r, j)));
    rot[7] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(j, k), __dmul_rn(r, i)));
    rot[8] = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(i, i), __dmul_rn(j, j))));
    double s[3], W[9];
    for (int a = 0; a < 3; ++a) s[a] = exp((double)sc.log_scales[g * 3 + a]);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) W[a * 3 + b] = __ddiv_rn(rot[b * 3 + a], s[a]);
    double rel[3];
    for (int a = 0; a < 3; ++a) rel[a] = __dsub_rn(fc.origin[a], (double)sc.means[g * 3 + a]);
    double ou[3], du[3];
    for (int a = 0; a < 3; ++a) {
        ou[a] = __dadd_rn(__dadd_rn(__dmul_rn(W[a * 3 + 0], rel[0]), __dmul_rn(W[a * 3 + 1], rel[1])),
                          __dmul_rn(W[a * 3 + 2], rel[2]));
        du[a] = __dadd_rn(__dadd_rn(__dmul_rn(W[a * 3 + 0], d[0]), __dmul_rn(W[a * 3 + 1], d[1])),
                          __dmul_rn(W[a * 3 + 2], d[2]));
    }
    double m0 = __dsub_rn(__dmul_rn(ou[1], du[2]), __dmul_rn(ou[2], du[1]));
    double m1 = __dsub_rn(__dmul_rn(ou[2], du[0]), __dmul_rn(ou[0], du[2]));
    double m2 = __dsub_rn(__dmul_rn(ou[0], du[1]), __dmul_rn(ou[1], du[0]));
    double dd = __dadd_rn(__dadd_rn(__dmul_rn(du[0], du[0]), __dmul_rn(du[1], du[1])), __dmul_rn(du[2], du[2]));
    double mm = __dadd_rn(__dadd_rn(__dmul_rn(m0, m0), __dmul_rn(m1, m1)), __dmul_rn(m2, m2));
    return __ddiv_rn(mm, dd);
}

struct PairEval {
    float du0, du1, du2, m0, m1, m2, rdd, kap, alpha, u, t;
};

// Shared by forward and backward: identical instruction sequence -> identical bits.
__device__ __forceinline__ void eval_pair(const Payload &P, float dx, float dy, float dz, const FrameConst &fc,
                                          const geer_scene &sc, uint32_t gid, const double d64[3], PairEval &e,
                                          int &rechecks) {
    const float4 r0 = P.r0, r1 = P.r1, r2 = P.r2;
    e.du0 = __fmaf_rn(r0.z, dz, __fmaf_rn(r0.y, dy, __fmul_rn(r0.x, dx)));
    e.du1 = __fmaf_rn(r1.z, dz, __fmaf_rn(r1.y, dy, __fmul_rn(r1.x, dx)));
    e.du2 = __fmaf_rn(r2.z, dz, __fmaf_rn(r2.y, dy, __fmul_rn(r2.x, dx)));
    const float o0 = r0.w, o1 = r1.w, o2 = r2.w;
    e.m0 = __fmaf_rn(o1, e.du2, -__fmul_rn(o2, e.du1));
    e.m1 = __fmaf_rn(o2, e.du0, -__fmul_rn(o0, e.du2));
    e.m2 = __fmaf_rn(o0, e.du1, -__fmul_rn(o1, e.du0));
    const float dd = __fmaf_rn(e.du2, e.du2, __fmaf_rn(e.du1, e.du1, __fmul_rn(e.du0, e.du0)));
    const float mm = __fmaf_rn(e.m2, e.m2, __fmaf_rn(e.m1, e.m1, __fmul_rn(e.m0, e.m0)));
    e.rdd = rcp_approx(dd);
    e.kap = __fmul_rn(mm, e.rdd);
    e.alpha = ex2_approx(__fmul_rn(e.kap, -0.72134752044448170f));  // exp(-kappa/2)
    float u = __fmul_rn(P.col.w, e.alpha);
    if (fc.cutoff) {
        bool inside = e.kap <= fc.lam2f;
        if (fabsf(__fsub_rn(e.kap, fc.lam2f)) <= P.ext.x) {
            inside = kappa_fp64(fc, sc, gid, d64) <= fc.lam2;
            ++rechecks;
        }
        u = inside ? u : 0.0f;
    }
    e.u = u;
    e.t = fminf(u, kMaxBlendTF);
}

// ------------------------------------------------------------------------------ K5

template <bool kBEAP>
__global__ void __launch_bounds__(kRasterThreads, 2)
    k_forward(FrameConst fc, geer_scene sc, const int4 *__restrict__ items, const int32_t *__restrict__ n_items,
              const int32_t *__restrict__ pix_list, const double2 *__restrict__ col_sc,
              const double2 *__restrict__ row_sc, const double *__restrict__ dir64, const int32_t *__restrict__ ranges,
              const uint32_t *__restrict__ order, const Payload *__restrict__ payload, float *__restrict__ color,
              float *__restrict__ remaining, int32_t *__restrict__ count, int32_t *__restrict__ n_eval,
              unsigned long long *__restrict__ rechecks_out) {
    __shared__ Payload sbuf[2][kFwdBatch];
    __shared__ uint32_t sgid[2][kFwdBatch];
    if ((int)blockIdx.x >= *n_items) return;
    const int4 it = items[blockIdx.x];
    const int tid = threadIdx.x;
    const bool valid = tid < it.z;
    const int p = valid ? pix_list[it.y + tid] : 0;
    double d64[3] = {0.0, 0.0, 1.0};
    if (valid) pixel_ray<kBEAP>(fc, p, col_sc, row_sc, dir64, d64);
    const float dx = (float)d64[0], dy = (float)d64[1], dz = (float)d64[2];

    const int e0 = ranges[it.x], e1 = ranges[it.x + 1];
    float cr = 0.f, cg = 0.f, cb = 0.f, rem = 1.0f;
    int cnt = 0, ne = 0, rechecks = 0;
    bool done = !valid;

    auto stage = [&](int buf, int base) {
        const int n = min(kFwdBatch, e1 - base);
        for (int i = tid; i < n * 5; i += kRasterThreads) {
            const int e = i / 5, part = i - e * 5;
            const uint32_t g = __ldg(order + base + e);
            cp_async16(reinterpret_cast<float4 *>(&sbuf[buf][e]) + part, reinterpret_cast<const float4 *>(payload + g) + part);
            if (part == 0) sgid[buf][e] = g;
        }
        cp_async_commit();
    };

    int buf = 0;
    if (e0 < e1) stage(0, e0);
    for (int base = e0; base < e1; base += kFwdBatch) {
        const bool more = base + kFwdBatch < e1;
        if (more) {
            stage(buf ^ 1, base + kFwdBatch);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (!done) {
            const int n = min(kFwdBatch, e1 - base);
            for (int j = 0; j < n; ++j) {
                if (!(rem >= kMinRemainingF)) {  // renderer.py:113 alive test, before the contribution
                    done = true;
                    break;
                }
                ++ne;
                const Payload &P = sbuf[buf][j];
                PairEval e;
                eval_pair(P, dx, dy, dz, fc, sc, sgid[buf][j], d64, e, rechecks);
                const float w = __fmul_rn(rem, e.t);
                cr = __fmaf_rn(w, P.col.x, cr);
                cg = __fmaf_rn(w, P.col.y, cg);
                cb = __fmaf_rn(w, P.col.z, cb);
                rem = __fmul_rn(rem, __fsub_rn(1.0f, e.t));
                cnt += e.t > 0.0f;
            }
        }
        buf ^= 1;
        if (!__syncthreads_or(!done)) break;
    }
    cp_async_wait<0>();  // no copy may be in flight when the CTA retires
    if (valid) {
        // renderer.py:118 background with the final remaining transmittance
        color[(int64_t)p * 3 + 0] = __fmaf_rn(rem, fc.bg[0], cr);
        color[(int64_t)p * 3 + 1] = __fmaf_rn(rem, fc.bg[1], cg);
        color[(int64_t)p * 3 + 2] = __fmaf_rn(rem, fc.bg[2], cb);
        remaining[p] = rem;
        count[p] = cnt;
        n_eval[p] = ne;
    }
    if (rechecks_out) {
        rechecks = __reduce_add_sync(0xffffffffu, rechecks);
        if ((tid & 31) == 0 && rechecks) atomicAdd(rechecks_out, (unsigned long long)rechecks);
    }
}

// ------------------------------------------------------------------------------ K6

// Reduce 16 per-lane values over the warp; afterwards lane L holds the total of
// value index (L >> 1) & 15 (both lanes of a pair hold it).
__device__ __forceinline__ float warp_transpose_reduce16(float v[16], int lane) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const bool hi = lane & 16;
        float send = hi ? v[k] : v[k + 8];
        float keep = hi ? v[k + 8] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const bool hi = lane & 8;
        float send = hi ? v[k] : v[k + 4];
        float keep = hi ? v[k + 4] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const bool hi = lane & 4;
        float send = hi ? v[k] : v[k + 2];
        float keep = hi ? v[k + 2] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    {
        const bool hi = lane & 2;
        float send = hi ? v[0] : v[1];
        float keep = hi ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

template <bool kBEAP>
__global__ void __launch_bounds__(kRasterThreads, 2)
    k_backward(FrameConst fc, geer_scene sc, const int4 *__restrict__ items, const int32_t *__restrict__ n_items,
               const int32_t *__restrict__ pix_list, const double2 *__restrict__ col_sc,
               const double2 *__restrict__ row_sc, const double *__restrict__ dir64,
               const int32_t *__restrict__ ranges, const uint32_t *__restrict__ order,
               const Payload *__restrict__ payload, const float *__restrict__ remaining,
               const int32_t *__restrict__ n_eval, const float *__restrict__ dl_dimage, float4 *__restrict__ accum) {
    constexpr int kWarps = kRasterThreads / 32;
    __shared__ Payload sbuf[kBwdBatch];
    __shared__ uint32_t sgid[kBwdBatch];
    __shared__ float red[kWarps][kBwdBatch][16];
    __shared__ int smax;
    if ((int)blockIdx.x >= *n_items) return;
    const int4 it = items[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool valid = tid < it.z;
    const int p = valid ? pix_list[it.y + tid] : 0;
    double d64[3] = {0.0, 0.0, 1.0};
    if (valid) pixel_ray<kBEAP>(fc, p, col_sc, row_sc, dir64, d64);
    const float dx = (float)d64[0], dy = (float)d64[1], dz = (float)d64[2];
    const int ne = valid ? n_eval[p] : 0;
    const float t_fin = valid ? remaining[p] : 0.f;
    float gl0 = 0.f, gl1 = 0.f, gl2 = 0.f;
    if (valid) {
        gl0 = dl_dimage[(int64_t)p * 3 + 0];
        gl1 = dl_dimage[(int64_t)p * 3 + 1];
        gl2 = dl_dimage[(int64_t)p * 3 + 2];
    }
    // renderer.py:279-280: background term scaled by the final remaining
    const float bgt0 = t_fin * fc.bg[0], bgt1 = t_fin * fc.bg[1], bgt2 = t_fin * fc.bg[2];
    if (tid == 0) smax = 0;
    __syncthreads();
    const int wmax = __reduce_max_sync(0xffffffffu, ne);
    if (lane == 0 && wmax > 0) atomicMax(&smax, wmax);
    __syncthreads();
    const int max_n = smax;
    if (max_n == 0) return;
    const int e0 = ranges[it.x];

    float T = t_fin;                  // transmittance in front of the current entry, walked back
    float s0 = 0.f, s1 = 0.f, s2 = 0.f;  // occlusion suffix (renderer.py:283)
    int dummy = 0;
    for (int hi = max_n; hi > 0; hi -= kBwdBatch) {
        const int lo = max(0, hi - kBwdBatch);
        const int n = hi - lo;
        for (int i = tid; i < n * 5; i += kRasterThreads) {
            const int e = i / 5, part = i - e * 5;
            const uint32_t g = __ldg(order + e0 + lo + e);
            cp_async16(reinterpret_cast<float4 *>(&sbuf[e]) + part, reinterpret_cast<const float4 *>(payload + g) + part);
            if (part == 0) sgid[e] = g;
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        const bool warp_live = __any_sync(0xffffffffu, lo < ne);
        for (int jj = n - 1; jj >= 0; --jj) {
            const int i = lo + jj;
            float v[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = 0.f;
            const bool active = i < ne;
            if (warp_live) {
                if (active) {
                    const Payload &P = sbuf[jj];
                    PairEval e;
                    eval_pair(P, dx, dy, dz, fc, sc, sgid[jj], d64, e, dummy);
                    const float omt = __fsub_rn(1.0f, e.t);
                    const float inv = 1.0f / omt;
                    T = __fdiv_rn(T, omt);  // T_i = T_{i+1} / (1 - t_i)
                    const float w = T * e.t;
                    const float c0 = P.col.x, c1 = P.col.y, c2 = P.col.z;
                    // renderer.py:284-287
                    const float dcdt0 = T * c0 - (s0 + bgt0) * inv;
                    const float dcdt1 = T * c1 - (s1 + bgt1) * inv;
                    const float dcdt2 = T * c2 - (s2 + bgt2) * inv;
                    const float dl_dt = dcdt0 * gl0 + dcdt1 * gl1 + dcdt2 * gl2;
                    s0 += w * c0;
                    s1 += w * c1;
                    s2 += w * c2;
                    v[13] = w * gl0;  // renderer.py:309 dcol
                    v[14] = w * gl1;
                    v[15] = w * gl2;
                    // renderer.py:289-302 (gate: t > 0 and u < 0.999)
                    if (e.t > 0.0f && e.u < kMaxBlendTF) {
                        v[12] = dl_dt * e.alpha;
                        const float dk = -0.5f * dl_dt * e.u;
                        const float coef = 2.0f * dk * e.rdd;  // dl_dm = coef * m
                        const float lm0 = coef * e.m0, lm1 = coef * e.m1, lm2 = coef * e.m2;
                        // dl_do = d_u x dl_dm
                        v[9] = e.du1 * lm2 - e.du2 * lm1;
                        v[10] = e.du2 * lm0 - e.du0 * lm2;
                        v[11] = e.du0 * lm1 - e.du1 * lm0;
                        // dl_dd = -(2 kappa dk / dd) d_u + dl_dm x o_u
                        const float sc_ = e.kap * coef;
                        const float o0 = P.r0.w, o1 = P.r1.w, o2 = P.r2.w;
                        const float dd0 = -sc_ * e.du0 + (lm1 * o2 - lm2 * o1);
                        const float dd1 = -sc_ * e.du1 + (lm2 * o0 - lm0 * o2);
                        const float dd2 = -sc_ * e.du2 + (lm0 * o1 - lm1 * o0);
                        // renderer.py:304 dW_rc = sum_p dl_dd (x) d_p
                        v[0] = dd0 * dx; v[1] = dd0 * dy; v[2] = dd0 * dz;
                        v[3] = dd1 * dx; v[4] = dd1 * dy; v[5] = dd1 * dz;
                        v[6] = dd2 * dx; v[7] = dd2 * dy; v[8] = dd2 * dz;
                    }
                }
                const float tot = warp_transpose_reduce16(v, lane);
                if ((lane & 1) == 0) red[warp][jj][lane >> 1] = tot;
            } else if (lane < 16) {
                red[warp][jj][lane] = 0.f;
            }
        }
        __syncthreads();
        // CTA reduction over warps; one float4 atomic per 4 partials
        for (int idx = tid; idx < n * 4; idx += kRasterThreads) {
            const int jj = idx >> 2, q = idx & 3;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                acc.x += red[w][jj][q * 4 + 0];
                acc.y += red[w][jj][q * 4 + 1];
                acc.z += red[w][jj][q * 4 + 2];
                acc.w += red[w][jj][q * 4 + 3];
            }
            if (acc.x != 0.f || acc.y != 0.f || acc.z != 0.f || acc.w != 0.f)
                atomicAdd(accum + (int64_t)sgid[jj] * 4 + q, acc);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------ small kernels

__global__ void k_sum_i32(const int32_t *v, int64_t n, unsigned long long *out) {
    unsigned long long s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += (unsigned long long)(v[i] > 0 ? v[i] : 0);
    s = __reduce_add_sync(0xffffffffu, (unsigned)s);  // per-thread partials are < 2^32
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}
__global__ void k_f64_f32(const double *in, float *out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)in[i];
}
__global__ void k_f32_f64(const float *in, double *out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}
__global__ void k_i32_i64(const int32_t *in, int64_t *out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)in[i];
}
__global__ void k_fill_bg(FrameConst fc, float *color, float *remaining, int32_t *count, int32_t *n_eval) {
    int64_t npx = (int64_t)fc.width * fc.height;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npx; i += (int64_t)gridDim.x * blockDim.x) {
        color[i * 3 + 0] = fc.bg[0];
        color[i * 3 + 1] = fc.bg[1];
        color[i * 3 + 2] = fc.bg[2];
        remaining[i] = 1.0f;
        count[i] = 0;
        if (n_eval) n_eval[i] = 0;
    }
}

static int grid_for(int64_t n) { return (int)lmin(lmax((n + 255) / 256, 1), 148 * 8); }

void launch_forward(const FrameConst &fc, const geer_scene &sc, int max_items, const int4 *items,
                    const int32_t *n_items, const int32_t *pix_list, const double2 *col_sc, const double2 *row_sc,
                    const double *dir64, const int32_t *ranges, const uint32_t *order, const Payload *payload,
                    float *color, float *remaining, int32_t *count, int32_t *n_eval, unsigned long long *rechecks,
                    cudaStream_t st) {
    if (max_items <= 0) return;
    if (fc.model == GEER_BEAP)
        k_forward<true><<<max_items, kRasterThreads, 0, st>>>(fc, sc, items, n_items, pix_list, col_sc, row_sc, dir64,
                                                              ranges, order, payload, color, remaining, count, n_eval,
                                                              rechecks);
    else
        k_forward<false><<<max_items, kRasterThreads, 0, st>>>(fc, sc, items, n_items, pix_list, col_sc, row_sc, dir64,
                                                               ranges, order, payload, color, remaining, count, n_eval,
                                                               rechecks);
}

void launch_backward(const FrameConst &fc, const geer_scene &sc, int max_items, const int4 *items,
                     const int32_t *n_items, const int32_t *pix_list, const double2 *col_sc, const double2 *row_sc,
                     const double *dir64, const int32_t *ranges, const uint32_t *order, const Payload *payload,
                     const float *remaining, const int32_t *n_eval, const float *dl_dimage, float4 *accum,
                     cudaStream_t st) {
    if (max_items <= 0) return;
    if (fc.model == GEER_BEAP)
        k_backward<true><<<max_items, kRasterThreads, 0, st>>>(fc, sc, items, n_items, pix_list, col_sc, row_sc, dir64,
                                                               ranges, order, payload, remaining, n_eval, dl_dimage,
                                                               accum);
    else
        k_backward<false><<<max_items, kRasterThreads, 0, st>>>(fc, sc, items, n_items, pix_list, col_sc, row_sc,
                                                                dir64, ranges, order, payload, remaining, n_eval,
                                                                dl_dimage, accum);
}

void launch_sum_i32(const int32_t *v, int64_t n, unsigned long long *out, cudaStream_t st) {
    k_sum_i32<<<grid_for(n), 256, 0, st>>>(v, n, out);
}
void launch_convert_f64_f32(const double *in, float *out, int64_t n, cudaStream_t st) {
    if (n > 0) k_f64_f32<<<grid_for(n), 256, 0, st>>>(in, out, n);
}
void launch_convert_f32_f64(const float *in, double *out, int64_t n, cudaStream_t st) {
    if (n > 0) k_f32_f64<<<grid_for(n), 256, 0, st>>>(in, out, n);
}
void launch_convert_i32_i64(const int32_t *in, int64_t *out, int64_t n, cudaStream_t st) {
    if (n > 0) k_i32_i64<<<grid_for(n), 256, 0, st>>>(in, out, n);
}
void launch_fill_background(const FrameConst &fc, float *color, float *remaining, int32_t *count, int32_t *n_eval,
                            cudaStream_t st) {
    int64_t npx = (int64_t)fc.width * fc.height;
    k_fill_bg<<<grid_for(npx), 256, 0, st>>>(fc, color, remaining, count, n_eval);
}

}  // namespace geer
