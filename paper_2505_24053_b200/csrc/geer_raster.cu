// geer_raster.cu — K5 forward raster and K6 reverse-order backward raster.
//
// One CTA per raster work item (a tile, or a <=256-pixel chunk of an oversized non-BEAP tile): a
// producer warp streams the tile's depth-sorted payload rows into a 3-stage shared-memory ring with
// TMA gather4 copies completed on mbarriers and turns each into an offset record, and 8 consumer warps
// (one pixel per lane, an 8x4 patch per warp) cull each stage against their patch, then walk the kept
// entries front to back:
//
//   d_u = W d, m = o_u x d_u from the item's offset records (fp64 products rounded once; see
//   make_record), kappa = |m|^2/|d_u|^2                       (core.py:184-199)
//   u = sigma exp(-kappa/2) [kappa <= lam^2], t = min(u, 0.999) (renderer.py:96-105)
//   C += rem t c; rem *= 1 - t; count += t > 0; stop when rem < 1e-4 (renderer.py:107-118)
//
// The per-pair math is written with explicit __f*_rn intrinsics so the forward and backward kernels
// evaluate bit-identical t values (the backward recovers T_i = T_{i+1} / (1 - t_i) exactly as the
// forward multiplied).  Pairs whose fp32 kappa lies within the error band of lam^2 are re-decided in
// fp64, and pixels whose stop test is too close to call are recomposited in fp64 by
// k_fixup, so cutoff decisions and contributor counts match the fp64 reference.  The backward
// (renderer.py:259-310) streams each tile's alive prefix back to front, forms the 16
// per-(pixel, Gaussian) partials, reduces them over the warp through a shared-memory transpose and
// issues one fp32 atomic per (entry, partial).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

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

// Pixel ray (world frame, fp64; camera.py:141-155 + renderer.py:77, or the K0 ray table).
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
__device__ __noinline__ double kappa_fp64(const float *__restrict__ means, const float *__restrict__ log_scales,
                                          const float *__restrict__ quats, double ox, double oy, double oz, int64_t g,
                                          double dx, double dy, double dz) {
    const double origin[3] = {ox, oy, oz};
    const double d[3] = {dx, dy, dz};
    double q0 = quats[g * 4 + 0], q1 = quats[g * 4 + 1], q2 = quats[g * 4 + 2], q3 = quats[g * 4 + 3];
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
    for (int a = 0; a < 3; ++a) s[a] = exp((double)log_scales[g * 3 + a]);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) W[a * 3 + b] = __ddiv_rn(rot[b * 3 + a], s[a]);
    double rel[3];
    for (int a = 0; a < 3; ++a) rel[a] = __dsub_rn(origin[a], (double)means[g * 3 + a]);
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

struct PairT {
    float kap, alpha, u, t, dd;
};

// |d_u|^2 and |m|^2 of (payload P, ray d) in fp64 via the cross product d_u = W d, m = o_u x d_u
// (core.py:184-199; explicit fma: the same rounding in every kernel that calls it).
__device__ __forceinline__ void norms64(const Payload &P, const double *dray, double &dd, double &mm) {
    const double d0 = dray[0], d1 = dray[1], d2 = dray[2];
    const double u0 = fma(P.q[2], d2, fma(P.q[1], d1, P.q[0] * d0));
    const double u1 = fma(P.q[5], d2, fma(P.q[4], d1, P.q[3] * d0));
    const double u2 = fma(P.q[8], d2, fma(P.q[7], d1, P.q[6] * d0));
    const double o0 = P.q[9], o1 = P.q[10], o2 = P.q[11];
    const double x0 = fma(o1, u2, -(o2 * u1)), x1 = fma(o2, u0, -(o0 * u2)), x2 = fma(o0, u1, -(o1 * u0));
    dd = fma(u2, u2, fma(u1, u1, u0 * u0));
    mm = fma(x2, x2, fma(x1, x1, x0 * x0));
}

// Blend quantities of a pair from its fp64 norms (fp32 from here on; the fp64 path of items without an
// offset frame):  u = sigma exp(-kappa/2) [kappa <= lam^2], t = min(u, 0.999)   (renderer.py:96-105)
// Returns true when the cutoff decision lies within the fp64 evaluation's own error bound (the
// forward then hands the pixel to the fp64 fix-up, which uses the reference formulation).
__device__ __forceinline__ bool finish_t(double dd, double mm, const Payload &P, const FrameConst &fc, PairT &e,
                                         int &rechecks) {
    const float sw = P.col.w;
    const float ddf = (float)dd;
    e.dd = ddf;
    e.kap = __fmul_rn((float)mm, rcp_approx(ddf));
    e.alpha = ex2_approx(__fmul_rn(e.kap, -0.72134752044448170f));  // exp(-kappa/2)
    float u = __fmul_rn(sw, e.alpha);
    bool uncertain = false;
    if (fc.cutoff) {
        bool inside = e.kap <= fc.lam2f;
        // kappa_fp32 carries ~3e-7 relative error plus the fp64 evaluation's bound ext.x: re-decide near lam^2
        if (fabsf(__fsub_rn(e.kap, fc.lam2f)) <= fc.cutoff_tol + P.ext.x) {
            const double k64 = mm / dd;
            inside = k64 <= fc.lam2;
            uncertain = fabs(k64 - fc.lam2) <= (double)P.ext.x;
            ++rechecks;
        }
        u = inside ? u : 0.0f;
    }
    e.u = u;
    e.t = fminf(u, kMaxBlendTF);
    return uncertain;
}

// Shared verbatim by the forward and backward kernels, so t is bit-identical in both.
__device__ __forceinline__ bool eval_t(const Payload &P, const double *dray, const FrameConst &fc, PairT &e,
                                       int &rechecks) {
    double dd, mm;
    norms64(P, dray, dd, mm);
    return finish_t(dd, mm, P, fc, e, rechecks);
}

// Relative bound on |t_fp32 - t_exact| / t for a pair of the fp64 path (fp64 kappa rounded to fp32, rcp/ex2 approximations).
__device__ __forceinline__ float t_rel_bound(float kap) { return 6e-7f + 3e-7f * kap; }

// ------------------------------------------------------------------------------ offset records
//
// Within a work item every pixel ray is d' = dc + x e1 + y e2 (ItemFrame), so per (item, Gaussian)
//   d_u = W d' = a + x b + y c           (a = W dc, b = W e1, c = W e2)
//   m   = o_u x d_u = ma + x mb + y mc   (ma = o_u x a, ...)
// The producer warp turns each streamed payload into a record of these vectors (fp64 products
// rounded once to fp32, m scaled by sqrt(kHalfLog2e)), the quadratic |d_u|^2 = D0 + D1 x + D2 y +
// D3 x^2 + D4 x y + D5 y^2 and two error bounds; per pair the consumers then evaluate
//   dd = |d_u|^2 (5 FFMA),  m (6 FFMA),  k = |m|^2 / dd = kHalfLog2e kappa,  u = sigma 2^-k
// in fp32.  The offsets x, y stay small (|x|, |y| <= ~0.02 for a 16-px tile), so the cancellation
// of the reference's cross product (o_u x d_u with |o_u| up to ~1e3) happens in fp64 once per
// (item, Gaussian), not per pair.  Record layout (float4 units):
//   [0] D0 D1 D2 D3   [1] D4 D5 sigma tol   [2] ma0 mb0 mc0 trel   [3] ma1 mb1 mc1 -   [4] ma2 mb2 mc2 -
//   [5] r g b -       backward only: [6] a0 b0 c0 ou0   [7] a1 b1 c1 ou1   [8] a2 b2 c2 ou2
// tol bounds |k_fp32 - kHalfLog2e kappa_ref| near the cutoff (pairs within tol of it are re-decided
// from the fp64 payload), trel bounds the relative error of t on the pairs that contribute.
constexpr int kRecF = 24;  // forward record floats
constexpr int kRecB = 36;  // backward record floats

// Offset coordinates of a pixel ray d in an item frame (x, y of d / (d . dc)).
__device__ __forceinline__ float2 pixel_xy(const ItemFrame &F, const double d[3]) {
    const double den = __fma_rn(d[2], F.dc[2], __fma_rn(d[1], F.dc[1], __dmul_rn(d[0], F.dc[0])));
    const double nx = __fma_rn(d[2], F.e1[2], __fma_rn(d[1], F.e1[1], __dmul_rn(d[0], F.e1[0])));
    const double ny = __fma_rn(d[2], F.e2[2], __fma_rn(d[1], F.e2[1], __dmul_rn(d[0], F.e2[0])));
    return make_float2((float)__ddiv_rn(nx, den), (float)__ddiv_rn(ny, den));
}

// A pixel's offsets: x, y (each duplicated into a pair for the packed fp32 FMAs) and the products.
struct PixXY {
    float2 x2, y2;
    float xx, xy, yy;
};
__device__ __forceinline__ PixXY make_pxy(float2 v) {
    return PixXY{make_float2(v.x, v.x), make_float2(v.y, v.y), __fmul_rn(v.x, v.x), __fmul_rn(v.x, v.y),
                 __fmul_rn(v.y, v.y)};
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// The record of payload P in frame F (one producer lane per entry; noinline: the forward and backward
// kernels run this one compiled body, so their records - and hence t - are bit-identical).  Only the
// cross product that cancels, ma = o_u x W dc (|o_u| up to ~1e3, |ma| down to ~0 for a Gaussian on
// the item's centre ray), is formed in fp64; the offset terms (x mb + y mc, |x|, |y| <= rx, ry) and
// the quadratic's coefficients are fp32, and their rounding is charged to the bounds (which carry
// a 1.5x margin, covering the approximate sqrt / rcp used to form them).
__device__ __noinline__ void make_record(const Payload &P, const ItemFrame &F, float thrk, float *rec, int grad) {
    const double *W = P.q;
    double a[3], b[3], c[3];
    float wmin2 = INFINITY;  // sigma_min(W)^2 = min row norm^2 (W = S^-1 R^T)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double w0 = W[i * 3 + 0], w1 = W[i * 3 + 1], w2 = W[i * 3 + 2];
        a[i] = __fma_rn(w2, F.dc[2], __fma_rn(w1, F.dc[1], __dmul_rn(w0, F.dc[0])));
        b[i] = __fma_rn(w2, F.e1[2], __fma_rn(w1, F.e1[1], __dmul_rn(w0, F.e1[0])));
        c[i] = __fma_rn(w2, F.e2[2], __fma_rn(w1, F.e2[1], __dmul_rn(w0, F.e2[0])));
        const float f0 = (float)w0, f1 = (float)w1, f2 = (float)w2;
        wmin2 = fminf(wmin2, f0 * f0 + f1 * f1 + f2 * f2);
    }
    // m = (o_u sqrt(kHalfLog2e)) x (a + x b + y c): the cancelling cross products in fp64
    const double o0 = __dmul_rn(P.q[9], kSqrtHalfLog2e), o1 = __dmul_rn(P.q[10], kSqrtHalfLog2e),
                 o2 = __dmul_rn(P.q[11], kSqrtHalfLog2e);
    auto cross = [&](const double *v, float *m) {
        m[0] = (float)__fma_rn(o1, v[2], -__dmul_rn(o2, v[1]));
        m[1] = (float)__fma_rn(o2, v[0], -__dmul_rn(o0, v[2]));
        m[2] = (float)__fma_rn(o0, v[1], -__dmul_rn(o1, v[0]));
    };
    float ma[3], mb[3], mc[3];
    cross(a, ma);
    cross(b, mb);
    cross(c, mc);
    const float af[3] = {(float)a[0], (float)a[1], (float)a[2]}, bf[3] = {(float)b[0], (float)b[1], (float)b[2]},
                cf[3] = {(float)c[0], (float)c[1], (float)c[2]};
    auto dot = [](const float *x, const float *y) {
        return __fmaf_rn(x[2], y[2], __fmaf_rn(x[1], y[1], __fmul_rn(x[0], y[0])));
    };
    const float D0 = dot(af, af), D1 = 2.0f * dot(af, bf), D2 = 2.0f * dot(af, cf);
    const float D3 = dot(bf, bf), D4 = 2.0f * dot(bf, cf), D5 = dot(cf, cf);
    // error bounds (u = 2^-24):
    //   |d dd| <= 16 u Sd, Sd = (|a| + rx |b| + ry |c|)^2  (coefficients from the rounded vectors,
    //   offsets, 5 FMA);  |d m| <= 4 u (|ma| + rx |mb| + ry |mc|)  (rounding of the fp64 products,
    //   offsets, 2 FMA);  dd >= ddlo over the item;  at k = thrk
    //   |d k| <= (2 sqrt(k dd) |d m| + |d m|^2 + k |d dd|) / dd + 6 u k   (rcp.approx + products),
    // plus the reference's own fp64 error ext.x.
    const float rx = F.rx, ry = F.ry, u = 5.9604645e-8f;
    const float na = sqrt_approx(D0), nb = sqrt_approx(D3), nc = sqrt_approx(D5);
    const float lin = na - rx * nb - ry * nc;
    const float ddlo = fmaxf(lin > 0.f ? 0.999f * lin * lin : 0.f, 0.98f * wmin2);  // |d'| >= 1
    const float idd = rcp_approx(ddlo);
    const float sd = (na + rx * nb + ry * nc) * (na + rx * nb + ry * nc);
    const float dm = 4.0f * u * (sqrt_approx(dot(ma, ma)) + rx * sqrt_approx(dot(mb, mb)) + ry * sqrt_approx(dot(mc, mc)));
    const float tol = 1.5f * (2.0f * sqrt_approx(thrk * idd) * dm + dm * dm * idd + thrk * (6.0f * u + 16.0f * u * sd * idd)) +
                      (float)kHalfLog2e * P.ext.x + 1e-30f;
    float4 *r4 = reinterpret_cast<float4 *>(rec);
    const float sig = P.col.w;
    // layout (rec_k): the coefficients that rec_k's packed FMAs combine sit side by side
    //   r4[0] = (ma0, ma1, mb0, mb1)   r4[1] = (mc0, mc1, ma2, D0)   r4[2] = (mb2, D1, mc2, D2)
    //   r4[3] = (D3, D4, D5, trel)     r4[4] = (sigma, tol, 0, 0)    r4[5] = colour
    //   backward: r4[6] = (a0, a1, b0, b1)   r4[7] = (c0, c1, a2, b2)   r4[8] = (c2, o_u)
    if (!(tol < 0.25f * thrk) || !(sd < 1e36f) || !(dm < 1e-3f * 1e18f)) {
        // fp32 cannot carry this Gaussian here (huge or degenerate W / o_u): every pair goes to the fp64
        // re-check (k = 0 lies within an infinite tol of the cutoff)
        r4[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        r4[1] = make_float4(0.f, 0.f, 0.f, 1.f);
        r4[2] = make_float4(0.f, 0.f, 0.f, 0.f);
        r4[3] = make_float4(0.f, 0.f, 0.f, 1e-5f);
        r4[4] = make_float4(sig, INFINITY, 0.f, 0.f);
    } else {
        r4[0] = make_float4(ma[0], ma[1], mb[0], mb[1]);
        r4[1] = make_float4(mc[0], mc[1], ma[2], D0);
        r4[2] = make_float4(mb[2], D1, mc[2], D2);
        r4[3] = make_float4(D3, D4, D5, 0.6931472f * tol + 1e-6f);
        r4[4] = make_float4(sig, tol, 0.f, 0.f);
    }
    r4[5] = make_float4(P.col.x, P.col.y, P.col.z, 0.f);
    if (grad) {
        r4[6] = make_float4(af[0], af[1], bf[0], bf[1]);
        r4[7] = make_float4(cf[0], cf[1], af[2], bf[2]);
        r4[8] = make_float4(cf[2], (float)P.q[9], (float)P.q[10], (float)P.q[11]);
    }
}

// ------------------------------------------------------------------------------ pipeline plumbing
//
// Each raster CTA = kConsumerWarps consumer warps (one pixel per lane) + 1 producer warp.  The
// producer streams the tile's entries through a ring of kStages shared-memory stages: it gathers
// the payload rows with TMA gather4 (completion counted on the stage's "landed" mbarrier), turns
// each into an offset record and then arrives on the stage's "full" mbarrier; the consumer warps
// release a stage through its "empty" mbarrier.  Consumer warps never meet at a CTA barrier: each
// warp retires as soon as its own 32 pixels are opaque, and the producer stops streaming once every
// consumer warp is done.

constexpr int kConsumerWarps = kRasterThreads / 32;  // 8
#ifndef GEER_STAGES
#define GEER_STAGES 3
#endif
constexpr int kStages = GEER_STAGES;
constexpr int kStageEntries = 32;  // one entry per producer lane
constexpr int kPipeThreads = kRasterThreads + 32;
#ifndef FWD_MIN_BLOCKS
#define FWD_MIN_BLOCKS 3
#endif

constexpr int kRingGroupBytes = 768;    // 4 x 176-B payloads (704 B), padded to a multiple of 128
constexpr int kRingGroups = kStageEntries / 4 + 1;
static_assert(sizeof(Payload) * 4 <= kRingGroupBytes, "ring layout");

template <bool kGrad>
struct __align__(128) PipeSmem {
    static constexpr int kNW = kConsumerWarps;
    static constexpr int kRec = kGrad ? kRecB : kRecF;
    // Entries land in groups of 4 (one TMA gather4 per group), each group 128-B aligned; group
    // kStageEntries / 4 holds the null entry (t = 0 for every ray).  Use ring_at.
    alignas(128) unsigned char ring[kStages][kRingGroups][kRingGroupBytes];
    alignas(16) float rec[kStages][kStageEntries][kRec];  // offset records (producer -> consumers)
    ItemFrame frame;                                        // the item's frame (producer copy)
    float4 wc[kNW][2];                                      // per consumer warp: culling patch, cone
    alignas(16) float red[kGrad ? kNW : 1][16][36];         // backward: per-warp transpose of the 16 partials
    uint32_t gid[kStages][kStageEntries];
    int count[kStages];  // entries in the stage; 0 = end of stream
    uint8_t idx[kStages][kNW][kStageEntries + 4];  // per warp: its kept entries, padded with null slots
    unsigned long long landed[kStages];  // TMA fill complete
    unsigned long long full[kStages];    // records written (consumers may read the stage)
    unsigned long long empty[kStages];
    int done_warps;
    int stop;  // producer will not fill any more stages
};

// The pipeline state lives at the start of the dynamic shared window, declared __align__(128) (TMA
// destinations; the compiler places the window after the static allocations at that alignment, so
// every member sits at a fixed offset).  Launches still reserve sizeof + 128 bytes.

__device__ __forceinline__ uint32_t ring_off(int j) { return (uint32_t)((j >> 2) * kRingGroupBytes + (j & 3) * (int)sizeof(Payload)); }
template <class Smem>
__device__ __forceinline__ Payload &ring_at(Smem &S, int s, int j) {
    return *reinterpret_cast<Payload *>(&S.ring[s][0][0] + ring_off(j));
}

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_drop(unsigned long long *bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive_drop.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long *bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
#ifdef GEER_WATCHDOG
// Diagnosis build: a barrier wait that lasts over 2 s prints where it is stuck and traps.
__device__ __forceinline__ unsigned long long wd_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __noinline__ void wd_wait(unsigned long long *bar, unsigned parity, int tag) {
    const unsigned long long t0 = wd_now();
    for (;;) {
        unsigned ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (wd_now() - t0 > 2000000000ull) {
            printf("WATCHDOG tag %d block %d thread %d bar %p parity %u\n", tag, (int)blockIdx.x, (int)threadIdx.x,
                   (void *)bar, parity);
            __trap();
        }
    }
}
#endif

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
#ifdef GEER_WATCHDOG
    wd_wait(bar, parity, 1);
    return;
#endif
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Wait with a suspend-time hint: the waiting warp sleeps in the barrier (woken when the phase
// completes or after ~ns) instead of spinning; used by the producer, whose spinning would take
// issue slots from the consumer warps it waits for.
__device__ __forceinline__ void mbar_wait_suspend(unsigned long long *bar, unsigned parity) {
#ifndef GEER_PRODUCER_SUSPEND_NS
#define GEER_PRODUCER_SUSPEND_NS 20000
#endif
#ifdef GEER_WATCHDOG
    wd_wait(bar, parity, 2);
    return;
#endif
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITS_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(GEER_PRODUCER_SUSPEND_NS)
        : "memory");
}
// One probe with a suspend-time hint (the producer's idle sleep; the result is not needed).
__device__ __forceinline__ void mbar_try_wait_suspend(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(GEER_PRODUCER_SUSPEND_NS)
        : "memory");
}
// TMA gather4: rows r[0..3] of a 2D row-major tensor (one row = one payload) into 4 consecutive
// rows at dst (128-B aligned), completion counted on bar (sm_100a UTMALDG.2D.GATHER4).
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *map, const uint32_t r[4],
                                            unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(smem_u32(bar))
        : "memory");
}

template <class Smem>
__device__ __forceinline__ void pipe_init(Smem &S) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&S.landed[s], 1);
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], Smem::kNW);
        }
        S.done_warps = 0;
        S.stop = 0;
        // null entry: W = I, o_u = 0, sigma = 0  ->  kappa = 0, t = 0 exactly (a no-op)
        for (int s = 0; s < kStages; ++s) {
            Payload &z = ring_at(S, s, kStageEntries);
            for (int i = 0; i < 12; ++i) z.q[i] = (i == 0 || i == 4 || i == 8) ? 1.0 : 0.0;
            z.col = make_float4(0.f, 0.f, 0.f, 0.f);
            z.ext = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
}

// True when no ray of a warp's cone can meet the Gaussian's lam-ellipsoid along its full line.
// A ray d meets it iff g(d) = d^T K d >= 0 (K from k_preprocess: the ellipsoid's visual cone,
// equivalent to kappa(d) <= lam^2).  For unit d within angle beta <= 45 deg of the cone axis c:
// g(d) <= cos^2(beta) g(c) + sin(2 beta) |P_perp K c| + sin^2(beta) lambda_max(K)  (for g(c) < 0).
// The test is made on squares, with a margin far above the fp32 error of K (entries <= ~1 after
// normalisation).  pc = (c, cos^2 beta); tb.z = lambda_max bound (+inf: never culled).
__device__ __forceinline__ bool cone_misses(const float4 &ta, const float4 &tb, const float4 &pc) {
    const float t00 = ta.x, t11 = ta.y, t22 = ta.z, t01 = ta.w, t02 = tb.x, t12 = tb.y, lmax = tb.z;  // K entries
    const float tc0 = t00 * pc.x + t01 * pc.y + t02 * pc.z;
    const float tc1 = t01 * pc.x + t11 * pc.y + t12 * pc.z;
    const float tc2 = t02 * pc.x + t12 * pc.y + t22 * pc.z;
    const float gc = tc0 * pc.x + tc1 * pc.y + tc2 * pc.z;
    const float p2 = fmaxf(tc0 * tc0 + tc1 * tc1 + tc2 * tc2 - gc * gc, 0.0f);  // |P_perp T c|^2
    const float c2 = pc.w, s2 = 1.0f - pc.w;                                      // cos^2, sin^2 beta
    const float tnorm = fabsf(t00) + fabsf(t11) + fabsf(t22) + 2.0f * (fabsf(t01) + fabsf(t02) + fabsf(t12));
    const float lhs = c2 * gc + s2 * fmaxf(lmax, 0.0f) + 1e-5f * tnorm + 1e-30f;  // must be < -sin(2b) p
    return lhs < 0.0f && lhs * lhs > 4.0f * s2 * c2 * p2;                          // sin^2(2b) = 4 s2 c2
}

// Producer warp: stream entries [first, first + n_total) (forward order) or the same range walked
// from the back (reverse) in stages of kStageEntries, then an end-of-stream sentinel (count 0).  It
// runs a non-blocking loop over two queues: issue the next fill (TMA gather4, completion on
// "landed") as soon as its slot is free, and finish the oldest landed fill (records written, "full"
// arrived), so neither a slow consumer warp nor a pending gather holds up the other queue.
// with_rec = false (items without a frame): no records, a fill is full once it has landed.
template <bool kReverse, class Smem>
__device__ __forceinline__ void pipe_produce(Smem &S, const uint32_t *__restrict__ order, const CUtensorMap *pay_map,
                                             float thrk, bool with_rec, int first, int n_total, bool stop_when_done,
                                             unsigned long long *streamed = nullptr) {
    constexpr bool kGrad = Smem::kRec == kRecB;
    const unsigned per_group = (unsigned)(4 * sizeof(Payload));
    const int lane = threadIdx.x & 31;
    const int n_fills = (n_total + kStageEntries - 1) / kStageEntries;
    // gid of this lane's entry in fill bb (the order load runs one fill ahead of the copies)
    auto load_gid = [&](int bb) -> uint32_t {
        const int done = kStageEntries * bb;
        const int n = min(kStageEntries, n_total - done);
        const int base = kReverse ? first + n_total - done - n : first + done;
        return lane < n ? __ldg(order + base + lane) : 0u;
    };
    // warp-uniform barrier probes (a completed phase stays complete until we act on the slot again)
    auto ready = [&](unsigned long long *bar, unsigned parity) {
        return __shfl_sync(0xffffffffu, (int)mbar_try_wait(bar, parity), 0) != 0;
    };
    int next = 0, fin = 0;  // next fill to issue (n_fills: the sentinel), oldest fill not yet full
    uint32_t g_next = load_gid(0);
#ifdef GEER_WATCHDOG
    unsigned long long t_prog = wd_now();
#endif
    for (;;) {
        // every consumer left (lane 0's reading, broadcast: the warp must take this branch as one)
        if (stop_when_done && __shfl_sync(0xffffffffu, *((volatile int *)&S.done_warps), 0) == Smem::kNW) break;
        bool progress = false;
        if (next <= n_fills && ready(&S.empty[next % kStages], ((next / kStages) & 1) ^ 1)) {
            const int s = next % kStages;
            if (next == n_fills) {  // sentinel
                if (lane == 0) {
                    S.count[s] = 0;
                    mbar_arrive(&S.full[s]);
                }
            } else {
                const int n = min(kStageEntries, n_total - kStageEntries * next);
                const uint32_t g = g_next;
                if (next + 1 < n_fills) g_next = load_gid(next + 1);
                if (lane < n) S.gid[s][lane] = g;
                __syncwarp();
                if (lane == 0) {
                    S.count[s] = n;
                    mbar_arrive_expect_tx(&S.landed[s], ((n + 3) >> 2) * per_group);
                }
                __syncwarp();
                // lane k < ceil(n / 4) gathers rows of entries 4k..4k+3 (a partial last group repeats
                // its last entry, so every gather moves 4 whole rows)
                uint32_t rows[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) rows[q] = __shfl_sync(0xffffffffu, g, min(4 * (lane & 7) + q, n - 1));
                if (lane < ((n + 3) >> 2)) tma_gather4(&S.ring[s][lane][0], pay_map, rows, &S.landed[s]);
            }
            ++next;
            progress = true;
        }
        const int issued = min(next, n_fills);
        if (fin < issued && ready(&S.landed[fin % kStages], (fin / kStages) & 1)) {
            const int sp = fin % kStages;
            if (with_rec && lane < S.count[sp]) make_record(ring_at(S, sp, lane), S.frame, thrk, &S.rec[sp][lane][0], kGrad);
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.full[sp]);
            ++fin;
            progress = true;
        }
        if (next > n_fills && fin == n_fills) break;
#ifdef GEER_WATCHDOG
        if (progress) t_prog = wd_now();
        else if (wd_now() - t_prog > 2000000000ull) {
            if (lane == 0)
                printf("WATCHDOG producer block %d next %d fin %d n_fills %d done %d count0 %d\n", (int)blockIdx.x, next,
                       fin, n_fills, *((volatile int *)&S.done_warps), S.count[0]);
            __trap();
        }
#endif
        if (!progress) {  // sleep on the gather we wait for, else on the slot we wait for
            if (fin < issued)
                mbar_try_wait_suspend(&S.landed[fin % kStages], (fin / kStages) & 1);
            else
                mbar_try_wait_suspend(&S.empty[next % kStages], ((next / kStages) & 1) ^ 1);
        }
    }
    if (lane == 0) *((volatile int *)&S.stop) = 1;
    const int issued = min(next, n_fills);
    if (streamed && lane == 0) atomicAdd(streamed, (unsigned long long)min(n_total, kStageEntries * issued));
    // No bulk copy may still be writing shared memory when the CTA retires: wait for the fills not
    // yet finished (each is the latest fill of its slot).
    for (int f = fin; f < issued; ++f) mbar_wait(&S.landed[f % kStages], (f / kStages) & 1);
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

constexpr uint32_t kColOff = 96;  // offsetof(Payload, col)
constexpr uint32_t kExtOff = 112; // offsetof(Payload, ext)
constexpr uint32_t kCullOff = 128;  // offsetof(Payload, cull)
static_assert(offsetof(Payload, col) == kColOff && offsetof(Payload, ext) == kExtOff &&
              offsetof(Payload, cull) == kCullOff, "payload layout");

// Per-warp culling of one stage (run by the consumer warp itself, one entry per lane): an entry is
// kept unless its PBF hull misses the warp's mirror-space patch or its visual cone misses the warp's
// ray cone (both conservative: a dropped entry has kappa > lam^2, i.e. t = 0, on every pixel of the
// warp).  Writes the warp's compacted, null-padded entry list; returns the kept count and (via m)
// the kept mask.
template <class Smem>
__device__ __forceinline__ int stage_keep(Smem &S, int s, int warp, int lane, int n, bool cull, uint32_t &m) {
    const uint32_t pa = smem_u32(&S.ring[s][0][0]) + ring_off(lane);  // this lane's entry of the stage
    bool ov = lane < n;
    if (cull && ov) {
        const float4 patch = S.wc[warp][0], pcone = S.wc[warp][1];
        const float4 bx = lds_f4(pa + kCullOff), k0 = lds_f4(pa + kCullOff + 16), k1 = lds_f4(pa + kCullOff + 32);
        ov = !(bx.y < patch.x || bx.x > patch.y || bx.w < patch.z || bx.z > patch.w) && !cone_misses(k0, k1, pcone);
    }
    m = __ballot_sync(0xffffffffu, ov);
    const int c = __popc(m);
    if (ov) S.idx[s][warp][__popc(m & ((1u << lane) - 1u))] = (uint8_t)lane;
    if (lane < 4) S.idx[s][warp][c + lane] = (uint8_t)kStageEntries;  // pad to a multiple of 4
    __syncwarp();
    return c;
}

// A consumer warp whose pixels are all opaque leaves the pipeline: it releases the current stage
// with arrive_drop and drops out of each later stage's "empty" barrier at the phase it would have
// released (waiting for that stage's fill first, so the phase is the right one), unless the
// producer has stopped filling.
template <class Smem>
__device__ __forceinline__ void pipe_drop_out(Smem &S, int s, unsigned phase) {
    const int lane = threadIdx.x & 31;
    for (int k = 0; k < kStages; ++k) {
        if (k > 0) {
            // Every decision here is made on lane 0's observation and broadcast: lanes that judged
            // "filled" and "producer stopped" differently would wait at different warp barriers
            // (this __syncwarp vs the epilogue's warp reductions) forever.
            bool ready = false;
            for (;;) {
                ready = __shfl_sync(0xffffffffu, (int)mbar_try_wait(&S.full[s], phase), 0) != 0;
                if (ready || __shfl_sync(0xffffffffu, *((volatile int *)&S.stop), 0)) break;
                __nanosleep(256);  // (a retired warp: do not take issue slots from the working ones)
            }
            if (!ready || __shfl_sync(0xffffffffu, S.count[s], 0) == 0) return;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_drop(&S.empty[s]);
        if (++s == kStages) {
            s = 0;
            phase ^= 1;
        }
    }
}

// ------------------------------------------------------------------------------ pair evaluation from records

// k = kHalfLog2e kappa, dd = |d_u|^2 and the scaled m of the record at shared address ra for pixel X
// (fp32 with explicit rounding: the forward and backward kernels evaluate bit-identical values).
// Also returns the record's (D4, D5, sigma, tol) and trel.
__device__ __forceinline__ void rec_k(uint32_t ra, const PixXY &X, float &k, float &dd, float (&m)[3], float4 &c1,
                                      float &trel) {
    const float4 A = lds_f4(ra), B = lds_f4(ra + 16), C = lds_f4(ra + 32), D = lds_f4(ra + 48), E = lds_f4(ra + 64);
    // (m0, m1) and (m2, the linear part of dd) as packed FMA pairs: per element the same FMA chain
    // (base + x b + y c) as scalar code, so the values do not depend on the packing
    const float2 m01 = __ffma2_rn(make_float2(B.x, B.y), X.y2,
                                  __ffma2_rn(make_float2(A.z, A.w), X.x2, make_float2(A.x, A.y)));
    const float2 m2d = __ffma2_rn(make_float2(C.z, C.w), X.y2,
                                  __ffma2_rn(make_float2(C.x, C.y), X.x2, make_float2(B.z, B.w)));
    dd = __fmaf_rn(D.z, X.yy, __fmaf_rn(D.y, X.xy, __fmaf_rn(D.x, X.xx, m2d.y)));
    m[0] = m01.x;
    m[1] = m01.y;
    m[2] = m2d.x;
    const float mm = __fmaf_rn(m[2], m[2], __fmaf_rn(m[1], m[1], __fmul_rn(m[0], m[0])));
    k = __fmul_rn(mm, rcp_approx(dd));
    c1 = make_float4(0.f, 0.f, E.x, E.y);  // (.z sigma, .w tol)
    trel = D.w;
}

// fp64 re-decision of a pair whose k lies within tol of the cutoff: kappa from the payload's W and o_u
// (the reference's cross product) for the fp64 ray.  Returns inside; kout = kHalfLog2e kappa64 (t then
// follows from it, so a record too coarse for fp32 still yields the right t); unc = even fp64 cannot
// decide (the pixel goes to the fix-up).
__device__ __forceinline__ bool recheck(const Payload &P, const double *dray, const FrameConst &fc, bool &unc,
                                        float &kout) {
    double dd, mm;
    norms64(P, dray, dd, mm);
    const double k64 = mm / dd;
    unc = fc.cutoff && fabs(k64 - fc.lam2) <= (double)P.ext.x;
    kout = (float)(kHalfLog2e * k64);
    return !fc.cutoff || k64 <= fc.lam2;
}

// ------------------------------------------------------------------------------ K5

// Forward pixel state with a running bound on |rem_fp32 - rem_fp64| (err): the alive test of
// renderer.py:113 is decided against rem64 in [rem - err, rem + err]; a pixel whose test (or a
// cutoff decision) is too close to call is stopped and redone in fp64 by k_fixup.
struct PixelState {
    float2 crg;  // (red, green): one packed FMA per update
    float cb;
    float r;     // remaining transmittance while the pixel is live, 0 once it stopped
    float rfin;  // remaining transmittance at the stop
    float err;   // bound on |r_fp32 - r_fp64|
    float efin;  // err at a threshold stop (-1: none)
    int cnt, ne, border;
};

// One front-to-back step (renderer.py:111-117) of a live pixel, followed by the alive test of the
// NEXT entry (renderer.py:113: remaining >= 1e-4), made here against the fp64 remaining known to lie
// in [r - err, r + err].  A pixel stops either surely opaque or "borderline" (test, or this entry's
// cutoff, too close to call: redone in fp64 by k_fixup; see pixel_border).  Stopped pixels carry
// r = 0, which turns every later update into a no-op without branches, and an entry with t = 0
// changes nothing, so skipping it (PBF culling, null padding entries) is exact.  trel bounds the
// relative error of t.
template <bool kUnc>
__device__ __forceinline__ void pixel_update(PixelState &ps, float trel, float t, const float4 &col, bool unc, int jne) {
    if (kUnc && unc) {  // rare: this entry's cutoff is undecidable in fp64 -> whole pixel to the fp64 fix-up
        ps.border |= ps.r > 0.0f ? 1 : 0;
        ps.rfin = ps.r > 0.0f ? ps.r : ps.rfin;
        ps.r = 0.0f;
    }
    const float w = __fmul_rn(ps.r, t);
    const float omt = __fsub_rn(1.0f, t);
    ps.crg = __ffma2_rn(make_float2(col.x, col.y), make_float2(w, w), ps.crg);
    ps.cb = __fmaf_rn(w, col.z, ps.cb);
    // |d r'| <= |d r| (1 - t) + r |d t| + rounding (none when t = 0: skipping such an entry - PBF
    // culling, a shorter list - stays an exact no-op),  |d t| <= t * trel
    ps.err = __fmaf_rn(ps.err, omt, __fmaf_rn(w, trel, w > 0.0f ? __fmul_rn(ps.r, 1.2e-7f) : 0.0f));
    ps.cnt += w > 0.0f ? 1 : 0;
    ps.r = __fmul_rn(ps.r, omt);
    const bool stop = (ps.r > 0.0f) & (__fsub_rn(ps.r, ps.err) < 1.00001e-4f);
    ps.rfin = stop ? ps.r : ps.rfin;
    ps.efin = stop ? ps.err : ps.efin;
    ps.ne = stop ? jne : ps.ne;  // alive entries: this one and every one before it (renderer.py:113)
    ps.r = stop ? 0.0f : ps.r;
}

// A pixel that stopped on the threshold is borderline when the fp64 remaining could still be >= 1e-4.
__device__ __forceinline__ bool pixel_border(const PixelState &ps) {
    return ps.border || (ps.r == 0.0f && ps.efin >= 0.0f && __fadd_rn(ps.rfin, ps.efin) >= 0.99999e-4f);
}

// The entries of one stage that this warp's culling keeps, front to back, four at a time (the list
// is padded with null entries, which are exact no-ops): the fp64 path of items without a frame.
template <class Smem>
__device__ __forceinline__ void consume_stage_generic(Smem &S, int s, int warp, int cnt, int base, const double *dray,
                                                      const FrameConst &fc, PixelState &ps, int &rechecks, int &went) {
    int k0 = 0;
    for (; k0 < cnt; k0 += 4) {
        if (k0 > 0 && !__any_sync(0xffffffffu, ps.r > 0.0f)) break;  // warp opaque
        const uint32_t q = *reinterpret_cast<const uint32_t *>(&S.idx[s][warp][k0]);
#pragma unroll 1
        for (int u = 0; u < 4; ++u) {
            const int j = (q >> (8 * u)) & 0xFF;
            const Payload &P = ring_at(S, s, j);
            PairT e;
            const bool unc = eval_t(P, dray, fc, e, rechecks);
            pixel_update<true>(ps, t_rel_bound(e.kap), e.t, P.col, unc, base + j + 1);
        }
    }
    went += k0 < cnt ? k0 : cnt;
}

// GG kept entries (stage indices jj) against the thread's pixel: the entries' t first (independent
// work), one warp vote for the rare fp64 cutoff re-decisions, then the serial pixel updates
// (without the undecidable-cutoff handling unless one occurred).  fc.thrkc is the cutoff in k units
// (+inf without the support cutoff: nothing is outside, nothing is near).
template <int GG, class Smem>
__device__ __forceinline__ void rec_group(Smem &S, int s, const int (&jj)[GG], int jbase, const PixXY &X,
                                          const double *dray, const FrameConst &fc, PixelState &ps, int &rechecks) {
    const uint32_t rb = smem_u32(&S.rec[s][0][0]);
    float t[GG], trel[GG];
    bool near[GG];
    bool any_near = false;
#pragma unroll
    for (int u = 0; u < GG; ++u) {
        float k, dd, m[3];
        float4 c1;
        rec_k(rb + (uint32_t)jj[u] * (kRecF * 4), X, k, dd, m, c1, trel[u]);
        near[u] = fabsf(__fsub_rn(k, fc.thrkc)) <= c1.w;
        any_near |= near[u];
        const float uu = __fmul_rn(c1.z, ex2_approx(-k));
        t[u] = k <= fc.thrkc ? fminf(uu, kMaxBlendTF) : 0.0f;
    }
    bool unc[GG];
#pragma unroll
    for (int u = 0; u < GG; ++u) unc[u] = false;
    bool any_unc = false;
    if (__any_sync(0xffffffffu, any_near)) {
#pragma unroll
        for (int u = 0; u < GG; ++u) {
            if (!near[u]) continue;
            float kr;
            const bool in64 = recheck(ring_at(S, s, jj[u]), dray, fc, unc[u], kr);
            const float uu = __fmul_rn(lds_f32(rb + (uint32_t)jj[u] * (kRecF * 4) + 64), ex2_approx(-kr));  // sigma
            t[u] = in64 ? fminf(uu, kMaxBlendTF) : 0.0f;
            any_unc |= unc[u];
            ++rechecks;
        }
        any_unc = __any_sync(0xffffffffu, any_unc);
    }
    if (!any_unc) {
#pragma unroll
        for (int u = 0; u < GG; ++u)
            pixel_update<false>(ps, trel[u], t[u], lds_f4(rb + (uint32_t)jj[u] * (kRecF * 4) + 80), false, jbase + jj[u]);
    } else {
#pragma unroll
        for (int u = 0; u < GG; ++u)
            pixel_update<true>(ps, trel[u], t[u], lds_f4(rb + (uint32_t)jj[u] * (kRecF * 4) + 80), unc[u], jbase + jj[u]);
    }
}

// Stage of an item with a frame: the warp's kept entries in groups of 4, then the last cnt % 4 one
// at a time (the null padding of the list is never evaluated).
template <class Smem>
__device__ __forceinline__ void consume_stage_rec(Smem &S, int s, int warp, int cnt, int base, const PixXY &X,
                                                  const double *dray, const FrameConst &fc, PixelState &ps,
                                                  int &rechecks, int &went) {
    const uint32_t ib = smem_u32(&S.idx[s][warp][0]);
    const int jbase = base + 1;
    int k0 = 0;
    for (; k0 + 4 <= cnt; k0 += 4) {
        if (k0 > 0 && !__any_sync(0xffffffffu, ps.r > 0.0f)) {  // warp opaque
            went += k0;
            return;
        }
        const uint32_t q = lds_u32(ib + k0);
        const int jj[4] = {(int)(q & 0xFF), (int)((q >> 8) & 0xFF), (int)((q >> 16) & 0xFF), (int)(q >> 24)};
        rec_group<4>(S, s, jj, jbase, X, dray, fc, ps, rechecks);
    }
#pragma unroll 1
    for (; k0 < cnt; ++k0) {
        if (k0 > 0 && !__any_sync(0xffffffffu, ps.r > 0.0f)) break;
        const int jj[1] = {(int)*(const uint8_t *)&S.idx[s][warp][k0]};
        rec_group<1>(S, s, jj, jbase, X, dray, fc, ps, rechecks);
    }
    went += k0;
}

// Per-warp culling regions and the frame of every raster work item, cached with the camera:
// wcull[(item * kConsumerWarps + warp) * 2 + {0, 1}] = patch, cone; iframe[item].  The culling
// regions are computed in fp32 from the camera-frame pixel rays and widened outward far beyond fp32
// rounding (1e-5 in mirror units, 2 % of sin^2 of the cone): a larger region only keeps more t = 0
// entries, so the culling stays exact.  The frame is fp64: dc = normalised sum of the item's world
// rays, e1 / e2 completing an orthonormal basis; rx, ry = max |x|, |y| of the item's pixel offsets
// (pixel_xy, the raster's own function), or rx = -1 when some ray is more than 60 deg from dc.
template <bool kBEAP>
__global__ void __launch_bounds__(kRasterThreads) k_warp_cull(FrameConst fc, const int4 *__restrict__ items,
                                                              const int32_t *__restrict__ n_items,
                                                              const int32_t *__restrict__ pix_list,
                                                              const double2 *__restrict__ col_sc,
                                                              const double2 *__restrict__ row_sc,
                                                              const double *__restrict__ dir64, float4 *__restrict__ wcull,
                                                              ItemFrame *__restrict__ iframe) {
    __shared__ double sred[kConsumerWarps][3];
    __shared__ float sxy[kConsumerWarps][3];
    __shared__ ItemFrame sF;
    if ((int)blockIdx.x >= n_items[0]) return;
    const int4 it = items[blockIdx.x];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool valid = tid < it.z;
    const int p = valid ? pix_list[it.y + tid] : 0;
    float c[3] = {0.f, 0.f, 1.f};  // camera-frame ray
    if (valid) {
        if (kBEAP) {  // camera.py:141-155 angles_to_dir
            const double2 cs = col_sc[p % fc.width], rs = row_sc[p / fc.width];
            const float x = (float)cs.x * (float)rs.y, y = (float)cs.y * (float)rs.x, z = (float)cs.y * (float)rs.y;
            const float inv = rsqrtf(x * x + y * y + z * z);
            c[0] = x * inv;
            c[1] = y * inv;
            c[2] = z * inv;
        } else {
            const double *d = dir64 + (int64_t)p * 3;
            for (int i = 0; i < 3; ++i)
                c[i] = (float)(fc.R[i * 3 + 0] * d[0] + fc.R[i * 3 + 1] * d[1] + fc.R[i * 3 + 2] * d[2]);
        }
    }
    // PBF patch: mirror coordinates m = tan(angle / 2) of the (x, z) and (y, z) projections
    float4 b = make_float4(-INFINITY, INFINITY, -INFINITY, INFINITY);
    if (c[2] > 1e-3f) {
        const float mx = c[0] / (sqrtf(c[0] * c[0] + c[2] * c[2]) + c[2]);
        const float my = c[1] / (sqrtf(c[1] * c[1] + c[2] * c[2]) + c[2]);
        b = make_float4(mx - 1e-5f, mx + 1e-5f, my - 1e-5f, my + 1e-5f);
    }
    if (!valid) b = make_float4(INFINITY, -INFINITY, INFINITY, -INFINITY);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        b.x = fminf(b.x, __shfl_xor_sync(0xffffffffu, b.x, o));
        b.y = fmaxf(b.y, __shfl_xor_sync(0xffffffffu, b.y, o));
        b.z = fminf(b.z, __shfl_xor_sync(0xffffffffu, b.z, o));
        b.w = fmaxf(b.w, __shfl_xor_sync(0xffffffffu, b.w, o));
    }
    const float4 patch = b;
    // ray cone: axis = normalised sum of the rays, sin^2(beta) = max |axis x ray|^2
    float sx = valid ? c[0] : 0.f, sy = valid ? c[1] : 0.f, sz = valid ? c[2] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
        sz += __shfl_xor_sync(0xffffffffu, sz, o);
    }
    const float nrm2 = sx * sx + sy * sy + sz * sz;
    float sin2 = 0.f;
    if (valid && nrm2 > 0.f) {
        const float inv = rsqrtf(nrm2);
        const float ax = sx * inv, ay = sy * inv, az = sz * inv;
        const float x0 = ay * c[2] - az * c[1], x1 = az * c[0] - ax * c[2], x2 = ax * c[1] - ay * c[0];
        sin2 = (x0 * x0 + x1 * x1 + x2 * x2) / (c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sin2 = fmaxf(sin2, __shfl_xor_sync(0xffffffffu, sin2, o));
    sin2 = fmaf(sin2, 1.02f, 1e-7f);
    float4 cone = make_float4(0.f, 0.f, 1.f, 0.f);  // cos^2 = 0 disables the test (beta > 45 deg)
    if (nrm2 > 0.f && sin2 < 0.5f) {
        const float inv = rsqrtf(nrm2);
        cone = make_float4(sx * inv, sy * inv, sz * inv, 1.0f - sin2);
    }
    if (lane == 0) {
        wcull[((int64_t)it.w * kConsumerWarps + warp) * 2 + 0] = patch;
        wcull[((int64_t)it.w * kConsumerWarps + warp) * 2 + 1] = cone;
    }
    // ---- the item frame (fp64 world rays, as the raster computes them)
    double d[3] = {0.0, 0.0, 0.0};
    if (valid) pixel_ray<kBEAP>(fc, p, col_sc, row_sc, dir64, d);
    double ws[3] = {d[0], d[1], d[2]};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        for (int i = 0; i < 3; ++i) ws[i] += __shfl_xor_sync(0xffffffffu, ws[i], o);
    if (lane == 0)
        for (int i = 0; i < 3; ++i) sred[warp][i] = ws[i];
    __syncthreads();
    if (tid == 0) {
        double sum[3] = {0.0, 0.0, 0.0};
        for (int w = 0; w < kConsumerWarps; ++w)
            for (int i = 0; i < 3; ++i) sum[i] += sred[w][i];
        const double nn = sqrt(sum[0] * sum[0] + sum[1] * sum[1] + sum[2] * sum[2]);
        ItemFrame F{};
        if (nn > 0.0) {
            for (int i = 0; i < 3; ++i) F.dc[i] = sum[i] / nn;
            int k = 0;  // the axis least aligned with dc
            for (int i = 1; i < 3; ++i)
                if (fabs(F.dc[i]) < fabs(F.dc[k])) k = i;
            double e[3] = {-F.dc[k] * F.dc[0], -F.dc[k] * F.dc[1], -F.dc[k] * F.dc[2]};
            e[k] += 1.0;
            const double en = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
            for (int i = 0; i < 3; ++i) F.e1[i] = e[i] / en;
            F.e2[0] = F.dc[1] * F.e1[2] - F.dc[2] * F.e1[1];
            F.e2[1] = F.dc[2] * F.e1[0] - F.dc[0] * F.e1[2];
            F.e2[2] = F.dc[0] * F.e1[1] - F.dc[1] * F.e1[0];
            const double e2n = sqrt(F.e2[0] * F.e2[0] + F.e2[1] * F.e2[1] + F.e2[2] * F.e2[2]);
            for (int i = 0; i < 3; ++i) F.e2[i] /= e2n;
            F.rx = 0.f;
        } else {
            F.rx = -1.f;
        }
        sF = F;
    }
    __syncthreads();
    float ax = 0.f, ay = 0.f, bad = sF.rx < 0.f ? 1.f : 0.f;
    if (valid && sF.rx >= 0.f) {
        const double den = d[0] * sF.dc[0] + d[1] * sF.dc[1] + d[2] * sF.dc[2];
        if (!(den > 0.5 * sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]))) {
            bad = 1.f;
        } else {
            const float2 xy = pixel_xy(sF, d);
            ax = fabsf(xy.x);
            ay = fabsf(xy.y);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ax = fmaxf(ax, __shfl_xor_sync(0xffffffffu, ax, o));
        ay = fmaxf(ay, __shfl_xor_sync(0xffffffffu, ay, o));
        bad = fmaxf(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    }
    if (lane == 0) {
        sxy[warp][0] = ax;
        sxy[warp][1] = ay;
        sxy[warp][2] = bad;
    }
    __syncthreads();
    if (tid == 0) {
        ItemFrame F = sF;
        float mx = 0.f, my = 0.f, mb = 0.f;
        for (int w = 0; w < kConsumerWarps; ++w) {
            mx = fmaxf(mx, sxy[w][0]);
            my = fmaxf(my, sxy[w][1]);
            mb = fmaxf(mb, sxy[w][2]);
        }
        F.rx = mb > 0.f ? -1.f : mx;
        F.ry = my;
        iframe[it.w] = F;
    }
}

#ifdef GEER_CTA_TIMING
// Tuning instrumentation (build with -DGEER_CTA_TIMING): per raster CTA start / end %globaltimer
// (ns), SM id and warp-entries, read back by geer_debug_cta_times (scripts/cta_timing.py).
__device__ unsigned long long g_cta_t0[1 << 16], g_cta_t1[1 << 16];
__device__ int g_cta_sm[1 << 16], g_cta_went[1 << 16];
__device__ unsigned long long g_cta_ts[1 << 16], g_cta_tf[1 << 16];  // setup done, first stage ready
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

constexpr int kFwdThreads = kPipeThreads;  // 8 consumer warps + the producer warp
#ifndef FWD_MIN_BLOCKS2
#define FWD_MIN_BLOCKS2 3
#endif
using FwdSmem = PipeSmem<false>;

// Copy an item frame into shared memory (the producer warp; 24 words).
__device__ __forceinline__ void load_frame(ItemFrame &dst, const ItemFrame *src, int lane) {
    const uint32_t *s = reinterpret_cast<const uint32_t *>(src);
    uint32_t *d = reinterpret_cast<uint32_t *>(&dst);
    if (lane < (int)(sizeof(ItemFrame) / 4)) d[lane] = __ldg(s + lane);
    __syncwarp();
}

// K5.  One pixel per consumer thread.
template <bool kBEAP>
__global__ void __launch_bounds__(kFwdThreads, FWD_MIN_BLOCKS2)
    k_forward(FrameConst fc, geer_scene sc, const int4 *__restrict__ items, const int32_t *__restrict__ n_items,
              const int32_t *__restrict__ pix_list, const double2 *__restrict__ col_sc,
              const double2 *__restrict__ row_sc, const double *__restrict__ dir64, const int32_t *__restrict__ ranges,
              const uint32_t *__restrict__ order, const __grid_constant__ CUtensorMap pay_map,
              const float4 *__restrict__ wcull, const ItemFrame *__restrict__ iframe, float *__restrict__ color,
              float *__restrict__ remaining, int32_t *__restrict__ count, int32_t *__restrict__ n_eval,
              unsigned long long *__restrict__ counters, int32_t *__restrict__ fixup_list) {
    constexpr int NW = kConsumerWarps;
    extern __shared__ __align__(128) unsigned char dsmem[];  // PipeSmem (dynamic: deep rings exceed 48 KB)
    FwdSmem &S = *reinterpret_cast<FwdSmem *>(dsmem);  // 128-B aligned base: TMA destinations, fixed offsets
    __shared__ double sray[kRasterThreads][3];  // fp64 pixel rays (re-checks, fp64 path)
    // n_items: [0] items with entries (work[0, n0)), [1] empty items (the tail of [0, n0 + n1))
    const int n_full = n_items[0];
    if ((int)blockIdx.x >= n_full + n_items[1]) return;
    const int4 it = items[(int)blockIdx.x < n_full ? (int)blockIdx.x : n_full + n_items[1] - 1 - ((int)blockIdx.x - n_full)];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if ((int)blockIdx.x >= n_full) {  // tile without entries: background only (renderer.py:118)
        for (int q = tid; q < it.z; q += blockDim.x) {
            const int p = pix_list[it.y + q];
            color[(int64_t)p * 3 + 0] = fc.bg[0];
            color[(int64_t)p * 3 + 1] = fc.bg[1];
            color[(int64_t)p * 3 + 2] = fc.bg[2];
            remaining[p] = 1.0f;
            count[p] = 0;
            n_eval[p] = 0;
        }
        return;
    }
    const int tr = fc.exhaustive ? 0 : it.x;  // exhaustive mode: one shared list [0, n_kept)
    const int e0 = ranges[tr], e1 = ranges[tr + 1];
#ifdef GEER_CTA_TIMING
    if (tid == 0 && blockIdx.x < (1u << 16)) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        g_cta_t0[blockIdx.x] = gtimer();
        g_cta_sm[blockIdx.x] = (int)smid;
        g_cta_t1[blockIdx.x] = 0;
        g_cta_went[blockIdx.x] = 0;
    }
#endif
    const ItemFrame *F = iframe + it.w;
    const bool framed = F->rx >= 0.f;  // uniform over the CTA
    // the producer starts streaming right away; the consumers set up their pixels meanwhile
    pipe_init(S);
    if (warp == NW) {
        load_frame(S.frame, F, lane);
        pipe_produce<false>(S, order, &pay_map, fc.thrk, framed, e0, e1 - e0, true, &counters[4]);
        return;
    }
    const int q = tid;
    const bool valid = q < it.z;
    const int p = valid ? pix_list[it.y + q] : 0;
    double d64[3] = {0.0, 0.0, 1.0};
    PixXY X = make_pxy(make_float2(0.f, 0.f));
    if (valid) {
        pixel_ray<kBEAP>(fc, p, col_sc, row_sc, dir64, d64);
        if (framed) X = make_pxy(pixel_xy(*F, d64));
    }
    if (lane < 2) S.wc[warp][lane] = wcull[((int64_t)it.w * kConsumerWarps + warp) * 2 + lane];  // (k_warp_cull)
    __syncwarp();
#ifdef GEER_CTA_TIMING
    if (tid == 0 && blockIdx.x < (1u << 16)) g_cta_ts[blockIdx.x] = gtimer();
#endif
    sray[q][0] = d64[0];
    sray[q][1] = d64[1];
    sray[q][2] = d64[2];
    const double *dray = sray[q];
    PixelState ps{make_float2(0.f, 0.f), 0.f, valid ? 1.0f : 0.0f, 1.0f, 0.f, -1.0f, 0, 0, 0};
    int rechecks = 0, went = 0;
    bool warp_live = __any_sync(0xffffffffu, valid);
    if (!warp_live && lane == 0) atomicAdd(&S.done_warps, 1);
    unsigned phase = 0;
    int s = 0, base = 0;
    for (;;) {
        mbar_wait(&S.full[s], phase);
#ifdef GEER_CTA_TIMING
        if (tid == 0 && base == 0 && blockIdx.x < (1u << 16)) g_cta_tf[blockIdx.x] = gtimer();
#endif
        const int n = S.count[s];
        if (n == 0) break;
        if (warp_live) {
            uint32_t m;
            const int cnt = stage_keep(S, s, warp, lane, n, fc.cull != 0, m);
            if (!framed)
                consume_stage_generic(S, s, warp, cnt, base, dray, fc, ps, rechecks, went);
            else
                consume_stage_rec(S, s, warp, cnt, base, X, dray, fc, ps, rechecks, went);
            warp_live = __any_sync(0xffffffffu, ps.r > 0.0f);
            if (!warp_live && lane == 0) atomicAdd(&S.done_warps, 1);
        }
        if (!warp_live) {  // every pixel of the warp opaque: leave the pipeline, stop issuing
            pipe_drop_out(S, s, phase);
            break;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);
        base += n;
        if (++s == kStages) {
            s = 0;
            phase ^= 1;
        }
    }
    if (ps.r > 0.0f) ps.ne = e1 - e0;  // alive through the whole list
    if (valid) {
        const float rem = ps.r > 0.0f ? ps.r : ps.rfin;  // live to the end of the list, or stopped
        // renderer.py:118 background with the final remaining transmittance
        color[(int64_t)p * 3 + 0] = __fmaf_rn(rem, fc.bg[0], ps.crg.x);
        color[(int64_t)p * 3 + 1] = __fmaf_rn(rem, fc.bg[1], ps.crg.y);
        color[(int64_t)p * 3 + 2] = __fmaf_rn(rem, fc.bg[2], ps.cb);
        remaining[p] = rem;
        count[p] = ps.cnt;
        n_eval[p] = ps.ne;
        if (pixel_border(ps)) {
            unsigned long long slot = atomicAdd(&counters[2], 1ull);
            fixup_list[slot] = (int32_t)(((int64_t)blockIdx.x << 8) | q);  // work item, pixel of the item
        }
    }
    rechecks = __reduce_add_sync(0xffffffffu, rechecks);
    if (lane == 0 && rechecks) atomicAdd(&counters[0], (unsigned long long)rechecks);
    if (lane == 0 && went) atomicAdd(&counters[3], (unsigned long long)went);
#ifdef GEER_CTA_TIMING
    if (lane == 0 && blockIdx.x < (1u << 16)) {
        atomicMax(&g_cta_t1[blockIdx.x], gtimer());
        atomicAdd(&g_cta_went[blockIdx.x], went);
    }
#endif
}

// ------------------------------------------------------------------------------ fp64 fix-up of borderline pixels

// One warp per borderline pixel: the pixel is recomposited in fp64 exactly as
// renderer.py:96-118 (kappa, u, t, remaining in fp64; the 1e-4 early-stop test
// on the fp64 remaining), so its early-stop decision is the reference's.  The tile's list is walked
// in batches of 128 entries: each entry's culling record is tested against the pixel's own ray
// first (the raster's exact PBF-hull and visual-cone tests, for a cone of one ray), and only the
// survivors - in list order, compacted into shared memory - get the fp64 evaluation.  A culled entry
// has t = 0: it changes neither remaining nor the count, and it is alive exactly when the survivors
// before it leave remaining >= 1e-4, so n_eval = position of the stopping survivor + 1.
template <bool kBEAP>
__device__ void fixup_pixel(FrameConst fc, const geer_scene &sc, const int4 *__restrict__ items,
                            const int32_t *__restrict__ pix_list, const double2 *__restrict__ col_sc,
                            const double2 *__restrict__ row_sc, const double *__restrict__ dir64,
                            const int32_t *__restrict__ ranges, const uint32_t *__restrict__ order,
                            const Payload *__restrict__ payload, int code, int lane, int32_t *surv,
                            float *__restrict__ color, float *__restrict__ remaining, int32_t *__restrict__ count,
                            int32_t *__restrict__ n_eval) {
    const int4 it = items[code >> 8];
    const int p = pix_list[it.y + (code & 255)];
    double d[3];
    pixel_ray<kBEAP>(fc, p, col_sc, row_sc, dir64, d);
    const int tr = fc.exhaustive ? 0 : it.x;  // exhaustive mode: one shared list [0, n_kept)
    const int e0 = ranges[tr], e1 = ranges[tr + 1];
    // the pixel's culling region: its mirror coordinates (+-1e-5) and a cone of one ray (k_warp_cull)
    float4 box = make_float4(-INFINITY, INFINITY, -INFINITY, INFINITY), cone = make_float4(0.f, 0.f, 1.f, 0.f);
    {
        float c[3];
        for (int i = 0; i < 3; ++i) c[i] = (float)(fc.R[i * 3 + 0] * d[0] + fc.R[i * 3 + 1] * d[1] + fc.R[i * 3 + 2] * d[2]);
        if (c[2] > 1e-3f) {
            const float mx = c[0] / (sqrtf(c[0] * c[0] + c[2] * c[2]) + c[2]);
            const float my = c[1] / (sqrtf(c[1] * c[1] + c[2] * c[2]) + c[2]);
            box = make_float4(mx - 1e-5f, mx + 1e-5f, my - 1e-5f, my + 1e-5f);
        }
        const float inv = rsqrtf(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
        cone = make_float4(c[0] * inv, c[1] * inv, c[2] * inv, 1.0f - 1e-7f);
    }
    double cr = 0, cg = 0, cb = 0, rem = 1.0;
    int cnt = 0, last = e0 - 1;  // last: the last alive survivor
    bool alive = true;
    // fp64 t of entry e (renderer.py:96-105 in fp64: the payload's cross product, the reference
    // formulation near the cutoff, K1's fp64 sigmoid from the payload, fp64 exp)
    auto eval64 = [&](int e, double &t, float4 &cl) {
        const uint32_t g = order[e];
        const Payload &P = payload[g];
        cl = P.col;
        double dd, mm;
        norms64(P, d, dd, mm);
        double kap = mm / dd;
        if (fc.cutoff && fabs(kap - fc.lam2) <= (double)P.ext.x)
            kap = kappa_fp64(sc.means, sc.log_scales, sc.quats, fc.origin[0], fc.origin[1], fc.origin[2], g, d[0], d[1],
                             d[2]);
        const double sig = __hiloint2double(__float_as_int(P.ext.z), __float_as_int(P.ext.y));  // K1's fp64 sigmoid
        double u = sig * exp(-0.5 * kap);
        if (fc.cutoff && !(kap <= fc.lam2)) u = 0.0;
        t = u < kMaxBlendT ? u : kMaxBlendT;
    };
    for (int sbase = e0; sbase < e1 && alive; sbase += 128) {
        // survivors of the batch, in list order
        int ns = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int e = sbase + 32 * k + lane;
            bool keep = e < e1;
            if (keep && fc.cull) {
                const Cull cl = payload[order[e]].cull;
                keep = !(cl.box.y < box.x || cl.box.x > box.y || cl.box.w < box.z || cl.box.z > box.w) &&
                       !cone_misses(cl.k0, cl.k1, cone);
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) surv[ns + __popc(m & ((1u << lane) - 1u))] = e;
            ns += __popc(m);
        }
        __syncwarp();
        for (int i0 = 0; i0 < ns && alive; i0 += 32) {
            const int n = min(32, ns - i0);
            double t = 0.0;
            float4 cl = make_float4(0.f, 0.f, 0.f, 0.f);
            const int e = lane < n ? surv[i0 + lane] : e1;
            if (lane < n) eval64(e, t, cl);
            // composite the survivors with a warp scan: rem before survivor j = rem * prod_{i<j} (1 - t_i);
            // the alive test (rem >= 1e-4, renderer.py:113) holds on a prefix since rem only decreases
            double P = lane < n ? 1.0 - t : 1.0;  // inclusive prefix product
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, P, o);
                if (lane >= o) P *= y;
            }
            const double up1 = __shfl_up_sync(0xffffffffu, P, 1);  // (every lane takes part in the shuffle)
            const double pex = lane == 0 ? 1.0 : up1;
            const double rb = rem * pex;
            const bool live = lane < n && rb >= kMinRemaining;
            const int na = __popc(__ballot_sync(0xffffffffu, live));
            double w = live ? rb * t : 0.0;
            double wr = w * cl.x, wg = w * cl.y, wb = w * cl.z;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                wr += __shfl_xor_sync(0xffffffffu, wr, o);
                wg += __shfl_xor_sync(0xffffffffu, wg, o);
                wb += __shfl_xor_sync(0xffffffffu, wb, o);
            }
            cr += wr;
            cg += wg;
            cb += wb;
            cnt += __popc(__ballot_sync(0xffffffffu, live && t > 0.0));
            const double pl = __shfl_sync(0xffffffffu, P, na > 0 ? na - 1 : 0);
            const int el = __shfl_sync(0xffffffffu, e, na > 0 ? na - 1 : 0);
            if (na > 0) {
                rem = rem * pl;
                last = el;
            }
            if (!(rem >= kMinRemaining)) alive = false;  // the entries after survivor `last` are not alive
        }
        __syncwarp();
    }
    const int ne = alive ? e1 - e0 : last - e0 + 1;
    if (lane == 0) {
        color[(int64_t)p * 3 + 0] = (float)(cr + rem * fc.bg[0]);
        color[(int64_t)p * 3 + 1] = (float)(cg + rem * fc.bg[1]);
        color[(int64_t)p * 3 + 2] = (float)(cb + rem * fc.bg[2]);
        remaining[p] = (float)rem;
        count[p] = cnt;
        n_eval[p] = ne;
    }
}

template <bool kBEAP>
__global__ void __launch_bounds__(128) k_fixup(FrameConst fc, geer_scene sc, const int4 *__restrict__ items,
                                               const int32_t *__restrict__ pix_list,
                                               const double2 *__restrict__ col_sc, const double2 *__restrict__ row_sc,
                                               const double *__restrict__ dir64, const int32_t *__restrict__ ranges,
                                               const uint32_t *__restrict__ order, const Payload *__restrict__ payload,
                                               const unsigned long long *__restrict__ counters,
                                               const int32_t *__restrict__ fixup_list, float *__restrict__ color,
                                               float *__restrict__ remaining, int32_t *__restrict__ count,
                                               int32_t *__restrict__ n_eval) {
    __shared__ int32_t surv[4][128];  // per warp: the batch's surviving entries
    const int lane = threadIdx.x & 31;
    const int n_fix = (int)counters[2];
    const int n_warps = (int)((gridDim.x * (int64_t)blockDim.x) >> 5);
    for (int wg = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); wg < n_fix; wg += n_warps)
        fixup_pixel<kBEAP>(fc, sc, items, pix_list, col_sc, row_sc, dir64, ranges, order, payload, fixup_list[wg], lane,
                           surv[threadIdx.x >> 5], color, remaining, count, n_eval);
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

// The same reduction through shared memory (red: this warp's 16 x 36 scratch): lane l stores its 16
// values as column l (conflict-free), then lane l sums half a row (partial l >> 1, lanes 16 (l & 1) ..
// + 15) with four 16-B loads (rows padded to 36 words: conflict-free) and one shuffle.  ~40 instead
// of ~62 instructions.
__device__ __forceinline__ float smem_transpose_reduce16(float (*red)[36], const float v[16], int lane) {
#pragma unroll
    for (int k = 0; k < 16; ++k) red[k][lane] = v[k];
    __syncwarp();
    const float4 *row = reinterpret_cast<const float4 *>(&red[lane >> 1][16 * (lane & 1)]);
    const float4 a = row[0], b = row[1], c = row[2], d = row[3];
    float sum = ((a.x + a.y) + (a.z + a.w)) + ((b.x + b.y) + (b.z + b.w)) + (((c.x + c.y) + (c.z + c.w)) + ((d.x + d.y) + (d.z + d.w)));
    __syncwarp();  // (the next entry overwrites the scratch)
    return sum + __shfl_xor_sync(0xffffffffu, sum, 1);
}

// The second half of smem_transpose_reduce16, for partials already stored as column `lane`.
__device__ __forceinline__ float smem_column_reduce16(float (*red)[36], int lane) {
    __syncwarp();
    const float4 *row = reinterpret_cast<const float4 *>(&red[lane >> 1][16 * (lane & 1)]);
    const float4 a = row[0], b = row[1], c = row[2], d = row[3];
    float sum = ((a.x + a.y) + (a.z + a.w)) + ((b.x + b.y) + (b.z + b.w)) + (((c.x + c.y) + (c.z + c.w)) + ((d.x + d.y) + (d.z + d.w)));
    __syncwarp();  // (the next entry overwrites the scratch)
    return sum + __shfl_xor_sync(0xffffffffu, sum, 1);
}

// Reverse-order backward (renderer.py:259-310).  The producer streams the
// tile's first max_n entries back to front; each lane walks its pixel's alive
// entries (index < n_eval) from the last to the first, recovering
// T_i = T_{i+1} / (1 - t_i) from the forward's final remaining, and the warp
// adds its 16 per-entry partials to the Gaussian's accumulators.
#ifndef BWD_MIN_BLOCKS
#define BWD_MIN_BLOCKS 3
#endif
using BwdSmem = PipeSmem<true>;
template <bool kBEAP>
__global__ void __launch_bounds__(kPipeThreads, BWD_MIN_BLOCKS)
    k_backward(FrameConst fc, geer_scene sc, const int4 *__restrict__ items, const int32_t *__restrict__ n_items,
               const int32_t *__restrict__ pix_list, const double2 *__restrict__ col_sc,
               const double2 *__restrict__ row_sc, const double *__restrict__ dir64,
               const int32_t *__restrict__ ranges, const uint32_t *__restrict__ order,
               const __grid_constant__ CUtensorMap pay_map, const float4 *__restrict__ wcull,
               const ItemFrame *__restrict__ iframe, const float *__restrict__ remaining,
               const int32_t *__restrict__ n_eval,
               const float *__restrict__ dl_dimage, float *__restrict__ accum) {
    extern __shared__ __align__(128) unsigned char dsmem[];
    BwdSmem &S = *reinterpret_cast<BwdSmem *>(dsmem);
    __shared__ double sray[kRasterThreads][3];
    __shared__ int smax;
    if ((int)blockIdx.x >= n_items[0]) return;  // tiles without entries have no gradient
    const int4 it = items[blockIdx.x];
    const int e0 = ranges[it.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool valid = warp < kConsumerWarps && tid < it.z;
    const int p = valid ? pix_list[it.y + tid] : 0;
    const int ne = valid ? n_eval[p] : 0;
    if (tid == 0) smax = 0;
    __syncthreads();
    const int wmax = __reduce_max_sync(0xffffffffu, ne);
    if (lane == 0 && wmax > 0) atomicMax(&smax, wmax);
    pipe_init(S);  // (its __syncthreads also publishes smax)
    const int max_n = smax;
    if (max_n == 0) return;
    const ItemFrame *F = iframe + it.w;
    const bool framed = F->rx >= 0.f;
    if (warp == kConsumerWarps) {
        load_frame(S.frame, F, lane);
        pipe_produce<true>(S, order, &pay_map, fc.thrk, framed, e0, max_n, false);
        return;
    }
    // the producer streams while the consumers set up their pixels
    double d64[3] = {0.0, 0.0, 1.0};
    PixXY X = make_pxy(make_float2(0.f, 0.f));
    float dx, dy, dz;  // the ray the gradient is formed with: d' = dc + x e1 + y e2 (framed) or d
    if (valid) pixel_ray<kBEAP>(fc, p, col_sc, row_sc, dir64, d64);
    if (framed) {
        const float2 xy = valid ? pixel_xy(*F, d64) : make_float2(0.f, 0.f);
        X = make_pxy(xy);
        dx = (float)(F->dc[0] + (double)xy.x * F->e1[0] + (double)xy.y * F->e2[0]);
        dy = (float)(F->dc[1] + (double)xy.x * F->e1[1] + (double)xy.y * F->e2[1]);
        dz = (float)(F->dc[2] + (double)xy.x * F->e1[2] + (double)xy.y * F->e2[2]);
    } else {
        dx = (float)d64[0];
        dy = (float)d64[1];
        dz = (float)d64[2];
    }
    if (lane < 2) S.wc[warp][lane] = wcull[((int64_t)it.w * kConsumerWarps + warp) * 2 + lane];  // (k_warp_cull)
    __syncwarp();
    sray[tid][0] = d64[0];
    sray[tid][1] = d64[1];
    sray[tid][2] = d64[2];
    const float t_fin = valid ? remaining[p] : 0.f;
    float gl0 = 0.f, gl1 = 0.f, gl2 = 0.f;
    if (valid) {
        gl0 = dl_dimage[(int64_t)p * 3 + 0];
        gl1 = dl_dimage[(int64_t)p * 3 + 1];
        gl2 = dl_dimage[(int64_t)p * 3 + 2];
    }
    // (x, y) components kept as pairs for the packed fp32 instructions
    const float2 gl01 = make_float2(gl0, gl1), dxy = make_float2(dx, dy);
    const float2 bgt01 = make_float2(t_fin * fc.bg[0], t_fin * fc.bg[1]);
    const float bgt2 = t_fin * fc.bg[2];
    float T = t_fin, s2 = 0.f;
    float2 s01 = make_float2(0.f, 0.f);
    int dummy = 0;
    unsigned phase = 0;
    int s = 0;
    int hi = max_n;  // local index one past the current stage
    for (;;) {
        mbar_wait(&S.full[s], phase);
        const int n = S.count[s];
        if (n == 0) break;
        const int lo = hi - n;
        if (lo < wmax) {  // some lane of this warp has alive entries in the stage
            // entries the culling keeps (culled ones have t = 0: no gradient, T unchanged), below wmax
            uint32_t msk;
            stage_keep(S, s, warp, lane, n, fc.cull != 0, msk);
            if (wmax - lo < 32) msk &= (1u << (wmax - lo)) - 1u;
            const uint32_t rb = smem_u32(&S.rec[s][0][0]);
            // one entry's gradient: T and suffix update, 16 partials, warp reduction, accumulators.
            // du, m, o: d_u = W d, m = o_u x d_u (m unscaled here) for the gradient ray (dx, dy, dz).
            auto entry = [&](const int jj, const PairT &e, const float *du, const float *mv, const float *o,
                             const float4 &col) {
                const int i = lo + jj;
                // t = 0 (or not alive) on every lane: T, the suffix and all 16 partials are unchanged
                if (!__any_sync(0xffffffffu, i < ne && e.t > 0.0f)) return;
#ifndef GEER_BWD_SHFL_REDUCE
                // the 16 partials go straight into this lane's column of the warp's transpose scratch
                // (each value's register dies at its store)
                float *colp = &S.red[warp][0][lane];
                auto put = [&](int k, float val) { colp[k * 36] = val; };
#else
                float v[16];
                auto put = [&](int k, float val) { v[k] = val; };
#endif
                const bool alive = i < ne;
                const float omt = __fsub_rn(1.0f, e.t);
                const float inv = rcp_approx(omt);  // 1 - t >= 0.001: ~1 ulp
                if (alive) T = T * inv;             // T_i = T_{i+1} / (1 - t_i)
                const float w = alive ? T * e.t : 0.0f;
                {
                    const float2 c01 = make_float2(col.x, col.y);
                    const float c2 = col.z;
                    // renderer.py:284-287
                    const float2 dcdt01 = __ffma2_rn(c01, make_float2(T, T),
                                                     __fmul2_rn(__fadd2_rn(s01, bgt01), make_float2(-inv, -inv)));
                    const float dcdt2 = T * c2 - (s2 + bgt2) * inv;
                    const float dl_dt = dcdt01.x * gl0 + dcdt01.y * gl1 + dcdt2 * gl2;
                    s01 = __ffma2_rn(c01, make_float2(w, w), s01);
                    s2 += w * c2;
                    const float2 dc01 = __fmul2_rn(gl01, make_float2(w, w));  // renderer.py:309 dcol
                    put(13, dc01.x);
                    put(14, dc01.y);
                    put(15, w * gl2);
                    // renderer.py:289-290 gate
                    const bool gate = alive && e.t > 0.0f && e.u < kMaxBlendTF;
                    put(12, gate ? dl_dt * e.alpha : 0.0f);
                    const float dk = -0.5f * dl_dt * e.u;
                    const float coef = gate ? 2.0f * dk * rcp_approx(e.dd) : 0.0f;  // dl_dm = coef * m
                    const float2 lm01 = __fmul2_rn(make_float2(mv[0], mv[1]), make_float2(coef, coef));
                    const float lm0 = lm01.x, lm1 = lm01.y, lm2 = coef * mv[2];
                    put(9, du[1] * lm2 - du[2] * lm1);  // dl_do = d_u x dl_dm
                    put(10, du[2] * lm0 - du[0] * lm2);
                    put(11, du[0] * lm1 - du[1] * lm0);
                    const float sc_ = e.kap * coef;  // dl_dd = -(2 kappa dk / dd) d_u + dl_dm x o_u
                    const float dd0 = -sc_ * du[0] + (lm1 * o[2] - lm2 * o[1]);
                    const float dd1 = -sc_ * du[1] + (lm2 * o[0] - lm0 * o[2]);
                    const float dd2 = -sc_ * du[2] + (lm0 * o[1] - lm1 * o[0]);
                    // renderer.py:304 dW_rc
                    const float2 w0 = __fmul2_rn(dxy, make_float2(dd0, dd0)), w1 = __fmul2_rn(dxy, make_float2(dd1, dd1)),
                                 w2 = __fmul2_rn(dxy, make_float2(dd2, dd2));
                    put(0, w0.x); put(1, w0.y); put(2, dd0 * dz);
                    put(3, w1.x); put(4, w1.y); put(5, dd1 * dz);
                    put(6, w2.x); put(7, w2.y); put(8, dd2 * dz);
                }
#ifdef GEER_BWD_SHFL_REDUCE
                const float tot = warp_transpose_reduce16(v, lane);
#else
                const float tot = smem_column_reduce16(S.red[warp], lane);
#endif
                // lane 2k adds partial k (predicated fire-and-forget reduction, no branch)
                float *dst = accum + (int64_t)S.gid[s][jj] * 16 + (lane >> 1);
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "setp.ne.u32 p, %2, 0;\n\t"
                    "@p red.global.add.f32 [%0], %1;\n\t}" ::"l"(dst),
                    "f"(tot), "r"((int)((lane & 1) == 0 && tot != 0.0f))
                    : "memory");
            };
            if (!framed) {  // fp64 path: t from the payload's fp64 cross product, gradient vectors in fp32
                while (msk) {
                    const int jj = 31 - __clz(msk);
                    msk &= ~(1u << jj);
                    const Payload &P = ring_at(S, s, jj);
                    PairT e;
                    eval_t(P, sray[tid], fc, e, dummy);
                    float du[3], mv[3], o[3];
                    for (int r = 0; r < 3; ++r) {
                        du[r] = (float)P.q[r * 3 + 0] * dx + (float)P.q[r * 3 + 1] * dy + (float)P.q[r * 3 + 2] * dz;
                        o[r] = (float)P.q[9 + r];
                    }
                    mv[0] = o[1] * du[2] - o[2] * du[1];
                    mv[1] = o[2] * du[0] - o[0] * du[2];
                    mv[2] = o[0] * du[1] - o[1] * du[0];
                    entry(jj, e, du, mv, o, P.col);
                }
            } else {
                while (msk) {
                    const int jj = 31 - __clz(msk);
                    msk &= ~(1u << jj);
                    // t exactly as the forward's rec_group computes it
                    const uint32_t ra = rb + (uint32_t)jj * (kRecB * 4);
                    float k, dd, trel, ms[3];
                    float4 c1;
                    rec_k(ra, X, k, dd, ms, c1, trel);
                    bool inside = k <= fc.thrkc;
                    if (fabsf(__fsub_rn(k, fc.thrkc)) <= c1.w) {  // (exactly the forward's re-check)
                        bool unc;
                        inside = recheck(ring_at(S, s, jj), sray[tid], fc, unc, k);
                    }
                    PairT e;
                    e.alpha = ex2_approx(-k);
                    e.u = inside ? __fmul_rn(c1.z, e.alpha) : 0.0f;
                    e.t = inside ? fminf(e.u, kMaxBlendTF) : 0.0f;
                    e.kap = k * (float)(1.0 / kHalfLog2e);
                    // gradient vectors for d' (kappa is scale-invariant in the ray: dW = dl/dd_u (x) d')
                    const float4 g0 = lds_f4(ra + 96), g1 = lds_f4(ra + 112), g2 = lds_f4(ra + 128);
                    const float2 du01 = __ffma2_rn(make_float2(g1.x, g1.y), X.y2,
                                                   __ffma2_rn(make_float2(g0.z, g0.w), X.x2, make_float2(g0.x, g0.y)));
                    const float du[3] = {du01.x, du01.y, __fmaf_rn(g2.x, X.y2.x, __fmaf_rn(g1.w, X.x2.x, g1.z))};
                    const float o[3] = {g2.y, g2.z, g2.w};
                    float mv[3];
                    if (c1.w < INFINITY) {  // the record's m and dd (entry-uniform branch)
                        constexpr float kInvS = (float)(1.0 / kSqrtHalfLog2e);
                        mv[0] = ms[0] * kInvS;
                        mv[1] = ms[1] * kInvS;
                        mv[2] = ms[2] * kInvS;
                        e.dd = dd;
                    } else {  // a record without fp32 vectors (fp64 re-check path): from d_u and o_u
                        mv[0] = o[1] * du[2] - o[2] * du[1];
                        mv[1] = o[2] * du[0] - o[0] * du[2];
                        mv[2] = o[0] * du[1] - o[1] * du[0];
                        e.dd = du[0] * du[0] + du[1] * du[1] + du[2] * du[2];
                    }
                    entry(jj, e, du, mv, o, lds_f4(ra + 80));
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[s]);
        hi = lo;
        if (++s == kStages) {
            s = 0;
            phase ^= 1;
        }
    }
}


// Exhaustive mode: ranges2 = {0, number of kept Gaussians} (they lead the depth order).
__global__ void k_exhaustive_ranges(const uint8_t *__restrict__ flags, int64_t n, int32_t *__restrict__ ranges2) {
    int c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += flags[i] & 1;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&ranges2[1], c);
}
void launch_exhaustive_ranges(const uint8_t *flags, int64_t n, int32_t *ranges2, cudaStream_t st) {
    cudaMemsetAsync(ranges2, 0, 2 * sizeof(int32_t), st);
    if (n > 0) k_exhaustive_ranges<<<(int)lmin((n + 255) / 256, 148 * 8), 256, 0, st>>>(flags, n, ranges2);
}

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

// Dynamic shared memory above 48 KB needs an explicit opt-in per kernel (done once).
static void raster_smem_optin() {
    static bool done = false;
    if (done) return;
    done = true;
    cudaFuncSetAttribute(k_forward<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FwdSmem) + 128);
    cudaFuncSetAttribute(k_forward<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FwdSmem) + 128);
    cudaFuncSetAttribute(k_backward<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BwdSmem) + 128);
    cudaFuncSetAttribute(k_backward<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BwdSmem) + 128);
}

void launch_forward(const FrameConst &fc, const geer_scene &sc, int max_items, const int4 *items,
                    const int32_t *n_items, const int32_t *pix_list, const double2 *col_sc, const double2 *row_sc,
                    const double *dir64, const int32_t *ranges, const uint32_t *order, const Payload *payload,
                    const CUtensorMap &pay_map, const float4 *wcull, const ItemFrame *iframe, float *color,
                    float *remaining, int32_t *count, int32_t *n_eval, unsigned long long *counters,
                    int32_t *fixup_list, cudaStream_t st) {
    if (max_items <= 0) return;
    raster_smem_optin();
    if (fc.model == GEER_BEAP) {
        k_forward<true><<<max_items, kFwdThreads, sizeof(FwdSmem) + 128, st>>>(
            fc, sc, items, n_items, pix_list, col_sc, row_sc, dir64, ranges, order, pay_map, wcull, iframe, color,
            remaining, count, n_eval, counters, fixup_list);
        k_fixup<true><<<148 * 8, 128, 0, st>>>(fc, sc, items, pix_list, col_sc, row_sc, dir64, ranges, order, payload,
                                               counters, fixup_list, color, remaining, count, n_eval);
    } else {
        k_forward<false><<<max_items, kFwdThreads, sizeof(FwdSmem) + 128, st>>>(
            fc, sc, items, n_items, pix_list, col_sc, row_sc, dir64, ranges, order, pay_map, wcull, iframe, color,
            remaining, count, n_eval, counters, fixup_list);
        k_fixup<false><<<148 * 8, 128, 0, st>>>(fc, sc, items, pix_list, col_sc, row_sc, dir64, ranges, order, payload,
                                                counters, fixup_list, color, remaining, count, n_eval);
    }
}

void launch_backward(const FrameConst &fc, const geer_scene &sc, int max_items, const int4 *items,
                     const int32_t *n_items, const int32_t *pix_list, const double2 *col_sc, const double2 *row_sc,
                     const double *dir64, const int32_t *ranges, const uint32_t *order, const CUtensorMap &pay_map,
                     const float4 *wcull, const ItemFrame *iframe, const float *remaining, const int32_t *n_eval,
                     const float *dl_dimage, float *accum, cudaStream_t st) {
    if (max_items <= 0) return;
    raster_smem_optin();
    if (fc.model == GEER_BEAP)
        k_backward<true><<<max_items, kPipeThreads, sizeof(BwdSmem) + 128, st>>>(
            fc, sc, items, n_items, pix_list, col_sc, row_sc, dir64, ranges, order, pay_map, wcull, iframe, remaining,
            n_eval, dl_dimage, accum);
    else
        k_backward<false><<<max_items, kPipeThreads, sizeof(BwdSmem) + 128, st>>>(
            fc, sc, items, n_items, pix_list, col_sc, row_sc, dir64, ranges, order, pay_map, wcull, iframe, remaining,
            n_eval, dl_dimage, accum);
}

void launch_warp_cull(const FrameConst &fc, int max_items, const int4 *items, const int32_t *n_items,
                      const int32_t *pix_list, const double2 *col_sc, const double2 *row_sc, const double *dir64,
                      float4 *wcull, ItemFrame *iframe, cudaStream_t st) {
    if (max_items <= 0) return;
    if (fc.model == GEER_BEAP)
        k_warp_cull<true><<<max_items, kRasterThreads, 0, st>>>(fc, items, n_items, pix_list, col_sc, row_sc, dir64, wcull, iframe);
    else
        k_warp_cull<false><<<max_items, kRasterThreads, 0, st>>>(fc, items, n_items, pix_list, col_sc, row_sc, dir64, wcull, iframe);
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

#ifdef GEER_CTA_TIMING
extern "C" int geer_debug_cta_phases(unsigned long long *ts, unsigned long long *tf, int n) {
    if (n > (1 << 16)) n = 1 << 16;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(ts, geer::g_cta_ts, sizeof(unsigned long long) * n);
    cudaMemcpyFromSymbol(tf, geer::g_cta_tf, sizeof(unsigned long long) * n);
    return (int)cudaGetLastError();
}
extern "C" int geer_debug_cta_times(unsigned long long *t0, unsigned long long *t1, int *sm, int *went, int n) {
    if (n > (1 << 16)) n = 1 << 16;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(t0, geer::g_cta_t0, sizeof(unsigned long long) * n);
    cudaMemcpyFromSymbol(t1, geer::g_cta_t1, sizeof(unsigned long long) * n);
    cudaMemcpyFromSymbol(sm, geer::g_cta_sm, sizeof(int) * n);
    cudaMemcpyFromSymbol(went, geer::g_cta_went, sizeof(int) * n);
    return (int)cudaGetLastError();
}
#endif
