// sm_100a kernels of the VQhull hot path (see DESIGN.md for the roofline of
// each one).  Reference behaviour each kernel reproduces is cited inline.
//
// Default pipeline (split root):
//   K_S poly_sample_kernel      16-gon filter polygon from a sample of the input
//   K_F root_filter_tma         (partition.cu) filter + survivors + find_extremes
//   KT  tail_kernel             (tail.cu) every recursion level in one launch
//   K0  tiny_hull_kernel        the whole hull of n <= kFinMax points in one CTA
// Kernels shared with the other root modes and the host-driven levels:
//   K1  extremes_kernel         find_extremes            geometry.cpp:7-36
//   KA  bootstrap_argmax_kernel bootstrap pass p,q,p     hull.cpp:228-235 (+ finiteness check vqhull_c.cpp:32-34)
//   KB  root_partition_kernel   levels 1+2 fused: the bootstrap split AND the
//                               two child partitions in ONE pass over the input
//   K2  level_kernel / level_tma  extract_blocks (fused classify + two-sided
//                               compaction + arg-max), all live segments of a
//                               level in one launch       extract_core.hpp:421-515
//   K3  planner_kernel          recursion driver: child -> segment/finisher
//                               tables, tile offsets       hull.cpp:78-115
//   K3' finisher_all_kernel     whole subtrees of small segments: a CTA each up to
//                               kFinMax points, a warp each up to kFinSmall
//                               (explicit stack)           hull.cpp:119-190
//   K4  size/emit kernels       in-order chain assembly    hull.cpp:59-73, 259-266
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

#include "common.cuh"
#include "hull_types.cuh"
#include "kernels.h"

namespace vqb {


// ===========================================================================
// K1: extremes.  lo = lexicographic min of (x, y, index); hi = max x, then
// max y, then min index.  y is read only on x ties, like the reference scan;
// the (x, y, index) total order makes the grid reduction independent of the
// visiting order.  Branch-free per point (compare + select); an exact x tie
// with the running extreme takes a warp-uniform slow path that reads y.
// ===========================================================================
struct ExtPartial {
    ExtKey lo, hi;
    uint32_t nonfinite, pad;
};

constexpr int kStreamUnroll = 4;  // double2 loads per array per thread per iteration

__global__ void __launch_bounds__(256) extremes_kernel(const double* __restrict__ xs,
                                                       const double* __restrict__ ys,
                                                       uint64_t n, ExtPartial* partials,
                                                       uint32_t* ticket, RootInfo* root) {
    VQB_PDL();
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    // running extremes (x, index); the first index wins among exact x ties
    // unless y decides (checked on the slow path)
    double lo_x = kInf, hi_x = -kInf;
    uint32_t lo_i = 0xffffffffu, hi_i = 0xffffffffu;
    bool bad = false;  // non-finite x (vqhull_c.cpp:32-34; y is checked by the pass that reads it)
    auto visit = [&](uint32_t i, double x) {
        bad |= nonfinite_bits(x);
        const bool lt = x < lo_x, gt = x > hi_x;
        const bool tie = (x == lo_x) | (x == hi_x);
        // grid-stride trip counts differ per lane: vote over the lanes that
        // are actually here (a full-mask vote would be undefined behaviour)
        if (__any_sync(__activemask(), tie)) {
            // exact x tie: smaller (larger) y wins; equal y keeps the earlier index
            if (x == lo_x && lo_i != 0xffffffffu && ys[i] < ys[lo_i]) lo_i = i;
            if (x == hi_x && hi_i != 0xffffffffu && ys[i] > ys[hi_i]) hi_i = i;
        }
        lo_i = lt ? i : lo_i;
        lo_x = lt ? x : lo_x;
        hi_i = gt ? i : hi_i;
        hi_x = gt ? x : hi_x;
    };
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t stride = gridDim.x * blockDim.x;
    const bool vec = (reinterpret_cast<uintptr_t>(xs) & 15u) == 0;
    if (vec) {
        const uint32_t npair = uint32_t(n / 2);
        const double2* x2 = reinterpret_cast<const double2*>(xs);
        uint32_t j = tid;
        for (; j + (kStreamUnroll - 1) * stride < npair; j += kStreamUnroll * stride) {
            double2 v[kStreamUnroll];
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u) v[u] = __ldcs(&x2[j + u * stride]);
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u) {
                visit(2 * (j + u * stride), v[u].x);
                visit(2 * (j + u * stride) + 1, v[u].y);
            }
        }
        for (; j < npair; j += stride) {
            const double2 v = __ldcs(&x2[j]);
            visit(2 * j, v.x);
            visit(2 * j + 1, v.y);
        }
        if ((n & 1) && tid == 0) visit(uint32_t(n - 1), xs[n - 1]);
    } else {
        for (uint32_t i = tid; i < n; i += stride) visit(i, xs[i]);
    }
    // NaN inputs never win a comparison; they are rejected by KA anyway
    ExtKey lo{lo_x, 0.0, lo_i, lo_i != 0xffffffffu};
    ExtKey hi{hi_x, 0.0, hi_i, hi_i != 0xffffffffu};
    if (lo.valid) lo.y = ys[lo_i];
    if (hi.valid) hi.y = ys[hi_i];
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        ExtKey a = shfl_key(lo, s);
        if (lo_better(a, lo)) lo = a;
        ExtKey b = shfl_key(hi, s);
        if (hi_better(b, hi)) hi = b;
    }
    __shared__ ExtKey s_lo[8], s_hi[8];
    __shared__ bool s_last;
    __shared__ uint32_t s_bad;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    if (bad) atomicOr(&s_bad, 1u);
    if (lane == 0) { s_lo[warp] = lo; s_hi[warp] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) {
            if (lo_better(s_lo[w], lo)) lo = s_lo[w];
            if (hi_better(s_hi[w], hi)) hi = s_hi[w];
        }
        partials[blockIdx.x].lo = lo;
        partials[blockIdx.x].hi = hi;
        partials[blockIdx.x].nonfinite = s_bad;
        __threadfence();
        const uint32_t t = atomicAdd(ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    ExtKey L, H;
    L.valid = H.valid = 0;
    uint32_t nb = 0;
    for (uint32_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
        ExtKey a, c;
        a.x = __ldcg(&partials[b].lo.x); a.y = __ldcg(&partials[b].lo.y);
        a.idx = __ldcg(&partials[b].lo.idx); a.valid = __ldcg(&partials[b].lo.valid);
        c.x = __ldcg(&partials[b].hi.x); c.y = __ldcg(&partials[b].hi.y);
        c.idx = __ldcg(&partials[b].hi.idx); c.valid = __ldcg(&partials[b].hi.valid);
        nb |= __ldcg(&partials[b].nonfinite);
        if (lo_better(a, L)) L = a;
        if (hi_better(c, H)) H = c;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        ExtKey a = shfl_key(L, s);
        if (lo_better(a, L)) L = a;
        ExtKey b = shfl_key(H, s);
        if (hi_better(b, H)) H = b;
        nb |= __shfl_xor_sync(kFull, nb, s);
    }
    __syncthreads();
    if (lane == 0 && nb) atomicOr(&s_bad, 2u);
    if (lane == 0) { s_lo[warp] = L; s_hi[warp] = H; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) {
            if (lo_better(s_lo[w], L)) L = s_lo[w];
            if (hi_better(s_hi[w], H)) H = s_hi[w];
        }
        root->p_idx = L.idx;
        root->q_idx = H.idx;
        root->px = L.x;
        root->py = L.y;
        root->qx = H.x;
        root->qy = H.y;
        root->nonfinite = (s_bad & 2u) ? 1u : 0u;
        *ticket = 0;  // re-arm for the next launch
    }
}

// ===========================================================================
// KA: bootstrap arg-max.  One read-only pass: which side of p->q / q->p each
// point falls on, |S1|, |S2|, and r1/r2 in the canonical order.  No writes:
// the split itself is recomputed (fused with the next level) by KB.
// Also folds in vqhull_compute's finiteness check (vqhull_c.cpp:32-34).
//  * left of p->q is A*D > B*C and left of q->p is C*B > D*A with the same
//    two products (IEEE products commute), and the second implies "not the
//    first", so mask_b &= ~mask_a (kernels.hpp:91) holds automatically;
//  * the q->p frame is the exact negation of the p->q frame, so one offset o
//    serves both sides: S1 prefers the smallest o, S2 the smallest -o (the
//    largest o); equal offsets (incl. +-0) go to the slow path's
//    lexicographic / first-index tie-break.
// ===========================================================================
struct RootPartial {
    uint32_t cnt1, cnt2, nonfinite, pad;
    Best b1, b2;
};


__global__ void __launch_bounds__(256) bootstrap_argmax_kernel(
    const double* __restrict__ xs, const double* __restrict__ ys, uint64_t n,
    RootPartial* partials, uint32_t* ticket, RootInfo* root) {
    VQB_PDL();
    const double px = root->px, py = root->py, qx = root->qx, qy = root->qy;
    const double adx = dsub(qx, px), ady = dsub(qy, py);  // frame of p->q (kernels.hpp:23-25)
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    uint32_t c1 = 0, c2 = 0;
    bool bad = false;
    double o1 = kInf, o2 = -kInf;  // S1: min o, S2: max o
    uint32_t i1 = 0xffffffffu, i2 = 0xffffffffu;
    auto visit = [&](uint32_t i, double ux, double uy) {
        bad |= nonfinite_bits(ux) | nonfinite_bits(uy);
        const double A = dsub(px, ux), B = dsub(py, uy);
        const double Cc = dsub(qx, ux), D = dsub(qy, uy);
        const double t1 = dmul(A, D), t2 = dmul(B, Cc);
        const bool la = t1 > t2;  // left of p->q
        const bool lb = t2 > t1;  // left of q->p (and therefore not of p->q)
        c1 += la;
        c2 += lb;
        const double o = lat_off(adx, ady, ux, uy);
        const bool maybe = (la && !(o > o1)) || (lb && !(o < o2));
        if (__any_sync(__activemask(), maybe)) {  // lanes may be in different iterations
            if (maybe) {
                const bool s = la;
                const double ob = s ? o1 : o2;
                const uint32_t ib = s ? i1 : i2;
                bool take = s ? (o < ob) : (o > ob);
                take |= ib == 0xffffffffu;
                if (!take && o == ob && i != ib) {  // exact tie: smaller (x, y), then index
                    const double xb = xs[ib], yb = ys[ib];
                    take = (ux != xb) ? (ux < xb) : ((uy != yb) ? (uy < yb) : (i < ib));
                }
                if (take && s) { o1 = o; i1 = i; }
                if (take && !s) { o2 = o; i2 = i; }
            }
        }
    };
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t stride = gridDim.x * blockDim.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(xs) | reinterpret_cast<uintptr_t>(ys)) & 15u) == 0;
    if (vec) {
        const uint32_t npair = uint32_t(n / 2);
        const double2* x2 = reinterpret_cast<const double2*>(xs);
        const double2* y2 = reinterpret_cast<const double2*>(ys);
        uint32_t j = tid;
        for (; j + (kStreamUnroll - 1) * stride < npair; j += kStreamUnroll * stride) {
            double2 vx[kStreamUnroll], vy[kStreamUnroll];
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u) {
                vx[u] = __ldcs(&x2[j + u * stride]);
                vy[u] = __ldcs(&y2[j + u * stride]);
            }
#pragma unroll
            for (int u = 0; u < kStreamUnroll; ++u) {
                visit(2 * (j + u * stride), vx[u].x, vy[u].x);
                visit(2 * (j + u * stride) + 1, vx[u].y, vy[u].y);
            }
        }
        for (; j < npair; j += stride) {
            const double2 vx = __ldcs(&x2[j]);
            const double2 vy = __ldcs(&y2[j]);
            visit(2 * j, vx.x, vy.x);
            visit(2 * j + 1, vx.y, vy.y);
        }
        if ((n & 1) && tid == 0) visit(uint32_t(n - 1), xs[n - 1], ys[n - 1]);
    } else {
        for (uint32_t i = tid; i < n; i += stride) visit(i, xs[i], ys[i]);
    }
    // thread candidates -> Best (S2's offset in its own frame is -o)
    Best b1 = best_none(), b2 = best_none();
    if (i1 != 0xffffffffu) { b1.off = o1; b1.x = xs[i1]; b1.y = ys[i1]; b1.idx = i1; b1.valid = 1; }
    if (i2 != 0xffffffffu) { b2.off = -o2; b2.x = xs[i2]; b2.y = ys[i2]; b2.idx = i2; b2.valid = 1; }
    uint32_t ubad = bad ? 1u : 0u;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        c1 += __shfl_xor_sync(kFull, c1, s);
        c2 += __shfl_xor_sync(kFull, c2, s);
        ubad |= __shfl_xor_sync(kFull, ubad, s);
    }
    b1 = warp_best(b1);
    b2 = warp_best(b2);
    __shared__ RootPartial s_p[8];
    __shared__ bool s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        s_p[warp].cnt1 = c1;
        s_p[warp].cnt2 = c2;
        s_p[warp].nonfinite = ubad;
        s_p[warp].b1 = b1;
        s_p[warp].b2 = b2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        RootPartial r = s_p[0];
        for (int w = 1; w < int(blockDim.x >> 5); ++w) {
            r.cnt1 += s_p[w].cnt1;
            r.cnt2 += s_p[w].cnt2;
            r.nonfinite |= s_p[w].nonfinite;
            if (prefer(s_p[w].b1, r.b1)) r.b1 = s_p[w].b1;
            if (prefer(s_p[w].b2, r.b2)) r.b2 = s_p[w].b2;
        }
        partials[blockIdx.x] = r;
        __threadfence();
        const uint32_t t = atomicAdd(ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (warp != 0) return;
    uint32_t C1 = 0, C2 = 0, BAD = 0;
    Best B1 = best_none(), B2 = best_none();
    for (uint32_t b = lane; b < gridDim.x; b += 32) {
        const RootPartial* p = &partials[b];
        C1 += __ldcg(&p->cnt1);
        C2 += __ldcg(&p->cnt2);
        BAD |= __ldcg(&p->nonfinite);
        Best x1, x2;
        x1.off = __ldcg(&p->b1.off); x1.x = __ldcg(&p->b1.x); x1.y = __ldcg(&p->b1.y);
        x1.idx = __ldcg(&p->b1.idx); x1.valid = __ldcg(&p->b1.valid);
        x2.off = __ldcg(&p->b2.off); x2.x = __ldcg(&p->b2.x); x2.y = __ldcg(&p->b2.y);
        x2.idx = __ldcg(&p->b2.idx); x2.valid = __ldcg(&p->b2.valid);
        if (prefer(x1, B1)) B1 = x1;
        if (prefer(x2, B2)) B2 = x2;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        C1 += __shfl_xor_sync(kFull, C1, s);
        C2 += __shfl_xor_sync(kFull, C2, s);
        BAD |= __shfl_xor_sync(kFull, BAD, s);
    }
    B1 = warp_best(B1);
    B2 = warp_best(B2);
    if (lane == 0) {
        root->cnt1 = C1;
        root->cnt2 = C2;
        root->nonfinite = BAD;
        root->r1 = B1;
        root->r2 = B2;
        *ticket = 0;
    }
}

// ===========================================================================
// K1' (default root stage) = K1 (extremes_kernel: find_extremes,
// geometry.cpp:7-36, over every point; x read for every point, y only on
// exact x ties; finiteness of x) + this sample kernel: the octagon filter's
// 8 vertices from a sample of the input (every 16th group of 1024 points, x
// and y): min/max x, y, x+y, x-y.  Two kernels, so the x stream keeps K1's
// small register footprint (occupancy, loads in flight).  The filter
// only needs its vertices to be input points (see poly_finish), not exact
// extremes, so a sample costs 1/16 of a y pass and loses almost nothing.  Finiteness of
// x is checked here, of y by the root pass that reads every y.
// ===========================================================================
struct PolyPartial {
    ExtKey lo, hi;
    double av[kPolyV];
    uint32_t ai[kPolyV];
    double sx, sy, sn;  // sums over the sample (centre of the filter's inner box)
    uint32_t nonfinite;
    uint32_t pad;
};

struct SamplePartial {
    double s[3];  // sample sums of x, y and the count
};

// monotone u32 key of a double rounded to f32 (larger value -> larger key)
__device__ __forceinline__ uint32_t f32_order_key(double v) {
    const uint32_t u = __float_as_uint(__double2float_rn(v));
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// diagnostics (VQHULL_SAMPLE_TRACE, build with -DVQB_STAMPS): %globaltimer
// stamps of the sample, filter and tail kernels; compiled out otherwise
__device__ unsigned long long g_strace[8];
#ifdef VQB_STAMPS
#define VQB_STAMP(...) __VA_ARGS__
#else
#define VQB_STAMP(...)
#endif
__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int kSampleShift = 9;  // groups of 512 pairs (1024 points, 8 KB of x and of y)
constexpr int kSampleUnroll = 4;  // double2 loads per array per thread in flight

// Last step of K1' (one warp, poly_finish_warp): p, q (exact, in the
// one-pass octagon root), the octagon filter (the sample's 8 directional
// extremes: mutually consistent, so in convex position up to rounding ties —
// exact p, q would not be, e.g. when one far point of a heavy-tailed input
// dominates), its chord forms and inner box, the emission frame.
// Every vertex is an input point, so the region right of all 8 chords (the
// octagon, or its kernel if rounding ties made it non-convex) lies in the
// hull.  M bounds |coordinates| of the vertices, hence of every point the
// filter can drop; the margin is 2^-32 M (~10^5 ulps of M), so the fused
// multiply-adds' rounding can never reach a dropped point and no reference
// predicate can see one as a hull or farthest candidate.  Outside
// 2^-400 <= M <= 2^500 (products could underflow/overflow): no filter.
// One warp: lane l owns vertex / chord j = l & 15 (each twice) and a share of
// the inside-tests, so a candidate region costs a few FMAs and one vote.
__device__ int g_inner_force = -1;  // set_filter_inner

__device__ __noinline__ void poly_finish_warp(const PolyPartial& F, const double* __restrict__ xs,
                                              const double* __restrict__ ys, RootInfo* root, bool with_pq) {
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    const int lane = threadIdx.x & 31, j = lane & (kPolyV - 1), half = lane >> 4;
    const ExtKey L = F.lo, H = F.hi;
    const uint32_t nb = F.nonfinite;
    RootInfo& R = *root;
    RootPoly& P = R.poly;
    bool ok = with_pq ? (L.valid && H.valid && nb == 0) : true;
    const uint32_t aj = F.ai[j];
    const uint32_t ij = aj != kNoIdx ? aj : (L.valid ? L.idx : 0u);  // n >= 1
    const double vxj = xs[ij], vyj = ys[ij];
    ok &= __all_sync(kFull, aj != kNoIdx);
    auto VX = [&](int k) { return __shfl_sync(kFull, vxj, k); };
    auto VY = [&](int k) { return __shfl_sync(kFull, vyj, k); };
    auto wmax = [&](double v) {
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, s));
        return v;
    };
    auto wmin = [&](double v) {
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) v = fmin(v, __shfl_xor_sync(kFull, v, s));
        return v;
    };
    const double M = wmax(fmax(fabs(vxj), fabs(vyj)));
    ok &= M >= 0x1p-400 && M <= 0x1p500;
    // chord j = V_j -> V_{j+1}
    const double nxj = VX((j + 1) & (kPolyV - 1)), nyj = VY((j + 1) & (kPolyV - 1));
    const double ex = nxj - vxj, ey = nyj - vyj;
    const bool deg = ex == 0.0 && ey == 0.0;  // degenerate chord: no constraint
    const double fa = deg ? 0.0 : -ey;
    const double fb = deg ? 0.0 : ex;
    const double fc = deg ? -1.0 : ey * vxj - ex * vyj;
    const double ft = deg ? 0.0 : -0x1p-32 * M * (fabs(ex) + fabs(ey));
    const int chords = __popc(__ballot_sync(kFull, !deg)) / 2;
    auto in_j = [&](double x, double y) { return __fma_rn(fa, x, __fma_rn(fb, y, fc)) < ft; };
    auto inside_pt = [&](double x, double y) { return __all_sync(kFull, in_j(x, y)); };
    auto inside_box = [&](double x0, double x1, double y0, double y1) {  // corners half, half + 2
        return __all_sync(kFull, in_j((half & 1) ? x1 : x0, y0) && in_j((half & 1) ? x1 : x0, y1));
    };
    // octagon {|X| < hx, |Y| < hy, |X| + |Y| < d} around (cx, cy): its
    // vertices (+-hx, +-min(hy, d - hx)), (+-min(hx, d - hy), +-hy)
    auto inside_oct = [&](double cx, double cy, double hx, double hy, double d) {
        const double a = fmin(hy, d - hx), b = fmin(hx, d - hy);
        const double sx = half ? -1.0 : 1.0;
        return __all_sync(kFull, in_j(cx + sx * hx, cy + a) && in_j(cx + sx * hx, cy - a) &&
                                     in_j(cx + sx * b, cy + hy) && in_j(cx + sx * b, cy - hy));
    };
    // inner box between the diagonal vertices (shrunk a little), kept only if
    // its 4 corners pass the test (the filter region is convex)
    const double cx0 = fmax(VX(2), VX(14)), cx1 = fmin(VX(6), VX(10));
    const double cy0 = fmax(VY(10), VY(14)), cy1 = fmin(VY(2), VY(6));
    double bx0 = kInf, bx1 = -kInf, by0 = kInf, by1 = -kInf;  // empty
    const double shrink[3] = {0x1p-20 * M, 0x1p-10 * M, 0.0625 * fmax(cx1 - cx0, cy1 - cy0)};
    for (int t = 0; t < 3; ++t) {
        const double x0 = cx0 + shrink[t], x1 = cx1 - shrink[t];
        const double y0 = cy0 + shrink[t], y1 = cy1 - shrink[t];
        if (x0 < x1 && y0 < y1 && inside_box(x0, x1, y0, y1)) {
            bx0 = x0; bx1 = x1; by0 = y0; by1 = y1;
            break;
        }
    }
    const double xmin = wmin(vxj), xmax = wmax(vxj), ymin = wmin(vyj), ymax = wmax(vyj);
    // second candidate: the largest box around the sample's mean with the
    // polygon's aspect (closed form per chord), verified like the first
    const bool mean_ok = F.sn > 0.0;
    const double mx = mean_ok ? F.sx / F.sn : 0.0, my = mean_ok ? F.sy / F.sn : 0.0;
    if (mean_ok) {
        const double W = 0.5 * (xmax - xmin), Hh = 0.5 * (ymax - ymin);
        if (inside_pt(mx, my) && W > 0.0 && Hh > 0.0) {
            const double f0 = fa * mx + fb * my + fc;
            const double g = fabs(fa) * W + fabs(fb) * Hh;
            double t = wmin(g > 0.0 ? fmin(1.0, (ft - f0) / g) : 1.0);
            for (int tries = 0; tries < 4 && t > 0.0; ++tries, t *= 0.5) {
                const double x0 = mx - 0.999 * t * W, x1 = mx + 0.999 * t * W;
                const double y0 = my - 0.999 * t * Hh, y1 = my + 0.999 * t * Hh;
                if (x0 < x1 && y0 < y1 && inside_box(x0, x1, y0, y1)) {
                    const double a_old = bx0 < bx1 ? (bx1 - bx0) * (by1 - by0) : 0.0;
                    if ((x1 - x0) * (y1 - y0) > a_old) { bx0 = x0; bx1 = x1; by0 = y0; by1 = y1; }
                    break;
                }
            }
        }
    }
    // the octagon, for the points outside the box: around the box centre (or
    // the mean), the polygon's own extents in x, y and x +- y, scaled by the
    // largest s that keeps its 8 vertices inside every chord (closed form)
    double ocx = 0.0, ocy = 0.0, ohx = -1.0, ohy = -1.0, od = -1.0;  // empty: |.| < -1 never holds
    double dcx = 0.0, dcy = 0.0, dr2 = -1.0;                           // empty disk
    {
        const bool have_box = bx0 < bx1;
        const double cx = have_box ? 0.5 * (bx0 + bx1) : mx, cy = have_box ? 0.5 * (by0 + by1) : my;
        if ((have_box || mean_ok) && inside_pt(cx, cy)) {
            const double Wx = wmax(fabs(vxj - cx)), Wy = wmax(fabs(vyj - cy));
            const double Wd = wmax(fabs(vxj - cx) + fabs(vyj - cy));
            const double a = fmin(Wy, Wd - Wx), b = fmin(Wx, Wd - Wy);
            const double f0 = fa * cx + fb * cy + fc;
            // this lane's chord against the vertices of its half
            const double sx = half ? -1.0 : 1.0;
            const double den[4] = {fa * sx * Wx + fb * a, fa * sx * Wx - fb * a, fa * sx * b + fb * Wy,
                                   fa * sx * b - fb * Wy};
            double s = kInf;
#pragma unroll
            for (int v = 0; v < 4; ++v)
                if (den[v] > 0.0) s = fmin(s, (ft - f0) / den[v]);
            s = 0.999 * wmin(s);
            for (int tries = 0; tries < 4 && s > 0.0 && s < kInf; ++tries, s *= 0.5) {
                const double hx = s * Wx, hy = s * Wy, d = s * Wd;
                if (hx > 0.0 && hy > 0.0 && inside_oct(cx, cy, hx, hy, d)) {
                    ocx = cx; ocy = cy; ohx = hx; ohy = hy; od = d;
                    break;
                }
            }
            // the disk around (cx, cy): radius = 0.999 x the distance to the
            // nearest chord line, ft - f0 being the chord's slack at the centre.
            // A slack within 2^-40 of the operands' scale (rounding of f0) voids
            // it.  For |P - C| < r: f_j(P) <= f_j(C) + |n_j| r < ft_j exactly,
            // so the disk lies inside every chord's margin; the pass kernel
            // tests fma(du, du, dw dw) < r^2 (1 - 2^-30), which bounds the true
            // distance below r through its three roundings.
            const double nrm = sqrt(fa * fa + fb * fb);
            const double slack = ft - f0;
            const double scale = fabs(fa * cx) + fabs(fb * cy) + fabs(fc);
            const double rj = deg ? kInf : (nrm > 0.0 && slack > 0x1p-40 * scale ? slack / nrm : -1.0);
            const double r = 0.999 * wmin(rj);
            if (r > 0.0 && r < kInf) {
                dcx = cx; dcy = cy; dr2 = r * r * (1.0 - 0x1p-30);
            }
        }
    }
    ok &= chords >= 2;  // all vertices equal: the test would constrain nothing
    if (lane < kPolyV) {
        P.vx[j] = vxj; P.vy[j] = vyj; P.vidx[j] = aj;
        P.fa[j] = fa; P.fb[j] = fb; P.fc[j] = fc; P.ft[j] = ft;
        P.fg[j] = ft - fc;
    }
    // the inner test that adds the most area (a uniform choice per call);
    // when the disk wins and the box adds next to nothing to it (< 1 % of the
    // disk's area lies in the box but outside the disk: 64 midpoint samples,
    // two per lane), the disk is tested alone (3)
    uint32_t inner_mode;
    {
        const double box_area = bx0 < bx1 ? (bx1 - bx0) * (by1 - by0) : 0.0;
        const double cut = fmax(0.0, ohx + ohy - od);
        const double oct_area = ohx > 0.0 ? 4.0 * ohx * ohy - 2.0 * cut * cut : 0.0;
        const double disk_area = dr2 > 0.0 ? 3.14159 * dr2 : 0.0;
        inner_mode = disk_area > 1.02 * fmax(oct_area, box_area) ? 2u : (oct_area > 1.02 * box_area ? 1u : 0u);
        if (inner_mode == 2u) {  // (warp-uniform)
            uint32_t box_out = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int sidx = lane + 32 * h;
                const double sx = bx0 + (bx1 - bx0) * (0.0625 + 0.125 * double(sidx & 7));
                const double sy = by0 + (by1 - by0) * (0.0625 + 0.125 * double(sidx >> 3));
                const bool out = bx0 < bx1 && (sx - dcx) * (sx - dcx) + (sy - dcy) * (sy - dcy) >= dr2;
                box_out += uint32_t(__popc(__ballot_sync(kFull, out)));
            }
            if (double(box_out) * (1.0 / 64.0) * box_area < 0.01 * disk_area) inner_mode = 3u;
        }
    }
    if (lane != 0) return;
    P.mref = M;
    P.bx0 = bx0; P.bx1 = bx1; P.by0 = by0; P.by1 = by1;
    P.ocx = ocx; P.ocy = ocy; P.ohx = ohx; P.ohy = ohy; P.od = od;
    P.dcx = dcx; P.dcy = dcy; P.dr2 = dr2;
    {
        P.oct_on = inner_mode;
        const int f = g_inner_force;  // test knob: a forced choice, when that region exists
        if (f == 0 || (f == 1 && ohx > 0.0) || (f >= 2 && f <= 3 && dr2 > 0.0)) P.oct_on = uint32_t(f);
        P.pad2 = 0u;
    }
    P.filter = ok ? 1u : 0u;
    if (!with_pq) return;
    P.nv = 2;  // emission frame: [p] chain(S1) [q] chain(S2)
    P.ex[0] = L.x; P.ey[0] = L.y; P.eidx[0] = L.idx;
    P.ex[1] = H.x; P.ey[1] = H.y; P.eidx[1] = H.idx;
    R.nonfinite = nb;
    R.p_idx = L.idx;
    R.q_idx = H.idx;
    R.px = L.x; R.py = L.y;
    R.qx = H.x; R.qy = H.y;
}

__global__ void __launch_bounds__(256, 2) poly_sample_kernel(const double* __restrict__ xs,
                                                            const double* __restrict__ ys, uint64_t n,
                                                            SamplePartial* partials, uint32_t* ticket,
                                                            unsigned long long* keys, RootInfo* root,
                                                            unsigned long long* side_ctr, int with_pq,
                                                            uint32_t smask) {
    VQB_PDL();
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    // slot j: the extreme of the functional of direction j (clockwise from
    // -x, see RootPoly): 0 min x, 1 min 2x-y, 2 min x-y, 3 min x-2y, 4 max y,
    // 5 max x+2y, 6 max x+y, 7 max 2x+y, 8 max x, 9 max 2x-y, 10 max x-y,
    // 11 max x-2y, 12 min y, 13 min x+2y, 14 min x+y, 15 min 2x+y
    double av[kPolyV];
    uint32_t ai[kPolyV];
#pragma unroll
    for (int a = 0; a < kPolyV; ++a) {
        av[a] = (a >= 4 && a <= 11) ? -kInf : kInf;
        ai[a] = kNoIdx;
    }
    double ssx = 0.0, ssy = 0.0;  // sample sums (non-finite input is rejected anyway)
    uint32_t ssn = 0;
    auto visit_xy = [&](uint32_t i, double x, double y) {
        const double s = __dadd_rn(x, y), d = __dsub_rn(x, y);
        const double u1 = __dadd_rn(x, s), u2 = __dadd_rn(y, s);  // 2x+y, x+2y
        const double u3 = __dadd_rn(x, d), u4 = __dsub_rn(d, y);  // 2x-y, x-2y
        ssx = __dadd_rn(ssx, x);
        ssy = __dadd_rn(ssy, y);
        ++ssn;
        const double val[kPolyV] = {x, u3, d, u4, y, u2, s, u1, x, u3, d, u4, y, u2, s, u1};
#pragma unroll
        for (int a = 0; a < kPolyV; ++a) {
            const bool maximize = (a >= 4 && a <= 11);
            const bool take = maximize ? val[a] > av[a] : val[a] < av[a];
            av[a] = take ? val[a] : av[a];
            ai[a] = take ? i : ai[a];
        }
    };
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t stride = gridDim.x * blockDim.x;
    VQB_STAMP(if (tid == 0) g_strace[0] = gtimer_ns();)
    const bool vec = ((reinterpret_cast<uintptr_t>(xs) | reinterpret_cast<uintptr_t>(ys)) & 15u) == 0;
    if (vec) {
        const uint32_t npair = uint32_t(n / 2);
        const double2* x2 = reinterpret_cast<const double2*>(xs);
        const double2* y2 = reinterpret_cast<const double2*>(ys);
        if ((n & 1) && tid == 0) visit_xy(uint32_t(n - 1), xs[n - 1], ys[n - 1]);
        // x and y of the sampled groups (every 16th run of 512 pairs)
        const uint32_t ngroups = (npair + (1u << kSampleShift) - 1) >> kSampleShift;
        const uint32_t nsg = (ngroups + smask) / (smask + 1);
        const uint32_t nsample = nsg << kSampleShift;
        auto pair_of = [&](uint32_t m) {
            return ((m >> kSampleShift) * (smask + 1) << kSampleShift) | (m & ((1u << kSampleShift) - 1));
        };
        uint32_t m = tid;
        for (; m + (kSampleUnroll - 1) * stride < nsample; m += kSampleUnroll * stride) {
            double2 v[kSampleUnroll], w[kSampleUnroll];
            uint32_t jj[kSampleUnroll];
#pragma unroll
            for (int u = 0; u < kSampleUnroll; ++u) {
                jj[u] = pair_of(m + u * stride);
                const uint32_t q = jj[u] < npair ? jj[u] : 0u;
                v[u] = __ldcs(&x2[q]);
                w[u] = __ldcs(&y2[q]);
            }
#pragma unroll
            for (int u = 0; u < kSampleUnroll; ++u) {
                if (jj[u] >= npair) continue;
                visit_xy(2 * jj[u], v[u].x, w[u].x);
                visit_xy(2 * jj[u] + 1, v[u].y, w[u].y);
            }
        }
        for (; m < nsample; m += stride) {
            const uint32_t q = pair_of(m);
            if (q >= npair) continue;
            const double2 v = __ldcs(&x2[q]);
            const double2 w = __ldcs(&y2[q]);
            visit_xy(2 * q, v.x, w.x);
            visit_xy(2 * q + 1, v.y, w.y);
        }
    } else {
        for (uint32_t i = tid; i < n; i += stride)
            if (((i >> (kSampleShift + 1)) & smask) == 0) visit_xy(i, xs[i], ys[i]);
    }
    VQB_STAMP(if (threadIdx.x == 0) atomicMax(&g_strace[1], gtimer_ns());)
    // Reductions.  A vertex only has to be SOME input point (see
    // poly_finish_warp), so the CTAs combine their directional extremes with
    // one 64-bit atomicMax per direction on {order key of the value rounded to
    // f32, ~index}: order-independent, hence deterministic, and no serial
    // fold.  The sample sums (box centre) are combined in a fixed order.
    __shared__ unsigned long long s_key[kPolyV][8];
    __shared__ double s_sum[3][8];
    __shared__ bool s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long key[kPolyV];
#pragma unroll
    for (int a = 0; a < kPolyV; ++a) {
        const bool maximize = (a >= 4 && a <= 11);
        key[a] = ai[a] == kNoIdx ? 0ull
                                 : (uint64_t(f32_order_key(maximize ? av[a] : -av[a])) << 32) | uint32_t(~ai[a]);
    }
    double sx = ssx, sy = ssy, sn = double(ssn);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int a = 0; a < kPolyV; ++a) {
            const unsigned long long k = __shfl_xor_sync(kFull, key[a], o);
            key[a] = k > key[a] ? k : key[a];
        }
        sx += __shfl_xor_sync(kFull, sx, o);
        sy += __shfl_xor_sync(kFull, sy, o);
        sn += __shfl_xor_sync(kFull, sn, o);
    }
    if (lane == 0) {
#pragma unroll
        for (int a = 0; a < kPolyV; ++a) s_key[a][warp] = key[a];
        s_sum[0][warp] = sx; s_sum[1][warp] = sy; s_sum[2][warp] = sn;
    }
    __syncthreads();
    if (threadIdx.x < kPolyV) {
        unsigned long long k = s_key[threadIdx.x][0];
        for (int w = 1; w < 8; ++w) k = s_key[threadIdx.x][w] > k ? s_key[threadIdx.x][w] : k;
        if (k) atomicMax(&keys[threadIdx.x], k);
    } else if (threadIdx.x < kPolyV + 3) {
        const int c = threadIdx.x - kPolyV;
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += s_sum[c][w];
        partials[blockIdx.x].s[c] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    VQB_STAMP(if (threadIdx.x == 0) g_strace[2] = gtimer_ns();)
    // sums over the CTA partials: strided per thread, then a fixed tree
    sx = sy = sn = 0.0;
    for (uint32_t c = threadIdx.x; c < gridDim.x; c += blockDim.x) {
        sx += __ldcg(&partials[c].s[0]);
        sy += __ldcg(&partials[c].s[1]);
        sn += __ldcg(&partials[c].s[2]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sx += __shfl_xor_sync(kFull, sx, o);
        sy += __shfl_xor_sync(kFull, sy, o);
        sn += __shfl_xor_sync(kFull, sn, o);
    }
    __syncthreads();
    if (lane == 0) { s_sum[0][warp] = sx; s_sum[1][warp] = sy; s_sum[2][warp] = sn; }
    __syncthreads();
    __shared__ PolyPartial s_fin;
    if (threadIdx.x == 0) {
        sx = sy = sn = 0.0;
        for (int w = 0; w < 8; ++w) { sx += s_sum[0][w]; sy += s_sum[1][w]; sn += s_sum[2][w]; }
        s_fin.sx = sx; s_fin.sy = sy; s_fin.sn = sn;
        // p, q and the finiteness of x come from K1 (one-pass octagon root)
        if (with_pq) {
            s_fin.lo = ExtKey{root->px, root->py, root->p_idx, 1u};
            s_fin.hi = ExtKey{root->qx, root->qy, root->q_idx, 1u};
            s_fin.nonfinite = root->nonfinite;
        } else {
            s_fin.lo = ExtKey{0.0, 0.0, kNoIdx, 0u};
            s_fin.hi = s_fin.lo;
            s_fin.nonfinite = 0u;
        }
        s_fin.pad = 0u;
    }
    if (threadIdx.x < kPolyV) {
        const unsigned long long k = __ldcg(&keys[threadIdx.x]);
        s_fin.ai[threadIdx.x] = k ? ~uint32_t(k) : kNoIdx;
        s_fin.av[threadIdx.x] = 0.0;  // unused: vertices are re-read by index
        keys[threadIdx.x] = 0ull;     // re-arm for the next call
    }
    __syncthreads();
    VQB_STAMP(if (threadIdx.x == 0) g_strace[3] = gtimer_ns();)
    if (threadIdx.x >= 32) return;
    poly_finish_warp(s_fin, xs, ys, root, with_pq != 0);
    if (threadIdx.x != 0) return;
    VQB_STAMP(g_strace[4] = gtimer_ns();)
    side_ctr[0] = 0ull;  // the root pass's counter (another root mode may have used it)
    *ticket = 0;
}

// ===========================================================================
// K3: planner — turns the child slots of a level into the next level's work:
// internal segments (m > kFinMax, tiled), finisher segments (2..kFinMax: a
// warp up to kFinSmall, a CTA above),
// leaves (m == 1: the node's chain is just its apex, hull.cpp:83) and empty
// slots.  One single-pass scan with decoupled look-back over slot chunks.
// ===========================================================================
constexpr int kPlanPer = 4;
constexpr int kPlanChunk = kThreads * kPlanPer;

struct PlanArgs {
    const ChildRec* slots;
    uint32_t nslots;      // level 2 only; deeper levels: 2 * prev->nseg
    const LevelInfo* prev;
    uint32_t fin_cap;     // FinRec array capacity (CTA-finisher segments fill it from the back)
    SegRec* segs;
    FinRec* fins;
    uint8_t* kind;
    uint32_t* link;
    LevelInfo* info;
    uint32_t* flags;
    PlanAgg* aggs;
    PlanAgg* incs;
    uint32_t epoch;
    uint32_t* ctr;
    uint32_t* seg_pcnt;
    uint32_t* seg_done;
    unsigned long long* seg_ctr;
    LevelInfo* next_info;  // zeroed here: the planner-free level kernel accumulates into it
};

__device__ __forceinline__ uint8_t kind_of(uint32_t m) {
    return m == 0 ? kEmpty : (m == 1 ? kLeaf : (m <= kFinMax ? kFin : kInternal));
}
__device__ __forceinline__ uint8_t kind_of_cap(uint32_t m, uint32_t fin_max) {
    return m == 0 ? kEmpty : (m == 1 ? kLeaf : (m <= fin_max ? kFin : kInternal));
}

// nblocks: CTAs running the planner (they claim slot chunks dynamically);
// the persistent tail kernel runs it on one CTA.
__device__ __noinline__ void planner_body(const PlanArgs& a, uint32_t nblocks) {
    __shared__ PlanAgg s_w[kWarps];
    __shared__ PlanAgg s_excl;
    __shared__ uint32_t s_chunk;
    // the level's size comes from the previous level on the device, so the
    // host can queue several levels without waiting for their counts
    const uint32_t nslots = a.prev ? 2u * a.prev->nseg : a.nslots;
    const uint32_t nchunks = (nslots + kPlanChunk - 1) / kPlanChunk;
    const uint64_t fin_chain_base = a.prev ? uint64_t(a.prev->fin_base) + a.prev->fin_total : 0ull;
    if (a.next_info && blockIdx.x == 0 && threadIdx.x < sizeof(LevelInfo) / 4)
        reinterpret_cast<uint32_t*>(a.next_info)[threadIdx.x] = 0u;
    if (nslots == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
        LevelInfo li;
        li.nslots = 0; li.nseg = 0; li.nfin = 0; li.ntiles = 0;
        li.out_total = 0; li.fin_total = 0; li.nleaf = 0;
        li.fin_base = uint32_t(fin_chain_base);
        li.nfin2 = 0; li.pad = 0;
        *a.info = li;
    }
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t c = atomicAdd(a.ctr, 1u);
            s_chunk = c;
            if (c >= nchunks && c == nchunks + nblocks - 1) *a.ctr = 0;
        }
        __syncthreads();
        const uint32_t chunk = s_chunk;
        if (chunk >= nchunks) break;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        // blocked: thread owns kPlanPer consecutive slots
        const uint64_t s0 = uint64_t(chunk) * kPlanChunk + uint64_t(threadIdx.x) * kPlanPer;
        uint32_t m[kPlanPer];
        PlanAgg mine;
        pl_clear(mine);
#pragma unroll
        for (int k = 0; k < kPlanPer; ++k) {
            const uint64_t s = s0 + k;
            m[k] = s < nslots ? a.slots[s].m : 0u;
            const uint8_t kd = s < nslots ? kind_of(m[k]) : kEmpty;
            mine.nseg += kd == kInternal;
            mine.nfin += kd == kFin && m[k] <= kFinSmall;
            mine.nfin2 += kd == kFin && m[k] > kFinSmall;
            mine.leaf += kd == kLeaf;
            mine.ntiles += kd == kInternal ? (m[k] + kTile - 1) / kTile : 0;
            mine.out += kd == kInternal ? m[k] : 0;
            mine.fin += kd == kFin ? m[k] : 0;
        }
        // block exclusive scan (warp inclusive scan, then warp totals)
        PlanAgg incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            PlanAgg o;
            o.nseg = __shfl_up_sync(kFull, incl.nseg, d);
            o.nfin = __shfl_up_sync(kFull, incl.nfin, d);
            o.nfin2 = __shfl_up_sync(kFull, incl.nfin2, d);
            o.ntiles = __shfl_up_sync(kFull, incl.ntiles, d);
            o.out = __shfl_up_sync(kFull, incl.out, d);
            o.fin = __shfl_up_sync(kFull, incl.fin, d);
            o.leaf = __shfl_up_sync(kFull, incl.leaf, d);
            if (lane >= d) pl_combine(incl, o);
        }
        if (lane == 31) s_w[warp] = incl;
        __syncthreads();
        if (threadIdx.x < 32) {
            PlanAgg tot;
            pl_clear(tot);
            for (int w = 0; w < kWarps; ++w) pl_combine(tot, s_w[w]);
            const PlanAgg ex = lookback<PlanAgg>(chunk, 0u, tot, a.flags, a.aggs, a.incs, a.epoch);
            if (threadIdx.x == 0) {
                s_excl = ex;
                if (chunk == nchunks - 1) {
                    PlanAgg all = ex;
                    pl_combine(all, tot);
                    LevelInfo li;
                    li.nslots = nslots;
                    li.nseg = all.nseg;
                    li.nfin = all.nfin;
                    li.ntiles = all.ntiles;
                    li.out_total = all.out;
                    li.fin_total = all.fin;
                    li.nleaf = all.leaf;
                    li.fin_base = uint32_t(fin_chain_base);
                    li.nfin2 = all.nfin2;
                    li.pad = 0;
                    *a.info = li;
                }
            }
        }
        __syncthreads();
        PlanAgg run = s_excl;
        for (int w = 0; w < warp; ++w) pl_combine(run, s_w[w]);
        // exclusive within warp
        PlanAgg wex = incl;
        wex.nseg -= mine.nseg; wex.nfin -= mine.nfin; wex.nfin2 -= mine.nfin2; wex.ntiles -= mine.ntiles;
        wex.out -= mine.out; wex.fin -= mine.fin; wex.leaf -= mine.leaf;
        pl_combine(run, wex);
#pragma unroll
        for (int k = 0; k < kPlanPer; ++k) {
            const uint64_t s = s0 + k;
            if (s >= nslots) break;
            const uint8_t kd = kind_of(m[k]);
            a.kind[s] = kd;
            if (kd == kInternal) {
                const ChildRec c = a.slots[s];
                SegRec g;
                g.px = c.px; g.py = c.py; g.rx = c.rx; g.ry = c.ry; g.qx = c.qx; g.qy = c.qy;
                g.bx = c.rx; g.by = c.ry;
                g.adx = dsub(c.rx, c.px); g.ady = dsub(c.ry, c.py);
                g.bdx = dsub(c.qx, c.rx); g.bdy = dsub(c.qy, c.ry);
                g.begin = c.begin;
                g.out = run.out;
                g.m = c.m;
                g.tile0 = run.ntiles;
                g.ntiles = (c.m + kTile - 1) / kTile;
                g.slot = uint32_t(s);
                a.segs[run.nseg] = g;
                a.seg_pcnt[run.nseg] = 0;
                a.seg_done[run.nseg] = 0;
                a.seg_ctr[run.nseg] = 0ull;
                a.link[s] = run.nseg;
                run.nseg += 1;
                run.ntiles += g.ntiles;
                run.out += c.m;
            } else if (kd == kFin) {
                FinRec f;
                f.c = a.slots[s];
                f.chain_base = fin_chain_base + run.fin;
                f.slot = uint32_t(s);
                f.pad = 0;
                // warp-finisher segments from the front of the FinRec array,
                // CTA-finisher segments from the back
                const uint32_t fi = m[k] <= kFinSmall ? run.nfin : a.fin_cap - 1u - run.nfin2;
                a.fins[fi] = f;
                a.link[s] = fi;
                run.nfin += m[k] <= kFinSmall;
                run.nfin2 += m[k] > kFinSmall;
                run.fin += m[k];
            } else {
                a.link[s] = 0;
                run.leaf += (kd == kLeaf);
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads) planner_kernel(const __grid_constant__ PlanArgs a) {
    VQB_PDL();
    planner_body(a, gridDim.x);
}

// tile -> segment map (binary search over the segments' first tiles)
__global__ void tilemap_kernel(const SegRec* segs, const LevelInfo* info, uint32_t* tile_seg) {
    VQB_PDL();
    const uint32_t nseg = info->nseg, ntiles = info->ntiles;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles;
         t += gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = nseg;  // find last k with tile0 <= t
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (segs[mid].tile0 <= t) lo = mid; else hi = mid;
        }
        tile_seg[t] = lo;
    }
}

// ===========================================================================
// K3': warp finisher.  One warp solves the whole subtree of a segment with
// m <= kFinSmall points in shared memory, depth-first with an explicit stack
// (the reference's chain_iterative, hull.cpp:119-190), emitting the chain
// in order: chain(L) ++ [r] ++ chain(R)  (assemble_chain, hull.cpp:59-73).
// Points are referenced by local ids; the two working arrays ping-pong per
// depth so a child's range never overlaps a pending sibling's.
// ===========================================================================
constexpr uint16_t kNoLid = 0xffffu;

struct FinFrame {
    uint16_t lo, hi, p, r, q, rcnt, rR;
    uint8_t buf, phase;
};

struct FinSmem {
    double x[kFinSmall + 3];
    double y[kFinSmall + 3];
    uint32_t gid[kFinSmall + 3];
    uint16_t work[2][kFinSmall];
    FinFrame stack[kFinSmall + 2];
};

// canonical order on local ids when the offsets tie exactly: smaller (x, y),
// then the smaller global (first-occurrence) index
__device__ __forceinline__ bool fin_tie_better(uint16_t a, uint16_t b, const FinSmem& S) {
    if (a == kNoLid || a == b) return false;
    if (b == kNoLid) return true;
    if (S.x[a] != S.x[b]) return S.x[a] < S.x[b];
    if (S.y[a] != S.y[b]) return S.y[a] < S.y[b];
    return S.gid[a] < S.gid[b];
}

__device__ __forceinline__ void fin_consider(unsigned long long& kb, uint16_t& lb, unsigned long long k,
                                             uint16_t l, const FinSmem& S) {
    if (k < kb || (k == kb && fin_tie_better(l, lb, S))) {
        kb = k;
        lb = l;
    }
}

__device__ __forceinline__ void fin_warp_best(unsigned long long& k, uint16_t& l, const FinSmem& S) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const unsigned long long ok = __shfl_xor_sync(kFull, k, s);
        const uint16_t ol = uint16_t(__shfl_xor_sync(kFull, uint32_t(l), s));
        fin_consider(k, l, ok, ol, S);
    }
}

// one warp: segments f = gw, gw + nw, ... of the front (warp) list
__device__ __forceinline__ void finisher_warp_body(FinSmem& S, uint32_t gw, uint32_t nw, const FinRec* fins,
                                                   const LevelInfo* info, const double* __restrict__ ix,
                                                   const double* __restrict__ iy,
                                                   const uint32_t* __restrict__ iid, uint32_t* chain,
                                                   uint32_t* fin_count_out) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    const uint32_t nfin = info->nfin;
    for (uint32_t f = gw; f < nfin; f += nw) {
        const FinRec rec = fins[f];
        const uint32_t m = rec.c.m;
        VQB_CHECK(m >= 2 && m <= kFinSmall, 30, m, f);
        for (uint32_t i = lane; i < m; i += 32) {
            S.x[i] = ix[rec.c.begin + i];
            S.y[i] = iy[rec.c.begin + i];
            S.gid[i] = iid[rec.c.begin + i];
            S.work[0][i] = uint16_t(i);
        }
        const uint16_t P0 = uint16_t(m), Q0 = uint16_t(m + 1), R0 = uint16_t(m + 2);
        if (lane == 0) {
            S.x[P0] = rec.c.px; S.y[P0] = rec.c.py; S.gid[P0] = 0xffffffffu;
            S.x[Q0] = rec.c.qx; S.y[Q0] = rec.c.qy; S.gid[Q0] = 0xffffffffu;
            S.x[R0] = rec.c.rx; S.y[R0] = rec.c.ry; S.gid[R0] = rec.c.r_idx;
            FinFrame& fr = S.stack[0];
            fr.lo = 0; fr.hi = uint16_t(m); fr.p = P0; fr.r = R0; fr.q = Q0;
            fr.buf = 0; fr.phase = 0; fr.rcnt = 0; fr.rR = 0;
        }
        __syncwarp();
        int depth = 1;
        uint32_t emitted = 0;
        const uint64_t cbase = rec.chain_base;
        uint32_t guard = 0;
        while (depth > 0) {
            if (++guard > 8 * kFinSmall + 64) {  // at most ~3 visits per node
                if (lane == 0) g_vqb_fault = 2u;
                break;
            }
            const FinFrame fr = S.stack[depth - 1];
            if (fr.phase == 0) {
                // partition the node's points against (p->r), (r->q) with the
                // fused farthest search, in the reference's exact predicates
                const double px = S.x[fr.p], py = S.y[fr.p];
                const double rx = S.x[fr.r], ry = S.y[fr.r];
                const double qx = S.x[fr.q], qy = S.y[fr.q];
                const double adx = dsub(rx, px), ady = dsub(ry, py);
                const double bdx = dsub(qx, rx), bdy = dsub(qy, ry);
                const int src = fr.buf, dst = fr.buf ^ 1;
                uint32_t nL = 0, nR = 0;
                unsigned long long kL = kNoKey, kR = kNoKey;
                uint16_t lL = kNoLid, lR = kNoLid;
                for (uint32_t b0 = fr.lo; b0 < fr.hi; b0 += 32) {
                    const uint32_t i = b0 + lane;
                    const bool v = i < fr.hi;
                    const uint16_t id = v ? S.work[src][i] : 0;
                    const double u = S.x[id], w = S.y[id];
                    const double A = dsub(px, u), B = dsub(py, w);
                    const double E = dsub(rx, u), F = dsub(ry, w);
                    const double Cc = dsub(qx, u), D = dsub(qy, w);
                    const bool la = v && left_diff(A, B, E, F);
                    const bool lb = v && !la && left_diff(E, F, Cc, D);
                    const unsigned ba = __ballot_sync(kFull, la);
                    const unsigned bb = __ballot_sync(kFull, lb);
                    if (la) {
                        S.work[dst][fr.lo + nL + __popc(ba & lt)] = id;
                        fin_consider(kL, lL, key_of(lat_off(adx, ady, u, w)), id, S);
                    }
                    if (lb) {
                        S.work[dst][fr.hi - 1 - nR - __popc(bb & lt)] = id;
                        fin_consider(kR, lR, key_of(lat_off(bdx, bdy, u, w)), id, S);
                    }
                    nL += __popc(ba);
                    nR += __popc(bb);
                }
                if (nL) fin_warp_best(kL, lL, S);
                if (nR) fin_warp_best(kR, lR, S);
                __syncwarp();
                // a one-point child is its own chain: emit it in place instead
                // of visiting it (hull.cpp:83, m <= 1 returns m)
                if (nL == 1) {
                    if (lane == 0) chain[cbase + emitted] = S.gid[lL];
                    ++emitted;
                }
                if (lane == 0) {
                    FinFrame& cur = S.stack[depth - 1];
                    cur.phase = 1;
                    cur.rcnt = uint16_t(nR);
                    cur.rR = nR ? lR : 0;
                    if (nL >= 2) {
                        FinFrame& ch = S.stack[depth];
                        ch.lo = fr.lo; ch.hi = uint16_t(fr.lo + nL);
                        ch.p = fr.p; ch.r = lL; ch.q = fr.r;
                        ch.buf = uint8_t(dst); ch.phase = 0; ch.rcnt = 0; ch.rR = 0;
                    }
                }
                __syncwarp();
                if (nL >= 2) ++depth;
            } else if (fr.phase == 1) {
                // chain(L) is out: emit r, then the right child
                if (lane == 0) {
                    VQB_CHECK(emitted < m, 31, emitted, m);
                    chain[cbase + emitted] = S.gid[fr.r];
                    if (fr.rcnt == 1) chain[cbase + emitted + 1] = S.gid[fr.rR];
                    FinFrame& cur = S.stack[depth - 1];
                    if (fr.rcnt >= 2) {
                        // tail call: the frame becomes its right child
                        cur.lo = uint16_t(fr.hi - fr.rcnt);
                        cur.p = fr.r; cur.r = fr.rR;  // q unchanged
                        cur.buf = uint8_t(fr.buf ^ 1); cur.phase = 0;
                        cur.rcnt = 0; cur.rR = 0;
                    } else {
                        cur.phase = 2;
                    }
                }
                emitted += 1 + (fr.rcnt == 1);
                __syncwarp();
            } else {
                --depth;  // the parent resumes at phase 1 (its left subtree is done)
            }
        }
        if (lane == 0) fin_count_out[f] = emitted;
        __syncwarp();
    }
}

// ===========================================================================
// K3'' CTA finisher: one CTA solves the whole subtree of a segment of
// kFinSmall < m <= CAP points in shared memory, LEVEL-SYNCHRONOUSLY: every
// node of the current depth is partitioned in the same pass (the reference's
// chain_recursive, hull.cpp:78-115, visited breadth-first), so the serial
// chain is the tree depth, not the node count (a warp walking the nodes one
// by one is latency-bound when every point is a hull vertex).  Points never
// move: each carries its node id, which becomes its child's id, then the
// child's next-depth node id.  Per depth:
//   (1) every live point is classified against its node's (p->r), (r->q)
//       with the reference's exact predicates (left_diff, kernels.hpp:28-30;
//       mask_b &= ~mask_a, :91) and its farthest key (the canonical order of
//       kernels.hpp:41-45 as an order-preserving u64) stays in a register; the
//       child's point count (warp-aggregated) and minimal key (shared atomic,
//       warp-reduced first when the whole warp shares one child — the top of
//       the subtree) are accumulated;
//   (2) the points holding their child's minimal key register as its apex; an
//       exact tie (real on circle-like inputs: ~2 children per segment) lists
//       the extra candidates, resolved by smaller (x, y), then smaller index
//       (first occurrence) on one thread;
//   (3) children with >= 2 points become the next depth's nodes (block scan),
//       one-point children are leaves (hull.cpp:83); the subtree's links;
//   (4) fresh accumulators for the next depth.
// Finally subtree sizes bottom-up and chain positions top-down give
// chain(L) ++ [r] ++ chain(R) (assemble_chain, hull.cpp:59-73).
// (An earlier version moved every point to its child's range each depth and
// recomputed the keys: ~2x the instructions; a one-warp-per-segment variant
// was latency-bound: profiles/r02_finisher_warp_bfs.md.)
// ===========================================================================
// diagnostics (VQHULL_FIN_TRACE, build with -DVQB_STAMPS): block 0's
// CTA-finisher per-depth timestamps
__device__ unsigned long long g_ftrace[64];
__device__ uint32_t g_ftrace_on;

constexpr int kFcThreads = 256;
constexpr uint16_t kDead = 0xffffu;
constexpr uint16_t kLinkEmpty = 0, kLinkLeaf = 0x4000, kLinkNode = 0x8000;  // kind | value
constexpr uint32_t kFcNoChild = 0xffffffffu;

// shared memory of the CTA finisher for segments of at most CAP points
// (kFinMax for the host-driven finisher kernel, kTailFinMax inside KT)
template <int CAP>
struct FinCtaSmemT {
    static constexpr int kCap = CAP;
    static constexpr int kNodes = CAP / 2;  // nodes of one depth hold >= 2 points each
    double x[CAP + 3];
    double y[CAP + 3];
    uint32_t gid[CAP + 3];
    uint32_t ccnt[CAP];             // per child: points | candidates << 16
    uint16_t pnode[CAP];            // per point: child id of the last depth (kDead: done)
    uint16_t np[2][kNodes], nr[2][kNodes], nq[2][kNodes], ntree[2][kNodes];
    uint16_t ccand[CAP];            // per child: its apex
    uint16_t cmap[CAP];             // per child: next-depth node id (kDead: none)
    uint16_t tlist[CAP];            // extra candidates of tied children
    uint16_t tapex[CAP + 1], tleft[CAP + 1], tright[CAP + 1];
    uint16_t lvl_start[CAP + 2];
    union {
        unsigned long long ckey[CAP];  // per child: minimal key (during the BFS)
        struct {
            uint16_t tsize[CAP + 1];
            uint16_t tstart[CAP + 1];
        } t;                           // subtree sizes / chain positions (emission)
    } u;
    uint32_t wsum[kFcThreads / 32];
    uint32_t ntie;
    uint32_t nnext;
};
using FinCtaSmem = FinCtaSmemT<int(kFinMax)>;

template <class SM>
__device__ __forceinline__ uint32_t fc_link_size(const SM& S, uint16_t l) {
    return (l & kLinkNode) ? S.u.t.tsize[l & 0x3fff] : ((l & kLinkLeaf) ? 1u : 0u);
}

template <int CAP>
__device__ __forceinline__ void finisher_cta_body(FinCtaSmemT<CAP>& S, const FinRec* fins, const LevelInfo* info,
                                                  uint32_t fin_cap, const double* __restrict__ ix,
                                                  const double* __restrict__ iy,
                                                  const uint32_t* __restrict__ iid, uint32_t* chain,
                                                  uint32_t* fin_count) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int kFcItems = (CAP + kFcThreads - 1) / kFcThreads;  // points per thread
    const uint32_t nfin2 = info->nfin2;
    for (uint32_t f = blockIdx.x; f < nfin2; f += gridDim.x) {
        const uint32_t fi = fin_cap - 1u - f;
        const FinRec rec = fins[fi];
        const uint32_t m = rec.c.m;
        VQB_CHECK(m > kFinSmall && m <= uint32_t(CAP), 32, m, f);
        const uint16_t P0 = uint16_t(m), Q0 = uint16_t(m + 1), R0 = uint16_t(m + 2);
        for (uint32_t i = tid; i < m; i += kFcThreads) {
            S.x[i] = ix[rec.c.begin + i];
            S.y[i] = iy[rec.c.begin + i];
            S.gid[i] = iid[rec.c.begin + i];
        }
        if (tid == 0) {
            S.x[P0] = rec.c.px; S.y[P0] = rec.c.py; S.gid[P0] = 0xffffffffu;
            S.x[Q0] = rec.c.qx; S.y[Q0] = rec.c.qy; S.gid[Q0] = 0xffffffffu;
            S.x[R0] = rec.c.rx; S.y[R0] = rec.c.ry; S.gid[R0] = rec.c.r_idx;
            S.np[0][0] = P0; S.nr[0][0] = R0; S.nq[0][0] = Q0; S.ntree[0][0] = 0;
            S.tapex[0] = R0; S.tleft[0] = kLinkEmpty; S.tright[0] = kLinkEmpty;
            S.lvl_start[0] = 0; S.lvl_start[1] = 1;
            S.ntie = 0;
            S.cmap[0] = 0;  // depth 0: every point's "child" 0 maps to node 0
        }
        if (tid < 2) {
            S.u.ckey[tid] = kNoKey;
            S.ccnt[tid] = 0;
        }
        __syncthreads();
        uint32_t nnodes = 1, ntree = 1;
        int cur = 0, depth = 0;
        VQB_STAMP(const bool ftr = g_ftrace_on && blockIdx.x == 0 && tid == 0;
                  if (ftr) { g_ftrace[0] = m; g_ftrace[1] = gtimer_ns(); })
        while (nnodes > 0) {
            VQB_STAMP(if (ftr && depth < 38) g_ftrace[2 + depth] = gtimer_ns();)
            if (depth > CAP + 2) {  // every depth consumes >= 1 apex
                if (tid == 0) g_vqb_fault = 5u;
                break;
            }
            const int nxt = cur ^ 1;
            // (1) classify in place; child counts and minimal keys
            uint32_t chv[kFcItems];
            unsigned long long keyv[kFcItems];
#pragma unroll
            for (int k = 0; k < kFcItems; ++k) {
                const uint32_t i = uint32_t(k) * kFcThreads + tid;
                chv[k] = kFcNoChild;
                keyv[k] = kNoKey;
                if (i >= m) continue;
                const uint16_t pc = depth == 0 ? uint16_t(0) : S.pnode[i];
                const uint16_t c = pc == kDead ? kDead : S.cmap[pc];
                if (c == kDead) {
                    if (depth > 0) S.pnode[i] = kDead;
                    continue;
                }
                const uint16_t p = S.np[cur][c], r = S.nr[cur][c], q = S.nq[cur][c];
                const double u = S.x[i], w = S.y[i];
                const double px = S.x[p], py = S.y[p], rx = S.x[r], ry = S.y[r];
                const double qx = S.x[q], qy = S.y[q];
                const double A = dsub(px, u), B = dsub(py, w);
                const double E = dsub(rx, u), F = dsub(ry, w);
                const double Cc = dsub(qx, u), D = dsub(qy, w);
                const bool la = left_diff(A, B, E, F);
                const bool lb = !la && left_diff(E, F, Cc, D);
                if (la || lb) {
                    const uint32_t ch = 2u * c + (lb ? 1u : 0u);
                    const double fx = lb ? dsub(qx, rx) : dsub(rx, px);
                    const double fy = lb ? dsub(qy, ry) : dsub(ry, py);
                    const unsigned long long key = key_of(lat_off(fx, fy, u, w));
                    chv[k] = ch;
                    keyv[k] = key;
                    S.pnode[i] = uint16_t(ch);
                } else {
                    S.pnode[i] = kDead;
                }
            }
#pragma unroll
            for (int k = 0; k < kFcItems; ++k) {
                const uint32_t ch = chv[k];
                const unsigned grp = __match_any_sync(kFull, ch);
                if (grp == kFull) {  // the whole warp in one child (or none)
                    unsigned long long key = keyv[k];
#pragma unroll
                    for (int s = 16; s > 0; s >>= 1) {
                        const unsigned long long o = __shfl_xor_sync(kFull, key, s);
                        key = o < key ? o : key;
                    }
                    if (ch != kFcNoChild && lane == 0) {
                        atomicAdd(&S.ccnt[ch], 32u);
                        if (key < S.u.ckey[ch]) atomicMin(&S.u.ckey[ch], key);
                    }
                } else if (ch != kFcNoChild) {
                    if (lane == __ffs(grp) - 1) atomicAdd(&S.ccnt[ch], uint32_t(__popc(grp)));
                    if (keyv[k] < S.u.ckey[ch]) atomicMin(&S.u.ckey[ch], keyv[k]);
                }
            }
            __syncthreads();
            VQB_STAMP(if (ftr && depth == 0) g_ftrace[40] = gtimer_ns();)
            // (2) apexes: the points holding their child's minimal key
#pragma unroll
            for (int k = 0; k < kFcItems; ++k) {
                const uint32_t ch = chv[k];
                if (ch == kFcNoChild || keyv[k] != S.u.ckey[ch]) continue;
                const uint32_t i = uint32_t(k) * kFcThreads + tid;
                if ((atomicAdd(&S.ccnt[ch], 0x10000u) >> 16) == 0) S.ccand[ch] = uint16_t(i);
                else S.tlist[atomicAdd(&S.ntie, 1u)] = uint16_t(i);
            }
            __syncthreads();
            VQB_STAMP(if (ftr && depth == 0) g_ftrace[41] = gtimer_ns();)
            if (S.ntie) {  // exact offset ties: smaller (x, y), then first index
                if (tid == 0) {
                    const uint32_t nt = S.ntie;
                    for (uint32_t t = 0; t < nt; ++t) {
                        const uint16_t i = S.tlist[t];
                        const uint16_t ch = S.pnode[i];
                        const uint16_t b = S.ccand[ch];
                        const bool better = S.x[i] != S.x[b] ? S.x[i] < S.x[b]
                                          : (S.y[i] != S.y[b] ? S.y[i] < S.y[b] : S.gid[i] < S.gid[b]);
                        if (better) S.ccand[ch] = i;
                    }
                    S.ntie = 0;
                }
                __syncthreads();
            }
            // (3) children -> next depth's nodes (block scan over "internal"), links, leaves
            const uint32_t nch = 2 * nnodes;
            uint32_t flags = 0, local = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t ch = 4u * tid + k;
                const bool in = ch < nch && (S.ccnt[ch] & 0xffffu) >= 2;
                flags |= uint32_t(in) << k;
                local += in;
            }
            uint32_t incl = local;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(kFull, incl, d);
                if (lane >= d) incl += o;
            }
            if (lane == 31) S.wsum[warp] = incl;
            __syncthreads();
            VQB_STAMP(if (ftr && depth == 0) g_ftrace[42] = gtimer_ns();)
            uint32_t base = 0;
            for (int w2 = 0; w2 < warp; ++w2) base += S.wsum[w2];
            uint32_t id = base + incl - local;  // first next-depth id of this thread's children
            if (tid == kFcThreads - 1) S.nnext = base + incl;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t ch = 4u * tid + k;
                if (ch >= nch) break;
                const int c = int(ch >> 1), s = int(ch & 1);
                const uint32_t cnt = S.ccnt[ch] & 0xffffu;
                const uint16_t t = S.ntree[cur][c];
                uint16_t link = kLinkEmpty;
                uint16_t map = kDead;
                if (cnt == 1) {
                    link = uint16_t(kLinkLeaf | S.ccand[ch]);
                } else if (cnt >= 2) {
                    const uint32_t nid = id++;
                    const uint16_t tnew = uint16_t(ntree + nid);
                    link = uint16_t(kLinkNode | tnew);
                    S.np[nxt][nid] = s ? S.nr[cur][c] : S.np[cur][c];
                    S.nq[nxt][nid] = s ? S.nq[cur][c] : S.nr[cur][c];
                    S.nr[nxt][nid] = S.ccand[ch];
                    S.ntree[nxt][nid] = tnew;
                    S.tapex[tnew] = S.ccand[ch];
                    S.tleft[tnew] = kLinkEmpty;
                    S.tright[tnew] = kLinkEmpty;
                    map = uint16_t(nid);
                }
                S.cmap[ch] = map;
                if (s) S.tright[t] = link; else S.tleft[t] = link;
            }
            __syncthreads();
            VQB_STAMP(if (ftr && depth == 0) g_ftrace[43] = gtimer_ns();)
            const uint32_t nn = S.nnext;
            // (4) fresh accumulators for the next depth's children (points
            // read their next node id through cmap in the next phase 1)
            for (uint32_t ch = tid; ch < 2 * nn; ch += kFcThreads) {
                S.u.ckey[ch] = kNoKey;
                S.ccnt[ch] = 0;
            }
            ntree += nn;
            ++depth;
            if (tid == 0) S.lvl_start[depth + 1] = uint16_t(ntree);
            nnodes = nn;
            cur = nxt;
            __syncthreads();
        }
        VQB_STAMP(if (ftr) { g_ftrace[62] = depth; g_ftrace[63] = gtimer_ns(); })
        // subtree sizes bottom-up, then chain positions top-down
        for (int d = depth - 1; d >= 0; --d) {
            for (uint32_t t = S.lvl_start[d] + tid; t < S.lvl_start[d + 1]; t += kFcThreads)
                S.u.t.tsize[t] = uint16_t(fc_link_size(S, S.tleft[t]) + 1u + fc_link_size(S, S.tright[t]));
            __syncthreads();
        }
        const uint64_t cb = rec.chain_base;
        if (tid == 0) S.u.t.tstart[0] = 0;
        __syncthreads();
        for (int d = 0; d < depth; ++d) {
            for (uint32_t t = S.lvl_start[d] + tid; t < S.lvl_start[d + 1]; t += kFcThreads) {
                const uint32_t s0 = S.u.t.tstart[t];
                const uint16_t L = S.tleft[t], R = S.tright[t];
                const uint32_t ap = s0 + fc_link_size(S, L);
                chain[cb + ap] = S.gid[S.tapex[t]];
                if (L & kLinkLeaf) chain[cb + s0] = S.gid[L & 0x3fff];
                else if (L & kLinkNode) S.u.t.tstart[L & 0x3fff] = uint16_t(s0);
                if (R & kLinkLeaf) chain[cb + ap + 1] = S.gid[R & 0x3fff];
                else if (R & kLinkNode) S.u.t.tstart[R & 0x3fff] = uint16_t(ap + 1);
            }
            __syncthreads();
        }
        if (tid == 0) fin_count[fi] = S.u.t.tsize[0];
        __syncthreads();
    }
}

// Both finishers of a level in one launch (kFcThreads per CTA): first the
// CTA segments (one CTA each), then the warp segments (one warp each), in the
// same shared memory.
template <int CAP>
union FinAllSmemT {
    FinCtaSmemT<CAP> cta;
    FinSmem warp[kFcThreads / 32];
};
using FinAllSmem = FinAllSmemT<int(kFinMax)>;

template <int CAP>
__device__ __forceinline__ void finisher_all_body(FinAllSmemT<CAP>& U, const FinRec* fins, const LevelInfo* info,
                                                  uint32_t fin_cap, const double* __restrict__ ix,
                                                  const double* __restrict__ iy,
                                                  const uint32_t* __restrict__ iid, uint32_t* chain,
                                                  uint32_t* fin_count) {
    finisher_cta_body(U.cta, fins, info, fin_cap, ix, iy, iid, chain, fin_count);
    __syncthreads();
    const uint32_t wpb = kFcThreads / 32;
    finisher_warp_body(U.warp[threadIdx.x >> 5], blockIdx.x * wpb + (threadIdx.x >> 5), gridDim.x * wpb, fins,
                       info, ix, iy, iid, chain, fin_count);
}

__global__ void __launch_bounds__(kFcThreads) finisher_all_kernel(const FinRec* fins, const LevelInfo* info,
                                                                  uint32_t fin_cap,
                                                                  const double* __restrict__ ix,
                                                                  const double* __restrict__ iy,
                                                                  const uint32_t* __restrict__ iid,
                                                                  uint32_t* chain, uint32_t* fin_count) {
    VQB_PDL();
    extern __shared__ __align__(16) unsigned char fc_dsm[];
    FinAllSmem& U = *reinterpret_cast<FinAllSmem*>(fc_dsm);
    finisher_all_body(U, fins, info, fin_cap, ix, iy, iid, chain, fin_count);
}

// ===========================================================================
// K4: in-order emission.  Bottom-up chain sizes, then top-down starts;
// every node writes its apex between its children's chains.
// Output = [p] ++ chain(S1) ++ [q if q != p] ++ chain(S2)  (hull.cpp:259-266)
// ===========================================================================
__global__ void size_kernel(uint32_t nslots, const uint8_t* kind, const uint32_t* link,
                            const uint32_t* fin_count, const uint32_t* child_size,
                            uint32_t* size) {
    VQB_PDL();
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < nslots;
         s += gridDim.x * blockDim.x) {
        const uint8_t k = kind[s];
        uint32_t v = 0;
        if (k == kLeaf) v = 1;
        else if (k == kFin) v = fin_count[link[s]];
        else if (k == kInternal) v = 1 + child_size[2 * link[s]] + child_size[2 * link[s] + 1];
        size[s] = v;
    }
}

__global__ void emit_kernel(uint32_t nslots, const uint8_t* kind, const uint32_t* link,
                            const ChildRec* slots, const FinRec* fins, const uint32_t* fin_count,
                            const uint32_t* chain, const uint32_t* start,
                            const uint32_t* child_size, uint32_t* child_start, uint32_t* out) {
    VQB_PDL();
    // one warp per slot: a finisher slot copies its whole chain (up to
    // kFinMax entries) with the warp's 32 lanes
    const int lane = threadIdx.x & 31;
    const uint32_t wpb = blockDim.x >> 5;
    for (uint32_t s = blockIdx.x * wpb + (threadIdx.x >> 5); s < nslots; s += gridDim.x * wpb) {
        const uint8_t k = kind[s];
        const uint32_t st = start[s];
        if (k == kLeaf) {
            if (lane == 0) out[st] = slots[s].r_idx;
        } else if (k == kInternal) {
            if (lane == 0) {
                const uint32_t L = link[s];
                const uint32_t sl = child_size[2 * L];
                out[st + sl] = slots[s].r_idx;
                child_start[2 * L] = st;
                child_start[2 * L + 1] = st + sl + 1;
            }
        } else if (k == kFin) {
            const uint32_t f = link[s];
            const uint32_t c = fin_count[f];
            const uint64_t b = fins[f].chain_base;
            for (uint32_t i = lane; i < c; i += 32) out[st + i] = chain[b + i];
        }
    }
}

// Whole emission of a small tree (few slots) in ONE CTA: bottom-up sizes,
// the root frame, top-down starts and writes — the same steps as
// size_kernel / poly_frame_kernel / emit_kernel, without one launch each.
// For a large tree the same kernel does its top levels (the many levels of
// few slots each), between the size launches and the emit launches of the
// levels below (E.below_size / E.below_start).
__global__ void __launch_bounds__(1024) emit_small_kernel(EmitAll E, const RootInfo* root, const uint32_t* chain,
                                                          uint32_t* out, uint32_t* h_out) {
    VQB_PDL();
    const int lane = threadIdx.x & 31;
    for (int l = E.nlev - 1; l >= 0; --l) {
        const EmitLevel& L = E.lv[l];
        const uint32_t* child_size = l + 1 < E.nlev ? E.lv[l + 1].size : E.below_size;
        for (uint32_t s = threadIdx.x; s < L.nslots; s += blockDim.x) {
            const uint8_t k = L.kind[s];
            uint32_t v = 0;
            if (k == kLeaf) v = 1;
            else if (k == kFin) v = L.fin_count[L.link[s]];
            else if (k == kInternal) v = 1 + child_size[2 * L.link[s]] + child_size[2 * L.link[s] + 1];
            L.size[s] = v;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const RootPoly& P = root->poly;
        uint32_t pos = 0;
        for (uint32_t j = 0; j < P.nv; ++j) {
            const bool same_prev = j > 0 && P.ex[j] == P.ex[j - 1] && P.ey[j] == P.ey[j - 1];
            const bool same_first = j > 0 && P.ex[j] == P.ex[0] && P.ey[j] == P.ey[0];
            if (!same_prev && !same_first) out[pos++] = P.eidx[j];
            E.lv[0].start[j] = pos;
            pos += E.lv[0].size[j];
        }
        *h_out = pos;
    }
    __syncthreads();
    const uint32_t wpb = blockDim.x >> 5;
    for (int l = 0; l < E.nlev; ++l) {
        const EmitLevel& L = E.lv[l];
        const uint32_t* csize = l + 1 < E.nlev ? E.lv[l + 1].size : E.below_size;
        uint32_t* cstart = l + 1 < E.nlev ? E.lv[l + 1].start : E.below_start;
        const bool has_child = cstart != nullptr;
        for (uint32_t s = threadIdx.x >> 5; s < L.nslots; s += wpb) {  // one warp per slot
            const uint8_t k = L.kind[s];
            const uint32_t st = L.start[s];
            if (k == kLeaf) {
                if (lane == 0) out[st] = L.slots[s].r_idx;
            } else if (k == kInternal && has_child) {
                if (lane == 0) {
                    const uint32_t c = L.link[s];
                    const uint32_t sl = csize[2 * c];
                    out[st + sl] = L.slots[s].r_idx;
                    cstart[2 * c] = st;
                    cstart[2 * c + 1] = st + sl + 1;
                }
            } else if (k == kFin) {
                const uint32_t f = L.link[s];
                const uint32_t c = L.fin_count[f];
                const uint64_t b = L.fins[f].chain_base;
                for (uint32_t i = lane; i < c; i += 32) out[st + i] = chain[b + i];
            }
        }
        __syncthreads();
    }
}

// Reference mode: the root polygon is (p, r1, q, r2) of the reference's
// first two recursion levels (hull.cpp:228-235); an empty side contributes
// no vertex (its r is replaced by the next vertex, emitted once).  Also
// re-arms the fast-mode side counters of the reference-mode root partition.
__global__ void legacy_poly_kernel(RootInfo* root, unsigned long long* side_ctr) {
    VQB_PDL();
    if (threadIdx.x != 0) return;
    side_ctr[0] = side_ctr[1] = 0ull;
    RootInfo& R = *root;
    RootPoly& P = R.poly;
    const bool h1 = R.cnt1 > 0, h2 = R.cnt2 > 0;
    P.ex[0] = R.px; P.ey[0] = R.py; P.eidx[0] = R.p_idx;
    P.ex[1] = h1 ? R.r1.x : R.qx; P.ey[1] = h1 ? R.r1.y : R.qy; P.eidx[1] = h1 ? R.r1.idx : R.q_idx;
    P.ex[2] = R.qx; P.ey[2] = R.qy; P.eidx[2] = R.q_idx;
    P.ex[3] = h2 ? R.r2.x : R.px; P.ey[3] = h2 ? R.r2.y : R.py; P.eidx[3] = h2 ? R.r2.idx : R.p_idx;
    P.nv = 4;
    P.filter = 0;
}

// Output frame: V_0 chain(slot 0) V_1 chain(slot 1) ... with repeated
// vertices written once (hull.cpp:259-266 for the reference-mode polygon:
// [p] chain(S1) [q if q != p] chain(S2), chain(S) = chain(S_1) [r] chain(S_2)).
__global__ void poly_frame_kernel(const RootInfo* root, const uint32_t* size2, uint32_t* start2,
                                  uint32_t* out, uint32_t* h_out) {
    VQB_PDL();
    if (threadIdx.x != 0) return;
    const RootPoly& P = root->poly;
    uint32_t pos = 0;
    for (uint32_t j = 0; j < P.nv; ++j) {
        const bool same_prev = j > 0 && P.ex[j] == P.ex[j - 1] && P.ey[j] == P.ey[j - 1];
        const bool same_first = j > 0 && P.ex[j] == P.ex[0] && P.ey[j] == P.ey[0];
        if (!same_prev && !same_first) out[pos++] = P.eidx[j];
        start2[j] = pos;
        pos += size2[j];
    }
    *h_out = pos;
}

// ===========================================================================
// K0: a whole hull of n <= kFinMax points in ONE CTA (tiny inputs, the
// candidates of a sharded hull): find_extremes (geometry.cpp:7-36) as a block
// reduction, then the bootstrap triangle (p, q, p) (hull.cpp:228-235) as one
// finisher segment — the finisher's chain of that segment is chain(S1) [q]
// chain(S2) — and the output [p] chain (hull.cpp:259-266).  No filter, no
// levels: one launch instead of sample + filter + recursion kernel.
// ===========================================================================

__global__ void __launch_bounds__(kFcThreads) tiny_hull_kernel(const __grid_constant__ TinyArgs A) {
    VQB_PDL();
    extern __shared__ __align__(16) unsigned char tn_dsm[];
    FinAllSmem& U = *reinterpret_cast<FinAllSmem*>(tn_dsm);
    __shared__ ExtKey s_lo[kFcThreads / 32], s_hi[kFcThreads / 32];
    __shared__ uint32_t s_bad[kFcThreads / 32];
    __shared__ uint32_t s_go;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t n = A.n;
    ExtKey lo{0.0, 0.0, kNoIdx, 0u}, hi{0.0, 0.0, kNoIdx, 0u};
    uint32_t bad = 0;
    for (uint32_t i = tid; i < n; i += kFcThreads) {
        const double x = A.xs[i], y = A.ys[i];
        A.iid[i] = i;
        bad |= uint32_t(nonfinite_bits(x) | nonfinite_bits(y));
        const ExtKey c{x, y, i, 1u};
        if (lo_better(c, lo)) lo = c;
        if (hi_better(c, hi)) hi = c;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const ExtKey a = shfl_key(lo, s);
        if (lo_better(a, lo)) lo = a;
        const ExtKey b = shfl_key(hi, s);
        if (hi_better(b, hi)) hi = b;
        bad |= __shfl_xor_sync(kFull, bad, s);
    }
    if (lane == 0) {
        s_lo[warp] = lo;
        s_hi[warp] = hi;
        s_bad[warp] = bad;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < kFcThreads / 32; ++w) {
            if (lo_better(s_lo[w], lo)) lo = s_lo[w];
            if (hi_better(s_hi[w], hi)) hi = s_hi[w];
            bad |= s_bad[w];
        }
        A.report[1] = bad;
        A.report[2] = 0u;
        s_go = 0u;
        if (!bad && lo.valid) {
            A.out[0] = lo.idx;
            if (lo.x == hi.x && lo.y == hi.y) {
                A.report[0] = 1u;  // all points equal: [p]
            } else {
                FinRec f;
                f.c.px = lo.x; f.c.py = lo.y;
                f.c.rx = hi.x; f.c.ry = hi.y;  // apex q
                f.c.qx = lo.x; f.c.qy = lo.y;
                f.c.begin = 0;
                f.c.m = n;
                f.c.r_idx = hi.idx;
                f.chain_base = 0;
                f.slot = 0;
                f.pad = 0;
                *A.fin = f;
                LevelInfo li;
                li.nslots = 1; li.nseg = 0; li.ntiles = 0; li.out_total = 0;
                li.fin_total = n; li.nleaf = 0; li.fin_base = 0; li.pad = 0;
                li.nfin = n <= kFinSmall ? 1u : 0u;  // warp list (front) or CTA list (back, fin_cap 1)
                li.nfin2 = n <= kFinSmall ? 0u : 1u;
                *A.info = li;
                s_go = 1u;
            }
        } else {
            A.report[0] = 0u;
        }
        __threadfence_block();
    }
    __syncthreads();
    if (!s_go) return;
    finisher_all_body(U, A.fin, A.info, 1u, A.xs, A.ys, A.iid, A.chain, A.fin_count);
    __syncthreads();
    const uint32_t c = *reinterpret_cast<volatile uint32_t*>(A.fin_count);
    for (uint32_t i = tid; i < c; i += kFcThreads) A.out[1 + i] = A.chain[i];
    if (tid == 0) {
        A.report[0] = 1u + c;
        A.report[2] = *reinterpret_cast<volatile uint32_t*>(&g_vqb_fault);
    }
}

void launch_tiny(const TinyArgs& a, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tiny_hull_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FinAllSmem)));
        attr = true;
    }
    pdl_launch(tiny_hull_kernel, 1, kFcThreads, sizeof(FinAllSmem), st, a);
}

// ===========================================================================
// Host-side launchers (C++ linkage, used by driver.cu)
// ===========================================================================
void launch_extremes(const double* xs, const double* ys, uint64_t n, void* partials,
                     uint32_t* ticket, RootInfo* root, int grid, cudaStream_t st) {
    pdl_launch(extremes_kernel, grid, 256, 0, st, xs, ys, n, static_cast<ExtPartial*>(partials), ticket,
                                          root);
}

void launch_bootstrap(const double* xs, const double* ys, uint64_t n, void* partials,
                      uint32_t* ticket, RootInfo* root, int grid, cudaStream_t st) {
    pdl_launch(bootstrap_argmax_kernel, grid, 256, 0, st, xs, ys, n, static_cast<RootPartial*>(partials),
                                                  ticket, root);
}

void launch_poly_sample(const double* xs, const double* ys, uint64_t n, void* partials,
                        uint32_t* ticket, unsigned long long* keys, RootInfo* root,
                        unsigned long long* side_ctr, int grid, bool with_pq, cudaStream_t st) {
    pdl_launch(poly_sample_kernel, grid, 256, 0, st, xs, ys, n, static_cast<SamplePartial*>(partials), ticket,
               keys, root, side_ctr, int(with_pq), sample_mask(n));
}

void fin_trace(bool on) {
    const uint32_t v = on ? 1u : 0u;
    cudaMemcpyToSymbol(g_ftrace_on, &v, 4);
}
void print_fin_trace() {
    unsigned long long t[64];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(t, g_ftrace, sizeof t);
    if (!t[1]) return;
    fprintf(stderr, "[fin] m=%llu depth=%llu total %.2f us:", t[0], t[62], (t[63] - t[1]) * 1e-3);
    for (int d = 0; d < 38 && d < int(t[62]); ++d) fprintf(stderr, " %.2f", (t[2 + d] - t[1]) * 1e-3);
    fprintf(stderr, " | depth0 phases:");
    for (int k = 40; k < 44; ++k) fprintf(stderr, " %.2f", (t[k] - t[1]) * 1e-3);
    fputc('\n', stderr);
    const unsigned long long z[64] = {};
    cudaMemcpyToSymbol(g_ftrace, z, sizeof z);
}

// one run of 1024 points in (mask + 1) is sampled: the largest power of two
// that still leaves >= kSampleMin sample points
#ifndef VQB_SAMPLE_MIN
#define VQB_SAMPLE_MIN 1500000ull
#endif
constexpr uint64_t kSampleMin = VQB_SAMPLE_MIN;
uint32_t sample_mask(uint64_t n) {
    static const uint64_t smin = getenv("VQHULL_SAMPLE_MIN") ? uint64_t(atoll(getenv("VQHULL_SAMPLE_MIN"))) : kSampleMin;
    uint64_t k = 1;
    while (k < 1024 && n / (2 * k) >= smin) k *= 2;
    return uint32_t(k - 1);
}

void print_sample_trace() {
    unsigned long long t[8];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(t, g_strace, sizeof t);
    fprintf(stderr, "[sample] stream end %.2f  fold %.2f  reduce %.2f  finish %.2f | filter start %.2f end %.2f | tail start %.2f us\n",
            (t[1] - t[0]) * 1e-3, (t[2] - t[0]) * 1e-3, (t[3] - t[0]) * 1e-3, (t[4] - t[0]) * 1e-3,
            (double(t[5]) - double(t[0])) * 1e-3, (double(t[6]) - double(t[0])) * 1e-3,
            (double(t[7]) - double(t[0])) * 1e-3);
    const unsigned long long z[8] = {0, 0, 0, 0, 0, ~0ull, 0, 0};
    cudaMemcpyToSymbol(g_strace, z, sizeof z);
}

size_t partial_bytes(int grid) {
    size_t m = sizeof(RootPartial) > sizeof(ExtPartial) ? sizeof(RootPartial) : sizeof(ExtPartial);
    m = m > sizeof(PolyPartial) ? m : sizeof(PolyPartial);
    return size_t(grid) * m;
}

void launch_planner(const ChildRec* slots, uint32_t nslots, const LevelInfo* prev, uint32_t nslots_bound,
                    SegRec* segs, FinRec* fins, uint8_t* kind, uint32_t* link, LevelInfo* info,
                    uint32_t* flags, void* aggs, void* incs, uint32_t epoch, uint32_t* ctr,
                    uint32_t* seg_pcnt, uint32_t* seg_done, unsigned long long* seg_ctr,
                    int max_grid, cudaStream_t st, LevelInfo* next_info) {
    PlanArgs a;
    a.next_info = next_info;
    a.seg_pcnt = seg_pcnt;
    a.seg_done = seg_done;
    a.seg_ctr = seg_ctr;
    a.slots = slots; a.nslots = nslots; a.prev = prev; a.fin_cap = nslots_bound > 0 ? nslots_bound : 1;
    a.segs = segs; a.fins = fins; a.kind = kind; a.link = link; a.info = info;
    a.flags = flags; a.aggs = static_cast<PlanAgg*>(aggs); a.incs = static_cast<PlanAgg*>(incs);
    a.epoch = epoch; a.ctr = ctr;
    const uint32_t chunks = (nslots_bound + kPlanChunk - 1) / kPlanChunk;
    int grid = int(chunks < uint32_t(max_grid) ? chunks : uint32_t(max_grid));
    if (grid < 1) grid = 1;
    pdl_launch(planner_kernel, grid, kThreads, 0, st, a);
}

void launch_tilemap(const SegRec* segs, const LevelInfo* info, uint32_t* tile_seg,
                    uint32_t ntiles_hint, cudaStream_t st) {
    uint32_t g = (ntiles_hint + 255) / 256;
    if (g < 1) g = 1;
    if (g > 1184) g = 1184;
    pdl_launch(tilemap_kernel, g, 256, 0, st, segs, info, tile_seg);
}

void launch_finisher(const FinRec* fins, const LevelInfo* info, uint32_t fin_cap, const double* ix,
                     const double* iy, const uint32_t* iid, uint32_t* chain, uint32_t* fin_count,
                     uint32_t nfin_hint, int max_grid, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(finisher_all_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FinAllSmem)));
        attr = true;
    }
    uint32_t g = nfin_hint;
    if (g < 1) g = 1;
    if (g > uint32_t(max_grid)) g = uint32_t(max_grid);
    pdl_launch(finisher_all_kernel, g, kFcThreads, sizeof(FinAllSmem), st, fins, info, fin_cap, ix, iy, iid, chain,
               fin_count);
}

int occupancy_finisher() {
    int b = 0;
    cudaFuncSetAttribute(finisher_all_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FinAllSmem)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, finisher_all_kernel, kFcThreads, sizeof(FinAllSmem));
    return b;
}

void launch_size(uint32_t nslots, const uint8_t* kind, const uint32_t* link,
                 const uint32_t* fin_count, const uint32_t* child_size, uint32_t* size,
                 cudaStream_t st) {
    uint32_t g = (nslots + 255) / 256;
    if (g < 1) g = 1;
    if (g > 1184) g = 1184;
    pdl_launch(size_kernel, g, 256, 0, st, nslots, kind, link, fin_count, child_size, size);
}

void launch_emit(uint32_t nslots, const uint8_t* kind, const uint32_t* link,
                 const ChildRec* slots, const FinRec* fins, const uint32_t* fin_count,
                 const uint32_t* chain, const uint32_t* start, const uint32_t* child_size,
                 uint32_t* child_start, uint32_t* out, cudaStream_t st) {
    uint32_t g = (nslots + 7) / 8;  // 8 warps (slots) per block
    if (g < 1) g = 1;
    if (g > 2368) g = 2368;
    pdl_launch(emit_kernel, g, 256, 0, st, nslots, kind, link, slots, fins, fin_count, chain, start,
                                   child_size, child_start, out);
}

void launch_emit_small(const EmitAll& e, const RootInfo* root, const uint32_t* chain, uint32_t* out,
                       uint32_t* h_out, cudaStream_t st) {
    pdl_launch(emit_small_kernel, 1, 1024, 0, st, e, root, chain, out, h_out);
}

void launch_legacy_poly(RootInfo* root, unsigned long long* side_ctr, cudaStream_t st) {
    pdl_launch(legacy_poly_kernel, 1, 32, 0, st, root, side_ctr);
}

void launch_poly_frame(const RootInfo* root, const uint32_t* size2, uint32_t* start2, uint32_t* out,
                       uint32_t* h_out, cudaStream_t st) {
    pdl_launch(poly_frame_kernel, 1, 32, 0, st, root, size2, start2, out, h_out);
}

size_t plan_agg_bytes() { return sizeof(PlanAgg); }

int occupancy_extremes() {
    int a = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, extremes_kernel, 256, 0);
    return a;
}
int occupancy_bootstrap() {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, bootstrap_argmax_kernel, 256, 0);
    return b;
}
int occupancy_poly_sample() {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, poly_sample_kernel, 256, 0);
    return b;
}

}  // namespace vqb

namespace vqb {
uint32_t* fault_word_ptr() {
    void* p = nullptr;
    cudaGetSymbolAddress(&p, g_vqb_fault);
    return static_cast<uint32_t*>(p);
}

uint32_t read_and_clear_fault() {
    uint32_t v = 0;
    cudaMemcpyFromSymbol(&v, g_vqb_fault, sizeof v);
#ifdef VQB_DEBUG
    if (v) {
        unsigned long long d[4];
        cudaMemcpyFromSymbol(d, g_vqb_dbg, sizeof d);
        fprintf(stderr, "[vqb debug] fault %u: a0=%llu a1=%llu block=%llu thread=%llu\n", v, d[0], d[1], d[2], d[3]);
    }
#endif
    if (v) {
        const uint32_t z = 0;
        cudaMemcpyToSymbol(g_vqb_fault, &z, sizeof z);
    }
    return v;
}
void set_filter_inner(int mode) { cudaMemcpyToSymbol(g_inner_force, &mode, sizeof mode); }

}  // namespace vqb
