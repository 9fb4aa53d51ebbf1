// The partition kernels of the hot path (sm_100a):
//
//   K_F root_filter_tma        the default root: polygon filter over every point
//   KB' root_filtered_tma      one-pass octagon root (level 1 behind the filter)
//   KB  root_partition_kernel  hull levels 1+2 fused over the caller's input
//   K2  level_kernel / level_tma  every live segment of one recursion level
//
// Both are the reference's extract_blocks (extract_core.hpp:421-515): f64
// orientation test against two edges with mask_b &= ~mask_a (kernels.hpp:91),
// order-preserving two-sided compaction (S1 from the left end of the range,
// S2 from the right end), and the fused farthest-point search in the
// canonical order (kernels.hpp:36-45).
//
// GPU structure (co-resident persistent CTAs, static tile schedule t -> CTA
// t mod G, next tile prefetched into registers):
//   classify -> warp ballots -> block scan -> publish the tile's counts
//   -> stage survivors in smem (input order) -> per-class arg-max
//   -> decoupled look-back over self-validating 8-byte status words
//   -> coalesced stores of the staged survivors to their final positions.
// The arg-max does not ride the look-back: each CTA keeps a running best per
// segment and publishes it once per segment visit; the CTA that completes a
// segment's tile count reduces those few partials and emits the children.
#include <type_traits>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "hull_types.cuh"
#include "kernels.h"

namespace vqb {

// ---------------------------------------------------------------------------
// Look-back status words.  Every word is 8 bytes = {tag: epoch<<2 | state,
// count: 32 bits}, so each one validates itself under PTX's 8-byte
// single-copy atomicity; aggregate and inclusive values live in separate
// slots, so a reader can never combine a fresh flag with stale counts.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pub_pair(unsigned long long* p, uint32_t tag, uint32_t c0,
                                         uint32_t c1) {
    const unsigned long long w0 = (static_cast<unsigned long long>(tag) << 32) | c0;
    const unsigned long long w1 = (static_cast<unsigned long long>(tag) << 32) | c1;
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1)
                 : "memory");
}

__device__ __forceinline__ ulonglong2 ld_pair(const unsigned long long* p) {
    ulonglong2 v;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                 : "=l"(v.x), "=l"(v.y)
                 : "l"(p)
                 : "memory");
    return v;
}

__device__ __forceinline__ uint32_t tag_of(unsigned long long w) { return uint32_t(w >> 32); }

// Inclusive counts of a finished tile (both words carry the inclusive tag).
__device__ __forceinline__ uint2 inclusive_of(const Status* s, uint32_t epoch) {
    const ulonglong2 i = ld_pair(s->inc);
    VQB_CHECK(tag_of(i.x) == ((epoch << 2) | kStInc) && tag_of(i.y) == ((epoch << 2) | kStInc), 40,
              tag_of(i.x), epoch);
    (void)epoch;
    return make_uint2(uint32_t(i.x), uint32_t(i.y));
}

// A tile announces its own counts as early as possible — right after its
// block scan — so successors rarely wait: INC for the first tile of its
// segment (nothing precedes it), AGG otherwise.
__device__ __forceinline__ void publish_counts(Status* s, bool first, uint32_t c0, uint32_t c1,
                                               uint32_t epoch) {
    if (first) pub_pair(s->inc, (epoch << 2) | kStInc, c0, c1);
    else pub_pair(s->agg, (epoch << 2) | kStAgg, c0, c1);
}

// Decoupled look-back over status words st[t * stride + side]; run by one
// full warp after the tile's own counts were published.  Returns the
// exclusive prefix (c0, c1) of `tile` inside the segment whose first tile is
// `first` and publishes the tile's inclusive counts.
__device__ uint2 lookback16(uint32_t tile, uint32_t first, uint32_t c0, uint32_t c1, Status* st,
                            uint32_t stride, uint32_t side, uint32_t epoch) {
    if (tile == first) return make_uint2(0u, 0u);
    const int lane = threadIdx.x & 31;
    const uint32_t tagA = (epoch << 2) | kStAgg, tagI = (epoch << 2) | kStInc;
    uint32_t acc0 = 0, acc1 = 0;
    int64_t pred = int64_t(tile) - 1;
    while (true) {
        const int64_t t = pred - lane;
        const bool in_seg = t >= int64_t(first);
        uint32_t state = 0, v0 = 0, v1 = 0;
        if (in_seg) {
            const Status* s = &st[uint64_t(t) * stride + side];
            uint32_t spins = 0;
            while (true) {
                const ulonglong2 i = ld_pair(s->inc);
                const ulonglong2 g = ld_pair(s->agg);
                if (tag_of(i.x) == tagI && tag_of(i.y) == tagI) {
                    state = kStInc;
                    v0 = uint32_t(i.x);
                    v1 = uint32_t(i.y);
                    break;
                }
                if (tag_of(g.x) == tagA && tag_of(g.y) == tagA) {
                    state = kStAgg;
                    v0 = uint32_t(g.x);
                    v1 = uint32_t(g.y);
                    break;
                }
                if (++spins > 4) __nanosleep(20);
                if (spins > (1u << 26)) {  // a bug, never wait forever
                    g_vqb_fault = 1u;
                    state = kStInc;
                    break;
                }
            }
        }
        const unsigned inc_mask = __ballot_sync(kFull, in_seg && state == kStInc);
        const int stop = inc_mask ? (__ffs(inc_mask) - 1) : 31;
        const bool take = in_seg && lane <= stop;
        v0 = take ? v0 : 0u;
        v1 = take ? v1 : 0u;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            v0 += __shfl_xor_sync(kFull, v0, s);
            v1 += __shfl_xor_sync(kFull, v1, s);
        }
        acc0 += v0;
        acc1 += v1;
        const unsigned seg_mask = __ballot_sync(kFull, in_seg);
        if (inc_mask || seg_mask != kFull) break;
        pred -= 32;
    }
    if (lane == 0)
        pub_pair(st[uint64_t(tile) * stride + side].inc, tagI, acc0 + c0, acc1 + c1);
    return make_uint2(acc0, acc1);
}

// Two 32-bit class counters packed in one u64, claimed with ONE atomic: the
// low half never carries into the high half because every count is < 2^32.
__device__ __forceinline__ uint2 claim_pair(unsigned long long* ctr, uint32_t c0, uint32_t c1) {
    const unsigned long long old =
        atomicAdd(ctr, static_cast<unsigned long long>(c0) | (static_cast<unsigned long long>(c1) << 32));
    return make_uint2(uint32_t(old), uint32_t(old >> 32));
}

__device__ __forceinline__ uint2 read_pair(const unsigned long long* ctr) {
    const unsigned long long v = __ldcg(ctr);
    return make_uint2(uint32_t(v), uint32_t(v >> 32));
}

// ---------------------------------------------------------------------------
// Tile staging
// ---------------------------------------------------------------------------
template <int NC>
struct TileSmem {
    double sx[kTile];
    double sy[kTile];
    uint32_t sid[kTile];
    uint32_t wcnt[NC][kItems * kWarps];
    uint32_t cbase[NC + 1];
    uint32_t cnt[NC];    // tile counts per class
    uint32_t excl[NC];   // offset of the tile inside its range, per class
    unsigned long long rkey[NC][kWarps];  // block reduction scratch
    uint32_t ridx[NC][kWarps];
};

// Ranks: per item 2 (NC=2) or 3 (NC=4) warp ballots encode every lane's
// class; each lane's rank is a popcount of the lanes before it in its class,
// and lanes 0..NC-1 record the per-class warp counts.  Then one warp scan per
// class over the (item, warp) counts.  cls[i] == NC means "no class".
template <int NC>
__device__ __forceinline__ void scan_tile(TileSmem<NC>& S, const int (&cls)[kItems],
                                          uint32_t (&rk)[kItems]) {
    static_assert(NC == 2 || NC == 4, "two or four classes");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const int c = cls[i];
        const bool v = c < NC;
        const unsigned V = __ballot_sync(kFull, v);
        const unsigned B0 = __ballot_sync(kFull, v && (c & 1));
        unsigned M, Mq;
        if (NC == 4) {
            const unsigned B1 = __ballot_sync(kFull, v && (c & 2));
            M = V & ((c & 1) ? B0 : ~B0) & ((c & 2) ? B1 : ~B1);
            Mq = V & ((lane & 1) ? B0 : ~B0) & ((lane & 2) ? B1 : ~B1);
        } else {
            M = V & ((c & 1) ? B0 : ~B0);
            Mq = V & ((lane & 1) ? B0 : ~B0);
        }
        rk[i] = __popc(M & lt);
        if (lane < NC) S.wcnt[lane][i * kWarps + warp] = __popc(Mq);
    }
    __syncthreads();
    static_assert(kItems * kWarps == 32, "one scan entry per lane");
    if (warp < NC) {
        const int c = warp;
        const uint32_t v = S.wcnt[c][lane];
        uint32_t incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += o;
        }
        S.wcnt[c][lane] = incl - v;
        if (lane == 31) S.cnt[c] = incl;
    }
    __syncthreads();
    if (threadIdx.x <= NC) {
        uint32_t acc = 0;
        for (int c = 0; c < int(threadIdx.x); ++c) acc += S.cnt[c];
        S.cbase[threadIdx.x] = acc;
    }
    __syncthreads();
}

// Survivors to the staging area in input order (class by class).
template <int NC>
__device__ __forceinline__ void stage_tile(TileSmem<NC>& S, const double (&ux)[kItems],
                                           const double (&uy)[kItems],
                                           const uint32_t (&uid)[kItems], const int (&cls)[kItems],
                                           const uint32_t (&rk)[kItems]) {
    const int warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const int c = cls[i];
        if (c < NC) {
            const uint32_t s = S.cbase[c] + S.wcnt[c][i * kWarps + warp] + rk[i];
            S.sx[s] = ux[i];
            S.sy[s] = uy[i];
            S.sid[s] = uid[i];
        }
    }
}

// Block-wide reduction of every thread's running (key, idx) candidate of
// class c; the winner goes to thread 0 only.
template <int NC>
__device__ __forceinline__ void block_key_best(TileSmem<NC>& S, int c, unsigned long long k,
                                               uint32_t i, const double* __restrict__ xs,
                                               const double* __restrict__ ys,
                                               unsigned long long& ko, uint32_t& io) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    warp_key_best(k, i, xs, ys);
    if (lane == 0) {
        S.rkey[c][warp] = k;
        S.ridx[c][warp] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ko = S.rkey[c][0];
        io = S.ridx[c][0];
        for (int w = 1; w < kWarps; ++w) {
            const unsigned long long kk = S.rkey[c][w];
            const uint32_t ii = S.ridx[c][w];
            if (kk < ko || (kk == ko && key_better(kk, ii, ko, io, xs, ys))) {
                ko = kk;
                io = ii;
            }
        }
    }
    __syncthreads();
}

// Stream the staged survivors to their final places.  base[c] is the first
// (fwd) / last (bwd) position of class c in its range.
template <int NC>
__device__ __forceinline__ void flush_tile(const TileSmem<NC>& S, const uint64_t (&base)[NC],
                                           const bool (&fwd)[NC], double* __restrict__ ox,
                                           double* __restrict__ oy, uint32_t* __restrict__ oid,
                                           uint64_t out_cap) {
    const uint32_t total = S.cbase[NC];
    for (uint32_t e = threadIdx.x; e < total; e += kThreads) {
        int c = 0;
        uint64_t b = base[0];
        bool f = fwd[0];
#pragma unroll
        for (int k = 1; k < NC; ++k) {
            if (e >= S.cbase[k]) {
                c = k;
                b = base[k];
                f = fwd[k];
            }
        }
        const uint64_t r = uint64_t(S.excl[c]) + (e - S.cbase[c]);
        const uint64_t pos = f ? b + r : b - r;
        VQB_CHECK(pos < out_cap, 10 + c, pos, out_cap);
#ifdef VQB_DEBUG
        if (pos >= out_cap) continue;
#endif
        ox[pos] = S.sx[e];
        oy[pos] = S.sy[e];
        oid[pos] = S.sid[e];
    }
}

__device__ __forceinline__ Best ldcg_best(const Best* p) {
    Best b;
    b.off = __ldcg(&p->off);
    b.x = __ldcg(&p->x);
    b.y = __ldcg(&p->y);
    b.idx = __ldcg(&p->idx);
    b.valid = __ldcg(&p->valid);
    return b;
}

// Branch-free running arg-max update of the candidate's class (one select
// chain for the incumbent, one predicated write-back); exact offset ties take
// a warp-uniform slow path that consults the coordinates.
template <int NC>
__device__ __forceinline__ void running_best(unsigned long long (&kb)[NC], uint32_t (&ib)[NC],
                                             int c, unsigned long long k, uint32_t id,
                                             const double* __restrict__ xs,
                                             const double* __restrict__ ys) {
    unsigned long long kc = kb[0];
    uint32_t ic = ib[0];
#pragma unroll
    for (int q = 1; q < NC; ++q) {
        kc = (c == q) ? kb[q] : kc;
        ic = (c == q) ? ib[q] : ic;
    }
    bool take = (c < NC) && (k < kc);
    const bool tie = (c < NC) && (k == kc) && (id != ic);
    if (__any_sync(kFull, tie)) {
        if (tie) take = key_better(k, id, kc, ic, xs, ys);
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        const bool w = take && (c == q);
        kb[q] = w ? k : kb[q];
        ib[q] = w ? id : ib[q];
    }
}

// ===========================================================================
// Scheduling.  Tile t belongs to CTA t mod G; CTAs visit their tiles in
// increasing order with the next tile prefetched into registers.
// Output offsets, two modes:
//   STABLE = false (default): one packed atomicAdd per tile side claims the
//     tile's place in each class's range; no tile ever waits for another.
//     The order of survivors inside S1/S2 follows claim order, which the
//     reference leaves unspecified (extract.hpp:14-18; its own parallel_extract
//     reorders), so every hull output is unchanged.
//   STABLE = true: decoupled look-back over self-validating status words gives
//     each survivor its input-order position (order-preserving compaction).
//     Launched cooperatively: all G CTAs are co-resident, so every look-back
//     waits only on running CTAs.
// ===========================================================================

// ===========================================================================
// KB: root partition — hull levels 1 and 2 fused (probe P5).
// Each input point is classified against the bootstrap edges p->q / q->p and
// then against its side's two child edges:
//   class 0: S1 ∧ left(p->r1)        class 1: S1 ∧ ¬0 ∧ left(r1->q)
//   class 2: S2 ∧ left(q->r2)        class 3: S2 ∧ ¬2 ∧ left(r2->p)
// exactly the sets of the reference's two second-level extract_subsets calls,
// with r11..r22 from the same pass.  Output: S1's range [0,|S1|) and S2's
// range [|S1|, |S1|+|S2|), each split two-sided.
// ===========================================================================
template <bool STABLE>
__global__ void __launch_bounds__(kThreads, kPartMinBlocks) root_partition_kernel(RootArgs a) {
    VQB_PDL();
    __shared__ TileSmem<4> S;
    __shared__ bool s_last;
    const RootInfo& R = *a.root;
    const double px = R.px, py = R.py, qx = R.qx, qy = R.qy;
    const double r1x = R.r1.x, r1y = R.r1.y, r2x = R.r2.x, r2y = R.r2.y;
    const uint32_t n1 = R.cnt1, n2 = R.cnt2;
    // child frames (kernels.hpp:23-25): 0: p->r1, 1: r1->q, 2: q->r2, 3: r2->p
    const double f0x = dsub(r1x, px), f0y = dsub(r1y, py);
    const double f1x = dsub(qx, r1x), f1y = dsub(qy, r1y);
    const double f2x = dsub(r2x, qx), f2y = dsub(r2y, qy);
    const double f3x = dsub(px, r2x), f3y = dsub(py, r2y);
    uint64_t base[4];
    const bool fwd[4] = {true, false, true, false};
    base[0] = 0;
    base[1] = uint64_t(n1) - 1;  // unused when empty
    base[2] = n1;
    base[3] = uint64_t(n1) + n2 - 1;
    // per-thread running arg-max of each class over all of this CTA's tiles
    unsigned long long kb[4] = {kNoKey, kNoKey, kNoKey, kNoKey};
    uint32_t ib[4] = {kNoIdx, kNoIdx, kNoIdx, kNoIdx};

    double ux[kItems], uy[kItems];
    uint32_t uid[kItems];
    bool inr[kItems];
    auto load = [&](uint32_t t) {
        const uint64_t start = uint64_t(t) * kTile;
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const uint64_t pos = start + uint64_t(i) * kThreads + threadIdx.x;
            inr[i] = pos < a.n;
            ux[i] = inr[i] ? ld_stream(a.xs + pos) : 0.0;
            uy[i] = inr[i] ? ld_stream(a.ys + pos) : 0.0;
            uid[i] = uint32_t(pos);
        }
    };
    uint32_t t = blockIdx.x;
    if (t < a.ntiles) load(t);
    while (t < a.ntiles) {
        int cls[kItems];
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const double u = ux[i], w = uy[i];
            const double A = dsub(px, u), B = dsub(py, w);
            const double Cc = dsub(qx, u), D = dsub(qy, w);
            const double t1 = dmul(A, D), t2 = dmul(B, Cc);
            const bool s1 = t1 > t2;           // left of p->q
            const bool s2 = !s1 && (t2 > t1);  // left of q->p
            // second level, side-selected operands
            const double rx = s1 ? r1x : r2x, ry = s1 ? r1y : r2y;
            const double P1x = s1 ? A : Cc, P1y = s1 ? B : D;
            const double Q2x = s1 ? Cc : A, Q2y = s1 ? D : B;
            const double E = dsub(rx, u), F = dsub(ry, w);
            const bool L = left_diff(P1x, P1y, E, F);         // left of (side start -> r)
            const bool Rr = !L && left_diff(E, F, Q2x, Q2y);  // left of (r -> side end)
            const int side = s1 ? 0 : 2;
            int c = (s1 || s2) ? (L ? side : (Rr ? side + 1 : 4)) : 4;
            c = inr[i] ? c : 4;
            cls[i] = c;
            // fused farthest-point search (extract_core.hpp:462-463)
            const double edx = s1 ? (L ? f0x : f1x) : (L ? f2x : f3x);
            const double edy = s1 ? (L ? f0y : f1y) : (L ? f2y : f3y);
            running_best<4>(kb, ib, c, key_of(lat_off(edx, edy, u, w)), uid[i], a.xs, a.ys);
        }
        uint32_t rk[kItems];
        scan_tile<4>(S, cls, rk);
        uint2 claimed = make_uint2(0u, 0u);
        if (threadIdx.x < 2) {
            const uint32_t side = threadIdx.x;
            if (STABLE)
                publish_counts(&a.status[uint64_t(t) * 2 + side], t == 0, S.cnt[2 * side],
                               S.cnt[2 * side + 1], a.epoch);
            else
                claimed = claim_pair(&a.side_ctr[side], S.cnt[2 * side], S.cnt[2 * side + 1]);
        }
        stage_tile<4>(S, ux, uy, uid, cls, rk);
        const uint32_t tn = t + gridDim.x;
        if (tn < a.ntiles) load(tn);  // in flight during the offsets and the stores
        if (STABLE) {
            if (threadIdx.x < 64) {
                const uint32_t side = threadIdx.x >> 5;
                claimed = lookback16(t, 0u, S.cnt[2 * side], S.cnt[2 * side + 1], a.status, 2u,
                                     side, a.epoch);
            }
        }
        if ((STABLE && (threadIdx.x & 31) == 0 && threadIdx.x < 64) || (!STABLE && threadIdx.x < 2)) {
            const uint32_t side = STABLE ? (threadIdx.x >> 5) : threadIdx.x;
            S.excl[2 * side] = claimed.x;
            S.excl[2 * side + 1] = claimed.y;
        }
        __syncthreads();
        flush_tile<4>(S, base, fwd, a.ox, a.oy, a.oid, a.out_cap);
        __syncthreads();
        t = tn;
    }
    // CTA arg-max partials; the last CTA out reduces them and emits the four
    // child nodes
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        unsigned long long ko;
        uint32_t io;
        block_key_best<4>(S, q, kb[q], ib[q], a.xs, a.ys, ko, io);
        if (threadIdx.x == 0) {
            const double edx = q == 0 ? f0x : (q == 1 ? f1x : (q == 2 ? f2x : f3x));
            const double edy = q == 0 ? f0y : (q == 1 ? f1y : (q == 2 ? f2y : f3y));
            a.cta_part[blockIdx.x * 4 + q] = best_from_key(ko, io, edx, edy, a.xs, a.ys);
        }
    }
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < 4) {
        const int c = warp;
        Best b = best_none();
        for (uint32_t k = lane; k < gridDim.x; k += 32) {
            const Best o = ldcg_best(&a.cta_part[k * 4 + c]);
            if (prefer(o, b)) b = o;
        }
        b = warp_best(b);
        if (lane == 0) {
            uint32_t m = 0;
            if (a.ntiles) {
                const uint2 w = STABLE
                    ? inclusive_of(&a.status[uint64_t(a.ntiles - 1) * 2 + (c >> 1)], a.epoch)
                    : read_pair(&a.side_ctr[c >> 1]);
                m = (c & 1) ? w.y : w.x;
            }
            ChildRec ch;
            // children: (p, r11, r1) (r1, r12, q) (q, r21, r2) (r2, r22, p)
            ch.px = c == 0 ? px : (c == 1 ? r1x : (c == 2 ? qx : r2x));
            ch.py = c == 0 ? py : (c == 1 ? r1y : (c == 2 ? qy : r2y));
            ch.qx = c == 0 ? r1x : (c == 1 ? qx : (c == 2 ? r2x : px));
            ch.qy = c == 0 ? r1y : (c == 1 ? qy : (c == 2 ? r2y : py));
            ch.rx = b.x;
            ch.ry = b.y;
            ch.r_idx = b.idx;
            ch.m = m;
            ch.begin = (c & 1) ? (c == 1 ? uint64_t(n1) - m : uint64_t(n1) + n2 - m)
                               : (c == 0 ? 0 : uint64_t(n1));
            a.children[c] = ch;
        }
    }
    if (threadIdx.x == 0) *a.ticket = 0;
}

// ===========================================================================
// K2: level kernel — all live segments of one recursion level in one launch.
// Tiles never straddle segments; a segment's tiles are consecutive ids.
// GENERAL = two unrelated edges (the extract_subsets API); otherwise the
// edges p->r and r->q share r (two subtractions saved per point).
// Each thread keeps a running best for the segment its CTA is visiting; on
// leaving a segment the CTA reduces them and publishes one partial; the CTA
// whose finished-tile count completes the segment reduces the partials and
// emits the two children.
// ===========================================================================
template <bool GENERAL, bool STABLE>
__device__ __forceinline__ void level_body(const LevelArgs& a) {
    __shared__ TileSmem<2> S;
    __shared__ SegRec s_seg[2];
    __shared__ uint32_t s_k[2];
    __shared__ SegRec s_cur;  // segment whose arg-max this CTA is accumulating
    __shared__ uint32_t s_cur_k, s_cur_tiles;
    __shared__ Best s_run[2];
    __shared__ bool s_last;
    __shared__ uint32_t s_ntiles;
    if (threadIdx.x == 0) {
        s_ntiles = a.info->ntiles;
        s_cur_k = 0xffffffffu;
        s_cur_tiles = 0;
    }
    __syncthreads();
    const uint32_t ntiles = s_ntiles;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long kb[2] = {kNoKey, kNoKey};
    uint32_t ib[2] = {kNoIdx, kNoIdx};

    auto finalize = [&]() {
        for (int c = 0; c < 2; ++c) {
            unsigned long long ko;
            uint32_t io;
            block_key_best<2>(S, c, kb[c], ib[c], a.gx, a.gy, ko, io);
            if (threadIdx.x == 0)
                s_run[c] = best_from_key(ko, io, c == 0 ? s_cur.adx : s_cur.bdx,
                                         c == 0 ? s_cur.ady : s_cur.bdy, a.gx, a.gy);
        }
        if (threadIdx.x == 0) {
            const uint32_t k = s_cur_k;
            const uint32_t slot = atomicAdd(&a.seg_pcnt[k], 1u);
            VQB_CHECK(slot < s_cur.ntiles && 2 * (uint64_t(s_cur.tile0) + slot) + 1 < a.part_cap,
                      50, slot, s_cur.ntiles);
            a.tile_part[2 * (uint64_t(s_cur.tile0) + slot)] = s_run[0];
            a.tile_part[2 * (uint64_t(s_cur.tile0) + slot) + 1] = s_run[1];
            __threadfence();
            const uint32_t done = atomicAdd(&a.seg_done[k], s_cur_tiles) + s_cur_tiles;
            s_last = (done == s_cur.ntiles);
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            if (warp < 2) {
                const int c = warp;
                const uint32_t np = __ldcg(&a.seg_pcnt[s_cur_k]);
                VQB_CHECK(np <= s_cur.ntiles, 51, np, s_cur.ntiles);
                Best b = best_none();
                for (uint32_t j = lane; j < np; j += 32) {
                    const Best o = ldcg_best(&a.tile_part[2 * (uint64_t(s_cur.tile0) + j) + c]);
                    if (prefer(o, b)) b = o;
                }
                b = warp_best(b);
                if (lane == 0) {
                    const SegRec& g = s_cur;
                    const uint2 w = STABLE
                        ? inclusive_of(&a.status[uint64_t(g.tile0) + g.ntiles - 1], a.epoch)
                        : read_pair(&a.seg_ctr[s_cur_k]);
                    const uint32_t m = c == 0 ? w.x : w.y;
                    ChildRec ch;
                    if (c == 0) {  // left of p->r: triangle (p, rL, r)
                        ch.px = g.px; ch.py = g.py; ch.qx = g.rx; ch.qy = g.ry;
                        ch.begin = g.out;
                    } else {       // left of r->q: triangle (r, rR, q)
                        ch.px = GENERAL ? g.bx : g.rx; ch.py = GENERAL ? g.by : g.ry;
                        ch.qx = g.qx; ch.qy = g.qy;
                        ch.begin = g.out + g.m - m;
                    }
                    ch.rx = b.x;
                    ch.ry = b.y;
                    ch.r_idx = b.idx;
                    ch.m = m;
                    VQB_CHECK(2 * uint64_t(s_cur_k) + c < a.children_cap, 57, s_cur_k, a.children_cap);
                    a.children[2 * uint64_t(s_cur_k) + c] = ch;
                }
            }
        }
        __syncthreads();
        kb[0] = kb[1] = kNoKey;
        ib[0] = ib[1] = kNoIdx;
    };

    double ux[kItems], uy[kItems];
    uint32_t uid[kItems];
    uint32_t cnt = 0;
    auto fetch = [&](uint32_t tt, int bb) {  // segment of tile tt -> s_seg[bb], then loads
        if (threadIdx.x == 0) {
            const uint32_t k = a.tile_seg[tt];
            VQB_CHECK(k < a.info->nseg, 21, k, tt);
            s_k[bb] = k;
            s_seg[bb] = a.segs[k];
        }
        __syncthreads();
        const SegRec& g = s_seg[bb];
        const uint32_t j = tt - g.tile0;
        const uint64_t start = g.begin + uint64_t(j) * kTile;
        cnt = min(uint32_t(kTile), g.m - j * uint32_t(kTile));
        VQB_CHECK(j < g.ntiles && start + cnt <= a.in_cap, 20, start + cnt, a.in_cap);
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const uint32_t r = uint32_t(i) * kThreads + threadIdx.x;
            const bool v = r < cnt;
            ux[i] = v ? ld_stream(a.ix + start + r) : 0.0;
            uy[i] = v ? ld_stream(a.iy + start + r) : 0.0;
            uid[i] = v ? ld_stream(a.iid + start + r) : 0u;
        }
    };

    int b = 0;
    uint32_t t = blockIdx.x;
    if (t < ntiles) fetch(t, b);
    while (t < ntiles) {
        // entering a new segment?  Every thread decides on the same snapshot
        // of the shared state (the branch guards barriers).
        const uint32_t k_now = s_k[b], k_cur = s_cur_k;
        __syncthreads();
        if (k_now != k_cur) {
            if (k_cur != 0xffffffffu) finalize();
            if (threadIdx.x == 0) {
                s_cur = s_seg[b];
                s_cur_k = k_now;
                s_cur_tiles = 0;
            }
            __syncthreads();
        }
        const SegRec& g = s_seg[b];
        int cls[kItems];
        {
            const double px = g.px, py = g.py, rx = g.rx, ry = g.ry, qx = g.qx, qy = g.qy;
            const double adx = g.adx, ady = g.ady, bdx = g.bdx, bdy = g.bdy;
#pragma unroll
            for (int i = 0; i < kItems; ++i) {
                const double u = ux[i], w = uy[i];
                bool la, lb;
                if (GENERAL) {
                    la = left_diff(dsub(px, u), dsub(py, w), dsub(rx, u), dsub(ry, w));
                    lb = !la && left_diff(dsub(g.bx, u), dsub(g.by, w), dsub(qx, u), dsub(qy, w));
                } else {
                    const double A = dsub(px, u), B = dsub(py, w);
                    const double E = dsub(rx, u), F = dsub(ry, w);
                    const double Cc = dsub(qx, u), D = dsub(qy, w);
                    la = left_diff(A, B, E, F);
                    lb = !la && left_diff(E, F, Cc, D);
                }
                const bool v = uint32_t(i) * kThreads + threadIdx.x < cnt;
                const int c = !v ? 2 : (la ? 0 : (lb ? 1 : 2));
                cls[i] = c;
                // fused farthest-point search
                const unsigned long long k = key_of(lat_off(la ? adx : bdx, la ? ady : bdy, u, w));
                running_best<2>(kb, ib, c, k, uid[i], a.gx, a.gy);
            }
        }
        const uint32_t tile0 = g.tile0;
        const uint64_t base[2] = {g.out, g.out + g.m - 1};
        const bool fwd[2] = {true, false};
        uint32_t rk[kItems];
        scan_tile<2>(S, cls, rk);
        uint2 claimed = make_uint2(0u, 0u);
        if (threadIdx.x == 0) {
            if (STABLE) publish_counts(&a.status[t], t == tile0, S.cnt[0], S.cnt[1], a.epoch);
            else claimed = claim_pair(&a.seg_ctr[k_now], S.cnt[0], S.cnt[1]);
        }
        stage_tile<2>(S, ux, uy, uid, cls, rk);
        const uint32_t tn = t + gridDim.x;
        if (tn < ntiles) fetch(tn, b ^ 1);  // in flight during the offsets and the stores
        if (STABLE && warp == 0)
            claimed = lookback16(t, tile0, S.cnt[0], S.cnt[1], a.status, 1u, 0u, a.epoch);
        if (threadIdx.x == 0) {
            S.excl[0] = claimed.x;
            S.excl[1] = claimed.y;
        }
        __syncthreads();
        flush_tile<2>(S, base, fwd, a.ox, a.oy, a.oid, a.out_cap);
        if (threadIdx.x == 0) ++s_cur_tiles;
        __syncthreads();
        t = tn;
        b ^= 1;
    }
    if (s_cur_k != 0xffffffffu) finalize();
}

template <bool GENERAL, bool STABLE>
__global__ void __launch_bounds__(kThreads, kPartMinBlocks) level_kernel(LevelArgs a) {
    VQB_PDL();
    level_body<GENERAL, STABLE>(a);
}

// ===========================================================================
// Fast mode (default): no staging.  Per item, 2-3 warp ballots give every
// lane its rank inside its class among the warp's earlier lanes; per-warp
// running class counts live in lanes 0..NC-1 and are broadcast by shuffle.
// One tiny block scan over (class, warp) totals and one packed atomic per
// side claim the tile's place; survivors are then stored straight from
// registers — each warp store instruction writes one contiguous run per
// class.  The order inside S1/S2 follows claim order (unspecified in the
// reference, extract.hpp:14-18).
// ===========================================================================
struct FastSmem {
    uint32_t wtot[4][kWarps];   // per (class, warp) counts of the tile
    uint32_t wbase[4][kWarps];  // exclusive offsets of each warp inside the tile's class run
    uint32_t claim[4];          // the tile's offset inside each class range
    unsigned long long rkey[4][kWarps];
    uint32_t ridx[4][kWarps];
};

// running arg-max with double incumbents: a candidate is examined closely
// only when it is at least as good as its class incumbent, which after the
// first tiles is rare, so the common path is one compare per point.
template <int NC>
__device__ __forceinline__ void running_best_d(double (&bo)[NC], uint32_t (&bi)[NC], int c,
                                               double off, uint32_t id,
                                               const double* __restrict__ xs,
                                               const double* __restrict__ ys) {
    double inc = bo[0];
#pragma unroll
    for (int q = 1; q < NC; ++q) inc = (c == q) ? bo[q] : inc;
    const bool maybe = (c < NC) && !(off > inc);  // off <= inc (incumbent +inf when empty)
    if (__any_sync(kFull, maybe)) {
        if (maybe) {
            uint32_t ic = bi[0];
#pragma unroll
            for (int q = 1; q < NC; ++q) ic = (c == q) ? bi[q] : ic;
            bool take = off < inc || ic == kNoIdx;
            if (!take && off == inc && id != ic) {  // exact offset tie: lexicographic, then index
                const double x = xs[id], y = ys[id], xb = xs[ic], yb = ys[ic];
                take = (x != xb) ? (x < xb) : ((y != yb) ? (y < yb) : (id < ic));
            }
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                if (take && c == q) {
                    bo[q] = off;
                    bi[q] = id;
                }
            }
        }
    }
}

template <int NC>
__device__ __forceinline__ void block_best_d(FastSmem& S, int c, double off, uint32_t i,
                                             const double* __restrict__ xs,
                                             const double* __restrict__ ys,
                                             double& oo, uint32_t& io) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long k = (i == kNoIdx) ? kNoKey : key_of(off);
    warp_key_best(k, i, xs, ys);
    if (lane == 0 && warp < kWarps) {  // a control warp (no points) does not contribute
        S.rkey[c][warp] = k;
        S.ridx[c][warp] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long ko = S.rkey[c][0];
        io = S.ridx[c][0];
        for (int w = 1; w < kWarps; ++w) {
            const unsigned long long kk = S.rkey[c][w];
            const uint32_t ii = S.ridx[c][w];
            if (kk < ko || (kk == ko && key_better(kk, ii, ko, io, xs, ys))) {
                ko = kk;
                io = ii;
            }
        }
        oo = 0.0;
    }
    __syncthreads();
}

// ranks of one item: returns the lane's rank among the warp's lanes of its
// class so far (earlier items included); wrun (lanes < NC) accumulates counts
template <int NC>
__device__ __forceinline__ uint32_t warp_rank(int c, uint32_t& wrun) {
    // class bits as ballots; a lane's same-class mask is V & ~(B0 ^ m0) &
    // ~(B1 ^ m1) & ... with m = all-ones where the lane's own bit is set
    static_assert(NC == 2 || NC == 4 || NC == 8, "class count");
    const int lane = threadIdx.x & 31;
    const bool v = c < NC;
    const unsigned V = __ballot_sync(kFull, v);
    unsigned M = V, Mq = V;
#pragma unroll
    for (int b = 0; (1 << b) < NC; ++b) {
        const unsigned bit = (unsigned(c) >> b) & 1u;
        const unsigned B = __ballot_sync(kFull, v && bit);
        const unsigned mb = 0u - bit, lb = 0u - ((unsigned(lane) >> b) & 1u);
        M &= ~(B ^ mb);
        Mq &= ~(B ^ lb);
    }
    const uint32_t before = __shfl_sync(kFull, wrun, c & (NC - 1));
    wrun += (lane < NC) ? __popc(Mq) : 0u;
    return before + __popc(M & lanemask_lt());
}

// tile-level: (class, warp) exclusive offsets + class totals (by warp 0)
template <int NC>
__device__ __forceinline__ void tile_scan_fast(FastSmem& S, uint32_t (&tot)[NC]) {
    const int lane = threadIdx.x & 31;
    static_assert(NC * kWarps <= 32, "one lane per (class, warp)");
    const int c = lane / kWarps, w = lane % kWarps;
    uint32_t v = (lane < NC * kWarps) ? S.wtot[c][w] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int d = 1; d < kWarps; d <<= 1) {
        const uint32_t o = __shfl_up_sync(kFull, incl, d, kWarps);
        if (w >= d) incl += o;
    }
    if (lane < NC * kWarps) S.wbase[c][w] = incl - v;
#pragma unroll
    for (int q = 0; q < NC; ++q) tot[q] = __shfl_sync(kFull, incl, q * kWarps + kWarps - 1);
}

// p, q, r1, r2 and the side counts of the current hull, copied device-to-
// device into the constant bank right after KA (stream-ordered, no host
// sync): the FP64 instructions read them as constant operands, which keeps
// 16 registers free for occupancy.
__constant__ RootInfo c_root;

void upload_root_consts(const RootInfo* d_root, cudaStream_t st) {
    cudaMemcpyToSymbolAsync(c_root, d_root, sizeof(RootInfo), 0, cudaMemcpyDeviceToDevice, st);
}

template <bool PREFETCH>
__global__ void __launch_bounds__(kThreads, PREFETCH ? 3 : kFastMinBlocks) root_partition_fast(RootArgs a) {
    VQB_PDL();
    __shared__ FastSmem S;
    __shared__ double2 s_frame[4];   // class frames (edx, edy)
    __shared__ uint32_t s_org[4][kWarps];  // per (class, warp): store origin of rank 0
    __shared__ bool s_last;
    const RootInfo& R = c_root;
    const double px = R.px, py = R.py, qx = R.qx, qy = R.qy;
    const double r1x = R.r1.x, r1y = R.r1.y, r2x = R.r2.x, r2y = R.r2.y;
    const uint32_t n1 = R.cnt1, n2 = R.cnt2;
    const uint32_t n = uint32_t(a.n);  // < 2^32 (checked by the driver)
    if (threadIdx.x == 0) {
        // child frames (kernels.hpp:23-25): 0: p->r1, 1: r1->q, 2: q->r2, 3: r2->p
        s_frame[0] = make_double2(dsub(r1x, px), dsub(r1y, py));
        s_frame[1] = make_double2(dsub(qx, r1x), dsub(qy, r1y));
        s_frame[2] = make_double2(dsub(r2x, qx), dsub(r2y, qy));
        s_frame[3] = make_double2(dsub(px, r2x), dsub(py, r2y));
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    double bo[4] = {kInf, kInf, kInf, kInf};
    uint32_t bi[4] = {kNoIdx, kNoIdx, kNoIdx, kNoIdx};

    double ux[kItems], uy[kItems], nx[kItems], ny[kItems];
    auto load = [&](uint32_t t, double (&lx)[kItems], double (&ly)[kItems]) {
        const uint32_t start = t * uint32_t(kTile) + threadIdx.x;
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const uint32_t pos = start + uint32_t(i) * kThreads;
            const bool in = pos < n;
            lx[i] = in ? ld_stream(a.xs + pos) : 0.0;
            ly[i] = in ? ld_stream(a.ys + pos) : 0.0;
        }
    };
    uint32_t t = blockIdx.x;
    if (t < a.ntiles) load(t, ux, uy);
    while (t < a.ntiles) {
        const uint32_t start = t * uint32_t(kTile) + threadIdx.x;
        const uint32_t tn = t + gridDim.x;
        if (PREFETCH && tn < a.ntiles) load(tn, nx, ny);  // next tile in flight during this one
        int cls[kItems];
        uint32_t rk[kItems];
        uint32_t wrun = 0;
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const uint32_t pos = start + uint32_t(i) * kThreads;
            const double u = ux[i], w = uy[i];
            const double A = dsub(px, u), B = dsub(py, w);
            const double Cc = dsub(qx, u), D = dsub(qy, w);
            const double t1 = dmul(A, D), t2 = dmul(B, Cc);
            const bool s1 = t1 > t2;           // left of p->q
            const bool s2 = !s1 && (t2 > t1);  // left of q->p
            const double rx = s1 ? r1x : r2x, ry = s1 ? r1y : r2y;
            const double P1x = s1 ? A : Cc, P1y = s1 ? B : D;
            const double Q2x = s1 ? Cc : A, Q2y = s1 ? D : B;
            const double E = dsub(rx, u), F = dsub(ry, w);
            const bool L = left_diff(P1x, P1y, E, F);
            const bool Rr = !L && left_diff(E, F, Q2x, Q2y);
            const int side = s1 ? 0 : 2;
            int c = (s1 || s2) ? (L ? side : (Rr ? side + 1 : 4)) : 4;
            c = (pos < n) ? c : 4;
            cls[i] = c;
            rk[i] = warp_rank<4>(c, wrun);
            const double2 fr = s_frame[c & 3];  // fused farthest-point search
            running_best_d<4>(bo, bi, c, lat_off(fr.x, fr.y, u, w), pos, a.xs, a.ys);
        }
        if (lane < 4) S.wtot[lane][warp] = wrun;
        __syncthreads();
        if (warp == 0) {
            uint32_t tot[4];
            tile_scan_fast<4>(S, tot);
            if (lane < 2) {
                const uint2 c2 = claim_pair(&a.side_ctr[lane], tot[2 * lane], tot[2 * lane + 1]);
                S.claim[2 * lane] = c2.x;
                S.claim[2 * lane + 1] = c2.y;
            }
            __syncwarp();
            // store origin of rank 0 of every (class, warp): forward classes
            // grow from the range start, backward ones shrink from its end
            if (lane < 4 * kWarps) {
                const int c = lane / kWarps, w = lane % kWarps;
                const uint32_t off = S.claim[c] + S.wbase[c][w];
                const uint32_t org = c == 0 ? 0u : (c == 1 ? n1 - 1u : (c == 2 ? n1 : n1 + n2 - 1u));
                s_org[c][w] = (c & 1) ? org - off : org + off;
            }
        }
        __syncthreads();
        // stores straight from registers
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const int c = cls[i];
            if (c < 4) {
                const uint32_t o = s_org[c][warp];
                const uint32_t p = (c & 1) ? o - rk[i] : o + rk[i];
                VQB_CHECK(p < a.out_cap, 12, p, a.out_cap);
                a.ox[p] = ux[i];
                a.oy[p] = uy[i];
                a.oid[p] = start + uint32_t(i) * kThreads;
            }
        }
        if (PREFETCH) {
#pragma unroll
            for (int i = 0; i < kItems; ++i) {
                ux[i] = nx[i];
                uy[i] = ny[i];
            }
        } else if (tn < a.ntiles) {
            load(tn, ux, uy);
        }
        t = tn;
    }
    // CTA partials -> last CTA emits the four children
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        double oo;
        uint32_t io;
        block_best_d<4>(S, q, bo[q], bi[q], a.xs, a.ys, oo, io);
        if (threadIdx.x == 0)
            a.cta_part[blockIdx.x * 4 + q] =
                best_from_key(io == kNoIdx ? kNoKey : 0ull, io, s_frame[q].x, s_frame[q].y, a.xs, a.ys);
    }
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (warp < 4) {
        const int c = warp;
        Best b = best_none();
        for (uint32_t k = lane; k < gridDim.x; k += 32) {
            const Best o = ldcg_best(&a.cta_part[k * 4 + c]);
            if (prefer(o, b)) b = o;
        }
        b = warp_best(b);
        if (lane == 0) {
            const uint2 w = read_pair(&a.side_ctr[c >> 1]);
            const uint32_t m = (c & 1) ? w.y : w.x;
            ChildRec ch;
            ch.px = c == 0 ? px : (c == 1 ? r1x : (c == 2 ? qx : r2x));
            ch.py = c == 0 ? py : (c == 1 ? r1y : (c == 2 ? qy : r2y));
            ch.qx = c == 0 ? r1x : (c == 1 ? qx : (c == 2 ? r2x : px));
            ch.qy = c == 0 ? r1y : (c == 1 ? qy : (c == 2 ? r2y : py));
            ch.rx = b.x;
            ch.ry = b.y;
            ch.r_idx = b.idx;
            ch.m = m;
            ch.begin = (c & 1) ? (c == 1 ? uint64_t(n1) - m : uint64_t(n1) + n2 - m)
                               : (c == 0 ? 0 : uint64_t(n1));
            a.children[c] = ch;
        }
    }
    if (threadIdx.x == 0) *a.ticket = 0;
}

// ===========================================================================
// KB with a TMA ring (default fast path when the inputs are 16-byte aligned).
// One thread streams the CTA's upcoming full tiles (x and y, 8 KB each) into
// a kRing-deep shared-memory ring with cp.async.bulk, completing on
// mbarriers; the warps read their items from shared memory.  No per-element
// load instructions and no prefetch registers; the static tile schedule
// knows every future tile, so the ring runs kRing tiles ahead.
// ===========================================================================
constexpr int kRing = 3;

struct RootRing {
    double x[kRing][kTile];
    double y[kRing][kTile];
    unsigned long long bar[kRing];
};

// 8 compute warps + 1 control warp (scan, claim, TMA refills): the claim's
// atomic round trip overlaps the compute warps' arg-max updates.
constexpr int kCtlThreads = kThreads + 32;

__global__ void __launch_bounds__(kCtlThreads, 3) root_partition_tma(RootArgs a) {
    VQB_PDL();
    extern __shared__ __align__(128) unsigned char dsm[];
    RootRing& ring = *reinterpret_cast<RootRing*>(dsm);
    __shared__ FastSmem S;
    __shared__ double2 s_frame[4];
    __shared__ uint32_t s_org[4][kWarps];
    __shared__ bool s_last;
    const RootInfo& R = c_root;
    const double px = R.px, py = R.py, qx = R.qx, qy = R.qy;
    const double r1x = R.r1.x, r1y = R.r1.y, r2x = R.r2.x, r2y = R.r2.y;
    const uint32_t n1 = R.cnt1, n2 = R.cnt2;
    const uint32_t n = uint32_t(a.n);
    const uint32_t G = gridDim.x;
    const uint32_t nfull = n / kTile;  // tiles streamed by TMA; a partial last tile is loaded directly
    auto issue = [&](uint32_t k) {     // thread 0: local tile k -> stage k % kRing
        const uint32_t t = blockIdx.x + k * G;
        if (t >= nfull) return;
        const int s = int(k % kRing);
        mbar_expect_tx(&ring.bar[s], 2u * kTile * 8u);
        tma_load_1d(ring.x[s], a.xs + uint64_t(t) * kTile, kTile * 8u, &ring.bar[s]);
        tma_load_1d(ring.y[s], a.ys + uint64_t(t) * kTile, kTile * 8u, &ring.bar[s]);
    };
    const bool ctl = threadIdx.x >= kThreads;  // the control warp
    if (threadIdx.x == kThreads) {
        s_frame[0] = make_double2(dsub(r1x, px), dsub(r1y, py));
        s_frame[1] = make_double2(dsub(qx, r1x), dsub(qy, r1y));
        s_frame[2] = make_double2(dsub(r2x, qx), dsub(r2y, qy));
        s_frame[3] = make_double2(dsub(px, r2x), dsub(py, r2y));
        for (int s = 0; s < kRing; ++s) mbar_init(&ring.bar[s], 1);
        mbar_fence_init();
        for (uint32_t k = 0; k < kRing; ++k) issue(k);
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    double bo[4] = {kInf, kInf, kInf, kInf};
    uint32_t bi[4] = {kNoIdx, kNoIdx, kNoIdx, kNoIdx};

    uint32_t k = 0;
    for (uint32_t t = blockIdx.x; t < a.ntiles; t += G, ++k) {
        const uint32_t start = t * uint32_t(kTile) + (threadIdx.x & (kThreads - 1));
        const int s = int(k % kRing);
        double ux[kItems], uy[kItems];
        int cls[kItems];
        uint32_t rk[kItems];
        if (!ctl) {
            if (t < nfull) {
                mbar_wait(&ring.bar[s], (k / kRing) & 1u);
#pragma unroll
                for (int i = 0; i < kItems; ++i) {
                    ux[i] = ring.x[s][i * kThreads + threadIdx.x];
                    uy[i] = ring.y[s][i * kThreads + threadIdx.x];
                }
            } else {
#pragma unroll
                for (int i = 0; i < kItems; ++i) {
                    const uint32_t pos = start + uint32_t(i) * kThreads;
                    ux[i] = pos < n ? a.xs[pos] : 0.0;
                    uy[i] = pos < n ? a.ys[pos] : 0.0;
                }
            }
            uint32_t wrun = 0;
#pragma unroll
            for (int i = 0; i < kItems; ++i) {
                const uint32_t pos = start + uint32_t(i) * kThreads;
                const double u = ux[i], w = uy[i];
                const double A = dsub(px, u), B = dsub(py, w);
                const double Cc = dsub(qx, u), D = dsub(qy, w);
                const double t1 = dmul(A, D), t2 = dmul(B, Cc);
                const bool s1 = t1 > t2;           // left of p->q
                const bool s2 = !s1 && (t2 > t1);  // left of q->p
                const double rx = s1 ? r1x : r2x, ry = s1 ? r1y : r2y;
                const double P1x = s1 ? A : Cc, P1y = s1 ? B : D;
                const double Q2x = s1 ? Cc : A, Q2y = s1 ? D : B;
                const double E = dsub(rx, u), F = dsub(ry, w);
                const bool L = left_diff(P1x, P1y, E, F);
                const bool Rr = !L && left_diff(E, F, Q2x, Q2y);
                const int side = s1 ? 0 : 2;
                int c = (s1 || s2) ? (L ? side : (Rr ? side + 1 : 4)) : 4;
                c = (pos < n) ? c : 4;
                cls[i] = c;
                rk[i] = warp_rank<4>(c, wrun);
            }
            if (lane < 4) S.wtot[lane][warp] = wrun;
        }
        __syncthreads();  // counts ready; every compute warp is done with stage s
        if (ctl) {
            uint32_t tot[4];
            tile_scan_fast<4>(S, tot);
            if (lane < 2) {
                const uint2 c2 = claim_pair(&a.side_ctr[lane], tot[2 * lane], tot[2 * lane + 1]);
                S.claim[2 * lane] = c2.x;
                S.claim[2 * lane + 1] = c2.y;
            }
            __syncwarp();
            if (lane < 4 * kWarps) {
                const int c = lane / kWarps, w = lane % kWarps;
                const uint32_t off = S.claim[c] + S.wbase[c][w];
                const uint32_t org = c == 0 ? 0u : (c == 1 ? n1 - 1u : (c == 2 ? n1 : n1 + n2 - 1u));
                s_org[c][w] = (c & 1) ? org - off : org + off;
            }
            if (lane == 0) {
                fence_proxy_async_smem();
                issue(k + kRing);  // refill stage s with the tile kRing ahead
            }
        } else {
#pragma unroll
            for (int i = 0; i < kItems; ++i) {  // fused farthest-point search, overlapping the claim
                const int c = cls[i];
                const double2 fr = s_frame[c & 3];
                running_best_d<4>(bo, bi, c, lat_off(fr.x, fr.y, ux[i], uy[i]),
                                  start + uint32_t(i) * kThreads, a.xs, a.ys);
            }
        }
        __syncthreads();
        if (!ctl) {
#pragma unroll
            for (int i = 0; i < kItems; ++i) {
                const int c = cls[i];
                if (c < 4) {
                    const uint32_t o = s_org[c][warp];
                    const uint32_t p = (c & 1) ? o - rk[i] : o + rk[i];
                    VQB_CHECK(p < a.out_cap, 12, p, a.out_cap);
                    a.ox[p] = ux[i];
                    a.oy[p] = uy[i];
                    a.oid[p] = start + uint32_t(i) * kThreads;
                }
            }
        }
    }
    // CTA partials -> last CTA emits the four children (the control warp's
    // candidates are empty)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        double oo;
        uint32_t io;
        block_best_d<4>(S, q, bo[q], bi[q], a.xs, a.ys, oo, io);
        if (threadIdx.x == 0)
            a.cta_part[blockIdx.x * 4 + q] =
                best_from_key(io == kNoIdx ? kNoKey : 0ull, io, s_frame[q].x, s_frame[q].y, a.xs, a.ys);
    }
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (warp < 4) {
        const int c = warp;
        Best b = best_none();
        for (uint32_t kk = lane; kk < gridDim.x; kk += 32) {
            const Best o = ldcg_best(&a.cta_part[kk * 4 + c]);
            if (prefer(o, b)) b = o;
        }
        b = warp_best(b);
        if (lane == 0) {
            const uint2 w = read_pair(&a.side_ctr[c >> 1]);
            const uint32_t m = (c & 1) ? w.y : w.x;
            ChildRec ch;
            ch.px = c == 0 ? px : (c == 1 ? r1x : (c == 2 ? qx : r2x));
            ch.py = c == 0 ? py : (c == 1 ? r1y : (c == 2 ? qy : r2y));
            ch.qx = c == 0 ? r1x : (c == 1 ? qx : (c == 2 ? r2x : px));
            ch.qy = c == 0 ? r1y : (c == 1 ? qy : (c == 2 ? r2y : py));
            ch.rx = b.x;
            ch.ry = b.y;
            ch.r_idx = b.idx;
            ch.m = m;
            ch.begin = (c & 1) ? (c == 1 ? uint64_t(n1) - m : uint64_t(n1) + n2 - m)
                               : (c == 0 ? 0 : uint64_t(n1));
            a.children[c] = ch;
        }
    }
    if (threadIdx.x == 0) *a.ticket = 0;
}

// ===========================================================================
// KB' (default): level 1 of the reference's recursion behind the octagon
// filter, over the caller's arrays.  Per point:
//  1. drop it if it is provably inside the octagon by the margin
//     (RootPoly): strictly inside the shrunk inner box (4 compares), or else
//     in the x window of its upper and lower chord (the chains L..R and R..L
//     are x-monotone, so no other chord is within mu), inside the octagon's
//     y range, and below both chords' rounded cross-product threshold;
//  2. otherwise the reference's bootstrap split (hull.cpp:228-235): left of
//     p->q -> S1, left of q->p -> S2 (kernels.hpp:60-66 expression), with the
//     fused farthest-point search of each side (one offset o of the p->q
//     frame: S1 minimises o, S2 minimises -o, the exact offset of its own
//     q->p frame).
// S1 grows forward from 0 and S2 backward from n-1 of the output buffer (one
// packed atomic claim per tile), so the two sides can never collide.
//
// Pipeline (8 compute warps + 1 control warp, no CTA-wide barrier per tile):
//  * the control warp streams tiles into a kRing4-deep shared-memory ring
//    with cp.async.bulk (mbarrier completion);
//  * compute warps classify tile k, post their per-warp counts (named barrier
//    A, arrive only), run the arg-max, then store tile k-1, whose offsets
//    the control warp published behind named barrier B — so the claim's
//    atomic round trip overlaps a whole tile of compute;
//  * stores re-read x and y from the ring stage, which the control warp
//    refills only once those stores are done (tile k-2's stage at step k).
// ===========================================================================
constexpr int kRing4 = 4;

struct RootRing4 {
    double x[kRing4][kTile];
    double y[kRing4][kTile];
    unsigned long long bar[kRing4];
};
// the filter pass's ring: two spare elements per stage for callers' arrays
// that are not 16-byte aligned (root_filter_tma)
struct FilterRing {
    double x[kRing4][kTile + 2];
    double y[kRing4][kTile + 2];
    unsigned long long bar[kRing4];
};

// named barriers with immediate ids (ptxas then reserves only those)
template <int ID>
__device__ __forceinline__ void named_sync_i(int count) {
    asm volatile("bar.sync %0, %1;" ::"n"(ID), "r"(count) : "memory");
}
template <int ID>
__device__ __forceinline__ void named_arrive_i(int count) {
    asm volatile("bar.arrive %0, %1;" ::"n"(ID), "r"(count) : "memory");
}
// barrier pair (base, base+1) selected by a parity bit
template <int BASE>
__device__ __forceinline__ void named_sync(int par, int count) {
    if (par) named_sync_i<BASE + 1>(count); else named_sync_i<BASE>(count);
}
template <int BASE>
__device__ __forceinline__ void named_arrive(int par, int count) {
    if (par) named_arrive_i<BASE + 1>(count); else named_arrive_i<BASE>(count);
}

__global__ void __launch_bounds__(kCtlThreads, 3) root_filtered_tma(RootArgs a) {
    VQB_PDL();
    extern __shared__ __align__(128) unsigned char dsm[];
    RootRing4& ring = *reinterpret_cast<RootRing4*>(dsm);
    __shared__ FastSmem S;
    __shared__ uint32_t s_wtot[2][2][kWarps];
    __shared__ uint32_t s_org[2][2][kWarps];
    __shared__ uint16_t s_q[kWarps][kTile / kWarps];             // a warp's points needing the slow path
    __shared__ uint16_t s_surv[2][kWarps][kTile / kWarps];       // survivors in rank order: idx | class << 10
    __shared__ uint32_t s_sn[2][kWarps];
    __shared__ bool s_last;
    const RootInfo& R = c_root;
    const RootPoly& P = R.poly;
    const double px = R.px, py = R.py, qx = R.qx, qy = R.qy;
    const uint32_t n = uint32_t(a.n);
    const uint32_t G = gridDim.x;
    const uint32_t nfull = n / kTile;
    const uint32_t nt = a.ntiles > blockIdx.x ? (a.ntiles - blockIdx.x + G - 1) / G : 0u;  // this CTA's tiles
    const bool ctl = threadIdx.x >= kThreads;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tid = threadIdx.x & (kThreads - 1);
    auto issue = [&](uint32_t k) {
        const uint32_t t = blockIdx.x + k * G;
        if (t >= nfull) return;
        const int s = int(k % kRing4);
        mbar_expect_tx(&ring.bar[s], 2u * kTile * 8u);
        tma_load_1d(ring.x[s], a.xs + uint64_t(t) * kTile, kTile * 8u, &ring.bar[s]);
        tma_load_1d(ring.y[s], a.ys + uint64_t(t) * kTile, kTile * 8u, &ring.bar[s]);
    };
    if (threadIdx.x == kThreads) {
        for (int s = 0; s < kRing4; ++s) mbar_init(&ring.bar[s], 1);
        mbar_fence_init();
        for (uint32_t k = 0; k < kRing4; ++k) issue(k);
    }
    __syncthreads();
    const double adx = dsub(qx, px), ady = dsub(qy, py);  // frame of p->q (kernels.hpp:23-25)
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    double bo[2] = {kInf, kInf};
    uint32_t bi[2] = {kNoIdx, kNoIdx};

    if (ctl) {
        // ---- control warp: refills, per-tile scan + claim + store origins
        const int c = (lane >> 3) & 1, w = lane & 7;
        for (uint32_t k = 0; k < nt; ++k) {
            const int par = int(k & 1);
            named_sync<1>(par, kCtlThreads);  // counts of tile k posted; tile k-2 stored
            if (lane == 0 && k >= 2) {
                fence_proxy_async_smem();
                issue(k - 2 + kRing4);  // refill tile k-2's stage
            }
            const uint32_t v = lane < 16 ? s_wtot[par][c][w] : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int d = 1; d < kWarps; d <<= 1) {
                const uint32_t o = __shfl_up_sync(kFull, incl, d, kWarps);
                if (w >= d) incl += o;
            }
            const uint32_t t0 = __shfl_sync(kFull, incl, kWarps - 1);
            const uint32_t t1 = __shfl_sync(kFull, incl, 2 * kWarps - 1);
            uint2 c2 = make_uint2(0u, 0u);
            if (lane == 0 && (t0 | t1)) c2 = claim_pair(&a.side_ctr[0], t0, t1);
            const uint32_t cl0 = __shfl_sync(kFull, c2.x, 0), cl1 = __shfl_sync(kFull, c2.y, 0);
            if (lane < 16) {
                const uint32_t off = (c ? cl1 : cl0) + incl - v;
                s_org[par][c][w] = c ? n - 1u - off : off;
            }
            named_arrive<3>(par, kCtlThreads);  // store origins of tile k published
        }
    } else {
        // ---- compute warps: every warp owns 128 points of a tile (4 per lane)
        const bool filter = P.filter != 0;
        const double bx0 = filter ? P.bx0 : kInf, bx1 = filter ? P.bx1 : -kInf;
        const double by0 = filter ? P.by0 : kInf, by1 = filter ? P.by1 : -kInf;
        bool bad = false;  // non-finite y (x was checked by K1'); never inside the box
        const unsigned lt = lanemask_lt();
        auto store_tile = [&](uint32_t k) {  // tile k's survivors, offsets behind barrier B
            const int par = int(k & 1);
            named_sync<3>(par, kCtlThreads);
            const uint32_t t = blockIdx.x + k * G;
            const uint32_t tbase = t * uint32_t(kTile);
            const int s = int(k % kRing4);
            const uint32_t sn = s_sn[par][warp];
            // the list holds each class's survivors in rank order: a
            // survivor's rank = number of earlier entries of its class
            uint32_t run0 = 0, run1 = 0;
            for (uint32_t j0 = 0; j0 < sn; j0 += 32) {
                const uint32_t j = j0 + lane;
                const uint32_t e = j < sn ? s_surv[par][warp][j] : 0xffffu;
                const uint32_t c = (e >> 10) & 1u;
                const unsigned b1 = __ballot_sync(kFull, j < sn && c == 1u);
                const unsigned b0 = __ballot_sync(kFull, j < sn) & ~b1;
                if (j < sn) {
                    const uint32_t idx = e & (kTile - 1);
                    const uint32_t rk = c ? run1 + __popc(b1 & lt) : run0 + __popc(b0 & lt);
                    const uint32_t o = s_org[par][c][warp];
                    const uint32_t p = c ? o - rk : o + rk;
                    VQB_CHECK(p < a.out_cap, 14, p, a.out_cap);
                    a.ox[p] = ring.x[s][idx];
                    a.oy[p] = ring.y[s][idx];
                    a.oid[p] = tbase + idx;
                }
                run0 += __popc(b0);
                run1 += __popc(b1);
            }
        };
        for (uint32_t k = 0; k < nt; ++k) {
            const uint32_t t = blockIdx.x + k * G;
            const uint32_t tbase = t * uint32_t(kTile);
            const int s = int(k % kRing4);
            const int par = int(k & 1);
            if (t < nfull) {
                mbar_wait(&ring.bar[s], (k / kRing4) & 1u);
            } else {  // the partial last tile is staged by the warps themselves
#pragma unroll
                for (int i = 0; i < kItems; ++i) {
                    const uint32_t idx = uint32_t(i) * kThreads + tid;
                    ring.x[s][idx] = tbase + idx < n ? a.xs[tbase + idx] : 0.0;
                    ring.y[s][idx] = tbase + idx < n ? a.ys[tbase + idx] : 0.0;
                }
                __syncwarp();
            }
            // phase A: strictly inside the inner box -> dropped at once
            uint32_t qn = 0;
#pragma unroll
            for (int i = 0; i < kItems; ++i) {
                const uint32_t idx = uint32_t(i) * kThreads + tid;
                const double u = ring.x[s][idx], w = ring.y[s][idx];
                const bool need = (tbase + idx < n) & !((u > bx0) & (u < bx1) & (w > by0) & (w < by1));
                const unsigned b = __ballot_sync(kFull, need);
                if (need) s_q[warp][qn + __popc(b & lt)] = uint16_t(idx);
                qn += __popc(b);
            }
            __syncwarp();
            // phase C: the rest, densely, 32 at a time
            uint32_t wrun = 0, sn = 0;
            for (uint32_t r0 = 0; r0 < qn; r0 += 32) {
                const uint32_t j = r0 + lane;
                const bool valid = j < qn;
                const uint32_t idx = valid ? s_q[warp][j] : 0u;
                const double u = ring.x[s][idx], w = ring.y[s][idx];
                int c = 2;
                if (valid) {
                    bad |= nonfinite_bits(w);
                    const double du = fabs(u - P.ocx), dw = fabs(w - P.ocy);
                    bool drop = filter && du < P.ohx && dw < P.ohy && du + dw < P.od;  // inner octagon
                    if (filter && !drop) {
                        drop = true;
#pragma unroll
                        for (int q = 0; q < kPolyV; ++q)  // inside by the margin w.r.t. every chord
                            drop &= __fma_rn(P.fa[q], u, __dmul_rn(P.fb[q], w)) < P.fg[q];
                    }
                    if (!drop) {
                        const double A = dsub(px, u), B = dsub(py, w);
                        const double Cc = dsub(qx, u), D = dsub(qy, w);
                        const double t1 = dmul(A, D), t2 = dmul(B, Cc);
                        c = t1 > t2 ? 0 : (t2 > t1 ? 1 : 2);  // left of p->q / of q->p
                    }
                }
                if (__any_sync(kFull, c < 2)) {
                    const double o = lat_off(adx, ady, u, w);  // fused farthest-point search
                    running_best_d<2>(bo, bi, c, c ? -o : o, tbase + idx, a.xs, a.ys);
                    (void)warp_rank<2>(c, wrun);  // per-class warp counts
                    const unsigned b = __ballot_sync(kFull, c < 2);
                    if (c < 2) s_surv[par][warp][sn + __popc(b & lt)] = uint16_t(idx | (uint32_t(c) << 10));
                    sn += __popc(b);
                }
            }
            if (lane < 2) s_wtot[par][lane][warp] = wrun;
            if (lane == 0) s_sn[par][warp] = sn;
            named_arrive<1>(par, kCtlThreads);
            if (k >= 1) store_tile(k - 1);
        }
        if (nt >= 1) store_tile(nt - 1);
        if (bad) atomicOr(&a.root_w->nonfinite, 1u);
    }
    __syncthreads();
    // CTA partials -> last CTA writes the two level-2 slots
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        double oo;
        uint32_t io;
        block_best_d<2>(S, q, bo[q], bi[q], a.xs, a.ys, oo, io);
        if (threadIdx.x == 0)
            a.cta_part[blockIdx.x * 2 + q] = best_from_key(io == kNoIdx ? kNoKey : 0ull, io, q ? -adx : adx,
                                                           q ? -ady : ady, a.xs, a.ys);
    }
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (warp < 2) {
        const int c = warp;
        Best b = best_none();
        for (uint32_t kk = lane; kk < gridDim.x; kk += 32) {
            const Best o = ldcg_best(&a.cta_part[kk * 2 + c]);
            if (prefer(o, b)) b = o;
        }
        b = warp_best(b);
        if (lane == 0) {
            const uint2 w = read_pair(&a.side_ctr[0]);
            const uint32_t m = c ? w.y : w.x;
            ChildRec ch;
            ch.px = c ? qx : px;
            ch.py = c ? qy : py;
            ch.qx = c ? px : qx;
            ch.qy = c ? py : qy;
            ch.rx = b.x;
            ch.ry = b.y;
            ch.r_idx = b.idx;
            ch.m = m;
            ch.begin = c ? uint64_t(n) - m : 0;
            a.children[c] = ch;
            if (c == 0) { a.root_w->cnt1 = m; a.root_w->r1 = b; }
            else { a.root_w->cnt2 = m; a.root_w->r2 = b; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a.side_ctr[0] = 0ull;  // re-arm for the next call
        *a.ticket = 0;
    }
}

// ===========================================================================
// KF (default root stage since the split root): pass 1 of the root, the
// octagon filter ALONE over the caller's arrays.  Per point: dropped when
// strictly inside the inner box, else when inside all 8 chords by the margin
// (the same RootPoly test as KB', so the same survivors); every survivor is
// appended to a dense list (x, y, input index) with one atomic claim per tile.
// Survivors also carry everything the reference's first level needs:
//  * find_extremes (geometry.cpp:7-36): a dropped point is strictly inside the
//    hull, so it can be neither the leftmost nor the rightmost point (nor one
//    of their exact duplicates) — lo/hi over the survivors ARE the input's
//    p and q, with the reference's tie-breaks and first-occurrence indices;
//  * finiteness of x and y (vqhull_c.cpp:32-34): a non-finite point never
//    passes the box (comparisons with NaN/inf are false) and never passes all
//    chords (the chord normals span the plane, so one form is +inf or NaN);
//  * the largest |coordinate| A of any survivor: the margin 2^-32 M is only
//    proven against rounding of predicates whose operands are <= 2^12 M, so
//    A > 2^12 M marks the call `unsafe` and the host reruns it unfiltered.
// The last CTA writes p, q and the first level's single slot: the bootstrap
// triangle (p, q, p) over all survivors (hull.cpp:228-235 — extract with
// edges p->q and q->p, then chain_recursive on each side), which the level
// machinery then partitions like any other segment.  Output frame: [p]
// chain(slot) where the slot's apex is q (hull.cpp:259-266; p == q means all
// points are equal: empty slot, output [p]).
// Bytes: 16 per input point + 20 per survivor; no arg-max, no classes.
// ===========================================================================
struct FilterPartial {
    ExtKey lo, hi;
    double amax;
    uint32_t nonfinite;
    uint32_t pad;
};

__device__ __forceinline__ void filter_warp_fold(ExtKey& lo, ExtKey& hi, double& amax, uint32_t& bad) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const ExtKey a = shfl_key(lo, s);
        if (lo_better(a, lo)) lo = a;
        const ExtKey b = shfl_key(hi, s);
        if (hi_better(b, hi)) hi = b;
        amax = fmax(amax, __shfl_xor_sync(kFull, amax, s));
        bad |= __shfl_xor_sync(kFull, bad, s);
    }
}

template <bool MIS>  // MIS: caller arrays not 16-byte aligned (the aligned instance carries no offsets)
__global__ void __launch_bounds__(kCtlThreads, 3) root_filter_tma(FilterArgs a) {
    VQB_PDL();
    VQB_STAMP(if (threadIdx.x == 0) atomicMin(&g_strace[5], gtimer_ns());)
    extern __shared__ __align__(128) unsigned char dsm[];
    using Ring = std::conditional_t<MIS, FilterRing, RootRing4>;
    Ring& ring = *reinterpret_cast<Ring*>(dsm);
    __shared__ uint32_t s_cnt[2][kWarps];                      // survivors per warp and tile
    __shared__ uint32_t s_org[2][kWarps];                      // their first output position
    __shared__ uint16_t s_q[kWarps][kTile / kWarps];           // a warp's points needing the chord test
    __shared__ uint16_t s_surv[2][kWarps][kTile / kWarps];     // a warp's survivors (tile-local index)
    __shared__ FilterPartial s_w[kCtlThreads / 32];
    __shared__ bool s_last;
    const RootPoly& P = c_root.poly;
    const uint32_t n = uint32_t(a.n);
    const uint32_t G = gridDim.x;
    // Caller arrays that are 8- but not 16-byte aligned (an odd offset into a
    // larger array): a tile's bulk copy starts at the 16-byte boundary below
    // its first element (one element early: a pointer that is not 16-byte
    // aligned is not the start of an allocation) and brings two elements
    // more; the points are read at a.xoff / a.yoff in the stage.  A tile whose
    // copy would run past the arrays' end is staged by the warps themselves,
    // like the partial last tile.
    constexpr bool mis = MIS;
    const uint32_t xoff = MIS ? a.xoff : 0u, yoff = MIS ? a.yoff : 0u;
    const uint32_t nfull = mis ? (n >= 2u ? (n - 2u) / kTile : 0u) : n / kTile;
    const uint32_t tile_bytes = (kTile + (mis ? 2u : 0u)) * 8u;
    const uint32_t nt = a.ntiles > blockIdx.x ? (a.ntiles - blockIdx.x + G - 1) / G : 0u;
    const bool ctl = threadIdx.x >= kThreads;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tid = threadIdx.x & (kThreads - 1);
    auto issue = [&](uint32_t k) {
        const uint32_t t = blockIdx.x + k * G;
        if (t >= nfull) return;
        const int s = int(k % kRing4);
        mbar_expect_tx(&ring.bar[s], 2u * tile_bytes);
        const unsigned long long pol = l2_evict_first_policy();
        tma_load_1d_stream(ring.x[s], a.xs - xoff + uint64_t(t) * kTile, tile_bytes, &ring.bar[s], pol);
        tma_load_1d_stream(ring.y[s], a.ys - yoff + uint64_t(t) * kTile, tile_bytes, &ring.bar[s], pol);
    };
    if (threadIdx.x == kThreads) {
        for (int s = 0; s < kRing4; ++s) mbar_init(&ring.bar[s], 1);
        mbar_fence_init();
        for (uint32_t k = 0; k < kRing4; ++k) issue(k);
    }
    __syncthreads();
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    ExtKey lo{kInf, 0.0, kNoIdx, 0u}, hi{-kInf, 0.0, kNoIdx, 0u};
    double amax = 0.0;
    uint32_t bad = 0;

    if (ctl) {
        // ---- control warp: refills, per-tile scan of the warp counts + claim
        for (uint32_t k = 0; k < nt; ++k) {
            const int par = int(k & 1);
            named_sync<1>(par, kCtlThreads);  // counts of tile k posted; tile k-2 stored
            if (lane == 0 && k >= 2) {
                fence_proxy_async_smem();
                issue(k - 2 + kRing4);  // refill tile k-2's stage
            }
            const uint32_t v = lane < kWarps ? s_cnt[par][lane] : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int d = 1; d < kWarps; d <<= 1) {
                const uint32_t o = __shfl_up_sync(kFull, incl, d);
                if (lane >= d) incl += o;
            }
            const uint32_t tot = __shfl_sync(kFull, incl, kWarps - 1);
            uint32_t base = 0;
            if (lane == 0 && tot) base = atomicAdd(a.ctr, tot);
            base = __shfl_sync(kFull, base, 0);
            if (lane < kWarps) s_org[par][lane] = base + incl - v;
            named_arrive<3>(par, kCtlThreads);  // store origins of tile k published
        }
    } else {
        // ---- compute warps: every warp owns 128 points of a tile (4 per lane)
        const uint32_t mode = P.filter != 0 ? P.oct_on : 0u;
        const double alim = 0x1p12 * P.mref;
        const bool filter = P.filter != 0;
        const double bx0 = filter ? P.bx0 : kInf, bx1 = filter ? P.bx1 : -kInf;
        const double by0 = filter ? P.by0 : kInf, by1 = filter ? P.by1 : -kInf;
        const unsigned lt = lanemask_lt();
        auto store_tile = [&](uint32_t k, uint32_t sn) {  // tile k's survivors, offsets behind barrier B
            const int par = int(k & 1);
            // (every warp syncs, survivors or not: the wait bounds the warps'
            // skew to one tile, which is what lets two barrier parities do)
            named_sync<3>(par, kCtlThreads);
            if (sn == 0) return;  // (warp-uniform) nothing to place
            const uint32_t tbase = (blockIdx.x + k * G) * uint32_t(kTile);
            const int s = int(k % kRing4);
            const uint32_t o = s_org[par][warp];
            for (uint32_t j = lane; j < sn; j += 32) {
                const uint32_t idx = s_surv[par][warp][j];
                const uint32_t p = o + j;
                VQB_CHECK(p < a.out_cap, 15, p, a.out_cap);
                const double u = ring.x[s][xoff + idx], w = ring.y[s][yoff + idx];
                a.ox[p] = u;
                a.oy[p] = w;
                a.oid[p] = tbase + idx;
                if (a.kx) {  // sharded hull: the certificate's copy (shard.cu)
                    a.kx[p] = u;
                    a.ky[p] = w;
                    a.kid[p] = tbase + idx;
                }
            }
        };
        // the tile loop, instantiated per inner test (a uniform choice per call:
        // each instance keeps only its own region's constants live)
        auto tiles = [&](auto mode_tag) {
        constexpr int kMode = decltype(mode_tag)::value;
        uint32_t sn_prev = 0;  // this warp's survivors of the tile before
        for (uint32_t k = 0; k < nt; ++k) {
            const uint32_t t = blockIdx.x + k * G;
            const uint32_t tbase = t * uint32_t(kTile);
            const int s = int(k % kRing4);
            const int par = int(k & 1);
            if (t < nfull) {
                mbar_wait(&ring.bar[s], (k / kRing4) & 1u);
            } else {  // the partial last tile is staged by the warps themselves
#pragma unroll
                for (int i = 0; i < kItems; ++i) {
                    const uint32_t idx = uint32_t(i) * kThreads + tid;
                    ring.x[s][xoff + idx] = tbase + idx < n ? a.xs[tbase + idx] : 0.0;
                    ring.y[s][yoff + idx] = tbase + idx < n ? a.ys[tbase + idx] : 0.0;
                }
                __syncwarp();
            }
            // phase A: strictly inside the inner box, or (a uniform choice,
            // when it adds coverage) inside the inner octagon or disk -> dropped
            uint32_t qn = 0;
            auto phase_a = [&](auto inner, auto with_box) {
#pragma unroll
                for (int i = 0; i < kItems; ++i) {
                    const uint32_t idx = uint32_t(i) * kThreads + tid;
                    const double u = ring.x[s][xoff + idx], w = ring.y[s][yoff + idx];
                    const bool in = (decltype(with_box)::value && ((u > bx0) & (u < bx1) & (w > by0) & (w < by1))) |
                                    inner(u, w);
                    const bool need = (tbase + idx < n) & !in;
                    const unsigned b = __ballot_sync(kFull, need);
                    if (need) s_q[warp][qn + __popc(b & lt)] = uint16_t(idx);
                    qn += __popc(b);
                }
            };
            if constexpr (kMode == 3) {  // the disk covers the box: one test
                phase_a([&](double u, double w) {
                    const double du = u - P.dcx, dw = w - P.dcy;
                    return __fma_rn(du, du, __dmul_rn(dw, dw)) < P.dr2;
                }, std::false_type{});
            } else if constexpr (kMode == 2) {
                phase_a([&](double u, double w) {
                    const double du = u - P.dcx, dw = w - P.dcy;
                    return __fma_rn(du, du, __dmul_rn(dw, dw)) < P.dr2;
                }, std::true_type{});
            } else if constexpr (kMode == 1) {
                phase_a([&](double u, double w) {
                    const double du = fabs(u - P.ocx), dw = fabs(w - P.ocy);
                    return (du < P.ohx) & (dw < P.ohy) & (du + dw < P.od);
                }, std::true_type{});
            } else {
                phase_a([](double, double) { return false; }, std::true_type{});
            }
            // phase C: the chord test for the rest, 32 at a time
            uint32_t sn = 0;
            auto chord_round = [&](uint32_t idx, bool valid) {
                const double u = ring.x[s][xoff + idx], w = ring.y[s][yoff + idx];
                bool keep = false;
                if (valid) {
                    bad |= uint32_t(nonfinite_bits(u) | nonfinite_bits(w));
                    bool drop = filter;
#pragma unroll
                    for (int q = 0; q < kPolyV; ++q)  // inside by the margin w.r.t. every chord
                        drop &= __fma_rn(P.fa[q], u, __dmul_rn(P.fb[q], w)) < P.fg[q];
                    keep = !drop;
                }
                const unsigned b = __ballot_sync(kFull, keep);
                if (keep) {
                    s_surv[par][warp][sn + __popc(b & lt)] = uint16_t(idx);
                    // the full (x, y, index) order only for a possible new extreme
                    // (lo/hi start at x = +-inf, so the first survivor enters)
                    if (u <= lo.x) {
                        const ExtKey c{u, w, tbase + idx, 1u};
                        if (lo_better(c, lo)) lo = c;
                    }
                    if (u >= hi.x) {
                        const ExtKey c{u, w, tbase + idx, 1u};
                        if (hi_better(c, hi)) hi = c;
                    }
                    // only whether it exceeds 2^12 M matters (the unsafe flag)
                    if ((fabs(u) > alim) | (fabs(w) > alim)) amax = kInf;
                }
                sn += __popc(b);
            };
            __syncwarp();
            for (uint32_t r0 = 0; r0 < qn; r0 += 32) {
                const uint32_t j = r0 + lane;
                chord_round(j < qn ? s_q[warp][j] : 0u, j < qn);
            }
            if (lane == 0) s_cnt[par][warp] = sn;
            named_arrive<1>(par, kCtlThreads);
            if (k >= 1) store_tile(k - 1, sn_prev);
            sn_prev = sn;
        }
        if (nt >= 1) store_tile(nt - 1, sn_prev);
        };
        if (mode == 3u) tiles(std::integral_constant<int, 3>{});
        else if (mode == 2u) tiles(std::integral_constant<int, 2>{});
        else if (mode == 1u) tiles(std::integral_constant<int, 1>{});
        else tiles(std::integral_constant<int, 0>{});
    }
    // CTA partial -> the last CTA folds them and writes p, q and the slot
    uint32_t nb = bad;
    filter_warp_fold(lo, hi, amax, nb);
    if (lane == 0) {
        s_w[warp].lo = lo; s_w[warp].hi = hi; s_w[warp].amax = amax; s_w[warp].nonfinite = nb;
    }
    __syncthreads();
    FilterPartial* part = static_cast<FilterPartial*>(a.part);
    if (threadIdx.x == 0) {
        for (int w = 1; w < kCtlThreads / 32; ++w) {
            if (lo_better(s_w[w].lo, lo)) lo = s_w[w].lo;
            if (hi_better(s_w[w].hi, hi)) hi = s_w[w].hi;
            amax = fmax(amax, s_w[w].amax);
            nb |= s_w[w].nonfinite;
        }
        part[blockIdx.x].lo = lo; part[blockIdx.x].hi = hi;
        part[blockIdx.x].amax = amax; part[blockIdx.x].nonfinite = nb;
        __threadfence();
        s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    lo = ExtKey{0.0, 0.0, kNoIdx, 0u};
    hi = lo;
    amax = 0.0;
    nb = 0;
    for (uint32_t c = threadIdx.x; c < gridDim.x; c += blockDim.x) {
        const FilterPartial* p = &part[c];
        ExtKey x, h;
        x.x = __ldcg(&p->lo.x); x.y = __ldcg(&p->lo.y); x.idx = __ldcg(&p->lo.idx); x.valid = __ldcg(&p->lo.valid);
        h.x = __ldcg(&p->hi.x); h.y = __ldcg(&p->hi.y); h.idx = __ldcg(&p->hi.idx); h.valid = __ldcg(&p->hi.valid);
        if (lo_better(x, lo)) lo = x;
        if (hi_better(h, hi)) hi = h;
        amax = fmax(amax, __ldcg(&p->amax));
        nb |= __ldcg(&p->nonfinite);
    }
    filter_warp_fold(lo, hi, amax, nb);
    __syncthreads();  // s_w reuse
    if (lane == 0) {
        s_w[warp].lo = lo; s_w[warp].hi = hi; s_w[warp].amax = amax; s_w[warp].nonfinite = nb;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int w = 1; w < kCtlThreads / 32; ++w) {
        if (lo_better(s_w[w].lo, lo)) lo = s_w[w].lo;
        if (hi_better(s_w[w].hi, hi)) hi = s_w[w].hi;
        amax = fmax(amax, s_w[w].amax);
        nb |= s_w[w].nonfinite;
    }
    const uint32_t s = *reinterpret_cast<volatile uint32_t*>(a.ctr);
    RootInfo& R = *a.root_w;
    RootPoly& Pw = R.poly;
    const bool unsafe = P.filter != 0 && !(amax <= 0x1p12 * P.mref);
    R.p_idx = lo.idx; R.px = lo.x; R.py = lo.y;
    R.q_idx = hi.idx; R.qx = hi.x; R.qy = hi.y;
    R.cnt1 = s; R.cnt2 = 0;
    R.nonfinite = nb;
    R.unsafe = unsafe ? 1u : 0u;
    Pw.nv = 1;  // output frame: [p] chain(slot 0)
    Pw.ex[0] = lo.x; Pw.ey[0] = lo.y; Pw.eidx[0] = lo.idx;
    ChildRec ch;
    ch.px = lo.x; ch.py = lo.y;
    ch.rx = hi.x; ch.ry = hi.y;  // apex q
    ch.qx = lo.x; ch.qy = lo.y;
    ch.begin = 0;
    const bool degenerate = !lo.valid || (lo.x == hi.x && lo.y == hi.y);
    ch.m = (degenerate || nb || unsafe) ? 0u : s;
    ch.r_idx = hi.idx;
    a.slot[0] = ch;
    *a.ctr = 0;  // re-arm for the next call
    *a.ticket = 0;
    VQB_STAMP(g_strace[6] = gtimer_ns();)
}

// ===========================================================================
// K2 for levels of many small segments (deep levels of circle-like inputs:
// thousands of segments of a few tiles each): one CTA owns whole segments.
// With no other CTA on the segment there is nothing to claim, publish or
// reduce across CTAs: output places are running per-class counts (class 0
// forward from the range start, class 1 backward from its end — the
// two-sided layout), the farthest point of each class is the CTA's own
// running best, and the CTA writes the two children itself
// (hull.cpp:95-112).  Classification and order exactly as level_tma.
// ===========================================================================
constexpr uint32_t kSegCtaTiles = 4;

struct SegCtaSmem {
    uint32_t wc[2][2][kWarps];               // counts per (tile parity, class, warp)
    unsigned long long rkey[2][2][kWarps];   // warp winners per (segment parity, class, warp)
    uint32_t ridx[2][2][kWarps];
};

// ===========================================================================
// K2 fast mode with a TMA ring (8 compute warps + 1 control warp).  The
// control warp's lane 0 maps each upcoming tile of the CTA to its segment and
// streams x, y and the indices into a kRing-deep shared-memory ring with
// cp.async.bulk (segment starts are arbitrary: the copy starts at the
// 16-byte-aligned element below and the consumer skips the head; buffers
// carry a small tail pad).  Per tile the control warp scans the warp counts
// and claims the tile's places in the segment's two child ranges with one
// packed atomic while the compute warps update the running arg-max.
// ===========================================================================
struct LevelRing {
    double x[kRing][kTile + 2];
    double y[kRing][kTile + 2];
    uint32_t id[kRing][kTile + 4];
    unsigned long long bar[kRing];
    SegRec seg[kRing];
    uint32_t k[kRing];
    uint32_t cnt[kRing];
    uint32_t dx[kRing];
    uint32_t di[kRing];
};

// Planner-free host levels: the warp that writes a finished segment's child
// slot s also plans it for the next level (what planner_body does for a whole
// level, kernels.cu): its kind; an internal child gets a SegRec, fresh
// per-segment counters and its entries of the tile -> segment map, a finisher
// child a FinRec with its chain position, a leaf is counted.  Places in the
// next level's tables come from atomics on its LevelInfo (their order is free:
// the output ranges of internal segments are disjoint either way), so the
// host launches no planner and no tile-map kernel between levels.  Lane 0
// holds ch; every lane of the warp calls.
__device__ __forceinline__ void plan_child(const LevelArgs& a, uint64_t s, const ChildRec& ch) {
    const int lane = threadIdx.x & 31;
    uint32_t j = 0, t0 = 0, ntl = 0;
    if (lane == 0) {
        const uint32_t m = ch.m;
        const uint8_t kd = kind_of(m);
        a.n_kind[s] = kd;
        if (kd == kInternal) {
            ntl = (m + kTile - 1) / kTile;
            {  // one packed atomic for the segment's index and its first tile
                const uint2 c2 = claim_pair(reinterpret_cast<unsigned long long*>(&a.n_info->nseg), 1u, ntl);
                j = c2.x;
                t0 = c2.y;
            }
            const uint32_t out = atomicAdd(&a.n_info->out_total, m);
            SegRec g;
            g.px = ch.px; g.py = ch.py; g.rx = ch.rx; g.ry = ch.ry; g.qx = ch.qx; g.qy = ch.qy;
            g.bx = ch.rx; g.by = ch.ry;
            g.adx = dsub(ch.rx, ch.px); g.ady = dsub(ch.ry, ch.py);  // EdgeFrame::make (kernels.hpp:23-25)
            g.bdx = dsub(ch.qx, ch.rx); g.bdy = dsub(ch.qy, ch.ry);
            g.begin = ch.begin;
            g.out = out;
            g.m = m;
            g.tile0 = t0;
            g.ntiles = ntl;
            g.slot = uint32_t(s);
            a.n_segs[j] = g;
            a.n_seg_pcnt[j] = 0;
            a.n_seg_done[j] = 0;
            a.n_seg_ctr[j] = 0ull;
            a.n_link[s] = j;
        } else if (kd == kFin) {
            uint32_t f, before;  // its place in the list, the finisher points planned before it
            if (m <= kFinSmall) {
                f = atomicAdd(&a.n_info->nfin, 1u);
                before = atomicAdd(&a.n_info->fin_total, m);
            } else {  // one packed atomic for both
                const uint2 c2 = claim_pair(reinterpret_cast<unsigned long long*>(&a.n_info->fin_total), m, 1u);
                before = c2.x;
                f = a.n_fin_cap - 1u - c2.y;
            }
            FinRec fr;
            fr.c = ch;
            fr.chain_base = uint64_t(a.info->fin_base) + a.info->fin_total + before;
            fr.slot = uint32_t(s);
            fr.pad = 0;
            a.n_fins[f] = fr;
            a.n_link[s] = f;
        } else {
            if (kd == kLeaf) atomicAdd(&a.n_info->nleaf, 1u);
            a.n_link[s] = 0;
        }
    }
    j = __shfl_sync(kFull, j, 0);
    t0 = __shfl_sync(kFull, t0, 0);
    ntl = __shfl_sync(kFull, ntl, 0);
    for (uint32_t t = lane; t < ntl; t += 32) a.n_tile_seg[t0 + t] = j;
}

// block 0 at the start of a planner-free level: the next level's slot count
// and chain base; the level after it starts from zero counters
__device__ __forceinline__ void plan_level_start(const LevelArgs& a) {
    if (!a.n_kind || blockIdx.x != 0) return;
    if (threadIdx.x < sizeof(LevelInfo) / 4) reinterpret_cast<uint32_t*>(a.nn_info)[threadIdx.x] = 0u;
    if (threadIdx.x == 0) {
        a.n_info->nslots = 2u * a.info->nseg;
        a.n_info->fin_base = a.info->fin_base + a.info->fin_total;
    }
}

// Segment-per-CTA levels, fed by the TMA ring: the control warp walks the
// CTA's segments (k = blockIdx.x, + gridDim.x, ...) tile by tile and keeps
// kRing tiles in flight, so the next segment's points are already in shared
// memory when the current one ends (a CTA owns 2-4 tiles per segment on
// these levels; unprefetched, every tile exposed a full load latency).
template <bool GENERAL>
__device__ __forceinline__ void level_segcta_tma(const LevelArgs& a, uint32_t nseg, LevelRing& ring,
                                                 SegCtaSmem& S) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool ctl = tid >= kThreads;
    const uint32_t G = gridDim.x;
    uint32_t it_k = blockIdx.x, it_j = 0;  // control lane: next (segment, tile) to load
    auto issue_next = [&](uint32_t n) {     // CTA-local tile n -> stage n % kRing
        if (it_k >= nseg) return;
        const int st = int(n % kRing);
        const SegRec& g = a.segs[it_k];
        const uint32_t m = g.m, ntl = g.ntiles;
        const uint32_t start = uint32_t(g.begin) + it_j * uint32_t(kTile);
        const uint32_t cnt = min(uint32_t(kTile), m - it_j * uint32_t(kTile));
        const uint32_t ax = start & ~1u, dx = start - ax;
        const uint32_t ai = start & ~3u, di = start - ai;
        const uint32_t bx = ((cnt + dx + 1u) & ~1u) * 8u;
        const uint32_t bi = ((cnt + di + 3u) & ~3u) * 4u;
        VQB_CHECK(uint64_t(ax) * 8 + bx <= a.in_cap * 8 && uint64_t(ai) * 4 + bi <= a.in_cap * 4, 24, start, cnt);
        ring.cnt[st] = cnt;
        ring.dx[st] = dx;
        ring.di[st] = di;
        mbar_expect_tx(&ring.bar[st], 2u * bx + bi);
        tma_load_1d(ring.x[st], a.ix + ax, bx, &ring.bar[st]);
        tma_load_1d(ring.y[st], a.iy + ax, bx, &ring.bar[st]);
        tma_load_1d(ring.id[st], a.iid + ai, bi, &ring.bar[st]);
        if (++it_j == ntl) {
            it_j = 0;
            it_k += G;
        }
    };
    if (tid == kThreads) {
        for (int st = 0; st < kRing; ++st) mbar_init(&ring.bar[st], 1);
        mbar_fence_init();
        for (uint32_t n = 0; n < uint32_t(kRing); ++n) issue_next(n);
    }
    __syncthreads();
    uint32_t n = 0;  // CTA-local tile counter (every thread)
    int sp = 0;      // parity of the CTA-local segment counter
    for (uint32_t k = blockIdx.x; k < nseg; k += G, sp ^= 1) {
        const SegRec g = a.segs[k];
        const double px = g.px, py = g.py, rx = g.rx, ry = g.ry, qx = g.qx, qy = g.qy;
        const double adx = g.adx, ady = g.ady, bdx = g.bdx, bdy = g.bdy;
        unsigned long long kb[2] = {kNoKey, kNoKey};
        uint32_t ib[2] = {kNoIdx, kNoIdx};
        uint32_t run0 = 0, run1 = 0;  // CTA-uniform running class counts
        for (uint32_t j = 0; j < g.ntiles; ++j, ++n) {
            const int st = int(n % kRing);
            int cls[kItems];
            double ux[kItems], uy[kItems];
            uint32_t uid[kItems], rk[kItems];
            if (!ctl) {
                const uint32_t cnt = ring.cnt[st], dx = ring.dx[st], di = ring.di[st];
                mbar_wait(&ring.bar[st], (n / kRing) & 1u);
                uint32_t wrun = 0;
#pragma unroll
                for (int i = 0; i < kItems; ++i) {
                    const uint32_t r = uint32_t(i) * kThreads + tid;
                    const bool v = r < cnt;
                    const double u = ring.x[st][dx + r], w = ring.y[st][dx + r];
                    ux[i] = u;
                    uy[i] = w;
                    uid[i] = ring.id[st][di + r];
                    bool la, lb;
                    if (GENERAL) {
                        la = left_diff(dsub(px, u), dsub(py, w), dsub(rx, u), dsub(ry, w));
                        lb = !la && left_diff(dsub(g.bx, u), dsub(g.by, w), dsub(qx, u), dsub(qy, w));
                    } else {
                        const double A = dsub(px, u), B = dsub(py, w);
                        const double E = dsub(rx, u), F = dsub(ry, w);
                        const double Cc = dsub(qx, u), D = dsub(qy, w);
                        la = left_diff(A, B, E, F);
                        lb = !la && left_diff(E, F, Cc, D);
                    }
                    const int c = !v ? 2 : (la ? 0 : (lb ? 1 : 2));
                    cls[i] = c;
                    rk[i] = warp_rank<2>(c, wrun);
                    const unsigned long long key = key_of(lat_off(c == 0 ? adx : bdx, c == 0 ? ady : bdy, u, w));
                    running_best<2>(kb, ib, c, key, uid[i], a.gx, a.gy);
                }
                if (lane < 2) S.wc[n & 1][lane][warp] = wrun;
            }
            // The tile's only CTA barrier: counts posted; the stage's points
            // are in registers.  Every warp then scans the 2 x 8 counts itself
            // (the counts are double-buffered by tile parity: a warp is at
            // most one tile ahead of another).
            __syncthreads();
            if (ctl) {
                if (lane == 0) {
                    fence_proxy_async_smem();
                    issue_next(n + kRing);  // refill this stage
                }
            } else {
                const int c16 = (lane >> 3) & 1, w8 = lane & 7;
                const uint32_t v = lane < 16 ? S.wc[n & 1][c16][w8] : 0u;
                uint32_t incl = v;
#pragma unroll
                for (int d = 1; d < kWarps; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(kFull, incl, d, kWarps);
                    if (w8 >= d) incl += o;
                }
                const uint32_t ex0 = __shfl_sync(kFull, incl - v, warp);
                const uint32_t ex1 = __shfl_sync(kFull, incl - v, kWarps + warp);
                const uint32_t tot0 = __shfl_sync(kFull, incl, kWarps - 1);
                const uint32_t tot1 = __shfl_sync(kFull, incl, 2 * kWarps - 1);
#pragma unroll
                for (int i = 0; i < kItems; ++i) {
                    const int c = cls[i];
                    if (c < 2) {
                        const uint32_t off = (c ? run1 + ex1 : run0 + ex0) + rk[i];
                        const uint64_t pos = c ? g.out + g.m - 1u - off : g.out + off;
                        VQB_CHECK(pos < a.out_cap, 16, pos, a.out_cap);
                        a.ox[pos] = ux[i];
                        a.oy[pos] = uy[i];
                        a.oid[pos] = uid[i];
                    }
                }
                run0 += tot0;
                run1 += tot1;
            }
        }
        // the segment's two children (farthest point: block reduction; the
        // warp winners are double-buffered by segment parity, so the next
        // segment starts without a second barrier)
        for (int c = 0; c < 2; ++c) {
            unsigned long long kk = kb[c];
            uint32_t ii = ib[c];
            if (!ctl) warp_key_best(kk, ii, a.gx, a.gy);
            if (lane == 0 && !ctl) {
                S.rkey[sp][c][warp] = kk;
                S.ridx[sp][c][warp] = ii;
            }
        }
        __syncthreads();
        if (warp < 2) {
            const int c = warp;
            ChildRec ch;
            if (lane == 0) {
                unsigned long long ko = S.rkey[sp][c][0];
                uint32_t io = S.ridx[sp][c][0];
                for (int w = 1; w < kWarps; ++w) {
                    const unsigned long long kk = S.rkey[sp][c][w];
                    const uint32_t ii = S.ridx[sp][c][w];
                    if (kk < ko || (kk == ko && key_better(kk, ii, ko, io, a.gx, a.gy))) {
                        ko = kk;
                        io = ii;
                    }
                }
                const Best b = best_from_key(ko, io, c == 0 ? adx : bdx, c == 0 ? ady : bdy, a.gx, a.gy);
                const uint32_t m = c == 0 ? run0 : run1;
                if (c == 0) {  // left of p->r: triangle (p, rL, r)
                    ch.px = g.px; ch.py = g.py; ch.qx = g.rx; ch.qy = g.ry;
                    ch.begin = g.out;
                } else {       // left of r->q: triangle (r, rR, q)
                    ch.px = GENERAL ? g.bx : g.rx; ch.py = GENERAL ? g.by : g.ry;
                    ch.qx = g.qx; ch.qy = g.qy;
                    ch.begin = g.out + g.m - m;
                }
                ch.rx = b.x;
                ch.ry = b.y;
                ch.r_idx = b.idx;
                ch.m = m;
                VQB_CHECK(2 * uint64_t(k) + c < a.children_cap, 58, k, a.children_cap);
                a.children[2 * uint64_t(k) + c] = ch;
            }
            if (a.n_kind) plan_child(a, 2 * uint64_t(k) + c, ch);
        }
    }
}

#ifndef VQB_LEVEL_MINB
#define VQB_LEVEL_MINB 3
#endif
template <bool GENERAL>
__global__ void __launch_bounds__(kCtlThreads, VQB_LEVEL_MINB) level_tma(LevelArgs a) {
    VQB_PDL();
    plan_level_start(a);
    {
        // (-DVQB_SEGCTA) many small segments (at most kSegCtaTiles tiles on
        // average): one CTA per segment, no cross-CTA claims or partials
        // (uniform branch).  Off by default since the wide path lost its third
        // barrier per tile: compiled into the same kernel the second path costs
        // the first one its registers (168 B of spills), and alone the wide path
        // is faster on every input measured (profiles/r02_ncu_summary.md).
        const uint32_t nseg = a.info->nseg, nt = a.info->ntiles;
#ifdef VQB_SEGCTA
        if (nseg >= gridDim.x && nt <= kSegCtaTiles * nseg) {
            __shared__ SegCtaSmem SC;
            extern __shared__ __align__(128) unsigned char dsm_sc[];
            level_segcta_tma<GENERAL>(a, nseg, *reinterpret_cast<LevelRing*>(dsm_sc), SC);
            return;
        }
#else
        (void)nseg; (void)nt;
#endif
    }
    extern __shared__ __align__(128) unsigned char dsm[];
    LevelRing& ring = *reinterpret_cast<LevelRing*>(dsm);
    __shared__ FastSmem S;
    __shared__ SegRec s_cur;
    __shared__ uint32_t s_org[2][kWarps];
    __shared__ Best s_run[2];
    __shared__ bool s_last;
    __shared__ uint32_t s_ntiles;
    const bool ctl = threadIdx.x >= kThreads;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t G = gridDim.x;
    auto issue = [&](uint32_t kk) {  // control lane: local tile kk -> stage kk % kRing
        // contiguous chunks of tiles per CTA: consecutive tiles of a CTA
        // mostly share a segment (one partial per segment visit, not per tile)
        const uint32_t chunk = (s_ntiles + G - 1) / G;
        const uint32_t t = blockIdx.x * chunk + kk;
        if (t >= s_ntiles || kk >= chunk) return;
        const int s = int(kk % kRing);
        const uint32_t sk = a.tile_seg[t];
        const SegRec g = a.segs[sk];
        const uint32_t j = t - g.tile0;
        const uint32_t start = uint32_t(g.begin) + j * uint32_t(kTile);
        const uint32_t cnt = min(uint32_t(kTile), g.m - j * uint32_t(kTile));
        const uint32_t ax = start & ~1u, dx = start - ax;
        const uint32_t ai = start & ~3u, di = start - ai;
        const uint32_t bx = ((cnt + dx + 1u) & ~1u) * 8u;
        const uint32_t bi = ((cnt + di + 3u) & ~3u) * 4u;
        VQB_CHECK(uint64_t(ax) * 8 + bx <= a.in_cap * 8 && uint64_t(ai) * 4 + bi <= a.in_cap * 4, 23, start, cnt);
        ring.seg[s] = g;
        ring.k[s] = sk;
        ring.cnt[s] = cnt;
        ring.dx[s] = dx;
        ring.di[s] = di;
        mbar_expect_tx(&ring.bar[s], 2u * bx + bi);
        tma_load_1d(ring.x[s], a.ix + ax, bx, &ring.bar[s]);
        tma_load_1d(ring.y[s], a.iy + ax, bx, &ring.bar[s]);
        tma_load_1d(ring.id[s], a.iid + ai, bi, &ring.bar[s]);
    };
    if (threadIdx.x == kThreads) {
        s_ntiles = a.info->ntiles;
        for (int s = 0; s < kRing; ++s) mbar_init(&ring.bar[s], 1);
        mbar_fence_init();
        for (uint32_t kk = 0; kk < kRing; ++kk) issue(kk);
    }
    __syncthreads();
    const uint32_t ntiles = s_ntiles;
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    double bo[2] = {kInf, kInf};
    uint32_t bi[2] = {kNoIdx, kNoIdx};

    // the current segment and the CTA's tile count in it: every thread keeps
    // them (they follow the same tile sequence), so a new tile needs no
    // snapshot barrier
    uint32_t cur_k = 0xffffffffu, cur_tiles = 0;
    auto finalize = [&]() {
        // both classes' winners first, then their coordinates in one round
        // trip (they are random accesses to the input)
        // (both classes through one barrier: block_best_d twice was four)
        {
            unsigned long long k0 = bi[0] == kNoIdx ? kNoKey : key_of(bo[0]);
            unsigned long long k1 = bi[1] == kNoIdx ? kNoKey : key_of(bo[1]);
            uint32_t i0 = bi[0], i1 = bi[1];
            warp_key_best(k0, i0, a.gx, a.gy);
            warp_key_best(k1, i1, a.gx, a.gy);
            if (lane == 0 && warp < kWarps) {  // (the control warp holds no points)
                S.rkey[0][warp] = k0; S.ridx[0][warp] = i0;
                S.rkey[1][warp] = k1; S.ridx[1][warp] = i1;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t io[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                unsigned long long ko = S.rkey[c][0];
                io[c] = S.ridx[c][0];
                for (int w = 1; w < kWarps; ++w) {
                    const unsigned long long kk2 = S.rkey[c][w];
                    const uint32_t ii = S.ridx[c][w];
                    if (kk2 < ko || (kk2 == ko && key_better(kk2, ii, ko, io[c], a.gx, a.gy))) {
                        ko = kk2;
                        io[c] = ii;
                    }
                }
            }
            const uint32_t io0 = io[0], io1 = io[1];
            const double x0 = io0 != kNoIdx ? a.gx[io0] : 0.0, y0 = io0 != kNoIdx ? a.gy[io0] : 0.0;
            const double x1 = io1 != kNoIdx ? a.gx[io1] : 0.0, y1 = io1 != kNoIdx ? a.gy[io1] : 0.0;
            Best b0 = best_none(), b1 = best_none();
            if (io0 != kNoIdx) {
                b0.x = x0; b0.y = y0; b0.idx = io0; b0.valid = 1u;
                b0.off = lat_off(s_cur.adx, s_cur.ady, x0, y0);
            }
            if (io1 != kNoIdx) {
                b1.x = x1; b1.y = y1; b1.idx = io1; b1.valid = 1u;
                b1.off = lat_off(s_cur.bdx, s_cur.bdy, x1, y1);
            }
            s_run[0] = b0;
            s_run[1] = b1;
        }
        // A segment whose tiles were all this CTA's (the rule on deep levels:
        // a CTA's tiles are a contiguous chunk) needs no partials: the CTA's
        // own winners are the segment's, its own claims the final counts.
        const bool own = cur_tiles == s_cur.ntiles;  // (uniform)
        if (threadIdx.x == 0 && !own) {
            const uint32_t k = cur_k;
            const uint32_t slot = atomicAdd(&a.seg_pcnt[k], 1u);
            VQB_CHECK(slot < s_cur.ntiles && 2 * (uint64_t(s_cur.tile0) + slot) + 1 < a.part_cap,
                      50, slot, s_cur.ntiles);
            a.tile_part[2 * (uint64_t(s_cur.tile0) + slot)] = s_run[0];
            a.tile_part[2 * (uint64_t(s_cur.tile0) + slot) + 1] = s_run[1];
            __threadfence();
            const uint32_t done = atomicAdd(&a.seg_done[k], cur_tiles) + cur_tiles;
            s_last = (done == s_cur.ntiles);
        }
        __syncthreads();
        if (own || s_last) {
            if (!own) __threadfence();
            if (warp < 2) {
                const int c = warp;
                Best b = best_none();
                if (own) {
                    b = s_run[c];
                } else {
                    const uint32_t np = __ldcg(&a.seg_pcnt[cur_k]);
                    for (uint32_t jj = lane; jj < np; jj += 32) {
                        const Best o = ldcg_best(&a.tile_part[2 * (uint64_t(s_cur.tile0) + jj) + c]);
                        if (prefer(o, b)) b = o;
                    }
                    b = warp_best(b);
                }
                ChildRec ch;
                if (lane == 0) {
                    const SegRec& g = s_cur;
                    const uint2 w = read_pair(&a.seg_ctr[cur_k]);
                    const uint32_t m = c == 0 ? w.x : w.y;
                    if (c == 0) {  // left of p->r: triangle (p, rL, r)
                        ch.px = g.px; ch.py = g.py; ch.qx = g.rx; ch.qy = g.ry;
                        ch.begin = g.out;
                    } else {       // left of r->q: triangle (r, rR, q)
                        ch.px = GENERAL ? g.bx : g.rx; ch.py = GENERAL ? g.by : g.ry;
                        ch.qx = g.qx; ch.qy = g.qy;
                        ch.begin = g.out + g.m - m;
                    }
                    ch.rx = b.x;
                    ch.ry = b.y;
                    ch.r_idx = b.idx;
                    ch.m = m;
                    VQB_CHECK(2 * uint64_t(cur_k) + c < a.children_cap, 57, cur_k, a.children_cap);
                    a.children[2 * uint64_t(cur_k) + c] = ch;
                }
                if (a.n_kind) plan_child(a, 2 * uint64_t(cur_k) + c, ch);
            }
        }
        __syncthreads();
        bo[0] = bo[1] = kInf;
        bi[0] = bi[1] = kNoIdx;
    };

    // Lagged stores (as in the filter pass): tile k is classified while the
    // control warp claims its output ranges, and tile k-1 — classes and ranks
    // kept in shared memory, coordinates still in its ring stage — is stored
    // in the same interval, so the claim's L2 round trip never stalls the
    // compute warps; the stage is refilled once its stores are done.
    __shared__ uint16_t s_cr[2][kTile];          // class << 8 | rank in the (class, warp) run
    __shared__ uint32_t s_og[2][2][kWarps];      // output origins per (tile parity, class, warp)
    auto store_tile = [&](uint32_t kt) {         // compute warps: tile kt's points to their places
        const int st = int(kt % kRing), par = int(kt & 1);
        const uint32_t dx = ring.dx[st], di = ring.di[st];
        const int warp_ = threadIdx.x >> 5;
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const uint32_t r = uint32_t(i) * kThreads + threadIdx.x;
            const uint32_t v = s_cr[par][r];
            const uint32_t c = v >> 8, rk = v & 0xffu;
            if (c < 2) {
                const uint32_t o = s_og[par][c][warp_];
                const uint32_t p = c ? o - rk : o + rk;
                VQB_CHECK(p < a.out_cap, 13, p, a.out_cap);
                a.ox[p] = ring.x[st][dx + r];
                a.oy[p] = ring.y[st][dx + r];
                a.oid[p] = ring.id[st][di + r];
            }
        }
    };
    uint32_t kk = 0;
    const uint32_t chunk = (ntiles + G - 1) / G;
    const uint32_t t_end = min(ntiles, (blockIdx.x + 1) * chunk);
    for (uint32_t t = blockIdx.x * chunk; t < t_end; ++t, ++kk) {
        const int s = int(kk % kRing), par = int(kk & 1);
        // entering a new segment?  (ring.k[s] was written two barriers ago)
        const uint32_t k_now = ring.k[s];
        if (k_now != cur_k) {
            if (cur_k != 0xffffffffu) finalize();
            if (threadIdx.x == 0) s_cur = ring.seg[s];
            cur_k = k_now;
            cur_tiles = 0;
            __syncthreads();
        }
        if (!ctl) {
            const SegRec& g = ring.seg[s];
            const uint32_t cnt = ring.cnt[s], dx = ring.dx[s], di = ring.di[s];
            const double adx = g.adx, ady = g.ady, bdx = g.bdx, bdy = g.bdy;
            mbar_wait(&ring.bar[s], (kk / kRing) & 1u);
            const double px = g.px, py = g.py, rx = g.rx, ry = g.ry, qx = g.qx, qy = g.qy;
            uint32_t wrun = 0;
#pragma unroll
            for (int i = 0; i < kItems; ++i) {
                const uint32_t r = uint32_t(i) * kThreads + threadIdx.x;
                const bool v = r < cnt;
                const double u = ring.x[s][dx + r], w = ring.y[s][dx + r];
                bool la, lb;
                if (GENERAL) {
                    la = left_diff(dsub(px, u), dsub(py, w), dsub(rx, u), dsub(ry, w));
                    lb = !la && left_diff(dsub(g.bx, u), dsub(g.by, w), dsub(qx, u), dsub(qy, w));
                } else {
                    const double A = dsub(px, u), B = dsub(py, w);
                    const double E = dsub(rx, u), F = dsub(ry, w);
                    const double Cc = dsub(qx, u), D = dsub(qy, w);
                    la = left_diff(A, B, E, F);
                    lb = !la && left_diff(E, F, Cc, D);
                }
                const int c = !v ? 2 : (la ? 0 : (lb ? 1 : 2));
                const uint32_t rk = warp_rank<2>(c, wrun);
                s_cr[par][r] = uint16_t((uint32_t(c) << 8) | rk);
                // fused farthest-point search (kernels.hpp:41-45)
                running_best_d<2>(bo, bi, c, lat_off(c == 0 ? adx : bdx, c == 0 ? ady : bdy, u, w),
                                  ring.id[s][di + r], a.gx, a.gy);
            }
            if (lane < 2) S.wtot[lane][warp] = wrun;
        }
        __syncthreads();  // A: tile kk's counts and ranks posted
        if (ctl) {
            uint32_t tot[2];
            tile_scan_fast<2>(S, tot);
            if (lane == 0) {
                const uint2 c2 = claim_pair(&a.seg_ctr[k_now], tot[0], tot[1]);
                S.claim[0] = c2.x;
                S.claim[1] = c2.y;
            }
            __syncwarp();
            if (lane < 2 * kWarps) {
                const int c = lane / kWarps, w = lane % kWarps;
                const uint32_t out = uint32_t(ring.seg[s].out), m = ring.seg[s].m;
                const uint32_t off = S.claim[c] + S.wbase[c][w];
                const uint32_t org = c == 0 ? out : out + m - 1u;
                s_og[par][c][w] = c ? org - off : org + off;
            }
        } else if (kk >= 1) {
            store_tile(kk - 1);  // overlaps the claim of tile kk
        }
        __syncthreads();  // B: tile kk's origins published; tile kk-1 stored
        if (ctl && lane == 0 && kk >= 1) {
            fence_proxy_async_smem();
            issue(kk - 1 + kRing);  // refill tile kk-1's stage
        }
        ++cur_tiles;
    }
    if (kk >= 1 && !ctl) store_tile(kk - 1);
    if (cur_k != 0xffffffffu) finalize();
}

// ===========================================================================
// launchers (the stable mode is launched cooperatively: co-resident CTAs)
// ===========================================================================
cudaError_t launch_root_partition(const RootArgs& a, int grid, bool stable, cudaStream_t st) {
    if (!stable) {
        const bool aligned = ((reinterpret_cast<uintptr_t>(a.xs) | reinterpret_cast<uintptr_t>(a.ys)) & 15u) == 0;
        if (aligned && !getenv("VQB_NO_TMA")) {
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(root_partition_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(RootRing)));
                attr = true;
            }
            pdl_launch(root_partition_tma, grid, kCtlThreads, sizeof(RootRing), st, a);
        } else {
            pdl_launch(root_partition_fast<true>, grid, kThreads, 0, st, a);  // unaligned caller arrays
        }
        return cudaGetLastError();
    }
    void* args[] = {const_cast<RootArgs*>(&a)};
    return cudaLaunchCooperativeKernel((const void*)root_partition_kernel<true>, dim3(grid),
                                       dim3(kThreads), args, 0, st);
}

cudaError_t launch_root_filtered(const RootArgs& a, int grid, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(root_filtered_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(RootRing4)));
        attr = true;
    }
    pdl_launch(root_filtered_tma, grid, kCtlThreads, sizeof(RootRing4), st, a);
    return cudaGetLastError();
}

cudaError_t launch_root_filter(const FilterArgs& a, int grid, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(root_filter_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FilterRing)));
        cudaFuncSetAttribute(root_filter_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FilterRing)));
        attr = true;
    }
    if (a.xoff | a.yoff) pdl_launch(root_filter_tma<true>, grid, kCtlThreads, sizeof(FilterRing), st, a);
    else pdl_launch(root_filter_tma<false>, grid, kCtlThreads, sizeof(RootRing4), st, a);
    return cudaGetLastError();
}

int occupancy_filter() {
    int b = 0;
    int c = 0;
    cudaFuncSetAttribute(root_filter_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FilterRing)));
    cudaFuncSetAttribute(root_filter_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FilterRing)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, root_filter_tma<false>, kCtlThreads, sizeof(FilterRing));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, root_filter_tma<true>, kCtlThreads, sizeof(FilterRing));
    b = b < c ? b : c;
    return b;
}

size_t filter_partial_bytes(int grid) { return size_t(grid) * sizeof(FilterPartial); }

int occupancy_filtered() {
    int b = 0;
    cudaFuncSetAttribute(root_filtered_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(RootRing4)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, root_filtered_tma, kCtlThreads, sizeof(RootRing4));
    return b;
}

cudaError_t launch_level(const LevelArgs& a, bool general, bool stable, int grid, cudaStream_t st) {
    if (!stable && !getenv("VQB_NO_TMA")) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(level_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(LevelRing)));
            cudaFuncSetAttribute(level_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(LevelRing)));
            attr = true;
        }
        if (general) pdl_launch(level_tma<true>, grid, kCtlThreads, sizeof(LevelRing), st, a);
        else pdl_launch(level_tma<false>, grid, kCtlThreads, sizeof(LevelRing), st, a);
        return cudaGetLastError();
    }
    if (!stable) {
        if (general) pdl_launch(level_kernel<true, false>, grid, kThreads, 0, st, a);
        else pdl_launch(level_kernel<false, false>, grid, kThreads, 0, st, a);
        return cudaGetLastError();
    }
    void* args[] = {const_cast<LevelArgs*>(&a)};
    const void* fn = general ? (const void*)level_kernel<true, true> : (const void*)level_kernel<false, true>;
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, 0, st);
}

int occupancy_root(bool stable) {
    int b = 0, c = 0;
    if (stable) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, root_partition_kernel<true>, kThreads, 0);
        return b;
    }
    cudaFuncSetAttribute(root_partition_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(RootRing)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, root_partition_fast<true>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, root_partition_tma, kCtlThreads, sizeof(RootRing));
    return b < c ? b : c;  // one grid size serves both fast-path kernels
}
int occupancy_level(bool stable) {
    int m = 1 << 30, b = 0;
    if (stable) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, level_kernel<false, true>, kThreads, 0); m = b < m ? b : m;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, level_kernel<true, true>, kThreads, 0); m = b < m ? b : m;
    } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, level_kernel<false, false>, kThreads, 0); m = b < m ? b : m;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, level_kernel<true, false>, kThreads, 0); m = b < m ? b : m;
        cudaFuncSetAttribute(level_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(LevelRing)));
        cudaFuncSetAttribute(level_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(LevelRing)));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, level_tma<false>, kCtlThreads, sizeof(LevelRing)); m = b < m ? b : m;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, level_tma<true>, kCtlThreads, sizeof(LevelRing)); m = b < m ? b : m;
    }
    return m;
}

}  // namespace vqb
