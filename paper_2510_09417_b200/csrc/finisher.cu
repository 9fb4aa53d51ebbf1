// K3 batch finisher: whole recursion subtrees of every segment of at most
// kFinMax points (hull.cpp:78-115, chain_recursive, visited breadth-first;
// DESIGN.md §2.9), several segments per CTA.
//
// A CTA takes a BATCH of consecutive finisher segments whose points fit its
// kFbCap point slots and walks all their subtrees together, one depth per
// round.  A point never moves.  It keeps, in registers, its coordinates and
// the chord (p, q) of the node it currently belongs to; the node is NAMED by
// the slot of its apex r (every node has its own apex, so the name is unique
// and needs no numbering pass), and child s of node a is accumulator 2a + s —
// used at exactly one depth of one batch, so the accumulators are initialised
// once per batch and never reset.  Per depth:
//   (1) r = xy[node]; the reference's two orientation tests (left_diff,
//       kernels.hpp:28-30; mask_b &= ~mask_a, :91) pick the child; the chord
//       becomes (p, r) or (r, q); the point's farthest key for that chord (the
//       canonical order of kernels.hpp:41-45 as an order-preserving u64) goes
//       to the child's minimum (warp-reduced first when a warp shares a child);
//       a point in neither subset is dropped;
//   (2) the points holding their child's minimal key install themselves as
//       its apex; an exact tie falls to the smaller (x, y), then the smaller
//       input index (first occurrence) — a compare-and-swap on the apex word;
//   (3) every live point reads its child's apex: that is its next node, or
//       itself, in which case it is a hull vertex of this depth and retires.
// Two CTA barriers per depth, no scans, no per-node tables: the apex words
// ARE the tree (apex[2a + s] = apex of child s of node a).  Then subtree sizes
// bottom-up and chain positions top-down give chain(L) ++ [r] ++ chain(R)
// (assemble_chain, hull.cpp:59-73) for every segment of the batch.
// (The round-1/2 CTA finisher kept per-depth node tables, a block scan and six
// barriers per depth at one segment per CTA: 246 warp instructions per 32
// point-depths on circle 1e7; profiles/r02_finisher_bfs.md.)
#include "hull_types.cuh"

namespace vqb {

#ifndef VQB_FB_THREADS
#define VQB_FB_THREADS 256
#endif
#ifndef VQB_FB_ITEMS
#define VQB_FB_ITEMS 3
#endif
#ifndef VQB_FB_MINB
#define VQB_FB_MINB 4  // 64 registers (a few spilled words): 4 CTAs per SM beat 3 at 76 registers (1.27 -> 1.10 ms on circle 1e7)
#endif
constexpr int kFbThreads = VQB_FB_THREADS;
constexpr int kFbItems = VQB_FB_ITEMS;             // point slots per thread
constexpr int kFbCap = kFbThreads * kFbItems;      // point slots per batch
constexpr int kFbSegs = 32;                        // segments per batch (one warp plans a batch)
constexpr int kFbSlots = kFbCap + 3 * kFbSegs;     // + (p, q, r) of every segment
constexpr uint32_t kFbNone = 0xffffffffu;
static_assert(kFinMax <= uint32_t(kFbCap), "a finisher segment must fit one batch");
static_assert(kFbSlots < 32768, "positions are 16-bit");

struct FbSmem {
    double2 xy[kFbSlots];
    uint32_t gid[kFbSlots];
    union {
        unsigned long long ckey[2 * kFbSlots];  // per child: minimal key (during the walk)
        struct {
            uint16_t tsize[kFbSlots];           // per vertex: its subtree's chain length
            uint16_t tstart[kFbSlots];          // per vertex: where its subtree's chain starts
        } t;                                    // (emission)
    } u;
    uint32_t apex[2 * kFbSlots];                // per child: its apex slot (kFbNone: empty child)
    uint16_t vlist[kFbCap];                     // the vertices in the order they retired (by depth)
    uint16_t dstart[kFbCap + 2];                // first vlist entry of each depth
    uint8_t sseg[kFbCap];                       // per point slot: its segment in the batch
    uint32_t seg_off[kFbSegs + 1];              // first point slot of each segment
    uint32_t seg_fi[kFbSegs];                   // its FinRec
    uint32_t seg_begin[kFbSegs];                // its first point in the level's buffer
    uint64_t seg_chain[kFbSegs];                // where its chain goes
    uint32_t nb;                                // segments in this batch
    uint32_t nv;                                // vertices so far
};

// exact key tie: a strictly preferred over b
__device__ __forceinline__ bool fb_tie_better(const FbSmem& S, uint32_t a, uint32_t b) {
    const double2 A = S.xy[a], B = S.xy[b];
    if (A.x != B.x) return A.x < B.x;
    if (A.y != B.y) return A.y < B.y;
    return S.gid[a] < S.gid[b];
}

__device__ __forceinline__ uint32_t fb_size(const FbSmem& S, uint32_t a) {
    return a == kFbNone ? 0u : uint32_t(S.u.t.tsize[a]);
}

// one list of FinRecs (entries first, first + dir, ...; count of them), this
// CTA's contiguous share of it
__device__ __forceinline__ void fb_run_list(FbSmem& S, const FinRec* fins, int64_t first, int dir, uint32_t count,
                                            const double* __restrict__ ix, const double* __restrict__ iy,
                                            const uint32_t* __restrict__ iid, uint32_t* chain,
                                            uint32_t* fin_count) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned lt = lanemask_lt();
    uint32_t f = uint32_t(uint64_t(count) * blockIdx.x / gridDim.x);
    const uint32_t f_end = uint32_t(uint64_t(count) * (blockIdx.x + 1) / gridDim.x);
    while (f < f_end) {
        // ---- plan the batch (warp 0); fresh accumulators (the others)
        if (warp == 0) {
            const bool have = f + lane < f_end;
            const uint32_t fi = uint32_t(first + int64_t(dir) * int64_t(f + lane));
            const uint32_t m = have ? fins[fi].c.m : 0u;
            VQB_CHECK(!have || (m >= 1 && m <= kFinMax), 32, m, fi);
            uint32_t incl = m;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(kFull, incl, d);
                if (lane >= d) incl += o;
            }
            const unsigned fit = __ballot_sync(kFull, have && incl <= uint32_t(kFbCap));
            const uint32_t nb = uint32_t(__popc(fit));  // a prefix of the lanes (incl is monotone), >= 1
            if (lane < int(nb)) {
                const FinRec rec = fins[fi];
                S.seg_off[lane] = incl - m;
                S.seg_fi[lane] = fi;
                S.seg_begin[lane] = uint32_t(rec.c.begin);
                S.seg_chain[lane] = rec.chain_base;
                const int b = kFbCap + 3 * lane;
                S.xy[b] = make_double2(rec.c.px, rec.c.py);
                S.xy[b + 1] = make_double2(rec.c.qx, rec.c.qy);
                S.xy[b + 2] = make_double2(rec.c.rx, rec.c.ry);
                S.gid[b + 2] = rec.c.r_idx;
                if (lane == int(nb) - 1) {
                    S.seg_off[nb] = incl;
                    S.nb = nb;
                    S.nv = 0;
                }
            }
        }
        for (int i = tid; i < 2 * kFbSlots; i += kFbThreads) {
            S.u.ckey[i] = kNoKey;
            S.apex[i] = kFbNone;
        }
        __syncthreads();
        const uint32_t nb = S.nb;
        const uint32_t total = S.seg_off[nb];

        // ---- load: point slot i = k * kFbThreads + tid
        double u[kFbItems], w[kFbItems], px[kFbItems], py[kFbItems], qx[kFbItems], qy[kFbItems];
        unsigned long long key[kFbItems];
        uint32_t node[kFbItems];   // live: its node (the apex's slot), then its child; kFbNone: retired
#pragma unroll
        for (int k = 0; k < kFbItems; ++k) {
            const uint32_t i = uint32_t(k) * kFbThreads + tid;
            node[k] = kFbNone;
            u[k] = w[k] = px[k] = py[k] = qx[k] = qy[k] = 0.0;
            if (i < total) {
                uint32_t lo = 0, hi = nb;  // segment: seg_off[lo] <= i < seg_off[lo + 1]
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (S.seg_off[mid] <= i) lo = mid; else hi = mid;
                }
                const uint32_t src = S.seg_begin[lo] + (i - S.seg_off[lo]);
                u[k] = ix[src];
                w[k] = iy[src];
                S.gid[i] = iid[src];
                S.xy[i] = make_double2(u[k], w[k]);
                const int b = kFbCap + 3 * int(lo);
                const double2 P = S.xy[b], Q = S.xy[b + 1];
                px[k] = P.x; py[k] = P.y; qx[k] = Q.x; qy[k] = Q.y;
                node[k] = uint32_t(b + 2);
                S.sseg[i] = uint8_t(lo);
            }
        }
        __syncthreads();

        // ---- the walk
        uint32_t depth = 0;
        for (;;) {
            bool any = false;
            // (1) classify; the child's minimal key
#pragma unroll
            for (int k = 0; k < kFbItems; ++k) {
                key[k] = kNoKey;
                if (node[k] == kFbNone) continue;
                const double2 R = S.xy[node[k]];
                const double A = dsub(px[k], u[k]), B = dsub(py[k], w[k]);
                const double E = dsub(R.x, u[k]), F = dsub(R.y, w[k]);
                const double Cc = dsub(qx[k], u[k]), D = dsub(qy[k], w[k]);
                const bool la = left_diff(A, B, E, F);
                const bool lb = !la && left_diff(E, F, Cc, D);
                if (la) {
                    qx[k] = R.x; qy[k] = R.y;
                } else if (lb) {
                    px[k] = R.x; py[k] = R.y;
                } else {
                    node[k] = kFbNone;
                    continue;
                }
                node[k] = 2u * node[k] + (lb ? 1u : 0u);  // its child, until (3)
                // EdgeFrame::make of the child's chord (kernels.hpp:23-25), lateral offset (:32-34)
                key[k] = key_of(lat_off(dsub(qx[k], px[k]), dsub(qy[k], py[k]), u[k], w[k]));
                any = true;
            }
#pragma unroll
            for (int k = 0; k < kFbItems; ++k) {
                const uint32_t c = node[k];
                const uint32_t c0 = __shfl_sync(kFull, c, 0);
                if (__all_sync(kFull, c == c0)) {  // the whole warp in one child (the top of a subtree), or retired
                    if (c0 != kFbNone) {
                        const uint32_t hi = uint32_t(key[k] >> 32);
                        const uint32_t mh = __reduce_min_sync(kFull, hi);
                        const uint32_t ml = __reduce_min_sync(kFull, hi == mh ? uint32_t(key[k]) : 0xffffffffu);
                        const unsigned long long mk = (static_cast<unsigned long long>(mh) << 32) | ml;
                        if (lane == 0 && mk < S.u.ckey[c0]) atomicMin(&S.u.ckey[c0], mk);
                    }
                } else if (c != kFbNone) {
                    if (key[k] < S.u.ckey[c]) atomicMin(&S.u.ckey[c], key[k]);
                }
            }
            const bool go = __syncthreads_or(any);
            // every warp has appended the vertices of the depths before this
            // one, and none appends before the next barrier
            if (tid == 0) S.dstart[depth] = uint16_t(S.nv);
            if (!go) break;
            // (2) the holders of the minimal key: the child's apex
#pragma unroll
            for (int k = 0; k < kFbItems; ++k) {
                const uint32_t c = node[k];
                if (c == kFbNone || key[k] != S.u.ckey[c]) continue;
                const uint32_t me = uint32_t(k) * kFbThreads + tid;
                uint32_t cur = atomicCAS(&S.apex[c], kFbNone, me);
                while (cur != kFbNone && fb_tie_better(S, me, cur)) {
                    const uint32_t old = atomicCAS(&S.apex[c], cur, me);
                    if (old == cur) break;
                    cur = old;
                }
            }
            __syncthreads();
            // (3) next node, or retire as this depth's vertex
#pragma unroll
            unsigned retired[kFbItems];
            uint32_t nret = 0;
#pragma unroll
            for (int k = 0; k < kFbItems; ++k) {
                const uint32_t c = node[k];
                bool ret = false;
                if (c != kFbNone) {
                    const uint32_t a = S.apex[c];
                    ret = a == uint32_t(k) * kFbThreads + tid;
                    node[k] = ret ? kFbNone : a;
                }
                retired[k] = __ballot_sync(kFull, ret);
                nret += uint32_t(__popc(retired[k]));
            }
            if (nret) {  // (warp-uniform) this warp's new vertices join the list of their depth
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&S.nv, nret);
                base = __shfl_sync(kFull, base, 0);
#pragma unroll
                for (int k = 0; k < kFbItems; ++k) {
                    if (retired[k] & (1u << lane))
                        S.vlist[base + uint32_t(__popc(retired[k] & lt))] = uint16_t(uint32_t(k) * kFbThreads + tid);
                    base += uint32_t(__popc(retired[k]));
                }
            }
            ++depth;
            if (depth > uint32_t(kFbCap)) {  // cannot happen: every depth retires >= 1 point of <= kFbCap
                if (tid == 0) g_vqb_fault = 5u;
                break;
            }
        }
        // ---- emission (ckey is dead: every thread is past its last (2)).
        // Sizes bottom-up, then positions top-down, over each depth's vertices.
        __syncthreads();
        for (int d = int(depth) - 1; d >= 0; --d) {
            for (uint32_t i = S.dstart[d] + tid; i < S.dstart[d + 1]; i += kFbThreads) {
                const uint32_t v = S.vlist[i];
                S.u.t.tsize[v] = uint16_t(fb_size(S, S.apex[2 * v]) + 1u + fb_size(S, S.apex[2 * v + 1]));
            }
            __syncthreads();
        }
        if (tid < int(nb)) {  // the segments' own apexes: chain(S1) ++ [r] ++ chain(S2)
            const uint32_t me = uint32_t(kFbCap + 3 * tid + 2);
            const uint32_t L = S.apex[2 * me], R = S.apex[2 * me + 1];
            const uint32_t pos = fb_size(S, L);
            chain[S.seg_chain[tid] + pos] = S.gid[me];
            if (L != kFbNone) S.u.t.tstart[L] = 0;
            if (R != kFbNone) S.u.t.tstart[R] = uint16_t(pos + 1);
            fin_count[S.seg_fi[tid]] = pos + 1u + fb_size(S, R);
        }
        __syncthreads();
        for (uint32_t d = 0; d < depth; ++d) {
            for (uint32_t i = S.dstart[d] + tid; i < S.dstart[d + 1]; i += kFbThreads) {
                const uint32_t v = S.vlist[i];
                const uint32_t L = S.apex[2 * v], R = S.apex[2 * v + 1];
                const uint32_t s0 = S.u.t.tstart[v];
                const uint32_t pos = s0 + fb_size(S, L);
                chain[S.seg_chain[S.sseg[v]] + pos] = S.gid[v];
                if (L != kFbNone) S.u.t.tstart[L] = uint16_t(s0);
                if (R != kFbNone) S.u.t.tstart[R] = uint16_t(pos + 1);
            }
            __syncthreads();
        }
        f += nb;
    }
}

__global__ void __launch_bounds__(kFbThreads, VQB_FB_MINB) finisher_batch_kernel(const FinRec* fins, const LevelInfo* info,
                                                                    uint32_t fin_cap,
                                                                    const double* __restrict__ ix,
                                                                    const double* __restrict__ iy,
                                                                    const uint32_t* __restrict__ iid,
                                                                    uint32_t* chain, uint32_t* fin_count) {
    VQB_PDL();
    extern __shared__ __align__(16) unsigned char fb_dsm[];
    FbSmem& S = *reinterpret_cast<FbSmem*>(fb_dsm);
    // the large segments (listed from the back of the table), then the small ones
    fb_run_list(S, fins, int64_t(fin_cap) - 1, -1, info->nfin2, ix, iy, iid, chain, fin_count);
    fb_run_list(S, fins, 0, 1, info->nfin, ix, iy, iid, chain, fin_count);
}

void launch_finisher_batch(const FinRec* fins, const LevelInfo* info, uint32_t fin_cap, const double* ix,
                           const double* iy, const uint32_t* iid, uint32_t* chain, uint32_t* fin_count,
                           uint32_t nfin_hint, int max_grid, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(finisher_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FbSmem)));
        attr = true;
    }
    uint32_t g = nfin_hint;
    if (g < 1) g = 1;
    if (g > uint32_t(max_grid)) g = uint32_t(max_grid);
    pdl_launch(finisher_batch_kernel, g, kFbThreads, sizeof(FbSmem), st, fins, info, fin_cap, ix, iy, iid, chain,
               fin_count);
}

int occupancy_finisher_batch() {
    int b = 0;
    cudaFuncSetAttribute(finisher_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FbSmem)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, finisher_batch_kernel, kFbThreads, sizeof(FbSmem));
    return b;
}

}  // namespace vqb
