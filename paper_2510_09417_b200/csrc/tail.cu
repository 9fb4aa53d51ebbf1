// KT: the persistent recursion kernel (included by device.cu).
//
// After the split root, the recursion below the bootstrap triangle is a
// sequence of small levels on most inputs (square 1e8: ~60k survivors, six
// levels of 1..32 segments).  Run level by level as separate launches
// (planner, finisher, tile map, K2) those levels are pure latency: four
// launches and their global round trips per level.  KT runs the same
// per-level steps inside ONE cooperative launch with one CTA per SM slot:
//
//   CTA 0: plan level l (planner_body: slot kinds, segment / finisher tables,
//          tile offsets) and the tile -> segment map
//   grid barrier
//   all:   K2 tiles of every internal segment (level_body: fused f64
//          classification, two-sided compaction, farthest point; the CTA
//          completing a segment writes its two children = level l+1's slots)
//          + every finisher segment (finisher_all_body)
//   grid barrier; stop when level l had no internal segment
//
// The tables it writes are exactly the host-driven path's (level(l) slots,
// kinds, links, FinRecs, LevelInfo), so emission is unchanged and the host
// can resume the level loop where KT stops: KT bails out at the first level
// whose slot count exceeds max_slots (deep, wide recursions such as points on
// a circle), leaving that level's slots for the host-driven kernels.
// Reference: chain_recursive / chain_iterative (hull.cpp:78-190), one call per
// segment there; here one launch for all levels.
#include <cooperative_groups.h>

namespace vqb {

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// CTA 0, thread 0: timestamp of phase ph of level li (diagnostics)
#define KT_TRACE(li, ph)                                                      \
    do {                                                                      \
        if (A.trace && blockIdx.x == 0 && threadIdx.x == 0)                   \
            A.trace[1 + (li) * 10 + (ph)] = global_ns();                      \
    } while (0)

// Single-CTA planner for a level of at most kTailSlots slots: the same
// tables as planner_body (kinds, links, SegRec / FinRec, LevelInfo, reset
// per-segment counters) from one block-wide scan — no chunk claims, no
// look-back — and the tile -> segment map by binary search over the
// segments' first tiles in shared memory.
__device__ __noinline__ void tail_plan(const TailArgs& A, const TailLevel& T, uint32_t nslots,
                                       const LevelInfo* prev, LevelInfo* info, int li) {
    __shared__ PlanAgg s_w[kWarps];
    __shared__ PlanAgg s_tot;
    __shared__ uint32_t s_tile0[kTailSlots];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t fin_chain_base = prev ? uint64_t(prev->fin_base) + prev->fin_total : 0ull;
    // rounds of kThreads slots (slot k * kThreads + tid), one block scan each:
    // a small level is one round with at most one slot per thread
    PlanAgg carry;
    pl_clear(carry);
    const uint32_t rounds = (nslots + kThreads - 1) / kThreads;
    for (uint32_t k = 0; k < rounds; ++k) {
        const uint32_t s = k * kThreads + uint32_t(tid);
        ChildRec c;
        uint32_t m = 0;
        if (s < nslots) {
            c = T.slots[s];
            m = c.m;
        }
        const uint8_t kd = s < nslots ? kind_of_cap(m, A.fin_max) : kEmpty;
        PlanAgg mine;
        pl_clear(mine);
        mine.nseg = kd == kInternal;
        mine.nfin = kd == kFin && m <= kFinSmall;
        mine.nfin2 = kd == kFin && m > kFinSmall;
        mine.leaf = kd == kLeaf;
        mine.ntiles = kd == kInternal ? (m + kTile - 1) / kTile : 0;
        mine.out = kd == kInternal ? m : 0;
        mine.fin = kd == kFin ? m : 0;
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
        PlanAgg run = carry, tot = carry;
        for (int w = 0; w < kWarps; ++w) {
            if (w < warp) pl_combine(run, s_w[w]);
            pl_combine(tot, s_w[w]);
        }
        __syncthreads();  // s_w is rewritten by the next round
        PlanAgg wex = incl;  // exclusive within the warp
        wex.nseg -= mine.nseg; wex.nfin -= mine.nfin; wex.nfin2 -= mine.nfin2; wex.ntiles -= mine.ntiles;
        wex.out -= mine.out; wex.fin -= mine.fin; wex.leaf -= mine.leaf;
        pl_combine(run, wex);
        carry = tot;
        if (s >= nslots) continue;
        T.kind[s] = kd;
        if (kd == kInternal) {
            SegRec g;
            g.px = c.px; g.py = c.py; g.rx = c.rx; g.ry = c.ry; g.qx = c.qx; g.qy = c.qy;
            g.bx = c.rx; g.by = c.ry;
            g.adx = dsub(c.rx, c.px); g.ady = dsub(c.ry, c.py);  // EdgeFrame::make (kernels.hpp:23-25)
            g.bdx = dsub(c.qx, c.rx); g.bdy = dsub(c.qy, c.ry);
            g.begin = c.begin;
            g.out = run.out;
            g.m = c.m;
            g.tile0 = run.ntiles;
            g.ntiles = (c.m + kTile - 1) / kTile;
            g.slot = s;
            T.segs[run.nseg] = g;
            s_tile0[run.nseg] = run.ntiles;
            A.seg_pcnt[run.nseg] = 0;
            A.seg_done[run.nseg] = 0;
            A.seg_ctr[run.nseg] = 0ull;
            T.link[s] = run.nseg;
        } else if (kd == kFin) {
            FinRec f;
            f.c = c;
            f.chain_base = fin_chain_base + run.fin;
            f.slot = s;
            f.pad = 0;
            // warp-finisher segments from the front, CTA-finisher ones from the back
            const uint32_t fi = m <= kFinSmall ? run.nfin : kTailSlots - 1u - run.nfin2;
            T.fins[fi] = f;
            T.link[s] = fi;
        } else {
            T.link[s] = 0;
        }
    }
    KT_TRACE(li, 6);
    if (tid == 0) {
        s_tot = carry;
        LevelInfo lv;
        lv.nslots = nslots;
        lv.nseg = carry.nseg;
        lv.nfin = carry.nfin;
        lv.ntiles = carry.ntiles;
        lv.out_total = carry.out;
        lv.fin_total = carry.fin;
        lv.nleaf = carry.leaf;
        lv.fin_base = uint32_t(fin_chain_base);
        lv.nfin2 = carry.nfin2;
        lv.pad = 0;
        *info = lv;
    }
    __syncthreads();
    KT_TRACE(li, 7);
    const uint32_t nseg = s_tot.nseg, ntiles = s_tot.ntiles;
    for (uint32_t t = tid; t < ntiles; t += kThreads) {
        uint32_t lo = 0, hi = nseg;  // last k with tile0 <= t
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (s_tile0[mid] <= t) lo = mid; else hi = mid;
        }
        A.tile_seg[t] = lo;
    }
}

// In-kernel emission (CTA 0, after the last level): the same in-order chain
// assembly as size_kernel / poly_frame_kernel / emit_kernel (hull.cpp:59-73,
// 259-266) with every level's slot sizes and starts in shared memory, for
// trees of at most kTailEmitSlots slots.  Output = [p] chain(root slot).
constexpr uint32_t kTailEmitSlots = 4096;
struct TailEmitSmem {
    uint32_t sz[kTailEmitSlots];
    uint32_t st[kTailEmitSlots];
    uint32_t kl[kTailEmitSlots];  // kind << 30 | link
    uint32_t off[kTailLevels + 1];
    uint32_t total;
};
static_assert(sizeof(TailEmitSmem) <= sizeof(FinAllSmemT<kTailFinMax>), "emission reuses the finisher's shared memory");

// returns false (nothing written) when the tree is too large
__device__ __noinline__ bool tail_emit(const TailArgs& A, TailEmitSmem& E, int nl) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        uint32_t o = 0;
        for (int li = 0; li < nl; ++li) {
            E.off[li] = o;
            o += A.info[A.l0 + li].nslots;
        }
        E.off[nl] = o;
        E.total = o;
    }
    __syncthreads();
    const uint32_t total = E.total;
    if (total > kTailEmitSlots || E.off[1] != 1u) return false;  // split root: one root slot
    for (uint32_t i = tid; i < total; i += kThreads) {
        int li = 0;
        while (E.off[li + 1] <= i) ++li;
        const TailLevel& T = A.lv[li];
        const uint32_t s = i - E.off[li];
        const uint32_t k = T.kind[s];
        const uint32_t ln = T.link[s];
        E.kl[i] = (k << 30) | ln;
        E.sz[i] = k == kLeaf ? 1u : (k == kFin ? T.fin_count[ln] : (k == kInternal ? 1u : 0u));
    }
    __syncthreads();
    for (int li = nl - 2; li >= 0; --li) {  // bottom-up subtree sizes (the last level has no internal slot)
        for (uint32_t i = E.off[li] + tid; i < E.off[li + 1]; i += kThreads) {
            const uint32_t kl = E.kl[i];
            if ((kl >> 30) == kInternal) {
                const uint32_t c = E.off[li + 1] + 2u * (kl & 0x3fffffffu);
                E.sz[i] += E.sz[c] + E.sz[c + 1];
            }
        }
        __syncthreads();
    }
    if (tid == 0) {  // frame: [p] chain(root slot)  (hull.cpp:259-266)
        A.out[0] = *A.p_idx;
        E.st[0] = 1;
        *A.h_out = 1u + E.sz[0];
    }
    __syncthreads();
    for (int li = 0; li + 1 < nl; ++li) {  // top-down starts
        for (uint32_t i = E.off[li] + tid; i < E.off[li + 1]; i += kThreads) {
            const uint32_t kl = E.kl[i];
            if ((kl >> 30) == kInternal) {
                const uint32_t c = E.off[li + 1] + 2u * (kl & 0x3fffffffu);
                E.st[c] = E.st[i];
                E.st[c + 1] = E.st[i] + E.sz[c] + 1u;
            }
        }
        __syncthreads();
    }
    // writes: apexes of internal slots and leaves one per thread, finisher
    // chains one per warp
    for (uint32_t i = tid; i < total; i += kThreads) {
        const uint32_t kl = E.kl[i], k = kl >> 30;
        if (k != kLeaf && k != kInternal) continue;
        int li = 0;
        while (E.off[li + 1] <= i) ++li;
        const uint32_t s = i - E.off[li];
        uint32_t pos = E.st[i];
        if (k == kInternal) pos += E.sz[E.off[li + 1] + 2u * (kl & 0x3fffffffu)];
        A.out[pos] = A.lv[li].slots[s].r_idx;
    }
    for (uint32_t i = warp; i < total; i += kWarps) {
        const uint32_t kl = E.kl[i];
        if ((kl >> 30) != kFin) continue;
        int li = 0;
        while (E.off[li + 1] <= i) ++li;
        const uint32_t f = kl & 0x3fffffffu;
        const uint32_t c = E.sz[i];
        const uint64_t b = A.lv[li].fins[f].chain_base;
        for (uint32_t j = lane; j < c; j += 32) A.out[E.st[i] + j] = A.chain[b + j];
    }
    return true;
}

// CTA 0 at exit: everything the host needs in ONE contiguous copy — state,
// h, the root verdicts and every processed level's LevelInfo.
__device__ __noinline__ void tail_report(const TailArgs& A, int nl) {
    uint32_t* r = A.report;
    if (threadIdx.x == 0) {
        const RootInfo* R = A.root;
        r[0] = A.state[0];
        r[1] = A.state[1];
        r[2] = *A.h_out;
        r[3] = R->nonfinite;
        r[4] = R->unsafe;
        r[5] = R->poly.filter;
        r[6] = R->cnt1;
        r[7] = *reinterpret_cast<volatile uint32_t*>(&g_vqb_fault);  // (its own copy would cost a memcpy)
    }
    const uint32_t* src = reinterpret_cast<const uint32_t*>(A.info + A.l0);
    const uint32_t words = uint32_t(nl) * uint32_t(sizeof(LevelInfo) / 4);
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) r[8 + i] = src[i];
}

__global__ void __launch_bounds__(kThreads, 2) tail_kernel(const __grid_constant__ TailArgs A) {
    VQB_PDL();
    extern __shared__ __align__(16) unsigned char tl_dsm[];
    FinAllSmemT<kTailFinMax>& U = *reinterpret_cast<FinAllSmemT<kTailFinMax>*>(tl_dsm);
    __shared__ uint32_t s_flag;
    cg::grid_group grid = cg::this_grid();
    // the cluster recursion (cluster_tail.cu) ran just before and did everything
    if (A.kc_done && *reinterpret_cast<volatile uint32_t*>(A.kc_done)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        A.state[0] = uint32_t(A.l0);
        A.state[1] = 0u;
        if (A.trace) A.trace[0] = global_ns();
        VQB_STAMP(g_strace[7] = global_ns();)
    }
    int in = A.in0;  // the buffer level l0 reads
    for (int li = 0;; ++li) {
        const int l = A.l0 + li;
        const TailLevel& T = A.lv[li];
        LevelInfo* info = A.info + l;
        const LevelInfo* prev = li ? A.info + (l - 1) : A.prev0;
        KT_TRACE(li, 0);
        // ---- plan (CTA 0)
        if (blockIdx.x == 0) {
            if (threadIdx.x == 0) {
                const uint32_t ns = prev ? 2u * prev->nseg : A.nslots0;
                // the last table set is only for children: stop before it
                const bool bail = ns > A.max_slots || li + 1 >= A.nlev;
                s_flag = bail ? 1u : 0u;
                if (bail) {
                    A.state[0] = uint32_t(l);
                    A.state[1] = 2u;
                }
            }
            __syncthreads();
            if (!s_flag) {
                tail_plan(A, T, prev ? 2u * prev->nseg : A.nslots0, prev, info, li);
                // a level with many points runs better through the host-driven
                // TMA-ring kernel: hand it over (the host re-plans it)
                if (threadIdx.x == 0 && info->ntiles > A.max_tiles) {
                    A.state[0] = uint32_t(l);
                    A.state[1] = 2u;
                }
            }
        }
        KT_TRACE(li, 1);
        grid.sync();
        KT_TRACE(li, 2);
        if (threadIdx.x == 0) s_flag = *reinterpret_cast<volatile uint32_t*>(&A.state[1]);
        __syncthreads();
        if (s_flag == 2u) {
            if (blockIdx.x == 0) tail_report(A, li);
            return;
        }
        // ---- work: K2 tiles, then the finisher segments
        LevelArgs la = {};
        la.gx = A.gx;
        la.gy = A.gy;
        la.segs = T.segs;
        la.tile_seg = A.tile_seg;
        la.info = info;
        la.ix = A.bx[in];
        la.iy = A.by[in];
        la.iid = A.bid[in];
        la.ox = A.bx[in ^ 1];
        la.oy = A.by[in ^ 1];
        la.oid = A.bid[in ^ 1];
        la.in_cap = A.buf_cap;
        la.out_cap = A.buf_cap;
        la.status_cap = 0;
        la.part_cap = A.part_cap;
        la.children_cap = 2ull * A.max_slots;
        la.segs_cap = A.max_slots;
        la.status = nullptr;
        la.epoch = 0;
        la.ctr = nullptr;
        la.tile_part = A.tile_part;
        la.seg_pcnt = A.seg_pcnt;
        la.seg_done = A.seg_done;
        la.seg_ctr = A.seg_ctr;
        la.children = A.lv[li + 1].slots;
        level_body<false, false>(la);
        __syncthreads();
        KT_TRACE(li, 3);
        finisher_all_body(U, T.fins, info, A.max_slots, A.bx[in], A.by[in], A.bid[in], A.chain, T.fin_count);
        KT_TRACE(li, 4);
        grid.sync();
        KT_TRACE(li, 5);
        if (info->nseg == 0) {  // no internal segment: the recursion ended at this level
            if (blockIdx.x != 0) return;
            const bool emitted = A.out && tail_emit(A, *reinterpret_cast<TailEmitSmem*>(tl_dsm), li + 1);
            if (threadIdx.x == 0) {
                A.state[0] = uint32_t(l);
                A.state[1] = emitted ? 3u : 1u;
            }
            __syncthreads();
            tail_report(A, li + 1);
            return;
        }
        in ^= 1;
    }
}

size_t tail_smem_bytes() { return sizeof(FinAllSmemT<kTailFinMax>); }

int occupancy_tail() {
    int b = 0;
    cudaFuncSetAttribute(tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FinAllSmemT<kTailFinMax>)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tail_kernel, kThreads, sizeof(FinAllSmemT<kTailFinMax>));
    return b;
}

cudaError_t launch_tail(const TailArgs& a, int grid, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FinAllSmemT<kTailFinMax>)));
        attr = true;
    }
    // cooperative (grid barriers) and, where the driver accepts the pair,
    // programmatic stream serialization so the launch overlaps the filter
    // pass's tail (the kernel's griddepcontrol.wait orders the data)
    static int pdl_ok = pdl_enabled() ? 1 : 0;
    if (pdl_ok) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = sizeof(FinAllSmemT<kTailFinMax>);
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, tail_kernel, a);
        if (e == cudaSuccess) return e;
        (void)cudaGetLastError();
        pdl_ok = 0;
    }
    void* args[] = {const_cast<TailArgs*>(&a)};
    return cudaLaunchCooperativeKernel((const void*)tail_kernel, dim3(grid), dim3(kThreads), args,
                                       sizeof(FinAllSmemT<kTailFinMax>), st);
}

}  // namespace vqb
