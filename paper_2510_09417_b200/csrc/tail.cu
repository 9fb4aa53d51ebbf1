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
            A.trace[1 + (li) * 6 + (ph)] = global_ns();                      \
    } while (0)

__global__ void __launch_bounds__(kThreads, 2) tail_kernel(TailArgs A) {
    VQB_PDL();
    extern __shared__ __align__(16) unsigned char tl_dsm[];
    FinAllSmem& U = *reinterpret_cast<FinAllSmem*>(tl_dsm);
    __shared__ uint32_t s_flag;
    cg::grid_group grid = cg::this_grid();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        A.state[0] = uint32_t(A.l0);
        A.state[1] = 0u;
        if (A.trace) A.trace[0] = global_ns();
    }
    int in = 0;  // level l0 reads buffer 0 (the root's output)
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
                PlanArgs pa;
                pa.slots = T.slots;
                pa.nslots = A.nslots0;
                pa.prev = prev;
                pa.fin_cap = A.max_slots;
                pa.segs = T.segs;
                pa.fins = T.fins;
                pa.kind = T.kind;
                pa.link = T.link;
                pa.info = info;
                pa.flags = A.flags;
                pa.aggs = static_cast<PlanAgg*>(A.aggs_v);
                pa.incs = static_cast<PlanAgg*>(A.incs_v);
                pa.epoch = A.epoch0 + uint32_t(li);
                pa.ctr = A.plan_ctr;
                pa.seg_pcnt = A.seg_pcnt;
                pa.seg_done = A.seg_done;
                pa.seg_ctr = A.seg_ctr;
                planner_body(pa, 1u);
                __syncthreads();
                const uint32_t nseg = info->nseg;
                for (uint32_t k = threadIdx.x; k < nseg; k += blockDim.x) {
                    const uint32_t t0 = T.segs[k].tile0, nt = T.segs[k].ntiles;
                    for (uint32_t t = 0; t < nt; ++t) A.tile_seg[t0 + t] = k;
                }
            }
        }
        KT_TRACE(li, 1);
        grid.sync();
        KT_TRACE(li, 2);
        if (threadIdx.x == 0) s_flag = *reinterpret_cast<volatile uint32_t*>(&A.state[1]);
        __syncthreads();
        if (s_flag == 2u) return;
        // ---- work: K2 tiles, then the finisher segments
        LevelArgs la;
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
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                A.state[0] = uint32_t(l);
                A.state[1] = 1u;
            }
            return;
        }
        in ^= 1;
    }
}

size_t tail_smem_bytes() { return sizeof(FinAllSmem); }

int occupancy_tail() {
    int b = 0;
    cudaFuncSetAttribute(tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FinAllSmem)));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tail_kernel, kThreads, sizeof(FinAllSmem));
    return b;
}

cudaError_t launch_tail(const TailArgs& a, int grid, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FinAllSmem)));
        attr = true;
    }
    void* args[] = {const_cast<TailArgs*>(&a)};
    return cudaLaunchCooperativeKernel((const void*)tail_kernel, dim3(grid), dim3(kThreads), args,
                                       sizeof(FinAllSmem), st);
}

}  // namespace vqb
