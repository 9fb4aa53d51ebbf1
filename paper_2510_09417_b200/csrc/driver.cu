// Host-side recursion driver and C ABI of the B200 VQhull hot path.
//
// One Engine per device owns the HBM workspace (point buffers, level tables,
// look-back words) and runs a hull as:
//   n <= kFinMax:  K0 one-CTA hull;
//   default:       K_S sample polygon -> K_F filter pass -> KT persistent
//                  recursion (+ emission) — captured once per input as a CUDA
//                  graph and replayed; wide levels continue host-driven:
//                  { planner -> finisher -> tile map -> K2 } per level -> emit;
//   other modes:   K1 extremes -> KA bootstrap -> KB fused levels 1+2 -> levels.
// The reference's equivalent is convex_hull (hull.cpp:207-267) driving
// chain_recursive/chain_iterative (hull.cpp:78-190), one call per segment;
// here a level is one launch (or one phase of KT) over all of its segments.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <initializer_list>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vqhull_b200.h"
#include "hull_types.cuh"
#include "kernels.h"

namespace vqb {

namespace {

thread_local std::string g_last_error;
// bumped whenever an engine buffer is (re)allocated: a captured hull graph
// is valid only while every pointer baked into it is
std::atomic<uint64_t> g_alloc_gen{0};

// VQHULL_TRACE=1: host-side progress trace on stderr (diagnostics)
const bool g_trace = getenv("VQHULL_TRACE") != nullptr;
#define VQB_TRACE(...)                          \
    do {                                        \
        if (g_trace) {                          \
            fprintf(stderr, "[vqhull] " __VA_ARGS__); \
            fputc('\n', stderr);                \
            fflush(stderr);                     \
        }                                       \
    } while (0)

struct CudaError {
    cudaError_t e;
};

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
#ifdef VQB_DEBUG
        fprintf(stderr, "[vqb debug] %s; device fault word %u\n", g_last_error.c_str(), read_and_clear_fault());
#endif
        throw CudaError{e};
    }
}

// Device buffer that only grows.  keep=true preserves the old contents.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void ensure(size_t bytes, cudaStream_t st, bool keep = false) {
        if (bytes <= cap) return;
        size_t ncap = std::max(bytes, cap + cap / 2);
        ncap = (ncap + 255) & ~size_t(255);
        void* np = nullptr;
        ck(cudaMallocAsync(&np, ncap, st), "cudaMallocAsync");
        g_alloc_gen.fetch_add(1);
        if (keep && p && cap) ck(cudaMemcpyAsync(np, p, cap, cudaMemcpyDeviceToDevice, st), "grow copy");
        if (p) ck(cudaFreeAsync(p, st), "cudaFreeAsync");
        p = np;
        cap = ncap;
    }
    void release() {
        if (p) cudaFree(p);
        if (p) g_alloc_gen.fetch_add(1);
        p = nullptr;
        cap = 0;
    }
};

struct PointBuf {
    DevBuf x, y, id;
    // +64 elements: the level kernel's TMA copies round segment ranges out to
    // 16-byte boundaries and may read a few elements past a segment's end
    void ensure(size_t n, cudaStream_t st) {
        x.ensure((n + 64) * 8, st);
        y.ensure((n + 64) * 8, st);
        id.ensure((n + 64) * 4, st);
    }
};

struct LevelTables {
    DevBuf slots, kind, link, size, start, segs, fins, fin_count;
};

struct TimedKernel {
    int family;  // 0 extremes 1 bootstrap 2 root 3 level 4 finisher 5 other
    cudaEvent_t a, b;
};

}  // namespace

class Engine {
   public:
    explicit Engine(int dev) : dev_(dev) {
        VQB_TRACE("engine: cudaSetDevice(%d)", dev);
        ck(cudaSetDevice(dev), "cudaSetDevice");
        VQB_TRACE("engine: context ready");
        ck(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev), "attr");
        // keep freed pool memory cached: per-call growth then costs nothing
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        VQB_TRACE("engine: occupancy queries");
        occ_root_ = std::max(1, occupancy_root(false));
        occ_root_stable_ = std::max(1, occupancy_root(true));
        occ_level_ = std::max(1, occupancy_level(false));
        occ_level_stable_ = std::max(1, occupancy_level(true));
        occ_fin_ = std::max(1, occupancy_finisher());
        occ_fb_ = std::max(1, occupancy_finisher_batch());
        occ_filt_ = std::max(1, occupancy_filtered());
        occ_filter_ = std::max(1, occupancy_filter());
        occ_tail_ = std::max(1, std::min(getenv("VQHULL_TAIL_OCC") ? atoi(getenv("VQHULL_TAIL_OCC")) : 1, occupancy_tail()));
        // VQHULL_KC=0: no cluster recursion (KT does every small recursion)
        use_kc_ = !(getenv("VQHULL_KC") && getenv("VQHULL_KC")[0] == '0') && kc_prepare() > 0;
        // one full wave each
        grid_ext_ = sms_ * std::max(1, std::min(8, occupancy_extremes()));
        grid_boot_ = sms_ * std::max(1, std::min(8, occupancy_bootstrap()));
        grid_poly_ = sms_ * std::max(1, std::min(8, occupancy_poly_sample()));
        if (const char* e = getenv("VQHULL_POLY_OCC"))  // experiments: K_S CTAs per SM
            grid_poly_ = sms_ * std::max(1, std::min(atoi(e), occupancy_poly_sample()));
        stream_grid_ = std::max(std::max(grid_ext_, grid_boot_), grid_poly_);
        VQB_TRACE("engine: allocations");
        ck(cudaMalloc(&ctrs_, 64 * sizeof(uint32_t)), "cudaMalloc ctrs");
        ck(cudaMemset(ctrs_, 0, 64 * sizeof(uint32_t)), "memset ctrs");
        ck(cudaMalloc(&root_, sizeof(RootInfo)), "cudaMalloc root");
        ck(cudaMalloc(&hword_, 64), "cudaMalloc h");
        ck(cudaMallocHost(&h_info_, sizeof(LevelInfo) * 2), "cudaMallocHost");
        ck(cudaMallocHost(&h_root_, sizeof(RootInfo)), "cudaMallocHost");
        ck(cudaMallocHost(&h_word_, 64), "cudaMallocHost");
        ck(cudaMallocHost(&h_dbl_, 8 * 32), "cudaMallocHost");
        fault_dev_ = fault_word_ptr();
        ck(cudaMallocHost(&h_tail_, report_bytes(kTailLevels)), "cudaMallocHost");
        partials_.ensure(partial_bytes(stream_grid_), nullptr);
        VQB_TRACE("engine: synchronize");
        ck(cudaDeviceSynchronize(), "init");
        VQB_TRACE("engine: ready");
    }

    int device() const { return dev_; }
    void set_timing(bool on) { timing_ = on; }
    const vqhull_stats& stats() const { return stats_; }
    std::mutex& mutex() { return mu_; }

    // Full hull on device arrays.  Writes the u32 index list to d_out (device,
    // capacity >= n) and returns h through *h.  Returns VQHULL_* code.
    int hull(const double* dx, const double* dy, uint64_t n, uint32_t* d_out, uint64_t* h,
             cudaStream_t st) {
        VQB_TRACE("hull: n=%llu", (unsigned long long)n);
        // the legacy default stream cannot be captured into a graph: use the
        // engine's own blocking stream, which orders with it both ways
        if (st == nullptr) st = own_stream();
        reset_stats(n);
        *h = 0;
        keep_valid_ = false;
        if (n == 0) return VQHULL_OK;
        if (n >= 0xffffffffull) return VQHULL_ESIZE;
        launches_ = 0;
        begin_timing(st);
        if (n <= kFinMax && !stable_ && !root_reference_ && !root_octagon_ && !force_reference_ && use_tiny_)
            return run_tiny(dx, dy, n, d_out, h, st);

        // ---- root stage: polygon + first partition (levels 1+2 in reference mode)
        // (f64 arrays are 8-byte aligned; the split root's filter pass also takes
        // arrays that are not 16-byte aligned, the one-pass octagon root does not)
        const bool aligned = ((reinterpret_cast<uintptr_t>(dx) | reinterpret_cast<uintptr_t>(dy)) & 15u) == 0;
        const bool aligned8 = ((reinterpret_cast<uintptr_t>(dx) | reinterpret_cast<uintptr_t>(dy)) & 7u) == 0;
        const bool filtered = !stable_ && !root_reference_ && !force_reference_ && !getenv("VQB_NO_TMA") &&
                              (root_octagon_ ? aligned : aligned8);
        const bool split = filtered && !root_octagon_;
        // the common small-recursion case (split root + KT) replays one
        // captured CUDA graph: sample, filter, KT and the report copy
        graph_run_ = split && n <= kLeanN && use_tail_ && use_graph_ && !timing_ && !tail_trace_ && !sync_each_ &&
                     !keep_req_ &&
                     run_graph(dx, dy, n, d_out, st);
        uint32_t nslots = graph_run_ ? 1u
                        : split ? run_root_split(dx, dy, n, st)
                                : (filtered ? run_root_filtered(dx, dy, n, st) : run_root_reference(dx, dy, n, st));
        // finiteness verdict, octagon verdict, sizes for the byte accounting
        const bool lean = n > kLeanN;
        const bool tail = split && !lean && use_tail_;
        if (!tail)  // (the tail kernel reports the root's verdicts with its own state)
            ck(cudaMemcpyAsync(h_root_, root_, sizeof(RootInfo), cudaMemcpyDeviceToHost, st), "d2h root");

        // ---- levels.  Every kernel of a level reads its counts from the
        // level's LevelInfo on the device (the planner derives its slot count
        // and chain base from the previous level's), and every table is sized
        // by host-side bounds, so the host queues kLevelBatch levels at a time
        // and synchronizes once per batch to learn whether the recursion has
        // ended.  Levels queued past the end find zero slots and do nothing.
        // lean mode (very large n): sizes come from the planner's exact
        // counts, one host sync per level, instead of n-sized bounds
        bufs_[0].ensure(n, st);
        if (!lean) {
            bufs_[1].ensure(n, st);
            chain_.ensure(n * 4 + 4, st, true);
        }
        const uint64_t seg_lim = n / (uint64_t(kFinMax) + 1);  // internal segments hold > kFinMax points
        uint32_t S = nslots;  // slot bound of the level being queued
        int in = 0;
        int lvl = 2;
        lmax_ = -1;
        tail_emitted_ = false;
        if (tail) {
            // KT: every level in one persistent launch while they stay small
            const int rc = graph_run_ ? finish_tail(graph_ta_, st, &lvl, &in, &S)
                                      : run_tail(dx, dy, n, nslots, d_out, st, &lvl, &in, &S);
            if (rc == VQHULL_EINVAL) return rc;
            if (rc < 0) return rerun_unfiltered(dx, dy, n, d_out, h, st);
        }
        // (VQHULL_LEVEL_BATCH overrides the batch: tests of the re-entry path)
        const int batch = lean ? 1 : (getenv("VQHULL_LEVEL_BATCH") ? std::max(1, atoi(getenv("VQHULL_LEVEL_BATCH")))
                                                                   : kLevelBatch);
        // planner-free levels (fast mode): each level kernel plans the next one
        // (plan_child, partition.cu); only the first host level runs the
        // planner and tile-map kernels.  The tile map and the per-segment
        // counters alternate between two sets (the level reads one, plans
        // into the other).
        const bool pfree = !stable_ && use_pf_;
        int par = 0;
        bool planned = false;
        while (lmax_ < 0) {
            const int first = lvl;
            for (int b = 0; b < batch; ++b, ++lvl) {
                uint32_t nseg_b = uint32_t(std::min<uint64_t>(S, seg_lim));
                uint32_t ntiles_b = uint32_t(n / kTile) + nseg_b + 1;
                const uint32_t S1 = std::max<uint32_t>(S, 1);
                LevelTables& T = level(lvl);
                ensure_tables(T, S1, st);
                ensure_lookback(std::max<uint32_t>((S1 + 1023) / 1024, ntiles_b), st);
                DevBuf& SA = par ? segaux2_ : segaux_;
                SA.ensure(segaux_bytes(S1), st);
                info_.ensure(size_t(lvl + 3) * sizeof(LevelInfo), st, true);
                LevelInfo* dinfo = info_.as<LevelInfo>() + lvl;
                const LevelInfo* dprev = lvl == 2 ? nullptr : info_.as<LevelInfo>() + (lvl - 1);
                if (!planned) {
                    const uint32_t ep = next_epoch();
                    tk(5, st, [&] {
                        launch_planner(T.slots.as<ChildRec>(), S, dprev, S, T.segs.as<SegRec>(), T.fins.as<FinRec>(),
                                       T.kind.as<uint8_t>(), T.link.as<uint32_t>(), dinfo, flags_.as<uint32_t>(),
                                       aggs_.p, incs_.p, ep, &ctrs_[2], seg_pcnt(SA), seg_done(SA, S1),
                                       seg_ctr(SA, S1), sms_ * 4, st, pfree ? dinfo + 1 : nullptr);
                    });
                }
                uint64_t out_bound = n;  // points of the next level
                if (lean) {
                    ck(cudaMemcpyAsync(h_info_, dinfo, sizeof(LevelInfo), cudaMemcpyDeviceToHost, st), "d2h info");
                    ck(cudaStreamSynchronize(st), "level sync");
                    if (lvl == 2 && h_root_->nonfinite) {
                        end_timing(st);
                        ck(cudaStreamSynchronize(st), "sync");
                        return VQHULL_EINVAL;
                    }
                    if (lvl == 2 && split && h_root_->unsafe) return rerun_unfiltered(dx, dy, n, d_out, h, st);
                    const LevelInfo li = *h_info_;
                    nseg_b = li.nseg;
                    ntiles_b = li.ntiles;
                    out_bound = li.out_total;
                    bufs_[in ^ 1].ensure(std::max<uint32_t>(li.out_total, 1), st);
                    chain_.ensure((uint64_t(li.fin_base) + li.fin_total) * 4 + 4, st, true);
                }
                // finishers: whole subtrees of every segment of <= kFinMax
                // points (a warp each up to kFinSmall, a CTA each above)
                tk(4, st, [&] {
                    if (use_fb_)
                        launch_finisher_batch(T.fins.as<FinRec>(), dinfo, S1, bufs_[in].x.as<double>(),
                                              bufs_[in].y.as<double>(), bufs_[in].id.as<uint32_t>(),
                                              chain_.as<uint32_t>(), T.fin_count.as<uint32_t>(), S1, sms_ * occ_fb_, st);
                    else
                        launch_finisher(T.fins.as<FinRec>(), dinfo, S1, bufs_[in].x.as<double>(),
                                        bufs_[in].y.as<double>(), bufs_[in].id.as<uint32_t>(), chain_.as<uint32_t>(),
                                        T.fin_count.as<uint32_t>(), S1, sms_ * occ_fin_, st);
                });
                // K2 over all internal segments of this level
                const int out = in ^ 1;
                DevBuf& TS = par ? tile_seg2_ : tile_seg_;
                TS.ensure(size_t(ntiles_b) * 4, st);
                part_.ensure(size_t(ntiles_b) * 2 * sizeof(Best), st);
                LevelTables& Tn = level(lvl + 1);
                Tn.slots.ensure(size_t(2) * std::max<uint32_t>(nseg_b, 1) * sizeof(ChildRec), st);
                LevelTables& Tc = level(lvl);
                if (!planned)
                    tk(5, st, [&] { launch_tilemap(Tc.segs.as<SegRec>(), dinfo, TS.as<uint32_t>(), ntiles_b, st); });
                {
                    const int grid = std::max(1, std::min<int>(int(ntiles_b), sms_ * (stable_ ? occ_level_stable_ : occ_level_)));
                    LevelArgs la = {};
                    la.gx = dx; la.gy = dy;
                    la.segs = Tc.segs.as<SegRec>(); la.tile_seg = TS.as<uint32_t>(); la.info = dinfo;
                    la.ix = bufs_[in].x.as<double>(); la.iy = bufs_[in].y.as<double>(); la.iid = bufs_[in].id.as<uint32_t>();
                    la.ox = bufs_[out].x.as<double>(); la.oy = bufs_[out].y.as<double>(); la.oid = bufs_[out].id.as<uint32_t>();
                    la.in_cap = bufs_[in].x.cap / 8; la.out_cap = bufs_[out].x.cap / 8;
                    la.status_cap = status_.cap / sizeof(Status); la.part_cap = part_.cap / sizeof(Best);
                    la.children_cap = Tn.slots.cap / sizeof(ChildRec); la.segs_cap = S1;
                    la.status = status_.as<Status>(); la.epoch = next_epoch(); la.ctr = &ctrs_[1];
                    la.tile_part = part_.as<Best>();
                    la.seg_pcnt = seg_pcnt(SA); la.seg_done = seg_done(SA, S1); la.seg_ctr = seg_ctr(SA, S1);
                    la.children = Tn.slots.as<ChildRec>();
                    if (pfree) {  // plan level lvl + 1 inside this launch
                        const uint32_t S1n = std::max<uint32_t>(2 * nseg_b, 1);
                        const uint64_t nseg_n = std::min<uint64_t>(S1n, seg_lim);
                        ensure_tables(Tn, S1n, st);
                        DevBuf& SAn = par ? segaux_ : segaux2_;
                        SAn.ensure(segaux_bytes(S1n), st);
                        DevBuf& TSn = par ? tile_seg_ : tile_seg2_;
                        TSn.ensure(size_t(out_bound / kTile + nseg_n + 1) * 4, st);
                        la.n_kind = Tn.kind.as<uint8_t>(); la.n_link = Tn.link.as<uint32_t>();
                        la.n_segs = Tn.segs.as<SegRec>(); la.n_fins = Tn.fins.as<FinRec>(); la.n_fin_cap = S1n;
                        la.n_info = dinfo + 1; la.nn_info = dinfo + 2;
                        la.n_tile_seg = TSn.as<uint32_t>();
                        la.n_seg_pcnt = seg_pcnt(SAn); la.n_seg_done = seg_done(SAn, S1n); la.n_seg_ctr = seg_ctr(SAn, S1n);
                    }
                    tk(3, st, [&] { ck(launch_level(la, false, stable_, grid, st), "level launch"); });
                }
                in = out;
                S = 2 * nseg_b;
                if (pfree) par ^= 1;
                planned = pfree;
            }
            ck(cudaMemcpyAsync(h_info_, info_.as<LevelInfo>() + (lvl - 1), sizeof(LevelInfo),
                               cudaMemcpyDeviceToHost, st), "d2h info");
            VQB_TRACE("hull: levels %d..%d sync", first, lvl - 1);
            ck(cudaStreamSynchronize(st), "level sync");
            if (first == 2 && h_root_->nonfinite) {
                end_timing(st);
                ck(cudaStreamSynchronize(st), "sync");
                return VQHULL_EINVAL;
            }
            if (first == 2 && split && h_root_->unsafe) return rerun_unfiltered(dx, dy, n, d_out, h, st);
            VQB_TRACE("hull: after level %d: nslots %u nseg %u out_total %u fin_total %u", lvl - 1, h_info_->nslots,
                      h_info_->nseg, h_info_->out_total, h_info_->fin_total);
            if (h_info_->nseg == 0) {
                // the recursion ended in this batch: fetch all level infos
                hinfo_.resize(lvl);
                ck(cudaMemcpyAsync(hinfo_.data() + 2, info_.as<LevelInfo>() + 2, sizeof(LevelInfo) * (lvl - 2),
                                   cudaMemcpyDeviceToHost, st), "d2h infos");
                ck(cudaStreamSynchronize(st), "info sync");
                for (int l = 2; l < lvl; ++l)
                    if (hinfo_[l].nseg == 0) { lmax_ = l; break; }
            } else if (uint64_t(lvl) > n + 8) {  // every level sheds >= 1 point per segment
                g_last_error = "recursion did not shrink (internal error)";
                throw CudaError{cudaErrorUnknown};
            }
        }
        for (int l = 2; l <= lmax_; ++l) {
            const LevelInfo& li = hinfo_[l];
            VQB_TRACE("level %d: slots %u internal %u (points %u) finisher %u+%u (points %u) leaves %u", l, li.nslots,
                      li.nseg, li.out_total, li.nfin, li.nfin2, li.fin_total, li.nleaf);
            // every point of this level's slots was written (20 B) by the
            // previous partition (KB for level 2, K2 otherwise)
            const uint64_t written = uint64_t(li.out_total) + li.fin_total + li.nleaf;
            if (l == 2) stats_.survivors_root = written;
            else stats_.bytes_levels += 20 * written;
            stats_.finisher_points += li.fin_total;
            stats_.finisher_segments += li.nfin + li.nfin2;
            stats_.bytes_finisher += uint64_t(li.fin_total) * 20 + uint64_t(li.fin_total) * 4;
            stats_.segments += li.nseg;
            stats_.level_points += li.out_total;
            stats_.bytes_levels += uint64_t(li.out_total) * 20;  // reads; writes counted next level
        }
        stats_.levels = uint32_t(lmax_);
        stats_.bytes_root_partition = 16 * n + 20 * stats_.survivors_root;
        stats_.root_filtered = filtered ? (split ? 2u : 1u) : 0u;
        if (filtered) stats_.root_filter_on = h_root_->poly.filter;

        // ---- emission: bottom-up sizes, root frame, top-down starts
        // (already done inside the persistent tail kernel for small trees)
        uint64_t total_slots = 0;
        for (int l = 2; l <= lmax_; ++l) total_slots += hinfo_[l].nslots;
        if (tail_emitted_) {
        } else if (lmax_ - 1 <= kEmitMaxLevels && total_slots <= kEmitSmallSlots) {
            // small tree: everything in one CTA
            EmitAll E;
            std::memset(&E, 0, sizeof E);
            E.nlev = lmax_ - 1;
            for (int l = 2; l <= lmax_; ++l) {
                LevelTables& T = level(l);
                EmitLevel& el = E.lv[l - 2];
                el.kind = T.kind.as<uint8_t>(); el.link = T.link.as<uint32_t>(); el.slots = T.slots.as<ChildRec>();
                el.fins = T.fins.as<FinRec>(); el.fin_count = T.fin_count.as<uint32_t>();
                el.size = T.size.as<uint32_t>(); el.start = T.start.as<uint32_t>();
                el.nslots = hinfo_[l].nslots;
            }
            tk(5, st, [&] { launch_emit_small(E, root_, chain_.as<uint32_t>(), d_out, hword_, st); });
        } else {
        // a large tree: its top levels (few slots each, many launches
        // otherwise) in the one-CTA kernel, the levels below one launch each
        int ltop = 1;  // last level done by the one-CTA kernel
        {
            uint64_t acc = 0;
            while (ltop + 1 < lmax_ && ltop - 1 < kEmitMaxLevels && acc + hinfo_[ltop + 1].nslots <= kEmitTopSlots) {
                acc += hinfo_[ltop + 1].nslots;
                ++ltop;
            }
            if (ltop < 4) ltop = 1;  // not worth a launch of its own
        }
        for (int l = lmax_; l > ltop && l >= 2; --l) {
            LevelTables& T = level(l);
            const uint32_t ns = hinfo_[l].nslots;
            const uint32_t* child_size = (l < lmax_) ? level(l + 1).size.as<uint32_t>() : nullptr;
            tk(5, st, [&] {
                launch_size(ns, T.kind.as<uint8_t>(), T.link.as<uint32_t>(), T.fin_count.as<uint32_t>(),
                            child_size, T.size.as<uint32_t>(), st);
            });
        }
        if (ltop >= 2) {
            EmitAll E;
            std::memset(&E, 0, sizeof E);
            E.nlev = ltop - 1;
            for (int l = 2; l <= ltop; ++l) {
                LevelTables& T = level(l);
                EmitLevel& el = E.lv[l - 2];
                el.kind = T.kind.as<uint8_t>(); el.link = T.link.as<uint32_t>(); el.slots = T.slots.as<ChildRec>();
                el.fins = T.fins.as<FinRec>(); el.fin_count = T.fin_count.as<uint32_t>();
                el.size = T.size.as<uint32_t>(); el.start = T.start.as<uint32_t>();
                el.nslots = hinfo_[l].nslots;
            }
            E.below_size = level(ltop + 1).size.as<uint32_t>();
            E.below_start = level(ltop + 1).start.as<uint32_t>();
            tk(5, st, [&] { launch_emit_small(E, root_, chain_.as<uint32_t>(), d_out, hword_, st); });
        } else {
            tk(5, st, [&] {
                launch_poly_frame(root_, level(2).size.as<uint32_t>(), level(2).start.as<uint32_t>(), d_out,
                                  hword_, st);
            });
        }
        for (int l = std::max(2, ltop + 1); l <= lmax_; ++l) {
            LevelTables& T = level(l);
            const uint32_t ns = hinfo_[l].nslots;
            const bool has_child = l < lmax_;
            tk(5, st, [&] {
                launch_emit(ns, T.kind.as<uint8_t>(), T.link.as<uint32_t>(), T.slots.as<ChildRec>(),
                            T.fins.as<FinRec>(), T.fin_count.as<uint32_t>(), chain_.as<uint32_t>(),
                            T.start.as<uint32_t>(), has_child ? level(l + 1).size.as<uint32_t>() : nullptr,
                            has_child ? level(l + 1).start.as<uint32_t>() : nullptr, d_out, st);
            });
        }
        }
        if (!tail_emitted_) {  // (the tail kernel's h came with its state)
            ck(cudaMemcpyAsync(h_word_, hword_, 4, cudaMemcpyDeviceToHost, st), "d2h h");
            ck(cudaMemcpyAsync(h_word_ + 1, fault_dev_, 4, cudaMemcpyDeviceToHost, st), "d2h fault");
            end_timing(st);
            VQB_TRACE("hull: final sync");
            ck(cudaStreamSynchronize(st), "final sync");
        }
        VQB_TRACE("hull: done");
        ck(cudaGetLastError(), "kernel launch");
        check_fault();
        *h = *h_word_;
        if (sample_trace_) print_sample_trace();
        if (fin_trace_) print_fin_trace();
        stats_.hull_size = *h;
        stats_.launches = launches_;
        stats_.bytes_moved = stats_.bytes_extremes + stats_.bytes_bootstrap + stats_.bytes_root_partition +
                             stats_.bytes_levels + stats_.bytes_finisher;
        collect_timing();
        return VQHULL_OK;
    }

    int find_extremes(const double* dx, const double* dy, uint64_t n, uint64_t* lo, uint64_t* hi,
                      cudaStream_t st) {
        if (n == 0) return VQHULL_EINVAL;
        if (n >= 0xffffffffull) return VQHULL_ESIZE;
        launch_extremes(dx, dy, n, partials_.p, &ctrs_[3], root_, grid_ext_, st);
        ck(cudaMemcpyAsync(h_root_, root_, sizeof(RootInfo), cudaMemcpyDeviceToHost, st), "d2h root");
        ck(cudaStreamSynchronize(st), "sync");
        ck(cudaGetLastError(), "launch");
        *lo = h_root_->p_idx;
        *hi = h_root_->q_idx;
        return VQHULL_OK;
    }

    int extract(double* dx, double* dy, uint64_t n, const double* ea, const double* eb, uint64_t* wl,
                uint64_t* wr, double* r1, int* h1, double* r2, int* h2, cudaStream_t st) {
        *wl = 0;
        *wr = n;
        *h1 = *h2 = 0;
        if (n == 0) return VQHULL_OK;
        if (n >= 0xffffffffull) return VQHULL_ESIZE;
        bufs_[0].ensure(n, st);
        bufs_[1].ensure(n, st);
        ck(cudaMemcpyAsync(bufs_[0].x.p, dx, n * 8, cudaMemcpyDeviceToDevice, st), "copy x");
        ck(cudaMemcpyAsync(bufs_[0].y.p, dy, n * 8, cudaMemcpyDeviceToDevice, st), "copy y");
        iota(bufs_[0].id.as<uint32_t>(), n, st);
        SegRec g;
        std::memset(&g, 0, sizeof g);
        g.px = ea[0]; g.py = ea[1]; g.rx = ea[2]; g.ry = ea[3];
        g.bx = eb[0]; g.by = eb[1]; g.qx = eb[2]; g.qy = eb[3];
        g.adx = ea[2] - ea[0]; g.ady = ea[3] - ea[1];  // EdgeFrame::make (kernels.hpp:23-25)
        g.bdx = eb[2] - eb[0]; g.bdy = eb[3] - eb[1];
        g.begin = 0; g.out = 0; g.m = uint32_t(n); g.tile0 = 0;
        g.ntiles = uint32_t((n + kTile - 1) / kTile);
        g.slot = 0;
        LevelInfo li;
        std::memset(&li, 0, sizeof li);
        li.nslots = 1; li.nseg = 1; li.ntiles = g.ntiles; li.out_total = uint32_t(n);
        scratch_.ensure(sizeof(SegRec) + sizeof(LevelInfo) + 2 * sizeof(ChildRec), st);
        char* sp = scratch_.as<char>();
        SegRec* dseg = reinterpret_cast<SegRec*>(sp);
        LevelInfo* dli = reinterpret_cast<LevelInfo*>(sp + sizeof(SegRec));
        ChildRec* dch = reinterpret_cast<ChildRec*>(sp + sizeof(SegRec) + sizeof(LevelInfo));
        ck(cudaMemcpyAsync(dseg, &g, sizeof g, cudaMemcpyHostToDevice, st), "h2d seg");
        ck(cudaMemcpyAsync(dli, &li, sizeof li, cudaMemcpyHostToDevice, st), "h2d info");
        tile_seg_.ensure(size_t(g.ntiles) * 4, st);
        ck(cudaMemsetAsync(tile_seg_.p, 0, size_t(g.ntiles) * 4, st), "memset tiles");
        ensure_lookback(g.ntiles, st);
        part_.ensure(size_t(g.ntiles) * 2 * sizeof(Best), st);
        segaux_.ensure(segaux_bytes(1), st);
        ck(cudaMemsetAsync(segaux_.p, 0, segaux_bytes(1), st), "memset seg aux");
        const int grid = std::max(1, std::min<int>(int(g.ntiles), sms_ * (stable_ ? occ_level_stable_ : occ_level_)));
        LevelArgs la = {};
        la.gx = bufs_[0].x.as<double>(); la.gy = bufs_[0].y.as<double>();
        la.segs = dseg; la.tile_seg = tile_seg_.as<uint32_t>(); la.info = dli;
        la.ix = bufs_[0].x.as<double>(); la.iy = bufs_[0].y.as<double>(); la.iid = bufs_[0].id.as<uint32_t>();
        la.ox = bufs_[1].x.as<double>(); la.oy = bufs_[1].y.as<double>(); la.oid = bufs_[1].id.as<uint32_t>();
        la.in_cap = bufs_[0].x.cap / 8; la.out_cap = bufs_[1].x.cap / 8;
        la.status_cap = status_.cap / sizeof(Status); la.part_cap = part_.cap / sizeof(Best);
        la.children_cap = 2; la.segs_cap = 1;
        la.status = status_.as<Status>(); la.epoch = next_epoch(); la.ctr = &ctrs_[1];
        la.tile_part = part_.as<Best>();
        la.seg_pcnt = seg_pcnt(); la.seg_done = seg_done(1); la.seg_ctr = seg_ctr(1);
        la.children = dch;
        ck(launch_level(la, true, stable_, grid, st), "extract launch");
        ChildRec ch[2];
        ck(cudaMemcpyAsync(ch, dch, sizeof ch, cudaMemcpyDeviceToHost, st), "d2h children");
        ck(cudaStreamSynchronize(st), "sync");
        ck(cudaGetLastError(), "launch");
        const uint64_t nl = ch[0].m, nr = ch[1].m;
        if (nl) ck(cudaMemcpyAsync(dx, bufs_[1].x.p, nl * 8, cudaMemcpyDeviceToDevice, st), "copy back");
        if (nl) ck(cudaMemcpyAsync(dy, bufs_[1].y.p, nl * 8, cudaMemcpyDeviceToDevice, st), "copy back");
        if (nr) ck(cudaMemcpyAsync(dx + (n - nr), bufs_[1].x.as<double>() + (n - nr), nr * 8,
                                   cudaMemcpyDeviceToDevice, st), "copy back");
        if (nr) ck(cudaMemcpyAsync(dy + (n - nr), bufs_[1].y.as<double>() + (n - nr), nr * 8,
                                   cudaMemcpyDeviceToDevice, st), "copy back");
        ck(cudaStreamSynchronize(st), "sync");
        *wl = nl;
        *wr = n - nr;
        *h1 = nl > 0;
        *h2 = nr > 0;
        if (nl) { r1[0] = ch[0].rx; r1[1] = ch[0].ry; }
        if (nr) { r2[0] = ch[1].rx; r2[1] = ch[1].ry; }
        return VQHULL_OK;
    }

    // Host -> device copy of caller arrays.  Page-locked (or registered)
    // memory goes to the copy engine as it is.  Pageable memory — what a
    // drop-in C caller of vqhull_compute passes — would be staged by the
    // driver through its own small pinned buffer at ~11 GB/s; here worker
    // threads copy 8 MB chunks into a ring of pinned buffers, each chunk
    // followed by its asynchronous H2D copy, so the host memcpy of one chunk
    // overlaps the PCIe transfer of the others (the copies stay ordered
    // before the hull on the stream).
    struct HostPart {
        void* dst;
        const void* src;
        size_t bytes;
    };
    static bool pageable(const void* p) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
            (void)cudaGetLastError();
            return true;
        }
        return at.type == cudaMemoryTypeUnregistered;
    }
    void h2d(std::initializer_list<HostPart> parts, cudaStream_t st) {
        static const bool staging = !(getenv("VQHULL_STAGING") && getenv("VQHULL_STAGING")[0] == '0');
        size_t total = 0;
        bool paged = false;
        for (const HostPart& q : parts) {
            total += q.bytes;
            paged |= q.bytes && pageable(q.src);
        }
        if (!staging || !paged || total < (size_t(64) << 20)) {
            for (const HostPart& q : parts)
                if (q.bytes) ck(cudaMemcpyAsync(q.dst, q.src, q.bytes, cudaMemcpyHostToDevice, st), "h2d");
            return;
        }
        constexpr size_t kChunk = size_t(8) << 20;
        constexpr int kBufsPerThread = 3;
        // (VQHULL_STAGE_THREADS overrides the worker count)
        static const int env_thr = getenv("VQHULL_STAGE_THREADS") ? atoi(getenv("VQHULL_STAGE_THREADS")) : 0;
        const int nthr = env_thr > 0 ? std::min(env_thr, 64)
                                     : int(std::max(1u, std::min(8u, std::thread::hardware_concurrency() / 2)));
        const size_t need = size_t(nthr) * kBufsPerThread * kChunk;
        if (stage_bytes_ < need) {
            if (stage_) cudaFreeHost(stage_);
            stage_ = nullptr;
            stage_bytes_ = 0;
            ck(cudaHostAlloc(&stage_, need, cudaHostAllocDefault), "cudaHostAlloc staging");
            stage_bytes_ = need;
        }
        struct Chunk {
            char* dst;
            const char* src;
            size_t bytes;
        };
        std::vector<Chunk> chunks;
        for (const HostPart& q : parts)
            for (size_t o = 0; o < q.bytes; o += kChunk)
                chunks.push_back({static_cast<char*>(q.dst) + o, static_cast<const char*>(q.src) + o,
                                  std::min(kChunk, q.bytes - o)});
        std::atomic<size_t> next{0};
        std::atomic<int> failed{0};
        auto work = [&](int t) {
            if (cudaSetDevice(dev_) != cudaSuccess) { failed = 1; return; }
            cudaEvent_t ev[kBufsPerThread];
            bool used[kBufsPerThread] = {};
            for (cudaEvent_t& e : ev)
                if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) { failed = 1; return; }
            char* base = static_cast<char*>(stage_) + size_t(t) * kBufsPerThread * kChunk;
            for (int b = 0; !failed; b = (b + 1) % kBufsPerThread) {
                const size_t i = next.fetch_add(1);
                if (i >= chunks.size()) break;
                if (used[b] && cudaEventSynchronize(ev[b]) != cudaSuccess) { failed = 1; break; }
                char* buf = base + size_t(b) * kChunk;
                std::memcpy(buf, chunks[i].src, chunks[i].bytes);
                if (cudaMemcpyAsync(chunks[i].dst, buf, chunks[i].bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
                    cudaEventRecord(ev[b], st) != cudaSuccess) { failed = 1; break; }
                used[b] = true;
            }
            for (int b = 0; b < kBufsPerThread; ++b) {
                if (used[b]) cudaEventSynchronize(ev[b]);  // the buffer is reused by the next call
                cudaEventDestroy(ev[b]);
            }
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < nthr; ++t) pool.emplace_back(work, t);
        work(0);
        for (std::thread& th : pool) th.join();
        if (failed) {
            (void)cudaGetLastError();
            g_last_error = "staged host-to-device copy failed";
            throw CudaError{cudaErrorUnknown};
        }
    }

    // host-input path (vqhull_compute)
    int compute_host(const double* xs, const double* ys, uint64_t n, uint32_t* h_out_u32, uint64_t* h,
                     cudaStream_t st) {
        VQB_TRACE("compute_host: n=%llu", (unsigned long long)n);
        if (n >= 0xffffffffull) return VQHULL_ESIZE;  // before any allocation or copy
        if (st == nullptr) st = own_stream();
        in_.x.ensure(n * 8, st);
        in_.y.ensure(n * 8, st);
        h2d({{in_.x.p, xs, size_t(n) * 8}, {in_.y.p, ys, size_t(n) * 8}}, st);
        out_.ensure(n * 4, st);
        const int rc = hull(in_.x.as<double>(), in_.y.as<double>(), n, out_.as<uint32_t>(), h, st);
        if (rc) return rc;
        if (*h) ck(cudaMemcpyAsync(h_out_u32, out_.p, *h * 4, cudaMemcpyDeviceToHost, st), "d2h idx");
        ck(cudaStreamSynchronize(st), "sync");
        return VQHULL_OK;
    }

    // ---- sharded hull (shard.cu) --------------------------------
    // Local stage of one shard: its hull, then the certificate, then the
    // candidates (every point not proven deep inside the local hull) sorted
    // by index, packed as rows {x, y, bits(offset + index)} behind a header
    // row {count, M_eff, A} (count -1: invalid input).  d_pack (device, room
    // for cap + 1 rows) may be null: the candidates stay in the engine for
    // repack().  floor_m > 0 (a merge's retry): no filter-pass shortcut, the
    // whole shard is tested with the margin scale max(M, floor_m).
    int shard(const double* dx, const double* dy, uint64_t n, uint64_t offset, double floor_m, double* d_pack,
              uint64_t cap, uint64_t* count, cudaStream_t st) {
        if (st == nullptr) st = own_stream();
        *count = 0;
        const double kInf = HUGE_VAL;
        shard_hdr_[0] = 0.0; shard_hdr_[1] = kInf; shard_hdr_[2] = 0.0;
        shard_k_ = 0;
        shard_offset_ = offset;
        if (n >= 0xffffffffull) return VQHULL_ESIZE;
        if (n == 0) return write_header(d_pack, st);
        out_.ensure(n * 4, st);
        uint64_t h = 0;
        keep_req_ = floor_m == 0.0;
        int rc;
        try {
            rc = hull(dx, dy, n, out_.as<uint32_t>(), &h, st);
        } catch (...) {
            keep_req_ = false;
            throw;
        }
        keep_req_ = false;
        if (rc == VQHULL_EINVAL) {  // non-finite input: every rank learns it from the merge
            shard_hdr_[0] = -1.0;
            return write_header(d_pack, st);
        }
        if (rc) return rc;
        const bool kept = floor_m == 0.0 && keep_valid_ && stats_.root_filtered == 2 && !stats_.root_reruns &&
                          stats_.root_filter_on;
        // the tested set: the filter pass's survivors, or the whole shard
        uint64_t m = n;
        ck(cudaMemcpyAsync(h_word_ + 4, &root_->cnt1, 4, cudaMemcpyDeviceToHost, st), "d2h survivors");
        ck(cudaMemcpyAsync(h_dbl_, &root_->poly.mref, 8, cudaMemcpyDeviceToHost, st), "d2h M");
        ck(cudaStreamSynchronize(st), "sync");
        if (kept) m = h_word_[4];
        const double m_kf = h_dbl_[0];
        cert_head_.ensure(sizeof(CertHead), st);
        cert_rec_.ensure(size_t(kCertMax) * sizeof(CertRec), st);
        cert_asc_.ensure(size_t(2 * kCertMax) * 4, st);
        cert_tab_.ensure(size_t(kCertBuckets) * 4, st);
        resid_.ensure(std::max<uint64_t>(m, 1), st);
        ck(cudaMemsetAsync(ctrs_ + 20, 0, 16, st), "memset cert counters");  // count, pad, amax bits (8-byte aligned)
        tk(5, st, [&] {
            launch_cert_build(out_.as<uint32_t>(), uint32_t(h), dx, dy, floor_m, cert_head_.as<CertHead>(),
                              cert_rec_.as<CertRec>(), cert_asc_.as<float>(), cert_tab_.as<uint32_t>(), st);
        });
        tk(5, st, [&] {
            launch_certify(kept ? keep_.x.as<double>() : dx, kept ? keep_.y.as<double>() : dy,
                           kept ? keep_.id.as<uint32_t>() : nullptr, m, nullptr, cert_head_.as<CertHead>(),
                           cert_rec_.as<CertRec>(), cert_asc_.as<float>(), cert_tab_.as<uint32_t>(),
                           resid_.x.as<double>(), resid_.y.as<double>(), resid_.id.as<uint32_t>(), ctrs_ + 20,
                           reinterpret_cast<unsigned long long*>(ctrs_ + 22), sms_ * 8, st);
        });
        CertHead ch;
        ck(cudaMemcpyAsync(h_word_ + 4, ctrs_ + 20, 16, cudaMemcpyDeviceToHost, st), "d2h cert counters");
        ck(cudaMemcpyAsync(h_dbl_ + 1, cert_head_.p, sizeof(CertHead), cudaMemcpyDeviceToHost, st), "d2h cert");
        ck(cudaStreamSynchronize(st), "sync");
        std::memcpy(&ch, h_dbl_ + 1, sizeof ch);
        const uint32_t k = h_word_[4];
        double amax;
        {
            uint64_t bits = uint64_t(h_word_[6]) | (uint64_t(h_word_[7]) << 32);
            std::memcpy(&amax, &bits, 8);
        }
        double m_eff = kInf;
        if (kept) m_eff = std::min(m_eff, m_kf);
        if (ch.valid) m_eff = std::min(m_eff, ch.Me);
        shard_hdr_[0] = double(k);
        shard_hdr_[1] = m_eff;
        shard_hdr_[2] = kept ? std::max(amax, m_kf) : amax;
        shard_k_ = k;
        stats_.shard_tested = m;
        stats_.shard_candidates = k;
        stats_.shard_cert_vertices = ch.K;
        // sort the candidates by index (first occurrence = smallest global index)
        if (k) {
            sorted_.ensure(size_t(k) * 12, st);  // sorted ids | permutation | iota
            const size_t tb = sort_temp_bytes(k);
            sort_tmp_.ensure(tb, st);
            int end_bit = 1;
            while (end_bit < 32 && (uint64_t(1) << end_bit) < n) ++end_bit;
            tk(5, st, [&] {
                ck(launch_sort_ids(sort_tmp_.p, tb, resid_.id.as<uint32_t>(), sorted_.as<uint32_t>(),
                                   sorted_.as<uint32_t>() + 2 * size_t(k), sorted_.as<uint32_t>() + k, k, end_bit, st),
                   "sort candidates");
            });
            launches_ += 2 + uint32_t((end_bit + 7) / 8);  // cub onesweep: histogram, scan, one pass per 8 bits (+ our iota)
        }
        stats_.launches = launches_;
        *count = k;
        return d_pack ? repack(d_pack, cap, st) : VQHULL_OK;
    }

    // the last shard()'s header and first min(count, cap) rows into d_pack
    int repack(double* d_pack, uint64_t cap, cudaStream_t st) {
        if (st == nullptr) st = own_stream();
        if (!d_pack) return VQHULL_EINVAL;
        const uint32_t c = uint32_t(std::min<uint64_t>(cap, 0xffffffffull));
        if (shard_k_)
            tk(5, st, [&] {
                launch_pack(resid_.x.as<double>(), resid_.y.as<double>(), sorted_.as<uint32_t>(),
                            sorted_.as<uint32_t>() + shard_k_, shard_k_, c, shard_offset_, d_pack, st);
            });
        return write_header(d_pack, st);
    }

    // Merge: nranks packs at a stride of stride_rows rows (header + rows, in
    // offset order).  Writes the global clockwise index list (host or device
    // out) or returns VQHULL_ERETRY with *floor_out: recompute every shard
    // with that margin floor (a shard's scale was too small for the largest
    // coordinate in play).
    int merge(const double* d_packs, uint32_t nranks, uint64_t stride_rows, uint64_t* out, uint64_t* count,
              double* floor_out, cudaStream_t st) {
        if (st == nullptr) st = own_stream();
        *count = 0;
        if (floor_out) *floor_out = 0.0;
        if (nranks == 0 || stride_rows == 0) return VQHULL_EINVAL;
        std::vector<double> hdr(size_t(nranks) * 3);
        ck(cudaMemcpy2DAsync(hdr.data(), 24, d_packs, stride_rows * 24, 24, nranks, cudaMemcpyDeviceToHost, st),
           "d2h headers");
        ck(cudaStreamSynchronize(st), "sync");
        double A = 0.0, Mmin = HUGE_VAL;
        std::vector<uint64_t> starts(nranks + 1, 0);
        for (uint32_t r = 0; r < nranks; ++r) {
            const double c = hdr[3 * r];
            if (!(c >= 0.0)) return VQHULL_EINVAL;  // a shard held a non-finite point (or garbage)
            if (c > double(stride_rows - 1)) {
                g_last_error = "merge: a shard's candidates exceed the pack stride (repack them)";
                return VQHULL_EINVAL;
            }
            starts[r + 1] = starts[r] + uint64_t(c);
            A = std::max(A, hdr[3 * r + 2]);
            Mmin = std::min(Mmin, hdr[3 * r + 1]);
        }
        if (!(A <= 0x1p12 * Mmin)) {  // the margins' rounding bound needs A <= 2^12 M on every shard
            if (floor_out) *floor_out = A * 0x1p-12;
            return VQHULL_ERETRY;
        }
        const uint64_t total = starts[nranks];
        stats_merge_ = total;
        if (total == 0) return VQHULL_OK;
        if (total >= 0xffffffffull) return VQHULL_ESIZE;
        mbuf_.ensure(total, st);
        mg_.ensure(total * 8, st);
        mstarts_.ensure(size_t(nranks + 1) * 8, st);
        ck(cudaMemcpyAsync(mstarts_.p, starts.data(), size_t(nranks + 1) * 8, cudaMemcpyHostToDevice, st),
           "h2d starts");
        ck(cudaStreamSynchronize(st), "sync");  // (starts is a host vector)
        ck(cudaMemsetAsync(ctrs_ + 24, 0, 4, st), "memset flag");
        launch_merge_gather(d_packs, stride_rows, mstarts_.as<uint64_t>(), nranks, total, mbuf_.x.as<double>(),
                            mbuf_.y.as<double>(), mg_.as<uint64_t>(), ctrs_ + 24, st);
        ck(cudaMemcpyAsync(h_word_ + 8, ctrs_ + 24, 4, cudaMemcpyDeviceToHost, st), "d2h flag");
        ck(cudaStreamSynchronize(st), "sync");
        if (h_word_[8]) {
            g_last_error = "merge: candidates are not in increasing global-index order (shards out of offset order)";
            return VQHULL_EINVAL;
        }
        out_.ensure(total * 4, st);
        uint64_t h = 0;
        const int rc = hull(mbuf_.x.as<double>(), mbuf_.y.as<double>(), total, out_.as<uint32_t>(), &h, st);
        if (rc) return rc;
        const bool dev = is_device_ptr_(out);
        uint64_t* dst = out;
        if (!dev) {
            mout_.ensure(std::max<uint64_t>(h, 1) * 8, st);
            dst = mout_.as<uint64_t>();
        }
        launch_map_gidx(out_.as<uint32_t>(), h, mg_.as<uint64_t>(), dst, st);
        stats_.launches += 2;  // gather + map
        if (!dev && h) ck(cudaMemcpyAsync(out, dst, h * 8, cudaMemcpyDeviceToHost, st), "d2h indices");
        ck(cudaStreamSynchronize(st), "sync");
        ck(cudaGetLastError(), "merge");
        *count = h;
        return VQHULL_OK;
    }

    uint64_t merged_candidates() const { return stats_merge_; }

    // a copy of host points [0, n) into the engine's input pair (multi-device driver)
    void load_host(const double* xs, const double* ys, uint64_t n, cudaStream_t st) {
        in_.x.ensure(n * 8, st);
        in_.y.ensure(n * 8, st);
        h2d({{in_.x.p, xs, size_t(n) * 8}, {in_.y.p, ys, size_t(n) * 8}}, st);
    }
    const double* in_x() const { return in_.x.as<double>(); }
    const double* in_y() const { return in_.y.as<double>(); }
    cudaStream_t stream() { return own_stream(); }

    DevBuf& out_buf() { return out_; }

    // frees the big per-call buffers (points, level tables, staging) and
    // returns the pool's cached memory to the device; the next call
    // re-allocates what it needs
    void trim() {
        ck(cudaDeviceSynchronize(), "trim sync");
        for (PointBuf* b : {&bufs_[0], &bufs_[1], &in_, &keep_, &resid_, &mbuf_}) {
            b->x.release();
            b->y.release();
            b->id.release();
        }
        for (LevelTables& T : levels_)
            for (DevBuf* d : {&T.slots, &T.kind, &T.link, &T.size, &T.start, &T.segs, &T.fins, &T.fin_count})
                d->release();
        for (DevBuf* d : {&tile_seg_, &tile_seg2_, &segaux2_, &chain_, &out_, &part_, &status_, &flags_, &aggs_, &incs_, &cert_head_,
                          &cert_rec_, &cert_asc_, &cert_tab_, &sorted_, &sort_tmp_, &mg_, &mstarts_, &mout_})
            d->release();
        for (GraphEntry& e : graphs_)
            if (e.exec) {
                cudaGraphExecDestroy(e.exec);
                e.exec = nullptr;
            }
        if (stage_) cudaFreeHost(stage_);
        stage_ = nullptr;
        stage_bytes_ = 0;
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev_) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
        ck(cudaDeviceSynchronize(), "trim sync");
    }

   private:
    // Default: K1' (8 exact directional extremes + finiteness) then KB'
    // (level 1 behind the octagon filter).  Returns the level-2 slot count.
    uint32_t run_root_filtered(const double* dx, const double* dy, uint64_t n, cudaStream_t st) {
        tk(0, st, [&] { launch_extremes(dx, dy, n, partials_.p, &ctrs_[3], root_, grid_ext_, st); });
        {
            // the sample is 1/16 of the points: a smaller grid
            const int g = std::max(1, std::min<int>(grid_poly_, int(n / ((uint64_t(sample_mask(n)) + 1) * 256 * 8)) + 1));
            tk(0, st, [&] { launch_poly_sample(dx, dy, n, partials_.p, &ctrs_[5], sample_keys(), root_, side_ctr(), g, true, st); });
        }
        upload_root_consts(root_, st);
        stats_.bytes_extremes = 8 * n + 16 * n / (sample_mask(n) + 1);  // x, then x and y of the sample
        stats_.bytes_bootstrap = 0;
        bufs_[0].ensure(n, st);
        const uint32_t ntiles_root = uint32_t((n + kTile - 1) / kTile);
        LevelTables& L2 = level(2);
        L2.slots.ensure(2 * sizeof(ChildRec), st);
        const int grid = std::max(1, std::min<int>(int(ntiles_root), sms_ * occ_filt_));
        part_.ensure(size_t(grid) * 2 * sizeof(Best), st);
        RootArgs ra;
        std::memset(&ra, 0, sizeof ra);
        ra.xs = dx; ra.ys = dy; ra.n = n; ra.root = root_; ra.root_w = root_;
        ra.ox = bufs_[0].x.as<double>(); ra.oy = bufs_[0].y.as<double>(); ra.oid = bufs_[0].id.as<uint32_t>();
        ra.out_cap = bufs_[0].x.cap / 8;
        ra.ticket = &ctrs_[4]; ra.cta_part = part_.as<Best>();
        ra.side_ctr = side_ctr();
        ra.children = L2.slots.as<ChildRec>(); ra.ntiles = ntiles_root;
        tk(2, st, [&] { ck(launch_root_filtered(ra, grid, st), "filtered root launch"); });
        return 2;
    }

    // KT (tail.cu): levels lvl.. in one cooperative launch.  Returns 0 and sets
    // lmax_ when the recursion ended inside it; otherwise 0 with (*lvl, *in,
    // *S) set to the level the host loop resumes at.  VQHULL_EINVAL for
    // non-finite input, -1 for an `unsafe` split root (caller reruns).
    int run_tail(const double* dx, const double* dy, uint64_t n, uint32_t nslots, uint32_t* d_out,
                 cudaStream_t st, int* lvl, int* in, uint32_t* S) {
        const TailArgs ta = tail_args(dx, dy, n, nslots, d_out, *lvl, st, *in);
        launch_tail_report(ta, st);
        return finish_tail(ta, st, lvl, in, S);
    }

    // KT's arguments (and every table it writes, allocated here)
    TailArgs tail_args(const double* dx, const double* dy, uint64_t n, uint32_t nslots, uint32_t* d_out, int l0,
                       cudaStream_t st, int in0 = 0) {
        const int nlev = kTailLevels;
        for (int li = 0; li < nlev; ++li) {
            LevelTables& T = level(l0 + li);
            T.kind.ensure(kTailSlots, st);
            T.link.ensure(size_t(kTailSlots) * 4, st);
            T.size.ensure(size_t(kTailSlots) * 4, st);
            T.start.ensure(size_t(kTailSlots) * 4, st);
            T.fin_count.ensure(size_t(kTailSlots) * 4, st);
            T.segs.ensure(size_t(kTailSlots) * sizeof(SegRec), st);
            T.fins.ensure(size_t(kTailSlots) * sizeof(FinRec), st);
            T.slots.ensure(size_t(2) * kTailSlots * sizeof(ChildRec), st, li == 0);  // level l0's slots are live
        }
        info_.ensure(size_t(l0 + nlev + 1) * sizeof(LevelInfo), st, true);
        const uint64_t tiles = n / kTile + kTailSlots + 1;
        ensure_lookback(kTailSlots / 1024 + 1, st);
        segaux_.ensure(segaux_bytes(kTailSlots), st);
        tile_seg_.ensure(tiles * 4, st);
        part_.ensure(tiles * 2 * sizeof(Best), st);
        bufs_[0].ensure(n, st);
        bufs_[1].ensure(n, st);
        chain_.ensure(n * 4 + 4, st, true);
        TailArgs ta;
        std::memset(&ta, 0, sizeof ta);
        for (int li = 0; li < nlev; ++li) {
            LevelTables& T = level(l0 + li);
            ta.lv[li].slots = T.slots.as<ChildRec>();
            ta.lv[li].segs = T.segs.as<SegRec>();
            ta.lv[li].fins = T.fins.as<FinRec>();
            ta.lv[li].kind = T.kind.as<uint8_t>();
            ta.lv[li].link = T.link.as<uint32_t>();
            ta.lv[li].fin_count = T.fin_count.as<uint32_t>();
        }
        ta.info = info_.as<LevelInfo>();
        ta.prev0 = l0 == 2 ? nullptr : info_.as<LevelInfo>() + (l0 - 1);
        ta.l0 = l0;
        ta.nlev = nlev;
        ta.nslots0 = nslots;
        ta.max_slots = kTailSlots;
        ta.max_tiles = tail_max_tiles();
        // segments of <= 768 points go to the CTA finisher (disk 1e6: 0.164 ->
        // 0.147 ms against the full 1024-point capacity; square unchanged)
        ta.fin_max = getenv("VQHULL_TAIL_FINMAX") ? std::min<uint32_t>(kTailFinMax, std::max(65, atoi(getenv("VQHULL_TAIL_FINMAX"))))
                                                  : 768u;
        ta.in0 = in0;
        for (int b = 0; b < 2; ++b) {
            ta.bx[b] = bufs_[b].x.as<double>();
            ta.by[b] = bufs_[b].y.as<double>();
            ta.bid[b] = bufs_[b].id.as<uint32_t>();
        }
        ta.buf_cap = std::min(bufs_[0].x.cap, bufs_[1].x.cap) / 8;
        ta.gx = dx;
        ta.gy = dy;
        ta.flags = flags_.as<uint32_t>();
        ta.aggs_v = aggs_.p;
        ta.incs_v = incs_.p;
        ta.epoch0 = reserve_epochs(nlev);
        ta.plan_ctr = &ctrs_[2];
        ta.seg_pcnt = seg_pcnt();
        ta.seg_done = seg_done(kTailSlots);
        ta.seg_ctr = seg_ctr(kTailSlots);
        ta.tile_seg = tile_seg_.as<uint32_t>();
        ta.tile_part = part_.as<Best>();
        ta.part_cap = part_.cap / sizeof(Best);
        ta.chain = chain_.as<uint32_t>();
        ta.state = &ctrs_[16];
        ta.out = l0 == 2 ? d_out : nullptr;  // (in-kernel emission needs the whole tree)
        ta.h_out = hword_;
        ta.p_idx = &root_->p_idx;
        ta.root = root_;
        report_.ensure(report_bytes(nlev), st);
        ta.report = report_.as<uint32_t>();
        // the cluster recursion first (it hands the call to KT when it cannot take it)
        ta.kc_done = (use_kc_ && l0 == 2 && ta.out) ? ctrs_ + 25 : nullptr;
        if (tail_trace_) {
            trace_.ensure(8 * (1 + 10 * kTailLevels), st);
            ta.trace = trace_.as<unsigned long long>();
        }
        return ta;
    }

    // KT's launch and the one copy of its report (stream-ordered, capturable)
    void launch_tail_report(const TailArgs& ta, cudaStream_t st) {
        const int l0 = ta.l0;
        if (ta.trace) ck(cudaMemsetAsync(ta.trace, 0, 8 * (1 + 10 * kTailLevels), st), "memset trace");
        if (ta.kc_done) tk(3, st, [&] { ck(launch_cluster_tail(ta, st), "cluster recursion launch"); });
        tk(3, st, [&] { ck(launch_tail(ta, tail_grid(), st), "tail launch"); });
        if (tail_trace_) {
            std::vector<unsigned long long> tr(1 + 10 * kTailLevels);
            ck(cudaMemcpyAsync(tr.data(), trace_.p, 8 * tr.size(), cudaMemcpyDeviceToHost, st), "d2h trace");
            ck(cudaStreamSynchronize(st), "trace sync");
            for (int li = 0; li < kTailLevels && tr[1 + li * 10]; ++li) {
                fprintf(stderr, "[kt] level %d:", l0 + li);
                for (int ph = 0; ph < 10; ++ph)
                    if (tr[1 + li * 10 + ph]) fprintf(stderr, " %d:%.2f", ph, (tr[1 + li * 10 + ph] - tr[0]) * 1e-3);
                fputc('\n', stderr);
            }
        }
        ck(cudaMemcpyAsync(h_tail_, ta.report, report_bytes(ta.nlev), cudaMemcpyDeviceToHost, st),
           "d2h tail report");
        end_timing(st);  // (re-recorded later if the host emits)
    }

    // after KT: one sync, then the report decides — finished (lmax_ set,
    // perhaps emitted) or the level the host loop resumes at
    int finish_tail(const TailArgs& ta, cudaStream_t st, int* lvl, int* in, uint32_t* S) {
        const int l0 = ta.l0, nlev = ta.nlev;
        const uint32_t nslots = ta.nslots0;
        VQB_TRACE("hull: tail sync");
        ck(cudaStreamSynchronize(st), "tail sync");
        const uint32_t at = h_tail_[0], how = h_tail_[1];
        h_word_[1] = h_tail_[7];  // the device fault word, copied by the kernel into its report
        stats_.tail_launches += 1;
        stats_.tail_levels += (how == 2 ? at : at + 1) - uint32_t(l0);
        *h_word_ = h_tail_[2];
        h_root_->nonfinite = h_tail_[3];
        h_root_->unsafe = h_tail_[4];
        h_root_->poly.filter = h_tail_[5];
        h_root_->cnt1 = h_tail_[6];
        if (h_root_->nonfinite) return VQHULL_EINVAL;
        if (h_root_->unsafe) return -1;
        const LevelInfo* li = reinterpret_cast<const LevelInfo*>(h_tail_ + 8) - 0;
        hinfo_.resize(std::max<size_t>(hinfo_.size(), size_t(l0 + nlev)));
        for (int l = l0; l < int(at) && l < l0 + nlev; ++l) hinfo_[l] = li[l - l0];
        if (how == 1 || how == 3) {
            hinfo_[at] = li[at - l0];
            if (l0 > 2) {  // the host-driven levels before this launch
                ck(cudaMemcpyAsync(hinfo_.data() + 2, info_.as<LevelInfo>() + 2, sizeof(LevelInfo) * (l0 - 2),
                                   cudaMemcpyDeviceToHost, st), "d2h infos");
                ck(cudaStreamSynchronize(st), "info sync");
            }
            lmax_ = int(at);
            tail_emitted_ = how == 3;
            VQB_TRACE("hull: tail finished at level %u", at);
        } else {
            if (how != 2 || int(at) < l0 || int(at) >= l0 + nlev) {
                g_last_error = "tail kernel did not report its state (internal error)";
                throw CudaError{cudaErrorUnknown};
            }
            *lvl = int(at);
            *in = (int(at) - l0) & 1;
            *S = int(at) == l0 ? nslots : 2u * li[at - 1 - l0].nseg;
            VQB_TRACE("hull: tail stopped before level %u (%u slots)", at, *S);
        }
        return 0;
    }

    // Captures (once per input / buffer set) and launches the graph of the
    // split root + KT + report copy.  Returns false when capture fails (the
    // caller then launches the same work directly).
    bool run_graph(const double* dx, const double* dy, uint64_t n, uint32_t* d_out, cudaStream_t st) {
        // allocate everything first: nothing may allocate inside the capture
        prepare_split(n, st);
        graph_ta_ = tail_args(dx, dy, n, 1u, d_out, 2, st);
        const GraphKey key{dx, dy, n, d_out, st, g_alloc_gen.load()};
        GraphEntry* hit = nullptr;
        for (GraphEntry& e : graphs_)
            if (e.exec && e.key == key) hit = &e;
        if (!hit) {
            // capture only an input seen twice in a row (one-off inputs, e.g.
            // the candidates of a sharded hull, run direct: a capture costs
            // more than it saves once)
            if (!(pending_ == key)) {
                pending_ = key;
                return false;
            }
            GraphEntry* slot = &graphs_[0];  // least recently used
            for (GraphEntry& e : graphs_)
                if (!e.exec || e.used < slot->used) slot = &e;
            if (slot->exec) {
                cudaGraphExecDestroy(slot->exec);
                slot->exec = nullptr;
            }
            cudaGraph_t g = nullptr;
            VQB_TRACE("hull: capturing the split-root graph");
            if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
                VQB_TRACE("hull: capture refused: %s", cudaGetErrorString(cudaGetLastError()));
                use_graph_ = false;
                return false;
            }
            const uint32_t saved = launches_;
            try {
                run_root_split(dx, dy, n, st);
                launch_tail_report(graph_ta_, st);
            } catch (...) {
                VQB_TRACE("hull: capture threw: %s", g_last_error.c_str());
                cudaStreamEndCapture(st, &g);
                if (g) cudaGraphDestroy(g);
                (void)cudaGetLastError();
                use_graph_ = false;
                launches_ = saved;
                return false;
            }
            slot->launches = launches_ - saved;
            launches_ = saved;
            const cudaError_t e = cudaStreamEndCapture(st, &g);
            if (e != cudaSuccess || !g || cudaGraphInstantiate(&slot->exec, g, 0) != cudaSuccess) {
                if (g) cudaGraphDestroy(g);
                VQB_TRACE("hull: capture failed: %s", cudaGetErrorString(cudaGetLastError()));
                slot->exec = nullptr;
                use_graph_ = false;
                return false;
            }
            cudaGraphDestroy(g);
            if (g_alloc_gen.load() != key.gen) {  // something allocated during the capture: do not trust it
                cudaGraphExecDestroy(slot->exec);
                slot->exec = nullptr;
                use_graph_ = false;
                return false;
            }
            slot->key = key;
            hit = slot;
        }
        hit->used = ++graph_clock_;
        VQB_TRACE("hull: graph launch");
        ck(cudaGraphLaunch(hit->exec, st), "graph launch");
        launches_ += hit->launches;
        stats_.bytes_extremes = 16 * n / (sample_mask(n) + 1);
        stats_.bytes_bootstrap = 0;
        return true;
    }

    // n <= kFinMax: the whole hull in one CTA (tiny_hull_kernel), one launch
    // and one synchronization
    int run_tiny(const double* dx, const double* dy, uint64_t n, uint32_t* d_out, uint64_t* h, cudaStream_t st) {
        tiny_.ensure(kFinMax * 8 + sizeof(FinRec) + sizeof(LevelInfo) + 64, st);
        char* p = tiny_.as<char>();
        TinyArgs ta;
        ta.xs = dx;
        ta.ys = dy;
        ta.n = uint32_t(n);
        ta.iid = reinterpret_cast<uint32_t*>(p);
        ta.chain = reinterpret_cast<uint32_t*>(p + kFinMax * 4);
        ta.fin = reinterpret_cast<FinRec*>(p + kFinMax * 8);
        ta.info = reinterpret_cast<LevelInfo*>(p + kFinMax * 8 + sizeof(FinRec));
        ta.fin_count = reinterpret_cast<uint32_t*>(p + kFinMax * 8 + sizeof(FinRec) + sizeof(LevelInfo));
        ta.report = ta.fin_count + 4;
        ta.out = d_out;
        tk(4, st, [&] { launch_tiny(ta, st); ck(cudaGetLastError(), "tiny launch"); });
        ck(cudaMemcpyAsync(h_tail_, ta.report, 12, cudaMemcpyDeviceToHost, st), "d2h tiny report");
        end_timing(st);
        ck(cudaStreamSynchronize(st), "tiny sync");
        h_word_[1] = h_tail_[2];  // the device fault word (copied by the kernel)
        check_fault();
        if (h_tail_[1]) return VQHULL_EINVAL;
        *h = h_tail_[0];
        stats_.hull_size = *h;
        stats_.launches = launches_;
        stats_.levels = 1;
        stats_.survivors_root = n;
        stats_.bytes_root_partition = 16 * n;
        stats_.bytes_moved = 16 * n + 4 * *h;
        collect_timing();
        return VQHULL_OK;
    }

    // the device fault word (finisher guard, debug bounds checks) arrives with
    // each call's last host copy: no extra synchronous read per hull
    void check_fault() {
        if (const uint32_t f = h_word_[1]) {
            h_word_[1] = 0;
            (void)read_and_clear_fault();
            g_last_error = "device fault code " + std::to_string(f);
            throw CudaError{cudaErrorUnknown};
        }
    }

    cudaStream_t own_stream() {
        if (!own_st_) ck(cudaStreamCreate(&own_st_), "cudaStreamCreate");
        return own_st_;
    }

    void prepare_split(uint64_t n, cudaStream_t st) {
        bufs_[0].ensure(n, st);
        level(2).slots.ensure(sizeof(ChildRec), st);
        const uint32_t ntiles = uint32_t((n + kTile - 1) / kTile);
        const int grid = std::max(1, std::min<int>(int(ntiles), sms_ * occ_filter_));
        fpart_.ensure(filter_partial_bytes(grid), st);
    }

    // Split root (default): K_S the octagon from a sample, then K_F the filter
    // alone over every point (survivors + exact p, q + finiteness); the first
    // level is the single bootstrap slot (p, q, p) over the survivors, which
    // the level machinery partitions like any other segment.  Returns 1.
    uint32_t run_root_split(const double* dx, const double* dy, uint64_t n, cudaStream_t st) {
        {
            const int g = std::max(1, std::min<int>(grid_poly_, int(n / ((uint64_t(sample_mask(n)) + 1) * 256 * 8)) + 1));
            tk(0, st, [&] { launch_poly_sample(dx, dy, n, partials_.p, &ctrs_[5], sample_keys(), root_, side_ctr(), g, false, st); });
        }
        upload_root_consts(root_, st);  // the filter's geometry -> constant bank (FP64 operands)
        stats_.bytes_extremes = 16 * n / (sample_mask(n) + 1);  // x and y of the sample
        stats_.bytes_bootstrap = 0;
        bufs_[0].ensure(n, st);
        const uint32_t ntiles = uint32_t((n + kTile - 1) / kTile);
        LevelTables& L2 = level(2);
        L2.slots.ensure(sizeof(ChildRec), st);
        const int grid = std::max(1, std::min<int>(int(ntiles), sms_ * occ_filter_));
        fpart_.ensure(filter_partial_bytes(grid), st);
        FilterArgs fa;
        std::memset(&fa, 0, sizeof fa);
        fa.xs = dx; fa.ys = dy; fa.n = n; fa.ntiles = ntiles;
        fa.xoff = uint32_t((reinterpret_cast<uintptr_t>(dx) >> 3) & 1u);
        fa.yoff = uint32_t((reinterpret_cast<uintptr_t>(dy) >> 3) & 1u);
        fa.ox = bufs_[0].x.as<double>(); fa.oy = bufs_[0].y.as<double>(); fa.oid = bufs_[0].id.as<uint32_t>();
        fa.out_cap = bufs_[0].x.cap / 8;
        fa.ctr = &ctrs_[12]; fa.ticket = &ctrs_[13]; fa.part = fpart_.p;
        fa.root_w = root_; fa.slot = L2.slots.as<ChildRec>();
        if (keep_req_) {  // sharded hull: the filter pass also keeps its survivors for the certificate
            keep_.ensure(n, st);
            fa.kx = keep_.x.as<double>(); fa.ky = keep_.y.as<double>(); fa.kid = keep_.id.as<uint32_t>();
            keep_valid_ = true;
        }
        tk(2, st, [&] { ck(launch_root_filter(fa, grid, st), "root filter launch"); });
        return 1;
    }

    // The split root's margin argument needs every survivor within 2^12 of
    // the octagon's scale; a heavy-tailed input that violates it (the
    // sample missed a far outlier) is hulled again without the filter.
    int rerun_unfiltered(const double* dx, const double* dy, uint64_t n, uint32_t* d_out, uint64_t* h,
                         cudaStream_t st) {
        VQB_TRACE("hull: survivor beyond 2^12 M, rerun unfiltered");
        end_timing(st);
        ck(cudaStreamSynchronize(st), "sync");
        force_reference_ = true;
        int rc;
        try {
            rc = hull(dx, dy, n, d_out, h, st);
        } catch (...) {
            force_reference_ = false;
            throw;
        }
        force_reference_ = false;
        stats_.root_reruns = 1;
        return rc;
    }

    // Reference mode: K1 find_extremes, KA bootstrap arg-max, KB levels 1+2
    // fused; polygon (p, r1, q, r2).  Returns the level-2 slot count.
    uint32_t run_root_reference(const double* dx, const double* dy, uint64_t n, cudaStream_t st) {
        tk(0, st, [&] { launch_extremes(dx, dy, n, partials_.p, &ctrs_[3], root_, grid_ext_, st); });
        tk(1, st, [&] { launch_bootstrap(dx, dy, n, partials_.p, &ctrs_[3], root_, grid_boot_, st); });
        launch_legacy_poly(root_, side_ctr(), st);  // also re-arms the side counters
        ++launches_;
        upload_root_consts(root_, st);  // p, q, r1, r2 -> constant bank for KB
        stats_.bytes_extremes = 8 * n;
        stats_.bytes_bootstrap = 16 * n;
        bufs_[0].ensure(n, st);
        const uint32_t ntiles_root = uint32_t((n + kTile - 1) / kTile);
        ensure_lookback(2 * ntiles_root, st);
        LevelTables& L2 = level(2);
        L2.slots.ensure(4 * sizeof(ChildRec), st);
        const int grid = std::max(1, std::min<int>(int(ntiles_root), sms_ * (stable_ ? occ_root_stable_ : occ_root_)));
        part_.ensure(size_t(grid) * 4 * sizeof(Best), st);
        RootArgs ra;
        std::memset(&ra, 0, sizeof ra);
        ra.xs = dx; ra.ys = dy; ra.n = n; ra.root = root_; ra.root_w = root_;
        ra.ox = bufs_[0].x.as<double>(); ra.oy = bufs_[0].y.as<double>(); ra.oid = bufs_[0].id.as<uint32_t>();
        ra.out_cap = bufs_[0].x.cap / 8;
        ra.status = status_.as<Status>(); ra.epoch = next_epoch();
        ra.ctr = &ctrs_[0]; ra.ticket = &ctrs_[4]; ra.cta_part = part_.as<Best>();
        ra.side_ctr = side_ctr();
        ra.children = L2.slots.as<ChildRec>(); ra.ntiles = ntiles_root;
        tk(2, st, [&] { ck(launch_root_partition(ra, grid, stable_, st), "root partition launch"); });
        return 4;
    }

    LevelTables& level(int l) {
        if (levels_.size() <= size_t(l)) levels_.resize(l + 1);
        return levels_[l];
    }

    uint32_t reserve_epochs(int k) {  // k consecutive epochs (persistent kernel levels)
        uint32_t e = next_epoch();
        if (e + uint32_t(k) >= 0x3fffffffu) {
            epoch_ = 0;
            e = next_epoch();
        }
        epoch_ += uint32_t(k);
        return e;
    }

    uint32_t next_epoch() {
        ++epoch_;
        if ((epoch_ & 0x3fffffffu) == 0) epoch_ = 1;
        return epoch_ & 0x3fffffffu;
    }

    // status words (partition kernels) and planner look-back arrays; fresh
    // words must not alias a live epoch, so growth zeroes them
    void ensure_lookback(uint32_t tiles, cudaStream_t st) {
        const size_t t = std::max<uint32_t>(tiles, 1);
        if (t * sizeof(Status) > status_.cap) {
            status_.ensure(t * sizeof(Status), st);
            ck(cudaMemsetAsync(status_.p, 0, status_.cap, st), "memset status");
        }
        if (t * 4 > flags_.cap) {
            flags_.ensure(t * 4, st);
            ck(cudaMemsetAsync(flags_.p, 0, flags_.cap, st), "memset flags");
        }
        aggs_.ensure(t * plan_agg_bytes(), st);
        incs_.ensure(t * plan_agg_bytes(), st);
    }

    void iota(uint32_t* d, uint64_t n, cudaStream_t st);

    void reset_stats(uint64_t n) {
        std::memset(&stats_, 0, sizeof stats_);
        stats_.n = n;
        timed_.clear();
        lmax_ = 2;
    }

    template <class F>
    void tk(int family, cudaStream_t st, F&& f) {
        if (timing_) {
            TimedKernel t;
            t.family = family;
            t.a = event();
            t.b = event();
            ck(cudaEventRecord(t.a, st), "event");
            f();
            ck(cudaEventRecord(t.b, st), "event");
            timed_.push_back(t);
        } else {
            f();
        }
        ++launches_;
        if (sync_each_) {  // VQHULL_SYNC_EACH=1: localize a faulting launch
            static const char* names[6] = {"extremes", "bootstrap", "root_partition", "level",
                                           "finisher", "planner/tilemap/emit"};
            char buf[96];
            snprintf(buf, sizeof buf, "launch %u (%s)", launches_, names[family]);
            VQB_TRACE("sync after %s", buf);
            ck(cudaStreamSynchronize(st), buf);
            ck(cudaGetLastError(), buf);
        }
    }
    bool sync_each_ = getenv("VQHULL_SYNC_EACH") != nullptr;

    cudaEvent_t event() {
        if (ev_used_ == events_.size()) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "cudaEventCreate");
            events_.push_back(e);
        }
        return events_[ev_used_++];
    }
    void begin_timing(cudaStream_t st) {
        ev_used_ = 0;
        if (timing_) {
            ev_begin_ = event();
            ck(cudaEventRecord(ev_begin_, st), "event");
        }
    }
    void end_timing(cudaStream_t st) {
        if (timing_) {
            ev_end_ = event();
            ck(cudaEventRecord(ev_end_, st), "event");
        }
    }
    void collect_timing() {
        if (!timing_) return;
        float fam[6] = {0, 0, 0, 0, 0, 0};
        for (auto& t : timed_) {
            float ms = 0;
            ck(cudaEventElapsedTime(&ms, t.a, t.b), "elapsed");
            fam[t.family] += ms;
        }
        float total = 0;
        ck(cudaEventElapsedTime(&total, ev_begin_, ev_end_), "elapsed");
        stats_.ms_extremes = fam[0];
        stats_.ms_bootstrap = fam[1];
        stats_.ms_root_partition = fam[2];
        stats_.ms_levels = fam[3];
        stats_.ms_finisher = fam[4];
        stats_.ms_other = fam[5];
        stats_.ms_total = total;
        stats_.timing_valid = 1;
    }

   private:
    int dev_ = 0;
    void* stage_ = nullptr;     // pinned staging ring of h2d()
    size_t stage_bytes_ = 0;
    int sms_ = 148;
    int occ_root_ = 1, occ_root_stable_ = 1, occ_level_ = 1, occ_level_stable_ = 1, occ_fin_ = 1, occ_fb_ = 1;
    // VQHULL_FIN_OLD=1: the one-segment-per-CTA finisher (A/B runs)
    bool use_fb_ = getenv("VQHULL_FIN_OLD") == nullptr;
    int stream_grid_ = 592, grid_ext_ = 592, grid_boot_ = 592, grid_poly_ = 592, occ_filt_ = 1, occ_filter_ = 1;
    bool force_reference_ = false;
    int occ_tail_ = 1;
    // VQHULL_TAIL=0: levels only through the host-driven kernels
    bool use_tail_ = !(getenv("VQHULL_TAIL") && getenv("VQHULL_TAIL")[0] == '0');
    uint32_t* h_tail_ = nullptr;
    bool tail_emitted_ = false;
    bool use_kc_ = false;
    DevBuf tiny_;  // the one-CTA path's scratch
    uint32_t* fault_dev_ = nullptr;
    // VQHULL_TINY=0: tiny inputs through the general pipeline (tests)
    bool use_tiny_ = !(getenv("VQHULL_TINY") && getenv("VQHULL_TINY")[0] == '0');
    static constexpr uint32_t kTailTilesPerCta = 2;  // KT takes levels of at most this many tiles per CTA
    // (VQHULL_TAIL_MAXTILES overrides the tile bound: tests of the hand-over paths)
    int tail_grid() const {  // (VQHULL_TAIL_GRID overrides: experiments)
        const char* e = getenv("VQHULL_TAIL_GRID");
        return e ? std::max(1, std::min(atoi(e), sms_ * occ_tail_)) : sms_ * occ_tail_;
    }
    uint32_t tail_max_tiles() const {
        const char* e = getenv("VQHULL_TAIL_MAXTILES");
        return e ? uint32_t(atoi(e)) : uint32_t(kTailTilesPerCta * sms_ * occ_tail_);
    }
    // captured split-root + KT graph (VQHULL_GRAPH=0 disables)
    bool use_graph_ = !(getenv("VQHULL_GRAPH") && getenv("VQHULL_GRAPH")[0] == '0');
    bool graph_run_ = false;
    cudaStream_t own_st_ = nullptr;
    bool sample_trace_ = getenv("VQHULL_SAMPLE_TRACE") != nullptr;
    bool fin_trace_ = getenv("VQHULL_FIN_TRACE") != nullptr && (fin_trace(true), true);
    struct GraphKey {
        const double* dx = nullptr;
        const double* dy = nullptr;
        uint64_t n = 0;
        uint32_t* out = nullptr;
        cudaStream_t st = nullptr;
        uint64_t gen = ~0ull;
        bool operator==(const GraphKey& o) const {
            return dx == o.dx && dy == o.dy && n == o.n && out == o.out && st == o.st && gen == o.gen;
        }
    };
    struct GraphEntry {
        GraphKey key;
        cudaGraphExec_t exec = nullptr;
        uint32_t launches = 0;
        uint64_t used = 0;
    };
    GraphEntry graphs_[4];  // small LRU cache of captured hulls (all share the engine's buffers)
    GraphKey pending_;
    uint64_t graph_clock_ = 0;
    TailArgs graph_ta_;
    DevBuf report_;
    static size_t report_bytes(int nlev) { return 32 + sizeof(LevelInfo) * size_t(nlev); }
    bool tail_trace_ = getenv("VQHULL_TAIL_TRACE") != nullptr;
    DevBuf trace_;  // set while rerunning an `unsafe` split-root call
    // VQHULL_ROOT=octagon: the one-pass filtered root (K1' + KB'), kept for comparison
    bool root_octagon_ = getenv("VQHULL_ROOT") != nullptr && std::string(getenv("VQHULL_ROOT")) == "octagon";
    bool root_reference_ = getenv("VQHULL_ROOT") != nullptr && std::string(getenv("VQHULL_ROOT")) == "reference";
    uint32_t* ctrs_ = nullptr;
    RootInfo* root_ = nullptr;
    uint32_t* hword_ = nullptr;
    LevelInfo* h_info_ = nullptr;
    RootInfo* h_root_ = nullptr;
    uint32_t* h_word_ = nullptr;
    DevBuf partials_, flags_, aggs_, incs_, tile_seg_, chain_, info_, scratch_, out_;
    DevBuf status_, part_, segaux_, fpart_;
    bool stable_ = getenv("VQHULL_STABLE") != nullptr && getenv("VQHULL_STABLE")[0] == '1';

    // per-segment scratch of the level kernel: partial count, finished tiles
    // (u32 each) and the fast mode's packed L/R counter (u64)
    static size_t segaux_bytes(uint32_t ns) { return size_t(ns) * 16 + 16; }
    static uint32_t* seg_pcnt(DevBuf& b) { return b.as<uint32_t>(); }
    static uint32_t* seg_done(DevBuf& b, uint32_t ns) { return b.as<uint32_t>() + ns; }
    static unsigned long long* seg_ctr(DevBuf& b, uint32_t ns) {
        return reinterpret_cast<unsigned long long*>(b.as<char>() + ((size_t(ns) * 8 + 7) & ~size_t(7)));
    }
    void ensure_tables(LevelTables& T, uint32_t S1, cudaStream_t st) {
        T.kind.ensure(S1, st);
        T.link.ensure(size_t(S1) * 4, st);
        T.size.ensure(size_t(S1) * 4, st);
        T.start.ensure(size_t(S1) * 4, st);
        T.segs.ensure(size_t(S1) * sizeof(SegRec), st);
        T.fins.ensure(size_t(S1) * sizeof(FinRec), st);
        T.fin_count.ensure(size_t(S1) * 4, st);
    }
    DevBuf tile_seg2_, segaux2_;  // the second tile-map / segment-counter set (planner-free levels)
    // VQHULL_PLANNER=1: the planner and tile-map kernels before every host level
    bool use_pf_ = !(getenv("VQHULL_PLANNER") && getenv("VQHULL_PLANNER")[0] == '1');
    uint32_t* seg_pcnt() { return segaux_.as<uint32_t>(); }
    uint32_t* seg_done(uint32_t ns) { return segaux_.as<uint32_t>() + ns; }
    unsigned long long* seg_ctr(uint32_t ns) {
        return reinterpret_cast<unsigned long long*>(segaux_.as<char>() + ((size_t(ns) * 8 + 7) & ~size_t(7)));
    }
    unsigned long long* side_ctr() { return reinterpret_cast<unsigned long long*>(ctrs_ + 8); }
    // the sample kernel's 8 directional keys (zero between calls)
    unsigned long long* sample_keys() { return reinterpret_cast<unsigned long long*>(ctrs_ + 32); }

   public:
    void set_stable(bool s) { stable_ = s; }
    void set_root_reference(bool r) {
        root_reference_ = r;
        root_octagon_ = false;
    }
    void set_root_mode(int m) {  // 0 split (default), 1 one-pass octagon, 2 reference
        root_reference_ = m == 2;
        root_octagon_ = m == 1;
    }
    bool stable() const { return stable_; }

   private:
    PointBuf bufs_[2];
    PointBuf in_;
    // sharded hull: the filter pass's survivor copy, the candidates, the merge
    PointBuf keep_, resid_, mbuf_;
    DevBuf cert_head_, cert_rec_, cert_asc_, cert_tab_, sorted_, sort_tmp_, mg_, mstarts_, mout_;
    bool keep_req_ = false, keep_valid_ = false;
    double shard_hdr_[3] = {0.0, 0.0, 0.0};
    uint32_t shard_k_ = 0;
    uint64_t shard_offset_ = 0;
    uint64_t stats_merge_ = 0;
    double* h_dbl_ = nullptr;  // pinned scratch (8 + CertHead)
    int write_header(double* d_pack, cudaStream_t st) {
        if (!d_pack) return VQHULL_OK;
        std::memcpy(h_dbl_ + 16, shard_hdr_, 24);
        ck(cudaMemcpyAsync(d_pack, h_dbl_ + 16, 24, cudaMemcpyHostToDevice, st), "h2d header");
        ck(cudaStreamSynchronize(st), "sync");
        return VQHULL_OK;
    }
    static bool is_device_ptr_(const void* p) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
    }
    std::deque<LevelTables> levels_;  // deque: references stay valid on growth
    std::vector<LevelInfo> hinfo_;  // host copies of the level infos (after the last batch)
    int lmax_ = 2;
    static constexpr int kLevelBatch = 8;  // levels queued per host synchronization (4: disk 1e8 +2 %, 16: +6 %)
    static constexpr uint64_t kLeanN = 1ull << 29;
    static constexpr uint64_t kEmitTopSlots = 2048;  // a large tree's top levels done by the one-CTA emission kernel
    static constexpr uint64_t kEmitSmallSlots = 1u << 14;  // trees this small: one emission kernel  // above: exact per-level sizing (one sync per level)
    uint32_t epoch_ = 0;
    uint32_t launches_ = 0;
    bool timing_ = false;
    std::vector<cudaEvent_t> events_;
    size_t ev_used_ = 0;
    cudaEvent_t ev_begin_ = nullptr, ev_end_ = nullptr;
    std::vector<TimedKernel> timed_;
    vqhull_stats stats_{};
    std::mutex mu_;
};

__global__ void iota_kernel(uint32_t* d, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        d[i] = uint32_t(i);
}

void Engine::iota(uint32_t* d, uint64_t n, cudaStream_t st) {
    iota_kernel<<<1184, 256, 0, st>>>(d, n);
}

__global__ void widen_kernel(const uint32_t* s, uint64_t* d, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        d[i] = s[i];
}

// ---------------------------------------------------------------------------
// engine registry (one per device)
// ---------------------------------------------------------------------------
namespace {
std::mutex g_reg_mu;
std::vector<std::unique_ptr<Engine>> g_engines;
thread_local bool g_timing = false;

Engine& engine_for(int dev) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    if (g_engines.size() <= size_t(dev)) g_engines.resize(dev + 1);
    if (!g_engines[dev]) g_engines[dev].reset(new Engine(dev));
    return *g_engines[dev];
}

Engine& engine() {
    int dev = 0;
    VQB_TRACE("engine(): cudaGetDevice");
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    return engine_for(dev);
}

// ---------------------------------------------------------------------------
// Single-process multi-GPU hull of host arrays: the
// points are cut into `shards` contiguous ranges, shard s runs on device
// s mod ndev (one host thread per device: its own H2D over its own PCIe link,
// its local hull and certificate, Engine::shard); the packed candidates are
// copied peer-to-peer to device 0, which merges them (Engine::merge).  Global
// indices are 64-bit, so n may exceed 2^32 - 1 as long as every shard stays
// below it.  More shards than devices run one after another per device
// (tests of the sharded path on one GPU).
// ---------------------------------------------------------------------------
int hull_multi(const double* xs, const double* ys, uint64_t n, int shards, uint64_t* out, uint64_t* count) {
    *count = 0;
    if (shards < 1) return VQHULL_EINVAL;
    if (n == 0) return VQHULL_OK;
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (ndev < 1) return VQHULL_ECUDA;
    const uint64_t S = uint64_t(shards);
    const uint64_t base = n / S, rem = n % S;
    if (base + (rem ? 1 : 0) >= 0xffffffffull) return VQHULL_ESIZE;
    std::vector<uint64_t> off(S), cnt(S), k(S, 0);
    for (uint64_t s = 0; s < S; ++s) {
        off[s] = s * base + std::min(s, rem);
        cnt[s] = base + (s < rem ? 1 : 0);
    }
    const int nd = int(std::min<uint64_t>(uint64_t(ndev), S));
    std::vector<void*> packs(S, nullptr);
    auto free_packs = [&] {
        for (uint64_t s = 0; s < S; ++s)
            if (packs[s]) {
                cudaSetDevice(int(s % uint64_t(nd)));
                cudaFree(packs[s]);
                packs[s] = nullptr;
            }
    };
    double floor_m = 0.0;
    int rc = VQHULL_OK;
    for (int attempt = 0; attempt < 2; ++attempt) {
        std::vector<int> rcs(nd, VQHULL_OK);
        std::vector<std::string> errs(nd);
        auto work = [&](int d) {
            try {
                ck(cudaSetDevice(d), "cudaSetDevice");
                Engine& e = engine_for(d);
                std::lock_guard<std::mutex> lk(e.mutex());
                cudaStream_t st = e.stream();
                for (uint64_t s = uint64_t(d); s < S; s += uint64_t(nd)) {
                    e.load_host(xs + off[s], ys + off[s], cnt[s], st);
                    int r = e.shard(e.in_x(), e.in_y(), cnt[s], off[s], floor_m, nullptr, 0, &k[s], st);
                    if (r) {
                        rcs[d] = r;
                        return;
                    }
                    if (packs[s]) cudaFree(packs[s]);
                    packs[s] = nullptr;
                    ck(cudaMalloc(&packs[s], (k[s] + 1) * 24), "cudaMalloc pack");
                    r = e.repack(static_cast<double*>(packs[s]), k[s], st);
                    if (r) {
                        rcs[d] = r;
                        return;
                    }
                    ck(cudaStreamSynchronize(st), "sync");
                }
            } catch (const CudaError&) {
                rcs[d] = VQHULL_ECUDA;
                errs[d] = g_last_error;
            }
        };
        std::vector<std::thread> th;
        for (int d = 1; d < nd; ++d) th.emplace_back(work, d);
        work(0);
        for (auto& t : th) t.join();
        for (int d = 0; d < nd; ++d)
            if (rcs[d]) {
                if (!errs[d].empty()) g_last_error = errs[d];
                free_packs();
                return rcs[d];
            }
        uint64_t kmax = 0;
        for (uint64_t s = 0; s < S; ++s) kmax = std::max(kmax, k[s]);
        const uint64_t stride = kmax + 1;
        ck(cudaSetDevice(0), "cudaSetDevice");
        Engine& e0 = engine_for(0);
        {
            std::lock_guard<std::mutex> lk(e0.mutex());
            cudaStream_t st = e0.stream();
            void* area = nullptr;
            ck(cudaMallocAsync(&area, S * stride * 24, st), "cudaMallocAsync merge area");
            for (uint64_t s = 0; s < S; ++s)
                ck(cudaMemcpyPeerAsync(static_cast<char*>(area) + s * stride * 24, 0, packs[s],
                                       int(s % uint64_t(nd)), (k[s] + 1) * 24, st),
                   "peer copy candidates");
            double fl = 0.0;
            try {
                rc = e0.merge(static_cast<const double*>(area), uint32_t(S), stride, out, count, &fl, st);
            } catch (...) {
                cudaFreeAsync(area, st);
                free_packs();
                throw;
            }
            ck(cudaFreeAsync(area, st), "cudaFreeAsync");
            ck(cudaStreamSynchronize(st), "sync");
            if (rc == VQHULL_ERETRY && attempt == 0) {
                floor_m = fl;
                continue;
            }
        }
        break;
    }
    free_packs();
    return rc;
}

// devices the drop-in entry point uses: VQHULL_GPUS, else 1 (or as many as
// the 32-bit per-device limit needs)
int compute_shards(uint64_t n) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
        cudaGetLastError();
        ndev = 0;
    }
    if (const char* e = getenv("VQHULL_GPUS")) {
        const int g = atoi(e);
        if (g >= 1) return g;
    }
    const uint64_t need = (n + 0xfffffffdull) / 0xfffffffeull;  // shards below 2^32 - 1 points
    return int(std::max<uint64_t>(1, need));
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
}  // namespace

}  // namespace vqb

// ===========================================================================
// C ABI
// ===========================================================================
using vqb::CudaError;
using vqb::Engine;

extern "C" {

const char* vqhull_b200_version(void) { return "vqhull-b200 0.1 (sm_100a)"; }

const char* vqhull_cuda_last_error(void) { return vqb::g_last_error.c_str(); }

int vqhull_cuda_available(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n > 0 ? 1 : 0;
}

int vqhull_cuda_set_timing(int enable) {
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        e.set_timing(enable != 0);
        return 0;
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_set_stable(int stable) {
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        e.set_stable(stable != 0);
        return 0;
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_trim(void) {
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        e.trim();
        return 0;
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_set_root_mode(int mode) {
    if (mode < 0 || mode > 2) return VQHULL_EINVAL;
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        e.set_root_mode(mode);
        return 0;
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_set_filter_inner(int mode) {
    if (mode < -1 || mode > 3) return VQHULL_EINVAL;
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        vqb::set_filter_inner(mode);
        return 0;
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_set_root_reference(int reference) {
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        e.set_root_reference(reference != 0);
        return 0;
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_get_stats(vqhull_stats* out) {
    if (!out) return VQHULL_EINVAL;
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        *out = e.stats();
        return 0;
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_compute(const double* xs, const double* ys, size_t n, int workers, size_t* out_indices,
                   size_t* out_count) {
    // argument checks of the reference, in its order (vqhull_c.cpp:29-34);
    // the finiteness scan is fused into the bootstrap kernel
    if (!out_count || workers < 1) return VQHULL_EINVAL;
    *out_count = 0;
    if (n == 0) return VQHULL_OK;
    if (!xs || !ys || !out_indices) return VQHULL_EINVAL;
    try {
        // several GPUs (VQHULL_GPUS, or n beyond one device's 32-bit range)
        const int shards = vqb::compute_shards(n);
        if (shards > 1 || getenv("VQHULL_GPUS")) {
            static_assert(sizeof(size_t) == sizeof(uint64_t), "size_t is 64-bit");
            uint64_t h = 0;
            const int rc = vqb::hull_multi(xs, ys, n, shards, reinterpret_cast<uint64_t*>(out_indices), &h);
            if (rc) return rc;
            *out_count = size_t(h);
            return VQHULL_OK;
        }
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        std::vector<uint32_t> tmp;
        uint32_t* dst = reinterpret_cast<uint32_t*>(out_indices);  // widened in place below
        uint64_t h = 0;
        const int rc = e.compute_host(xs, ys, n, dst, &h, nullptr);
        if (rc) return rc;
        // widen u32 -> size_t in place, back to front
        for (uint64_t i = h; i-- > 0;) out_indices[i] = size_t(dst[i]);
        *out_count = size_t(h);
        return VQHULL_OK;
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_hull_u32(const double* d_xs, const double* d_ys, uint64_t n, uint32_t* d_out,
                         uint64_t* out_count, void* stream) {
    if (!out_count) return VQHULL_EINVAL;
    *out_count = 0;
    if (n == 0) return VQHULL_OK;
    if (!d_xs || !d_ys || !d_out) return VQHULL_EINVAL;
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        uint64_t h = 0;
        const int rc = e.hull(d_xs, d_ys, n, d_out, &h, static_cast<cudaStream_t>(stream));
        if (rc) return rc;
        *out_count = h;
        return VQHULL_OK;
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_hull(const double* d_xs, const double* d_ys, uint64_t n, uint64_t* out_indices,
                     uint64_t* out_count, void* stream) {
    if (!out_count) return VQHULL_EINVAL;
    *out_count = 0;
    if (n == 0) return VQHULL_OK;
    if (!d_xs || !d_ys || !out_indices) return VQHULL_EINVAL;
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        e.out_buf().ensure(n * 4, st);
        uint64_t h = 0;
        const int rc = e.hull(d_xs, d_ys, n, e.out_buf().as<uint32_t>(), &h, st);
        if (rc) return rc;
        if (h) {
            if (vqb::is_device_ptr(out_indices)) {
                vqb::widen_kernel<<<592, 256, 0, st>>>(e.out_buf().as<uint32_t>(), out_indices, h);
                vqb::ck(cudaStreamSynchronize(st), "sync");
            } else {
                std::vector<uint32_t> tmp(h);
                vqb::ck(cudaMemcpyAsync(tmp.data(), e.out_buf().p, h * 4, cudaMemcpyDeviceToHost, st), "d2h");
                vqb::ck(cudaStreamSynchronize(st), "sync");
                for (uint64_t i = 0; i < h; ++i) out_indices[i] = tmp[i];
            }
        }
        *out_count = h;
        return VQHULL_OK;
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_find_extremes(const double* d_xs, const double* d_ys, uint64_t n, uint64_t* lo,
                              uint64_t* hi, void* stream) {
    if (!lo || !hi) return VQHULL_EINVAL;
    if (n > 0 && (!d_xs || !d_ys)) return VQHULL_EINVAL;
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        return e.find_extremes(d_xs, d_ys, n, lo, hi, static_cast<cudaStream_t>(stream));
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_extract_subsets(double* d_xs, double* d_ys, uint64_t n, const double* edge_a,
                                const double* edge_b, uint64_t* w_l, uint64_t* w_r, double* r1,
                                int* has_r1, double* r2, int* has_r2, void* stream) {
    if (!edge_a || !edge_b || !w_l || !w_r || !r1 || !r2 || !has_r1 || !has_r2) return VQHULL_EINVAL;
    if (n > 0 && (!d_xs || !d_ys)) return VQHULL_EINVAL;
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        return e.extract(d_xs, d_ys, n, edge_a, edge_b, w_l, w_r, r1, has_r1, r2, has_r2,
                         static_cast<cudaStream_t>(stream));
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_hull_multi(const double* xs, const double* ys, uint64_t n, int num_shards,
                           uint64_t* out_indices, uint64_t* out_count) {
    if (!out_count) return VQHULL_EINVAL;
    *out_count = 0;
    if (n == 0) return VQHULL_OK;
    if (!xs || !ys || !out_indices || num_shards < 1) return VQHULL_EINVAL;
    try {
        return vqb::hull_multi(xs, ys, n, num_shards, out_indices, out_count);
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_shard_candidates(const double* d_xs, const double* d_ys, uint64_t n, uint64_t offset,
                                 double margin_floor, double* d_pack, uint64_t cap_rows, uint64_t* count,
                                 void* stream) {
    if (!count) return VQHULL_EINVAL;
    *count = 0;
    if (n > 0 && (!d_xs || !d_ys)) return VQHULL_EINVAL;
    if (!(margin_floor >= 0.0)) return VQHULL_EINVAL;
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        return e.shard(d_xs, d_ys, n, offset, margin_floor, d_pack, cap_rows, count,
                       static_cast<cudaStream_t>(stream));
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_shard_repack(double* d_pack, uint64_t cap_rows, void* stream) {
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        return e.repack(d_pack, cap_rows, static_cast<cudaStream_t>(stream));
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

int vqhull_cuda_merge_candidates(const double* d_packs, uint32_t nranks, uint64_t stride_rows,
                                 uint64_t* out_indices, uint64_t* out_count, double* margin_floor,
                                 void* stream) {
    if (!out_count || !d_packs || !out_indices) return VQHULL_EINVAL;
    *out_count = 0;
    try {
        Engine& e = vqb::engine();
        std::lock_guard<std::mutex> lk(e.mutex());
        return e.merge(d_packs, nranks, stride_rows, out_indices, out_count, margin_floor,
                       static_cast<cudaStream_t>(stream));
    } catch (const CudaError&) {
        return VQHULL_ECUDA;
    }
}

}  // extern "C"
