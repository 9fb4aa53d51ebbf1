// KC: the cluster-resident recursion (included by device.cu).
//
// After the split root's filter pass, most inputs leave a few tens of
// thousands of survivors (square 1e8: ~47k; disk 1e6: ~25k) whose recursion
// is a handful of narrow levels.  KT runs those levels on the whole GPU with
// two grid barriers and chains of L2 round trips per level (~15 us each).
// KC runs them in ONE thread-block cluster (16 CTAs, distributed shared
// memory): every CTA holds a contiguous share of the survivors in shared
// memory for the whole recursion, and the points never move — each carries
// the id of its node, then of its child, exactly like the CTA finisher.  Per
// level (the reference's chain_recursive, hull.cpp:78-115, breadth-first):
//   (1) every CTA classifies its points against their node's (p->r), (r->q)
//       with the reference's exact predicates (left_diff, kernels.hpp:28-30;
//       mask_b &= ~mask_a, :91) and accumulates, per child, its point count
//       and minimal farthest key (the canonical order of kernels.hpp:41-45);
//   cluster barrier;
//   (2) every CTA reduces the 16 CTAs' counts and keys over DSMEM (the same
//       values in every CTA: no broadcast round) and marks its own points
//       holding a child's minimal key (ties inside a CTA: smaller (x, y),
//       then smaller input index);
//   cluster barrier;
//   (3) every CTA picks each child's apex among the 16 CTAs' candidates (an
//       exact tie across CTAs: the same order), builds the next level's node
//       table (children with >= 2 points; one-point children are leaves,
//       hull.cpp:83) and re-labels its points; CTA 0 records the tree.
// Per-CTA accumulators are double-buffered by level parity, so a CTA never
// clears an array another CTA may still be reading: two cluster barriers per
// level.  CTA 0 then writes the clockwise list [p] chain(root)
// (assemble_chain, hull.cpp:59-73; hull.cpp:259-266) and KT's report.  KC
// hands the call to KT (which then runs as before) when the survivors do not
// fit, a level has more than kKcNodes nodes, or the tree outgrows its tables.
#include <cooperative_groups.h>

namespace vqb {

namespace kc_cg = cooperative_groups;

constexpr int kKcCtas = 16;         // cluster size (non-portable: 16 CTAs of one GPC)
constexpr int kKcThreads = 512;
constexpr int kKcPts = 4096;        // survivors per CTA (capacity 64k)
constexpr int kKcNodes = 256;       // nodes per level
constexpr int kKcChildren = 2 * kKcNodes;
constexpr int kKcTree = 2048;       // internal tree nodes (hull vertices from internal nodes)
constexpr int kKcLeaves = 2048;
constexpr int kKcLevels = kTailLevels - 1;
constexpr int kKcWarps = kKcThreads / 32;
constexpr int kKcWarpPts = kKcPts / kKcWarps;  // points a warp owns (256)
constexpr int kKcRounds = kKcWarpPts / 32;     // its rounds of 32 (8)
constexpr uint32_t kKcNone = 0xffffffffu;
constexpr uint16_t kKcDead = 0xffffu;

struct KcNode {
    double px, py, rx, ry, qx, qy;
};

struct KcSmem {
    double x[kKcPts];
    double y[kKcPts];
    uint16_t pn[kKcPts];                    // node id (between levels) / child id (in a level) / dead
    uint16_t lst[kKcThreads / 32][kKcPts / (kKcThreads / 32)];  // each warp's live points
    // per child, double-buffered by level parity (read remotely over DSMEM)
    uint32_t lcnt[2][kKcChildren];
    unsigned long long lkey[2][kKcChildren];
    uint32_t lncand[2][kKcChildren];
    uint32_t lcand[2][kKcChildren];         // local index of this CTA's candidate
    // replicated per-level state (every CTA computes the same values)
    KcNode node[2][kKcNodes];
    uint16_t ntree[2][kKcNodes];            // tree id of each node
    uint32_t gcnt[kKcChildren];
    unsigned long long gkey[kKcChildren];
    uint16_t cmap[kKcChildren];
    uint32_t wsum[kKcThreads / 32], wsum2[kKcThreads / 32];
    uint16_t tlist[kKcPts];                 // local extra candidates (ties)
    uint32_t ntie;
    // the tree (CTA 0): internal nodes t: apex (rank << 16 | local index), links (kind | id)
    uint32_t tapex[kKcTree];
    uint32_t tleft[kKcTree], tright[kKcTree];
    uint32_t tsize[kKcTree], tstart[kKcTree];
    uint32_t leaf_gid[kKcLeaves];
    uint16_t lvl_start[kKcLevels + 2];
    LevelInfo info[kKcLevels + 1];
    uint32_t bail;
};
constexpr uint32_t kKcLinkEmpty = 0, kKcLinkLeaf = 0x40000000u, kKcLinkNode = 0x80000000u;

__device__ __forceinline__ uint32_t kc_link_size(const KcSmem& S, uint32_t l) {
    return (l & kKcLinkNode) ? S.tsize[l & 0x3fffffffu] : ((l & kKcLinkLeaf) ? 1u : 0u);
}

__global__ void __launch_bounds__(kKcThreads, 1) cluster_tail_kernel(const __grid_constant__ TailArgs A) {
    VQB_PDL();
    extern __shared__ __align__(16) unsigned char kc_dsm[];
    KcSmem& S = *reinterpret_cast<KcSmem*>(kc_dsm);
    kc_cg::cluster_group cluster = kc_cg::this_cluster();
    const uint32_t rank = cluster.block_rank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned lt = lanemask_lt();
    const ChildRec slot = A.lv[0].slots[0];   // the bootstrap triangle (p, q, p) over the survivors
    const uint32_t m = slot.m;
    // hand the call to KT: nothing to do here, or too many points
    if (m < 2 || m > uint32_t(kKcCtas * kKcPts)) {
        if (rank == 0 && tid == 0) *A.kc_done = 0u;
        return;
    }
    const uint32_t lo = uint32_t((uint64_t(rank) * m) / kKcCtas);
    const uint32_t hi = uint32_t((uint64_t(rank + 1) * m) / kKcCtas);
    const uint32_t np = hi - lo;
    const double* gx = A.bx[0];
    const double* gy = A.by[0];
    const uint32_t* gid = A.bid[0];
    for (uint32_t i = tid; i < np; i += kKcThreads) {
        S.x[i] = gx[lo + i];
        S.y[i] = gy[lo + i];
        S.pn[i] = 0;
    }
    // warp w owns points [w * P, (w + 1) * P) and walks only its live ones
    const uint32_t P = (np + kKcWarps - 1) / kKcWarps;
    uint32_t wn = warp * P < np ? min(P, np - warp * P) : 0u;  // (warp-uniform)
    for (uint32_t j = lane; j < wn; j += 32) S.lst[warp][j] = uint16_t(warp * P + j);
    for (uint32_t c = tid; c < 2u * kKcChildren; c += kKcThreads) {
        const uint32_t b = c / kKcChildren, k = c % kKcChildren;
        S.lcnt[b][k] = 0;
        S.lkey[b][k] = kNoKey;
        S.lncand[b][k] = 0;
        S.lcand[b][k] = kKcNone;
    }
    if (tid == 0) {
        KcNode& r0 = S.node[0][0];
        r0.px = slot.px; r0.py = slot.py; r0.rx = slot.rx; r0.ry = slot.ry; r0.qx = slot.qx; r0.qy = slot.qy;
        S.ntree[0][0] = 0;
        S.tapex[0] = slot.r_idx;
        S.tleft[0] = kKcLinkEmpty;
        S.tright[0] = kKcLinkEmpty;
        S.lvl_start[0] = 0;
        S.lvl_start[1] = 1;
        S.ntie = 0;
        S.bail = 0;
        LevelInfo& li = S.info[0];
        li.nslots = 1; li.nseg = 1; li.nfin = 0; li.ntiles = 0; li.out_total = m; li.fin_total = 0;
        li.nleaf = 0; li.fin_base = 0; li.nfin2 = 0; li.pad = 0;
    }
    cluster.sync();  // every CTA's accumulators are clear before anyone accumulates
    uint32_t nn = 1, ntree = 1, nleaf = 0;
    int cur = 0, depth = 0;
    bool ok = true;
    while (true) {
        const int b = depth & 1, nxt = cur ^ 1;
        // (1) classify this CTA's live points; per-child counts and minimal
        // keys (each lane's keys stay in registers for the candidate pass)
        uint32_t chv[kKcRounds];
        unsigned long long keyv[kKcRounds];
#pragma unroll
        for (int k = 0; k < kKcRounds; ++k) {
            chv[k] = kKcNone;
            keyv[k] = kNoKey;
            if (uint32_t(k) * 32 >= wn) continue;  // (warp-uniform)
            const uint32_t j = uint32_t(k) * 32 + lane;
            uint32_t ch = kKcNone;
            unsigned long long key = kNoKey;
            if (j < wn) {
                const uint32_t i = S.lst[warp][j];
                const uint16_t c = S.pn[i];
                const KcNode& nd = S.node[cur][c];
                const double u = S.x[i], w = S.y[i];
                const double Aa = dsub(nd.px, u), B = dsub(nd.py, w);
                const double E = dsub(nd.rx, u), F = dsub(nd.ry, w);
                const double Cc = dsub(nd.qx, u), D = dsub(nd.qy, w);
                const bool la = left_diff(Aa, B, E, F);
                const bool lb = !la && left_diff(E, F, Cc, D);
                if (la || lb) {
                    ch = 2u * c + (lb ? 1u : 0u);
                    const double fx = lb ? dsub(nd.qx, nd.rx) : dsub(nd.rx, nd.px);
                    const double fy = lb ? dsub(nd.qy, nd.ry) : dsub(nd.ry, nd.py);
                    key = key_of(lat_off(fx, fy, u, w));
                    S.pn[i] = uint16_t(ch);
                } else {
                    S.pn[i] = kKcDead;
                }
            }
            chv[k] = ch;
            keyv[k] = key;
            const unsigned grp = __match_any_sync(kFull, ch);
            if (grp == kFull) {  // the whole warp in one child (or none)
#pragma unroll
                for (int s = 16; s > 0; s >>= 1) {
                    const unsigned long long o = __shfl_xor_sync(kFull, key, s);
                    key = o < key ? o : key;
                }
                if (ch != kKcNone && lane == 0) {
                    atomicAdd(&S.lcnt[b][ch], 32u);
                    if (key < S.lkey[b][ch]) atomicMin(&S.lkey[b][ch], key);
                }
            } else if (ch != kKcNone) {
                if (lane == __ffs(grp) - 1) atomicAdd(&S.lcnt[b][ch], uint32_t(__popc(grp)));
                if (key < S.lkey[b][ch]) atomicMin(&S.lkey[b][ch], key);
            }
        }
        cluster.sync();  // A: every CTA's counts and keys of this level
        // (2) cluster-wide counts and minimal keys (each CTA, redundantly)
        const uint32_t nch = 2 * nn;
        for (uint32_t c = tid; c < nch; c += kKcThreads) {
            uint32_t cv[kKcCtas];
            unsigned long long kv[kKcCtas];
#pragma unroll
            for (int r = 0; r < kKcCtas; ++r) {  // all 32 remote loads in flight at once
                const KcSmem* R = cluster.map_shared_rank(&S, r);
                cv[r] = R->lcnt[b][c];
                kv[r] = R->lkey[b][c];
            }
            uint32_t cnt = 0;
            unsigned long long key = kNoKey;
#pragma unroll
            for (int r = 0; r < kKcCtas; ++r) {
                cnt += cv[r];
                key = kv[r] < key ? kv[r] : key;
            }
            S.gcnt[c] = cnt;
            S.gkey[c] = key;
        }
        __syncthreads();
        // this CTA's candidates: its points holding their child's minimal key
#pragma unroll
        for (int k = 0; k < kKcRounds; ++k) {
            const uint32_t ch = chv[k];
            if (ch == kKcNone || keyv[k] != S.gkey[ch]) continue;
            const uint32_t i = S.lst[warp][uint32_t(k) * 32 + lane];
            if (atomicAdd(&S.lncand[b][ch], 1u) == 0) S.lcand[b][ch] = i;
            else S.tlist[atomicAdd(&S.ntie, 1u)] = uint16_t(i);
        }
        __syncthreads();
        if (S.ntie) {  // ties inside this CTA: smaller (x, y), then smaller input index
            if (tid == 0) {
                for (uint32_t t = 0; t < S.ntie; ++t) {
                    const uint32_t i = S.tlist[t];
                    const uint16_t ch = S.pn[i];
                    const uint32_t bc = S.lcand[b][ch];
                    const bool better = S.x[i] != S.x[bc] ? S.x[i] < S.x[bc]
                                      : (S.y[i] != S.y[bc] ? S.y[i] < S.y[bc] : gid[lo + i] < gid[lo + bc]);
                    if (better) S.lcand[b][ch] = i;
                }
                S.ntie = 0;
            }
            __syncthreads();
        }
        cluster.sync();  // B: every CTA's candidates
        // (3) apexes across the cluster (each CTA, redundantly): the 16 CTAs'
        // candidate slots at once, then the coordinates of the (almost always
        // single) candidate; the apex is recorded as (rank, local index) and
        // its input index looked up only at emission
        // (nch <= kKcChildren <= kKcThreads: child c = tid, so the apex stays in
        // this thread's registers for the node table below — no barrier between)
        double apx = 0.0, apy = 0.0;
        uint32_t apref = kKcNone;
        if (tid < nch) {
            const uint32_t c = tid;
            uint32_t lv[kKcCtas];
#pragma unroll
            for (int r = 0; r < kKcCtas; ++r) lv[r] = cluster.map_shared_rank(&S, r)->lcand[b][c];
            double bx = 0.0, by = 0.0;
            uint32_t bref = kKcNone;
            int ncand = 0, r1 = 0;
            uint32_t l1 = 0;
#pragma unroll
            for (int r = 0; r < kKcCtas; ++r)
                if (lv[r] != kKcNone) {
                    ++ncand;
                    r1 = r;
                    l1 = lv[r];
                }
            if (ncand == 1) {
                const KcSmem* R = cluster.map_shared_rank(&S, r1);
                bx = R->x[l1];
                by = R->y[l1];
                bref = (uint32_t(r1) << 16) | l1;
            } else if (ncand > 1) {  // an exact key tie across CTAs: smaller (x, y), then index
                uint32_t bg = kKcNone;
                for (int r = 0; r < kKcCtas; ++r) {
                    if (lv[r] == kKcNone) continue;
                    const KcSmem* R = cluster.map_shared_rank(&S, r);
                    const double x = R->x[lv[r]], y = R->y[lv[r]];
                    const uint32_t g = gid[uint32_t((uint64_t(r) * m) / kKcCtas) + lv[r]];
                    if (bg == kKcNone || (x != bx ? x < bx : (y != by ? y < by : g < bg))) {
                        bx = x;
                        by = y;
                        bg = g;
                        bref = (uint32_t(r) << 16) | lv[r];
                    }
                }
            }
            apx = bx;
            apy = by;
            apref = bref;
        }
        // next level's nodes (block scan over the internal children), leaves, links
        uint32_t nnext = 0, nlv = 0, out_pts = 0;
        {
            const uint32_t c = tid;  // nch <= kKcChildren <= kKcThreads: one child per thread
            const bool valid = c < nch;
            const uint32_t cnt = valid ? S.gcnt[c] : 0u;
            const bool internal = cnt >= 2, leaf = cnt == 1;
            const unsigned bi = __ballot_sync(kFull, internal), bl = __ballot_sync(kFull, leaf);
            uint32_t pts = internal ? cnt : 0u;
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) pts += __shfl_xor_sync(kFull, pts, s);
            if (lane == 0) {
                S.wsum[warp] = uint32_t(__popc(bi)) | (uint32_t(__popc(bl)) << 16);
                S.wsum2[warp] = pts;
            }
            __syncthreads();
            uint32_t basei = 0, basel = 0;
            for (int w = 0; w < kKcThreads / 32; ++w) {
                const uint32_t v = S.wsum[w];
                if (w < warp) {
                    basei += v & 0xffffu;
                    basel += v >> 16;
                }
                nnext += v & 0xffffu;
                nlv += v >> 16;
                out_pts += S.wsum2[w];
            }
            const bool fits = nnext <= uint32_t(kKcNodes) && ntree + nnext <= uint32_t(kKcTree) &&
                              nleaf + nlv <= uint32_t(kKcLeaves) && depth + 1 < kKcLevels;
            if (fits && valid) {
                const uint32_t nid = basei + __popc(bi & lt);
                const uint32_t lid = nleaf + basel + __popc(bl & lt);
                const int pc = int(c >> 1), side = int(c & 1);
                const KcNode& nd = S.node[cur][pc];
                uint32_t link = kKcLinkEmpty;
                uint16_t map = kKcDead;
                if (internal) {
                    const uint32_t tnew = ntree + nid;
                    KcNode& nn2 = S.node[nxt][nid];
                    nn2.px = side ? nd.rx : nd.px;
                    nn2.py = side ? nd.ry : nd.py;
                    nn2.qx = side ? nd.qx : nd.rx;
                    nn2.qy = side ? nd.qy : nd.ry;
                    nn2.rx = apx;
                    nn2.ry = apy;
                    S.ntree[nxt][nid] = uint16_t(tnew);
                    link = kKcLinkNode | tnew;
                    map = uint16_t(nid);
                    if (rank == 0) {
                        S.tapex[tnew] = apref;
                        S.tleft[tnew] = kKcLinkEmpty;
                        S.tright[tnew] = kKcLinkEmpty;
                    }
                } else if (leaf) {
                    link = kKcLinkLeaf | lid;
                    if (rank == 0) S.leaf_gid[lid] = apref;
                }
                S.cmap[c] = map;
                if (rank == 0) {
                    const uint32_t t = S.ntree[cur][pc];
                    if (side) S.tright[t] = link;
                    else S.tleft[t] = link;
                }
            }
            if (!fits) ok = false;
        }
        if (!ok) break;  // (uniform: every thread saw the same totals)
        // the other accumulator buffer for the next level: its last remote
        // readers finished before barrier A of this level
        for (uint32_t c = tid; c < 2 * nnext; c += kKcThreads) {
            S.lcnt[b ^ 1][c] = 0;
            S.lkey[b ^ 1][c] = kNoKey;
            S.lncand[b ^ 1][c] = 0;
            S.lcand[b ^ 1][c] = kKcNone;
        }
        __syncthreads();  // cmap complete
        {  // points follow their child to its next node id; the warp's live list shrinks in place
            uint32_t w2 = 0;
            for (uint32_t j0 = 0; j0 < wn; j0 += 32) {
                const uint32_t j = j0 + lane;
                uint32_t i = 0;
                bool alive = false;
                if (j < wn) {
                    i = S.lst[warp][j];
                    const uint16_t ch = S.pn[i];
                    const uint16_t nd = ch == kKcDead ? kKcDead : S.cmap[ch];
                    S.pn[i] = nd;
                    alive = nd != kKcDead;
                }
                const unsigned bal = __ballot_sync(kFull, alive);
                __syncwarp();  // every lane has read its entry before any is overwritten
                if (alive) S.lst[warp][w2 + __popc(bal & lt)] = uint16_t(i);
                w2 += __popc(bal);
            }
            wn = w2;
        }
        ntree += nnext;
        nleaf += nlv;
        ++depth;
        if (tid == 0) {
            S.lvl_start[depth + 1] = uint16_t(ntree);
            LevelInfo& li = S.info[depth];
            li.nslots = nch; li.nseg = nnext; li.nfin = 0; li.ntiles = 0; li.out_total = out_pts;
            li.fin_total = 0; li.nleaf = nlv; li.fin_base = 0; li.nfin2 = 0; li.pad = 0;
        }
        nn = nnext;
        cur = nxt;
        // (no barrier: the relabelling above is warp-local, and everything the
        // next level reads was complete at "cmap complete")
        if (nn == 0) break;
    }
    cluster.sync();  // no CTA leaves while another may read its shared memory
    if (rank != 0) return;
    if (!ok) {
        if (tid == 0) *A.kc_done = 0u;
        return;
    }
    // [p] chain(root): subtree sizes bottom-up, positions top-down
    for (int d = depth - 1; d >= 0; --d) {
        for (uint32_t t = S.lvl_start[d] + tid; t < S.lvl_start[d + 1]; t += kKcThreads)
            S.tsize[t] = kc_link_size(S, S.tleft[t]) + 1u + kc_link_size(S, S.tright[t]);
        __syncthreads();
    }
    if (tid == 0) S.tstart[0] = 1;  // out[0] = p
    __syncthreads();
    uint32_t* out = A.out;
    auto ref_gid = [&](uint32_t ref) {  // (rank, local index) -> input index
        const uint32_t r = ref >> 16, li = ref & 0xffffu;
        return gid[uint32_t((uint64_t(r) * m) / kKcCtas) + li];
    };
    for (uint32_t t = tid + 1; t < ntree; t += kKcThreads) S.tapex[t] = ref_gid(S.tapex[t]);  // (0: the root's q)
    for (uint32_t t = tid; t < nleaf; t += kKcThreads) S.leaf_gid[t] = ref_gid(S.leaf_gid[t]);
    __syncthreads();
    for (int d = 0; d < depth; ++d) {
        for (uint32_t t = S.lvl_start[d] + tid; t < S.lvl_start[d + 1]; t += kKcThreads) {
            const uint32_t s0 = S.tstart[t];
            const uint32_t L = S.tleft[t], R = S.tright[t];
            const uint32_t ap = s0 + kc_link_size(S, L);
            out[ap] = S.tapex[t];
            if (L & kKcLinkLeaf) out[s0] = S.leaf_gid[L & 0x3fffffffu];
            else if (L & kKcLinkNode) S.tstart[L & 0x3fffffffu] = s0;
            if (R & kKcLinkLeaf) out[ap + 1] = S.leaf_gid[R & 0x3fffffffu];
            else if (R & kKcLinkNode) S.tstart[R & 0x3fffffffu] = ap + 1;
        }
        __syncthreads();
    }
    // KT's report: finished and emitted at level l0 + depth
    uint32_t* r = A.report;
    if (tid == 0) {
        const uint32_t h = 1u + S.tsize[0];
        out[0] = *A.p_idx;
        *A.h_out = h;
        const RootInfo* Rt = A.root;
        r[0] = uint32_t(A.l0 + depth);
        r[1] = 3u;
        r[2] = h;
        r[3] = Rt->nonfinite;
        r[4] = Rt->unsafe;
        r[5] = Rt->poly.filter;
        r[6] = Rt->cnt1;
        r[7] = *reinterpret_cast<volatile uint32_t*>(&g_vqb_fault);
        A.state[0] = uint32_t(A.l0 + depth);
        A.state[1] = 3u;
        *A.kc_done = 1u;
    }
    const uint32_t* src = reinterpret_cast<const uint32_t*>(S.info);
    const uint32_t words = uint32_t(depth + 1) * uint32_t(sizeof(LevelInfo) / 4);
    for (uint32_t i = tid; i < words; i += kKcThreads) r[8 + i] = src[i];
}

size_t kc_smem_bytes() { return sizeof(KcSmem); }

// 0 when the device cannot host the cluster (the caller then skips KC)
int kc_prepare() {
    cudaFuncSetAttribute(cluster_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(KcSmem)));
    cudaFuncSetAttribute(cluster_tail_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kKcCtas);
    cfg.blockDim = dim3(kKcThreads);
    cfg.dynamicSmemBytes = sizeof(KcSmem);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kKcCtas;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, cluster_tail_kernel, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return clusters;
}

cudaError_t launch_cluster_tail(const TailArgs& a, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kKcCtas);
    cfg.blockDim = dim3(kKcThreads);
    cfg.dynamicSmemBytes = sizeof(KcSmem);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kKcCtas;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, cluster_tail_kernel, a);
}

}  // namespace vqb
