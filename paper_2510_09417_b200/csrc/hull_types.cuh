// Device data layout of the B200 VQhull driver.
#pragma once

#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace vqb {

// Points in HBM are structure-of-arrays, as in the reference PointSet
// (geometry.hpp:86-125): x[], y[] as f64, plus the carried u32 input index in
// every buffer after the root pass (the root pass reads the caller's arrays
// and uses the position as the index).

constexpr int kThreads = 256;               // partition CTA size
constexpr int kItems = 4;                   // points per thread per tile
constexpr int kTile = kThreads * kItems;    // points per partition tile
constexpr int kWarps = kThreads / 32;
constexpr int kPartMinBlocks = 3;           // resident partition CTAs per SM (register cap)
constexpr int kFastMinBlocks = 4;           // fast-mode kernels (no staging)
constexpr uint32_t kFinSmall = 64;          // segments of 2..64 points: warp finisher
#ifndef VQB_FIN_MAX
#define VQB_FIN_MAX 768
#endif
constexpr uint32_t kFinMax = VQB_FIN_MAX;           // 65..768 points: CTA finisher (4 per SM; 1024: 3 per SM, 8 % slower on circle 1e7); larger: tiled level kernel
constexpr uint32_t kTailFinMax = 1024;      // inside the persistent tail kernel (2048 measured: faster on disk 1e6, slower on square 1e8 and disk 1e7)

// Root stage geometry.  The recursion itself always follows the reference
// (level 1 splits by p->q, hull.cpp:228-235); a polygon of kPolyV input
// points (directional extremes of a sample) is only a FILTER in front of it:
// a point provably inside the polygon by a margin far above the predicates'
// rounding can never be a farthest point or a lone subset member, so dropping
// it cannot change the reference's output.
//  * vx/vy/vidx: V_j = the sample's extreme along direction j, the 16
//    directions (-1,0), (-2,1), (-1,1), (-1,2), (0,1), (1,2), (1,1), (2,1),
//    (1,0), ... clockwise from -x; chord j = V_j -> V_{j+1 mod 16};
//  * two inner regions verified inside the filter region, tested before any
//    chord: an open box (every point) and an octagon = box' ∩ diamond
//    (points outside the box);
//  * emission frame: nv vertices, slot j between V_j and V_{j+1}, repeated
//    vertices written once: nv = 2 (p, q) for the one-pass filtered root,
//    4 (p, r1, q, r2) for the fused levels-1+2 root, 1 (p) for the split root.
constexpr int kPolyV = 16;
struct RootPoly {
    double vx[kPolyV], vy[kPolyV];
    uint32_t vidx[kPolyV];
    double ex[4], ey[4];        // emission frame vertices
    uint32_t eidx[4];
    uint32_t nv;
    uint32_t filter;            // 1: the polygon filter may drop points
    // chord j as a linear form f_j(P) = fa*x + fb*y + fc = cross(V_{j+1} - V_j,
    // P - V_j) (> 0: left of the chord, outside); P is dropped when
    // f_j(P) < ft_j for all chords (ft_j = -margin * |chord|_1)
    double fa[kPolyV], fb[kPolyV], fc[kPolyV], ft[kPolyV];
    // the pass kernels' form of the test: fma(fa, x, fb * y) < fg = ft - fc
    // (two constant operands per chord, error <= ~6 eps |e| M << margin)
    double fg[kPolyV];
    double bx0, bx1, by0, by1;  // open box verified to lie inside the filter region
    // octagon |x - ocx| < ohx, |y - ocy| < ohy, |x - ocx| + |y - ocy| < od,
    // verified (its 8 vertices) to lie inside the filter region
    double ocx, ocy, ohx, ohy, od;
    // disk |P - (dcx, dcy)|^2 < dr2 (radius: the distance to the nearest chord
    // line, shrunk), by construction inside every chord's margin
    double dcx, dcy, dr2;
    uint32_t oct_on;            // K_F's fast inner test: 0 box, 1 box | octagon, 2 box | disk (the largest area)
    uint32_t pad2;
    double mref;                // M: max |coordinate| of the vertices (the margin is 2^-32 M)
};

// K1 + pass A results, one per hull call (device resident).
struct RootInfo {
    // K1: find_extremes (geometry.cpp:7-36)
    uint32_t p_idx, q_idx;
    double px, py, qx, qy;
    // pass A: bootstrap partition counts + arg-max (hull.cpp:228-235)
    uint32_t cnt1, cnt2;
    Best r1, r2;
    uint32_t nonfinite;
    uint32_t unsafe;            // split root: a survivor exceeds 2^12 M (margin argument void) -> rerun unfiltered
    RootPoly poly;
};

// One node of the recursion tree as produced by its parent's partition:
// triangle (p, r, q) where r is the node's apex (its hull vertex), and the
// node's candidate points, which live contiguously at [begin, begin+m) of the
// buffer the parent wrote.  hull.cpp:95-112 (chain_recursive children).
struct ChildRec {
    double px, py, rx, ry, qx, qy;
    uint64_t begin;
    uint32_t m;
    uint32_t r_idx;
};

// A node that is partitioned by the tiled level kernel (m > kFinMax).
// Edge A = p->r, edge B = b->q (b == r except for the general-edge extract
// API).  Frames: (adx, ady) = r - p, (bdx, bdy) = q - b  (kernels.hpp:23-25).
struct SegRec {
    double px, py, rx, ry, qx, qy;
    double bx, by;
    double adx, ady, bdx, bdy;
    uint64_t begin;   // input buffer position of the first point
    uint64_t out;     // output buffer base of its two-sided range
    uint32_t m;
    uint32_t tile0;   // first tile id of this segment in the level launch
    uint32_t ntiles;
    uint32_t slot;    // this node's slot in the level's slot table
};

// A node solved entirely by one warp (m <= kFinSmall) or one CTA (m <= kFinMax).
struct FinRec {
    ChildRec c;
    uint64_t chain_base;  // where its in-order chain is written
    uint32_t slot;
    uint32_t pad;
};

// Node kinds in the slot tables.
enum : uint8_t { kEmpty = 0, kLeaf = 1, kFin = 2, kInternal = 3 };

// Per-level planner output.
struct LevelInfo {
    uint32_t nslots;
    uint32_t nfin;
    // (nseg, ntiles) and (fin_total, nfin2) are 8-byte aligned pairs: the level
    // kernels advance each pair with ONE packed 64-bit atomic per planned child
    uint32_t nseg;
    uint32_t ntiles;
    uint32_t out_total;   // points handed to the level kernel
    uint32_t nleaf;
    uint32_t fin_total;   // points handed to the finisher
    uint32_t nfin2;       // CTA-finisher segments (FinRec array from the back)
    uint32_t fin_base;    // first chain entry of this level's finisher segments
    uint32_t pad;
};
static_assert(offsetof(LevelInfo, nseg) % 8 == 0 && offsetof(LevelInfo, ntiles) == offsetof(LevelInfo, nseg) + 4 &&
              offsetof(LevelInfo, fin_total) % 8 == 0 && offsetof(LevelInfo, nfin2) == offsetof(LevelInfo, fin_total) + 4,
              "packed LevelInfo pairs");

// Look-back status of one tile (one side) of the partition kernels: two
// 8-byte words for the aggregate and two for the inclusive prefix, each
// {tag = epoch << 2 | state, 32-bit count} (see partition.cu).
struct __align__(16) Status {
    unsigned long long agg[2];
    unsigned long long inc[2];
};

struct RootArgs {
    const double* xs;
    const double* ys;
    uint64_t n;
    const RootInfo* root;
    double* ox;
    double* oy;
    uint32_t* oid;
    uint64_t out_cap;    // debug bounds
    Status* status;      // stable mode: 2 per tile (side S1, side S2)
    unsigned long long* side_ctr;  // fast mode: packed class counters per side
    uint32_t epoch;
    uint32_t* ctr;       // tile claim counter
    uint32_t* ticket;    // CTA exit ticket
    Best* cta_part;      // 4 per CTA (8 in octagon mode)
    ChildRec* children;  // 4 slots (8 in octagon mode)
    uint32_t ntiles;
    RootInfo* root_w;    // filtered root: side counts and apexes for the stats
};

// Split root, pass 1 (root_filter_tma): the octagon filter over the caller's
// arrays; survivors (x, y, index) are compacted to o*, the exact extremes of
// the survivors (= find_extremes of the input) give p and q, and the last CTA
// writes the first level's single slot (p, q, p) — the reference's bootstrap
// triangle (hull.cpp:228-235).
struct FilterArgs {
    const double* xs;
    const double* ys;
    uint64_t n;
    uint32_t ntiles;
    double* ox;
    double* oy;
    uint32_t* oid;
    uint64_t out_cap;    // debug bounds
    uint32_t* ctr;       // survivor counter
    uint32_t* ticket;    // CTA exit ticket
    void* part;          // per-CTA partials
    RootInfo* root_w;
    ChildRec* slot;      // the first level's slot table (1 slot)
    double* kx;          // sharded hull: a second copy of the survivors (nullptr: none)
    double* ky;
    uint32_t* kid;
    uint32_t xoff, yoff; // xs / ys sit this many elements (0 or 1) above a 16-byte boundary
};

struct LevelArgs {
    const double* gx;    // the hull's input arrays (index -> coordinates, arg-max ties)
    const double* gy;
    const SegRec* segs;
    const uint32_t* tile_seg;
    const LevelInfo* info;
    const double* ix;
    const double* iy;
    const uint32_t* iid;
    double* ox;
    double* oy;
    uint32_t* oid;
    uint64_t in_cap, out_cap;  // debug bounds
    uint64_t status_cap, part_cap, children_cap, segs_cap;
    Status* status;      // 1 per tile
    uint32_t epoch;
    uint32_t* ctr;
    Best* tile_part;     // 2 per tile (per-CTA segment partials, indexed tile0 + slot)
    uint32_t* seg_pcnt;  // per segment: partials published
    uint32_t* seg_done;  // per segment: tiles finished
    unsigned long long* seg_ctr;  // fast mode: packed L/R counters per segment
    ChildRec* children;  // 2 per segment
    // the next level's plan, written by the level kernel as each segment
    // finishes (planner-free host levels; n_kind == nullptr: the host runs the
    // planner kernel instead): kinds, links, SegRec / FinRec tables, the tile
    // -> segment map, zeroed per-segment counters, and LevelInfo counters
    // (atomics); nn_info (the level after) is zeroed for the next launch
    uint8_t* n_kind;
    uint32_t* n_link;
    SegRec* n_segs;
    FinRec* n_fins;
    uint32_t n_fin_cap;
    LevelInfo* n_info;
    LevelInfo* nn_info;
    uint32_t* n_tile_seg;
    uint32_t* n_seg_pcnt;
    uint32_t* n_seg_done;
    unsigned long long* n_seg_ctr;
};

// Persistent recursion kernel (tail.cu): per level, the host-allocated tables
// it fills (the same tables the host-driven level loop uses).
struct TailLevel {
    ChildRec* slots;
    SegRec* segs;
    FinRec* fins;
    uint8_t* kind;
    uint32_t* link;
    uint32_t* fin_count;
};
constexpr int kTailLevels = 40;
constexpr uint32_t kTailSlots = 4096;  // slot capacity of the persistent kernel's level tables
struct TailArgs {
    TailLevel lv[kTailLevels];
    LevelInfo* info;          // LevelInfo array indexed by level
    const LevelInfo* prev0;   // info of level l0 - 1 (nullptr: level l0 has nslots0 slots)
    int l0, nlev;
    uint32_t nslots0;
    uint32_t max_slots;       // table capacity; a level with more slots is left to the host
    uint32_t max_tiles;       // a level with more tiles is left to the host's TMA-ring kernel
    uint32_t fin_max;         // segments up to this size go to the finishers (<= kTailFinMax)
    int in0;                  // buffer read by level l0
    double* bx[2];
    double* by[2];
    uint32_t* bid[2];
    uint64_t buf_cap;
    const double* gx;
    const double* gy;
    uint32_t* flags;          // planner look-back
    void* aggs_v;
    void* incs_v;
    uint32_t epoch0;
    uint32_t* plan_ctr;
    uint32_t* seg_pcnt;
    uint32_t* seg_done;
    unsigned long long* seg_ctr;
    uint32_t* tile_seg;
    Best* tile_part;
    uint64_t part_cap;
    uint32_t* chain;
    uint32_t* state;          // [0] level, [1] 1 = finished at that level, 2 = stopped before it
    unsigned long long* trace;  // optional (VQHULL_TAIL_TRACE): CTA 0's %globaltimer per level phase
    uint32_t* out;            // in-kernel emission: index list (nullptr: the host emits)
    uint32_t* h_out;          // its length
    const uint32_t* p_idx;    // &RootInfo::p_idx (the frame vertex)
    const RootInfo* root;
    uint32_t* report;         // [8 words: state, h, nonfinite, unsafe, filter, survivors, 0] + level infos
    uint32_t* kc_done;        // set to 1 by the cluster recursion (KC) when it did the whole call
};

// Sharded hull certificate (shard.cu): polygon of at most kCertMax vertices
// of the local hull, the three chord forms per vertex, the wedge table.
constexpr uint32_t kCertMax = 16384;
constexpr uint32_t kCertBuckets = 16384;
struct CertHead {
    uint32_t K;        // vertices (0: no certificate)
    uint32_t j0;       // vertex of the smallest angle around c
    uint32_t valid;
    uint32_t pad;
    double cx, cy;     // centre, verified inside conv(Q)
    double M;          // max |coordinate| of the vertices and c
    double Me;         // margin scale max(M, floor): margin 2^-32 Me
};
struct CertRec {
    double ra, rb, rg;  // chord c -> v_j        (drop side: fma(a, x, b*y) < g)
    double ba, bb, bg;  // chord v_j -> c
    double ea, eb, eg;  // chord v_j -> v_{j+1}
};

// One-CTA hull of a tiny input (kernels.cu, tiny_hull_kernel).
struct TinyArgs {
    const double* xs;
    const double* ys;
    uint32_t n;
    uint32_t* iid;        // scratch: positions 0..n-1 (the segment's carried indices)
    FinRec* fin;          // one FinRec
    LevelInfo* info;      // its counts (warp or CTA list)
    uint32_t* chain;
    uint32_t* fin_count;
    uint32_t* out;        // index list (device)
    uint32_t* report;     // [0] h, [1] non-finite
};

// Emission of a small recursion tree in one kernel: per level, the slot
// tables (levels 2 .. 2 + nlev - 1).
constexpr int kEmitMaxLevels = 48;
struct EmitLevel {
    const uint8_t* kind;
    const uint32_t* link;
    const ChildRec* slots;
    const FinRec* fins;
    const uint32_t* fin_count;
    uint32_t* size;
    uint32_t* start;
    uint32_t nslots;
    uint32_t pad;
};
struct EmitAll {
    EmitLevel lv[kEmitMaxLevels];
    int nlev;
    // the level below the last one listed, emitted by its own launches
    // (nullptr: the listed levels are the whole tree)
    const uint32_t* below_size;
    uint32_t* below_start;
};

// Look-back payload of the planner scan.
struct PlanAgg {
    uint32_t nseg, nfin, nfin2, ntiles, out, fin, leaf;
};

__device__ __forceinline__ void pl_clear(PlanAgg& a) {
    a.nseg = a.nfin = a.nfin2 = a.ntiles = a.out = a.fin = a.leaf = 0;
}
__device__ __forceinline__ void pl_combine(PlanAgg& a, const PlanAgg& b) {
    a.nseg += b.nseg;
    a.nfin += b.nfin;
    a.nfin2 += b.nfin2;
    a.ntiles += b.ntiles;
    a.out += b.out;
    a.fin += b.fin;
    a.leaf += b.leaf;
}
__device__ __forceinline__ void pl_store(PlanAgg* d, const PlanAgg& a) { *d = a; }
__device__ __forceinline__ PlanAgg pl_load(const PlanAgg* s) {
    PlanAgg a;
    a.nseg = __ldcg(&s->nseg);
    a.nfin = __ldcg(&s->nfin);
    a.nfin2 = __ldcg(&s->nfin2);
    a.ntiles = __ldcg(&s->ntiles);
    a.out = __ldcg(&s->out);
    a.fin = __ldcg(&s->fin);
    a.leaf = __ldcg(&s->leaf);
    return a;
}
__device__ __forceinline__ PlanAgg pl_shfl(const PlanAgg& a, int x) {
    PlanAgg o;
    o.nseg = __shfl_xor_sync(kFull, a.nseg, x);
    o.nfin = __shfl_xor_sync(kFull, a.nfin, x);
    o.nfin2 = __shfl_xor_sync(kFull, a.nfin2, x);
    o.ntiles = __shfl_xor_sync(kFull, a.ntiles, x);
    o.out = __shfl_xor_sync(kFull, a.out, x);
    o.fin = __shfl_xor_sync(kFull, a.fin, x);
    o.leaf = __shfl_xor_sync(kFull, a.leaf, x);
    return o;
}

}  // namespace vqb
