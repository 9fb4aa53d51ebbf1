// Shared device-side building blocks of the B200 VQhull hot path.
//
// Numerics: every predicate and offset below is the reference's exact f64
// expression (kernels.hpp:19-45), evaluated with explicit round-to-nearest
// intrinsics (__dsub_rn / __dmul_rn) so no FMA contraction can occur even if
// the translation unit were compiled with --fmad=true.  Products that the
// reference forms as a*b are formed here either as a*b or b*a; IEEE
// multiplication is exactly commutative, so the rounded values are identical.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace vqb {

constexpr unsigned kFull = 0xffffffffu;

// set by a kernel that detected an impossible state (bounded spin expired,
// runaway loop); the driver checks it after every hull and reports an error
static __device__ uint32_t g_vqb_fault = 0;
// debug builds (-DVQB_DEBUG) record the first failed bounds check here
static __device__ unsigned long long g_vqb_dbg[4];
#ifdef VQB_DEBUG
#define VQB_CHECK(cond, code, a0, a1)                                        \
    do {                                                                     \
        if (!(cond)) {                                                       \
            if (atomicCAS(&g_vqb_fault, 0u, (unsigned)(code)) == 0u) {       \
                g_vqb_dbg[0] = (unsigned long long)(a0);                     \
                g_vqb_dbg[1] = (unsigned long long)(a1);                     \
                g_vqb_dbg[2] = blockIdx.x;                                   \
                g_vqb_dbg[3] = threadIdx.x;                                  \
            }                                                                \
        }                                                                    \
    } while (0)
#else
#define VQB_CHECK(cond, code, a0, a1) \
    do {                              \
    } while (0)
#endif  // per-TU; only kernels.cu launches kernels

// ---------------------------------------------------------------------------
// Canonical farthest order (kernels.hpp:36-45): the strictly smaller lateral
// offset wins, an exact tie falls to the lexicographically smaller point.
// We extend the order by the input index so that, among copies of the same
// coordinates, the FIRST occurrence is the one carried forward: this is the
// index vqhull_compute would map the vertex to (vqhull_c.cpp:51-61).
// ---------------------------------------------------------------------------
struct __align__(16) Best {
    double off;
    double x;
    double y;
    uint32_t idx;    // global input index (first-occurrence tie-break)
    uint32_t valid;  // 0 = side empty
};

__host__ __device__ __forceinline__ Best best_none() {
    Best b;
    b.off = 0.0;
    b.x = 0.0;
    b.y = 0.0;
    b.idx = 0xffffffffu;
    b.valid = 0u;
    return b;
}

// true when a is strictly preferred over b
__device__ __forceinline__ bool prefer(const Best& a, const Best& b) {
    if (!a.valid) return false;
    if (!b.valid) return true;
    if (a.off != b.off) return a.off < b.off;
    if (a.x != b.x) return a.x < b.x;
    if (a.y != b.y) return a.y < b.y;
    return a.idx < b.idx;
}

__device__ __forceinline__ void consider(Best& b, bool take, double off, double x,
                                         double y, uint32_t idx) {
    Best c;
    c.off = off;
    c.x = x;
    c.y = y;
    c.idx = idx;
    c.valid = take ? 1u : 0u;
    if (prefer(c, b)) b = c;
}

__device__ __forceinline__ Best shfl_best(const Best& b, int src_lane_xor) {
    Best o;
    o.off = __shfl_xor_sync(kFull, b.off, src_lane_xor);
    o.x = __shfl_xor_sync(kFull, b.x, src_lane_xor);
    o.y = __shfl_xor_sync(kFull, b.y, src_lane_xor);
    o.idx = __shfl_xor_sync(kFull, b.idx, src_lane_xor);
    o.valid = __shfl_xor_sync(kFull, b.valid, src_lane_xor);
    return o;
}

// butterfly: every lane ends with the warp's best
__device__ __forceinline__ Best warp_best(Best b) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        Best o = shfl_best(b, s);
        if (prefer(o, b)) b = o;
    }
    return b;
}

// ---------------------------------------------------------------------------
// Orientation predicate of the reference, frame_left_of (kernels.hpp:28-30):
//   (e.px - ux) * (e.qy - uy) > (e.py - uy) * (e.qx - ux)
// expressed on the precomputed differences of the query point to p and q.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// left of (P -> Q) given (Px-ux, Py-uy) and (Qx-ux, Qy-uy)
__device__ __forceinline__ bool left_diff(double pdx, double pdy, double qdx, double qdy) {
    return dmul(pdx, qdy) > dmul(pdy, qdx);
}

// Programmatic dependent launch: a kernel waits for its stream predecessor
// to complete (and its writes to be visible) before touching memory, then at
// once lets its own successor be launched, so launch latency and CTA
// placement of the next kernel overlap this one (no-ops without the launch
// attribute).  Must be the first statement of every kernel launched with
// pdl_launch.
#define VQB_PDL() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")

// Inf or NaN (exponent all ones), by the bits
__device__ __forceinline__ bool nonfinite_bits(double v) {
    return (__double2hiint(v) & 0x7ff00000) == 0x7ff00000;
}

// lateral offset e.dy*ux - e.dx*uy (kernels.hpp:32-34)
__device__ __forceinline__ double lat_off(double edx, double edy, double ux, double uy) {
    return dsub(dmul(edy, ux), dmul(edx, uy));
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------------------
// Register-light running arg-max.  A candidate is (key, idx): key is an
// order-preserving u64 image of its lateral offset (after +0.0, so -0 and +0
// map to the same key: they compare equal as doubles), idx its input index.
// Smaller key = strictly smaller offset = preferred (kernels.hpp:41-45).  Only
// an exact offset tie needs the coordinates: they are fetched from the input
// arrays through idx, and the reference's lexicographic (x, y) rule plus the
// first-occurrence index rule decide.  Equivalent to prefer() on Best.
// ---------------------------------------------------------------------------
// find_extremes key (geometry.cpp:7-36): lo = lexicographic min of (x, y,
// index); hi = max x, then max y, then min index.
struct ExtKey {
    double x, y;
    uint32_t idx;
    uint32_t valid;
};

__device__ __forceinline__ bool lo_better(const ExtKey& a, const ExtKey& b) {
    if (!a.valid) return false;
    if (!b.valid) return true;
    if (a.x != b.x) return a.x < b.x;
    if (a.y != b.y) return a.y < b.y;
    return a.idx < b.idx;
}
__device__ __forceinline__ bool hi_better(const ExtKey& a, const ExtKey& b) {
    if (!a.valid) return false;
    if (!b.valid) return true;
    if (a.x != b.x) return a.x > b.x;
    if (a.y != b.y) return a.y > b.y;
    return a.idx < b.idx;
}
__device__ __forceinline__ ExtKey shfl_key(const ExtKey& k, int x) {
    ExtKey o;
    o.x = __shfl_xor_sync(kFull, k.x, x);
    o.y = __shfl_xor_sync(kFull, k.y, x);
    o.idx = __shfl_xor_sync(kFull, k.idx, x);
    o.valid = __shfl_xor_sync(kFull, k.valid, x);
    return o;
}

constexpr unsigned long long kNoKey = ~0ull;
constexpr uint32_t kNoIdx = 0xffffffffu;

__device__ __forceinline__ unsigned long long key_of(double off) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(off + 0.0));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// candidate (k, i) strictly preferred over incumbent (kb, ib)?
__device__ __forceinline__ bool key_better(unsigned long long k, uint32_t i, unsigned long long kb,
                                           uint32_t ib, const double* __restrict__ xs,
                                           const double* __restrict__ ys) {
    if (k != kb) return k < kb;
    if (i == ib || i == kNoIdx) return false;
    if (ib == kNoIdx) return true;
    const double x = xs[i], y = ys[i], xb = xs[ib], yb = ys[ib];
    if (x != xb) return x < xb;
    if (y != yb) return y < yb;
    return i < ib;
}

__device__ __forceinline__ void key_consider(unsigned long long& kb, uint32_t& ib,
                                             unsigned long long k, uint32_t i,
                                             const double* __restrict__ xs,
                                             const double* __restrict__ ys) {
    if (k < kb || (k == kb && key_better(k, i, kb, ib, xs, ys))) {
        kb = k;
        ib = i;
    }
}

// butterfly: every lane ends with the warp's preferred candidate
__device__ __forceinline__ void warp_key_best(unsigned long long& k, uint32_t& i,
                                              const double* __restrict__ xs,
                                              const double* __restrict__ ys) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const unsigned long long ok = __shfl_xor_sync(kFull, k, s);
        const uint32_t oi = __shfl_xor_sync(kFull, i, s);
        if (ok < k || (ok == k && key_better(ok, oi, k, i, xs, ys))) {
            k = ok;
            i = oi;
        }
    }
}

// Materialise a (key, idx) candidate as a Best: coordinates from the input,
// offset recomputed with the same frame (identical rounding).
__device__ __forceinline__ Best best_from_key(unsigned long long k, uint32_t i, double edx,
                                              double edy, const double* __restrict__ xs,
                                              const double* __restrict__ ys) {
    Best b = best_none();
    if (i != kNoIdx && k != kNoKey) {
        b.x = xs[i];
        b.y = ys[i];
        b.off = lat_off(edx, edy, b.x, b.y);
        b.idx = i;
        b.valid = 1u;
    }
    return b;
}

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk) global -> shared, completed on an mbarrier.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// generic-proxy accesses of shared memory ordered before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// streaming variant: the lines are marked evict-first in L2, so a pass over
// gigabytes does not flush what the next kernels reuse (their tables, the
// survivors, instructions)
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_1d_stream(void* dst, const void* src, uint32_t bytes,
                                                   unsigned long long* bar, unsigned long long policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
    uint32_t done;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}

// ---------------------------------------------------------------------------
// Memory-ordering primitives for the decoupled look-back.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ double ld_cg_f64(const double* p) { return __ldcg(p); }

// streaming loads of data read exactly once
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) { return __ldcs(p); }

// ---------------------------------------------------------------------------
// Look-back payload: per class the element count and the best candidate.
// Combination is associative and commutative (sum; canonical arg-max).
// ---------------------------------------------------------------------------
template <int NC>
struct __align__(16) Agg {
    uint32_t cnt[NC];
    Best best[NC];
};

template <int NC>
__device__ __forceinline__ void agg_clear(Agg<NC>& a) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        a.cnt[c] = 0;
        a.best[c] = best_none();
    }
}

template <int NC>
__device__ __forceinline__ void agg_combine(Agg<NC>& a, const Agg<NC>& b) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        a.cnt[c] += b.cnt[c];
        if (prefer(b.best[c], a.best[c])) a.best[c] = b.best[c];
    }
}

template <int NC>
__device__ __forceinline__ void agg_store(Agg<NC>* dst, const Agg<NC>& a) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        dst->cnt[c] = a.cnt[c];
        dst->best[c] = a.best[c];
    }
}

template <int NC>
__device__ __forceinline__ Agg<NC> agg_load_cg(const Agg<NC>* src) {
    Agg<NC> a;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        a.cnt[c] = __ldcg(&src->cnt[c]);
        a.best[c].off = __ldcg(&src->best[c].off);
        a.best[c].x = __ldcg(&src->best[c].x);
        a.best[c].y = __ldcg(&src->best[c].y);
        a.best[c].idx = __ldcg(&src->best[c].idx);
        a.best[c].valid = __ldcg(&src->best[c].valid);
    }
    return a;
}

template <int NC>
__device__ __forceinline__ Agg<NC> shfl_agg(const Agg<NC>& a, int lane_xor) {
    Agg<NC> o;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        o.cnt[c] = __shfl_xor_sync(kFull, a.cnt[c], lane_xor);
        o.best[c] = shfl_best(a.best[c], lane_xor);
    }
    return o;
}

// Tile status words: (epoch << 2) | state.  A fresh epoch per launch makes
// stale words from earlier launches read as "not yet published".
constexpr uint32_t kStAgg = 1u;
constexpr uint32_t kStInc = 2u;

__device__ __forceinline__ uint32_t status_word(uint32_t epoch, uint32_t st) {
    return (epoch << 2) | st;
}

// Payload concept for the look-back: clear / combine / store / load_cg / shfl.
template <int NC>
__device__ __forceinline__ void pl_clear(Agg<NC>& a) { agg_clear(a); }
template <int NC>
__device__ __forceinline__ void pl_combine(Agg<NC>& a, const Agg<NC>& b) { agg_combine(a, b); }
template <int NC>
__device__ __forceinline__ void pl_store(Agg<NC>* d, const Agg<NC>& a) { agg_store(d, a); }
template <int NC>
__device__ __forceinline__ Agg<NC> pl_load(const Agg<NC>* s) { return agg_load_cg(s); }
template <int NC>
__device__ __forceinline__ Agg<NC> pl_shfl(const Agg<NC>& a, int x) { return shfl_agg(a, x); }

// Decoupled look-back, run by ONE full warp of the tile that owns `tile`.
// `first` is the global id of the segment's first tile (tiles of a segment are
// consecutive ids and are claimed in increasing order, so every predecessor is
// owned by a running CTA that publishes without waiting).  Publishes the
// tile's aggregate, walks back, publishes the inclusive value, and returns the
// exclusive prefix to every lane.
template <class T>
__device__ T lookback(uint32_t tile, uint32_t first, const T& local, uint32_t* flags,
                      T* aggs, T* incs, uint32_t epoch) {
    const int lane = threadIdx.x & 31;
    T excl;
    pl_clear(excl);
    if (tile == first) {
        if (lane == 0) {
            pl_store(&incs[tile], local);
            __threadfence();
            st_release(&flags[tile], status_word(epoch, kStInc));
        }
        __syncwarp();
        return excl;
    }
    if (lane == 0) {
        pl_store(&aggs[tile], local);
        __threadfence();
        st_release(&flags[tile], status_word(epoch, kStAgg));
    }
    __syncwarp();
    int64_t pred = int64_t(tile) - 1;  // highest predecessor not yet folded in
    while (true) {
        const int64_t t = pred - lane;
        const bool in_seg = t >= int64_t(first);
        uint32_t st = 0;
        if (in_seg) {
            const uint32_t want_hi = epoch << 2;
            uint32_t w;
            uint32_t spins = 0;
            while (true) {
                w = ld_acquire(&flags[t]);
                if ((w & ~3u) == want_hi && (w & 3u) != 0) break;
                if (++spins > 4) __nanosleep(64);
                if (spins > (1u << 25)) {  // ~seconds: a bug, never wait forever
                    w = kStInc;
                    g_vqb_fault = 1u;
                    break;
                }
            }
            st = w & 3u;
        }
        const unsigned inc_mask = __ballot_sync(kFull, in_seg && st == kStInc);
        // lanes up to (and including) the nearest inclusive tile contribute
        const int stop = inc_mask ? (__ffs(inc_mask) - 1) : 31;
        T mine;
        pl_clear(mine);
        if (in_seg && lane <= stop) mine = (st == kStInc) ? pl_load(&incs[t]) : pl_load(&aggs[t]);
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            T o = pl_shfl(mine, s);
            pl_combine(mine, o);
        }
        pl_combine(excl, mine);
        const unsigned seg_mask = __ballot_sync(kFull, in_seg);
        if (inc_mask) break;
        if (seg_mask != kFull) break;  // window reached the first tile (defensive)
        pred -= 32;
    }
    if (lane == 0) {
        T inc = excl;
        pl_combine(inc, local);
        pl_store(&incs[tile], inc);
        __threadfence();
        st_release(&flags[tile], status_word(epoch, kStInc));
    }
    __syncwarp();
    return excl;
}

// Register-light look-back for the partition payloads: the exclusive prefix
// accumulates in shared memory (*excl) and the window is reduced one class at
// a time, so at most one Best is live per lane.  Same protocol as lookback<>.
template <int NC>
__device__ void lookback_agg(uint32_t tile, uint32_t first, const Agg<NC>& local, Agg<NC>& excl,
                             uint32_t* flags, Agg<NC>* aggs, Agg<NC>* incs, uint32_t epoch) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) agg_clear(excl);
    if (tile == first) {
        if (lane == 0) {
            agg_store(&incs[tile], local);
            __threadfence();
            st_release(&flags[tile], status_word(epoch, kStInc));
        }
        __syncwarp();
        return;
    }
    if (lane == 0) {
        agg_store(&aggs[tile], local);
        __threadfence();
        st_release(&flags[tile], status_word(epoch, kStAgg));
    }
    __syncwarp();
    int64_t pred = int64_t(tile) - 1;
    while (true) {
        const int64_t t = pred - lane;
        const bool in_seg = t >= int64_t(first);
        uint32_t st = 0;
        if (in_seg) {
            const uint32_t want_hi = epoch << 2;
            uint32_t w;
            uint32_t spins = 0;
            while (true) {
                w = ld_acquire(&flags[t]);
                if ((w & ~3u) == want_hi && (w & 3u) != 0) break;
                if (++spins > 4) __nanosleep(64);
                if (spins > (1u << 25)) {
                    w = kStInc;
                    g_vqb_fault = 1u;
                    break;
                }
            }
            st = w & 3u;
        }
        const unsigned inc_mask = __ballot_sync(kFull, in_seg && st == kStInc);
        const int stop = inc_mask ? (__ffs(inc_mask) - 1) : 31;
        const bool take = in_seg && lane <= stop;
        const Agg<NC>* src = (st == kStInc) ? &incs[in_seg ? t : 0] : &aggs[in_seg ? t : 0];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            uint32_t v = take ? __ldcg(&src->cnt[c]) : 0u;
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(kFull, v, s);
            Best b = best_none();
            if (take) {
                b.off = __ldcg(&src->best[c].off);
                b.x = __ldcg(&src->best[c].x);
                b.y = __ldcg(&src->best[c].y);
                b.idx = __ldcg(&src->best[c].idx);
                b.valid = __ldcg(&src->best[c].valid);
            }
            b = warp_best(b);
            if (lane == 0) {
                excl.cnt[c] += v;
                if (prefer(b, excl.best[c])) excl.best[c] = b;
            }
        }
        const unsigned seg_mask = __ballot_sync(kFull, in_seg);
        if (inc_mask) break;
        if (seg_mask != kFull) break;
        pred -= 32;
    }
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            incs[tile].cnt[c] = excl.cnt[c] + local.cnt[c];
            incs[tile].best[c] = prefer(local.best[c], excl.best[c]) ? local.best[c] : excl.best[c];
        }
        __threadfence();
        st_release(&flags[tile], status_word(epoch, kStInc));
    }
    __syncwarp();
}

}  // namespace vqb

#if defined(__CUDACC__)
#include <cstdlib>
namespace vqb {
inline bool pdl_enabled() {
    static const bool on = getenv("VQB_NO_PDL") == nullptr;
    return on;
}
// <<<grid, block, smem, st>>> with programmatic stream serialization
template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
}  // namespace vqb
#endif
