// Sharded hull: the per-shard candidate certificate and the
// merge-side gather, exact by construction.
//
// Each shard computes its local hull L (the ordinary pipeline).  The hull of
// the union of local hulls is NOT the reference's answer in general: the
// reference's f64 predicates are not robust, so a global recursion can keep a
// near-collinear point that a shard's recursion discarded (circle 1e7:
// 9,994,016 vs 9,994,044 vertices).  Instead a shard sends every
// point it cannot PROVE irrelevant to the global recursion:
//
//   F_r = { P in shard r : P is not provably inside conv(L_r) by the margin }
//
// where "provably inside by the margin" is the polygon-filter test of the
// split root, applied to one wedge triangle (c, v_i, v_{i+1})
// of L_r (c a point verified inside conv(L_r)): P right of the three chords
// c -> v_i, v_i -> v_{i+1}, v_{i+1} -> c by 2^-32 M |chord|_1 (M bounds the
// vertices), evaluated with fused multiply-adds whose rounding (<= ~6 eps |e| M)
// is far below the margin.  Then the mu-ball around P lies in the triangle,
// hence in conv(L_r), hence in the hull of the points left in play, and the
// drop argument of the filter applies unchanged: such a point can never be a
// farthest point nor the lone member of a subset of the global recursion.
// The merge hulls F = union of the F_r (ordered by global index, so duplicates
// resolve to their first occurrence) with the ordinary pipeline: the result
// is the reference's global recursion over all points.  The rounding bound
// behind the margin needs every coordinate in play within 2^12 M; each shard
// reports its M and the largest |coordinate| it holds, the merge checks the
// condition across shards and, if a shard's scale is too small, asks for its
// candidates again with a margin floor (VQHULL_ERETRY).
//
// Which points a shard tests: the split root's filter pass already dropped
// the points inside its 16-gon by the same argument (they are deep inside
// conv(F) too: the 16-gon's vertices are in F or certified inside conv(L_r)),
// so with the filter on the certificate runs over the filter pass's survivors
// only (kept by that pass, FilterArgs::kx); otherwise over the whole shard.
//
// Wedge lookup: the vertex angles around c are decreasing along the clockwise
// hull; a 16384-bucket table of the ascending sequence gives each point's
// wedge in O(1) (f32 atan2).  The lookup only chooses which triangle to test:
// a wrong choice can only keep a point, never drop one.
#include <cub/cub.cuh>

#include <cstdint>
#include <cstdio>

#include "common.cuh"
#include "hull_types.cuh"
#include "kernels.h"

namespace vqb {

namespace {

constexpr float kPiF = 3.14159265358979323846f;

// chord u -> w as the filter's linear form (poly_finish_warp): f(P) =
// cross(w - u, P - u) = fa x + fb y + fc; the drop-side test is
// fma(fa, x, fb * y) < fg with fg = -mu |w - u|_1 - fc.  Degenerate chords
// never pass (fg = -inf).
__device__ __forceinline__ void chord_form(double ux, double uy, double wx, double wy, double mu,
                                           double& fa, double& fb, double& fg) {
    const double ex = wx - ux, ey = wy - uy;
    if (ex == 0.0 && ey == 0.0) {
        fa = 0.0;
        fb = 0.0;
        fg = -__longlong_as_double(0x7ff0000000000000ll);
        return;
    }
    fa = -ey;
    fb = ex;
    const double fc = ey * ux - ex * uy;
    const double ft = -mu * (fabs(ex) + fabs(ey));
    fg = ft - fc;
}

__device__ __forceinline__ bool chord_in(double fa, double fb, double fg, double x, double y) {
    return __fma_rn(fa, x, __dmul_rn(fb, y)) < fg;
}

__device__ __forceinline__ float wedge_angle(double x, double y, double cx, double cy) {
    return atan2f(__double2float_rn(y - cy), __double2float_rn(x - cx));
}

// order-preserving image of a non-negative double for atomicMax
__device__ __forceinline__ unsigned long long mag_key(double a) {
    return static_cast<unsigned long long>(__double_as_longlong(a));
}

}  // namespace

// ---------------------------------------------------------------------------
// cert_build_kernel: one CTA.  Polygon Q = K vertices of the local hull
// (every vertex when h <= kCertMax, else an even subsample: still input
// points in clockwise order), centre c = their mean, M, the chord forms, the
// angle table.  valid = 0 disables the certificate (every tested point stays).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) cert_build_kernel(const uint32_t* __restrict__ hull, uint32_t h,
                                                          const double* __restrict__ xs,
                                                          const double* __restrict__ ys, double floor_m,
                                                          CertHead* head, CertRec* rec, float* asc,
                                                          uint32_t* tab) {
    __shared__ double s_red[32][3];
    __shared__ float s_fmin[32];
    __shared__ uint32_t s_imin[32];
    __shared__ uint32_t s_bad;
    const uint32_t K = h < kCertMax ? h : kCertMax;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto vert = [&](uint32_t j) -> uint32_t {
        return K == h ? hull[j] : hull[uint32_t((uint64_t(j) * h) / K)];
    };
    if (tid == 0) s_bad = 0u;
    // sums and max |coordinate|
    double sx = 0.0, sy = 0.0, m = 0.0;
    for (uint32_t j = tid; j < K; j += blockDim.x) {
        const uint32_t v = vert(j);
        const double x = xs[v], y = ys[v];
        sx += x;
        sy += y;
        m = fmax(m, fmax(fabs(x), fabs(y)));
        if (!(fabs(x) <= 0x1p1000) || !(fabs(y) <= 0x1p1000)) atomicOr(&s_bad, 1u);
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        sx += __shfl_xor_sync(kFull, sx, s);
        sy += __shfl_xor_sync(kFull, sy, s);
        m = fmax(m, __shfl_xor_sync(kFull, m, s));
    }
    if (lane == 0) {
        s_red[warp][0] = sx;
        s_red[warp][1] = sy;
        s_red[warp][2] = m;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0.0, b = 0.0, c = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
            a += s_red[w][0];
            b += s_red[w][1];
            c = fmax(c, s_red[w][2]);
        }
        s_red[0][0] = K ? a / double(K) : 0.0;
        s_red[0][1] = K ? b / double(K) : 0.0;
        s_red[0][2] = c;
    }
    __syncthreads();
    const double cx = s_red[0][0], cy = s_red[0][1];
    const double M = fmax(s_red[0][2], fmax(fabs(cx), fabs(cy)));
    const double Me = fmax(M, floor_m);  // margin scale (a floor from the merge's scale check)
    const double mu = 0x1p-32 * Me;
    bool ok = K >= 3 && s_bad == 0u && M >= 0x1p-400 && M <= 0x1p500 && Me <= 0x1p500;
    // chord forms and angles; c must lie strictly right of every edge chord
    // (then c is inside conv(Q): right of every chord of a closed polygon)
    float fmin_v = 3.0e38f;
    uint32_t imin = 0;
    for (uint32_t j = tid; j < K && ok; j += blockDim.x) {
        const uint32_t v = vert(j), w = vert(j + 1 == K ? 0 : j + 1);
        const double vx = xs[v], vy = ys[v], wx = xs[w], wy = ys[w];
        CertRec r;
        chord_form(cx, cy, vx, vy, mu, r.ra, r.rb, r.rg);  // c -> v_j
        chord_form(vx, vy, cx, cy, mu, r.ba, r.bb, r.bg);  // v_j -> c
        chord_form(vx, vy, wx, wy, mu, r.ea, r.eb, r.eg);  // v_j -> v_{j+1}
        rec[j] = r;
        if (!chord_in(r.ea, r.eb, r.eg, cx, cy)) atomicOr(&s_bad, 2u);
        const float a = wedge_angle(vx, vy, cx, cy);
        asc[K + j] = a;  // angle by vertex (scratch: second half of asc)
        if (a < fmin_v) {
            fmin_v = a;
            imin = j;
        }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const float o = __shfl_xor_sync(kFull, fmin_v, s);
        const uint32_t oi = __shfl_xor_sync(kFull, imin, s);
        if (o < fmin_v || (o == fmin_v && oi < imin)) {
            fmin_v = o;
            imin = oi;
        }
    }
    if (lane == 0) {
        s_fmin[warp] = fmin_v;
        s_imin[warp] = imin;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w)
            if (s_fmin[w] < s_fmin[0] || (s_fmin[w] == s_fmin[0] && s_imin[w] < s_imin[0])) {
                s_fmin[0] = s_fmin[w];
                s_imin[0] = s_imin[w];
            }
    }
    __syncthreads();
    ok = ok && s_bad == 0u;
    const uint32_t j0 = s_imin[0];
    // ascending sequence: asc[t] = angle of vertex (j0 - t) mod K
    if (ok)
        for (uint32_t t = tid; t < K; t += blockDim.x) {
            const uint32_t j = (j0 + K - (t % K)) % K;
            asc[t] = asc[K + j];
        }
    __syncthreads();
    // bucket b starts at angle -pi + b * 2pi / B: tab[b] = #{t : asc[t] < start}
    // (binary search; asc is ascending up to rounding ties, which only cost
    // a few extra steps of the per-point walk)
    if (ok)
        for (uint32_t b = tid; b < kCertBuckets; b += blockDim.x) {
            const float start = -kPiF + (2.0f * kPiF) * (float(b) / float(kCertBuckets));
            uint32_t lo = 0, hi = K;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (asc[mid] < start) lo = mid + 1;
                else hi = mid;
            }
            tab[b] = lo;
        }
    if (tid == 0) {
        CertHead H;
        H.K = ok ? K : 0u;
        H.j0 = j0;
        H.valid = ok ? 1u : 0u;
        H.pad = 0u;
        H.cx = cx;
        H.cy = cy;
        H.M = M;
        H.Me = Me;
        *head = H;
    }
}

// ---------------------------------------------------------------------------
// certify_kernel: every tested point either passes its wedge triangle's three
// chord tests (dropped) or is appended to the residual (x, y, local index).
// Also the largest |coordinate| of every tested point (the merge's scale
// check).  Warp-aggregated appends, one atomic per warp and round.
// ---------------------------------------------------------------------------
template <bool kIdx>
__global__ void __launch_bounds__(256) certify_kernel(const double* __restrict__ xs, const double* __restrict__ ys,
                                                      const uint32_t* __restrict__ ids, uint64_t n_host,
                                                      const uint32_t* __restrict__ n_dev,
                                                      const CertHead* __restrict__ head,
                                                      const CertRec* __restrict__ rec,
                                                      const float* __restrict__ asc,
                                                      const uint32_t* __restrict__ tab, double* __restrict__ rx,
                                                      double* __restrict__ ry, uint32_t* __restrict__ rid,
                                                      uint32_t* __restrict__ rcount,
                                                      unsigned long long* __restrict__ amax_bits) {
    const uint64_t n = n_dev ? uint64_t(*n_dev) : n_host;
    const CertHead H = *head;
    const bool valid = H.valid != 0u;
    const uint32_t K = H.K;
    const unsigned lt = lanemask_lt();
    const int lane = threadIdx.x & 31;
    double amax = 0.0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    // warp-uniform loop bound: every lane takes part in the ballots
    const uint64_t base0 = uint64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u);
    for (uint64_t base = base0; base < n; base += stride) {
        const uint64_t i = base + lane;
        const bool live = i < n;
        double x = 0.0, y = 0.0;
        uint32_t id = 0;
        if (live) {
            x = xs[i];
            y = ys[i];
            id = kIdx ? ids[i] : uint32_t(i);
            amax = fmax(amax, fmax(fabs(x), fabs(y)));
        }
        bool drop = false;
        if (live && valid && fabs(x) <= H.M && fabs(y) <= H.M) {
            const float phi = wedge_angle(x, y, H.cx, H.cy);
            int b = int((phi + kPiF) * (float(kCertBuckets) / (2.0f * kPiF)));
            b = b < 0 ? 0 : (b >= int(kCertBuckets) ? int(kCertBuckets) - 1 : b);
            uint32_t t = tab[b];
            for (int s = 0; s < 64 && t < K && asc[t] <= phi; ++s) ++t;
            // wedge between vertex i = (j0 - t) mod K (larger angle) and i + 1
            const uint32_t vi = (H.j0 + K - (t % K)) % K;
            const uint32_t vn = vi + 1 == K ? 0u : vi + 1;
            const CertRec& a = rec[vi];
            drop = chord_in(a.ra, a.rb, a.rg, x, y) && chord_in(a.ea, a.eb, a.eg, x, y) &&
                   chord_in(rec[vn].ba, rec[vn].bb, rec[vn].bg, x, y);
        }
        const bool keep = live && !drop;
        const unsigned bal = __ballot_sync(kFull, keep);
        if (bal) {
            uint32_t o = 0;
            if (lane == 0) o = atomicAdd(rcount, uint32_t(__popc(bal)));
            o = __shfl_sync(kFull, o, 0);
            if (keep) {
                const uint32_t p = o + uint32_t(__popc(bal & lt));
                rx[p] = x;
                ry[p] = y;
                rid[p] = id;
            }
        }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) amax = fmax(amax, __shfl_xor_sync(kFull, amax, s));
    if (lane == 0 && amax > 0.0) atomicMax(amax_bits, mag_key(amax));
}

// pack: header row {count, M_eff, A} + rows {x, y, bits(offset + id)} in the
// sorted order (perm), the first min(count, cap) of them
__global__ void pack_kernel(const double* __restrict__ rx, const double* __restrict__ ry,
                            const uint32_t* __restrict__ sorted_id, const uint32_t* __restrict__ perm,
                            uint32_t count, uint32_t cap, uint64_t offset, double* __restrict__ pack) {
    const uint32_t m = count < cap ? count : cap;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
        const uint32_t s = perm[t];
        double* row = pack + 3 * (uint64_t(t) + 1);
        row[0] = rx[s];
        row[1] = ry[s];
        row[2] = __longlong_as_double(static_cast<long long>(offset + sorted_id[t]));
    }
}

__global__ void iota32_kernel(uint32_t* d, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) d[i] = i;
}

// merge gather: rows of every rank's pack (headers already read by the host)
// into contiguous (x, y, gidx), and whether the global indices come strictly
// increasing (ranks in offset order)
__device__ __forceinline__ const double* merge_row(const double* packs, uint64_t stride_rows,
                                                   const uint64_t* starts, uint32_t nranks, uint64_t t) {
    uint32_t lo = 0, hi = nranks;  // rank r holds [starts[r], starts[r+1])
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (starts[mid] <= t) lo = mid;
        else hi = mid;
    }
    return packs + 3 * (uint64_t(lo) * stride_rows + 1 + (t - starts[lo]));
}

__global__ void merge_gather_kernel(const double* __restrict__ packs, uint64_t stride_rows,
                                    const uint64_t* __restrict__ starts, uint32_t nranks, uint64_t total,
                                    double* __restrict__ mx, double* __restrict__ my,
                                    uint64_t* __restrict__ mg, uint32_t* __restrict__ unsorted) {
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += uint64_t(gridDim.x) * blockDim.x) {
        const double* row = merge_row(packs, stride_rows, starts, nranks, t);
        const uint64_t g = static_cast<uint64_t>(__double_as_longlong(row[2]));
        mx[t] = row[0];
        my[t] = row[1];
        mg[t] = g;
        if (t > 0) {
            const double* prev = merge_row(packs, stride_rows, starts, nranks, t - 1);
            if (!(static_cast<uint64_t>(__double_as_longlong(prev[2])) < g)) *unsorted = 1u;
        }
    }
}

// final indices: positions in the merged (index-ordered) set -> global indices
__global__ void map_gidx_kernel(const uint32_t* __restrict__ pos, uint64_t h, const uint64_t* __restrict__ mg,
                                uint64_t* __restrict__ out) {
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < h; t += uint64_t(gridDim.x) * blockDim.x)
        out[t] = mg[pos[t]];
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
void launch_cert_build(const uint32_t* hull, uint32_t h, const double* xs, const double* ys, double floor_m,
                       CertHead* head, CertRec* rec, float* asc, uint32_t* tab, cudaStream_t st) {
    cert_build_kernel<<<1, 1024, 0, st>>>(hull, h, xs, ys, floor_m, head, rec, asc, tab);
}

void launch_certify(const double* xs, const double* ys, const uint32_t* ids, uint64_t n_host,
                    const uint32_t* n_dev, const CertHead* head, const CertRec* rec, const float* asc,
                    const uint32_t* tab, double* rx, double* ry, uint32_t* rid, uint32_t* rcount,
                    unsigned long long* amax_bits, int grid, cudaStream_t st) {
    if (ids)
        certify_kernel<true><<<grid, 256, 0, st>>>(xs, ys, ids, n_host, n_dev, head, rec, asc, tab, rx, ry, rid,
                                                    rcount, amax_bits);
    else
        certify_kernel<false><<<grid, 256, 0, st>>>(xs, ys, ids, n_host, n_dev, head, rec, asc, tab, rx, ry, rid,
                                                     rcount, amax_bits);
}

size_t sort_temp_bytes(uint32_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), int(n < 1 ? 1 : n));
    return bytes;
}

cudaError_t launch_sort_ids(void* temp, size_t temp_bytes, const uint32_t* keys_in, uint32_t* keys_out,
                            uint32_t* vals_in, uint32_t* vals_out, uint32_t n, int end_bit, cudaStream_t st) {
    iota32_kernel<<<(n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184, 256, 0, st>>>(vals_in, n);
    return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, int(n), 0,
                                           end_bit, st);
}

void launch_pack(const double* rx, const double* ry, const uint32_t* sorted_id, const uint32_t* perm,
                 uint32_t count, uint32_t cap, uint64_t offset, double* pack, cudaStream_t st) {
    const uint32_t m = count < cap ? count : cap;
    if (!m) return;
    pack_kernel<<<(m + 255) / 256 < 1184 ? (m + 255) / 256 : 1184, 256, 0, st>>>(rx, ry, sorted_id, perm, count,
                                                                                cap, offset, pack);
}

void launch_merge_gather(const double* packs, uint64_t stride_rows, const uint64_t* starts, uint32_t nranks,
                         uint64_t total, double* mx, double* my, uint64_t* mg, uint32_t* unsorted,
                         cudaStream_t st) {
    if (!total) return;
    const uint64_t g = (total + 255) / 256;
    merge_gather_kernel<<<g < 1184 ? unsigned(g) : 1184u, 256, 0, st>>>(packs, stride_rows, starts, nranks, total,
                                                                        mx, my, mg, unsorted);
}

void launch_map_gidx(const uint32_t* pos, uint64_t h, const uint64_t* mg, uint64_t* out, cudaStream_t st) {
    if (!h) return;
    const uint64_t g = (h + 255) / 256;
    map_gidx_kernel<<<g < 1184 ? unsigned(g) : 1184u, 256, 0, st>>>(pos, h, mg, out);
}

}  // namespace vqb
