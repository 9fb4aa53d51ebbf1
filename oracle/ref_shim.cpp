// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Thin extern "C" shim over the UNMODIFIED reference library (VQhull,
// /root/reference/proj/src, compiled in place by oracle/Makefile into
// oracle/_ref/libvqhull_ref.so).  It exists so that tests/, the golden-vector
// generator and bench.py's reference / cpu_baseline legs can drive the real
// reference through ctypes.  Every function forwards to the reference's own
// public C++ API; nothing here re-implements reference behaviour.
//
//   ref_convex_hull      -> vqhull::convex_hull          (hull.hpp:58)
//   ref_bench_hull       -> run_bench_points semantics   (bench.cpp:99-148)
//   ref_find_extremes    -> vqhull::find_extremes        (geometry.hpp:135-138)
//   ref_extract_subsets  -> vqhull::extract_subsets      (extract.hpp:79-82)
//   ref_generate         -> vqhull::generate             (dataset.hpp:50)
//   ref_generate_square  -> rng::uniform01 (dataset.hpp:30) for BASELINE
//                           config 2's harness-defined square, x = 2U(2i)-1,
//                           y = 2U(2i+1)-1 (the reference has no square kind)
//   ref_scale_baseline   -> stream_scale_baseline        (bench.hpp:32, bench.cpp:33-74)
//   ref_trace_hull       -> HullTrace + bytes_model      (hull.hpp:26-36, bench.cpp:16-21)
//   ref_monotone_chain   -> monotone_chain_hull          (bench.hpp:87)
//   vqhull_compute       is exported by the reference itself (vqhull_c.h:23)
#include <algorithm>
#include <chrono>
#include <cstring>
#include <cstdint>
#include <thread>
#include <vector>

#include "vqhull/bench.hpp"
#include "vqhull/config.hpp"
#include "vqhull/dataset.hpp"
#include "vqhull/extract.hpp"
#include "vqhull/geometry.hpp"
#include "vqhull/hull.hpp"

using namespace vqhull;

namespace {
PointSet load(const double* xs, const double* ys, size_t n) {
    PointSet p(n);
    if (n) {
        std::memcpy(p.xs(), xs, n * sizeof(double));
        std::memcpy(p.ys(), ys, n * sizeof(double));
    }
    return p;
}
}  // namespace

extern "C" {

int ref_avx512_available() { return avx512_available() ? 1 : 0; }

unsigned ref_hw_threads() { return std::thread::hardware_concurrency(); }

// Hull coordinates in the reference's output order.  Returns 0 / 1 on error.
int ref_convex_hull(const double* xs, const double* ys, size_t n, int workers,
                    int lanes, int simd_portable, int max_depth,
                    double* out_x, double* out_y, size_t out_cap, size_t* out_count) {
    try {
        PointSet pts = load(xs, ys, n);
        Config cfg;
        cfg.workers = workers;
        cfg.lanes = lanes;
        cfg.simd = simd_portable ? SimdMode::Portable : SimdMode::Auto;
        cfg.max_depth = max_depth;
        const HullPolygon h = convex_hull(pts, cfg);
        *out_count = h.size();
        if (h.size() > out_cap) return 2;
        for (size_t i = 0; i < h.size(); ++i) {
            out_x[i] = h.vertices[i].x;
            out_y[i] = h.vertices[i].y;
        }
        *out_count = h.size();
        return 0;
    } catch (...) {
        return 1;
    }
}

// run_bench_points semantics: every repetition hulls a fresh copy; the clock
// covers convex_hull only (extremes through assembly), never the copy.
int ref_bench_hull(const double* xs, const double* ys, size_t n, int workers,
                   int reps, double* seconds, size_t* hull_size) {
    try {
        const PointSet base = load(xs, ys, n);
        Config cfg;
        cfg.workers = workers;
        for (int r = 0; r < reps; ++r) {
            PointSet scratch = base;
            const auto t0 = std::chrono::steady_clock::now();
            const HullPolygon h = convex_hull(scratch, cfg);
            const auto t1 = std::chrono::steady_clock::now();
            seconds[r] = std::chrono::duration<double>(t1 - t0).count();
            *hull_size = h.size();
        }
        return 0;
    } catch (...) {
        return 1;
    }
}

int ref_find_extremes(const double* xs, const double* ys, size_t n,
                      size_t* lo, size_t* hi) {
    try {
        const auto e = find_extremes(xs, ys, n);
        *lo = e.first;
        *hi = e.second;
        return 0;
    } catch (...) {
        return 1;
    }
}

// In-place extraction on caller arrays.  edge = {px, py, qx, qy}.
int ref_extract_subsets(double* xs, double* ys, size_t n, const double* ea,
                        const double* eb, int lanes, int simd_portable,
                        size_t* w_l, size_t* w_r, double* r1, int* has_r1,
                        double* r2, int* has_r2) {
    try {
        Config cfg;
        cfg.lanes = lanes;
        cfg.simd = simd_portable ? SimdMode::Portable : SimdMode::Auto;
        const DirectedEdge a{{ea[0], ea[1]}, {ea[2], ea[3]}};
        const DirectedEdge b{{eb[0], eb[1]}, {eb[2], eb[3]}};
        const ExtractOutcome o = extract_subsets(xs, ys, n, a, b, cfg);
        *w_l = o.w_l;
        *w_r = o.w_r;
        *has_r1 = o.r1.has_value();
        *has_r2 = o.r2.has_value();
        if (o.r1) { r1[0] = o.r1->x; r1[1] = o.r1->y; }
        if (o.r2) { r2[0] = o.r2->x; r2[1] = o.r2->y; }
        return 0;
    } catch (...) {
        return 1;
    }
}

// kind: 0 kuzmin, 1 circle, 2 disk (DatasetKind order, dataset.hpp:12)
int ref_generate(int kind, uint64_t n, uint64_t seed, int workers, double* xs,
                 double* ys) {
    try {
        DatasetSpec spec;
        spec.kind = static_cast<DatasetKind>(kind);
        spec.n = n;
        spec.seed = seed;
        const PointSet p = generate(spec, workers);
        std::memcpy(xs, p.xs(), n * sizeof(double));
        std::memcpy(ys, p.ys(), n * sizeof(double));
        return 0;
    } catch (...) {
        return 1;
    }
}

// points [first, first + n) of the square stream; the fill is split over
// `workers` threads like generate() (the bytes do not depend on the split)
int ref_generate_square(uint64_t seed, uint64_t first, uint64_t n, int workers, double* xs,
                        double* ys) {
    try {
        if (workers < 1) workers = 1;
        auto fill = [&](uint64_t b, uint64_t e) {
            for (uint64_t i = b; i < e; ++i) {
                const uint64_t k = first + i;
                xs[i] = 2.0 * rng::uniform01(seed, 2 * k) - 1.0;
                ys[i] = 2.0 * rng::uniform01(seed, 2 * k + 1) - 1.0;
            }
        };
        std::vector<std::thread> th;
        const uint64_t chunk = (n + uint64_t(workers) - 1) / uint64_t(workers);
        for (int t = 1; t < workers; ++t) {
            const uint64_t b = chunk * uint64_t(t);
            if (b >= n) break;
            th.emplace_back(fill, b, std::min(n, b + chunk));
        }
        fill(0, std::min(n, chunk));
        for (auto& t : th) t.join();
        return 0;
    } catch (...) {
        return 1;
    }
}

// the reference's STREAM-Scale ceiling (best-of-reps GB/s, 16 B per element)
double ref_scale_baseline(uint64_t buffer_bytes, int reps, int workers) {
    try {
        return stream_scale_baseline(buffer_bytes ? buffer_bytes : default_scale_bytes(), reps, workers).gbps;
    } catch (...) {
        return -1.0;
    }
}

uint64_t ref_rng_at(uint64_t seed, uint64_t index) { return rng::at(seed, index); }
double ref_uniform01(uint64_t seed, uint64_t index) { return rng::uniform01(seed, index); }

// Traced single-worker hull: byte model, number of partition calls, hull size
// and (optionally) the per-call records {points, s1, s2, chain2_moved}.
int ref_trace_hull(const double* xs, const double* ys, size_t n,
                   uint64_t* model_bytes, size_t* n_calls, size_t* hull_size,
                   uint64_t* calls_out, size_t calls_cap) {
    try {
        PointSet pts = load(xs, ys, n);
        HullTrace trace;
        Config cfg;
        cfg.trace = &trace;
        const HullPolygon h = convex_hull(pts, cfg);
        *model_bytes = bytes_model(trace);
        *n_calls = trace.calls.size();
        *hull_size = h.size();
        if (calls_out) {
            for (size_t i = 0; i < trace.calls.size() && i < calls_cap; ++i) {
                calls_out[4 * i + 0] = trace.calls[i].points;
                calls_out[4 * i + 1] = trace.calls[i].s1;
                calls_out[4 * i + 2] = trace.calls[i].s2;
                calls_out[4 * i + 3] = trace.calls[i].chain2_moved;
            }
        }
        return 0;
    } catch (...) {
        return 1;
    }
}

int ref_monotone_chain(const double* xs, const double* ys, size_t n,
                       double* out_x, double* out_y, size_t* out_count) {
    try {
        const PointSet pts = load(xs, ys, n);
        const std::vector<Point> h = monotone_chain_hull(pts);
        for (size_t i = 0; i < h.size(); ++i) {
            out_x[i] = h[i].x;
            out_y[i] = h[i].y;
        }
        *out_count = h.size();
        return 0;
    } catch (...) {
        return 1;
    }
}

}  // extern "C"
