// vqhull_b200.hpp — C++ host API of the B200 hot path, header-only, over the
// C ABI of vqhull_b200.h.
//
// Mirrors the reference's C++ surface for this path (VQhull,
// proj/include/vqhull): the same type and function names, argument meaning
// and error behaviour, so a caller of the reference can switch namespaces:
//
//   reference (proj/include/vqhull)           this header (namespace vqhull_b200)
//   Point, DirectedEdge      geometry.hpp:14-28   Point, DirectedEdge
//   PointSet                 geometry.hpp:90-125  PointSet (SoA, host)
//   find_extremes            geometry.hpp:135-138 find_extremes (throws on empty)
//   ExtractOutcome           extract.hpp:19-24    ExtractOutcome
//   extract_subsets          extract.hpp:79-82    extract_subsets (in place)
//   HullPolygon              hull.hpp:17-22       HullPolygon (+ input indices)
//   convex_hull              hull.hpp:58          convex_hull (input kept; the
//                                                 reference consumes it)
//   convex_hull_copy         hull.hpp:61          convex_hull_copy
//
// Every call runs on the GPU (cuda device 0 of the calling thread); there is
// no CPU fallback — a missing device surfaces as std::runtime_error.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "vqhull_b200.h"

namespace vqhull_b200 {

struct Point {
    double x = 0.0;
    double y = 0.0;
    friend bool operator==(const Point& a, const Point& b) { return a.x == b.x && a.y == b.y; }
};

struct DirectedEdge {
    Point p;
    Point q;
};

class PointSet {
   public:
    PointSet() = default;
    explicit PointSet(std::size_t n) : xs_(n, 0.0), ys_(n, 0.0) {}
    std::size_t size() const { return xs_.size(); }
    bool empty() const { return xs_.empty(); }
    void reserve(std::size_t n) { xs_.reserve(n); ys_.reserve(n); }
    void push_back(Point p) { xs_.push_back(p.x); ys_.push_back(p.y); }
    Point operator[](std::size_t i) const { return {xs_[i], ys_[i]}; }
    void set(std::size_t i, Point p) { xs_[i] = p.x; ys_[i] = p.y; }
    double* xs() { return xs_.data(); }
    double* ys() { return ys_.data(); }
    const double* xs() const { return xs_.data(); }
    const double* ys() const { return ys_.data(); }

   private:
    std::vector<double> xs_, ys_;
};

struct HullPolygon {
    std::vector<Point> vertices;       // clockwise from the leftmost(-lowest) point
    std::vector<std::size_t> indices;  // first-occurrence input index of each vertex
    std::size_t size() const { return vertices.size(); }
    bool empty() const { return vertices.empty(); }
};

struct ExtractOutcome {
    std::size_t w_l = 0;
    std::size_t w_r = 0;
    std::optional<Point> r1;
    std::optional<Point> r2;
};

// Accepted for source compatibility with the reference's Config
// (config.hpp:36-57); the GPU path has no worker/lane/block knobs.  `stable`
// selects order-preserving partition offsets (vqhull_cuda_set_stable).
struct Config {
    int workers = 1;
    bool stable = false;
    void validate() const {
        if (workers < 1) throw std::invalid_argument("workers must be >= 1");
    }
};

namespace detail {
inline void check(int rc, const char* what) {
    if (rc == VQHULL_OK) return;
    if (rc == VQHULL_EINVAL) throw std::invalid_argument(std::string(what) + ": invalid argument");
    if (rc == VQHULL_ESIZE) throw std::length_error(std::string(what) + ": too many points for one device");
    throw std::runtime_error(std::string(what) + ": " + vqhull_cuda_last_error());
}

struct DeviceArrays {  // RAII device copy of a PointSet
    double* x = nullptr;
    double* y = nullptr;
    std::size_t n = 0;
    explicit DeviceArrays(const double* hx, const double* hy, std::size_t count) : n(count) {
        if (!n) return;
        if (cudaMalloc(&x, n * sizeof(double)) != cudaSuccess ||
            cudaMalloc(&y, n * sizeof(double)) != cudaSuccess) {
            release();
            throw std::runtime_error("cudaMalloc failed");
        }
        cudaMemcpy(x, hx, n * sizeof(double), cudaMemcpyHostToDevice);
        cudaMemcpy(y, hy, n * sizeof(double), cudaMemcpyHostToDevice);
    }
    ~DeviceArrays() { release(); }
    DeviceArrays(const DeviceArrays&) = delete;
    DeviceArrays& operator=(const DeviceArrays&) = delete;
    void release() {
        if (x) cudaFree(x);
        if (y) cudaFree(y);
        x = y = nullptr;
    }
};
}  // namespace detail

// find_extremes (geometry.cpp:7-36): leftmost (ties: lowest y, first index),
// rightmost (ties: highest y, first index).  Throws on an empty set.
inline std::pair<std::size_t, std::size_t> find_extremes(const PointSet& points) {
    if (points.empty()) throw std::invalid_argument("find_extremes: empty input");
    detail::DeviceArrays d(points.xs(), points.ys(), points.size());
    uint64_t lo = 0, hi = 0;
    detail::check(vqhull_cuda_find_extremes(d.x, d.y, points.size(), &lo, &hi, nullptr),
                  "find_extremes");
    return {std::size_t(lo), std::size_t(hi)};
}

// extract_subsets (extract.hpp:75-82), in place on the host arrays.
inline ExtractOutcome extract_subsets(double* xs, double* ys, std::size_t n,
                                      const DirectedEdge& edge_a, const DirectedEdge& edge_b,
                                      const Config& cfg = {}) {
    cfg.validate();
    ExtractOutcome out;
    out.w_r = n;
    if (n == 0) return out;
    detail::DeviceArrays d(xs, ys, n);
    const double ea[4] = {edge_a.p.x, edge_a.p.y, edge_a.q.x, edge_a.q.y};
    const double eb[4] = {edge_b.p.x, edge_b.p.y, edge_b.q.x, edge_b.q.y};
    uint64_t wl = 0, wr = 0;
    double r1[2], r2[2];
    int h1 = 0, h2 = 0;
    detail::check(vqhull_cuda_set_stable(cfg.stable ? 1 : 0), "extract_subsets");
    detail::check(vqhull_cuda_extract_subsets(d.x, d.y, n, ea, eb, &wl, &wr, r1, &h1, r2, &h2, nullptr),
                  "extract_subsets");
    cudaMemcpy(xs, d.x, n * sizeof(double), cudaMemcpyDeviceToHost);
    cudaMemcpy(ys, d.y, n * sizeof(double), cudaMemcpyDeviceToHost);
    out.w_l = wl;
    out.w_r = wr;
    if (h1) out.r1 = Point{r1[0], r1[1]};
    if (h2) out.r2 = Point{r2[0], r2[1]};
    return out;
}

// convex_hull (hull.hpp:58): vertices clockwise from the leftmost(-lowest)
// point, collinear edge-interior points never emitted; plus their
// first-occurrence input indices (vqhull_c.cpp:51-61).
inline HullPolygon convex_hull(const PointSet& points, const Config& cfg = {}) {
    cfg.validate();
    HullPolygon h;
    const std::size_t n = points.size();
    if (n == 0) return h;
    detail::check(vqhull_cuda_set_stable(cfg.stable ? 1 : 0), "convex_hull");
    std::vector<std::size_t> idx(n);
    std::size_t cnt = 0;
    detail::check(vqhull_compute(points.xs(), points.ys(), n, cfg.workers, idx.data(), &cnt),
                  "convex_hull");
    idx.resize(cnt);
    h.vertices.reserve(cnt);
    for (std::size_t i : idx) h.vertices.push_back(points[i]);
    h.indices = std::move(idx);
    return h;
}

inline HullPolygon convex_hull_copy(const PointSet& points, const Config& cfg = {}) {
    return convex_hull(points, cfg);
}

}  // namespace vqhull_b200
