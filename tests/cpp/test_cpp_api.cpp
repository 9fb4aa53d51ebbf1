// C++ parity tests of the B200 path through include/vqhull_b200.hpp.  They
// restate the reference's own C++ test cases (proj/tests/test_hull.cpp,
// test_extract.cpp, test_geometry.cpp) against the GPU implementation; built
// and run by tests/test_cpp_api.py (-m gpu).  Exit code 0 = all passed.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "vqhull_b200.hpp"

using namespace vqhull_b200;

static int failures = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                    \
        }                                                                  \
    } while (0)

#define STEP(name) std::fprintf(stderr, "[cpp] %s\n", name)

static PointSet pts(std::initializer_list<Point> l) {
    PointSet p;
    for (const Point& q : l) p.push_back(q);
    return p;
}

int main() {
    // test_hull.cpp:71-115 degenerate hulls
    STEP("degenerate hulls");
    CHECK(convex_hull(PointSet{}).empty());
    {
        const HullPolygon h = convex_hull(pts({{0, 0}}));
        CHECK(h.size() == 1 && h.vertices[0] == (Point{0, 0}));
    }
    {
        PointSet p;
        for (int i = 0; i < 100; ++i) p.push_back({3, -4});
        const HullPolygon h = convex_hull(p);
        CHECK(h.size() == 1 && h.vertices[0] == (Point{3, -4}) && h.indices[0] == 0);
    }
    {
        const HullPolygon h = convex_hull(pts({{5, 1}, {-2, 7}}));
        CHECK(h.size() == 2 && h.vertices[0] == (Point{-2, 7}) && h.vertices[1] == (Point{5, 1}));
    }
    {
        PointSet p;
        for (int i = 0; i < 10; ++i) p.push_back({double(i), double(i)});
        const HullPolygon h = convex_hull(p);
        CHECK(h.size() == 2 && h.vertices[0] == (Point{0, 0}) && h.vertices[1] == (Point{9, 9}));
    }
    {
        PointSet p;
        for (int i = 0; i < 7; ++i) p.push_back({2, double(i - 3)});
        const HullPolygon h = convex_hull(p);
        CHECK(h.size() == 2 && h.vertices[0] == (Point{2, -3}) && h.vertices[1] == (Point{2, 3}));
    }
    // test_hull.cpp:117-130 unit square with center
    STEP("unit square with center");
    {
        const HullPolygon h = convex_hull(pts({{1, 1}, {0, 0}, {0.5, 0.5}, {0, 1}, {1, 0}}));
        CHECK(h.size() == 4);
        CHECK(h.vertices[0] == (Point{0, 0}) && h.vertices[1] == (Point{0, 1}));
        CHECK(h.vertices[2] == (Point{1, 1}) && h.vertices[3] == (Point{1, 0}));
    }
    // test_hull.cpp:220-240 deep recursion on a convex power-of-two curve
    STEP("deep recursion on a convex power-of-two curve");
    {
        const int m = 600;
        PointSet p;
        for (int i = 0; i < m; ++i) p.push_back({std::ldexp(1.0, i), std::ldexp(1.0, -i)});
        for (bool stable : {false, true}) {
            Config cfg;
            cfg.stable = stable;
            const HullPolygon h = convex_hull(p, cfg);
            CHECK(h.size() == std::size_t(m));
            CHECK(h.vertices[0] == (Point{1, 1}) && h.vertices[1] == p[m - 1]);
            for (int i = 2; i < m; ++i) CHECK(h.vertices[std::size_t(i)] == p[std::size_t(m - i)]);
        }
    }
    // test_hull.cpp:320-345 C interface semantics (index 5 duplicates 0)
    STEP("C interface semantics (index 5 duplicates 0)");
    {
        const double xs[] = {0, 4, 4, 0, 2, 0};
        const double ys[] = {0, 0, 4, 4, 2, 0};
        std::size_t idx[6] = {99, 99, 99, 99, 99, 99};
        std::size_t count = 0;
        CHECK(vqhull_compute(xs, ys, 6, 1, idx, &count) == 0);
        CHECK(count == 4 && idx[0] == 0 && idx[1] == 3 && idx[2] == 2 && idx[3] == 1);
        std::size_t c = 7;
        CHECK(vqhull_compute(nullptr, nullptr, 0, 1, nullptr, &c) == 0 && c == 0);
        CHECK(vqhull_compute(nullptr, ys, 6, 1, idx, &c) == 1);
        CHECK(vqhull_compute(xs, ys, 6, 0, idx, &c) == 1);
        const double bad_x[] = {0, std::nan("")};
        const double bad_y[] = {0, 1};
        CHECK(vqhull_compute(bad_x, bad_y, 2, 1, idx, &c) == 1);
    }
    // test_geometry.cpp:32-51 find_extremes tie-breaks
    STEP("find_extremes tie-breaks");
    {
        CHECK(find_extremes(pts({{0, 0}})) == (std::pair<std::size_t, std::size_t>{0, 0}));
        CHECK(find_extremes(pts({{1, 5}, {-2, 0}, {3, 1}})) == (std::pair<std::size_t, std::size_t>{1, 2}));
        CHECK(find_extremes(pts({{0, 1}, {0, -1}, {0, 0}})) == (std::pair<std::size_t, std::size_t>{1, 0}));
        bool threw = false;
        try {
            find_extremes(PointSet{});
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    // test_extract.cpp:183-210 eight points around an edge
    STEP("eight points around an edge");
    for (bool stable : {false, true}) {
        PointSet p = pts({{1, 1}, {2, -1}, {3, 2}, {1, 0}, {0.5, -3}, {2, 4}, {3, 0}, {2.5, -0.5}});
        Config cfg;
        cfg.stable = stable;
        const ExtractOutcome o = extract_subsets(p.xs(), p.ys(), 8, {{0, 0}, {4, 0}}, {{4, 0}, {0, 0}}, cfg);
        CHECK(o.w_l == 3 && o.w_r == 5);
        CHECK(o.r1 && *o.r1 == (Point{2, 4}));
        CHECK(o.r2 && *o.r2 == (Point{0.5, -3}));
    }
    if (failures) {
        std::fprintf(stderr, "%d check(s) failed\n", failures);
        return 1;
    }
    std::printf("cpp api: all checks passed\n");
    return 0;
}
