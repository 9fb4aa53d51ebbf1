// Seeded synthetic point sets (host tooling; not on the hot path).
//
// The reference's counter-based generators (dataset.cpp:32-75): point i of
// stream `seed` draws u(2i) and u(2i+1) with
//   u(k) = (splitmix64_mix(seed + (k+1) * 0x9e3779b97f4a7c15) >> 11) * 2^-53.
// The radial/angle transforms use the host libm (cos/sin are not bitwise
// reproducible on the GPU), so inputs are generated here and copied to HBM.
// Compiled with -ffp-contract=off so e.g. inv*inv - 1.0 is not fused.
// kind 3 ("square") is the harness-defined BASELINE config 2:
//   x = 2u(2i) - 1, y = 2u(2i+1) - 1   (exact in f64).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;
constexpr double kTwoPi = 6.283185307179586476925286766559;  // 2*pi rounded to f64

inline uint64_t mix(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ull;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebull;
    z ^= z >> 31;
    return z;
}

inline double u01(uint64_t seed, uint64_t k) {
    return double(mix(seed + (k + 1) * kGamma) >> 11) * 0x1.0p-53;
}

void point(int kind, uint64_t seed, uint64_t i, double& x, double& y) {
    switch (kind) {
        case 0: {  // kuzmin
            const double u = u01(seed, 2 * i);
            const double inv = 1.0 / (1.0 - u);
            const double r = std::sqrt(inv * inv - 1.0);
            const double t = kTwoPi * u01(seed, 2 * i + 1);
            x = r * std::cos(t);
            y = r * std::sin(t);
            break;
        }
        case 1: {  // circle
            const double t = kTwoPi * u01(seed, 2 * i);
            x = std::cos(t);
            y = std::sin(t);
            break;
        }
        case 2: {  // disk
            const double r = std::sqrt(u01(seed, 2 * i));
            const double t = kTwoPi * u01(seed, 2 * i + 1);
            x = r * std::cos(t);
            y = r * std::sin(t);
            break;
        }
        default: {  // square [-1, 1]^2
            x = 2.0 * u01(seed, 2 * i) - 1.0;
            y = 2.0 * u01(seed, 2 * i + 1) - 1.0;
            break;
        }
    }
}

}  // namespace

extern "C" int vqhull_generate(int kind, uint64_t seed, uint64_t first, uint64_t n, double* xs,
                               double* ys, int threads) {
    if (kind < 0 || kind > 3) return 1;
    if (n == 0) return 0;
    if (!xs || !ys) return 1;
    auto run = [=](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i) point(kind, seed, first + i, xs[i], ys[i]);
    };
    if (threads <= 1 || n < (1u << 16)) {
        run(0, n);
        return 0;
    }
    const uint64_t chunk = (n + threads - 1) / uint64_t(threads);
    std::vector<std::thread> th;
    for (int t = 1; t < threads; ++t) {
        const uint64_t b = chunk * uint64_t(t);
        if (b >= n) break;
        th.emplace_back(run, b, std::min(n, b + chunk));
    }
    run(0, std::min(n, chunk));
    for (auto& t : th) t.join();
    return 0;
}
