// Golden vectors for the text point format: std::to_chars(double) shortest
// form, as the reference's append_double (proj/src/io.cpp:26-30) writes it.
// Build + run: g++ -std=c++17 -O1 tests/golden/make_to_chars.cpp -o /tmp/mtc && /tmp/mtc > tests/golden/to_chars.txt
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <cmath>

static void emit(double v) {
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v);
    *r.ptr = 0;
    std::uint64_t bits;
    std::memcpy(&bits, &v, 8);
    std::printf("%016llx %s\n", (unsigned long long)bits, buf);
}

int main() {
    const double fixed[] = {0.0, -0.0, 1.0, -1.0, 100.0, 1e5, 1e15, 1e16, 1e17, 1e21, 1e22, 123456.0,
                            1234567.0, 0.1, 0.5, 0.001, 0.0001, 1e-5, 1e-7, 1.5e-7, 3.14159, 2.5e10,
                            1e100, 1e-100, 5e-324, 1.7976931348623157e308, 2.2250738585072014e-308,
                            123e18, 1e23, 9007199254740993.0, 0.30000000000000004, 12300.0, 1.23e-4};
    for (double v : fixed) emit(v);
    std::mt19937_64 g(7);
    for (int i = 0; i < 3000; ++i) {
        std::uint64_t b = g();
        double v;
        std::memcpy(&v, &b, 8);
        if (v != v || v - v != 0) continue;  // skip NaN / inf
        emit(v);
    }
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    for (int i = 0; i < 2000; ++i) {
        double v = u(g) * std::pow(10.0, double(int(g() % 40) - 20));
        emit(v);
    }
    for (int e = -25; e <= 25; ++e) { emit(std::pow(10.0, e)); emit(3 * std::pow(10.0, e)); }
    return 0;
}
