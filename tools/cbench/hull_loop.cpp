// Host-overhead probe: back-to-back vqhull_cuda_hull_u32 calls from C++ (no
// Python), device-resident input.  Usage: hull_loop KIND N SEED [REPS]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#include "vqhull_b200.h"

int main(int argc, char** argv) {
    const int kind = argc > 1 ? atoi(argv[1]) : 3;
    const uint64_t n = argc > 2 ? uint64_t(atof(argv[2])) : 100000000ull;
    const uint64_t seed = argc > 3 ? uint64_t(atoll(argv[3])) : 2;
    const int reps = argc > 4 ? atoi(argv[4]) : 20;
    std::vector<double> xs(n), ys(n);
    vqhull_generate(kind, seed, 0, n, xs.data(), ys.data(), 16);
    double *dx, *dy;
    uint32_t* dout;
    cudaMalloc(&dx, n * 8);
    cudaMalloc(&dy, n * 8);
    cudaMalloc(&dout, n * 4);
    cudaMemcpy(dx, xs.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, ys.data(), n * 8, cudaMemcpyHostToDevice);
    uint64_t h = 0;
    for (int i = 0; i < 3; ++i) vqhull_cuda_hull_u32(dx, dy, n, dout, &h, nullptr);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, nullptr);
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) vqhull_cuda_hull_u32(dx, dy, n, dout, &h, nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    cudaEventRecord(b, nullptr);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("kind %d n %llu h %llu: %.4f ms/hull (events), %.4f ms/hull (host clock)\n", kind,
           (unsigned long long)n, (unsigned long long)h, ms / reps,
           std::chrono::duration<double, std::milli>(t1 - t0).count() / reps);
    return 0;
}
