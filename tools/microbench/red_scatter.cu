// Microbenchmark: scatter-accumulate into a frame-interleaved variable array (the
// single-pass "posterior accumulate" BP variant of DESIGN.md 7c).  Each warp walks
// edge slots e, variable v = perm[e]; lane l adds a float4 (4 frames) to acc[v][l].
//   mode 0: red.global.add.v4.f32          (one vector reduction per lane)
//   mode 1: 2 x red.global.add.u64         (biased fixed point, 2 frames per u64; deterministic)
//   mode 2: 4 x red.global.add.u32         (fixed point, 1 frame per op; deterministic)
//   mode 3: plain ld + st float4 (racy; the non-atomic bound)
//   mode 4: ld float4 only (gather bound)
// V variables x 32 lanes x 16 B; V = 65536 -> 33.5 MB (L2-resident), V = 1M -> 537 MB (HBM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 red_scatter.cu -o red_scatter
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(const int *__restrict__ perm, int E, float4 *acc, float4 *sink) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int e = warp; e < E; e += nw) {
        const int v = __ldg(perm + e);
        float4 *p = acc + (size_t)v * 32 + lane;
        const float a = 0.25f * (float)(e & 7);
        if (MODE == 0) {
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(a), "f"(a), "f"(a)
                         : "memory");
        } else if (MODE == 1) {
            unsigned long long *q = reinterpret_cast<unsigned long long *>(p);
            const unsigned long long w = (unsigned long long)(e & 1023) | ((unsigned long long)(e & 511) << 32);
            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(q), "l"(w) : "memory");
            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(q + 1), "l"(w) : "memory");
        } else if (MODE == 2) {
            unsigned *q = reinterpret_cast<unsigned *>(p);
            const unsigned w = (unsigned)(e & 1023);
#pragma unroll
            for (int c = 0; c < 4; ++c) asm volatile("red.global.add.u32 [%0], %1;" ::"l"(q + c), "r"(w) : "memory");
        } else if (MODE == 3) {
            float4 x = *p;
            x.x += a; x.y += a; x.z += a; x.w += a;
            *p = x;
        } else {
            const float4 x = *p;
            s.x += x.x; s.y += x.y; s.z += x.z; s.w += x.w;
        }
    }
    if (MODE == 4 && s.x == 12345.f) sink[0] = s;
}

int main(int argc, char **argv) {
    const int V = argc > 1 ? atoi(argv[1]) : 65536;
    const int E = (int)(3.37 * V);
    std::vector<int> h(E);
    std::mt19937 rng(1);
    for (int e = 0; e < E; ++e) h[e] = (int)(rng() % V);
    int *perm;
    float4 *acc, *sink;
    cudaMalloc(&perm, E * 4);
    cudaMalloc(&acc, (size_t)V * 32 * 16);
    cudaMalloc(&sink, 16);
    cudaMemcpy(perm, h.data(), E * 4, cudaMemcpyHostToDevice);
    cudaMemset(acc, 0, (size_t)V * 32 * 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char *names[] = {"red.v4.f32", "2x red.u64", "4x red.u32", "ld+st f4", "ld f4"};
    for (int mode = 0; mode < 5; ++mode) {
        for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
            auto run = [&]() {
                switch (mode) {
                    case 0: k<0><<<blocks, 256>>>(perm, E, acc, sink); break;
                    case 1: k<1><<<blocks, 256>>>(perm, E, acc, sink); break;
                    case 2: k<2><<<blocks, 256>>>(perm, E, acc, sink); break;
                    case 3: k<3><<<blocks, 256>>>(perm, E, acc, sink); break;
                    default: k<4><<<blocks, 256>>>(perm, E, acc, sink); break;
                }
            };
            for (int w = 0; w < 3; ++w) run();
            cudaEventRecord(a);
            const int R = 10;
            for (int r = 0; r < R; ++r) run();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double us = 1e3 * ms / R;
            const double bytes = (double)E * 32 * 16;  // payload bytes per launch (16 B per lane-edge)
            printf("V=%d E=%d %-12s blocks=%5d  %8.1f us  %7.0f GB/s payload\n", V, E, names[mode], blocks, us,
                   bytes / us * 1e-3);
        }
    }
    cudaError_t err = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(err));
    return 0;
}
