// Microbenchmark: random 4-byte DSMEM loads/stores across a thread-block cluster
// (sizing the cluster-resident decoder of DESIGN.md "next step").
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 dsmem_random.cu -o dsmem_random
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int WORDS = 24 * 1024;  // 96 KB per CTA

template <int MODE>  // 0 = local random stores, 1 = remote random stores, 2 = remote random loads
__global__ void k(int iters, unsigned long long *cycles, float *sink) {
    extern __shared__ float buf[];
    cg::cluster_group cl = cg::this_cluster();
    const int nb = cl.num_blocks();
    for (int i = threadIdx.x; i < WORDS; i += blockDim.x) buf[i] = (float)i;
    cl.sync();
    unsigned x = 2654435761u * (threadIdx.x + 1) + 97u * blockIdx.x;
    float acc = 0.f;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
        for (int u = 0; u < 8; ++u) {
            x = x * 1664525u + 1013904223u;
            const int dst = MODE == 0 ? cl.block_rank() : (int)((x >> 24) % nb);
            const int off = (int)((x >> 2) % WORDS);
            float *p = cl.map_shared_rank(buf, dst) + off;
            if (MODE == 2) acc += *p;
            else *p = (float)it;
        }
    }
    cl.sync();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
    if (acc == 12345.f) *sink = acc;
}

template <int MODE>
void run(int csize, const char *name) {
    int iters = 200, threads = 512, sms = 148;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, WORDS * 4);
    if (csize > 8) cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    int blocks = (sms / csize) * csize;
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = WORDS * 4;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    unsigned long long *cyc;
    float *sink;
    cudaMalloc(&cyc, 8);
    cudaMalloc(&sink, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, k<MODE>, iters, cyc, sink);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, k<MODE>, iters, cyc, sink);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)blocks * threads * iters * 8 * 4;
    printf("%-22s cluster %2d: %s  %.3f ms  %.1f GB/s total (%.1f per SM), %.2f B/clk/SM at 1.9 GHz\n", name, csize,
           cudaGetErrorString(e), ms, bytes / ms / 1e6, bytes / ms / 1e6 / blocks,
           bytes / (ms * 1e-3) / blocks / 1.9e9);
}

int main() {
    for (int c : {8, 16}) {
        run<0>(c, "local random st");
        run<1>(c, "remote random st");
        run<2>(c, "remote random ld");
    }
    return 0;
}
