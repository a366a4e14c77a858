// Register vectors of S frames per lane (S = 1, 2, 4) and their 4S-byte loads/stores.
#pragma once
#include <cuda_runtime.h>

namespace cvsr {

template <int S>
struct FV {
    float c[S];
};

template <int S>
__device__ __forceinline__ FV<S> ldv(const float *p) {
    FV<S> r;
    if constexpr (S == 4) {
        const float4 v = *reinterpret_cast<const float4 *>(p);
        r.c[0] = v.x; r.c[1] = v.y; r.c[2] = v.z; r.c[3] = v.w;
    } else if constexpr (S == 2) {
        const float2 v = *reinterpret_cast<const float2 *>(p);
        r.c[0] = v.x; r.c[1] = v.y;
    } else {
        r.c[0] = *p;
    }
    return r;
}

template <int S>
__device__ __forceinline__ void stv(float *p, const FV<S> &v) {
    if constexpr (S == 4) *reinterpret_cast<float4 *>(p) = make_float4(v.c[0], v.c[1], v.c[2], v.c[3]);
    else if constexpr (S == 2) *reinterpret_cast<float2 *>(p) = make_float2(v.c[0], v.c[1]);
    else *p = v.c[0];
}

template <int S>
__device__ __forceinline__ FV<S> splat(float x) {
    FV<S> r;
#pragma unroll
    for (int s = 0; s < S; ++s) r.c[s] = x;
    return r;
}

__device__ __forceinline__ uint32_t cmpu(const uint4 &v, int s) { return s == 0 ? v.x : s == 1 ? v.y : s == 2 ? v.z : v.w; }

}  // namespace cvsr
