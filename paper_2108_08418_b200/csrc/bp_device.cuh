// Device helpers shared by the BP kernels (bp_kernels.cu, layer_kernels.cu): MUFU wrappers,
// the check-node update in registers (sum/difference form of the tanh rule, header of
// bp_kernels.cu) and the mbarrier / bulk-copy (TMA) primitives.
#pragma once
#include "common.cuh"
#include "vec.cuh"

namespace cvsr {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2f(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcpf(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// a (+) b = 1 - (1 - a)(1 - b)
__device__ __forceinline__ float cplus(float a, float b) { return fmaf(b, 1.0f - a, a); }
__device__ __forceinline__ uint32_t sgnbit(float x) { return __float_as_uint(x) >> 31; }
__device__ __forceinline__ float clampf(float x, float lim) { return fminf(fmaxf(x, -lim), lim); }

// this lane's active bit per sub-tile, and "any" over the lane's S frames
template <int S>
__device__ __forceinline__ uint32_t lane_act(const uint4 &m, int lane) {
    uint32_t a = 0u;
#pragma unroll
    for (int s = 0; s < S; ++s) a |= ((cmpu(m, s) >> lane) & 1u) << s;
    return a;
}

// ------------------------------------------------------------------ check nodes

// q (log2 units) -> r (log2 units), in registers.
// "Sum/difference" form of the tanh rule: with u = 2^-|q| every edge is the pair
// (1, u) ~ (D + N, D - N) of t = N / D = (1 - u) / (1 + u), and a product of t's
// is tracked as (S, Delta) = (prod D + prod N, prod D - prod N) up to a common
// factor:  (S1, d1) x (S2, d2) = (S1 S2 + d1 d2, S1 d2 + d1 S2).  Every term is
// non-negative (no cancellation), the leave-one-out pairs come from prefix and
// suffix products, and |r| = ln((1 + P) / (1 - P)) = lg2(S) - lg2(Delta) in log2
// units: 3 MUFU per edge (ex2, 2 lg2) and no reciprocal.  A zero message gives
// S = Delta, r = 0 exactly; an empty fold (degree-1 check) gives Delta = 0,
// |r| = +inf -> Q_MAX.
template <int DC>
__device__ __forceinline__ void cn_update(float (&q)[DC], uint32_t sbit, float qmax2) {
    if constexpr (DC == 2) {
        // two edges: the box-plus over the single other edge is that edge itself, so
        // r_e = (1 - 2 s) clamp(q_other) exactly -- no transcendental; a dummy other edge
        // (degree-1 check) gives the empty-fold value Q_MAX
        const float m0 = fminf(fabsf(q[1]), qmax2), m1 = fminf(fabsf(q[0]), qmax2);
        const uint32_t g0 = sbit ^ sgnbit(q[1]), g1 = sbit ^ sgnbit(q[0]);
        q[0] = g0 ? -m0 : m0;
        q[1] = g1 ? -m1 : m1;
        return;
    }
    float u[DC];
    uint32_t par = sbit;
#pragma unroll
    for (int i = 0; i < DC; ++i) {
        u[i] = ex2f(-fabsf(q[i]));
        par ^= sgnbit(q[i]);
    }
    float ps[DC], pd[DC];
    ps[0] = 1.0f;
    pd[0] = 0.0f;
#pragma unroll
    for (int i = 1; i < DC; ++i) {
        ps[i] = fmaf(u[i - 1], pd[i - 1], ps[i - 1]);
        pd[i] = fmaf(u[i - 1], ps[i - 1], pd[i - 1]);
    }
    float ss = 1.0f, sd = 0.0f;
#pragma unroll
    for (int i = DC - 1; i >= 0; --i) {
        const float S = fmaf(ps[i], ss, pd[i] * sd);
        const float D = fmaf(ps[i], sd, pd[i] * ss);
        const float mag = fmaxf(fminf(lg2f(S) - lg2f(D), qmax2), 0.0f);
        const float ns = fmaf(u[i], sd, ss);
        sd = fmaf(u[i], ss, sd);
        ss = ns;
        q[i] = (par ^ sgnbit(q[i])) ? -mag : mag;
    }
}

// One check for the S frames of this lane.  DC is the code's maximum check
// degree; a check of degree deg < DC is padded with "certain" dummy edges
// (|q| = 200 in log2 units: w = 0, the neutral element of (+), sign +), which
// are neither loaded nor stored: one code body per code keeps the i-cache hot.
constexpr float DUMMY_Q = 200.0f;

// the S frames of this lane (frames that are not active keep their message)
template <int DC, int S>
__device__ __forceinline__ void cn_lanes(FV<S> (&q)[DC], uint32_t sb, uint32_t al, float qmax2) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
        if (!((al >> s) & 1u)) continue;
        float a[DC];
#pragma unroll
        for (int k = 0; k < DC; ++k) a[k] = q[k].c[s];
        cn_update<DC>(a, (sb >> s) & 1u, qmax2);
#pragma unroll
        for (int k = 0; k < DC; ++k) q[k].c[s] = a[k];
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// per-thread asynchronous global -> shared copy of 4 or 8 bytes (cp.async.ca, LDGSTS)
template <int BYTES>
__device__ __forceinline__ void cp_async_g2s(void *dst, const void *src) {
    static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16, "cp.async size");
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES) : "memory");
}
// the mbarrier tracks this thread's prior cp.async copies: one pending arrival is added now and
// arrives when they have landed
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// make this thread's mbarrier.init visible (to the async proxy) before any use
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// order this thread's generic-proxy shared-memory accesses before later async-proxy (bulk copy)
// accesses of the same bytes
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// programmatic dependent launch: wait until the preceding grid of the stream has completed and
// its memory operations are visible (a no-op when the kernel was not launched as a dependent)
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// let the next (dependent) grid of the stream launch once every CTA of this grid has called it
__device__ __forceinline__ void griddep_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace cvsr
