// Alice-side LLR kernels.
//
// Conditional LLR of slice j (PAPER.md:114 step 4; reading A-2), log domain:
//   log P_b(x) from log Q(z) = ln(erfcx(z/sqrt2)/2) - z^2/2 (z >= 0),
//                              log1p(-erfc(-z/sqrt2)/2)      (z < 0),
//   bins entirely above (below) the mean use the upper (lower) tail,
//   straddling bins use (erf(hi/sqrt2) + erf(-lo/sqrt2))/2 (no cancellation);
//   ln N_beta = log-sum-exp over the admissible bins, which are enumerated
//   directly (labels agreeing with the known bits), so every lane runs the
//   same trip count 2^(m - |K|).
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"
#include "vec.cuh"

namespace cvsr {

constexpr float RSQRT2 = 0.70710678118654752f;

// Upper-tail pieces of the standard normal at |z|: Q(|z|) = t * exp(e),
// t = erfcx(|z|/sqrt2)/2, e = -z^2/2 (erfcx keeps t accurate in the far tail).
struct Tail {
    float t, e;
};
__device__ __forceinline__ Tail tail_of(float z) {
    const float a = fabsf(z);
    return Tail{0.5f * erfcxf(a * RSQRT2), -0.5f * a * a};
}

// log P(lo <= Z < hi), Z ~ N(0,1), lo < hi (either may be infinite).  The bin is
// mirrored to the upper half when it lies below 0; then
//   a >= 0 (whole bin in the upper tail): log Q(a) + log(1 - Q(b)/Q(a))
//   a < 0 < b (straddles the mean)      : log(1 - Q(|a|) - Q(b))
// Both forms use the same two erfcx evaluations; the selection is branch-free.
__device__ __forceinline__ float log_bin(float lo, float hi, bool lo_inf, bool hi_inf) {
    const bool mirror = !hi_inf && hi <= 0.0f;
    const float a = mirror ? -hi : lo, b = mirror ? -lo : hi;
    const bool a_inf = mirror ? false : lo_inf;   // a = -inf only if lo = -inf (not mirrored)
    const bool b_inf = mirror ? lo_inf : hi_inf;  // b = +inf
    const Tail ta = tail_of(a_inf ? 0.0f : a), tb = tail_of(b_inf ? 0.0f : b);
    const float lqa = __logf(ta.t) + ta.e;                      // log Q(|a|)
    const float lqb = b_inf ? -INFINITY : __logf(tb.t) + tb.e;  // log Q(b)
    // tail form (a >= 0): log Q(a) + log(-expm1(log Q(b) - log Q(a)))
    const float tail = b_inf ? lqa : lqa + __logf(-expm1f(lqb - lqa));
    // straddle form (a < 0 < b): 1 - Q(|a|) - Q(b); a = -inf gives Q(|a|) -> 0
    const float qa = a_inf ? 0.0f : ta.t * __expf(ta.e);
    const float qb = b_inf ? 0.0f : tb.t * __expf(tb.e);
    const float strad = log1pf(-(qa + qb));
    if (a_inf && b_inf) return 0.0f;
    return (!a_inf && a >= 0.0f) ? tail : strad;
}

__device__ __forceinline__ float log_add(float a, float b) {
    const float mx = fmaxf(a, b), mn = fminf(a, b);
    if (mx == -INFINITY) return -INFINITY;
    return mx + log1pf(__expf(mn - mx));
}

__device__ __forceinline__ uint32_t gray_inv(uint32_t g) {
    g ^= g >> 1;
    g ^= g >> 2;
    g ^= g >> 4;
    return g;
}

// unclamped ln N_0 - ln N_1 (+-1e30 when one side is empty)
__device__ float llr_raw(const float *se, int m, int j, uint32_t kmask, uint32_t kappa, float x, float inv_sigma) {
    const int nb = 1 << m;
    const uint32_t free_mask = (uint32_t)(nb - 1) & ~kmask;
    const uint32_t base = kappa & kmask;
    float ln0 = -INFINITY, ln1 = -INFINITY;
    uint32_t sub = 0u;
    do {
        const uint32_t g = base | sub;
        const int b = (int)gray_inv(g);
        const bool lo_inf = (b == 0), hi_inf = (b == nb - 1);
        const float lo = lo_inf ? 0.0f : (se[b - 1] - x) * inv_sigma;
        const float hi = hi_inf ? 0.0f : (se[b] - x) * inv_sigma;
        const float lp = log_bin(lo, hi, lo_inf, hi_inf);
        if ((g >> j) & 1u) ln1 = log_add(ln1, lp);
        else ln0 = log_add(ln0, lp);
        sub = (sub - free_mask) & free_mask;
    } while (sub);
    if (ln0 == -INFINITY) return -1e30f;
    if (ln1 == -INFINITY) return 1e30f;
    return ln0 - ln1;
}

__device__ __forceinline__ float llr_clamp(float L, float llr_max) { return fminf(fmaxf(L, -llr_max), llr_max); }

__device__ float llr_cond(const float *se, int m, int j, uint32_t kmask, uint32_t kappa, float x, float inv_sigma,
                          float llr_max) {
    return llr_clamp(llr_raw(se, m, j, kmask, kappa, x, inv_sigma), llr_max);
}

// index of the known-bit pattern kappa among the 2^|K| patterns (bits of K in order)
__device__ __forceinline__ int combo_of(uint32_t kmask, uint32_t kappa) {
    int c = 0, t = 0;
    for (uint32_t mk = kmask; mk; mk &= mk - 1, ++t) c |= (int)((kappa >> (__ffs(mk) - 1)) & 1u) << t;
    return c;
}
__device__ __forceinline__ uint32_t kappa_of(uint32_t kmask, int combo) {
    uint32_t k = 0u;
    int t = 0;
    for (uint32_t mk = kmask; mk; mk &= mk - 1, ++t) k |= (uint32_t)((combo >> t) & 1) << (__ffs(mk) - 1);
    return k;
}

__global__ void k_llr_table(LlrParams p, float *__restrict__ table, int combos) {
    __shared__ float se[256];
    for (int i = threadIdx.x; i < 255; i += blockDim.x) se[i] = p.edges[i];
    __syncthreads();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= combos * LLR_NTAB) return;
    const int combo = idx / LLR_NTAB, i = idx % LLR_NTAB;
    const float x = -LLR_XMAX + (float)(i - 1) * LLR_H;
    table[idx] = llr_raw(se, p.m, p.j, p.known_mask, kappa_of(p.known_mask, combo), x, p.inv_sigma);
}

// window table: table4[combo][i] = (table[i], table[i+1], table[i+2], table[i+3]) -- the 4 values
// one interpolation reads, as one aligned 16-byte load (the 4 scalar loads per symbol were the
// L1 wavefront bound of the LLR kernels: 82 % of the global-load wavefront peak)
__global__ void k_llr_window(const float *__restrict__ table, float4 *__restrict__ table4, int combos) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= combos * LLR_NWIN) return;
    const int combo = idx / LLR_NWIN, i = idx % LLR_NWIN;
    const float *f = table + (size_t)combo * LLR_NTAB + i;
    table4[idx] = make_float4(f[0], f[1], f[2], f[3]);
}

// L(x) from the table (cubic Lagrange through grid points i-1..i+2) or exactly
__device__ __forceinline__ float llr_eval(const LlrParams &p, const float *se, uint32_t kappa, float x) {
    const float u = (x + LLR_XMAX) * (1.0f / LLR_H);
    if (p.table4 && u >= 0.0f && u < 4095.0f) {
        const int i = (int)u;
        const float t = u - (float)i;
        const float4 f = __ldg(p.table4 + (size_t)combo_of(p.known_mask, kappa) * LLR_NWIN + i);  // .x: point i-1
        const float tm1 = t - 1.0f, tm2 = t - 2.0f, tp1 = t + 1.0f;
        const float L = (-t * tm1 * tm2 * (1.0f / 6.0f)) * f.x + (tp1 * tm1 * tm2 * 0.5f) * f.y +
                        (-tp1 * t * tm2 * 0.5f) * f.z + (tp1 * t * tm1 * (1.0f / 6.0f)) * f.w;
        return llr_clamp(L, p.llr_max);
    }
    return llr_cond(se, p.m, p.j, p.known_mask, kappa, x, p.inv_sigma, p.llr_max);
}

// public API: natural layout out[f][v]
__global__ void k_llr_slice(LlrParams p, const float *__restrict__ x, const uint8_t *__restrict__ known_label,
                            int64_t count, float *__restrict__ out) {
    __shared__ float se[256];
    for (int i = threadIdx.x; i < 255; i += blockDim.x) se[i] = p.edges[i];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t kappa = p.known_mask ? known_label[i] : 0u;
        out[i] = llr_eval(p, se, kappa, x[i]);
    }
}

// L(x) from the table for the known-bit pattern with table index `combo` (bit t =
// slice kj[t]); exact evaluation off the grid
__device__ __forceinline__ float llr_eval_combo(const LlrParams &p, const float *se, uint32_t combo, float x) {
    const float u = (x + LLR_XMAX) * (1.0f / LLR_H);
    if (p.table4 && u >= 0.0f && u < 4095.0f) {
        const int i = (int)u;
        const float t = u - (float)i;
        const float4 f = __ldg(p.table4 + (size_t)combo * LLR_NWIN + i);  // .x: grid point i-1
        const float tm1 = t - 1.0f, tm2 = t - 2.0f, tp1 = t + 1.0f;
        const float L = (-t * tm1 * tm2 * (1.0f / 6.0f)) * f.x + (tp1 * tm1 * tm2 * 0.5f) * f.y +
                        (-tp1 * t * tm2 * 0.5f) * f.z + (tp1 * t * tm1 * (1.0f / 6.0f)) * f.w;
        return llr_clamp(L, p.llr_max);
    }
    return llr_cond(se, p.m, p.j, p.known_mask, kappa_of(p.known_mask, (int)combo), x, p.inv_sigma, p.llr_max);
}

// decoder feed: conditional LLR written straight into the interleaved arena
// L[t][v][lane][S] (fused transpose, log2 units); known bits read from the
// packed slices.  NK = number of known slices (compile time: the table index is
// assembled with NK unrolled bit extractions, no per-symbol mask walking).  A block
// covers LLR_VB groups of 32 variables of one tile (the edge table is staged once per
// block).  hb != nullptr (layered schedule): the initial hard decisions hb[t][v] =
// [L < 0] of the tile's active frames are written as well (k_layer_init's job).
constexpr int LLR_VB = 4;
template <int S, int NK>
__global__ void __launch_bounds__(256) k_llr_interleaved(LlrParams p, const float *__restrict__ x, int32_t F,
                                                         int32_t n, float *__restrict__ L, uint4 *__restrict__ hb,
                                                         const uint4 *__restrict__ tile_active) {
    __shared__ float se[256];
    __shared__ float sm[LANES * S][33];
    for (int i = threadIdx.x; i < 255; i += blockDim.x) se[i] = p.edges[i];
    const int t = blockIdx.y;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int Wn = words_of(n);
    const uint4 act = hb ? tile_active[t] : make_uint4(0u, 0u, 0u, 0u);
    for (int g = 0; g < LLR_VB; ++g) {
        const int v0 = (blockIdx.x * LLR_VB + g) * 32;
        if (v0 >= n) break;  // block-uniform
        __syncthreads();     // se staged / sm free again
        const int v = v0 + tx;
        const uint32_t *kb[NK > 0 ? NK : 1];
#pragma unroll
        for (int k = 0; k < NK; ++k) kb[k] = p.known_bits[p.kj[k]] + (v0 >> 5);
        for (int fl = ty; fl < LANES * S; fl += 8) {
            const int f = t * LANES * S + fl;
            float val = 0.0f;
            if (f < F && v < n) {
                uint32_t combo = 0u;
#pragma unroll
                for (int k = 0; k < NK; ++k) combo |= ((__ldg(kb[k] + (size_t)f * Wn) >> tx) & 1u) << k;
                val = llr_eval_combo(p, se, combo, x[(size_t)f * n + v]);
            }
            sm[fl][tx] = val * LOG2E;  // arena: log2 units
        }
        __syncthreads();
        for (int vl = ty; vl < 32; vl += 8) {
            const int vv = v0 + vl;
            if (vv < n) {  // warp-uniform
                FV<S> o;
#pragma unroll
                for (int s = 0; s < S; ++s) o.c[s] = sm[s * LANES + tx][vl];
                stv<S>(L + (((size_t)t * n + vv) * LANES + tx) * S, o);
                if (hb) {
                    uint32_t w[SUBS] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (int s = 0; s < S; ++s) w[s] = __ballot_sync(0xffffffffu, o.c[s] < 0.0f) & cmpu(act, s);
                    if (tx == 0) hb[(size_t)t * n + vv] = make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
        }
    }
}

__global__ void k_llr_biawgn(const float *__restrict__ y, int64_t count, float sigma2, float llr_max,
                             float *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = fminf(fmaxf(2.0f * y[i] / sigma2, -llr_max), llr_max);
}

static int grid_for(int64_t work, int block) {
    int64_t g = (work + block - 1) / block;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

// table for p (p.table is the destination); returns false when the grid is too coarse for sigma_n
bool launch_llr_table(const LlrParams &p, float *table, float4 *table4, cudaStream_t s) {
    if (LLR_H * p.inv_sigma > 0.02f) return false;
    const int combos = 1 << __builtin_popcount(p.known_mask);
    const int total = combos * LLR_NTAB;
    k_llr_table<<<(total + 255) / 256, 256, 0, s>>>(p, table, combos);
    k_llr_window<<<(combos * LLR_NWIN + 255) / 256, 256, 0, s>>>(table, table4, combos);
    return true;
}

void launch_llr_slice(const LlrParams &p, const float *x, const uint8_t *known_label, int32_t F, int32_t n,
                      float *out, cudaStream_t s) {
    const int64_t count = (int64_t)F * n;
    k_llr_slice<<<grid_for(count, 256), 256, 0, s>>>(p, x, known_label, count, out);
}

void launch_llr_biawgn(const float *y, int64_t count, float sigma2, float llr_max, float *out, cudaStream_t s) {
    k_llr_biawgn<<<grid_for(count, 256), 256, 0, s>>>(y, count, sigma2, llr_max, out);
}

template <int S>
static void launch_llr_il_s(const LlrParams &p, const float *x, int32_t F, int32_t n, dim3 grid, float *L, uint4 *hb,
                            const uint4 *act, cudaStream_t s) {
    switch (p.nk) {
        case 0: k_llr_interleaved<S, 0><<<grid, 256, 0, s>>>(p, x, F, n, L, hb, act); break;
        case 1: k_llr_interleaved<S, 1><<<grid, 256, 0, s>>>(p, x, F, n, L, hb, act); break;
        case 2: k_llr_interleaved<S, 2><<<grid, 256, 0, s>>>(p, x, F, n, L, hb, act); break;
        case 3: k_llr_interleaved<S, 3><<<grid, 256, 0, s>>>(p, x, F, n, L, hb, act); break;
        case 4: k_llr_interleaved<S, 4><<<grid, 256, 0, s>>>(p, x, F, n, L, hb, act); break;
        case 5: k_llr_interleaved<S, 5><<<grid, 256, 0, s>>>(p, x, F, n, L, hb, act); break;
        case 6: k_llr_interleaved<S, 6><<<grid, 256, 0, s>>>(p, x, F, n, L, hb, act); break;
        default: k_llr_interleaved<S, 7><<<grid, 256, 0, s>>>(p, x, F, n, L, hb, act); break;
    }
}

void launch_llr_interleaved(const LlrParams &p, const float *x, int32_t F, int32_t n, int tiles, int subs, float *L,
                            uint4 *hb, const uint4 *tile_active, cudaStream_t s) {
    dim3 grid((n + 32 * LLR_VB - 1) / (32 * LLR_VB), tiles);
    if (subs == 4) launch_llr_il_s<4>(p, x, F, n, grid, L, hb, tile_active, s);
    else if (subs == 2) launch_llr_il_s<2>(p, x, F, n, grid, L, hb, tile_active, s);
    else launch_llr_il_s<1>(p, x, F, n, grid, L, hb, tile_active, s);
}

}  // namespace cvsr
