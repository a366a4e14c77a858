// Toeplitz privacy amplification on the GPU (Step 6).
//
// y = T x over GF(2), T[i][j] = t[i - j + n_in - 1] (seed t of n_in + n_out - 1 bits),
// i.e. y_i = (t * x)[n_in - 1 + i] mod 2 for the integer convolution t * x.  The
// convolution is computed exactly with a number-theoretic transform modulo the
// prime p = 15 * 2^27 + 1 (primitive root 31): every coefficient is at most
// n_in < p, and a cyclic length N >= n_in + n_out - 1 leaves the window
// [n_in - 1, n_in + n_out - 2] free of wrap-around.  Transform layout:
//   forward = decimation in frequency (natural in, bit-reversed out),
//   inverse = decimation in time (bit-reversed in, natural out),
// so no bit-reversal permutation is ever materialised.  Stages with butterfly
// half-size >= 4096 run as radix-2^r passes over global memory (one thread per
// group of 2^r elements, r <= 4 stages per pass, coalesced by construction);
// the 12 lowest stages of the forward transform, the pointwise product with the
// seed's transform and the 12 lowest stages of the inverse run in ONE
// shared-memory kernel per 4096-element block.  Values are kept in [0, p); the
// twiddles and the seed transform are stored in Montgomery form (R = 2^32) so a
// product is one Montgomery multiplication.
#include <stdint.h>

#include <cuda_runtime.h>

#include "common.cuh"

namespace cvsr {
namespace pa {

constexpr uint32_t P = 2013265921u;  // 15 * 2^27 + 1
constexpr uint32_t G = 31u;          // primitive root mod P
constexpr int MAX_LOG_N = 27;
constexpr int MID_LOG = 12;          // stages handled in shared memory

constexpr uint32_t neg_inv_p() {     // -P^-1 mod 2^32 by Newton iteration
    uint32_t x = P;                  // P * P = 1 mod 8
    for (int i = 0; i < 5; ++i) x *= 2u - P * x;
    return 0u - x;
}
constexpr uint32_t PINV = neg_inv_p();
static_assert((uint32_t)(P * (0u - PINV)) == 1u, "Montgomery constant");

__host__ __device__ __forceinline__ uint32_t mont_mul(uint32_t a, uint32_t b) {
    const uint64_t t = (uint64_t)a * b;
    const uint32_t m = (uint32_t)t * PINV;
    const uint32_t u = (uint32_t)((t + (uint64_t)m * P) >> 32);
    return u >= P ? u - P : u;
}
// a w mod P for a fixed w with wq = floor(w 2^32 / P) (Shoup): 3 32-bit multiplies, no 64-bit product
__device__ __forceinline__ uint32_t mul_shoup(uint32_t a, uint32_t w, uint32_t wq) {
    const uint32_t q = __umulhi(a, wq);
    const uint32_t r = a * w - q * P;
    return r >= P ? r - P : r;
}
__device__ __forceinline__ uint32_t addp(uint32_t a, uint32_t b) {
    const uint32_t r = a + b;
    return r >= P ? r - P : r;
}
__device__ __forceinline__ uint32_t subp(uint32_t a, uint32_t b) { return a >= b ? a - b : a + P - b; }

__host__ __device__ inline uint32_t mulmod(uint32_t a, uint32_t b) { return (uint32_t)((uint64_t)a * b % P); }
__host__ __device__ inline uint32_t powmod(uint32_t b, uint64_t e) {
    uint32_t r = 1u;
    while (e) {
        if (e & 1u) r = mulmod(r, b);
        b = mulmod(b, b);
        e >>= 1;
    }
    return r;
}
__host__ __device__ inline uint32_t to_mont(uint32_t a) { return (uint32_t)(((uint64_t)a << 32) % P); }

// twiddles: T[h - 1 + j] = w_2h^(+-j) in Montgomery form, h = 1, 2, ..., N/2, j < h
__global__ void k_twiddles(uint32_t *__restrict__ tw, uint32_t *__restrict__ twi, uint2 *__restrict__ sh,
                           uint2 *__restrict__ shi, int64_t N) {
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < N - 1;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int lg = 63 - __clzll((unsigned long long)(idx + 1));  // h = 2^lg <= idx + 1 < 2h
        const int64_t h = 1LL << lg, j = idx - (h - 1);
        const uint64_t step = (uint64_t)(P - 1) / (uint64_t)(2 * h);  // w_2h = G^step
        const uint64_t e = (step * (uint64_t)j) % (P - 1);
        const uint32_t w = powmod(G, e), wi = powmod(G, (P - 1 - e) % (P - 1));
        tw[idx] = to_mont(w);
        twi[idx] = to_mont(wi);
        if (idx < (1 << MID_LOG)) {  // the shared-memory stages use Shoup pairs (w, floor(w 2^32 / P))
            sh[idx] = make_uint2(w, (uint32_t)(((uint64_t)w << 32) / P));
            shi[idx] = make_uint2(wi, (uint32_t)(((uint64_t)wi << 32) / P));
        }
    }
}

// bits (LSB first) -> values 0/1, zero-padded to N
__global__ void k_unpack(const uint32_t *__restrict__ bits, int64_t nbits, uint32_t *__restrict__ a, int64_t N) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = i < nbits ? (__ldg(bits + (i >> 5)) >> (i & 31)) & 1u : 0u;
}

// Twiddles of a radix-2^RB pass from ONE table load per thread: for the pass's top
// stage (half-size H = d 2^(RB-1)) b = w_2H^off; stage sh (half-size h = d 2^sh) needs
// w_2h^(off + q' d) = b^(2^(RB-1-sh)) * w_(2^(sh+1))^q', the second factor from the
// tiny head of the table (index 2^sh - 1 + q').

// forward DIF stages s_hi .. s_hi - RB + 1 (half-size >= 2^MID_LOG), one thread per group;
// xbits != null: the input is the packed bit string (first pass), values 0/1
template <int RB>
__global__ void __launch_bounds__(256) k_dif_pass(uint32_t *__restrict__ a, const uint32_t *__restrict__ tw,
                                                  int s_hi, int64_t N, const uint32_t *__restrict__ xbits,
                                                  int64_t nbits) {
    constexpr int Q = 1 << RB;
    const int S0 = s_hi - RB + 1;
    const int64_t d = 1LL << S0, groups = N >> RB;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t off = g & (d - 1), base = ((g >> S0) << (S0 + RB)) + off;
        uint32_t v[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int64_t i = base + q * d;
            v[q] = xbits ? (i < nbits ? (__ldg(xbits + (i >> 5)) >> (i & 31)) & 1u : 0u) : a[i];
        }
        uint32_t b = __ldg(tw + (d << (RB - 1)) - 1 + off);  // w_2H^off
#pragma unroll
        for (int sh = RB - 1; sh >= 0; --sh) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                if (q & (1 << sh)) continue;
                const int qq = q & ((1 << sh) - 1);
                const uint32_t w = qq ? mont_mul(b, __ldg(tw + (1 << sh) - 1 + qq)) : b;
                const uint32_t x = v[q], y = v[q + (1 << sh)];
                v[q] = addp(x, y);
                v[q + (1 << sh)] = mont_mul(subp(x, y), w);
            }
            b = mont_mul(b, b);
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) a[base + q * d] = v[q];
    }
}

// inverse DIT stages s_lo .. s_lo + RB - 1 (inverse twiddle table, same derivation)
template <int RB>
__global__ void __launch_bounds__(256) k_dit_pass(uint32_t *__restrict__ a, const uint32_t *__restrict__ twi,
                                                  int s_lo, int64_t N, const uint32_t *__restrict__, int64_t) {
    constexpr int Q = 1 << RB;
    const int S0 = s_lo;
    const int64_t d = 1LL << S0, groups = N >> RB;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t off = g & (d - 1), base = ((g >> S0) << (S0 + RB)) + off;
        uint32_t v[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) v[q] = a[base + q * d];
        uint32_t bs[RB];  // bs[sh] = w_2h^-off for stage sh
        bs[RB - 1] = __ldg(twi + (d << (RB - 1)) - 1 + off);
#pragma unroll
        for (int sh = RB - 2; sh >= 0; --sh) bs[sh] = mont_mul(bs[sh + 1], bs[sh + 1]);
#pragma unroll
        for (int sh = 0; sh < RB; ++sh) {
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                if (q & (1 << sh)) continue;
                const int qq = q & ((1 << sh) - 1);
                const uint32_t w = qq ? mont_mul(bs[sh], __ldg(twi + (1 << sh) - 1 + qq)) : bs[sh];
                const uint32_t x = v[q], y = mont_mul(v[q + (1 << sh)], w);
                v[q] = addp(x, y);
                v[q + (1 << sh)] = subp(x, y);
            }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) a[base + q * d] = v[q];
    }
}

// the lowest lb stages of the forward DIF of a block of B = 2^lb contiguous values, then
// (tm != null) the pointwise product with the seed transform and the lowest lb stages of
// the inverse DIT, in shared memory
__global__ void __launch_bounds__(512) k_ntt_mid(uint32_t *__restrict__ a, const uint2 *__restrict__ tw,
                                                 const uint2 *__restrict__ twi, const uint32_t *__restrict__ tm,
                                                 int lb) {
    __shared__ uint32_t s[1 << MID_LOG];
    const int B = 1 << lb;
    uint32_t *blk = a + (int64_t)blockIdx.x * B;
    for (int i = threadIdx.x; i < B; i += blockDim.x) s[i] = blk[i];
    __syncthreads();
    for (int st = lb - 1; st >= 0; --st) {
        const int h = 1 << st;
        for (int b = threadIdx.x; b < B / 2; b += blockDim.x) {
            const int j = b & (h - 1), i = ((b >> st) << (st + 1)) + j;
            const uint32_t x = s[i], y = s[i + h];
            const uint2 w = __ldg(tw + h - 1 + j);
            s[i] = addp(x, y);
            s[i + h] = mul_shoup(subp(x, y), w.x, w.y);
        }
        __syncthreads();
    }
    if (tm) {
        const uint32_t *tb = tm + (int64_t)blockIdx.x * B;
        for (int i = threadIdx.x; i < B; i += blockDim.x) s[i] = mont_mul(s[i], __ldg(tb + i));
        __syncthreads();
        for (int st = 0; st < lb; ++st) {
            const int h = 1 << st;
            for (int b = threadIdx.x; b < B / 2; b += blockDim.x) {
                const int j = b & (h - 1), i = ((b >> st) << (st + 1)) + j;
                const uint2 w = __ldg(twi + h - 1 + j);
                const uint32_t x = s[i], y = mul_shoup(s[i + h], w.x, w.y);
                s[i] = addp(x, y);
                s[i + h] = subp(x, y);
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < B; i += blockDim.x) blk[i] = s[i];
}

// Specialisation for full 4096-value blocks (lb = MID_LOG = 12): 512 threads own 8 values
// each; the 12 stages per direction run as 4 radix-8 steps entirely in registers
// (compile-time indices, 12 butterflies per thread and step, one barrier per step).
// Shared memory is padded by one word per 32 (conflict-free except 2-way in one step).
__device__ __forceinline__ int pad32(int i) { return i + (i >> 5); }

template <int S0, bool FWD>
__device__ __forceinline__ void mid8(uint32_t *s, const uint2 *__restrict__ tab, int g) {
    constexpr int d = 1 << S0;
    const int off = g & (d - 1), base = ((g >> S0) << (S0 + 3)) + off;
    uint32_t v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = s[pad32(base + q * d)];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int sh = FWD ? 2 - k : k;
        const int h = d << sh;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q & (1 << sh)) continue;
            const uint2 w = __ldg(tab + h - 1 + off + (q & ((1 << sh) - 1)) * d);
            const uint32_t x = v[q];
            if (FWD) {
                const uint32_t y = v[q + (1 << sh)];
                v[q] = addp(x, y);
                v[q + (1 << sh)] = mul_shoup(subp(x, y), w.x, w.y);
            } else {
                const uint32_t y = mul_shoup(v[q + (1 << sh)], w.x, w.y);
                v[q] = addp(x, y);
                v[q + (1 << sh)] = subp(x, y);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) s[pad32(base + q * d)] = v[q];
}

__global__ void __launch_bounds__(512) k_ntt_mid12(uint32_t *__restrict__ a, const uint2 *__restrict__ tw,
                                                   const uint2 *__restrict__ twi, const uint32_t *__restrict__ tm) {
    __shared__ uint32_t s[4096 + 128];
    uint32_t *blk = a + (int64_t)blockIdx.x * 4096;
    const int g = threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) s[pad32(g + 512 * k)] = blk[g + 512 * k];
    __syncthreads();
    mid8<9, true>(s, tw, g);
    __syncthreads();
    mid8<6, true>(s, tw, g);
    __syncthreads();
    mid8<3, true>(s, tw, g);
    __syncthreads();
    mid8<0, true>(s, tw, g);
    __syncthreads();
    if (tm) {
        const uint32_t *tb = tm + (int64_t)blockIdx.x * 4096;
#pragma unroll
        for (int k = 0; k < 8; ++k) s[pad32(g + 512 * k)] = mont_mul(s[pad32(g + 512 * k)], __ldg(tb + g + 512 * k));
        __syncthreads();
        mid8<0, false>(s, twi, g);
        __syncthreads();
        mid8<3, false>(s, twi, g);
        __syncthreads();
        mid8<6, false>(s, twi, g);
        __syncthreads();
        mid8<9, false>(s, twi, g);
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) blk[g + 512 * k] = s[pad32(g + 512 * k)];
}

__global__ void k_to_mont(uint32_t *__restrict__ a, int64_t N) {
    const uint32_t r2 = to_mont(to_mont(1u));  // R^2 mod P: mont_mul(x, R^2) = x R
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = mont_mul(a[i], r2);
}

// y_i = (N^-1 c[n_in - 1 + i]) & 1, packed LSB first; one warp per output word
__global__ void __launch_bounds__(256) k_pack_window(const uint32_t *__restrict__ c, int64_t n_in, int64_t n_out,
                                                     uint32_t ninv_mont, uint32_t *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int64_t words = (n_out + 31) / 32;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < words;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t i = w * 32 + lane;
        const uint32_t b = i < n_out ? mont_mul(c[n_in - 1 + i], ninv_mont) & 1u : 0u;
        const uint32_t word = __ballot_sync(0xffffffffu, b);
        if (lane == 0) y[w] = word;
    }
}

static int grid_for(int64_t work, int block) {
    int64_t g = (work + block - 1) / block;
    if (g > 148 * 16) g = 148 * 16;
    return (int)(g < 1 ? 1 : g);
}

template <typename K>
static void launch_radix(K k1, K k2, K k3, K k4, int rb, uint32_t *a, const uint32_t *tw, int s, int64_t N,
                         const uint32_t *xbits, int64_t nbits, cudaStream_t st) {
    const int g = grid_for(N >> rb, 256);
    switch (rb) {
        case 1: k1<<<g, 256, 0, st>>>(a, tw, s, N, xbits, nbits); break;
        case 2: k2<<<g, 256, 0, st>>>(a, tw, s, N, xbits, nbits); break;
        case 3: k3<<<g, 256, 0, st>>>(a, tw, s, N, xbits, nbits); break;
        default: k4<<<g, 256, 0, st>>>(a, tw, s, N, xbits, nbits); break;
    }
}

// forward DIF of a (natural in, bit-reversed out) when tm == null; with tm: forward,
// pointwise product with tm (Montgomery form, bit-reversed) and inverse DIT (natural out,
// scaled by N).  The input is the packed bit string xbits of nbits bits, unpacked on the
// fly by the first pass.  Returns the number of kernel launches.
static int ntt_run(uint32_t *a, const uint32_t *tw, const uint32_t *twi, const uint2 *sh, const uint2 *shi,
                   const uint32_t *tm, int lg, const uint32_t *xbits, int64_t nbits, cudaStream_t st) {
    const int64_t N = 1LL << lg;
    const int lb = lg < MID_LOG ? lg : MID_LOG;
    int launches = 0;
    if (lg == lb) {  // no global pass to fuse the unpacking into
        k_unpack<<<grid_for(N, 256), 256, 0, st>>>(xbits, nbits, a, N);
        ++launches;
        xbits = nullptr;
    }
    for (int s_hi = lg - 1; s_hi >= lb;) {  // global DIF passes, highest stages first
        const int rb = (s_hi - lb + 1) >= 4 ? 4 : (s_hi - lb + 1);
        launch_radix(k_dif_pass<1>, k_dif_pass<2>, k_dif_pass<3>, k_dif_pass<4>, rb, a, tw, s_hi, N, xbits, nbits,
                     st);
        xbits = nullptr;
        ++launches;
        s_hi -= rb;
    }
    if (lb == MID_LOG) k_ntt_mid12<<<(unsigned)(N >> lb), 512, 0, st>>>(a, sh, shi, tm);
    else k_ntt_mid<<<(unsigned)(N >> lb), 512, 0, st>>>(a, sh, shi, tm, lb);
    ++launches;
    if (!tm) return launches;
    for (int s_lo = lb; s_lo < lg;) {  // global DIT passes, lowest remaining stages first
        const int rb = (lg - s_lo) >= 4 ? 4 : (lg - s_lo);
        launch_radix(k_dit_pass<1>, k_dit_pass<2>, k_dit_pass<3>, k_dit_pass<4>, rb, a, twi, s_lo, N, nullptr, 0,
                     st);
        ++launches;
        s_lo += rb;
    }
    return launches;
}

}  // namespace pa
}  // namespace cvsr

using namespace cvsr::pa;

struct cvsr_pa_plan {
    int device = 0;
    int lg = 0;
    int64_t n_in = 0, n_out = 0, N = 0;
    uint32_t *mem = nullptr;
    uint32_t *tw = nullptr, *twi = nullptr, *tm = nullptr, *work = nullptr;
    uint2 *sh = nullptr, *shi = nullptr;  // Shoup pairs of the first 2^MID_LOG twiddles
};

cudaStream_t cvsr_internal_ctx_stream(cvsr_ctx *ctx);
cvsr_status cvsr_internal_fail(cvsr_status st, const char *msg);
cvsr_status cvsr_internal_launched(cvsr_ctx *ctx, int n);
int cvsr_internal_ctx_device(cvsr_ctx *ctx);

extern "C" {

cvsr_status cvsr_pa_plan_create(cvsr_ctx *ctx, int64_t n_in, int64_t n_out, const uint32_t *seed_bits_host,
                                cvsr_pa_plan **out) {
    if (!ctx || !seed_bits_host || !out) return cvsr_internal_fail(CVSR_EINVAL, "pa: null argument");
    *out = nullptr;
    if (n_in < 1 || n_out < 1 || n_out > n_in) return cvsr_internal_fail(CVSR_ESHAPE, "pa: need 1 <= n_out <= n_in");
    const int64_t need = n_in + n_out - 1;
    int lg = 1;  // N >= 2 so the shared-memory kernel always applies the product
    while ((1LL << lg) < need) ++lg;
    if (lg > MAX_LOG_N) return cvsr_internal_fail(CVSR_ESHAPE, "pa: n_in + n_out - 1 exceeds 2^27");
    cvsr_pa_plan *p = new cvsr_pa_plan();
    p->device = cvsr_internal_ctx_device(ctx);
    p->lg = lg;
    p->n_in = n_in;
    p->n_out = n_out;
    p->N = 1LL << lg;
    const int64_t N = p->N;
    if (cudaMalloc(&p->mem, (size_t)N * 4 * 4 + 2 * (size_t)(1 << MID_LOG) * 8) != cudaSuccess) {
        cudaGetLastError();
        delete p;
        return cvsr_internal_fail(CVSR_ENOMEM, "pa: plan buffers");
    }
    p->tw = p->mem;
    p->twi = p->mem + N;
    p->tm = p->mem + 2 * N;
    p->work = p->mem + 3 * N;
    p->sh = reinterpret_cast<uint2 *>(p->mem + 4 * N);
    p->shi = p->sh + (1 << MID_LOG);
    cudaStream_t st = cvsr_internal_ctx_stream(ctx);
    const int64_t sw = (need + 31) / 32;
    uint32_t *seed_dev = nullptr;
    if (cudaMallocAsync(&seed_dev, (size_t)sw * 4, st) != cudaSuccess ||
        cudaMemcpyAsync(seed_dev, seed_bits_host, (size_t)sw * 4, cudaMemcpyHostToDevice, st) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(p->mem);
        delete p;
        return cvsr_internal_fail(CVSR_ECUDA, "pa: seed upload");
    }
    int launches = 0;
    k_twiddles<<<grid_for(N - 1, 256), 256, 0, st>>>(p->tw, p->twi, p->sh, p->shi, N);
    ++launches;
    launches += ntt_run(p->tm, p->tw, p->twi, p->sh, p->shi, nullptr, lg, seed_dev, need, st);
    k_to_mont<<<grid_for(N, 256), 256, 0, st>>>(p->tm, N);
    ++launches;
    cudaFreeAsync(seed_dev, st);
    if (cvsr_status r = cvsr_internal_launched(ctx, launches)) {
        cudaFree(p->mem);
        delete p;
        return r;
    }
    *out = p;
    return CVSR_OK;
}

cvsr_status cvsr_pa_plan_info(const cvsr_pa_plan *p, int64_t *n_in, int64_t *n_out, int64_t *ntt_size) {
    if (!p) return cvsr_internal_fail(CVSR_EINVAL, "pa: null plan");
    if (n_in) *n_in = p->n_in;
    if (n_out) *n_out = p->n_out;
    if (ntt_size) *ntt_size = p->N;
    return CVSR_OK;
}

cvsr_status cvsr_pa_hash(cvsr_ctx *ctx, const cvsr_pa_plan *p, int32_t blocks, const uint32_t *x_bits,
                         uint32_t *y_bits) {
    if (!ctx || !p) return cvsr_internal_fail(CVSR_EINVAL, "pa: null context or plan");
    if (blocks < 0) return cvsr_internal_fail(CVSR_ESHAPE, "pa: blocks < 0");
    if (blocks == 0) return CVSR_OK;
    if (!x_bits || !y_bits) return cvsr_internal_fail(CVSR_EINVAL, "pa: null buffer");
    if (p->device != cvsr_internal_ctx_device(ctx)) return cvsr_internal_fail(CVSR_EINVAL, "pa: plan on another device");
    cudaStream_t st = cvsr_internal_ctx_stream(ctx);
    const int64_t wi = (p->n_in + 31) / 32, wo = (p->n_out + 31) / 32;
    const uint32_t ninv = to_mont(powmod((uint32_t)(p->N % P), P - 2));
    int launches = 0;
    for (int32_t b = 0; b < blocks; ++b) {
        launches += ntt_run(p->work, p->tw, p->twi, p->sh, p->shi, p->tm, p->lg, x_bits + b * wi, p->n_in, st);
        k_pack_window<<<grid_for(wo * 32, 256), 256, 0, st>>>(p->work, p->n_in, p->n_out, ninv, y_bits + b * wo);
        ++launches;
    }
    return cvsr_internal_launched(ctx, launches);
}

void cvsr_pa_plan_free(cvsr_pa_plan *p) {
    if (!p) return;
    cudaFree(p->mem);
    delete p;
}

}  // extern "C"
