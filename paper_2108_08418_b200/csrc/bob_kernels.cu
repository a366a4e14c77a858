// Bob-side kernels (quantise, slice bits, syndrome) and reconcile bookkeeping.
#include "common.cuh"
#include "kernels.cuh"

namespace cvsr {

constexpr unsigned FULLB = 0xffffffffu;

struct QEdges {
    float e[255];
};

// K1: b = #{k : y >= e_k} (branchless binary search over the sorted fp32 table,
// comparisons only => bit-exact), label = b ^ (b >> 1)
__device__ __forceinline__ uint8_t quantise_one(float y, const float *se, int m) {
    int b = 0;
    for (int s = 1 << (m - 1); s; s >>= 1)
        if (y >= se[b + s - 1]) b += s;
    return (uint8_t)(b ^ (b >> 1));
}

__global__ void k_quantise(QEdges q, int m, const float *__restrict__ y, int64_t count, uint8_t *__restrict__ label) {
    __shared__ float se[256];
    for (int i = threadIdx.x; i < 255; i += blockDim.x) se[i] = q.e[i];
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(y) & 15) == 0) && ((reinterpret_cast<uintptr_t>(label) & 3) == 0);
    if (vec) {
        const int64_t n4 = count / 4;
        const float4 *y4 = reinterpret_cast<const float4 *>(y);
        uchar4 *l4 = reinterpret_cast<uchar4 *>(label);
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
            const float4 v = y4[i];
            uchar4 o;
            o.x = quantise_one(v.x, se, m);
            o.y = quantise_one(v.y, se, m);
            o.z = quantise_one(v.z, se, m);
            o.w = quantise_one(v.w, se, m);
            l4[i] = o;
        }
        for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
            label[i] = quantise_one(y[i], se, m);
    } else {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
            label[i] = quantise_one(y[i], se, m);
    }
}

// S_j packed: warp per (frame, 32-var word)
__global__ void __launch_bounds__(BLOCK) k_slice_bits(const uint8_t *__restrict__ label, int32_t n, int32_t j,
                                                       uint32_t *__restrict__ bits) {
    const int f = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Wn = words_of(n);
    const int w = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (w >= Wn) return;
    const int v = w * 32 + lane;
    const uint32_t b = (v < n) ? (label[(size_t)f * n + v] >> j) & 1u : 0u;
    const uint32_t word = __ballot_sync(FULLB, b);
    if (lane == 0) bits[(size_t)f * Wn + w] = word;
}

// K2: s_j[c] = XOR_{v in row c} bit_j(label[v]); warp per (frame, 32-check word), lane = check
__global__ void __launch_bounds__(BLOCK) k_syndrome(CodeDev cd, const uint8_t *__restrict__ label, int32_t j,
                                                     uint32_t *__restrict__ synd) {
    const int f = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Wm = words_of(cd.M);
    const int w = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (w >= Wm) return;
    const int c = w * 32 + lane;
    uint32_t par = 0u;
    if (c < cd.M) {
        const uint8_t *lab = label + (size_t)f * cd.n;
        const int beg = cd.row_ptr[c], end = cd.row_ptr[c + 1];
        for (int e = beg; e < end; ++e) par ^= lab[cd.col_idx[e]];
        par = (par >> j) & 1u;
    }
    const uint32_t word = __ballot_sync(FULLB, par);
    if (lane == 0) synd[(size_t)f * Wm + w] = word;
}

// K2 from packed slice bits (bits[f][Wn], an 8 KB row per frame at N_R = 2^16 stays in L1)
__global__ void __launch_bounds__(BLOCK) k_syndrome_bits(CodeDev cd, const uint32_t *__restrict__ bits,
                                                          uint32_t *__restrict__ synd) {
    const int f = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Wm = words_of(cd.M), Wn = words_of(cd.n);
    const int w = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (w >= Wm) return;
    const int c = w * 32 + lane;
    uint32_t par = 0u;
    if (c < cd.M) {
        const uint32_t *b = bits + (size_t)f * Wn;
        const int beg = cd.row_ptr[c], end = cd.row_ptr[c + 1];
        for (int e = beg; e < end; ++e) {
            const int v = cd.col_idx[e];
            par ^= b[v >> 5] >> (v & 31);
        }
        par &= 1u;
    }
    const uint32_t word = __ballot_sync(FULLB, par);
    if (lane == 0) synd[(size_t)f * Wm + w] = word;
}

// simulation check: counts {ok frames, ok frames with any label mismatch, mismatching bytes}
__global__ void k_count_errors(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b,
                               const uint8_t *__restrict__ ok, int32_t n, unsigned long long *counts) {
    const int f = blockIdx.x;
    if (!ok[f]) return;
    unsigned long long cnt = 0;
    for (int v = threadIdx.x; v < n; v += blockDim.x) cnt += (a[(size_t)f * n + v] != b[(size_t)f * n + v]);
    __shared__ unsigned long long s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULLB, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&s, cnt);
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(&counts[0], 1ull);
        if (s) {
            atomicAdd(&counts[1], 1ull);
            atomicAdd(&counts[2], s);
        }
    }
}

// After slice j: record D_j, attempt/converged masks, kill failed frames (reading A-13).
// attempt[f] bit j: slice j attempted; attempt[F + f] bit j: slice j converged/disclosed.
__global__ void k_slice_done(DecState ds, int32_t m, int32_t j, int disclosed, uint8_t *alive, uint8_t *attempt,
                             int32_t *iters_out) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= ds.frames || !alive[f]) return;
    attempt[f] |= (uint8_t)(1u << j);
    if (disclosed) {
        iters_out[(size_t)f * m + j] = 0;
        attempt[ds.frames + f] |= (uint8_t)(1u << j);
        return;
    }
    iters_out[(size_t)f * m + j] = ds.iters[f];
    if (ds.conv[f]) attempt[ds.frames + f] |= (uint8_t)(1u << j);
    else alive[f] = 0;
}

struct BitPtrs {
    const uint32_t *p[8];
};

__global__ void k_assemble(BitPtrs bits, int32_t m, const uint8_t *__restrict__ attempt, int32_t n,
                           uint8_t *__restrict__ label_out) {
    const int f = blockIdx.y;
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int Wn = words_of(n);
    const uint32_t am = attempt[f];
    uint32_t lab = 0u;
    for (int j = 0; j < m; ++j)
        if ((am >> j) & 1u) lab |= ((bits.p[j][(size_t)f * Wn + (v >> 5)] >> (v & 31)) & 1u) << j;
    label_out[(size_t)f * n + v] = (uint8_t)lab;
}

__global__ void k_fill_i32(int32_t *p, int64_t count, int32_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_fill_u8(uint8_t *p, int64_t count, uint8_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// acc[0] ok frames; acc[1+j] attempted; acc[9+j] converged; acc[17+j] sum D_j (attempted)
__global__ void k_frame_stats(const uint8_t *__restrict__ alive, const uint8_t *__restrict__ attempt,
                              const int32_t *__restrict__ iters, int32_t F, int32_t m, unsigned long long *acc) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= F) return;
    if (alive[f]) atomicAdd(&acc[0], 1ull);
    const uint32_t am = attempt[f], cm = attempt[F + f];
    for (int j = 0; j < m; ++j) {
        if ((am >> j) & 1u) {
            atomicAdd(&acc[1 + j], 1ull);
            atomicAdd(&acc[17 + j], (unsigned long long)iters[(size_t)f * m + j]);
        }
        if ((cm >> j) & 1u) atomicAdd(&acc[9 + j], 1ull);
    }
}

// ---------------------------------------------------------------- launchers
static int grid_for(int64_t work, int block) {
    int64_t g = (work + block - 1) / block;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

void launch_quantise(const float *edges_host, int m, const float *y, int64_t count, uint8_t *label, cudaStream_t s) {
    QEdges q;
    for (int i = 0; i < 255; ++i) q.e[i] = (i < (1 << m) - 1) ? edges_host[i] : 0.0f;
    k_quantise<<<grid_for(count / 4 + 1, 256), 256, 0, s>>>(q, m, y, count, label);
}

void launch_slice_bits(const uint8_t *label, int32_t F, int32_t n, int32_t j, uint32_t *bits, cudaStream_t s) {
    dim3 grid((words_of(n) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, F);
    k_slice_bits<<<grid, BLOCK, 0, s>>>(label, n, j, bits);
}

void launch_syndrome(const CodeDev &cd, const uint8_t *label, int32_t F, int32_t j, uint32_t *synd, cudaStream_t s) {
    dim3 grid((words_of(cd.M) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, F);
    k_syndrome<<<grid, BLOCK, 0, s>>>(cd, label, j, synd);
}

void launch_syndrome_bits(const CodeDev &cd, const uint32_t *bits, int32_t F, uint32_t *synd, cudaStream_t s) {
    dim3 grid((words_of(cd.M) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, F);
    k_syndrome_bits<<<grid, BLOCK, 0, s>>>(cd, bits, synd);
}

void launch_count_errors(const uint8_t *a, const uint8_t *b, const uint8_t *ok, int32_t F, int32_t n,
                         unsigned long long *counts, cudaStream_t s) {
    k_count_errors<<<F, 256, 0, s>>>(a, b, ok, n, counts);
}

void launch_slice_done(const DecState &ds, int32_t m, int32_t j, int disclosed, uint8_t *alive, uint8_t *attempt,
                       int32_t *iters_out, cudaStream_t s) {
    k_slice_done<<<(ds.frames + 255) / 256, 256, 0, s>>>(ds, m, j, disclosed, alive, attempt, iters_out);
}

void launch_assemble(const uint32_t *const *bits, int32_t m, const uint8_t *attempt, int32_t F, int32_t n,
                     uint8_t *label_out, cudaStream_t s) {
    BitPtrs bp;
    for (int j = 0; j < 8; ++j) bp.p[j] = (j < m) ? bits[j] : nullptr;
    dim3 grid((n + 255) / 256, F);
    k_assemble<<<grid, 256, 0, s>>>(bp, m, attempt, n, label_out);
}

void launch_fill_i32(int32_t *p, int64_t count, int32_t v, cudaStream_t s) {
    k_fill_i32<<<grid_for(count, 256), 256, 0, s>>>(p, count, v);
}

void launch_fill_u8(uint8_t *p, int64_t count, uint8_t v, cudaStream_t s) {
    k_fill_u8<<<grid_for(count, 256), 256, 0, s>>>(p, count, v);
}

void launch_frame_stats(const uint8_t *alive, const uint8_t *attempt, const int32_t *iters, int32_t F, int32_t m,
                        unsigned long long *acc, cudaStream_t s) {
    k_frame_stats<<<(F + 255) / 256, 256, 0, s>>>(alive, attempt, iters, F, m, acc);
}

}  // namespace cvsr

namespace cvsr {

// ---------------------------------------------------------------- verification hash
// Polynomial hash over GF(p), p = 2^61 - 1 ("apply the same hash
// function to their reconciled strings and exchange the hash results"):
//   h_f = sum_{i=0}^{W-1} w_i * key^(i+1) mod p,
// w_i = the i-th little-endian 32-bit word of frame f's label bytes (zero-padded).
constexpr unsigned long long P61 = (1ull << 61) - 1ull;

__device__ __forceinline__ unsigned long long mulmod61(unsigned long long a, unsigned long long b) {
    const unsigned long long lo = a * b, hi = __umul64hi(a, b);
    unsigned long long r = (lo & P61) + ((lo >> 61) | (hi << 3));
    r = (r & P61) + (r >> 61);
    return r >= P61 ? r - P61 : r;
}

__device__ __forceinline__ unsigned long long addmod61(unsigned long long a, unsigned long long b) {
    const unsigned long long r = a + b;
    return r >= P61 ? r - P61 : r;
}

__device__ unsigned long long powmod61(unsigned long long b, unsigned long long e) {
    unsigned long long r = 1ull;
    while (e) {
        if (e & 1ull) r = mulmod61(r, b);
        b = mulmod61(b, b);
        e >>= 1;
    }
    return r;
}

__device__ __forceinline__ uint32_t label_word(const uint8_t *__restrict__ lab, int n, int i, bool aligned) {
    const int b0 = 4 * i;
    if (aligned) return __ldg(reinterpret_cast<const uint32_t *>(lab) + i);
    uint32_t w = 0u;
    for (int k = 0; k < 4 && b0 + k < n; ++k) w |= (uint32_t)lab[b0 + k] << (8 * k);
    return w;
}

// Block per frame; word i goes to thread t = i mod T (coalesced loads), and
//   h = sum_t key^(t+1) * sum_k w_{t+kT} (key^T)^k,
// each inner sum by Horner in K = key^T, then a block reduction.  Exact modular
// arithmetic, so the result is independent of T and bit-identical to the definition.
// NL = 2 hashes label_a and label_b together and writes ok[f] &= (h_a == h_b).
template <int NL>
__global__ void __launch_bounds__(256) k_frame_hash(const uint8_t *__restrict__ label_a,
                                                   const uint8_t *__restrict__ label_b, int32_t n,
                                                   unsigned long long key, unsigned long long *__restrict__ out_a,
                                                   unsigned long long *__restrict__ out_b,
                                                   const uint8_t *__restrict__ ok_in, uint8_t *__restrict__ ok_out) {
    const int f = blockIdx.x, T = blockDim.x, t = threadIdx.x;
    const int W = (n + 3) / 4;
    const bool aligned = (n & 3) == 0;
    const uint8_t *la = label_a + (size_t)f * n;
    const uint8_t *lb = NL == 2 ? label_b + (size_t)f * n : nullptr;
    const unsigned long long K = powmod61(key, (unsigned long long)T);
    unsigned long long ha = 0ull, hb = 0ull;
    const int kmax = t < W ? (W - 1 - t) / T : -1;
    for (int k = kmax; k >= 0; --k) {
        const int i = t + k * T;
        ha = addmod61(mulmod61(ha, K), label_word(la, n, i, aligned));
        if (NL == 2) hb = addmod61(mulmod61(hb, K), label_word(lb, n, i, aligned));
    }
    const unsigned long long kt = powmod61(key, (unsigned long long)(t + 1));
    __shared__ unsigned long long s[2][256];
    s[0][t] = mulmod61(ha, kt);
    if (NL == 2) s[1][t] = mulmod61(hb, kt);
    __syncthreads();
    for (int o = T / 2; o > 0; o >>= 1) {
        if (t < o) {
            s[0][t] = addmod61(s[0][t], s[0][t + o]);
            if (NL == 2) s[1][t] = addmod61(s[1][t], s[1][t + o]);
        }
        __syncthreads();
    }
    if (t == 0) {
        if (out_a) out_a[f] = s[0][0];
        if (NL == 2) {
            if (out_b) out_b[f] = s[1][0];
            ok_out[f] = (uint8_t)(ok_in[f] && s[0][0] == s[1][0]);
        }
    }
}

void launch_frame_hash(const uint8_t *label, int32_t F, int32_t n, unsigned long long key, unsigned long long *out,
                       cudaStream_t s) {
    k_frame_hash<1><<<F, 256, 0, s>>>(label, nullptr, n, key, out, nullptr, nullptr, nullptr);
}

void launch_verify(const uint8_t *label_a, const uint8_t *label_b, const uint8_t *ok_in, int32_t F, int32_t n,
                   unsigned long long key, uint8_t *ok_out, unsigned long long *ha, unsigned long long *hb,
                   cudaStream_t s) {
    k_frame_hash<2><<<F, 256, 0, s>>>(label_a, label_b, n, key, ha, hb, ok_in, ok_out);
}

}  // namespace cvsr
