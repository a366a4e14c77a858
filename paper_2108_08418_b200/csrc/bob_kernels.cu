// Bob-side kernels (quantise, slice bits, syndrome) and reconcile bookkeeping.
#include <stdlib.h>

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

// bit j of each byte of x, as a nibble (byte 0 -> bit 0): the four bits land in
// bits 28..31 of the product without carries (movemask by multiplication)
__device__ __forceinline__ uint32_t byte_bits(uint32_t x, int j) {
    return (((x >> j) & 0x01010101u) * 0x10204080u) >> 28;
}

// S_j packed: thread per (frame, 32-var word); 32 label bytes in, one word out
__global__ void __launch_bounds__(BLOCK) k_slice_bits(const uint8_t *__restrict__ label, int32_t F, int32_t n,
                                                       int32_t j, uint32_t *__restrict__ bits) {
    const int Wn = words_of(n);
    const int64_t total = (int64_t)F * Wn;
    const bool vec = (n & 31) == 0 && (reinterpret_cast<uintptr_t>(label) & 15) == 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = i / Wn;
        const int w = (int)(i - f * Wn);
        const uint8_t *lab = label + (size_t)f * n + (size_t)w * 32;
        uint32_t word = 0u;
        if (vec) {
            const uint4 a = __ldg(reinterpret_cast<const uint4 *>(lab));
            const uint4 b = __ldg(reinterpret_cast<const uint4 *>(lab) + 1);
            const uint32_t x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int k = 0; k < 8; ++k) word |= byte_bits(x[k], j) << (4 * k);
        } else {
            const int cnt = min(32, n - w * 32);
            for (int k = 0; k < cnt; ++k) word |= (uint32_t)((lab[k] >> j) & 1u) << k;
        }
        bits[i] = word;
    }
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

// Same, FB frames per block: their packed rows are staged in shared memory and each
// check's column indices are read once for all FB frames (the code structure is the
// same for every frame, so per-frame re-reads of col_idx were the dominant traffic).
template <int FB>
__global__ void __launch_bounds__(BLOCK) k_syndrome_bits_smem(CodeDev cd, const uint32_t *__restrict__ bits,
                                                               int32_t F, uint32_t *__restrict__ synd) {
    extern __shared__ uint32_t srow[];  // [FB][Wn]
    const int Wm = words_of(cd.M), Wn = words_of(cd.n);
    const int f0 = blockIdx.x * FB;
    const int nf = min(FB, F - f0);
    for (int i = threadIdx.x; i < FB * Wn; i += blockDim.x) {
        const int k = i / Wn;
        srow[i] = k < nf ? bits[(size_t)(f0 + k) * Wn + (i - k * Wn)] : 0u;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int w = threadIdx.x >> 5; w < Wm; w += WARPS_PER_BLOCK) {
        const int c = w * 32 + lane;
        uint32_t par[FB];
#pragma unroll
        for (int k = 0; k < FB; ++k) par[k] = 0u;
        if (c < cd.M) {
            const int beg = cd.row_ptr[c], end = cd.row_ptr[c + 1];
            for (int e = beg; e < end; ++e) {
                const int v = cd.col_idx[e];
#pragma unroll
                for (int k = 0; k < FB; ++k) par[k] ^= srow[k * Wn + (v >> 5)] >> (v & 31);
            }
        }
#pragma unroll
        for (int k = 0; k < FB; ++k) {
            const uint32_t word = __ballot_sync(FULLB, par[k] & 1u);
            if (lane == 0 && k < nf) synd[(size_t)(f0 + k) * Wm + w] = word;
        }
    }
}

// Bit-sliced syndrome (default for cvsr_syndrome): the packed rows [F][Wn] are transposed to
// sl[v][g] = bits of variable v for frames 32 g .. 32 g + 31 (G4 words per variable, a multiple of
// 4), then a warp takes 32 consecutive checks (lane = check) and 4 frame groups: per edge one
// 16-byte gather of the variable's 128 frames' bits instead of one 32-byte sector per frame, and
// the column indices are read once per 128 frames.  A 32 x 32 bit transpose turns the checks'
// parity words back into the frames' syndrome words.  Same XOR as k_syndrome_bits: bit-exact.
__global__ void __launch_bounds__(256) k_bits_to_sliced(const uint32_t *__restrict__ bits, int32_t F, int32_t n,
                                                        int32_t G4, uint32_t *__restrict__ sl) {
    __shared__ uint32_t sm[32][33];
    const int Wn = words_of(n);
    const int w0 = blockIdx.x * 32, g = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = warp; r < 32; r += 8) {
        const int f = g * 32 + r, w = w0 + lane;
        sm[r][lane] = (f < F && w < Wn) ? bits[(size_t)f * Wn + w] : 0u;
    }
    __syncthreads();
    for (int c = warp; c < 32; c += 8) {
        const int w = w0 + c;
        if (w >= Wn) break;  // warp-uniform
        const uint32_t y = transpose32(sm[lane][c], lane);  // lane i: variable 32 w + i, bit r = frame 32 g + r
        const int v = w * 32 + lane;
        if (v < n) sl[(size_t)v * G4 + g] = y;
    }
}

__global__ void __launch_bounds__(BLOCK) k_syndrome_sliced(CodeDev cd, const uint32_t *__restrict__ sl, int32_t G4,
                                                           int32_t F, uint32_t *__restrict__ synd) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Wm = words_of(cd.M);
    const int w = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (w >= Wm) return;  // warp-uniform
    const int q = blockIdx.y;  // frame groups 4 q .. 4 q + 3
    const int c = w * 32 + lane;
    uint4 par = make_uint4(0u, 0u, 0u, 0u);
    if (c < cd.M) {
        const int beg = cd.row_ptr[c], end = cd.row_ptr[c + 1];
#pragma unroll 4
        for (int e = beg; e < end; ++e) {
            const uint4 b = __ldg(reinterpret_cast<const uint4 *>(sl + (size_t)cd.col_idx[e] * G4) + q);
            par.x ^= b.x;
            par.y ^= b.y;
            par.z ^= b.z;
            par.w ^= b.w;
        }
    }
    const uint32_t pw[4] = {par.x, par.y, par.z, par.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t y = transpose32(pw[k], lane);  // lane f: bit i = parity of check 32 w + i, frame 32 g + f
        const int f = (4 * q + k) * 32 + lane;
        if (f < F) synd[(size_t)f * Wm + w] = y;
    }
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

// bit k of w spread to byte k of the result for k = 0..3 (inverse of byte_bits)
__device__ __forceinline__ uint32_t spread_nibble(uint32_t nib) {
    return (nib * 0x00204081u) & 0x01010101u;
}

// thread per (frame, 32-symbol word): m packed words in, 32 label bytes out
__global__ void __launch_bounds__(256) k_assemble(BitPtrs bits, int32_t m, const uint8_t *__restrict__ attempt,
                                                  int32_t F, int32_t n, uint8_t *__restrict__ label_out) {
    const int Wn = words_of(n);
    const int64_t total = (int64_t)F * Wn;
    const bool vec = (n & 31) == 0 && (reinterpret_cast<uintptr_t>(label_out) & 15) == 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = i / Wn;
        const int w = (int)(i - f * Wn);
        const uint32_t am = attempt[f];
        uint32_t out[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        for (int j = 0; j < m; ++j) {
            if (!((am >> j) & 1u)) continue;
            const uint32_t word = bits.p[j][i];
#pragma unroll
            for (int k = 0; k < 8; ++k) out[k] |= spread_nibble((word >> (4 * k)) & 0xFu) << j;
        }
        uint8_t *dst = label_out + (size_t)f * n + (size_t)w * 32;
        if (vec) {
            reinterpret_cast<uint4 *>(dst)[0] = make_uint4(out[0], out[1], out[2], out[3]);
            reinterpret_cast<uint4 *>(dst)[1] = make_uint4(out[4], out[5], out[6], out[7]);
        } else {
            const int cnt = min(32, n - w * 32);
            for (int k = 0; k < cnt; ++k) dst[k] = (uint8_t)(out[k >> 2] >> (8 * (k & 3)));
        }
    }
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
    k_slice_bits<<<grid_for((int64_t)F * words_of(n), BLOCK), BLOCK, 0, s>>>(label, F, n, j, bits);
}

void launch_syndrome(const CodeDev &cd, const uint8_t *label, int32_t F, int32_t j, uint32_t *synd, cudaStream_t s) {
    dim3 grid((words_of(cd.M) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, F);
    k_syndrome<<<grid, BLOCK, 0, s>>>(cd, label, j, synd);
}

int32_t syndrome_sliced_groups(int32_t F) { return ((words_of(F) + 3) / 4) * 4; }

static bool syndrome_sliced_enabled() {
    static const int v = [] {
        const char *e = getenv("CVSR_SYND_SLICED");
        return (e && *e) ? atoi(e) : 1;
    }();
    return v != 0;
}

int launch_syndrome_bits(const CodeDev &cd, const uint32_t *bits, int32_t F, uint32_t *synd, uint32_t *sliced,
                         cudaStream_t s) {
    if (sliced && syndrome_sliced_enabled()) {
        const int32_t G4 = syndrome_sliced_groups(F);
        // every group including the padding ones (frames >= F are written as zeros)
        k_bits_to_sliced<<<dim3((words_of(cd.n) + 31) / 32, G4), 256, 0, s>>>(bits, F, cd.n, G4, sliced);
        k_syndrome_sliced<<<dim3((words_of(cd.M) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, G4 / 4), BLOCK, 0, s>>>(
            cd, sliced, G4, F, synd);
        return 2;
    }
    // stage FB frames' rows in shared memory when they fit (<= 96 KB per block) and the
    // batch still fills the GPU with blocks; otherwise the per-frame kernel
    const size_t row = (size_t)words_of(cd.n) * 4;
    auto smem_launch = [&](auto kern, int fb) {
        const size_t bytes = row * fb;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        kern<<<(F + fb - 1) / fb, BLOCK, bytes, s>>>(cd, bits, F, synd);
    };
    if (row * 8 <= 96 * 1024 && F >= 8 * 148) smem_launch(k_syndrome_bits_smem<8>, 8);
    else if (row * 4 <= 96 * 1024 && F >= 4 * 148) smem_launch(k_syndrome_bits_smem<4>, 4);
    else if (row * 2 <= 96 * 1024 && F >= 2 * 148) smem_launch(k_syndrome_bits_smem<2>, 2);
    else {
        dim3 grid((words_of(cd.M) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, F);
        k_syndrome_bits<<<grid, BLOCK, 0, s>>>(cd, bits, synd);
    }
    return 1;
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
    k_assemble<<<grid_for((int64_t)F * words_of(n), 256), 256, 0, s>>>(bp, m, attempt, F, n, label_out);
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
// NL = 2 hashes label_a and label_b together; NK independent keys (hash h[f][k] per key);
// ok[f] &= (h_a == h_b for every key).
struct HashKeys {
    unsigned long long k[CVSR_HASH_KEYS];
};

// One block per frame, FH_T threads: thread t runs Horner over its words i = t + k T with K = key^T
// (6 independent chains for 2 labels x 3 keys), so h_t = sum_k w_{t+kT} key^{kT}; the block sums
// h_t key^{t+1} = sum_i w_i key^{i+1} (independent of T).  1024 threads: the chains are
// latency-bound 64-bit multiplies: with fewer frames than 2 blocks per SM and long frames (C4: 125
// frames of 250k words) 1024 threads per block (hash check 0.63 -> 0.38 ms per step); otherwise
// 256, since each thread's powers of the keys cost about as much as 16 words (C2: 0.39 vs 0.68 ms).
constexpr int FH_T = 1024;
static int frame_hash_threads(int32_t F, int32_t n) {
    return (F < 2 * 148 && (n + 3) / 4 >= 64 * FH_T) ? FH_T : 256;
}
template <int NL, int NK>
__global__ void __launch_bounds__(FH_T) k_frame_hash(const uint8_t *__restrict__ label_a,
                                                    const uint8_t *__restrict__ label_b, int32_t n, HashKeys keys,
                                                    unsigned long long *__restrict__ out_a,
                                                    unsigned long long *__restrict__ out_b,
                                                    const uint8_t *__restrict__ ok_in, uint8_t *__restrict__ ok_out) {
    const int f = blockIdx.x, T = blockDim.x, t = threadIdx.x;
    const int W = (n + 3) / 4;
    const bool aligned = (n & 3) == 0;
    const uint8_t *la = label_a + (size_t)f * n;
    const uint8_t *lb = NL == 2 ? label_b + (size_t)f * n : nullptr;
    unsigned long long K[NK], h[NL][NK];
#pragma unroll
    for (int q = 0; q < NK; ++q) {
        K[q] = powmod61(keys.k[q], (unsigned long long)T);
        h[0][q] = 0ull;
        if (NL == 2) h[NL - 1][q] = 0ull;
    }
    const int kmax = t < W ? (W - 1 - t) / T : -1;
    for (int k = kmax; k >= 0; --k) {
        const int i = t + k * T;
        const uint32_t wa = label_word(la, n, i, aligned);
        const uint32_t wb = NL == 2 ? label_word(lb, n, i, aligned) : 0u;
#pragma unroll
        for (int q = 0; q < NK; ++q) {
            h[0][q] = addmod61(mulmod61(h[0][q], K[q]), wa);
            if (NL == 2) h[NL - 1][q] = addmod61(mulmod61(h[NL - 1][q], K[q]), wb);
        }
    }
    // h_t key^{t+1}, summed over the warp by shuffles, then over the warps
    __shared__ unsigned long long sw[NL * NK][FH_T / 32];
    const int lane = t & 31, warp = t >> 5;
#pragma unroll
    for (int q = 0; q < NK; ++q) {
        const unsigned long long kt = powmod61(keys.k[q], (unsigned long long)(t + 1));
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            unsigned long long v = mulmod61(h[l][q], kt);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = addmod61(v, __shfl_xor_sync(0xffffffffu, v, o));
            if (lane == 0) sw[l * NK + q][warp] = v;
        }
    }
    __syncthreads();
    if (warp == 0) {
        const int nw = T / 32;
        unsigned long long tot[NL * NK];
#pragma unroll
        for (int r = 0; r < NL * NK; ++r) {
            unsigned long long v = lane < nw ? sw[r][lane] : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = addmod61(v, __shfl_xor_sync(0xffffffffu, v, o));
            tot[r] = v;
        }
        if (lane == 0) {
            bool eq = true;
#pragma unroll
            for (int q = 0; q < NK; ++q) {
                if (out_a) out_a[(size_t)f * NK + q] = tot[q];
                if (NL == 2) {
                    if (out_b) out_b[(size_t)f * NK + q] = tot[NK + q];
                    eq = eq && tot[q] == tot[NK + q];
                }
            }
            if (NL == 2) ok_out[f] = (uint8_t)(ok_in[f] && eq);
        }
    }
}

void launch_frame_hash(const uint8_t *label, int32_t F, int32_t n, unsigned long long key, unsigned long long *out,
                       cudaStream_t s) {
    HashKeys k{};
    k.k[0] = key;
    k_frame_hash<1, 1><<<F, frame_hash_threads(F, n), 0, s>>>(label, nullptr, n, k, out, nullptr, nullptr, nullptr);
}

void launch_verify(const uint8_t *label_a, const uint8_t *label_b, const uint8_t *ok_in, int32_t F, int32_t n,
                   const unsigned long long *keys, uint8_t *ok_out, unsigned long long *ha, unsigned long long *hb,
                   cudaStream_t s) {
    HashKeys k{};
    for (int q = 0; q < CVSR_HASH_KEYS; ++q) k.k[q] = keys[q];
    k_frame_hash<2, CVSR_HASH_KEYS><<<F, frame_hash_threads(F, n), 0, s>>>(label_a, label_b, n, k, ha, hb, ok_in,
                                                                            ok_out);
}

}  // namespace cvsr
