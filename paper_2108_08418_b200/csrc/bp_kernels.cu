// Sum-product BP kernels for sm_100a.
//
// Layout ("frame-interleaved arena"): a tile holds T = 32 frames, one per warp
// lane.  For every edge slot (CSR position) the 32 frames' messages are 128
// contiguous bytes, so each warp-level access is one fully-used 128-byte line.
// Messages are stored IN PLACE: the CN pass reads V2C q_e and overwrites it
// with C2V r_e; the VN pass reads r_e and overwrites it with the next q_e.
//
// Algorithm (PAPER.md:189 BP decoder, PAPER.md:231 message passes; SURVEY.md
// §8(c) O5 readings A-8 flooding, A-10 V2C clamp, A-12 stopping rule):
//   CN: r_e = (1 - 2 s_c) * BOXPLUS_{e' != e} q_e'
//       evaluated in the phi domain, phi(x) = -ln tanh(x/2) (self-inverse):
//       |r_e| = phi( sum_{e' != e} phi(|q_e'|) ),  sign = prod of the other signs.
//       The extrinsic sum is formed without "total minus own" cancellation:
//       ext_e = S_ex                       for the edge of largest phi (argmax),
//             = (S_ex - phi_e) + phi_max   otherwise,
//       where S_ex = sum of all phi except the max (then ext_e >= S/2, so its
//       relative error stays O(d_c eps)).
//   VN: post_v = L_v + sum_e r_e ; q_e = clamp(post_v - r_e, +-Q_MAX);
//       xhat_v = [post_v < 0].
//   The syndrome test H xhat = s of iteration k-1 is fused into CN pass k.
#include "common.cuh"
#include "kernels.cuh"

namespace cvsr {

constexpr unsigned FULL = 0xffffffffu;
// phi is evaluated at max(x, PHI_XMIN) so that phi <= 60 stays finite
// (phi(2e^-60) = 60); an exact 0 message then yields |r| ~ 1e-26 on the
// other edges instead of exactly 0 (far inside the 1e-4 parity tolerance).
constexpr float PHI_XMIN = 1.7516230e-26f;

// phi(x) = ln((1 + e^-x) / (1 - e^-x)) for x > 0, cancellation-safe:
//  x >= 4      : 2 atanh(u) = 2u (1 + u^2/3 + u^4/5), u = e^-x   (no 1+tiny rounding)
//  x <  0.375  : 1 - e^-x from its Taylor series (no 1 - u cancellation)
__device__ __forceinline__ float phi_f(float x) {
    x = fmaxf(x, PHI_XMIN);
    const float u = __expf(-x);
    const float u2 = u * u;
    const float big = 2.0f * u * fmaf(u2, fmaf(u2, 0.2f, 0.33333334f), 1.0f);
    const float dp = x * fmaf(-x, fmaf(-x, fmaf(-x, fmaf(-x, fmaf(-x, 1.0f / 720.0f, 1.0f / 120.0f),
                                                        1.0f / 24.0f), 1.0f / 6.0f), 0.5f), 1.0f);
    const float d = (x < 0.375f) ? dp : (1.0f - u);
    const float small = __logf(__fdividef(1.0f + u, d));
    return (x >= 4.0f) ? big : small;
}

template <int DC>
__device__ __forceinline__ void cn_core(float *__restrict__ m, uint32_t sbit, float qmax) {
    float q[DC], ph[DC];
#pragma unroll
    for (int i = 0; i < DC; ++i) q[i] = m[(size_t)i * T];
    uint32_t par = sbit;
#pragma unroll
    for (int i = 0; i < DC; ++i) {
        ph[i] = phi_f(fabsf(q[i]));
        par ^= __float_as_uint(q[i]) >> 31;
    }
    float pmax = ph[0], sex = 0.0f;
    int amax = 0;
#pragma unroll
    for (int i = 1; i < DC; ++i) {
        sex += fminf(ph[i], pmax);
        amax = (ph[i] > pmax) ? i : amax;
        pmax = fmaxf(ph[i], pmax);
    }
#pragma unroll
    for (int i = 0; i < DC; ++i) {
        const float ext = (i == amax) ? sex : (sex - ph[i]) + pmax;
        const float mag = fminf(phi_f(ext), qmax);
        const uint32_t sg = par ^ (__float_as_uint(q[i]) >> 31);
        m[(size_t)i * T] = sg ? -mag : mag;
    }
}

// any degree: two passes, the second re-reads q (L1-resident) and recomputes phi
__device__ __noinline__ void cn_generic(float *__restrict__ m, int deg, uint32_t sbit, float qmax) {
    uint32_t par = sbit;
    float pmax = -1.0f, sex = 0.0f;
    int amax = 0;
    for (int i = 0; i < deg; ++i) {
        const float qi = m[(size_t)i * T];
        const float p = phi_f(fabsf(qi));
        par ^= __float_as_uint(qi) >> 31;
        if (i == 0) {
            pmax = p;
        } else {
            sex += fminf(p, pmax);
            amax = (p > pmax) ? i : amax;
            pmax = fmaxf(p, pmax);
        }
    }
    for (int i = 0; i < deg; ++i) {
        const float qi = m[(size_t)i * T];
        const float p = phi_f(fabsf(qi));
        const float ext = (i == amax) ? sex : (sex - p) + pmax;
        const float mag = fminf(phi_f(ext), qmax);
        const uint32_t sg = par ^ (__float_as_uint(qi) >> 31);
        m[(size_t)i * T] = sg ? -mag : mag;
    }
}

__global__ void __launch_bounds__(BLOCK) k_cn(CodeDev cd, DecState ds, float qmax, int check_only) {
    const int ti = blockIdx.y;
    if (ti >= ds.counts[0]) return;
    const int t = ds.active_list[ti];
    const uint32_t active = ds.tile_active[t];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * WARPS_PER_BLOCK + warp;
    __shared__ uint32_t s_unsat;
    if (threadIdx.x == 0) s_unsat = 0u;
    __syncthreads();
    int beg = 0, deg = 0;
    uint32_t s = 0u;
    if (c < cd.M) {
        beg = cd.row_ptr[c];
        deg = cd.row_ptr[c + 1] - beg;
        s = ds.st[(size_t)t * cd.M + c];
        // fused syndrome test of decision k-1: lanes split the row's edges
        const uint32_t *hbt = ds.hb + (size_t)t * cd.n;
        uint32_t w = 0u;
        for (int i0 = 0; i0 < deg; i0 += 32) {
            const int i = i0 + lane;
            w ^= (i < deg) ? hbt[cd.col_idx[beg + i]] : 0u;
        }
        const uint32_t p = s ^ __reduce_xor_sync(FULL, w);
        const uint32_t u = p & active;
        if (lane == 0 && u) atomicOr(&s_unsat, u);
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_unsat) atomicOr(&ds.tile_unsat[t], s_unsat);
    if (check_only || c >= cd.M || !((active >> lane) & 1u)) return;
    float *m = ds.msg + ((size_t)t * cd.E + beg) * T + lane;
    const uint32_t sbit = (s >> lane) & 1u;
    switch (deg) {
        case 1: cn_core<1>(m, sbit, qmax); break;
        case 2: cn_core<2>(m, sbit, qmax); break;
        case 3: cn_core<3>(m, sbit, qmax); break;
        case 4: cn_core<4>(m, sbit, qmax); break;
        case 5: cn_core<5>(m, sbit, qmax); break;
        case 6: cn_core<6>(m, sbit, qmax); break;
        case 7: cn_core<7>(m, sbit, qmax); break;
        case 8: cn_core<8>(m, sbit, qmax); break;
        case 9: cn_core<9>(m, sbit, qmax); break;
        case 10: cn_core<10>(m, sbit, qmax); break;
        case 11: cn_core<11>(m, sbit, qmax); break;
        case 12: cn_core<12>(m, sbit, qmax); break;
        default: cn_generic(m, deg, sbit, qmax); break;
    }
}

template <int DV, bool FIRST>
__device__ __forceinline__ float vn_core(float *__restrict__ mt, int sl, float Lv, float qmax, bool act) {
    if (FIRST) {
        const float q = fminf(fmaxf(Lv, -qmax), qmax);
#pragma unroll
        for (int i = 0; i < DV; ++i) {
            const int slot = __shfl_sync(FULL, sl, i);
            if (act) mt[(size_t)slot * T] = q;
        }
        return Lv;
    }
    int slot[DV];
    float r[DV];
#pragma unroll
    for (int i = 0; i < DV; ++i) slot[i] = __shfl_sync(FULL, sl, i);
    float post = Lv;
    if (act) {
#pragma unroll
        for (int i = 0; i < DV; ++i) r[i] = mt[(size_t)slot[i] * T];
#pragma unroll
        for (int i = 0; i < DV; ++i) post += r[i];
#pragma unroll
        for (int i = 0; i < DV; ++i) mt[(size_t)slot[i] * T] = fminf(fmaxf(post - r[i], -qmax), qmax);
    }
    return post;
}

template <bool FIRST>
__device__ __noinline__ float vn_generic(float *__restrict__ mt, const int32_t *__restrict__ slots, int deg,
                                         float Lv, float qmax, bool act) {
    float post = Lv;
    if (!act) return post;
    if (FIRST) {
        const float q = fminf(fmaxf(Lv, -qmax), qmax);
        for (int i = 0; i < deg; ++i) mt[(size_t)slots[i] * T] = q;
        return post;
    }
    for (int i = 0; i < deg; ++i) post += mt[(size_t)slots[i] * T];
    for (int i = 0; i < deg; ++i) {
        float *p = mt + (size_t)slots[i] * T;
        *p = fminf(fmaxf(post - *p, -qmax), qmax);
    }
    return post;
}

template <bool FIRST>
__global__ void __launch_bounds__(BLOCK) k_vn(CodeDev cd, DecState ds, float qmax, float *post_dbg) {
    const int ti = blockIdx.y;
    if (ti >= ds.counts[0]) return;
    const int t = ds.active_list[ti];
    const uint32_t active = ds.tile_active[t];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int v = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (v >= cd.n) return;
    const int beg = cd.col_ptr[v];
    const int deg = cd.col_ptr[v + 1] - beg;
    const bool act = (active >> lane) & 1u;
    const size_t lv = ((size_t)t * cd.n + v) * T + lane;
    const float Lv = ds.L[lv];
    float *mt = ds.msg + (size_t)t * cd.E * T + lane;
    const int sl = (lane < deg) ? cd.csc_slot[beg + lane] : 0;
    float post;
    switch (deg) {
        case 0: post = Lv; break;
        case 1: post = vn_core<1, FIRST>(mt, sl, Lv, qmax, act); break;
        case 2: post = vn_core<2, FIRST>(mt, sl, Lv, qmax, act); break;
        case 3: post = vn_core<3, FIRST>(mt, sl, Lv, qmax, act); break;
        case 4: post = vn_core<4, FIRST>(mt, sl, Lv, qmax, act); break;
        case 5: post = vn_core<5, FIRST>(mt, sl, Lv, qmax, act); break;
        case 6: post = vn_core<6, FIRST>(mt, sl, Lv, qmax, act); break;
        case 7: post = vn_core<7, FIRST>(mt, sl, Lv, qmax, act); break;
        case 8: post = vn_core<8, FIRST>(mt, sl, Lv, qmax, act); break;
        default: post = vn_generic<FIRST>(mt, cd.csc_slot + beg, deg, Lv, qmax, act); break;
    }
    const uint32_t word = __ballot_sync(FULL, act && post < 0.0f);
    if (lane == 0) {
        uint32_t *h = ds.hb + (size_t)t * cd.n + v;
        *h = FIRST ? (word & active) : ((word & active) | (*h & ~active));
    }
    if (post_dbg && act) post_dbg[lv] = post;
}

// Block-wide exclusive scan of 0/1 flags (blockDim.x multiple of 32, <= 1024).
__device__ __forceinline__ int block_scan_flag(bool flag, int *s_warp, int *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t b = __ballot_sync(FULL, flag);
    const int within = __popc(b & ((1u << lane) - 1u));
    if (lane == 0) s_warp[warp] = __popc(b);
    __syncthreads();
    if (warp == 0) {
        int x = (lane < nw) ? s_warp[lane] : 0;
        int incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane < nw) s_warp[lane] = incl - x;
        if (lane == 31) s_warp[32] = incl;
    }
    __syncthreads();
    const int r = s_warp[warp] + within;
    *total = s_warp[32];
    __syncthreads();
    return r;
}

// Convergence bookkeeping after CN pass k (which tested decision k-1).
// Single block; loops over tiles.  final_pass: k = max_iter + 1.
__global__ void __launch_bounds__(1024) k_status(DecState ds, int k, int max_iter, int final_pass,
                                                 int32_t *host_counts) {
    __shared__ int s_warp[33];
    __shared__ int s_lanes;
    if (threadIdx.x == 0) s_lanes = 0;
    __syncthreads();
    int n_act = 0, n_ret = 0, lanes = 0;
    for (int t0 = 0; t0 < ds.tiles; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        uint32_t rem = 0u, newly = 0u;
        if (t < ds.tiles) {
            const uint32_t a = ds.tile_active[t];
            const uint32_t u = ds.tile_unsat[t];
            if (a) {
                ds.tile_unsat[t] = 0u;
                const uint32_t done = a & ~u;
                rem = a & u;
                uint32_t d = done;
                while (d) {
                    const int l = __ffs(d) - 1;
                    d &= d - 1;
                    ds.iters[t * T + l] = k - 1;
                    ds.conv[t * T + l] = 1;
                }
                if (final_pass) {
                    uint32_t f = rem;
                    while (f) {
                        const int l = __ffs(f) - 1;
                        f &= f - 1;
                        ds.iters[t * T + l] = max_iter;
                        ds.conv[t * T + l] = 0;
                    }
                    newly = a;
                    rem = 0u;
                } else {
                    newly = done;
                }
                ds.tile_active[t] = rem;
            }
            ds.tile_newly[t] = newly;
        }
        int tot;
        const int pa = block_scan_flag(rem != 0u, s_warp, &tot);
        if (rem) ds.active_list[n_act + pa] = t;
        n_act += tot;
        const int pr = block_scan_flag(newly != 0u, s_warp, &tot);
        if (newly) ds.retire_list[n_ret + pr] = t;
        n_ret += tot;
        int v = __popc(rem);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if ((threadIdx.x & 31) == 0) atomicAdd(&s_lanes, v);
    }
    __syncthreads();
    lanes = s_lanes;
    if (threadIdx.x == 0) {
        ds.counts[0] = n_act;
        ds.counts[1] = n_ret;
        ds.counts[2] = lanes;
        if (host_counts) {
            volatile int32_t *h = host_counts;
            h[0] = n_act;
            h[1] = n_ret;
            h[2] = lanes;
        }
    }
}

// Write the hard decisions of retired lanes as packed bits (32x32 bit transpose by ballots).
__global__ void __launch_bounds__(BLOCK) k_retire(DecState ds, int32_t n, uint32_t *bits_out) {
    const int ti = blockIdx.y;
    if (ti >= ds.counts[1]) return;
    const int t = ds.retire_list[ti];
    const uint32_t newly = ds.tile_newly[t];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Wn = words_of(n);
    const int w = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (w >= Wn) return;
    const int v = w * 32 + lane;
    const uint32_t word = (v < n) ? ds.hb[(size_t)t * n + v] : 0u;
    uint32_t mine = 0u;
#pragma unroll
    for (int f = 0; f < 32; ++f) {
        const uint32_t b = __ballot_sync(FULL, (word >> f) & 1u);
        if (lane == f) mine = b;
    }
    const int frame = t * T + lane;
    if (((newly >> lane) & 1u) && frame < ds.frames) bits_out[(size_t)frame * Wn + w] = mine;
}

// natural [F][rows] -> interleaved [tiles][rows][T] (zero-fill missing frames)
__global__ void k_to_interleaved(const float *__restrict__ src, float *__restrict__ dst, int32_t F, int64_t rows) {
    __shared__ float sm[32][33];
    const int t = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int fl = ty; fl < 32; fl += 8) {
        const int f = t * T + fl;
        const int64_t r = r0 + tx;
        sm[fl][tx] = (f < F && r < rows) ? src[(size_t)f * rows + r] : 0.0f;
    }
    __syncthreads();
    for (int rl = ty; rl < 32; rl += 8) {
        const int64_t r = r0 + rl;
        if (r < rows) dst[((size_t)t * rows + r) * T + tx] = sm[tx][rl];
    }
}

// interleaved [tiles][rows][T] -> natural [F][rows]
__global__ void k_from_interleaved(const float *__restrict__ src, float *__restrict__ dst, int32_t F, int64_t rows) {
    __shared__ float sm[32][33];
    const int t = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int rl = ty; rl < 32; rl += 8) {
        const int64_t r = r0 + rl;
        sm[rl][tx] = (r < rows) ? src[((size_t)t * rows + r) * T + tx] : 0.0f;
    }
    __syncthreads();
    for (int fl = ty; fl < 32; fl += 8) {
        const int f = t * T + fl;
        const int64_t r = r0 + tx;
        if (f < F && r < rows) dst[(size_t)f * rows + r] = sm[tx][fl];
    }
}

// public syndrome [F][Wm] -> per-tile lane-bit words st[t][c]
__global__ void __launch_bounds__(BLOCK) k_synd_transpose(const uint32_t *__restrict__ synd, int32_t F, int32_t M,
                                                           uint32_t *__restrict__ st) {
    const int t = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Wm = words_of(M);
    const int w = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (w >= Wm) return;
    const int f = t * T + lane;
    const uint32_t word = (f < F) ? synd[(size_t)f * Wm + w] : 0u;
    uint32_t mine = 0u;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        const uint32_t b = __ballot_sync(FULL, (word >> k) & 1u);
        if (lane == k) mine = b;
    }
    const int c = w * 32 + lane;
    if (c < M) st[(size_t)t * M + c] = mine;
}

// initial tile state: active lanes = valid frames (& alive mask if given)
__global__ void k_init_tiles(DecState ds, const uint8_t *__restrict__ alive) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ds.tiles) return;
    uint32_t a = 0u;
    for (int l = 0; l < T; ++l) {
        const int f = t * T + l;
        if (f < ds.frames && (!alive || alive[f])) a |= 1u << l;
    }
    ds.tile_active[t] = a;
    ds.tile_unsat[t] = 0u;
    ds.tile_newly[t] = 0u;
    ds.active_list[t] = t;
}

__global__ void k_set_counts(DecState ds, int32_t n_active) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        ds.counts[0] = n_active;
        ds.counts[1] = 0;
        ds.counts[2] = 0;
    }
}

// ---------------------------------------------------------------- launchers

void launch_cn(const CodeDev &cd, const DecState &ds, int grid_tiles, float qmax, int check_only, cudaStream_t s) {
    if (grid_tiles <= 0) return;
    dim3 grid((cd.M + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, grid_tiles);
    k_cn<<<grid, BLOCK, 0, s>>>(cd, ds, qmax, check_only);
}

void launch_vn(const CodeDev &cd, const DecState &ds, int grid_tiles, float qmax, bool first, float *post_dbg,
               cudaStream_t s) {
    if (grid_tiles <= 0) return;
    dim3 grid((cd.n + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, grid_tiles);
    if (first) k_vn<true><<<grid, BLOCK, 0, s>>>(cd, ds, qmax, post_dbg);
    else k_vn<false><<<grid, BLOCK, 0, s>>>(cd, ds, qmax, post_dbg);
}

void launch_status(const DecState &ds, int k, int max_iter, int final_pass, int32_t *host_counts, cudaStream_t s) {
    k_status<<<1, 1024, 0, s>>>(ds, k, max_iter, final_pass, host_counts);
}

void launch_retire(const DecState &ds, int32_t n, int grid_tiles, uint32_t *bits_out, cudaStream_t s) {
    if (grid_tiles <= 0) return;
    dim3 grid((words_of(n) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, grid_tiles);
    k_retire<<<grid, BLOCK, 0, s>>>(ds, n, bits_out);
}

void launch_to_interleaved(const float *src, float *dst, int32_t F, int64_t rows, int tiles, cudaStream_t s) {
    dim3 grid((unsigned)((rows + 31) / 32), tiles);
    k_to_interleaved<<<grid, 256, 0, s>>>(src, dst, F, rows);
}

void launch_from_interleaved(const float *src, float *dst, int32_t F, int64_t rows, int tiles, cudaStream_t s) {
    dim3 grid((unsigned)((rows + 31) / 32), tiles);
    k_from_interleaved<<<grid, 256, 0, s>>>(src, dst, F, rows);
}

void launch_synd_transpose(const uint32_t *synd, int32_t F, int32_t M, uint32_t *st, int tiles, cudaStream_t s) {
    dim3 grid((words_of(M) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, tiles);
    k_synd_transpose<<<grid, BLOCK, 0, s>>>(synd, F, M, st);
}

void launch_init_tiles(const DecState &ds, const uint8_t *alive, cudaStream_t s) {
    k_init_tiles<<<(ds.tiles + 255) / 256, 256, 0, s>>>(ds, alive);
}

void launch_set_counts(const DecState &ds, int32_t n_active, cudaStream_t s) {
    k_set_counts<<<1, 32, 0, s>>>(ds, n_active);
}

}  // namespace cvsr
