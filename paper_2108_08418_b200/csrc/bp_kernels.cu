// Sum-product BP kernels for sm_100a.
//
// Layout ("frame-interleaved arena"): a tile holds T = 32 frames, one per warp
// lane.  For every edge slot (CSR position) the 32 frames' messages are 128
// contiguous bytes, so each warp-level access is one fully-used 128-byte line.
// Messages are stored IN PLACE: the CN pass reads V2C q_e and overwrites it
// with C2V r_e; the VN pass reads r_e and overwrites it with the next q_e.
// Arena values are in log2 units (LLR * log2 e): every exp/log below is then a
// single MUFU ex2/lg2, and the conversion happens once at the arena boundary
// (LLR load, trace dumps).  A warp processes one check (or variable) for TPW
// tiles at once, so each warp has TPW x degree independent 128-byte requests
// in flight.
//
// Algorithm (PAPER.md:189 BP decoder, PAPER.md:231 message passes; SURVEY.md
// §8(c) O5 readings A-8 flooding, A-10 V2C clamp, A-12 stopping rule):
//   CN: r_e = (1 - 2 s_c) * BOXPLUS_{e' != e} q_e'.  With t = tanh(|q|/2) the
//       magnitude is 2 atanh(P_e), P_e = prod_{e' != e} t_e'.  It is evaluated
//       through complements, which never cancel:
//         w = 1 - t = 2u / (1 + u),  u = e^-|q|
//         c_e = 1 - P_e = (+)_{e' != e} w_e',   a (+) b = a + b - ab  (prefix/suffix)
//         |r_e| = ln((1 + P_e) / (1 - P_e)) = ln((2 - c_e) / c_e)
//       (4 MUFU per edge; a zero message gives w = 1, c = 1, r = 0 exactly; a
//       degree-1 check gives c = 0, |r| = +inf -> Q_MAX, the empty-fold rule).
//       Sign = syndrome bit XOR the other edges' signs.
//   VN: post_v = L_v + sum_e r_e ; q_e = clamp(post_v - r_e, +-Q_MAX);
//       xhat_v = [post_v < 0].
//   The syndrome test H xhat = s of iteration k-1 is fused into CN pass k.
#include "common.cuh"
#include "kernels.cuh"

namespace cvsr {

constexpr unsigned FULL = 0xffffffffu;
constexpr int TPW = 4;  // tiles per warp

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

// q (log2 units) -> r (log2 units), in registers
template <int DC>
__device__ __forceinline__ void cn_update(float (&q)[DC], uint32_t sbit, float qmax2) {
    float w[DC];
    uint32_t par = sbit;
#pragma unroll
    for (int i = 0; i < DC; ++i) {
        const float u = ex2f(-fabsf(q[i]));
        w[i] = 2.0f * u * rcpf(1.0f + u);
        par ^= sgnbit(q[i]);
    }
    float pre[DC];
    pre[0] = 0.0f;
#pragma unroll
    for (int i = 1; i < DC; ++i) pre[i] = cplus(pre[i - 1], w[i - 1]);
    float suf = 0.0f;
#pragma unroll
    for (int i = DC - 1; i >= 0; --i) {
        const float c = cplus(pre[i], suf);
        const float mag = fmaxf(fminf(lg2f((2.0f - c) * rcpf(c)), qmax2), 0.0f);
        suf = cplus(suf, w[i]);
        q[i] = (par ^ sgnbit(q[i])) ? -mag : mag;
    }
}

struct TileSet {
    int t[TPW];
    uint32_t act[TPW];
};

__device__ __forceinline__ TileSet load_tiles(const DecState &ds, int g) {
    TileSet ts;
    const int cnt = ds.counts[0];
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
        const int idx = g * TPW + i;
        const bool valid = idx < cnt;
        ts.t[i] = valid ? ds.active_list[idx] : 0;
        ts.act[i] = valid ? ds.tile_active[ts.t[i]] : 0u;
    }
    return ts;
}

template <int DC>
__device__ __forceinline__ void cn_tiles(const CodeDev &cd, const DecState &ds, const TileSet &ts, int beg,
                                         const uint32_t (&s)[TPW], int lane, float qmax2) {
    float q[TPW][DC];
    float *base[TPW];
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
        base[i] = ds.msg + ((size_t)ts.t[i] * cd.E + beg) * T + lane;
        const bool a = (ts.act[i] >> lane) & 1u;
#pragma unroll
        for (int k = 0; k < DC; ++k) q[i][k] = a ? base[i][(size_t)k * T] : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
        if (!((ts.act[i] >> lane) & 1u)) continue;
        cn_update<DC>(q[i], (s[i] >> lane) & 1u, qmax2);
#pragma unroll
        for (int k = 0; k < DC; ++k) base[i][(size_t)k * T] = q[i][k];
    }
}

// any degree up to MAX_DC (checks above 12 are rare: none in the shipped ensembles);
// w and suffix complements live in thread-local arrays.
__device__ __noinline__ void cn_tiles_generic(const CodeDev cd, const DecState ds, const TileSet ts, int beg,
                                              int deg, const uint32_t *s, int lane, float qmax2) {
    float wl[MAX_DC], sf[MAX_DC + 1];
    uint32_t sg[MAX_DC / 32];
    for (int i = 0; i < TPW; ++i) {
        if (!((ts.act[i] >> lane) & 1u)) continue;
        float *m = ds.msg + ((size_t)ts.t[i] * cd.E + beg) * T + lane;
        uint32_t par = (s[i] >> lane) & 1u;
        for (int k = 0; k < MAX_DC / 32; ++k) sg[k] = 0u;
        for (int k = 0; k < deg; ++k) {
            const float qk = m[(size_t)k * T];
            const uint32_t b = sgnbit(qk);
            par ^= b;
            sg[k >> 5] |= b << (k & 31);
            const float u = ex2f(-fabsf(qk));
            wl[k] = 2.0f * u * rcpf(1.0f + u);
        }
        sf[deg] = 0.0f;
        for (int k = deg - 1; k >= 0; --k) sf[k] = cplus(sf[k + 1], wl[k]);
        float pre = 0.0f;
        for (int k = 0; k < deg; ++k) {
            const float c = cplus(pre, sf[k + 1]);
            const float mag = fmaxf(fminf(lg2f((2.0f - c) * rcpf(c)), qmax2), 0.0f);
            m[(size_t)k * T] = (((sg[k >> 5] >> (k & 31)) & 1u) ^ par) ? -mag : mag;
            pre = cplus(pre, wl[k]);
        }
    }
}

__global__ void __launch_bounds__(BLOCK, 3) k_cn(CodeDev cd, DecState ds, float qmax2, int check_only) {
    const int g = blockIdx.y;
    if (g * TPW >= ds.counts[0]) return;
    const TileSet ts = load_tiles(ds, g);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * WARPS_PER_BLOCK + warp;
    __shared__ uint32_t s_unsat[TPW];
    if (threadIdx.x < TPW) s_unsat[threadIdx.x] = 0u;
    __syncthreads();
    int beg = 0, deg = 0;
    uint32_t s[TPW];
    if (c < cd.M) {
        beg = cd.row_ptr[c];
        deg = cd.row_ptr[c + 1] - beg;
        // fused syndrome test of decision k-1: lanes split the row's edges
        uint32_t w[TPW];
#pragma unroll
        for (int i = 0; i < TPW; ++i) w[i] = 0u;
        for (int i0 = 0; i0 < deg; i0 += 32) {
            const int e = i0 + lane;
            const int v = (e < deg) ? cd.col_idx[beg + e] : 0;
#pragma unroll
            for (int i = 0; i < TPW; ++i)
                if (e < deg && ts.act[i]) w[i] ^= ds.hb[(size_t)ts.t[i] * cd.n + v];
        }
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
            s[i] = ts.act[i] ? ds.st[(size_t)ts.t[i] * cd.M + c] : 0u;
            const uint32_t u = (s[i] ^ __reduce_xor_sync(FULL, w[i])) & ts.act[i];
            if (lane == 0 && u) atomicOr(&s_unsat[i], u);
        }
    }
    __syncthreads();
    if (threadIdx.x < TPW && s_unsat[threadIdx.x]) atomicOr(&ds.tile_unsat[ts.t[threadIdx.x]], s_unsat[threadIdx.x]);
    if (check_only || c >= cd.M) return;
    switch (deg) {
        case 1: cn_tiles<1>(cd, ds, ts, beg, s, lane, qmax2); break;
        case 2: cn_tiles<2>(cd, ds, ts, beg, s, lane, qmax2); break;
        case 3: cn_tiles<3>(cd, ds, ts, beg, s, lane, qmax2); break;
        case 4: cn_tiles<4>(cd, ds, ts, beg, s, lane, qmax2); break;
        case 5: cn_tiles<5>(cd, ds, ts, beg, s, lane, qmax2); break;
        case 6: cn_tiles<6>(cd, ds, ts, beg, s, lane, qmax2); break;
        case 7: cn_tiles<7>(cd, ds, ts, beg, s, lane, qmax2); break;
        case 8: cn_tiles<8>(cd, ds, ts, beg, s, lane, qmax2); break;
        case 9: cn_tiles<9>(cd, ds, ts, beg, s, lane, qmax2); break;
        case 10: cn_tiles<10>(cd, ds, ts, beg, s, lane, qmax2); break;
        default: cn_tiles_generic(cd, ds, ts, beg, deg, s, lane, qmax2); break;
    }
}

template <int DV, bool FIRST>
__device__ __forceinline__ void vn_tiles(const CodeDev &cd, const DecState &ds, const TileSet &ts, int v, int sl,
                                         int lane, float qmax2, float *post_dbg) {
    int slot[DV > 0 ? DV : 1];
#pragma unroll
    for (int k = 0; k < DV; ++k) slot[k] = __shfl_sync(FULL, sl, k);
    float Lv[TPW];
    float r[TPW][DV > 0 ? DV : 1];
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
        const bool a = (ts.act[i] >> lane) & 1u;
        Lv[i] = a ? ds.L[((size_t)ts.t[i] * cd.n + v) * T + lane] : 0.0f;
        if (!FIRST) {
            const float *mt = ds.msg + (size_t)ts.t[i] * cd.E * T + lane;
#pragma unroll
            for (int k = 0; k < DV; ++k) r[i][k] = a ? mt[(size_t)slot[k] * T] : 0.0f;
        }
    }
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
        const bool a = (ts.act[i] >> lane) & 1u;
        float post = Lv[i];
        if (!FIRST) {
#pragma unroll
            for (int k = 0; k < DV; ++k) post += r[i][k];
        }
        if (a) {
            float *mt = ds.msg + (size_t)ts.t[i] * cd.E * T + lane;
#pragma unroll
            for (int k = 0; k < DV; ++k)
                mt[(size_t)slot[k] * T] = fminf(fmaxf(FIRST ? post : post - r[i][k], -qmax2), qmax2);
            if (post_dbg) post_dbg[((size_t)ts.t[i] * cd.n + v) * T + lane] = post;
        }
        const uint32_t word = __ballot_sync(FULL, a && post < 0.0f);
        if (lane == 0 && ts.act[i]) {
            uint32_t *h = ds.hb + (size_t)ts.t[i] * cd.n + v;
            *h = FIRST ? (word & ts.act[i]) : ((word & ts.act[i]) | (*h & ~ts.act[i]));
        }
    }
}

template <bool FIRST>
__device__ __noinline__ void vn_tiles_generic(const CodeDev cd, const DecState ds, const TileSet ts, int v,
                                              int beg, int deg, int lane, float qmax2, float *post_dbg) {
    const int32_t *slots = cd.csc_slot + beg;
    for (int i = 0; i < TPW; ++i) {
        const bool a = (ts.act[i] >> lane) & 1u;
        float *mt = ds.msg + (size_t)ts.t[i] * cd.E * T + lane;
        float post = a ? ds.L[((size_t)ts.t[i] * cd.n + v) * T + lane] : 0.0f;
        if (a) {
            if (!FIRST)
                for (int k = 0; k < deg; ++k) post += mt[(size_t)slots[k] * T];
            for (int k = 0; k < deg; ++k) {
                float *p = mt + (size_t)slots[k] * T;
                *p = fminf(fmaxf(FIRST ? post : post - *p, -qmax2), qmax2);
            }
            if (post_dbg) post_dbg[((size_t)ts.t[i] * cd.n + v) * T + lane] = post;
        }
        const uint32_t word = __ballot_sync(FULL, a && post < 0.0f);
        if (lane == 0 && ts.act[i]) {
            uint32_t *h = ds.hb + (size_t)ts.t[i] * cd.n + v;
            *h = FIRST ? (word & ts.act[i]) : ((word & ts.act[i]) | (*h & ~ts.act[i]));
        }
    }
}

template <bool FIRST>
__global__ void __launch_bounds__(BLOCK, 3) k_vn(CodeDev cd, DecState ds, float qmax2, float *post_dbg) {
    const int g = blockIdx.y;
    if (g * TPW >= ds.counts[0]) return;
    const TileSet ts = load_tiles(ds, g);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int v = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (v >= cd.n) return;
    const int beg = cd.col_ptr[v];
    const int deg = cd.col_ptr[v + 1] - beg;
    const int sl = (lane < deg) ? cd.csc_slot[beg + lane] : 0;
    switch (deg) {
        case 0: vn_tiles<0, FIRST>(cd, ds, ts, v, sl, lane, qmax2, post_dbg); break;
        case 1: vn_tiles<1, FIRST>(cd, ds, ts, v, sl, lane, qmax2, post_dbg); break;
        case 2: vn_tiles<2, FIRST>(cd, ds, ts, v, sl, lane, qmax2, post_dbg); break;
        case 3: vn_tiles<3, FIRST>(cd, ds, ts, v, sl, lane, qmax2, post_dbg); break;
        case 4: vn_tiles<4, FIRST>(cd, ds, ts, v, sl, lane, qmax2, post_dbg); break;
        case 5: vn_tiles<5, FIRST>(cd, ds, ts, v, sl, lane, qmax2, post_dbg); break;
        case 6: vn_tiles<6, FIRST>(cd, ds, ts, v, sl, lane, qmax2, post_dbg); break;
        case 7: vn_tiles<7, FIRST>(cd, ds, ts, v, sl, lane, qmax2, post_dbg); break;
        case 8: vn_tiles<8, FIRST>(cd, ds, ts, v, sl, lane, qmax2, post_dbg); break;
        default: vn_tiles_generic<FIRST>(cd, ds, ts, v, beg, deg, lane, qmax2, post_dbg); break;
    }
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
__global__ void k_to_interleaved(const float *__restrict__ src, float *__restrict__ dst, int32_t F, int64_t rows,
                                 float scale) {
    __shared__ float sm[32][33];
    const int t = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int fl = ty; fl < 32; fl += 8) {
        const int f = t * T + fl;
        const int64_t r = r0 + tx;
        sm[fl][tx] = (f < F && r < rows) ? src[(size_t)f * rows + r] * scale : 0.0f;
    }
    __syncthreads();
    for (int rl = ty; rl < 32; rl += 8) {
        const int64_t r = r0 + rl;
        if (r < rows) dst[((size_t)t * rows + r) * T + tx] = sm[tx][rl];
    }
}

// interleaved [tiles][rows][T] -> natural [F][rows]
__global__ void k_from_interleaved(const float *__restrict__ src, float *__restrict__ dst, int32_t F, int64_t rows,
                                   float scale) {
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
        if (f < F && r < rows) dst[(size_t)f * rows + r] = sm[tx][fl] * scale;
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

// qmax is in natural LLR units; the arena works in log2 units
void launch_cn(const CodeDev &cd, const DecState &ds, int grid_tiles, float qmax, int check_only, cudaStream_t s) {
    if (grid_tiles <= 0) return;
    dim3 grid((cd.M + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, (grid_tiles + TPW - 1) / TPW);
    k_cn<<<grid, BLOCK, 0, s>>>(cd, ds, qmax * LOG2E, check_only);
}

void launch_vn(const CodeDev &cd, const DecState &ds, int grid_tiles, float qmax, bool first, float *post_dbg,
               cudaStream_t s) {
    if (grid_tiles <= 0) return;
    dim3 grid((cd.n + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, (grid_tiles + TPW - 1) / TPW);
    if (first) k_vn<true><<<grid, BLOCK, 0, s>>>(cd, ds, qmax * LOG2E, post_dbg);
    else k_vn<false><<<grid, BLOCK, 0, s>>>(cd, ds, qmax * LOG2E, post_dbg);
}

void launch_status(const DecState &ds, int k, int max_iter, int final_pass, int32_t *host_counts, cudaStream_t s) {
    k_status<<<1, 1024, 0, s>>>(ds, k, max_iter, final_pass, host_counts);
}

void launch_retire(const DecState &ds, int32_t n, int grid_tiles, uint32_t *bits_out, cudaStream_t s) {
    if (grid_tiles <= 0) return;
    dim3 grid((words_of(n) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, grid_tiles);
    k_retire<<<grid, BLOCK, 0, s>>>(ds, n, bits_out);
}

void launch_to_interleaved(const float *src, float *dst, int32_t F, int64_t rows, int tiles, float scale,
                           cudaStream_t s) {
    dim3 grid((unsigned)((rows + 31) / 32), tiles);
    k_to_interleaved<<<grid, 256, 0, s>>>(src, dst, F, rows, scale);
}

void launch_from_interleaved(const float *src, float *dst, int32_t F, int64_t rows, int tiles, float scale,
                             cudaStream_t s) {
    dim3 grid((unsigned)((rows + 31) / 32), tiles);
    k_from_interleaved<<<grid, 256, 0, s>>>(src, dst, F, rows, scale);
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
