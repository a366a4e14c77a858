// Row-layered BP schedule (reading R-9) for sm_100a.
#include <stdlib.h>

#include <algorithm>

#include "bp_device.cuh"
#include "common.cuh"
#include "kernels.cuh"
#include "vec.cuh"

namespace cvsr {

// ------------------------------------------------------------------ row-layered schedule
//
// Reading R-9 (PAPER.md:189 names sum-product BP without fixing its
// schedule): the checks are greedily coloured into layers that share no variable
// (cvsr_code_load) and one iteration updates the layers in order, each against
// the posteriors the previous layers left:
//     q_e = post_v - r_e,   r_e <- (1 - 2 s_c) BOXPLUS_{e' != e} clamp(q_e'),   post_v <- q_e + r_e.
// Arena use: ds.L holds the running posterior post_v (initialised to L_v), ds.msg
// holds r_e (initialised to 0), ds.hb the hard decisions [post_v < 0].  No VN pass:
// a layer kernel reads and writes one posterior line and one message line per
// edge (16 B per edge-frame per iteration, as flooding's CN + VN), but the
// schedule converges in about half the iterations (tools/layered_study.py).
// The syndrome test of an iteration is k_cn with check_only = 1.  Same CN
// arithmetic as k_cn (cn_lanes), so results differ from the oracle's fp64 only by
// rounding.

// hb = [L < 0] for the active frames; r = 0 is a memset by the caller
template <int S>
__global__ void __launch_bounds__(BLOCK) k_layer_init(CodeDev cd, DecState ds) {
    const int ti = blockIdx.y;
    if (ti >= ds.counts[0]) return;
    const int t = ds.active_list[ti];
    const uint4 act = ds.tile_active[t];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int v = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (v >= cd.n) return;
    const FV<S> p = ldv<S>(ds.L + (((size_t)t * cd.n + v) * LANES + lane) * S);
    uint32_t wd[SUBS] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int s = 0; s < S; ++s) wd[s] = __ballot_sync(FULL, p.c[s] < 0.0f) & cmpu(act, s);
    if (lane == 0) ds.hb[(size_t)t * cd.n + v] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
}

// one check of tile t: DC = code's maximum check degree (>= deg).  lo/deg/sbits describe the
// check; v(k) returns the variable of its k-th edge (indices were fetched by the caller).
template <int DC, int S, typename VarOf>
__device__ __forceinline__ void layer_check(const CodeDev &cd, const DecState &ds, int t, const uint4 &act, int lo,
                                            int deg, uint32_t sb, VarOf var_of, int lane, float qmax2) {
    if constexpr (DC >= 6) {
        // degree-2 checks in a code with a large maximum degree (MET-style type-A checks): a
        // 2-edge body instead of DC - 2 dummy edges (deg is warp-uniform)
        if (deg <= 2) {
            layer_check<2, S>(cd, ds, t, act, lo, deg, sb, var_of, lane, qmax2);
            return;
        }
    }
    const uint32_t al = lane_act<S>(act, lane);
    float *mt = ds.msg + ((size_t)t * cd.E + lo) * LANES * S + (size_t)lane * S;
    float *Lt = ds.L + (size_t)t * cd.n * LANES * S + (size_t)lane * S;
    int v[DC];
    FV<S> qu[DC], q[DC];
#pragma unroll
    for (int k = 0; k < DC; ++k) {
        v[k] = var_of(k);
        if (k < deg) {
            const FV<S> p = ldv<S>(Lt + (size_t)v[k] * LANES * S);
            const FV<S> r = ldv<S>(mt + (size_t)k * LANES * S);
#pragma unroll
            for (int s = 0; s < S; ++s) {
                qu[k].c[s] = p.c[s] - r.c[s];
                q[k].c[s] = clampf(qu[k].c[s], qmax2);
            }
        } else {
            q[k] = splat<S>(DUMMY_Q);
        }
    }
    cn_lanes<DC, S>(q, sb, al, qmax2);
#pragma unroll
    for (int k = 0; k < DC; ++k) {
        if (k < deg) {
            FV<S> p;
#pragma unroll
            for (int s = 0; s < S; ++s) p.c[s] = qu[k].c[s] + q[k].c[s];  // (retired frames' values are dead)
            uint32_t wd[SUBS] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int s = 0; s < S; ++s) wd[s] = __ballot_sync(FULL, p.c[s] < 0.0f) & cmpu(act, s);
            if (al) {
                stv<S>(mt + (size_t)k * LANES * S, q[k]);
                stv<S>(Lt + (size_t)v[k] * LANES * S, p);
            }
            if (lane == 0) ds.hb[(size_t)t * cd.n + v[k]] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
        }
    }
}

#ifndef CVSR_LAYER_MINB
#define CVSR_LAYER_MINB 4
#endif
#ifndef CVSR_LAYER_CPW
#define CVSR_LAYER_CPW 4
#endif
constexpr int LCPW = CVSR_LAYER_CPW;  // checks per warp in k_layer
// A warp takes CPW checks of the layer.  When CPW x DC <= 32 their check ids, row bounds and
// column indices are fetched up front with one load per lane (no dependent index loads per
// check); otherwise per check.
// Blocks per SM: the most that ptxas fits without spills (64 / 80 / 128 registers per thread
// for 4 / 3 / 2 blocks of 256 threads; -Xptxas -v of this build)
__host__ __device__ constexpr int layer_minb(int DC, int S) {
    return S == 1 ? (DC <= 7 ? CVSR_LAYER_MINB : (DC <= 10 ? 3 : 2))
                  : (S == 2 ? (DC <= 5 ? CVSR_LAYER_MINB : (DC <= 6 ? 3 : 2)) : (DC <= 3 ? 3 : 2));
}
template <int DC, int S>
__global__ void __launch_bounds__(BLOCK, layer_minb(DC, S)) k_layer(CodeDev cd, DecState ds, int lbeg, int lcnt,
                                                                    float qmax2) {
    const int ti = blockIdx.y;
    if (ti >= ds.counts[0]) return;
    const int t = ds.active_list[ti];
    const uint4 act = ds.tile_active[t];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = (blockIdx.x * WARPS_PER_BLOCK + warp) * LCPW;
    const int nc = min(LCPW, lcnt - i0);
    if (nc <= 0) return;
    const int myc = lane < nc ? cd.layer_chk[lbeg + i0 + lane] : 0;
    const int mylo = lane < nc ? cd.row_ptr[myc] : 0;
    const int myhi = lane < nc ? cd.row_ptr[myc + 1] : 0;
    const uint4 *stt = ds.st + (size_t)t * cd.M;
    if constexpr (LCPW * DC <= LANES) {
        const int ii = lane / DC, kk = lane - ii * DC;
        const int lo_ii = __shfl_sync(FULL, mylo, ii < LCPW ? ii : 0);
        const int hi_ii = __shfl_sync(FULL, myhi, ii < LCPW ? ii : 0);
        const int myv = (ii < nc && kk < hi_ii - lo_ii) ? cd.col_idx[lo_ii + kk] : 0;
#pragma unroll 1
        for (int i = 0; i < nc; ++i) {
            const int lo = __shfl_sync(FULL, mylo, i), deg = __shfl_sync(FULL, myhi, i) - lo;
            const int c = __shfl_sync(FULL, myc, i);
            const uint32_t sb = lane_act<S>(stt[lbeg + i0 + i], lane);  // rows in layer order
            layer_check<DC, S>(cd, ds, t, act, lo, deg, sb,
                               [&](int k) { return __shfl_sync(FULL, myv, i * DC + k); }, lane, qmax2);
        }
    } else {
#pragma unroll 1
        for (int i = 0; i < nc; ++i) {
            const int lo = __shfl_sync(FULL, mylo, i), deg = __shfl_sync(FULL, myhi, i) - lo;
            const int c = __shfl_sync(FULL, myc, i);
            const uint32_t sb = lane_act<S>(stt[lbeg + i0 + i], lane);  // rows in layer order
            const int myv = lane < deg ? cd.col_idx[lo + lane] : 0;
            layer_check<DC, S>(cd, ds, t, act, lo, deg, sb, [&](int k) { return __shfl_sync(FULL, myv, k); },
                               lane, qmax2);
        }
    }
}

// ------------------------------------------------------------------ TMA-staged layer kernel
//
// k_layer_tma<DC, S>: same check update and arena as k_layer, but the lines a check reads are
// staged in shared memory by bulk asynchronous copies (cp.async.bulk, the TMA engine's
// non-tensor path) instead of register loads, so the number of bytes in flight no longer
// depends on registers.  Each warp owns P (2-3) stages and walks LT_CH checks of the layer:
//   issue:   every lane copies its S frames of the posterior lines of the check's variables
//            (cp.async, 4 S bytes per lane and line, gathered; the stage's mbarrier tracks them),
//            lane 0 arms the mbarrier with the message bytes and copies the check's deg message
//            lines with one bulk copy (one contiguous span: CSR slots are contiguous);
//   compute: after the mbarrier phase completes, every lane reads its S frames of each line
//            from shared memory, runs the sum/difference CN update (cn_update) per frame and
//            writes r_e and post_v = q_e + r_e back into the stage, plus the hard decisions;
//   store:   lane-vectorised stores of the deg message lines and deg posterior lines;
//   refill:  the stage is re-armed with check i + P.
// (Measured against storing r_e / post_v straight from registers, which needs all S frames'
// q_e in registers and scalar stores: C4 95.6 vs 88.8 ms per step, C2 57.6 vs 51.6.)
// Checks of one layer share no variable, so prefetching the next checks' posterior lines while
// the current check is being written is exact.  The arithmetic is k_layer's operation for
// operation (results are bit-identical).
constexpr int LT_WARPS = 8;  // warps per block (k_layer_tmap, and k_layer_tma for S = 1)
// k_layer_tma: 4 warps per block at 4 frames per lane (512-byte lines: a warp's two stages take
// 14 KB at check degree 7, so 8-warp blocks would leave one block per SM) and at 2 frames per
// lane (CVSR_LT_WARPS2; the same warps per SM in smaller blocks shorten each layer's tail: C4
// 104.4 -> 102.9 ms, C2 42.7 -> 42.0 ms with 8 / 4 warps; 2 and 6 warps measured in between)
#ifndef CVSR_LT_WARPS2
#define CVSR_LT_WARPS2 4
#endif
__host__ __device__ constexpr int lt_warps(int S) { return S == 4 ? 4 : (S == 2 ? CVSR_LT_WARPS2 : 8); }
#ifndef CVSR_LT_CH
#define CVSR_LT_CH 4
#endif
#ifndef CVSR_LT_STAGE_KB
#define CVSR_LT_STAGE_KB 3
#endif
constexpr int LT_CH = CVSR_LT_CH;  // checks per warp
#ifndef CVSR_LT_CH2
#define CVSR_LT_CH2 12
#endif
constexpr int LT_CH2 = CVSR_LT_CH2;  // degree <= 2 checks per warp (codes with DC >= 6)
#ifndef CVSR_LT_CH2_WAVES
#define CVSR_LT_CH2_WAVES 4  // shorter tail chunks below this many waves of warps
#endif
static_assert(LT_CH <= 32 && LT_CH2 <= 32, "a chunk's descriptors are held one per lane");

template <int DC, int S>
struct LtLayout {
    static constexpr int LINE = LANES * S;                 // floats per line
    static constexpr int STAGE = 2 * DC * LINE;            // floats: DC posterior lines, then DC message lines
    // stages per warp: 3 while a stage is at most CVSR_LT_STAGE_KB, else 2 (shared memory per SM)
    static constexpr int P = (STAGE * 4 <= CVSR_LT_STAGE_KB * 1024) ? 3 : 2;
    // degree <= 2 checks of codes with DC >= 6 (MET type-A checks): the stages are re-cut into NS2
    // slots of 2 posterior + 2 message lines, so a warp has NS2 such checks in flight, and a warp
    // takes LT_CH2 of them
    static constexpr bool PAIRS = DC >= 6;
    static constexpr int NS2 = PAIRS ? P * DC / 2 : 0;
    static constexpr int NB = NS2 > P ? NS2 : P;  // mbarriers per warp
    static constexpr int VIDX = LT_CH * DC > 2 * LT_CH2 ? LT_CH * DC : 2 * LT_CH2;
    static constexpr size_t RAW = (size_t)P * STAGE * 4 + NB * 8 + (size_t)VIDX * 4;
    static constexpr size_t WARP_BYTES = (RAW + 127) & ~(size_t)127;
    static constexpr size_t BLOCK_BYTES = WARP_BYTES * lt_warps(S);
    // blocks per SM the shared memory allows (228 KB per SM, 1 KB reserved per block), at most 4
    static constexpr int SMEM_BLOCKS = (int)((228 * 1024) / (BLOCK_BYTES + 1024));
#ifdef CVSR_LT_MINB
    static constexpr int BLOCKS = CVSR_LT_MINB;
#else
    static constexpr int BLOCKS = SMEM_BLOCKS < 1 ? 1 : (SMEM_BLOCKS > 4 ? 4 : SMEM_BLOCKS);
#endif
};

// the check update of one check from its stage: DCT = compute width (>= deg; DCL = the stage
// layout's DC).  Results overwrite the stage: posterior lines <- post_v, message lines <- r_e.
#ifndef CVSR_LT_VLOAD
#define CVSR_LT_VLOAD 0
#endif
template <int DCT, int DCL, int S>
__device__ __forceinline__ void lt_compute(float *__restrict__ sp, int deg, uint32_t sb, int lane, float qmax2,
                                           bool first = false) {
    constexpr int LINE = LANES * S;
    float *pp = sp + lane * S;               // posterior lines
    float *rp = sp + DCL * LINE + lane * S;  // message lines
#if CVSR_LT_VLOAD
    // all S frames of each line with one vector shared-memory load (no 2-way bank conflicts)
    float qv[S][DCT];
#pragma unroll
    for (int k = 0; k < DCT; ++k) {
        if (k < deg) {
            const FV<S> p = ldv<S>(pp + k * LINE), r = first ? splat<S>(0.0f) : ldv<S>(rp + k * LINE);
#pragma unroll
            for (int s = 0; s < S; ++s) qv[s][k] = p.c[s] - r.c[s];
        } else {
#pragma unroll
            for (int s = 0; s < S; ++s) qv[s][k] = DUMMY_Q;
        }
    }
#endif
#pragma unroll(S == 4 ? 1 : S)
    for (int s = 0; s < S; ++s) {
        float qu[DCT], a[DCT];
#pragma unroll
        for (int k = 0; k < DCT; ++k) {
#if CVSR_LT_VLOAD
            qu[k] = qv[s][k];
#else
            qu[k] = (k < deg) ? pp[k * LINE + s] - (first ? 0.0f : rp[k * LINE + s]) : DUMMY_Q;
#endif
            a[k] = (k < deg) ? clampf(qu[k], qmax2) : DUMMY_Q;
        }
        cn_update<DCT>(a, (sb >> s) & 1u, qmax2);
#pragma unroll
        for (int k = 0; k < DCT; ++k) {
            if (k < deg) {
                rp[k * LINE + s] = a[k];
                pp[k * LINE + s] = qu[k] + a[k];
            }
        }
    }
}

// lane-vectorised stores of r_e and post_v of one check from its stage, and the hard decisions
// [post_v < 0] of the tile's active frames (one word per sub-tile, stored together).  DCT = the
// compile-time bound of the loop (the check's exact degree when EXACT, else >= deg).
template <int DCT, int DCL, int S, bool EXACT>
__device__ __forceinline__ void lt_store(const float *__restrict__ sp, int deg, int lo, const int *__restrict__ vrow,
                                         uint32_t al, const uint4 &act, int lane, float *__restrict__ mw,
                                         float *__restrict__ Lw, uint32_t *__restrict__ hbt) {
    constexpr int LINE = LANES * S;
#pragma unroll
    for (int k = 0; k < DCT; ++k) {
        if (EXACT || k < deg) {
            const FV<S> post = ldv<S>(sp + k * LINE + lane * S);
            if (al) {
                stv<S>(mw + (size_t)(lo + k) * LINE, ldv<S>(sp + (DCL + k) * LINE + lane * S));
                stv<S>(Lw + (size_t)vrow[k] * LINE, post);
            }
            uint32_t w[S];
#pragma unroll
            for (int q = 0; q < S; ++q) w[q] = __ballot_sync(FULL, post.c[q] < 0.0f) & cmpu(act, q);
            if (lane == 0) {
                uint32_t *h = hbt + (size_t)vrow[k] * 4;
                if constexpr (S == 1) h[0] = w[0];
                else if constexpr (S == 2) *reinterpret_cast<uint2 *>(h) = make_uint2(w[0], w[1]);
                else *reinterpret_cast<uint4 *>(h) = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    }
}

// one check: compute (lt_compute; deg passed as DCT when exact, so no edge is a padded dummy and
// no degree predicate remains) and store
template <int DCT, int DCL, int S, bool EXACT>
__device__ __forceinline__ void lt_check(float *__restrict__ sp, int deg, uint32_t sb, int lane, float qmax2,
                                         bool first, int lo, const int *__restrict__ vrow, uint32_t al,
                                         const uint4 &act, float *__restrict__ mw, float *__restrict__ Lw,
                                         uint32_t *__restrict__ hbt) {
    lt_compute<DCT, DCL, S>(sp, EXACT ? DCT : deg, sb, lane, qmax2, first);
    __syncwarp();
    lt_store<DCT, DCL, S, EXACT>(sp, EXACT ? DCT : deg, lo, vrow, al, act, lane, mw, Lw, hbt);
}

#ifndef CVSR_LT_EXACT
#define CVSR_LT_EXACT 1
#endif
// exact-degree bodies are used up to this maximum check degree: measured faster on C2 (degrees 4/5:
// 43.8 vs 46.6 ms per step); on C4 (6/7, 8/9) slower with 8-warp blocks (86.0 vs 84.3 ms, i-cache)
// and faster with the final 4-warp blocks and MET tail chunks (96.0 vs 97.4 ms; C4fast 74.2 vs 75.2;
// C3 11.5 vs 11.3: its degree-6 core checks are few and the kernel's registers rise 76 -> 96)
#ifndef CVSR_LT_EXACT_MAXDC
#define CVSR_LT_EXACT_MAXDC 12
#endif
// k_layer_tma's pipeline for a chunk of nc <= LT_CH2 degree <= 2 checks (layer positions g0 ..):
// NS2 slots of 2 posterior + 2 message lines cut from the warp's stages, one mbarrier each.  Same
// per-check steps and arithmetic as the general path (lt_check<2, ...>), so results are identical;
// only more checks are in flight per warp and a warp's prologue is shared by LT_CH2 checks.
template <int DC, int S>
__device__ __forceinline__ void lt_pairs(const CodeDev &cd, const DecState &ds, int g0, int nc, int ti, int lane,
                                         unsigned char *wb, float qmax2, int first, int early) {
    using LY = LtLayout<DC, S>;
    constexpr int LINE = LY::LINE;
    constexpr int NS = LY::NS2;
    constexpr int SLOT = 4 * LINE;  // floats
    float *stage = reinterpret_cast<float *>(wb);
    uint64_t *bar = reinterpret_cast<uint64_t *>(wb + (size_t)LY::P * LY::STAGE * 4);
    int *vidx = reinterpret_cast<int *>(bar + LY::NB);
    int4 dsc = make_int4(0, 0, 0, 0);
    if (nc > 0) {
        if (lane == 0) {
#pragma unroll
            for (int p = 0; p < NS; ++p) mbar_init(&bar[p], 1);
            mbar_init_fence();
        }
        if (lane < nc) dsc = cd.layer_desc[g0 + lane];
        for (int f = lane; f < 2 * LT_CH2; f += LANES)
            vidx[f] = (f >> 1) < nc ? cd.layer_col[(size_t)(g0 + (f >> 1)) * DC + (f & 1)] : 0;
        __syncwarp();
    }
    const int mylo = dsc.x, myhi = dsc.x + dsc.y;
    const int npre = min(NS, nc);
    int t = 0;
    uint4 act = make_uint4(0u, 0u, 0u, 0u), mys = make_uint4(0u, 0u, 0u, 0u);
    const float *Lt = nullptr, *mt = nullptr;
    auto issue_msg = [&](int i, int p) {
        const int lo = __shfl_sync(FULL, mylo, i), deg = __shfl_sync(FULL, myhi, i) - lo;
        if (lane == 0 && deg > 0 && !first) {
            mbar_expect_tx(&bar[p], (uint32_t)deg * LINE * 4u);
            bulk_g2s(stage + (size_t)p * SLOT + 2 * LINE, mt + (size_t)lo * LINE, (uint32_t)deg * LINE * 4, &bar[p]);
        }
    };
    auto issue_post = [&](int i, int p) {
        const int lo = __shfl_sync(FULL, mylo, i), deg = __shfl_sync(FULL, myhi, i) - lo;
        float *sp = stage + (size_t)p * SLOT;
        const int *vr = vidx + i * 2;
#pragma unroll
        for (int k = 0; k < 2; ++k)
            if (k < deg) cp_async_g2s<4 * S>(sp + k * LINE + lane * S, Lt + (size_t)vr[k] * LINE + lane * S);
        cp_async_mbar_arrive(&bar[p]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar[p]);
    };
    auto tile_meta = [&]() -> bool {
        if (ti >= ds.counts[0] || nc <= 0) return false;
        t = ds.active_list[ti];
        act = ds.tile_active[t];
        if (lane < nc) mys = ds.st[(size_t)t * cd.M + g0 + lane];
        Lt = ds.L + (size_t)t * cd.n * LINE;
        mt = ds.msg + (size_t)t * cd.E * LINE;
        return true;
    };
    bool live = true;
    if (early) {
        live = tile_meta();
        if (live)
            for (int i = 0; i < npre; ++i) issue_msg(i, i);
    }
    griddep_wait();
    griddep_launch_dependents();
    if (!early) {
        live = tile_meta();
        if (live)
            for (int i = 0; i < npre; ++i) issue_msg(i, i);
    }
    if (!live) return;
    for (int i = 0; i < npre; ++i) issue_post(i, i);
    const uint32_t al = lane_act<S>(act, lane);
    uint32_t *hbt = reinterpret_cast<uint32_t *>(ds.hb + (size_t)t * cd.n);
    float *Lw = ds.L + (size_t)t * cd.n * LINE + lane * S;
    float *mw = ds.msg + (size_t)t * cd.E * LINE + lane * S;
    uint32_t phase = 0u;
    for (int i = 0; i < nc; ++i) {
        const int p = i % NS;
        mbar_wait(&bar[p], (phase >> p) & 1u);
        phase ^= 1u << p;
        const int lo = __shfl_sync(FULL, mylo, i), deg = __shfl_sync(FULL, myhi, i) - lo;
        uint4 sw;
        sw.x = __shfl_sync(FULL, mys.x, i);
        sw.y = (S > 1) ? __shfl_sync(FULL, mys.y, i) : 0u;
        sw.z = (S > 2) ? __shfl_sync(FULL, mys.z, i) : 0u;
        sw.w = (S > 2) ? __shfl_sync(FULL, mys.w, i) : 0u;
        const uint32_t sb = lane_act<S>(sw, lane);
        lt_check<2, 2, S, false>(stage + (size_t)p * SLOT, deg, sb, lane, qmax2, first != 0, lo, vidx + i * 2, al, act,
                                 mw, Lw, hbt);
        fence_proxy_async_smem();
        __syncwarp();
        if (i + NS < nc) {
            issue_msg(i + NS, p);
            issue_post(i + NS, p);
        }
    }
}

template <int DC, int S>
__global__ void __launch_bounds__(lt_warps(S) * 32, LtLayout<DC, S>::BLOCKS)
    k_layer_tma(CodeDev cd, DecState ds, int lbeg, int lcnt, int nbig, int ch2, float qmax2, int first, int early) {
    using LY = LtLayout<DC, S>;
    constexpr int LINE = LY::LINE;
    constexpr int P = LY::P;
    extern __shared__ __align__(128) unsigned char lt_smem[];
    const int ti = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * lt_warps(S) + warp;  // the warp's chunk in the layer
    const int nch = (nbig + LT_CH - 1) / LT_CH;      // chunks of degree > 2 checks
    unsigned char *wb = lt_smem + (size_t)warp * LY::WARP_BYTES;
    if constexpr (LY::PAIRS) {
        if (gw >= nch) {  // warp-uniform: a chunk of the layer's degree <= 2 tail
            const int j0 = nbig + (gw - nch) * ch2;
            lt_pairs<DC, S>(cd, ds, lbeg + j0, min(ch2, lcnt - j0), ti, lane, wb, qmax2, first, early);
            return;
        }
    }
    const int i0 = gw * LT_CH;
    const int nc = min(LT_CH, nbig - i0);
    float *stage = reinterpret_cast<float *>(wb);
    uint64_t *bar = reinterpret_cast<uint64_t *>(wb + (size_t)P * LY::STAGE * 4);
    int *vidx = reinterpret_cast<int *>(bar + LY::NB);
    // Prologue (it may overlap the previous layer's grid when launched as a programmatic
    // dependent): the chunk's descriptors {row start, degree, check id} and padded column indices,
    // independent coalesced loads (layer_desc / layer_col in layer order).  When `early` (the
    // previous kernel of the stream is a layer kernel of the same iteration, so the tile lists,
    // syndrome rows and compaction of this iteration are complete -- every CTA of that kernel
    // passed its griddep_wait before this grid launched) the tile, its syndrome rows and the
    // message lines of the first P checks (written by this layer's own kernel one iteration ago)
    // are fetched here too; only the posterior lines wait for the previous layer.
    const int g0 = lbeg + i0;
    int4 dsc = make_int4(0, 0, 0, 0);
    if (nc > 0) {
        if (lane == 0) {
#pragma unroll
            for (int p = 0; p < P; ++p) mbar_init(&bar[p], 1);
            mbar_init_fence();
        }
        if (lane < nc) dsc = cd.layer_desc[g0 + lane];
        for (int f = lane; f < LT_CH * DC; f += LANES) vidx[f] = f < nc * DC ? cd.layer_col[(size_t)g0 * DC + f] : 0;
        __syncwarp();  // barrier init and vidx visible to the whole warp
    }
    const int mylo = dsc.x, myhi = dsc.x + dsc.y;
    const int npre = min(P, nc);
    int t = 0;
    uint4 act = make_uint4(0u, 0u, 0u, 0u), mys = make_uint4(0u, 0u, 0u, 0u);
    const float *Lt = nullptr, *mt = nullptr;
    // stage p of check i: lane 0 arms the stage's mbarrier with the message bytes and copies the
    // deg message lines, one contiguous CSR span, with one bulk copy (first iteration: r = 0,
    // reading R-9 init, nothing to load); every lane copies its S frames of the deg posterior
    // lines (cp.async tracked by the same mbarrier) and lane 0 arrives once they are registered
    auto issue_msg = [&](int i, int p) {
        const int lo = __shfl_sync(FULL, mylo, i), deg = __shfl_sync(FULL, myhi, i) - lo;
        if (lane == 0 && deg > 0 && !first) {
            mbar_expect_tx(&bar[p], (uint32_t)deg * LINE * 4u);
            bulk_g2s(stage + (size_t)p * LY::STAGE + DC * LINE, mt + (size_t)lo * LINE, (uint32_t)deg * LINE * 4,
                     &bar[p]);
        }
    };
    auto issue_post = [&](int i, int p) {
        const int lo = __shfl_sync(FULL, mylo, i), deg = __shfl_sync(FULL, myhi, i) - lo;
        float *sp = stage + (size_t)p * LY::STAGE;
        const int *vr = vidx + i * DC;
#pragma unroll
        for (int k = 0; k < DC; ++k)
            if (k < deg) cp_async_g2s<4 * S>(sp + k * LINE + lane * S, Lt + (size_t)vr[k] * LINE + lane * S);
        cp_async_mbar_arrive(&bar[p]);
        __syncwarp();  // every lane's pending-count increment precedes lane 0's arrival
        if (lane == 0) mbar_arrive(&bar[p]);
    };
    auto tile_meta = [&]() -> bool {
        if (ti >= ds.counts[0] || nc <= 0) return false;
        t = ds.active_list[ti];
        act = ds.tile_active[t];
        // syndrome rows (in layer order for the layered schedule)
        if (lane < nc) mys = ds.st[(size_t)t * cd.M + g0 + lane];
        Lt = ds.L + (size_t)t * cd.n * LINE;
        mt = ds.msg + (size_t)t * cd.E * LINE;
        return true;
    };
    bool live = true;
    if (early) {
        live = tile_meta();
        if (live)
            for (int i = 0; i < npre; ++i) issue_msg(i, i);
    }
    griddep_wait();  // the previous layer's posteriors (and, if !early, this iteration's lists)
    griddep_launch_dependents();
    if (!early) {
        live = tile_meta();
        if (live)
            for (int i = 0; i < npre; ++i) issue_msg(i, i);
    }
    if (!live) return;
    for (int i = 0; i < npre; ++i) issue_post(i, i);
    const uint32_t al = lane_act<S>(act, lane);
    uint32_t *hbt = reinterpret_cast<uint32_t *>(ds.hb + (size_t)t * cd.n);
    float *Lw = ds.L + (size_t)t * cd.n * LINE + lane * S;
    float *mw = ds.msg + (size_t)t * cd.E * LINE + lane * S;
    uint32_t phase = 0u;
    for (int i = 0; i < nc; ++i) {
        const int p = i % P;
        mbar_wait(&bar[p], (phase >> p) & 1u);
        phase ^= 1u << p;
        const int lo = __shfl_sync(FULL, mylo, i), deg = __shfl_sync(FULL, myhi, i) - lo;
        uint4 sw;
        sw.x = __shfl_sync(FULL, mys.x, i);
        sw.y = (S > 1) ? __shfl_sync(FULL, mys.y, i) : 0u;
        sw.z = (S > 2) ? __shfl_sync(FULL, mys.z, i) : 0u;
        sw.w = (S > 2) ? __shfl_sync(FULL, mys.w, i) : 0u;
        const uint32_t sb = lane_act<S>(sw, lane);
        float *sp = stage + (size_t)p * LY::STAGE;
        const int *vrow = vidx + i * DC;
        const bool f1 = first != 0;
        // exact-degree bodies for the two largest degrees (the irregular codes' checks take two
        // consecutive degrees; no padded dummy edges, no degree predicates), the 2-edge body for
        // MET type-A checks, and the padded body otherwise
        if (DC >= 6 && deg <= 2) {
            lt_check<2, DC, S, false>(sp, deg, sb, lane, qmax2, f1, lo, vrow, al, act, mw, Lw, hbt);
        } else if constexpr (CVSR_LT_EXACT && DC <= CVSR_LT_EXACT_MAXDC) {
            if (deg == DC)
                lt_check<DC, DC, S, true>(sp, deg, sb, lane, qmax2, f1, lo, vrow, al, act, mw, Lw, hbt);
            else if (DC > 3 && deg == DC - 1)
                lt_check<(DC > 3 ? DC - 1 : DC), DC, S, true>(sp, deg, sb, lane, qmax2, f1, lo, vrow, al, act, mw, Lw,
                                                            hbt);
            else
                lt_check<DC, DC, S, false>(sp, deg, sb, lane, qmax2, f1, lo, vrow, al, act, mw, Lw, hbt);
        } else {
            lt_check<DC, DC, S, false>(sp, deg, sb, lane, qmax2, f1, lo, vrow, al, act, mw, Lw, hbt);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (i + P < nc) {
            issue_msg(i + P, p);
            issue_post(i + P, p);
        }
    }
}

// ------------------------------------------------------------------ persistent layer kernel
//
// k_layer_tmap<DC, S>: k_layer_tma's check update with a persistent grid.  The layer's work items
// (tile, chunk of LT_CH checks) are spread over all resident warps (item = warp id + k x warps);
// each warp runs ONE stage ring over the concatenated checks of its items, so the ring never
// drains between items, and each item's metadata -- descriptors, syndrome rows, padded column
// indices and the tile's active mask -- is copied into shared memory by cp.async one item ahead
// (tracked by a per-buffer mbarrier), so no dependent index load stalls the warp.  Results are
// bit-identical to k_layer_tma (same arithmetic per check; checks of a layer are independent).
template <int DC, int S>
struct LtpLayout {
    using LY = LtLayout<DC, S>;
    static constexpr int META = 16 * LT_CH * 2 + 16 + 4 * LT_CH * DC;  // desc, st rows, act, vidx
    static constexpr int META_AL = (META + 15) & ~15;
    static constexpr int BARS = ((LY::P + 2) * 8 + 15) & ~15;  // stage + metadata barriers, 16-B aligned
    static constexpr size_t RAW = (size_t)LY::P * LY::STAGE * 4 + BARS + 2 * (size_t)META_AL;
    static constexpr size_t WARP_BYTES = (RAW + 127) & ~(size_t)127;
    static constexpr size_t BLOCK_BYTES = WARP_BYTES * LT_WARPS;
    static constexpr int SMEM_BLOCKS = (int)((228 * 1024) / (BLOCK_BYTES + 1024));
    static constexpr int BLOCKS = SMEM_BLOCKS < 1 ? 1 : (SMEM_BLOCKS > 4 ? 4 : SMEM_BLOCKS);
};

template <int DC, int S>
__global__ void __launch_bounds__(LT_WARPS * 32, LtpLayout<DC, S>::BLOCKS)
    k_layer_tmap(CodeDev cd, DecState ds, int lbeg, int lcnt, float qmax2) {
    using LY = LtLayout<DC, S>;
    using LP = LtpLayout<DC, S>;
    constexpr int LINE = LY::LINE;
    constexpr int P = LY::P;
    extern __shared__ __align__(128) unsigned char lt_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cpt = (lcnt + LT_CH - 1) / LT_CH;
    const int n_items = ds.counts[0] * cpt;
    // dynamic work distribution: items are grabbed from ds.counts[8]; the last warp to run out
    // resets the counters for the next launch (ds.counts[9] counts exited warps)
    const int total_warps = gridDim.x * LT_WARPS;
    auto grab = [&]() {
        int v = 0;
        if (lane == 0) v = atomicAdd(&ds.counts[8], 1);
        return __shfl_sync(FULL, v, 0);
    };
    auto leave = [&]() {
        if (lane == 0) {
            __threadfence();
            if (atomicAdd(&ds.counts[9], 1) == total_warps - 1) {
                ds.counts[8] = 0;
                ds.counts[9] = 0;
                __threadfence();
            }
        }
    };
    int it_cur = grab();
    if (it_cur >= n_items) {
        leave();
        return;
    }
    unsigned char *wb = lt_smem + (size_t)warp * LP::WARP_BYTES;
    float *stage = reinterpret_cast<float *>(wb);
    uint64_t *bar = reinterpret_cast<uint64_t *>(wb + (size_t)P * LY::STAGE * 4);
    uint64_t *mbar = bar + P;  // metadata barriers of the two item buffers
    unsigned char *meta0 = wb + (size_t)P * LY::STAGE * 4 + LP::BARS;
    if (lane == 0) {
#pragma unroll
        for (int p = 0; p < P + 2; ++p) mbar_init(&bar[p], 1);
        mbar_init_fence();
    }
    __syncwarp();
    // metadata buffer b: desc[LT_CH] int4 | strow[LT_CH] uint4 | act uint4 | vidx[LT_CH * DC] int
    auto m_desc = [&](int b) { return reinterpret_cast<int4 *>(meta0 + (size_t)b * LP::META_AL); };
    auto m_st = [&](int b) { return reinterpret_cast<uint4 *>(meta0 + (size_t)b * LP::META_AL + 16 * LT_CH); };
    auto m_act = [&](int b) { return reinterpret_cast<uint4 *>(meta0 + (size_t)b * LP::META_AL + 32 * LT_CH); };
    auto m_vidx = [&](int b) { return reinterpret_cast<int *>(meta0 + (size_t)b * LP::META_AL + 32 * LT_CH + 16); };
    struct Item {
        int t, nc, g0, b;
        bool valid;
    };
    auto make = [&](int item, int t, int b) {
        Item x;
        x.valid = item < n_items;
        x.b = b;
        x.t = t;
        x.nc = 0;
        x.g0 = 0;
        if (x.valid) {
            const int ch = item % cpt;
            x.g0 = lbeg + ch * LT_CH;
            x.nc = min(LT_CH, lcnt - ch * LT_CH);
        }
        return x;
    };
    auto tile_of = [&](int item) { return item < n_items ? ds.active_list[item / cpt] : 0; };
    // asynchronous metadata copy of an item into its buffer (every lane copies its part)
    auto fetch = [&](const Item &x) {
        if (!x.valid) return;
        if (lane < x.nc) {
            cp_async_g2s<16>(m_desc(x.b) + lane, cd.layer_desc + x.g0 + lane);
            cp_async_g2s<16>(m_st(x.b) + lane, ds.st + (size_t)x.t * cd.M + x.g0 + lane);
        }
        if (lane == 31) cp_async_g2s<16>(m_act(x.b), ds.tile_active + x.t);
        int *vx = m_vidx(x.b);
        for (int f = lane; f < x.nc * DC; f += LANES) cp_async_g2s<4>(vx + f, cd.layer_col + (size_t)x.g0 * DC + f);
        cp_async_mbar_arrive(&mbar[x.b]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&mbar[x.b]);
    };
    uint32_t mph = 0u;  // phase bit per metadata buffer
    auto meta_wait = [&](const Item &x) {
        mbar_wait(&mbar[x.b], (mph >> x.b) & 1u);
        mph ^= 1u << x.b;
    };
    // stage p of check i of item x (see k_layer_tma)
    auto issue = [&](const Item &x, int i, int p) {
        const int4 d = m_desc(x.b)[i];
        const int lo = d.x, deg = d.y;
        float *sp = stage + (size_t)p * LY::STAGE;
        const int *vr = m_vidx(x.b) + i * DC;
        const float *Lt = ds.L + (size_t)x.t * cd.n * LINE;
        const float *mt = ds.msg + (size_t)x.t * cd.E * LINE;
#pragma unroll
        for (int k = 0; k < DC; ++k)
            if (k < deg) cp_async_g2s<4 * S>(sp + k * LINE + lane * S, Lt + (size_t)vr[k] * LINE + lane * S);
        cp_async_mbar_arrive(&bar[p]);
        __syncwarp();
        if (lane == 0) {
            mbar_arrive_tx(&bar[p], (uint32_t)deg * LINE * 4u);
            if (deg > 0) bulk_g2s(sp + DC * LINE, mt + (size_t)lo * LINE, (uint32_t)deg * LINE * 4, &bar[p]);
        }
    };
    int it_nxt = grab(), it_nn = grab();
    Item cur = make(it_cur, tile_of(it_cur), 0);
    Item nxt = make(it_nxt, tile_of(it_nxt), 1);
    int t_nn = tile_of(it_nn);
    fetch(cur);
    fetch(nxt);
    meta_wait(cur);
    bool nxt_active = false;
    int iss_sel = 0, iss_i = 0;  // issue cursor: item (0 = cur, 1 = nxt) and check
    int issued = 0, done = 0;
    auto try_issue = [&]() -> bool {
        if (iss_sel == 0 && iss_i >= cur.nc) {
            iss_sel = 1;
            iss_i = 0;
        }
        if (iss_sel == 1) {
            if (!nxt.valid || iss_i >= nxt.nc) return false;
            if (!nxt_active) {
                meta_wait(nxt);
                nxt_active = true;
            }
            issue(nxt, iss_i, issued % P);
        } else {
            issue(cur, iss_i, issued % P);
        }
        ++iss_i;
        ++issued;
        return true;
    };
    while (issued < P && try_issue()) {
    }
    int ci = 0;
    for (;;) {
        const int p = done % P;
        mbar_wait(&bar[p], (uint32_t)(done / P) & 1u);
        {
            const int4 d = m_desc(cur.b)[ci];
            const int lo = d.x, deg = d.y;
            const uint4 act = *m_act(cur.b);
            const uint32_t sb = lane_act<S>(m_st(cur.b)[ci], lane);
            const uint32_t al = lane_act<S>(act, lane);
            float *sp = stage + (size_t)p * LY::STAGE;
            const int *vrow = m_vidx(cur.b) + ci * DC;
            uint32_t *hbt = reinterpret_cast<uint32_t *>(ds.hb + (size_t)cur.t * cd.n);
            float *Lw = ds.L + (size_t)cur.t * cd.n * LINE + lane * S;
            float *mw = ds.msg + (size_t)cur.t * cd.E * LINE + lane * S;
            if (CVSR_LT_EXACT && deg == DC) {
                lt_check<DC, DC, S, true>(sp, deg, sb, lane, qmax2, false, lo, vrow, al, act, mw, Lw, hbt);
            } else if (CVSR_LT_EXACT && DC > 3 && deg == DC - 1) {
                lt_check<(DC > 3 ? DC - 1 : DC), DC, S, true>(sp, deg, sb, lane, qmax2, false, lo, vrow, al, act, mw,
                                                            Lw, hbt);
            } else if (DC >= 6 && deg <= 2) {
                lt_check<2, DC, S, false>(sp, deg, sb, lane, qmax2, false, lo, vrow, al, act, mw, Lw, hbt);
            } else {
                lt_check<DC, DC, S, false>(sp, deg, sb, lane, qmax2, false, lo, vrow, al, act, mw, Lw, hbt);
            }
        }
        fence_proxy_async_smem();
        __syncwarp();
        ++done;
        ++ci;
        if (ci == cur.nc) {
            if (!nxt.valid) {
                leave();
                break;
            }
            // the next item becomes current; its successor's metadata goes to the freed buffer
            const bool was_active = nxt_active;
            cur = nxt;
            ci = 0;
            if (iss_sel == 0) iss_i = 0;
            iss_sel = 0;
            if (!was_active) meta_wait(cur);
            nxt_active = false;
            it_nxt = it_nn;
            it_nn = (it_nn < n_items) ? grab() : n_items;
            nxt = make(it_nxt, t_nn, 1 - cur.b);
            t_nn = tile_of(it_nn);
            fetch(nxt);
        }
        while (issued < done + P && try_issue()) {
        }
    }
}

template <int DC, int S>
static void launch_layer_tmap_t(const CodeDev &cd, const DecState &ds, int grid_tiles, int lbeg, int lcnt, float q2,
                                cudaStream_t s) {
    static int max_blocks = 0;
    constexpr size_t smem = LtpLayout<DC, S>::BLOCK_BYTES;
    if (max_blocks == 0) {
        cudaFuncSetAttribute(k_layer_tmap<DC, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int dev = 0, n_sm = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_layer_tmap<DC, S>, LT_WARPS * 32, smem);
        max_blocks = (per_sm > 0 ? per_sm : 1) * n_sm;
    }
    const long long items = (long long)grid_tiles * ((lcnt + LT_CH - 1) / LT_CH);
    const long long want = (items + LT_WARPS - 1) / LT_WARPS;
    const int grid = (int)(want < max_blocks ? want : max_blocks);
    if (grid > 0) k_layer_tmap<DC, S><<<grid, LT_WARPS * 32, smem, s>>>(cd, ds, lbeg, lcnt, q2);
}

template <int S>
static bool launch_layer_tmap_s(const CodeDev &cd, const DecState &ds, int grid_tiles, int lbeg, int lcnt, float q2,
                                cudaStream_t s) {
    switch (cd.max_dc) {
        case 1: case 2: launch_layer_tmap_t<2, S>(cd, ds, grid_tiles, lbeg, lcnt, q2, s); return true;
        case 3: launch_layer_tmap_t<3, S>(cd, ds, grid_tiles, lbeg, lcnt, q2, s); return true;
        case 4: launch_layer_tmap_t<4, S>(cd, ds, grid_tiles, lbeg, lcnt, q2, s); return true;
        case 5: launch_layer_tmap_t<5, S>(cd, ds, grid_tiles, lbeg, lcnt, q2, s); return true;
        case 6: launch_layer_tmap_t<6, S>(cd, ds, grid_tiles, lbeg, lcnt, q2, s); return true;
        case 7: launch_layer_tmap_t<7, S>(cd, ds, grid_tiles, lbeg, lcnt, q2, s); return true;
        case 8: launch_layer_tmap_t<8, S>(cd, ds, grid_tiles, lbeg, lcnt, q2, s); return true;
        case 9: launch_layer_tmap_t<9, S>(cd, ds, grid_tiles, lbeg, lcnt, q2, s); return true;
        case 10: launch_layer_tmap_t<10, S>(cd, ds, grid_tiles, lbeg, lcnt, q2, s); return true;
        case 11: case 12: launch_layer_tmap_t<12, S>(cd, ds, grid_tiles, lbeg, lcnt, q2, s); return true;
        default: return false;
    }
}

// ------------------------------------------------------------------ syndrome test (layered)
//
// H xhat = s for every active frame of the listed tiles (stopping rule A-12, decision of the
// previous iteration): one thread per (check, tile) XORs the hard-decision words of the check's
// variables (bit = lane, component = sub-tile) into its syndrome word; any nonzero bit marks that
// frame unsatisfied.  Unlike the check-only k_cn (a warp per 4 checks), every thread has its own
// independent gathers in flight.
template <int S>
__global__ void __launch_bounds__(256) k_synd_test(CodeDev cd, DecState ds) {
    const int ti = blockIdx.y;
    if (ti >= ds.counts[0]) return;
    const int t = ds.active_list[ti];
    const uint4 act = ds.tile_active[t];
    __shared__ uint32_t s_unsat[SUBS];
    if (threadIdx.x < SUBS) s_unsat[threadIdx.x] = 0u;
    __syncthreads();
    const int i = blockIdx.x * 256 + threadIdx.x;  // layer-order position (st rows are in layer order)
    uint32_t u[SUBS] = {0u, 0u, 0u, 0u};
    if (i < cd.M) {
        const uint4 sw = ds.st[(size_t)t * cd.M + i];
        u[0] = sw.x;
        u[1] = sw.y;
        u[2] = sw.z;
        u[3] = sw.w;
        const uint4 *hbt = ds.hb + (size_t)t * cd.n;
        const int4 d = cd.layer_desc[i];
#pragma unroll 4
        for (int e = d.x; e < d.x + d.y; ++e) {
            const uint4 h = hbt[cd.col_idx[e]];
            u[0] ^= h.x;
            if (S > 1) u[1] ^= h.y;
            if (S > 2) {
                u[2] ^= h.z;
                u[3] ^= h.w;
            }
        }
    }
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < S; ++q) {
        const uint32_t v = __reduce_or_sync(FULL, u[q]) & cmpu(act, q);
        if (lane == 0 && v) atomicOr(&s_unsat[q], v);
    }
    __syncthreads();
    if (threadIdx.x < S && s_unsat[threadIdx.x])
        atomicOr(reinterpret_cast<uint32_t *>(&ds.tile_unsat[t]) + threadIdx.x, s_unsat[threadIdx.x]);
}

// Same test with the check's padded column indices from layer_col (DC = layer_dc, one row of
// consecutive words per check) and TT tiles per thread: every index load and then every
// hard-decision gather of the TT tiles is issued before the first XOR, so a thread has up to
// TT x DC independent gathers in flight instead of a dependent index -> gather chain per edge.
constexpr int ST_TT = 2;
template <int S, int DC>
__global__ void __launch_bounds__(256) k_synd_test_w(CodeDev cd, DecState ds) {
    __shared__ uint32_t s_unsat[ST_TT][SUBS];
    if (threadIdx.x < ST_TT * SUBS) s_unsat[threadIdx.x / SUBS][threadIdx.x % SUBS] = 0u;
    __syncthreads();
    const int i = blockIdx.x * 256 + threadIdx.x;  // layer-order position (st rows are in layer order)
    const int nt = min(ST_TT, ds.counts[0] - (int)blockIdx.y * ST_TT);
    if (nt <= 0) return;  // block-uniform
    int tt[ST_TT];
    uint4 act[ST_TT];
#pragma unroll
    for (int k = 0; k < ST_TT; ++k) {
        tt[k] = k < nt ? ds.active_list[blockIdx.y * ST_TT + k] : 0;
        act[k] = k < nt ? ds.tile_active[tt[k]] : make_uint4(0u, 0u, 0u, 0u);
    }
    uint4 u[ST_TT];
#pragma unroll
    for (int k = 0; k < ST_TT; ++k) u[k] = make_uint4(0u, 0u, 0u, 0u);
    if (i < cd.M) {
        const int deg = cd.layer_desc[i].y;
        int col[DC];
#pragma unroll
        for (int e = 0; e < DC; ++e) col[e] = cd.layer_col[(size_t)i * DC + e];
#pragma unroll
        for (int k = 0; k < ST_TT; ++k) {
            if (k < nt) {
                const uint4 *hbt = ds.hb + (size_t)tt[k] * cd.n;
                uint4 a = ds.st[(size_t)tt[k] * cd.M + i];
#pragma unroll
                for (int e = 0; e < DC; ++e) {
                    if (e < deg) {
                        const uint4 h = hbt[col[e]];
                        a.x ^= h.x;
                        if (S > 1) a.y ^= h.y;
                        if (S > 2) {
                            a.z ^= h.z;
                            a.w ^= h.w;
                        }
                    }
                }
                u[k] = a;
            }
        }
    }
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < ST_TT; ++k) {
        const uint32_t w4[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
        for (int q = 0; q < S; ++q) {
            const uint32_t v = __reduce_or_sync(FULL, w4[q]) & cmpu(act[k], q);
            if (lane == 0 && v) atomicOr(&s_unsat[k][q], v);
        }
    }
    __syncthreads();
    if (threadIdx.x < ST_TT * S) {
        const int k = threadIdx.x / S, q = threadIdx.x % S;
        if (k < nt && s_unsat[k][q])
            atomicOr(reinterpret_cast<uint32_t *>(&ds.tile_unsat[tt[k]]) + q, s_unsat[k][q]);
    }
}

static bool synd_test_w_enabled() {
    static const int v = [] {
        const char *e = getenv("CVSR_SYND_TEST_W");
        return (e && *e) ? atoi(e) : 1;
    }();
    return v != 0;
}

template <int S>
static bool launch_synd_test_w(const CodeDev &cd, const DecState &ds, int grid_tiles, cudaStream_t s) {
    dim3 grid((cd.M + 255) / 256, (grid_tiles + ST_TT - 1) / ST_TT);
    switch (cd.layer_dc) {
        case 2: k_synd_test_w<S, 2><<<grid, 256, 0, s>>>(cd, ds); return true;
        case 3: k_synd_test_w<S, 3><<<grid, 256, 0, s>>>(cd, ds); return true;
        case 4: k_synd_test_w<S, 4><<<grid, 256, 0, s>>>(cd, ds); return true;
        case 5: k_synd_test_w<S, 5><<<grid, 256, 0, s>>>(cd, ds); return true;
        case 6: k_synd_test_w<S, 6><<<grid, 256, 0, s>>>(cd, ds); return true;
        case 7: k_synd_test_w<S, 7><<<grid, 256, 0, s>>>(cd, ds); return true;
        case 8: k_synd_test_w<S, 8><<<grid, 256, 0, s>>>(cd, ds); return true;
        case 9: k_synd_test_w<S, 9><<<grid, 256, 0, s>>>(cd, ds); return true;
        case 10: k_synd_test_w<S, 10><<<grid, 256, 0, s>>>(cd, ds); return true;
        default: return false;
    }
}

void launch_synd_test(const CodeDev &cd, const DecState &ds, int grid_tiles, cudaStream_t s) {
    if (grid_tiles <= 0) return;
    if (synd_test_w_enabled() && cd.layer_col) {
        if (ds.subs == 4 && launch_synd_test_w<4>(cd, ds, grid_tiles, s)) return;
        if (ds.subs == 2 && launch_synd_test_w<2>(cd, ds, grid_tiles, s)) return;
        if (ds.subs == 1 && launch_synd_test_w<1>(cd, ds, grid_tiles, s)) return;
    }
    dim3 grid((cd.M + 255) / 256, grid_tiles);
    if (ds.subs == 4) k_synd_test<4><<<grid, 256, 0, s>>>(cd, ds);
    else if (ds.subs == 2) k_synd_test<2><<<grid, 256, 0, s>>>(cd, ds);
    else k_synd_test<1><<<grid, 256, 0, s>>>(cd, ds);
}

// programmatic dependent launch of the layer kernels (CVSR_LAYER_PDL=0: plain stream order)
static bool layer_pdl_enabled() {
    static const int v = [] {
        const char *e = getenv("CVSR_LAYER_PDL");
        return (e && *e) ? atoi(e) : 1;
    }();
    return v != 0;
}

// degree <= 2 layer tails in LT_CH2-check chunks with NS2 slots (CVSR_LAYER_PAIRS=0: LT_CH chunks)
static bool layer_pairs_enabled() {
    static const int v = [] {
        const char *e = getenv("CVSR_LAYER_PAIRS");
        return (e && *e) ? atoi(e) : 1;
    }();
    return v != 0;
}

// message lines of the first stages fetched before the dependency wait (CVSR_LAYER_EARLY=0: after)
static bool layer_early_enabled() {
    static const int v = [] {
        const char *e = getenv("CVSR_LAYER_EARLY");
        return (e && *e) ? atoi(e) : 1;
    }();
    return v != 0;
}

template <int DC, int S>
static void launch_layer_tma_t(const CodeDev &cd, const DecState &ds, int grid_tiles, int l, float q2,
                               int first, int early, cudaStream_t s) {
    static bool attr = false;
    constexpr size_t smem = LtLayout<DC, S>::BLOCK_BYTES;
    if (!attr) {
        cudaFuncSetAttribute(k_layer_tma<DC, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    const int lbeg = cd.layer_off[l], lcnt = cd.layer_off[l + 1] - lbeg;
    // degree <= 2 tail in LT_CH2-check chunks (codes with DC >= 6), the rest in LT_CH-check chunks
    const int nbig = (LtLayout<DC, S>::PAIRS && layer_pairs_enabled()) ? cd.layer_nbig[l] : lcnt;
    // chunk length of the tail: LT_CH2 while that leaves at least 4 waves of warps (resident warps
    // per GPU from the occupancy of this instantiation), else shorter (C3's many small MET layers:
    // 12-check chunks left 1.3 waves, 11.7 -> 12.8 ms per step)
    static int resident = 0;
    if (!resident) {
        int per_sm = 0, dev = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_layer_tma<DC, S>, lt_warps(S) * 32,
                                                      LtLayout<DC, S>::BLOCK_BYTES);
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        resident = std::max(1, per_sm * lt_warps(S) * sms);
    }
    int ch2 = LT_CH2;
    const int64_t tail = (int64_t)(lcnt - nbig) * grid_tiles;
    static const int waves = [] {
        const char *e = getenv("CVSR_LAYER_CH2_WAVES");  // test / tuning switch (0: always LT_CH2)
        return (e && *e) ? atoi(e) : CVSR_LT_CH2_WAVES;
    }();
    while (ch2 > LT_CH && tail < (int64_t)waves * resident * ch2) ch2 -= LT_CH;
    const int chunks = (nbig + LT_CH - 1) / LT_CH + (lcnt - nbig + ch2 - 1) / ch2;
    const dim3 grid((chunks + lt_warps(S) - 1) / lt_warps(S), grid_tiles);
    if (!layer_pdl_enabled()) {
        k_layer_tma<DC, S><<<grid, lt_warps(S) * 32, smem, s>>>(cd, ds, lbeg, lcnt, nbig, ch2, q2, first, 0);
        return;
    }
    // programmatic dependent launch: the grid is launched while the previous layer's last wave
    // runs, its CTAs do the code-constant prologue and wait (griddep_wait) for that grid to finish
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = dim3(lt_warps(S) * 32);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, k_layer_tma<DC, S>, cd, ds, lbeg, lcnt, nbig, ch2, q2, first, early);
}

template <int S>
static bool launch_layer_tma_s(const CodeDev &cd, const DecState &ds, int grid_tiles, int l, float q2, int first,
                               int early, cudaStream_t s) {
    switch (cd.max_dc) {
        case 1: case 2: launch_layer_tma_t<2, S>(cd, ds, grid_tiles, l, q2, first, early, s); return true;
        case 3: launch_layer_tma_t<3, S>(cd, ds, grid_tiles, l, q2, first, early, s); return true;
        case 4: launch_layer_tma_t<4, S>(cd, ds, grid_tiles, l, q2, first, early, s); return true;
        case 5: launch_layer_tma_t<5, S>(cd, ds, grid_tiles, l, q2, first, early, s); return true;
        case 6: launch_layer_tma_t<6, S>(cd, ds, grid_tiles, l, q2, first, early, s); return true;
        case 7: launch_layer_tma_t<7, S>(cd, ds, grid_tiles, l, q2, first, early, s); return true;
        case 8: launch_layer_tma_t<8, S>(cd, ds, grid_tiles, l, q2, first, early, s); return true;
        case 9: launch_layer_tma_t<9, S>(cd, ds, grid_tiles, l, q2, first, early, s); return true;
        case 10: launch_layer_tma_t<10, S>(cd, ds, grid_tiles, l, q2, first, early, s); return true;
        case 11: case 12: launch_layer_tma_t<12, S>(cd, ds, grid_tiles, l, q2, first, early, s); return true;
        default: return false;
    }
}

// TMA-staged layer kernel on/off (CVSR_LAYER_TMA=0: the register-staged k_layer)
static bool layer_tma_enabled() {
    static const int v = [] {
        const char *e = getenv("CVSR_LAYER_TMA");
        return (e && *e) ? atoi(e) : 1;
    }();
    return v != 0;
}

// persistent layer kernel (k_layer_tmap, CVSR_LAYER_PERSIST=1; default off): it removes the
// index-load stalls but costs 14 % more instructions and the kernel is then issue-bound (full-tile
// ncu: 4.38 vs 4.57 TB/s; C4 step 93.8 vs 85.8 ms, C2 50.4 vs 46.2 ms)
static bool layer_persist_enabled() {
    static const int v = [] {
        const char *e = getenv("CVSR_LAYER_PERSIST");
        return (e && *e) ? atoi(e) : 0;
    }();
    return v != 0;
}

// frames per lane of the layered kernels: 2 (64-frame tiles) for k_layer_tma at every supported
// check degree (its registers do not hold whole lines: C4 88.8 vs 100.0 ms per step with one
// frame per lane) and for k_layer up to degree 6; 1 for k_layer above (no spills)
int layer_subs(int32_t max_dc) { return (layer_tma_enabled() || max_dc <= 6) ? 2 : 1; }

template <int S>
static bool launch_layer_s(const CodeDev &cd, const DecState &ds, dim3 grid, int lbeg, int lcnt, float q2,
                           cudaStream_t s) {
    switch (cd.max_dc) {
        case 1: case 2: k_layer<2, S><<<grid, BLOCK, 0, s>>>(cd, ds, lbeg, lcnt, q2); return true;
        case 3: k_layer<3, S><<<grid, BLOCK, 0, s>>>(cd, ds, lbeg, lcnt, q2); return true;
        case 4: k_layer<4, S><<<grid, BLOCK, 0, s>>>(cd, ds, lbeg, lcnt, q2); return true;
        case 5: k_layer<5, S><<<grid, BLOCK, 0, s>>>(cd, ds, lbeg, lcnt, q2); return true;
        case 6: k_layer<6, S><<<grid, BLOCK, 0, s>>>(cd, ds, lbeg, lcnt, q2); return true;
        case 7: k_layer<7, S><<<grid, BLOCK, 0, s>>>(cd, ds, lbeg, lcnt, q2); return true;
        case 8: k_layer<8, S><<<grid, BLOCK, 0, s>>>(cd, ds, lbeg, lcnt, q2); return true;
        case 9: k_layer<9, S><<<grid, BLOCK, 0, s>>>(cd, ds, lbeg, lcnt, q2); return true;
        case 10: k_layer<10, S><<<grid, BLOCK, 0, s>>>(cd, ds, lbeg, lcnt, q2); return true;
        case 11: case 12: k_layer<12, S><<<grid, BLOCK, 0, s>>>(cd, ds, lbeg, lcnt, q2); return true;
        default: return false;
    }
}

bool layered_supported(const CodeDev &cd) { return cd.n_layers > 0 && cd.max_dc <= 12; }

void launch_layer_init(const CodeDev &cd, const DecState &ds, int grid_tiles, cudaStream_t s) {
    if (grid_tiles <= 0) return;
    dim3 grid((cd.n + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, grid_tiles);
    if (ds.subs == 4) k_layer_init<4><<<grid, BLOCK, 0, s>>>(cd, ds);
    else if (ds.subs == 2) k_layer_init<2><<<grid, BLOCK, 0, s>>>(cd, ds);
    else k_layer_init<1><<<grid, BLOCK, 0, s>>>(cd, ds);
}

// all layers of one iteration (returns the number of launches)
// whether launch_layers(first = true) itself treats r as 0 (k_layer_tma); otherwise the caller
// zeroes the message arena before the first iteration
bool layers_zero_first() { return layer_tma_enabled() && !layer_persist_enabled(); }

int launch_layers(const CodeDev &cd, const DecState &ds, int grid_tiles, float qmax, bool first, cudaStream_t s) {
    if (grid_tiles <= 0) return 0;
    const float q2 = qmax * LOG2E;
    const bool tma = layer_tma_enabled();
    const int per_block = tma ? lt_warps(ds.subs) * LT_CH : WARPS_PER_BLOCK * LCPW;
    for (int l = 0; l < cd.n_layers; ++l) {
        const int lbeg = cd.layer_off[l], lcnt = cd.layer_off[l + 1] - lbeg;
        dim3 grid((lcnt + per_block - 1) / per_block, grid_tiles);
        if (tma && layer_persist_enabled() && ds.subs <= 2) {
            if (ds.subs == 2) launch_layer_tmap_s<2>(cd, ds, grid_tiles, lbeg, lcnt, q2, s);
            else launch_layer_tmap_s<1>(cd, ds, grid_tiles, lbeg, lcnt, q2, s);
            continue;
        }
        if (tma) {
            const int f = first ? 1 : 0;
            // the tile lists / messages may be read before the dependency wait only when the
            // previous kernel of the stream is the layer kernel launched just above
            const int early = (l > 0 && layer_pdl_enabled() && layer_early_enabled()) ? 1 : 0;
            if (ds.subs == 4) launch_layer_tma_s<4>(cd, ds, grid_tiles, l, q2, f, early, s);
            else if (ds.subs == 2) launch_layer_tma_s<2>(cd, ds, grid_tiles, l, q2, f, early, s);
            else launch_layer_tma_s<1>(cd, ds, grid_tiles, l, q2, f, early, s);
            continue;
        }
        if (ds.subs == 4) launch_layer_s<4>(cd, ds, grid, lbeg, lcnt, q2, s);
        else if (ds.subs == 2) launch_layer_s<2>(cd, ds, grid, lbeg, lcnt, q2, s);
        else launch_layer_s<1>(cd, ds, grid, lbeg, lcnt, q2, s);
    }
    return cd.n_layers;
}

}  // namespace cvsr
