// Sum-product BP kernels for sm_100a.
//
// Layout ("frame-interleaved arena"): a tile holds 32 S frames (S = 1, 2, 4);
// lane l of a warp owns frames {32 S t + 32 s + l : s < S} as one float/float2/
// float4.  For every edge slot (CSR position) the tile's messages are 128 S
// contiguous bytes, so a warp moves one 128 S-byte line per edge with one
// 4 S-byte access per lane.  Messages are stored IN PLACE: the CN pass reads
// V2C q_e and overwrites it with C2V r_e; the VN pass reads r_e and overwrites
// it with the next q_e.  Arena values are in log2 units (LLR * log2 e): every
// exp/log below is a single MUFU ex2/lg2; conversion happens once at the arena
// boundary (LLR load, trace dumps).  Each warp handles CPW consecutive checks
// so that one row_ptr load serves several rows, and the syndrome test is
// reduced after the message pass so its gathers overlap the message traffic.
// Variables are processed per degree class (one launch per class).
//
// Algorithm (PAPER.md:189 BP decoder, PAPER.md:231 message passes; SURVEY.md
// §8(c) O5 readings A-8 flooding, A-10 V2C clamp, A-12 stopping rule):
//   CN: r_e = (1 - 2 s_c) * BOXPLUS_{e' != e} q_e'.  With t = tanh(|q|/2) the
//       magnitude is 2 atanh(P_e), P_e = prod_{e' != e} t_e'.  With u = e^-|q|,
//       t = (1 - u) / (1 + u) = N / D, and the product is carried as the pair
//       (S, Delta) = (prod D + prod N, prod D - prod N) (up to a common factor):
//         edge e = (1, u_e),   (S1, d1) x (S2, d2) = (S1 S2 + d1 d2, S1 d2 + d1 S2)
//         |r_e| = ln((1 + P_e) / (1 - P_e)) = ln S_e - ln Delta_e   (prefix/suffix)
//       All terms are non-negative, so nothing cancels; 3 MUFU per edge (ex2 and
//       two lg2), no reciprocal and no "total minus own".  A zero message gives
//       S = Delta, r = 0 exactly; a degree-1 check gives Delta = 0, |r| = +inf ->
//       Q_MAX, the empty-fold rule.  (Checks of degree > 12 use the complement
//       form w = 1 - t, c = 1 - prod(1 - w), |r| = ln((2 - c)/c) in cn_check_generic,
//       whose products cannot overflow for any degree.)
//       Sign = syndrome bit XOR the other edges' signs.
//   VN: post_v = L_v + sum_e r_e ; q_e = clamp(post_v - r_e, +-Q_MAX);
//       xhat_v = [post_v < 0].
//   The syndrome test H xhat = s of iteration k-1 is fused into CN pass k.
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"
#include "vec.cuh"

#include "bp_device.cuh"

namespace cvsr {

#ifndef CVSR_CPW
#define CVSR_CPW 4
#endif
constexpr int CPW = CVSR_CPW;  // checks per warp

template <int DC, int S>
__device__ __forceinline__ void cn_check(float *__restrict__ m, int deg, uint32_t sb, uint32_t al, float qmax2) {
    if (!al) return;
    if constexpr (DC >= 5) {
        // degree-2 checks in a code with a large maximum degree (the type-A checks of the
        // MET-style codes, 96 % of their checks): a 2-edge body instead of DC - 2 dummy edges
        if (deg <= 2) {
            cn_check<2, S>(m, deg, sb, al, qmax2);
            return;
        }
    }
    FV<S> q[DC];
#pragma unroll
    for (int k = 0; k < DC; ++k) q[k] = (k < deg) ? ldv<S>(m + (size_t)k * LANES * S) : splat<S>(DUMMY_Q);
    cn_lanes<DC, S>(q, sb, al, qmax2);
#pragma unroll
    for (int k = 0; k < DC; ++k)
        if (k < deg) stv<S>(m + (size_t)k * LANES * S, q[k]);
}

// any degree up to MAX_DC (codes with a check degree > 8): w and suffix
// complements in thread-local arrays
template <int S>
__device__ __noinline__ void cn_check_generic(float *__restrict__ m, int deg, uint32_t sb, uint32_t al, float qmax2) {
    float wl[MAX_DC], sf[MAX_DC + 1];
    for (int s = 0; s < S; ++s) {
        if (!((al >> s) & 1u)) continue;
        uint32_t par = (sb >> s) & 1u;
        for (int k = 0; k < deg; ++k) {
            const float qk = m[(size_t)k * LANES * S + s];
            par ^= sgnbit(qk);
            const float u = ex2f(-fabsf(qk));
            wl[k] = 2.0f * u * rcpf(1.0f + u);
        }
        sf[deg] = 0.0f;
        for (int k = deg - 1; k >= 0; --k) sf[k] = cplus(sf[k + 1], wl[k]);
        float pre = 0.0f;
        for (int k = 0; k < deg; ++k) {
            float *p = m + (size_t)k * LANES * S + s;
            const float c = cplus(pre, sf[k + 1]);
            const float mag = fmaxf(fminf(lg2f((2.0f - c) * rcpf(c)), qmax2), 0.0f);
            pre = cplus(pre, wl[k]);
            *p = (par ^ sgnbit(*p)) ? -mag : mag;
        }
    }
}

// One group of up to CPW consecutive checks of tile t (rp: lane i <= nc holds
// row_ptr[c0 + i]).  Returns this group's unsatisfied-lane words (syndrome test
// of decision k-1), already masked by act.
template <int DCT, int S>
__device__ __forceinline__ uint4 cn_group(const CodeDev &cd, const DecState &ds, int t, const uint4 &act, int c0, int nc,
                                          int rp, int lane, float qmax2, int check_only) {
    int lo[CPW + 1];
#pragma unroll
    for (int i = 0; i <= CPW; ++i) lo[i] = __shfl_sync(FULL, rp, i <= nc ? i : nc);
    const int ebeg = lo[0], eend = lo[nc];
    // this lane's syndrome bits (S per check) for the CN signs; the full syndrome words are
    // re-read (cache hit) for the parity test after the message pass, keeping registers low
    const uint4 *stt = ds.st + (size_t)t * cd.M + c0;
    uint32_t sbits = 0u;
#pragma unroll
    for (int i = 0; i < CPW; ++i)
        if (i < nc) sbits |= lane_act<S>(stt[i], lane) << (i * S);
    // hard-decision word of this lane's edge (first 32 edges), issued before the message pass
    const uint4 *hbt = ds.hb + (size_t)t * cd.n;
    int e = ebeg + lane;
    uint4 h = make_uint4(0u, 0u, 0u, 0u);
    if (e < eend) h = hbt[cd.col_idx[e]];
    if (!check_only) {
        const uint32_t al = lane_act<S>(act, lane);
        float *mt = ds.msg + (size_t)t * cd.E * LANES * S + (size_t)lane * S;
#pragma unroll
        for (int i = 0; i < CPW; ++i) {
            if (i < nc) {
                const int deg = lo[i + 1] - lo[i];
                float *m = mt + (size_t)lo[i] * LANES * S;
                const uint32_t sb = (sbits >> (i * S)) & ((1u << S) - 1u);
                if constexpr (DCT > 0) cn_check<DCT, S>(m, deg, sb, al, qmax2);  // DCT = max_dc >= deg
                else cn_check_generic<S>(m, deg, sb, al, qmax2);
            }
        }
    }
    // syndrome test of decision k-1 (H xhat = s), chunks of 32 edges
    uint4 par[CPW];
#pragma unroll
    for (int i = 0; i < CPW; ++i) par[i] = (i < nc) ? stt[i] : make_uint4(0u, 0u, 0u, 0u);
    for (int e0 = ebeg;;) {
#pragma unroll
        for (int i = 0; i < CPW; ++i) {
            const bool in = (i < nc) && e >= lo[i] && e < lo[i + 1];
            par[i].x ^= __reduce_xor_sync(FULL, in ? h.x : 0u);
            if (S > 1) par[i].y ^= __reduce_xor_sync(FULL, in ? h.y : 0u);
            if (S > 2) {
                par[i].z ^= __reduce_xor_sync(FULL, in ? h.z : 0u);
                par[i].w ^= __reduce_xor_sync(FULL, in ? h.w : 0u);
            }
        }
        e0 += 32;
        if (e0 >= eend) break;
        e = e0 + lane;
        h = make_uint4(0u, 0u, 0u, 0u);
        if (e < eend) h = hbt[cd.col_idx[e]];
    }
    uint4 u = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
        u.x |= par[i].x; u.y |= par[i].y; u.z |= par[i].z; u.w |= par[i].w;
    }
    u.x &= act.x; u.y &= act.y; u.z &= act.z; u.w &= act.w;
    return u;
}

template <int DCT, int S>  // DCT = max check degree (templated body) or 0 = generic
#ifndef CVSR_CN_MINB16
#define CVSR_CN_MINB16 5
#endif
#ifndef CVSR_CN_MINB20
#define CVSR_CN_MINB20 4
#endif
__global__ void __launch_bounds__(BLOCK, (DCT > 0 && DCT * S <= 16) ? CVSR_CN_MINB16
                                         : (DCT > 0 && DCT * S <= 20) ? CVSR_CN_MINB20
                                         : (DCT > 0 && DCT * S <= 24) ? 4
                                                                      : (DCT * S <= 32 ? 3 : 2))
    k_cn(CodeDev cd, DecState ds, float qmax2, int check_only) {
    const int ti = blockIdx.y;
    if (ti >= ds.counts[0]) return;
    const int t = ds.active_list[ti];
    const uint4 act = ds.tile_active[t];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ uint32_t s_unsat[SUBS];
    __shared__ int s_done;
    if (threadIdx.x < SUBS) s_unsat[threadIdx.x] = 0u;
    if (threadIdx.x == 0) s_done = 0;
    __syncthreads();
    const int c0 = (blockIdx.x * WARPS_PER_BLOCK + warp) * CPW;
    const int nc = min(CPW, cd.M - c0);
    if (nc > 0) {
        const int rp = (lane <= nc) ? cd.row_ptr[c0 + lane] : 0;
        const uint4 u = cn_group<DCT, S>(cd, ds, t, act, c0, nc, rp, lane, qmax2, check_only);
        if (lane < S) {
            const uint32_t v = cmpu(u, lane);
            if (v) atomicOr(&s_unsat[lane], v);
        }
    }
    // last warp of the block publishes the block's unsatisfied lanes (no barrier in the hot part)
    __threadfence_block();
    int last = 0;
    if (lane == 0) last = (atomicAdd(&s_done, 1) == WARPS_PER_BLOCK - 1);
    last = __shfl_sync(FULL, last, 0);
    if (last && lane < S) {
        const uint32_t v = atomicOr(&s_unsat[lane], 0u);
        if (v) atomicOr(reinterpret_cast<uint32_t *>(&ds.tile_unsat[t]) + lane, v);
    }
}

// ------------------------------------------------------------------ check nodes, TMA-streamed
//
// The CN pass is a pure stream over the arena: for tile t the messages of checks
// [c0, c0 + CPI) are ONE contiguous span of (row_ptr[c0 + CPI] - row_ptr[c0]) x
// 128 S bytes (CSR slot order, frame-interleaved rows).  A persistent CTA walks
// work items (tile, group of CPI checks); one producer lane streams each item's
// span into a shared-memory ring with cp.async.bulk (TMA bulk copy, mbarrier
// complete_tx), CPI consumer warps take one check each, read their DC lines
// from shared memory, and store C2V straight to global memory.  Loads no longer
// occupy registers, so the number of bytes in flight is set by the ring depth
// instead of by occupancy.  Same arithmetic and stores as k_cn (cn_update), so
// results are bit-identical.

constexpr int CPI = 8;                 // checks per work item = consumer warps per CTA
constexpr int CN_TMA_THREADS = (CPI + 1) * 32;
constexpr int CN_TMA_MAX_STAGES = 8;

// one check of one item: DC lines from the stage, release the stage, update, store
template <int DC, int S>
__device__ __forceinline__ void cn_tma_item(const float *__restrict__ sm, float *__restrict__ m, int deg, uint32_t sb,
                                            uint32_t al, float qmax2, uint64_t *empty_bar, int lane) {
    constexpr int ROW = LANES * S;
    FV<S> q[DC];
    if (al) {
#pragma unroll
        for (int k = 0; k < DC; ++k) q[k] = (k < deg) ? ldv<S>(sm + (size_t)k * ROW) : splat<S>(DUMMY_Q);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_bar);
    if (al) {
        cn_lanes<DC, S>(q, sb, al, qmax2);
#pragma unroll
        for (int k = 0; k < DC; ++k)
            if (k < deg) stv<S>(m + (size_t)k * ROW, q[k]);
    }
}

template <int DCT, int S>
__global__ void __launch_bounds__(CN_TMA_THREADS, 2) k_cn_tma(CodeDev cd, DecState ds, float qmax2, int groups,
                                                           int nstage, int stage_bytes) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + CN_TMA_MAX_STAGES;
    unsigned char *ring = smem + 2 * CN_TMA_MAX_STAGES * sizeof(uint64_t);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_items = ds.counts[0] * groups;
    if (threadIdx.x == 0) {
        for (int i = 0; i < nstage; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], CPI);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    constexpr int ROW = LANES * S;  // floats per edge row of a tile
    if (warp == CPI) {
        // producer warp: the lanes look up 32 items' spans at once, then one lane issues
        // the bulk copies in order (no dependent global load on the issue path)
        int stage = 0;
        uint32_t phase = 0;
        for (int base = blockIdx.x; base < n_items; base += 32 * gridDim.x) {
            const int my = base + lane * gridDim.x;
            int t = 0, e0 = 0, e1 = 0;
            if (my < n_items) {
                t = ds.active_list[my / groups];
                const int c0 = (my % groups) * CPI;
                e0 = cd.row_ptr[c0];
                e1 = cd.row_ptr[min(c0 + CPI, cd.M)];
            }
            const int nb = min(32, (n_items - base + gridDim.x - 1) / gridDim.x);
            for (int j = 0; j < nb; ++j) {
                const int tj = __shfl_sync(FULL, t, j), e0j = __shfl_sync(FULL, e0, j),
                          e1j = __shfl_sync(FULL, e1, j);
                if (lane == 0) {
                    mbar_wait(&empty[stage], phase ^ 1u);
                    const uint32_t bytes = (uint32_t)(e1j - e0j) * ROW * 4u;
                    mbar_arrive_tx(&full[stage], bytes);
                    if (bytes)
                        bulk_g2s(ring + (size_t)stage * stage_bytes, ds.msg + ((size_t)tj * cd.E + e0j) * ROW, bytes,
                                 &full[stage]);
                }
                __syncwarp();
                if (++stage == nstage) { stage = 0; phase ^= 1u; }
            }
        }
        return;
    }
    // consumers: warp w owns check c0 + w of every item.  The per-item metadata is
    // software-pipelined two items deep: A = (tile, row range) for item i + 2,
    // B = (hard-decision words, syndrome word, active mask) for item i + 1, so the
    // dependent gather chain row_ptr -> col_idx -> hb overlaps the compute of item i.
    struct MetaA { int t, lo, deg, e0; bool valid; };
    struct MetaB { MetaA a; uint4 h, stc, act; };
    auto load_a = [&](int it) {
        MetaA m{0, 0, 0, 0, false};
        if (it < n_items) {
            m.t = ds.active_list[it / groups];
            const int c0 = (it % groups) * CPI, c = c0 + warp;
            m.e0 = cd.row_ptr[c0];
            if (c < cd.M) {
                m.valid = true;
                m.lo = cd.row_ptr[c];
                m.deg = cd.row_ptr[c + 1] - m.lo;
            }
        }
        return m;
    };
    auto load_b = [&](const MetaA &a, int it) {
        MetaB m;
        m.a = a;
        m.h = make_uint4(0u, 0u, 0u, 0u);
        m.stc = make_uint4(0u, 0u, 0u, 0u);
        m.act = make_uint4(0u, 0u, 0u, 0u);
        if (it < n_items) {
            m.act = ds.tile_active[a.t];
            if (a.valid) {
                const int c = (it % groups) * CPI + warp;
                m.stc = ds.st[(size_t)a.t * cd.M + c];
                if (lane < a.deg) m.h = ds.hb[(size_t)a.t * cd.n + cd.col_idx[a.lo + lane]];
            }
        }
        return m;
    };
    int stage = 0;
    uint32_t phase = 0;
    int pub_t = -1;
    uint32_t pub = 0u;  // unsatisfied bits of tile pub_t already published by this warp (lane s < S)
    const int G = gridDim.x;
    MetaB cur = load_b(load_a(blockIdx.x), blockIdx.x);
    MetaA nxt = load_a(blockIdx.x + G);
    for (int it = blockIdx.x; it < n_items; it += G) {
        const MetaB b_next = load_b(nxt, it + G);
        const MetaA a_next = load_a(it + 2 * G);
        const int t = cur.a.t, lo = cur.a.lo, deg = cur.a.deg;
        const bool have = cur.a.valid;
        mbar_wait(&full[stage], phase);
        const uint32_t al = have ? lane_act<S>(cur.act, lane) : 0u;
        {
            const float *sm = reinterpret_cast<const float *>(ring + (size_t)stage * stage_bytes) +
                              (size_t)(lo - cur.a.e0) * ROW + lane * S;
            float *m = ds.msg + ((size_t)t * cd.E + lo) * ROW + lane * S;
            const uint32_t sb = lane_act<S>(cur.stc, lane);
            cn_tma_item<DCT, S>(sm, m, deg, sb, al, qmax2, &empty[stage], lane);
        }
        if (++stage == nstage) { stage = 0; phase ^= 1u; }
        // parity of the check under decision k-1, masked by the active frames
        uint4 par = cur.stc;
        par.x ^= __reduce_xor_sync(FULL, cur.h.x);
        if (S > 1) par.y ^= __reduce_xor_sync(FULL, cur.h.y);
        if (S > 2) {
            par.z ^= __reduce_xor_sync(FULL, cur.h.z);
            par.w ^= __reduce_xor_sync(FULL, cur.h.w);
        }
        if (t != pub_t) { pub_t = t; pub = 0u; }
        if (lane < S && have) {
            const uint32_t v = cmpu(par, lane) & cmpu(cur.act, lane) & ~pub;
            if (v) {
                atomicOr(reinterpret_cast<uint32_t *>(&ds.tile_unsat[t]) + lane, v);
                pub |= v;
            }
        }
        cur = b_next;
        nxt = a_next;
    }
}

// ------------------------------------------------------------------ variable nodes
//
// Per degree class: every warp takes VPW variables of degree DV, loads all
// their slot indices with one coalesced load (class-major slot table), then
// issues all VPW x (DV + 1) line loads before using any of them.

template <int S>
__device__ __forceinline__ void vn_finish(const DecState &ds, const CodeDev &cd, int t, int v, const FV<S> &post,
                                          const uint4 &act, uint32_t any, int lane, float *post_dbg) {
    // hard decisions (frames retired by the preceding status pass were copied out already)
    uint32_t wd[SUBS] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int s = 0; s < S; ++s) wd[s] = __ballot_sync(FULL, post.c[s] < 0.0f) & cmpu(act, s);
    if (lane == 0) ds.hb[(size_t)t * cd.n + v] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    if (post_dbg && any) stv<S>(post_dbg + (((size_t)t * cd.n + v) * LANES + lane) * S, post);
}

// one block-chunk of a variable-degree class for tile t (chunk = block index within the class)
template <int DV, int VPW_, bool FIRST, int S>
__device__ __forceinline__ void vn_chunk(const CodeDev &cd, const DecState &ds, int cls, int t, const uint4 &act,
                                         int chunk, float qmax2, float *post_dbg) {
    // the warp's variables and slot indices are fetched with one load per lane
    static_assert(VPW_ <= LANES && VPW_ * DV <= LANES, "VPW x DV slot indices must fit one warp load");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int w0 = (chunk * WARPS_PER_BLOCK + warp) * VPW_;
    const int cnt = cd.vc_cnt[cls];
    const int nv = min(VPW_, cnt - w0);
    if (nv <= 0) return;
    const int vv = (lane < nv) ? cd.vc_vars[cd.vc_off[cls] + w0 + lane] : 0;
    const int sl = (lane < nv * DV) ? cd.vc_slots[cd.vc_soff[cls] + (int64_t)w0 * DV + lane] : 0;
    const uint32_t any = lane_act<S>(act, lane);
    int v[VPW_];
    FV<S> Lv[VPW_];
#pragma unroll
    for (int i = 0; i < VPW_; ++i) {
        v[i] = __shfl_sync(FULL, vv, i);
        Lv[i] = (i < nv && any) ? ldv<S>(ds.L + (((size_t)t * cd.n + v[i]) * LANES + lane) * S) : splat<S>(0.0f);
    }
    float *mt = ds.msg + (size_t)t * cd.E * LANES * S + (size_t)lane * S;
    int slot[VPW_][DV];
#pragma unroll
    for (int i = 0; i < VPW_; ++i)
#pragma unroll
        for (int k = 0; k < DV; ++k) slot[i][k] = __shfl_sync(FULL, sl, i * DV + k);
    if (FIRST) {
#pragma unroll
        for (int i = 0; i < VPW_; ++i) {
            if (i >= nv) break;
            if (any) {
                FV<S> q;
#pragma unroll
                for (int s = 0; s < S; ++s) q.c[s] = clampf(Lv[i].c[s], qmax2);
#pragma unroll
                for (int k = 0; k < DV; ++k) stv<S>(mt + (size_t)slot[i][k] * LANES * S, q);
            }
            vn_finish<S>(ds, cd, t, v[i], Lv[i], act, any, lane, post_dbg);
        }
        return;
    }
    FV<S> r[VPW_][DV];
#pragma unroll
    for (int i = 0; i < VPW_; ++i)
#pragma unroll
        for (int k = 0; k < DV; ++k)
            r[i][k] = (i < nv && any) ? ldv<S>(mt + (size_t)slot[i][k] * LANES * S) : splat<S>(0.0f);
#pragma unroll
    for (int i = 0; i < VPW_; ++i) {
        if (i >= nv) break;
        FV<S> post = Lv[i];
#pragma unroll
        for (int k = 0; k < DV; ++k)
#pragma unroll
            for (int s = 0; s < S; ++s) post.c[s] += r[i][k].c[s];
        if (any) {
#pragma unroll
            for (int k = 0; k < DV; ++k) {
                FV<S> q;
#pragma unroll
                for (int s = 0; s < S; ++s) q.c[s] = clampf(post.c[s] - r[i][k].c[s], qmax2);
                stv<S>(mt + (size_t)slot[i][k] * LANES * S, q);
            }
        }
        vn_finish<S>(ds, cd, t, v[i], post, act, any, lane, post_dbg);
    }
}

template <int DV, int VPW_, bool FIRST, int S>
#ifndef CVSR_VN_MINB
#define CVSR_VN_MINB 3
#endif
__global__ void __launch_bounds__(BLOCK, CVSR_VN_MINB) k_vn_cls(CodeDev cd, DecState ds, int cls, float qmax2,
                                                     float *post_dbg) {
    const int ti = blockIdx.y;
    if (ti >= ds.counts[0]) return;
    const int t = ds.active_list[ti];
    const uint4 act = ds.tile_active[t];
    vn_chunk<DV, VPW_, FIRST, S>(cd, ds, cls, t, act, blockIdx.x, qmax2, post_dbg);
}

// any degree: one variable per warp, slots read per edge (mixed / large-degree classes)
template <bool FIRST, int S>
__device__ __noinline__ void vn_generic_chunk(const CodeDev &cd, const DecState &ds, int cls, int t, uint4 act,
                                              int chunk, float qmax2, float *post_dbg) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int w = chunk * WARPS_PER_BLOCK + warp;
    if (w >= cd.vc_cnt[cls]) return;
    const int v = cd.vc_vars[cd.vc_off[cls] + w];
    const int beg = cd.col_ptr[v], deg = cd.col_ptr[v + 1] - beg;
    const int32_t *slots = cd.csc_slot + beg;
    const uint32_t any = lane_act<S>(act, lane);
    float *mt = ds.msg + (size_t)t * cd.E * LANES * S + (size_t)lane * S;
    FV<S> post = any ? ldv<S>(ds.L + (((size_t)t * cd.n + v) * LANES + lane) * S) : splat<S>(0.0f);
    if (any) {
        if (!FIRST)
            for (int k = 0; k < deg; ++k) {
                const FV<S> r = ldv<S>(mt + (size_t)slots[k] * LANES * S);
#pragma unroll
                for (int s = 0; s < S; ++s) post.c[s] += r.c[s];
            }
        for (int k = 0; k < deg; ++k) {
            float *p = mt + (size_t)slots[k] * LANES * S;
            const FV<S> r = FIRST ? splat<S>(0.0f) : ldv<S>(p);
            FV<S> q;
#pragma unroll
            for (int s = 0; s < S; ++s) q.c[s] = clampf(post.c[s] - r.c[s], qmax2);
            stv<S>(p, q);
        }
    }
    vn_finish<S>(ds, cd, t, v, post, act, any, lane, post_dbg);
}

template <bool FIRST, int S>
__global__ void __launch_bounds__(BLOCK) k_vn_generic(CodeDev cd, DecState ds, int cls, float qmax2,
                                                      float *post_dbg) {
    const int ti = blockIdx.y;
    if (ti >= ds.counts[0]) return;
    const int t = ds.active_list[ti];
    vn_generic_chunk<FIRST, S>(cd, ds, cls, t, ds.tile_active[t], blockIdx.x, qmax2, post_dbg);
}

// ------------------------------------------------------------------ scheduling

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

__device__ __forceinline__ void mark_frames(const DecState &ds, int t, int s, uint32_t bits, int32_t it, uint8_t cv) {
    while (bits) {
        const int l = __ffs(bits) - 1;
        bits &= bits - 1;
        const int slot = t * ds.tile_frames + s * LANES + l;
        const int f = ds.slot_frame ? ds.slot_frame[slot] : slot;
        ds.iters[f] = it;
        ds.conv[f] = cv;
    }
}

// Convergence bookkeeping after CN pass k (which tested decision k-1).
// Single block; loops over tiles.  final_pass: k = max_iter + 1.
// k < 0: the iteration number is the device counter counts[3] + 1 (CUDA-graph replays,
// where launch arguments are frozen); every call stores its iteration in counts[3].
__global__ void __launch_bounds__(1024) k_status(DecState ds, int k_arg, int max_iter, int final_pass,
                                                 int32_t *host_counts) {
    __shared__ int s_warp[33];
    __shared__ int s_lanes;
    const int k = k_arg >= 0 ? k_arg : ds.counts[3] + 1;
    if (threadIdx.x == 0) s_lanes = 0;
    __syncthreads();
    int n_act = 0, n_ret = 0;
    for (int t0 = 0; t0 < ds.tiles; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        uint4 rem = make_uint4(0u, 0u, 0u, 0u), newly = make_uint4(0u, 0u, 0u, 0u);
        if (t < ds.tiles) {
            const uint4 a = ds.tile_active[t];
            if (a.x | a.y | a.z | a.w) {
                const uint4 u = ds.tile_unsat[t];
                ds.tile_unsat[t] = make_uint4(0u, 0u, 0u, 0u);
                for (int s = 0; s < ds.subs; ++s) {
                    const uint32_t as = cmpu(a, s), us = cmpu(u, s);
                    mark_frames(ds, t, s, as & ~us, k - 1, 1);
                    if (final_pass) mark_frames(ds, t, s, as & us, max_iter, 0);
                }
                if (final_pass) {
                    newly = a;
                } else {
                    newly = make_uint4(a.x & ~u.x, a.y & ~u.y, a.z & ~u.z, a.w & ~u.w);
                    rem = make_uint4(a.x & u.x, a.y & u.y, a.z & u.z, a.w & u.w);
                }
                ds.tile_active[t] = rem;
            }
            ds.tile_newly[t] = newly;
        }
        const bool ra = (rem.x | rem.y | rem.z | rem.w) != 0u;
        const bool rn = (newly.x | newly.y | newly.z | newly.w) != 0u;
        int tot;
        const int pa = block_scan_flag(ra, s_warp, &tot);
        if (ra) ds.active_list[n_act + pa] = t;
        n_act += tot;
        const int pr = block_scan_flag(rn, s_warp, &tot);
        if (rn) ds.retire_list[n_ret + pr] = t;
        n_ret += tot;
        int v = __popc(rem.x) + __popc(rem.y) + __popc(rem.z) + __popc(rem.w);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_lanes, v);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ds.counts[0] = n_act;
        ds.counts[1] = n_ret;
        ds.counts[2] = s_lanes;
        ds.counts[3] = k;
        if (host_counts) {
            volatile int32_t *h = host_counts;
            h[0] = n_act;
            h[1] = n_ret;
            h[2] = s_lanes;
        }
    }
}

// ------------------------------------------------------------------ fused iteration
//
// One persistent launch per BP iteration: blocks grab work items in order
// [CN chunks of tile t0][VN chunks of t0][CN of t1][VN of t1]...; the last CN
// block of a tile performs that tile's convergence bookkeeping (status) and
// releases the tile; VN blocks of the tile wait for the release.  Processing
// one tile's VN right after its CN means the tile's freshly written C2V lines
// are read back from L2 and overwritten in L2 by the next V2C values, so most
// of the CN -> VN hand-off never reaches HBM (tiles are sized to fit L2).
// Items are grabbed in order and a VN block only waits for CN items that were
// grabbed earlier by running blocks, so the wait always terminates.

__host__ __device__ constexpr int vpw_for(int d, int S) {
    return d == 1 ? 6 : d == 2 ? 4 : (d <= 4 ? (S < 4 ? 4 : 2) : 4 / S);
}

template <bool FIRST, int S>
__device__ __forceinline__ void vn_dispatch(const CodeDev &cd, const DecState &ds, int c, int t, const uint4 &act,
                                            int chunk, float qmax2, float *post_dbg) {
    switch (cd.vc_deg[c]) {
        case 1: vn_chunk<1, vpw_for(1, S), FIRST, S>(cd, ds, c, t, act, chunk, qmax2, post_dbg); break;
        case 2: vn_chunk<2, vpw_for(2, S), FIRST, S>(cd, ds, c, t, act, chunk, qmax2, post_dbg); break;
        case 3: vn_chunk<3, vpw_for(3, S), FIRST, S>(cd, ds, c, t, act, chunk, qmax2, post_dbg); break;
        case 4: vn_chunk<4, vpw_for(4, S), FIRST, S>(cd, ds, c, t, act, chunk, qmax2, post_dbg); break;
        case 5: vn_chunk<5, vpw_for(5, S), FIRST, S>(cd, ds, c, t, act, chunk, qmax2, post_dbg); break;
        case 6: vn_chunk<6, vpw_for(6, S), FIRST, S>(cd, ds, c, t, act, chunk, qmax2, post_dbg); break;
        case 7: vn_chunk<7, vpw_for(7, S), FIRST, S>(cd, ds, c, t, act, chunk, qmax2, post_dbg); break;
        case 8: vn_chunk<8, vpw_for(8, S), FIRST, S>(cd, ds, c, t, act, chunk, qmax2, post_dbg); break;
        default: vn_generic_chunk<FIRST, S>(cd, ds, c, t, act, chunk, qmax2, post_dbg); break;
    }
}

template <int DCT, int S>
__global__ void __launch_bounds__(BLOCK, 3) k_iter(CodeDev cd, DecState dsc, DecState dsv, FusedPlan plan, int k,
                                                   float qmax2) {
    __shared__ int s_item, s_last;
    __shared__ uint32_t s_unsat[SUBS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_act = dsc.counts[0];
    const int n_cn = plan.n_cn, n_vn = plan.items_per_tile - plan.n_cn;
    const int n_items = n_act * plan.items_per_tile;
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(dsc.fused_work, 1);
        if (threadIdx.x < SUBS) s_unsat[threadIdx.x] = 0u;
        __syncthreads();
        const int item = s_item;
        if (item >= n_items) break;
        // phase 0: CN(t_0); phase j in [1, n_act): CN(t_j) then VN(t_{j-1}); phase n_act: VN(t_{n_act-1}).
        // A tile's VN items come one CN phase after its CN items, so they rarely wait.
        int ti, r;
        bool is_cn;
        if (item < n_cn) {
            ti = 0;
            r = item;
            is_cn = true;
        } else {
            const int i2 = item - n_cn;
            const int j = i2 / (n_cn + n_vn) + 1;
            r = i2 - (j - 1) * (n_cn + n_vn);
            if (j < n_act && r < n_cn) {
                ti = j;
                is_cn = true;
            } else {
                ti = j - 1;
                r = (j < n_act) ? r - n_cn : r;
                is_cn = false;
            }
        }
        const int t = dsc.active_list[ti];
        if (is_cn) {
            const uint4 act = __ldcg(&dsc.tile_active[t]);
            const int c0 = (r * WARPS_PER_BLOCK + warp) * CPW;
            const int nc = min(CPW, cd.M - c0);
            if (nc > 0) {
                const int rp = (lane <= nc) ? cd.row_ptr[c0 + lane] : 0;
                const uint4 u = cn_group<DCT, S>(cd, dsc, t, act, c0, nc, rp, lane, qmax2, 0);
                if (lane < S) {
                    const uint32_t v = cmpu(u, lane);
                    if (v) atomicOr(&s_unsat[lane], v);
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
#pragma unroll
                for (int q = 0; q < S; ++q)
                    if (s_unsat[q]) atomicOr(reinterpret_cast<uint32_t *>(&dsc.tile_unsat[t]) + q, s_unsat[q]);
                __threadfence();
                s_last = (atomicAdd(&dsc.cn_done[t], 1) == plan.n_cn - 1);
            }
            __syncthreads();
            if (s_last) {
                // status of tile t: frames whose decision k-1 satisfied every check stop (D = k-1)
                __threadfence();
                const uint4 a = __ldcg(&dsc.tile_active[t]);
                const uint4 u = __ldcg(&dsc.tile_unsat[t]);
                if (threadIdx.x < LANES * S) {
                    const int q = threadIdx.x >> 5;
                    if (((cmpu(a, q) & ~cmpu(u, q)) >> lane) & 1u) {
                        const int f = t * dsc.tile_frames + q * LANES + lane;
                        dsc.iters[f] = k - 1;
                        dsc.conv[f] = 1;
                    }
                }
                if (threadIdx.x == 0) {
                    dsc.tile_newly[t] = make_uint4(a.x & ~u.x, a.y & ~u.y, a.z & ~u.z, a.w & ~u.w);
                    dsc.tile_active[t] = make_uint4(a.x & u.x, a.y & u.y, a.z & u.z, a.w & u.w);
                    dsc.tile_unsat[t] = make_uint4(0u, 0u, 0u, 0u);
                    __threadfence();
                    atomicExch(&dsc.cn_ready[t], k);
                }
            }
        } else {
            int c = 0;
            while (c < plan.n_cls - 1 && r >= plan.cls_chunks[c]) r -= plan.cls_chunks[c++];
            if (threadIdx.x == 0) {
                while (atomicAdd(&dsv.cn_ready[t], 0) != k) __nanosleep(64);
                __threadfence();
            }
            __syncthreads();
            const uint4 act = __ldcg(&dsv.tile_active[t]);
            if (act.x | act.y | act.z | act.w) vn_dispatch<false, S>(cd, dsv, c, t, act, r, qmax2, nullptr);
        }
        __syncthreads();
    }
}

// after a fused iteration: active / retire lists of the processed tiles, counters reset
__global__ void __launch_bounds__(1024) k_list(DecState ds, int32_t *host_counts) {
    __shared__ int s_warp[33];
    __shared__ int s_lanes;
    if (threadIdx.x == 0) s_lanes = 0;
    __syncthreads();
    int n_act = 0, n_ret = 0;
    for (int t0 = 0; t0 < ds.tiles; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        uint4 rem = make_uint4(0u, 0u, 0u, 0u), newly = make_uint4(0u, 0u, 0u, 0u);
        if (t < ds.tiles) {
            if (ds.cn_done[t] > 0) {  // processed this iteration
                rem = ds.tile_active[t];
                newly = ds.tile_newly[t];
                ds.cn_done[t] = 0;
            } else {
                ds.tile_newly[t] = make_uint4(0u, 0u, 0u, 0u);
            }
        }
        const bool ra = (rem.x | rem.y | rem.z | rem.w) != 0u;
        const bool rn = (newly.x | newly.y | newly.z | newly.w) != 0u;
        int tot;
        const int pa = block_scan_flag(ra, s_warp, &tot);
        if (ra) ds.active_list[n_act + pa] = t;
        n_act += tot;
        const int pr = block_scan_flag(rn, s_warp, &tot);
        if (rn) ds.retire_list[n_ret + pr] = t;
        n_ret += tot;
        int v = __popc(rem.x) + __popc(rem.y) + __popc(rem.z) + __popc(rem.w);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_lanes, v);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ds.counts[0] = n_act;
        ds.counts[1] = n_ret;
        ds.counts[2] = s_lanes;
        *ds.fused_work = 0;
        if (host_counts) {
            volatile int32_t *h = host_counts;
            h[0] = n_act;
            h[1] = n_ret;
            h[2] = s_lanes;
        }
    }
}

// Write the hard decisions of retired frames as packed bits (32x32 bit transposes by ballots).
// Grid-stride over (retired tile, block of WARPS_PER_BLOCK words): most iterations retire no tile,
// and a grid sized for every tile's words was ~8k blocks that only read the count and exit.
__global__ void __launch_bounds__(BLOCK) k_retire(DecState ds, int32_t n, uint32_t *bits_out) {
    const int nr = ds.counts[1];
    const int Wn = words_of(n);
    const int nwb = (Wn + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t item = blockIdx.x; item < (int64_t)nr * nwb; item += gridDim.x) {
        const int ti = (int)(item / nwb);
        const int w = (int)(item - (int64_t)ti * nwb) * WARPS_PER_BLOCK + warp;
        if (w >= Wn) continue;  // warp-uniform
        const int t = ds.retire_list[ti];
        const uint4 newly = ds.tile_newly[t];
        const int v = w * 32 + lane;
        const uint4 word = (v < n) ? ds.hb[(size_t)t * n + v] : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int s = 0; s < SUBS; ++s) {
            const uint32_t ns = cmpu(newly, s);
            if (!ns) continue;
            // lane i holds bit f = decision of variable 32 w + i for frame lane f; lane f needs the
            // word over the 32 variables: a 32 x 32 bit transpose (5 shuffle rounds of block swaps)
            const uint32_t mine = transpose32(cmpu(word, s), lane);
            const int slot = t * ds.tile_frames + s * LANES + lane;
            const int frame = ds.slot_frame ? ds.slot_frame[slot] : slot;
            if (((ns >> lane) & 1u) && frame >= 0 && frame < ds.frames) bits_out[(size_t)frame * Wn + w] = mine;
        }
    }
}

// natural [F][rows] -> interleaved [tiles][rows][32][S] (zero-fill missing frames), times scale
template <int S>
__global__ void __launch_bounds__(256) k_to_interleaved(const float *__restrict__ src, float *__restrict__ dst,
                                                        int32_t F, int64_t rows, float scale) {
    __shared__ float sm[LANES * S][33];
    const int t = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int fl = ty; fl < LANES * S; fl += 8) {
        const int f = t * LANES * S + fl;
        const int64_t r = r0 + tx;
        sm[fl][tx] = (f < F && r < rows) ? src[(size_t)f * rows + r] * scale : 0.0f;
    }
    __syncthreads();
    for (int rl = ty; rl < 32; rl += 8) {
        const int64_t r = r0 + rl;
        if (r < rows) {
            FV<S> v;
#pragma unroll
            for (int s = 0; s < S; ++s) v.c[s] = sm[s * LANES + tx][rl];
            stv<S>(dst + (((size_t)t * rows + r) * LANES + tx) * S, v);
        }
    }
}

// interleaved [tiles][rows][32][S] -> natural [F][rows], times scale
template <int S>
__global__ void __launch_bounds__(256) k_from_interleaved(const float *__restrict__ src, float *__restrict__ dst,
                                                          int32_t F, int64_t rows, float scale) {
    __shared__ float sm[LANES * S][33];
    const int t = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int rl = ty; rl < 32; rl += 8) {
        const int64_t r = r0 + rl;
        const FV<S> v = (r < rows) ? ldv<S>(src + (((size_t)t * rows + r) * LANES + tx) * S) : splat<S>(0.0f);
#pragma unroll
        for (int s = 0; s < S; ++s) sm[s * LANES + tx][rl] = v.c[s];
    }
    __syncthreads();
    for (int fl = ty; fl < LANES * S; fl += 8) {
        const int f = t * LANES * S + fl;
        const int64_t r = r0 + tx;
        if (f < F && r < rows) dst[(size_t)f * rows + r] = sm[fl][tx] * scale;
    }
}

// public syndrome [F][Wm] -> per-tile lane-bit words st[t][c] (uint4 over sub-tiles)
__global__ void __launch_bounds__(BLOCK) k_synd_transpose(const uint32_t *__restrict__ synd, int32_t F, int32_t M,
                                                           int subs, uint4 *__restrict__ st,
                                                           const int32_t *__restrict__ pos) {
    const int t = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Wm = words_of(M);
    const int w = blockIdx.x * WARPS_PER_BLOCK + warp;
    if (w >= Wm) return;
    uint32_t mine[SUBS] = {0u, 0u, 0u, 0u};
    for (int s = 0; s < subs; ++s) {
        const int f = t * LANES * subs + s * LANES + lane;
        const uint32_t word = (f < F) ? synd[(size_t)f * Wm + w] : 0u;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint32_t b = __ballot_sync(FULL, (word >> k) & 1u);
            if (lane == k) mine[s] = b;
        }
    }
    const int c = w * 32 + lane;
    if (c < M) st[(size_t)t * M + (pos ? pos[c] : c)] = make_uint4(mine[0], mine[1], mine[2], mine[3]);
}

// initial tile state: active frames = valid frames (& alive mask if given)
__global__ void k_init_tiles(DecState ds, const uint8_t *__restrict__ alive) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ds.tiles) return;
    uint32_t a[SUBS] = {0u, 0u, 0u, 0u};
    for (int s = 0; s < ds.subs; ++s) {
        for (int l = 0; l < LANES; ++l) {
            const int f = t * ds.tile_frames + s * LANES + l;
            if (f < ds.frames && (!alive || alive[f])) a[s] |= 1u << l;
        }
    }
    ds.tile_active[t] = make_uint4(a[0], a[1], a[2], a[3]);
    ds.tile_unsat[t] = make_uint4(0u, 0u, 0u, 0u);
    ds.tile_newly[t] = make_uint4(0u, 0u, 0u, 0u);
    ds.active_list[t] = t;
    if (ds.cn_done) {
        ds.cn_done[t] = 0;
        ds.cn_ready[t] = -1;
        if (t == 0) *ds.fused_work = 0;
    }
}

__global__ void k_set_counts(DecState ds, int32_t n_active) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        ds.counts[0] = n_active;
        ds.counts[1] = 0;
        ds.counts[2] = 0;
        ds.counts[8] = 0;  // work-item counter of the persistent layer kernel (k_layer_tmap)
        ds.counts[9] = 0;  // its exit counter
    }
}

// ------------------------------------------------------------------ frame compaction
//
// When most frames of the active tiles have converged, the still-active frames
// are moved densely into a second arena (same layout), so the remaining
// iterations touch fewer tiles and sectors.  All active frames are at the same
// iteration (flooding), so a move carries only their state: messages, LLRs,
// syndrome bits and current hard decisions; slot_frame keeps the frame ids.

// Single block: rank the active slots of the source tiles (in slot order) and
// set up the destination tiles: dst_src[r] = source slot of destination slot r.
__global__ void __launch_bounds__(1024) k_compact_plan(DecState src, DecState dst, int32_t *dst_src,
                                                       int32_t *host_counts) {
    __shared__ int s_warp[33];
    const int T = src.tile_frames;
    const int n_act_tiles = src.counts[0];
    int base = 0;
    for (int i0 = 0; i0 < n_act_tiles * T; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        bool a = false;
        int slot = 0;
        if (i < n_act_tiles * T) {
            const int t = src.active_list[i / T];
            const int r = i % T;
            slot = t * T + r;
            a = (cmpu(src.tile_active[t], r / LANES) >> (r % LANES)) & 1u;
        }
        int tot;
        const int rk = block_scan_flag(a, s_warp, &tot);
        if (a) {
            dst_src[base + rk] = slot;
            dst.slot_frame[base + rk] = src.slot_frame ? src.slot_frame[slot] : slot;
        }
        base += tot;
    }
    __syncthreads();
    const int A = base, tiles_new = (A + T - 1) / T;
    for (int r = A + threadIdx.x; r < tiles_new * T; r += blockDim.x) {
        dst_src[r] = -1;
        dst.slot_frame[r] = -1;
    }
    // every tile of the arena gets fresh state: tiles past tiles_new become empty
    for (int t = threadIdx.x; t < src.tiles; t += blockDim.x) {
        uint32_t m[SUBS] = {0u, 0u, 0u, 0u};
        for (int q = 0; q < src.subs; ++q) {
            const int lo = t * T + q * LANES;
            const int cnt = min(max(A - lo, 0), LANES);
            m[q] = cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u);
        }
        dst.tile_active[t] = make_uint4(m[0], m[1], m[2], m[3]);
        dst.tile_unsat[t] = make_uint4(0u, 0u, 0u, 0u);
        dst.tile_newly[t] = make_uint4(0u, 0u, 0u, 0u);
        if (t < tiles_new) dst.active_list[t] = t;
    }
    if (threadIdx.x == 0) {
        dst.counts[0] = tiles_new;
        dst.counts[1] = 0;
        dst.counts[2] = A;
        if (host_counts) {
            volatile int32_t *h = host_counts;
            h[0] = tiles_new;
            h[1] = 0;
            h[2] = A;
        }
    }
}

// dst[t'][row][lane][s] = src[slot dst_src(t', s, lane)] for float rows (messages, LLRs)
// A warp moves CR consecutive rows of destination tile t; the slot map of its lanes
// (S source slots each) is loaded once and reused for every row.
#ifndef CVSR_CR_ROWS
#define CVSR_CR_ROWS 8
#endif
constexpr int CR_ROWS = CVSR_CR_ROWS;  // rows per warp, float rows

template <int S>
__global__ void __launch_bounds__(256) k_compact_rows(const float *__restrict__ src, float *__restrict__ dst,
                                                      int64_t rows, const int32_t *__restrict__ dst_src,
                                                      const int32_t *__restrict__ counts) {
    const int t = blockIdx.y;
    if (t >= counts[0]) return;
    const int lane = threadIdx.x & 31;
    const int64_t r0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * CR_ROWS;
    if (r0 >= rows) return;
    size_t base[S];  // source element offset of row 0 for each of this lane's S slots, or SIZE_MAX
#pragma unroll
    for (int q = 0; q < S; ++q) {
        const int so = dst_src[t * LANES * S + q * LANES + lane];
        base[q] = ~size_t(0);
        if (so >= 0) {
            const int st = so / (LANES * S), rem = so % (LANES * S);
            base[q] = ((size_t)st * rows * LANES + (rem % LANES)) * S + rem / LANES;
        }
    }
    const int nr = (int)(rows - r0 < CR_ROWS ? rows - r0 : CR_ROWS);
#pragma unroll 4
    for (int i = 0; i < nr; ++i) {
        const int64_t r = r0 + i;
        FV<S> v;
#pragma unroll
        for (int q = 0; q < S; ++q) v.c[q] = base[q] != ~size_t(0) ? src[base[q] + (size_t)r * LANES * S] : 0.0f;
        stv<S>(dst + (((size_t)t * rows + r) * LANES + lane) * S, v);
    }
}

// dst[t'][row] bit (s, lane) = src bit of slot dst_src(t', s, lane) for uint4 bit rows (st, hb).
// Thread per row (coalesced uint4 loads and stores); the tile's slot map sits in shared
// memory and the source word is re-loaded only when the source tile changes.
__global__ void __launch_bounds__(256) k_compact_bits(const uint4 *__restrict__ src, uint4 *__restrict__ dst,
                                                      int64_t rows, int subs, const int32_t *__restrict__ dst_src,
                                                      const int32_t *__restrict__ counts) {
    const int t = blockIdx.y;
    if (t >= counts[0]) return;
    __shared__ int smap[LANES * SUBS];
    const int slots = LANES * subs;
    for (int i = threadIdx.x; i < slots; i += blockDim.x) smap[i] = dst_src[t * slots + i];
    __syncthreads();
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        uint32_t w[SUBS] = {0u, 0u, 0u, 0u};
        int cur_t = -1;
        uint4 cur = make_uint4(0u, 0u, 0u, 0u);
        for (int i = 0; i < slots; ++i) {
            const int so = smap[i];
            if (so < 0) continue;
            const int st = so / slots, rem = so - st * slots;
            if (st != cur_t) {
                cur = src[(size_t)st * rows + r];
                cur_t = st;
            }
            w[i / LANES] |= ((cmpu(cur, rem / LANES) >> (rem % LANES)) & 1u) << (i % LANES);
        }
        dst[(size_t)t * rows + r] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// ---------------------------------------------------------------- shared-memory decoder
//
// Small codes (all E messages and n LLRs of a frame fit in shared memory): one CTA
// decodes one frame for all its iterations, so no message crosses HBM after the
// LLRs are read (the on-chip decoder for small N_R).  The
// arithmetic is that of the interleaved kernels, in the same order (cn_update on
// the same dummy-padded edge lists, variable sums in CSC slot order, the same
// clamps), so results are bit-identical to the interleaved path; the iteration
// bookkeeping follows k_status (a frame whose decision k-1 satisfies H x = s at
// pass k stops with D = k-1; after max_iter it fails with D = max_iter).

__device__ __forceinline__ uint32_t sbit(const uint32_t *w, int i) { return (w[i >> 5] >> (i & 31)) & 1u; }

template <int DCT>
__global__ void __launch_bounds__(512) k_decode_smem(CodeDev cd, DecState ds, int max_iter, float qmax2,
                                                     uint32_t *__restrict__ bits_out) {
    extern __shared__ float smem_f[];
    const int f = blockIdx.x;
    const int T = ds.tile_frames, S = ds.subs;
    const int t = f / T, r = f % T, sub = r / LANES, l = r % LANES;
    if (!((cmpu(ds.tile_active[t], sub) >> l) & 1u)) return;  // frame stopped in an earlier slice
    const int n = cd.n, M = cd.M, E = cd.E;
    const int Wn = words_of(n), Wm = words_of(M);
    float *msg = smem_f;
    float *L = msg + E;
    uint32_t *hb = reinterpret_cast<uint32_t *>(L + n);
    uint32_t *sy = hb + Wn;
    __shared__ int s_unsat;
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
    for (int v = tid; v < n; v += nthr) L[v] = ds.L[(((size_t)t * n + v) * LANES + l) * S + sub];
    for (int w = tid; w < Wm; w += nthr) {
        uint32_t word = 0u;
        const int c1 = min(M, 32 * w + 32);
        for (int c = 32 * w; c < c1; ++c) word |= ((cmpu(ds.st[(size_t)t * M + c], sub) >> l) & 1u) << (c & 31);
        sy[w] = word;
    }
    __syncthreads();
    // first VN pass: q = clamp(L), decision 0
    for (int v0 = warp * LANES; v0 < n; v0 += nwarps * LANES) {
        const int v = v0 + lane;
        float lv = 0.0f;
        if (v < n) {
            lv = L[v];
            const float q = clampf(lv, qmax2);
            for (int p = cd.col_ptr[v]; p < cd.col_ptr[v + 1]; ++p) msg[cd.csc_slot[p]] = q;
        }
        const uint32_t word = __ballot_sync(FULL, v < n && lv < 0.0f);
        if (lane == 0) hb[v0 >> 5] = word;
    }
    __syncthreads();
    int it = max_iter;
    uint8_t cv = 0;
    for (int k = 1; k <= max_iter + 1; ++k) {
        // syndrome test of decision k-1
        if (tid == 0) s_unsat = 0;
        __syncthreads();
        for (int c = tid; c < M; c += nthr) {
            uint32_t par = sbit(sy, c);
            for (int e = cd.row_ptr[c]; e < cd.row_ptr[c + 1]; ++e) par ^= sbit(hb, cd.col_idx[e]);
            if (par) s_unsat = 1;
        }
        __syncthreads();
        if (!s_unsat) {
            it = k - 1;
            cv = 1;
            break;
        }
        if (k == max_iter + 1) break;
        // CN pass k
        for (int c = tid; c < M; c += nthr) {
            const int e0 = cd.row_ptr[c], deg = cd.row_ptr[c + 1] - e0;
            const uint32_t sb = sbit(sy, c);
            if (DCT >= 5 && deg <= 2) {  // same special case as cn_check
                float q[2];
#pragma unroll
                for (int i = 0; i < 2; ++i) q[i] = i < deg ? msg[e0 + i] : DUMMY_Q;
                cn_update<2>(q, sb, qmax2);
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    if (i < deg) msg[e0 + i] = q[i];
            } else {
                float q[DCT];
#pragma unroll
                for (int i = 0; i < DCT; ++i) q[i] = i < deg ? msg[e0 + i] : DUMMY_Q;
                cn_update<DCT>(q, sb, qmax2);
#pragma unroll
                for (int i = 0; i < DCT; ++i)
                    if (i < deg) msg[e0 + i] = q[i];
            }
        }
        __syncthreads();
        // VN pass k: posterior in CSC slot order, extrinsic V2C, decision k
        for (int v0 = warp * LANES; v0 < n; v0 += nwarps * LANES) {
            const int v = v0 + lane;
            float post = 0.0f;
            if (v < n) {
                const int p0 = cd.col_ptr[v], p1 = cd.col_ptr[v + 1];
                post = L[v];
                for (int p = p0; p < p1; ++p) post += msg[cd.csc_slot[p]];
                for (int p = p0; p < p1; ++p) {
                    const int e = cd.csc_slot[p];
                    msg[e] = clampf(post - msg[e], qmax2);
                }
            }
            const uint32_t word = __ballot_sync(FULL, v < n && post < 0.0f);
            if (lane == 0) hb[v0 >> 5] = word;
        }
        __syncthreads();
    }
    if (tid == 0) {
        ds.iters[f] = it;
        ds.conv[f] = cv;
    }
    for (int w = tid; w < Wn; w += nthr) bits_out[(size_t)f * Wn + w] = hb[w];
}

size_t decode_smem_bytes(const CodeDev &cd) {
    return (size_t)(cd.E + cd.n) * 4 + (size_t)(words_of(cd.n) + words_of(cd.M)) * 4;
}

// returns false when the code is not eligible (max check degree > 12)
bool launch_decode_smem(const CodeDev &cd, const DecState &ds, int max_iter, float qmax, uint32_t *bits_out,
                        cudaStream_t s) {
    const size_t bytes = decode_smem_bytes(cd);
    const float q2 = qmax * LOG2E;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        kern<<<ds.frames, 512, bytes, s>>>(cd, ds, max_iter, q2, bits_out);
    };
    switch (cd.max_dc) {
        case 1: case 2: go(k_decode_smem<2>); return true;
        case 3: go(k_decode_smem<3>); return true;
        case 4: go(k_decode_smem<4>); return true;
        case 5: go(k_decode_smem<5>); return true;
        case 6: go(k_decode_smem<6>); return true;
        case 7: go(k_decode_smem<7>); return true;
        case 8: go(k_decode_smem<8>); return true;
        case 9: go(k_decode_smem<9>); return true;
        case 10: go(k_decode_smem<10>); return true;
        case 11: case 12: go(k_decode_smem<12>); return true;
        default: return false;
    }
}

// ---------------------------------------------------------------- launchers

// qmax is in natural LLR units; the arena works in log2 units.  The kernel body
// is chosen by the code's maximum check degree and the tile width S.
template <int S>
static void launch_cn_s(const CodeDev &cd, const DecState &ds, dim3 grid, float q2, int check_only, cudaStream_t s) {
    switch (cd.max_dc) {
        case 1: case 2: k_cn<2, S><<<grid, BLOCK, 0, s>>>(cd, ds, q2, check_only); break;
        case 3: k_cn<3, S><<<grid, BLOCK, 0, s>>>(cd, ds, q2, check_only); break;
        case 4: k_cn<4, S><<<grid, BLOCK, 0, s>>>(cd, ds, q2, check_only); break;
        case 5: k_cn<5, S><<<grid, BLOCK, 0, s>>>(cd, ds, q2, check_only); break;
        case 6: k_cn<6, S><<<grid, BLOCK, 0, s>>>(cd, ds, q2, check_only); break;
        case 7: k_cn<7, S><<<grid, BLOCK, 0, s>>>(cd, ds, q2, check_only); break;
        case 8: k_cn<8, S><<<grid, BLOCK, 0, s>>>(cd, ds, q2, check_only); break;
        case 9: k_cn<9, S><<<grid, BLOCK, 0, s>>>(cd, ds, q2, check_only); break;
        case 10: k_cn<10, S><<<grid, BLOCK, 0, s>>>(cd, ds, q2, check_only); break;
        case 11: case 12: k_cn<12, S><<<grid, BLOCK, 0, s>>>(cd, ds, q2, check_only); break;
        default: k_cn<0, S><<<grid, BLOCK, 0, s>>>(cd, ds, q2, check_only); break;
    }
}

// TMA-streamed CN pass (k_cn_tma): ring of nstage stages of CPI x DCT rows per CTA,
// persistent grid of (CTAs per SM) x SMs.  Opt-in (CVSR_CN_TMA=1): it measured
// slower than k_cn; CVSR_CN_RING_KB sets the ring budget per CTA.
static int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}

template <int DCT, int S>
static void launch_cn_tma_t(const CodeDev &cd, const DecState &ds, int grid_tiles, float q2, cudaStream_t s) {
    static int ctas_per_sm = -1, nstage = 0, stage_bytes = 0, n_sm = 0;
    if (ctas_per_sm < 0) {
        stage_bytes = CPI * DCT * LANES * S * 4;
        const int budget = env_int("CVSR_CN_RING_KB", 96) * 1024;
        nstage = budget / stage_bytes;
        nstage = nstage < 2 ? 2 : (nstage > CN_TMA_MAX_STAGES ? CN_TMA_MAX_STAGES : nstage);
        const int smem = 128 + nstage * stage_bytes;
        cudaFuncSetAttribute(k_cn_tma<DCT, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, k_cn_tma<DCT, S>, CN_TMA_THREADS, smem);
        if (ctas_per_sm < 1) ctas_per_sm = 1;
    }
    const int groups = (cd.M + CPI - 1) / CPI;
    const long long items = (long long)groups * grid_tiles;
    const int grid = (int)(items < (long long)ctas_per_sm * n_sm ? items : (long long)ctas_per_sm * n_sm);
    k_cn_tma<DCT, S><<<grid, CN_TMA_THREADS, 128 + nstage * stage_bytes, s>>>(cd, ds, q2, groups, nstage,
                                                                               stage_bytes);
}

template <int S>
static bool launch_cn_tma_s(const CodeDev &cd, const DecState &ds, int grid_tiles, float q2, cudaStream_t s) {
    switch (cd.max_dc) {
        case 1: case 2: launch_cn_tma_t<2, S>(cd, ds, grid_tiles, q2, s); return true;
        case 3: launch_cn_tma_t<3, S>(cd, ds, grid_tiles, q2, s); return true;
        case 4: launch_cn_tma_t<4, S>(cd, ds, grid_tiles, q2, s); return true;
        case 5: launch_cn_tma_t<5, S>(cd, ds, grid_tiles, q2, s); return true;
        case 6: launch_cn_tma_t<6, S>(cd, ds, grid_tiles, q2, s); return true;
        case 7: launch_cn_tma_t<7, S>(cd, ds, grid_tiles, q2, s); return true;
        case 8: launch_cn_tma_t<8, S>(cd, ds, grid_tiles, q2, s); return true;
        default: return false;
    }
}

void launch_cn(const CodeDev &cd, const DecState &ds, int grid_tiles, float qmax, int check_only, cudaStream_t s) {
    if (grid_tiles <= 0) return;
    static const int use_tma = env_int("CVSR_CN_TMA", 0);
    if (use_tma && !check_only) {
        const float q2t = qmax * LOG2E;
        bool done = false;
        if (ds.subs == 4) done = launch_cn_tma_s<4>(cd, ds, grid_tiles, q2t, s);
        else if (ds.subs == 2) done = launch_cn_tma_s<2>(cd, ds, grid_tiles, q2t, s);
        else done = launch_cn_tma_s<1>(cd, ds, grid_tiles, q2t, s);
        if (done) return;
    }
    const int per_block = WARPS_PER_BLOCK * CPW;
    dim3 grid((cd.M + per_block - 1) / per_block, grid_tiles);
    const float q2 = qmax * LOG2E;
    if (ds.subs == 4) launch_cn_s<4>(cd, ds, grid, q2, check_only, s);
    else if (ds.subs == 2) launch_cn_s<2>(cd, ds, grid, q2, check_only, s);
    else launch_cn_s<1>(cd, ds, grid, q2, check_only, s);
}

template <int DV, int VPW_, bool FIRST, int S>
static void launch_vn_cls(const CodeDev &cd, const DecState &ds, int cls, int grid_tiles, float q2, float *post_dbg,
                          cudaStream_t s) {
    const int per_block = WARPS_PER_BLOCK * VPW_;
    dim3 grid((cd.vc_cnt[cls] + per_block - 1) / per_block, grid_tiles);
    k_vn_cls<DV, VPW_, FIRST, S><<<grid, BLOCK, 0, s>>>(cd, ds, cls, q2, post_dbg);
}

// registers: VPW x (DV + 1) line buffers of S floats
template <bool FIRST, int S>
static int launch_vn_t(const CodeDev &cd, const DecState &ds, int grid_tiles, float q2, float *post_dbg,
                       cudaStream_t s) {
    constexpr int X = 4 / S;  // more variables per warp when the lines are narrower
    int launched = 0;
    for (int c = 0; c < cd.n_vclass; ++c) {
        if (cd.vc_cnt[c] <= 0) continue;
        ++launched;
        switch (cd.vc_deg[c]) {
            case 1: launch_vn_cls<1, 6, FIRST, S>(cd, ds, c, grid_tiles, q2, post_dbg, s); break;
            case 2: launch_vn_cls<2, 4, FIRST, S>(cd, ds, c, grid_tiles, q2, post_dbg, s); break;
            case 3: launch_vn_cls<3, 2 * (X > 1 ? 2 : 1), FIRST, S>(cd, ds, c, grid_tiles, q2, post_dbg, s); break;
            case 4: launch_vn_cls<4, 2 * (X > 1 ? 2 : 1), FIRST, S>(cd, ds, c, grid_tiles, q2, post_dbg, s); break;
            case 5: launch_vn_cls<5, X, FIRST, S>(cd, ds, c, grid_tiles, q2, post_dbg, s); break;
            case 6: launch_vn_cls<6, X, FIRST, S>(cd, ds, c, grid_tiles, q2, post_dbg, s); break;
            case 7: launch_vn_cls<7, X, FIRST, S>(cd, ds, c, grid_tiles, q2, post_dbg, s); break;
            case 8: launch_vn_cls<8, X, FIRST, S>(cd, ds, c, grid_tiles, q2, post_dbg, s); break;
            default: {
                dim3 grid((cd.vc_cnt[c] + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, grid_tiles);
                k_vn_generic<FIRST, S><<<grid, BLOCK, 0, s>>>(cd, ds, c, q2, post_dbg);
            }
        }
    }
    return launched;
}

// returns the number of kernels launched (one per variable-degree class)
int launch_vn(const CodeDev &cd, const DecState &ds, int grid_tiles, float qmax, bool first, float *post_dbg,
              cudaStream_t s) {
    if (grid_tiles <= 0) return 0;
    const float q2 = qmax * LOG2E;
    if (ds.subs == 4) return first ? launch_vn_t<true, 4>(cd, ds, grid_tiles, q2, post_dbg, s)
                                   : launch_vn_t<false, 4>(cd, ds, grid_tiles, q2, post_dbg, s);
    if (ds.subs == 2) return first ? launch_vn_t<true, 2>(cd, ds, grid_tiles, q2, post_dbg, s)
                                   : launch_vn_t<false, 2>(cd, ds, grid_tiles, q2, post_dbg, s);
    return first ? launch_vn_t<true, 1>(cd, ds, grid_tiles, q2, post_dbg, s)
                 : launch_vn_t<false, 1>(cd, ds, grid_tiles, q2, post_dbg, s);
}

FusedPlan make_plan(const CodeDev &cd, int subs) {
    FusedPlan p{};
    p.n_cn = (cd.M + WARPS_PER_BLOCK * CPW - 1) / (WARPS_PER_BLOCK * CPW);
    p.n_cls = cd.n_vclass;
    p.items_per_tile = p.n_cn;
    for (int c = 0; c < cd.n_vclass; ++c) {
        const int d = cd.vc_deg[c];
        const int vpw = (d >= 1 && d <= 8) ? vpw_for(d, subs) : 1;
        p.cls_chunks[c] = (cd.vc_cnt[c] + WARPS_PER_BLOCK * vpw - 1) / (WARPS_PER_BLOCK * vpw);
        p.items_per_tile += p.cls_chunks[c];
    }
    return p;
}

template <int DCT, int S>
static void launch_iter_t(const CodeDev &cd, const DecState &dsc, const DecState &dsv, const FusedPlan &plan, int k,
                          float q2, cudaStream_t s) {
    static int grid = 0;
    if (!grid) {
        int per_sm = 0, dev = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_iter<DCT, S>, BLOCK, 0);
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        grid = (per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148);
    }
    k_iter<DCT, S><<<grid, BLOCK, 0, s>>>(cd, dsc, dsv, plan, k, q2);
}

template <int S>
static void launch_iter_s(const CodeDev &cd, const DecState &dsc, const DecState &dsv, const FusedPlan &plan, int k,
                          float q2, cudaStream_t s) {
    switch (cd.max_dc) {
        case 1: case 2: launch_iter_t<2, S>(cd, dsc, dsv, plan, k, q2, s); break;
        case 3: launch_iter_t<3, S>(cd, dsc, dsv, plan, k, q2, s); break;
        case 4: launch_iter_t<4, S>(cd, dsc, dsv, plan, k, q2, s); break;
        case 5: launch_iter_t<5, S>(cd, dsc, dsv, plan, k, q2, s); break;
        case 6: launch_iter_t<6, S>(cd, dsc, dsv, plan, k, q2, s); break;
        case 7: launch_iter_t<7, S>(cd, dsc, dsv, plan, k, q2, s); break;
        case 8: launch_iter_t<8, S>(cd, dsc, dsv, plan, k, q2, s); break;
        default: launch_iter_t<0, S>(cd, dsc, dsv, plan, k, q2, s); break;
    }
}

void launch_iter(const CodeDev &cd, const DecState &dsc, const DecState &dsv, const FusedPlan &plan, int k,
                 float qmax, cudaStream_t s) {
    const float q2 = qmax * LOG2E;
    if (dsc.subs == 4) launch_iter_s<4>(cd, dsc, dsv, plan, k, q2, s);
    else if (dsc.subs == 2) launch_iter_s<2>(cd, dsc, dsv, plan, k, q2, s);
    else launch_iter_s<1>(cd, dsc, dsv, plan, k, q2, s);
}

void launch_list(const DecState &ds, int32_t *host_counts, cudaStream_t s) {
    k_list<<<1, 1024, 0, s>>>(ds, host_counts);
}

void launch_status(const DecState &ds, int k, int max_iter, int final_pass, int32_t *host_counts, cudaStream_t s) {
    k_status<<<1, 1024, 0, s>>>(ds, k, max_iter, final_pass, host_counts);
}

void launch_retire(const DecState &ds, int32_t n, int grid_tiles, uint32_t *bits_out, cudaStream_t s) {
    if (grid_tiles <= 0) return;
    const int64_t items = (int64_t)((words_of(n) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK) * grid_tiles;
    k_retire<<<(unsigned)std::min<int64_t>(items, 148 * 8), BLOCK, 0, s>>>(ds, n, bits_out);
}

void launch_to_interleaved(const float *src, float *dst, int32_t F, int64_t rows, int tiles, int subs, float scale,
                           cudaStream_t s) {
    dim3 grid((unsigned)((rows + 31) / 32), tiles);
    if (subs == 4) k_to_interleaved<4><<<grid, 256, 0, s>>>(src, dst, F, rows, scale);
    else if (subs == 2) k_to_interleaved<2><<<grid, 256, 0, s>>>(src, dst, F, rows, scale);
    else k_to_interleaved<1><<<grid, 256, 0, s>>>(src, dst, F, rows, scale);
}

void launch_from_interleaved(const float *src, float *dst, int32_t F, int64_t rows, int tiles, int subs, float scale,
                             cudaStream_t s) {
    dim3 grid((unsigned)((rows + 31) / 32), tiles);
    if (subs == 4) k_from_interleaved<4><<<grid, 256, 0, s>>>(src, dst, F, rows, scale);
    else if (subs == 2) k_from_interleaved<2><<<grid, 256, 0, s>>>(src, dst, F, rows, scale);
    else k_from_interleaved<1><<<grid, 256, 0, s>>>(src, dst, F, rows, scale);
}

void launch_synd_transpose(const uint32_t *synd, int32_t F, int32_t M, int subs, uint4 *st, int tiles,
                           const int32_t *pos, cudaStream_t s) {
    dim3 grid((words_of(M) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK, tiles);
    k_synd_transpose<<<grid, BLOCK, 0, s>>>(synd, F, M, subs, st, pos);
}

void launch_init_tiles(const DecState &ds, const uint8_t *alive, cudaStream_t s) {
    k_init_tiles<<<(ds.tiles + 127) / 128, 128, 0, s>>>(ds, alive);
}

// move the active frames of `src` densely into `dst` (state after a VN pass); returns launches
int launch_compact(const CodeDev &cd, const DecState &src, const DecState &dst, int32_t *dst_src, int max_tiles,
                   int32_t *host_counts, bool move_hb, cudaStream_t s) {
    k_compact_plan<<<1, 1024, 0, s>>>(src, dst, dst_src, host_counts);
    const int64_t fr = 8 * CR_ROWS;  // float rows per block
    const dim3 gE((unsigned)((cd.E + fr - 1) / fr), max_tiles), gN((unsigned)((cd.n + fr - 1) / fr), max_tiles),
        gNb((unsigned)((cd.n + 255) / 256), max_tiles), gM((unsigned)((cd.M + 255) / 256), max_tiles);
    if (src.subs == 4) {
        k_compact_rows<4><<<gE, 256, 0, s>>>(src.msg, dst.msg, cd.E, dst_src, dst.counts);
        k_compact_rows<4><<<gN, 256, 0, s>>>(src.L, dst.L, cd.n, dst_src, dst.counts);
    } else if (src.subs == 2) {
        k_compact_rows<2><<<gE, 256, 0, s>>>(src.msg, dst.msg, cd.E, dst_src, dst.counts);
        k_compact_rows<2><<<gN, 256, 0, s>>>(src.L, dst.L, cd.n, dst_src, dst.counts);
    } else {
        k_compact_rows<1><<<gE, 256, 0, s>>>(src.msg, dst.msg, cd.E, dst_src, dst.counts);
        k_compact_rows<1><<<gN, 256, 0, s>>>(src.L, dst.L, cd.n, dst_src, dst.counts);
    }
    k_compact_bits<<<gM, 256, 0, s>>>(src.st, dst.st, cd.M, src.subs, dst_src, dst.counts);
    if (!move_hb) return 5;
    k_compact_bits<<<gNb, 256, 0, s>>>(src.hb, dst.hb, cd.n, src.subs, dst_src, dst.counts);
    return 6;
}

void launch_set_counts(const DecState &ds, int32_t n_active, cudaStream_t s) {
    k_set_counts<<<1, 32, 0, s>>>(ds, n_active);
}


}  // namespace cvsr
