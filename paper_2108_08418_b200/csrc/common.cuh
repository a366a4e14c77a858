// Internal definitions of the cvsr CUDA library (sm_100a).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cvsr.h"

namespace cvsr {

// Frames per tile: 32 warp lanes x S frames per lane (S = 1, 2 or 4, chosen per
// decode from the batch size: a float, float2 or float4 per lane).  Frame f of
// tile t sits at lane (f mod 32), component s = (f / 32) mod S ("sub-tile"),
// i.e. f = 32 S t + 32 s + lane.  Edge messages of the 32 S frames of a tile
// are stored contiguously per edge slot ("frame-interleaved arena", SURVEY.md
// §2.6 row 45): a warp moves one 128 S-byte line per edge.
constexpr int LANES = 32;
constexpr int SUBS = 4;  // maximum S
constexpr int WARPS_PER_BLOCK = 8;
constexpr int BLOCK = 32 * WARPS_PER_BLOCK;
// largest check degree supported (cvsr_code_load rejects larger rows with CVSR_ECODE)
constexpr int MAX_DC = 128;
// variable-degree classes kept separate (more distinct degrees share a generic class)
constexpr int MAX_VCLASS = 16;
// layers of the row-layered schedule (codes needing more colours decode with flooding only)
constexpr int MAX_LAYERS = 48;
// arena values are LLR * log2(e)
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// Device view of a loaded parity-check matrix (SURVEY.md §1 layer B1).
struct CodeDev {
    int32_t n;          // variables (N_R)
    int32_t M;          // checks
    int64_t E;          // edges (G)
    const int32_t *row_ptr;   // [M+1]  CSR by check
    const int32_t *col_idx;   // [E]    variable of each CSR edge
    const int32_t *col_ptr;   // [n+1]  CSC by variable
    const int32_t *csc_slot;  // [E]    CSR position of each CSC entry
    int32_t max_dc, max_dv;
    // variables bucketed by degree (VN launches per class):
    const int32_t *vc_vars;   // [n]  variables sorted by (degree, index)
    const int32_t *vc_slots;  // [E]  their CSR slots, class-major, deg slots per variable
    int32_t n_vclass;
    int32_t vc_deg[MAX_VCLASS];    // degree of class (or -1: mixed degrees, generic path)
    int32_t vc_off[MAX_VCLASS];    // first position in vc_vars
    int32_t vc_cnt[MAX_VCLASS];    // number of variables
    int64_t vc_soff[MAX_VCLASS];   // first position in vc_slots
    // row-layered schedule (reading R-9): checks grouped by greedy colour, no two checks of a
    // layer share a variable; layer l is layer_chk[layer_off[l] .. layer_off[l + 1])
    const int32_t *layer_chk;      // [M]
    int32_t n_layers;              // 0: more than MAX_LAYERS colours (layered schedule unavailable)
    int32_t layer_off[MAX_LAYERS + 1];
    // the same checks in layer order as self-contained descriptors, so a warp's chunk of checks
    // needs no dependent index loads: layer_desc[i] = {row_ptr[c], degree, c, 0} for
    // c = layer_chk[i]; layer_col[i * layer_dc + k] = col_idx[row_ptr[c] + k] (0-padded to the
    // layered kernels' compute width layer_dc); null when the layered kernels do not apply
    const int4 *layer_desc;        // [M]
    const int32_t *layer_pos;      // [M] position of check c in layer order (inverse of layer_chk)
    const int32_t *layer_col;      // [M * layer_dc]
    int32_t layer_dc;
    // checks of layer l with degree > 2 (a layer is sorted by degree, so they come first; the
    // degree <= 2 tail is taken in longer chunks by k_layer_tma, host copy)
    int32_t layer_nbig[MAX_LAYERS];
};

// Per-decode device state (lives in the context's scratch arena).  Syndrome rows st are in check
// order for the flooding schedule and in layer order (row i = check layer_chk[i]) for the layered
// schedule (launch_synd_transpose's pos argument).
// Masks and bit words are uint4: component s holds the 32 lanes of sub-tile s.
struct DecState {
    int32_t tiles;
    int32_t frames;
    int32_t subs;           // S: frames per lane
    int32_t tile_frames;    // 32 S
    float *msg;             // [tiles][E][32][S]  in-place V2C/C2V message per edge slot (log2 units)
    float *L;               // [tiles][n][32][S]  channel LLR (log2 units)
    uint4 *hb;              // [tiles][n]      hard decisions, bit = lane (components >= S unused)
    uint4 *st;              // [tiles][M]      syndrome bits, bit = lane
    uint4 *tile_active;     // [tiles] frames still iterating
    uint4 *tile_unsat;      // [tiles] frames with >= 1 unsatisfied check in this CN pass
    uint4 *tile_newly;      // [tiles] frames retired by the last status pass
    int32_t *active_list;   // [tiles]
    int32_t *retire_list;   // [tiles]
    int32_t *counts;        // [4]: n_active, n_retire, total active lanes, pad
    int32_t *iters;         // [frames] D of the current decode
    uint8_t *conv;          // [frames]
    // fused-iteration scheduler (k_iter): second hard-decision buffer, work counter, per-tile sync
    uint4 *hb2;             // [tiles][n]
    int32_t *fused_work;    // [1]
    int32_t *cn_done;       // [tiles] CN chunks finished this iteration
    int32_t *cn_ready;      // [tiles] iteration whose CN + status of the tile completed
    // frame compaction: frame id of each slot (slot = 32 S t + 32 s + lane), nullptr = identity
    int32_t *slot_frame;
};

// work items of one fused iteration per tile: CN chunks then per-class VN chunks
struct FusedPlan {
    int32_t n_cn;
    int32_t n_cls;
    int32_t cls_chunks[MAX_VCLASS];
    int32_t items_per_tile;
};

// Conditional-LLR parameters for the reconcile LLR kernel.
struct LlrParams {
    int32_t m;
    int32_t j;
    uint32_t known_mask;
    float sigma_n;
    float inv_sigma;
    float llr_max;
    const uint32_t *known_bits[8];  // packed [F][Wn] per known slice (nullptr if unknown)
    int32_t nk;                     // number of known slices
    int32_t kj[8];                  // their indices, ascending (bit t of a table combo = slice kj[t])
    const float *table;             // [2^|K|][LLR_NTAB] unclamped L on the x grid (nullptr: exact only)
    const float4 *table4;           // [2^|K|][LLR_NWIN] windows (table[i .. i+3]) of the same values
    float edges[255];
};

// Tabulated conditional LLR: L(x) for one known-bit pattern is a smooth function
// of x; it is tabulated (exact log-domain formula) on a uniform grid and read by
// cubic Lagrange interpolation, falling back to the exact formula outside the grid
// or when the grid is coarse relative to sigma_n.
constexpr int LLR_NTAB = 4096 + 3;
constexpr float LLR_XMAX = 10.0f;
constexpr float LLR_H = 2.0f * LLR_XMAX / 4096.0f;
// interpolation windows: window i = the 4 grid values of interval i's cubic (one 16-byte load)
constexpr int LLR_NWIN = 4095;

__host__ __device__ inline int32_t words_of(int64_t bits) { return (int32_t)((bits + 31) / 32); }

#ifdef __CUDACC__
// Bit-matrix transpose across a warp (all 32 lanes): lane r holds row r (bit c = element [r][c]);
// returns column `lane` (bit r = element [r][lane]).  Round j swaps the j x j off-diagonal blocks
// between lane r and lane r ^ j.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
    constexpr uint32_t M[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int j = 16 >> k;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & ~M[k]) | ((y & ~M[k]) >> j)) : ((x & M[k]) | ((y & M[k]) << j));
    }
    return x;
}
#endif

// compute width of the layered kernels for a code's maximum check degree (the template DC of
// k_layer / k_layer_tma): exact for 3..10, 2 for degrees <= 2, 12 for 11..12; 0 = unsupported
inline int32_t layer_width(int32_t max_dc) {
    return max_dc <= 2 ? 2 : (max_dc <= 10 ? max_dc : (max_dc <= 12 ? 12 : 0));
}

// frames per lane for a batch: the smallest S in {1, 2, 4} whose tiles are not
// mostly empty (S = 4 once there are more than 64 frames)
inline int choose_subs(int32_t frames) { return frames <= 32 ? 1 : (frames <= 64 ? 2 : 4); }

}  // namespace cvsr
