/*
 * cvsr.h -- C ABI of the B200-native sliced-reconciliation hot path
 * (Ai & Malaney, arXiv 2108.08418; "PAPER.md" = the paper's text).
 *
 * The library (paper_2108_08418_b200/libcvsr.so, sm_100a) implements the
 * data-parallel hot path named by BASELINE.json's north star and scoped by
 * Gray-labelled constant-step quantisation (Bob), slice
 * syndromes (Bob), per-slice LLRs conditioned on already-known slices
 * (Alice), and syndrome-based sum-product BP (flooding, or row-layered per
 * cvsr_decode_opts.flags) over many independent LDPC sub-blocks ("frames")
 * with per-frame early termination.
 *
 * Conventions (apply to every entry point unless stated):
 *  - Ownership.  Every data buffer argument is CALLER-OWNED DEVICE memory of
 *    the context's device (e.g. a torch tensor's data_ptr()), except where a
 *    parameter is documented "host".  The library owns only cvsr_ctx (stream
 *    handle + a grow-only scratch arena) and cvsr_code (immutable after load).
 *  - Asynchrony.  Calls validate their arguments on the host, enqueue kernels
 *    on the context stream and return; outputs are valid after the stream
 *    (or cvsr_ctx_sync) completes.  Entry points that fill a host struct
 *    (cvsr_reconcile with stats_out != NULL, cvsr_count_errors) synchronise.
 *    cvsr_decode and cvsr_reconcile drive the BP iterations from the host:
 *    they keep the stream LOOKAHEAD (3) iterations ahead of a mapped
 *    progress counter and therefore return when the last iteration has been
 *    enqueued (at most a few iterations before the stream drains); batches of
 *    at most two tiles replay 8-iteration CUDA graphs instead (CVSR_GRAPH=0
 *    disables).
 *  - Errors.  The return status is the only error channel.  Argument and
 *    shape validation happens before any launch, so on a validation error
 *    nothing is written.  Asynchronous CUDA faults are sticky and reported
 *    as CVSR_ECUDA by the next call or by cvsr_ctx_sync.  Non-convergence of
 *    a frame is never an error; it is reported through flags.
 *    cvsr_last_error() returns a thread-local message for the last failure.
 *  - Threading.  A cvsr_ctx is single-threaded.  A cvsr_code is read-only
 *    and may be shared by contexts on the same device.
 *  - Determinism.  Results are bit-identical for any batch size, frame order
 *    and GPU count: no floating-point atomics on any path.
 *  - Environment switches (read once per process; defaults in brackets):
 *    CVSR_SMEM [1] / CVSR_SMEM_KB [40]: one-CTA-per-frame on-chip decoder for
 *    codes whose messages + LLRs fit in that many KB; CVSR_GRAPH [1]: CUDA
 *    graph replay of the iteration loop for single-tile batches;
 *    CVSR_COMPACT [1] / CVSR_COMPACT_FRAC [0.65]: frame compaction;
 *    CVSR_SUBS [auto]: frames per lane (1, 2, 4); CVSR_FUSED [0] and
 *    CVSR_CN_TMA [0]: experimental schedulers.  The SMEM, GRAPH,
 *    COMPACT, SUBS and FUSED variants are tested bit-identical to the default
 *    path.  CVSR_SCHEDULE [flooding]: "layered" makes the row-layered
 *    schedule the default of calls whose cvsr_decode_opts.flags leave the
 *    schedule unset (CVSR_SCHED_DEFAULT); the flags select it per call.
 *    Layered-path variants, all tested bit-identical to the default:
 *    CVSR_LAYER_TMA [1] (0: register-staged k_layer), CVSR_LAYER_PERSIST [0]
 *    (persistent k_layer_tmap), CVSR_LAYER_PDL [1] (layer kernels launched as
 *    programmatic dependents), CVSR_LAYER_EARLY [1] (tile lists and first
 *    message lines read before the dependency wait), CVSR_LAYER_PAIRS [1]
 *    (degree <= 2 layer tails in longer chunks; CVSR_LAYER_CH2_WAVES [4]: 12-check
 *    chunks only above that many waves of warps), CVSR_SYND_TEST_W [1]
 *    (syndrome test from the padded layer rows, two tiles per thread);
 *    CVSR_SYND_SLICED [1]: cvsr_syndrome through bit-sliced 32-frame words.
 *  - Layouts.  "frame-major" arrays are [frames][n] row-major.  Packed bit
 *    vectors put bit i at bit (i mod 32) of 32-bit word floor(i/32); a
 *    vector of B bits occupies ceil(B/32) words per frame; padding bits are
 *    0 on output and ignored on input.  Labels are uint8 Gray codes with bit
 *    j = slice j and bit 0 the LSB (PAPER.md:114 footnote "the least
 *    significant bit is l_0").
 */
#ifndef CVSR_H
#define CVSR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CVSR_ABI_VERSION 2

typedef int32_t cvsr_status;
#define CVSR_OK 0
#define CVSR_EINVAL (-1)  /* bad argument value / null pointer                 */
#define CVSR_ESHAPE (-2)  /* inconsistent sizes                                */
#define CVSR_ENOMEM (-3)  /* device or host allocation failed                  */
#define CVSR_ECUDA  (-4)  /* CUDA runtime error (sticky for asynchronous faults)*/
#define CVSR_ECODE  (-5)  /* malformed parity-check matrix                     */

typedef struct cvsr_ctx cvsr_ctx;
typedef struct cvsr_code cvsr_code;

/* Thread-local message describing the last non-OK status ("" if none). */
const char *cvsr_last_error(void);
/* Returns CVSR_ABI_VERSION of the loaded library. */
int32_t cvsr_abi_version(void);

/* ------------------------------------------------------------- context */
/* Create a context on CUDA device `device`; `cuda_stream` is a cudaStream_t
 * (NULL = the legacy default stream).  The stream is borrowed, not owned. */
cvsr_status cvsr_ctx_create(int32_t device, void *cuda_stream, cvsr_ctx **out);
/* Re-point the context at another borrowed stream of the same device. */
cvsr_status cvsr_ctx_set_stream(cvsr_ctx *ctx, void *cuda_stream);
/* Wait for all work on the context stream; surfaces asynchronous faults. */
cvsr_status cvsr_ctx_sync(cvsr_ctx *ctx);
/* Number of kernels this context has launched so far (diagnostics/bench). */
int64_t cvsr_ctx_launch_count(const cvsr_ctx *ctx);
void cvsr_ctx_destroy(cvsr_ctx *ctx);
/* Diagnostics: when enabled, the BP scheduler brackets its launches with CUDA
 * events on the context stream, per kernel class: 0 = check-node pass (k_cn),
 * 1 = variable-node pass (k_vn), 2 = initialisation (conditional LLR + first
 * V2C write), 3 = control (status/retire).  cvsr_ctx_kernel_times
 * synchronises, returns device milliseconds and launch counts per class in
 * HOST arrays ms_out[4], launches_out[4], and resets the accumulators. */
cvsr_status cvsr_ctx_set_profiling(cvsr_ctx *ctx, int32_t enable);
cvsr_status cvsr_ctx_kernel_times(cvsr_ctx *ctx, double *ms_out, int64_t *launches_out);

/* ------------------------------------------------------------- code H_j */
/* Load a parity-check matrix H (n_checks x n_vars) given as HOST CSR by
 * check: row_ptr[n_checks+1] (row_ptr[0] = 0, non-decreasing), col_idx[E]
 * (0 <= col < n_vars, no duplicate within a row).  G = E non-zeros
 * (PAPER.md:189).  The arrays are copied; the library builds the device
 * CSR + CSC + edge-permutation layout (SURVEY.md §1 layer B1).
 * Errors: CVSR_EINVAL (null/negative), CVSR_ECODE (malformed rows, empty
 * variable columns are allowed), CVSR_ENOMEM, CVSR_ECUDA. */
cvsr_status cvsr_code_load(cvsr_ctx *ctx, int32_t n_vars, int32_t n_checks, const int32_t *row_ptr,
                           const int32_t *col_idx, cvsr_code **out);
/* host outputs; any may be NULL */
cvsr_status cvsr_code_info(const cvsr_code *code, int32_t *n_vars, int32_t *n_checks, int64_t *n_edges);
void cvsr_code_free(cvsr_code *code);

/* ------------------------------------------------------------- Bob */
/* Constant-step quantiser M(.) (PAPER.md:114 step 1): m in
 * [1,8]; edges[0 .. 2^m-2] strictly ascending fp32 bin edges (reading A-3:
 * integer multiples of the step, symmetric about 0; outer bins unbounded).
 * Passed by host pointer. */
typedef struct {
    int32_t m;
    float edges[255];
} cvsr_quantiser;

/* label[i] = g(b), b = #{k : y[i] >= edges[k]}, g(b) = b ^ (b >> 1) (Gray
 * labelling).  Bit-exact (fp32 comparisons only; ties go to the
 * upper bin).  y: float[count] (any layout), label_out: uint8[count].
 * Inputs must be finite (NaN is undefined). */
cvsr_status cvsr_quantise(cvsr_ctx *ctx, const cvsr_quantiser *q, const float *y, int64_t count,
                          uint8_t *label_out);

/* Slice S_j = bit j of each label (PAPER.md:114 step 2), packed:
 * label uint8[frames][n] -> bits_out uint32[frames][ceil(n/32)]. */
cvsr_status cvsr_slice_bits(cvsr_ctx *ctx, const uint8_t *label, int32_t frames, int32_t n, int32_t slice_j,
                            uint32_t *bits_out);

/* Syndrome s_j = H_j S_j over GF(2) (PAPER.md:89, PAPER.md:114 steps 2-3):
 * label uint8[frames][n_vars] -> synd_out uint32[frames][ceil(n_checks/32)]. */
cvsr_status cvsr_syndrome(cvsr_ctx *ctx, const cvsr_code *code, const uint8_t *label, int32_t frames,
                          int32_t slice_j, uint32_t *synd_out);

/* ------------------------------------------------------------- Alice: LLR */
/* Conditional LLR of slice j (PAPER.md:114 step 4; reading A-2):
 * L = clamp(ln N_0 - ln N_1, +-llr_max), N_beta = sum of Gaussian bin
 * probabilities P_b(x) = Phi((e_{b+1}-x)/sigma_n) - Phi((e_b-x)/sigma_n) over
 * bins whose Gray label agrees with known_label on known_mask and has bit j =
 * beta.  Positive L means bit 0.  Evaluated in the log domain (fp32).
 * x float[frames][n]; known_label uint8[frames][n] (may be NULL iff
 * known_mask == 0; bit j of known_mask must be 0); llr_out float[frames][n]. */
cvsr_status cvsr_llr_slice(cvsr_ctx *ctx, const cvsr_quantiser *q, const float *x, int32_t frames, int32_t n,
                           float sigma_n, int32_t slice_j, uint32_t known_mask, const uint8_t *known_label,
                           float llr_max, float *llr_out);

/* BI-AWGN channel LLR (config C1, reading A-16): llr = clamp(2y/sigma2). */
cvsr_status cvsr_llr_biawgn(cvsr_ctx *ctx, const float *y, int64_t count, float sigma2, float llr_max,
                            float *llr_out);

/* ------------------------------------------------------------- Alice: BP */
/* max_iter >= 0 (reading A-9); msg_clamp = Q_MAX > 0, the V2C clamp
 * (reading A-10, 40); flags bits 0-1 = BP schedule (PAPER.md:189 names
 * sum-product BP without fixing its schedule):
 *   CVSR_SCHED_DEFAULT   the process default (env CVSR_SCHEDULE=layered, else flooding);
 *   CVSR_SCHED_FLOODING  flooding: all checks, then all variables (reading A-8);
 *   CVSR_SCHED_LAYERED   row-layered (reading R-9): the checks are greedily
 *     coloured in index order into layers that share no variable (check c takes the
 *     smallest colour not used by an earlier check sharing a variable) and an iteration
 *     updates the layers in order against the running posteriors:
 *     q_e = post_v - r_e, r_e <- (1 - 2 s_c) BOXPLUS_{e' != e} clamp(q_e'), post_v <- q_e + r_e.
 *     Same stopping rule as flooding.  A code that needs more than 48 layers or has a
 *     check degree > 12 is decoded with flooding instead (cvsr_stats.schedule reports
 *     what ran).  Other flag bits must be 0. */
#define CVSR_SCHED_DEFAULT 0
#define CVSR_SCHED_FLOODING 1
#define CVSR_SCHED_LAYERED 2
#define CVSR_SCHED_MASK 3
typedef struct {
    int32_t max_iter;
    float msg_clamp;
    int32_t flags;
} cvsr_decode_opts;

/* Syndrome-based sum-product BP (SURVEY.md §8(c)
 * O5, flooding, or O5' row-layered per opts->flags) of `frames` independent
 * sub-blocks sharing code H (flooding shown; layered: see CVSR_SCHED_LAYERED):
 *  k = 0 decision xhat = [L < 0]; iterations k = 1..max_iter of
 *  CN r_e = (1-2 s_c) BOXPLUS_{e' != e} q_e', VN post = L + sum r,
 *  q_e = clamp(post - r_e), xhat = [post < 0]; a frame stops at the first k
 *  with H xhat = s (converged, iters = k) else iters = max_iter, converged = 0.
 * llr float[frames][n_vars]; synd uint32[frames][ceil(n_checks/32)];
 * bits_out uint32[frames][ceil(n_vars/32)]; converged_out uint8[frames];
 * iters_out int32[frames]. */
cvsr_status cvsr_decode(cvsr_ctx *ctx, const cvsr_code *code, const float *llr, const uint32_t *synd,
                        int32_t frames, const cvsr_decode_opts *opts, uint32_t *bits_out, uint8_t *converged_out,
                        int32_t *iters_out);

/* Parity/debug: exactly k_iters >= 1 iterations, no early stop; c2v_out
 * float[frames][E] = C2V messages r_e of iteration k in CSR edge order,
 * post_out float[frames][n_vars] = posteriors of iteration k.  Either output
 * may be NULL.  flags: the schedule, as cvsr_decode_opts.flags
 * (CVSR_SCHED_LAYERED on a code the layered schedule does not support:
 * CVSR_EINVAL). */
cvsr_status cvsr_decode_trace(cvsr_ctx *ctx, const cvsr_code *code, const float *llr, const uint32_t *synd,
                              int32_t frames, int32_t k_iters, float msg_clamp, int32_t flags, float *c2v_out,
                              float *post_out);

/* ------------------------------------------------------------- scheduler */
/* Per-run statistics (host struct).  Slice arrays are indexed by slice j. */
typedef struct {
    int64_t frames;           /* frames processed                                     */
    int64_t frames_ok;        /* frames whose every coded slice converged             */
    int64_t bits_reconciled;  /* m * n per ok frame                     */
    int64_t attempted[8];     /* frames that reached slice j                          */
    int64_t converged[8];     /* frames whose slice j converged (disclosed: attempted)*/
    int64_t iters_sum[8];     /* sum of BP iterations D_j over attempted frames       */
    int64_t edge_iters[8];    /* sum over attempted frames of E_j * D_j               */
    double alice_seconds;     /* device time of the call (CUDA events)                */
    int32_t schedule[8];      /* schedule slice j ran with: 0 disclosed, CVSR_SCHED_FLOODING or
                                 CVSR_SCHED_LAYERED                                    */
} cvsr_stats;

/* Multi-stage sliced reconciliation, Alice's side (PAPER.md:114 steps 4-6,
 * Fig. 3), for `frames` sub-blocks of n symbols.
 *  m in [1,8]; codes: HOST array of m code pointers, codes[j] == NULL means
 *  slice j is disclosed (synd[j] then holds Bob's packed slice bits);
 *  order: HOST int32[m], a permutation of 0..m-1 (decode order);
 *  q: quantiser; sigma_n: noise std (reading A-5/A-18); x float[frames][n];
 *  synd: HOST array of m DEVICE pointers, synd[j] uint32[frames][ceil(M_j/32)]
 *  (or [frames][ceil(n/32)] for a disclosed slice);
 *  opts: BP options (llr clamp is fixed at msg_clamp as well, reading A-11);
 *  outputs: label_out uint8[frames][n] (Alice's labels: bits of attempted
 *  slices), frame_ok uint8[frames], iters int32[frames][m] (D_j; 0 for a
 *  disclosed slice; -1 if not attempted because an earlier slice failed,
 *  reading A-13).  stats_out: optional HOST struct; if non-NULL the call
 *  synchronises and fills it. */
cvsr_status cvsr_reconcile(cvsr_ctx *ctx, int32_t m, const cvsr_code *const *codes, const int32_t *order,
                           const cvsr_quantiser *q, float sigma_n, const float *x, const uint32_t *const *synd,
                           int32_t frames, int32_t n, const cvsr_decode_opts *opts, uint8_t *label_out,
                           uint8_t *frame_ok, int32_t *iters, cvsr_stats *stats_out);

/* Verification hash (Step 5: both parties "apply the same hash
 * function to their reconciled strings and exchange the hash results"):
 * hash_out[f] = sum_{i<W} w_i * key^(i+1) mod p, p = 2^61 - 1, where w_i is the
 * i-th little-endian 32-bit word of frame f's labels (uint8[frames][n],
 * zero-padded to W = ceil(n/4) words).  A universal hash: two different
 * strings collide with probability <= W/p over a uniformly random key in
 * [1, p-1].  key must be in [1, 2^61 - 2]; hash_out uint64[frames] (device). */
cvsr_status cvsr_frame_hash(cvsr_ctx *ctx, const uint8_t *label, int32_t frames, int32_t n, uint64_t key,
                            uint64_t *hash_out);

/* Both sides of the PAPER.md:90 check in one launch (simulation: Bob's labels
 * are on the same device), with CVSR_HASH_KEYS independent keys: hashes
 * label_alice and label_bob (uint8[frames][n]) with cvsr_frame_hash's definition
 * under each key keys[q] (HOST array; each in [1, 2^61 - 2], drawn independently
 * and uniformly per check) and writes verified_out[f] = frame_ok[f] && h_alice[f][q]
 * == h_bob[f][q] for every q (uint8, 0/1).  Two different strings pass with
 * probability <= (W/(p-1))^CVSR_HASH_KEYS over the keys, W = ceil(n/4): <= 2^-122
 * up to n = 5e6 (reading R-6; the 2^-120 target of the reference specification).
 * verified_out may alias frame_ok.  hash_alice_out / hash_bob_out
 * (uint64[frames][CVSR_HASH_KEYS]) may be NULL.  A frame that fails is discarded
 * (reading R-6: per-sub-block abort instead of restarting the whole protocol). */
#define CVSR_HASH_KEYS 3
cvsr_status cvsr_verify(cvsr_ctx *ctx, const uint8_t *label_alice, const uint8_t *label_bob, const uint8_t *frame_ok,
                        int32_t frames, int32_t n, const uint64_t *keys, uint8_t *verified_out, uint64_t *hash_alice_out,
                        uint64_t *hash_bob_out);

/* ------------------------------------------------------------ privacy amplification
 * Toeplitz hashing (Step 6: "apply a 2-universal hashing function on
 * their reconciled string"; reading R-8 of DESIGN.md): the n_in + n_out - 1 seed
 * bits t define T in {0,1}^{n_out x n_in}, T[i][j] = t[i - j + n_in - 1], and
 * y = T x over GF(2).  Computed exactly as the window [n_in - 1, n_in + n_out - 2]
 * of the integer convolution t * x by a number-theoretic transform modulo
 * 15 * 2^27 + 1 of size N = 2^ceil(log2(n_in + n_out - 1)).
 * Bit strings are packed LSB first: bit i at bit (i % 32) of uint32 word i / 32.
 * Limits: 1 <= n_out <= n_in, n_in + n_out - 1 <= 2^27.  The plan owns 16 N bytes
 * of device memory (twiddles, the seed's transform, one work array) on the
 * context's device; one plan serves one stream at a time. */
typedef struct cvsr_pa_plan cvsr_pa_plan;
cvsr_status cvsr_pa_plan_create(cvsr_ctx *ctx, int64_t n_in, int64_t n_out, const uint32_t *seed_bits_host,
                                cvsr_pa_plan **out);
cvsr_status cvsr_pa_plan_info(const cvsr_pa_plan *p, int64_t *n_in, int64_t *n_out, int64_t *ntt_size);
/* x_bits: device uint32[blocks][ceil(n_in/32)]; y_bits: device uint32[blocks][ceil(n_out/32)]
 * (bits past n_out in the last word are 0).  Every block is hashed with the plan's seed. */
cvsr_status cvsr_pa_hash(cvsr_ctx *ctx, const cvsr_pa_plan *p, int32_t blocks, const uint32_t *x_bits,
                         uint32_t *y_bits);
void cvsr_pa_plan_free(cvsr_pa_plan *p);

/* Simulation-only check against Bob's labels (both uint8[frames][n]):
 * counts_out HOST int64[3] = {frames ok, ok frames whose labels differ from
 * Bob's (undetected errors), differing label bytes over ok frames}.  Syncs. */
cvsr_status cvsr_count_errors(cvsr_ctx *ctx, const uint8_t *label_alice, const uint8_t *label_bob,
                              const uint8_t *frame_ok, int32_t frames, int32_t n, int64_t *counts_out);

/* ------------------------------------------------------------- session */
/* One batch of the whole hot path (Bob + Alice) with library-owned device
 * buffers: cvsr_session_run = cvsr_quantise(y) -> cvsr_syndrome (coded
 * slices) / cvsr_slice_bits (disclosed slices) -> cvsr_reconcile(x).  The
 * codes must stay loaded while the session lives.  Errors as above; on
 * CVSR_ECUDA the session must be destroyed. */
typedef struct cvsr_session cvsr_session;
cvsr_status cvsr_session_create(cvsr_ctx *ctx, int32_t m, const cvsr_code *const *codes, const int32_t *order,
                                const cvsr_quantiser *q, float sigma_n, int32_t n, int32_t frames,
                                const cvsr_decode_opts *opts, cvsr_session **out);
/* x, y: DEVICE float[frames][n]; stats_out optional (synchronises). */
cvsr_status cvsr_session_run(cvsr_session *s, const float *x, const float *y, cvsr_stats *stats_out);
/* x_host, y_host: HOST float[frames][n] (pinned for overlap); copies them in,
 * runs the step and copies Alice's labels (label_host uint8[frames][n],
 * nullable), frame_ok_host uint8[frames] and iters_host int32[frames][m]
 * (nullable) back; synchronises.  This is the end-to-end entry point.  For
 * batches of >= 512 frames the work is split into 4 frame chunks so that the
 * next chunk's host-to-device copy and the previous chunk's device-to-host
 * copy overlap the current chunk's kernels; results do not depend on it. */
cvsr_status cvsr_session_run_host(cvsr_session *s, const float *x_host, const float *y_host, uint8_t *label_host,
                                  uint8_t *frame_ok_host, int32_t *iters_host, cvsr_stats *stats_out);

/* Streaming variant for a sequence of batches (the serving loop): batch b's
 * inputs x_host[b], y_host[b] (pinned host, float[frames][n]) are copied in
 * while batch b-1 is reconciled, and batch b's results (label_host[b]
 * uint8[frames][n], may be NULL; frame_ok_host[b] uint8[frames]) are copied out
 * while batch b+1 runs, using a second device buffer set allocated on the first
 * call.  Results per batch equal cvsr_session_run_host's.  Synchronous: returns
 * after the last result copy.  Per-batch statistics are not collected. */
cvsr_status cvsr_session_run_host_stream(cvsr_session *s, int32_t n_batches, const float *const *x_host,
                                         const float *const *y_host, uint8_t *const *label_host,
                                         uint8_t *const *frame_ok_host);

/* Hash verification inside the session step: keys != NULL (HOST
 * array of CVSR_HASH_KEYS keys, as cvsr_verify) makes every later run / run_host
 * call end with cvsr_verify on the session's labels, so frame_ok (device buffer
 * and frame_ok_host) reports "converged AND all hashes equal".  keys = NULL turns
 * it off (default).  stats_out counts are taken before the hash check. */
cvsr_status cvsr_session_set_verify(cvsr_session *s, const uint64_t *keys);

/* device pointers of the session's result buffers (any output may be NULL) */
cvsr_status cvsr_session_buffers(const cvsr_session *s, uint8_t **label_bob, uint8_t **label_alice,
                                 uint8_t **frame_ok, int32_t **iters);
void cvsr_session_destroy(cvsr_session *s);

#ifdef __cplusplus
}
#endif
#endif /* CVSR_H */
