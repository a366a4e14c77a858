/*
 * cvsr ORACLE -- plain, slow, fp64 CPU reference of the sliced-reconciliation
 * hot path of Ai & Malaney, arXiv 2108.08418 ("PAPER.md" below).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * in paper_2108_08418_b200/ (and includes nothing from it); the only common
 * inputs are the seeded data produced by cvsr_inputs/.
 *
 * Every function follows the plain definition (quantiser, syndrome) or the
 * algorithm step by step in the order of SURVEY.md §8(c) O2-O6, which fixes
 * the readings of PAPER.md where the paper is silent (A-1 .. A-22).  No
 * blocking, fusion or reordering: OpenMP parallelism is over independent
 * frames only.  Floating point is double throughout.
 *
 * Bit packing (SURVEY.md §8(b) conventions): bit i of a packed vector lives
 * at bit (i mod 32) of 32-bit word floor(i/32); padding bits are 0.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL (-1)

static int32_t words_of(int64_t bits) { return (int32_t)((bits + 31) / 32); }

static int get_bit(const uint32_t *w, int64_t i) { return (int)((w[i >> 5] >> (i & 31)) & 1u); }
static void set_bit(uint32_t *w, int64_t i, int b) {
    if (b) w[i >> 5] |= (1u << (i & 31));
    else w[i >> 5] &= ~(1u << (i & 31));
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------
 * O2  Quantiser M(.) with Gray labelling.
 * PAPER.md:114 step 1 ("constant-step quantisation function M(.)")
 * ("2^5 bins centered on zero"), PAPER.md:87 ("Using Gray Labelling"),
 * PAPER.md:114 footnote ("the least significant bit is l_0").
 * Definition (readings A-3, A-4): b(y) = #{k : y >= e_k} over the fp32 edge
 * table e_1 < ... < e_{2^m-1}; label = b XOR (b >> 1).  Comparison in float
 * (the inputs' precision), so ties go to the upper bin.
 * ---------------------------------------------------------------------- */
int orc_quantise(int32_t m, const float *edges, const float *y, int64_t count, uint8_t *label) {
    if (m < 1 || m > 8 || !edges || !y || !label || count < 0) return ORC_EINVAL;
    const int32_t ne = (1 << m) - 1;
    for (int64_t i = 0; i < count; ++i) {
        int32_t b = 0;
        for (int32_t k = 0; k < ne; ++k)
            if (y[i] >= edges[k]) b += 1;
        label[i] = (uint8_t)(b ^ (b >> 1));
    }
    return ORC_OK;
}

/* Slice extraction S_j = (l_j^0 ... l_j^{N_R-1}) (PAPER.md:114 step 2), packed. */
int orc_slice_bits(const uint8_t *label, int32_t frames, int32_t n, int32_t j, uint32_t *bits_out) {
    if (!label || !bits_out || frames < 0 || n < 0 || j < 0 || j > 7) return ORC_EINVAL;
    const int32_t W = words_of(n);
    for (int32_t f = 0; f < frames; ++f) {
        uint32_t *w = bits_out + (int64_t)f * W;
        memset(w, 0, sizeof(uint32_t) * (size_t)W);
        for (int32_t i = 0; i < n; ++i) set_bit(w, i, (label[(int64_t)f * n + i] >> j) & 1);
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------
 * O3  Syndrome s_j = H_j S_j over GF(2) ("encodes ... into syndrome
 * bits", PAPER.md:114 step 2).  Plain definition: s[c] = XOR of S_j[v] over
 * the columns v of row c.
 * ---------------------------------------------------------------------- */
int orc_syndrome(int32_t n, int32_t n_checks, const int32_t *row_ptr, const int32_t *col_idx,
                 const uint8_t *label, int32_t frames, int32_t j, uint32_t *synd_out) {
    if (n <= 0 || n_checks <= 0 || !row_ptr || !col_idx || !label || !synd_out || j < 0 || j > 7)
        return ORC_EINVAL;
    const int32_t W = words_of(n_checks);
    for (int32_t f = 0; f < frames; ++f) {
        const uint8_t *lab = label + (int64_t)f * n;
        uint32_t *s = synd_out + (int64_t)f * W;
        memset(s, 0, sizeof(uint32_t) * (size_t)W);
        for (int32_t c = 0; c < n_checks; ++c) {
            int par = 0;
            for (int32_t e = row_ptr[c]; e < row_ptr[c + 1]; ++e) par ^= (lab[col_idx[e]] >> j) & 1;
            set_bit(s, c, par);
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------
 * O4  Conditional LLR of slice j (PAPER.md:114 step 4: Alice "uses her
 * quadrature values as side information"; reading A-2: conditioned on the
 * hard decisions of the already-known slices K).
 *   y = x + n, n ~ N(0, sigma_n^2) (reading A-5)
 *   P_b(x) = Phi((e_{b+1}-x)/sigma_n) - Phi((e_b-x)/sigma_n), e_0=-inf, e_{2^m}=+inf
 *   N_beta = sum{ P_b : bits_K(g(b)) = kappa, bit_j(g(b)) = beta }
 *   L = clamp(ln N_0 - ln N_1, -LLR_MAX, +LLR_MAX)   (positive => bit 0)
 * Evaluated in the log domain.
 * ---------------------------------------------------------------------- */
static const double SQRT1_2 = 0.70710678118654752440;
static const double HALF_LOG_2PI = 0.91893853320467274178;

/* log Q(z), Q(z) = P(N(0,1) > z) (PAPER.md eq. after eq:R_Finite defines Q) */
static double log_q(double z) {
    if (z < 0.0) return log1p(-0.5 * erfc(-z * SQRT1_2));
    if (z < 35.0) return log(0.5 * erfc(z * SQRT1_2));
    /* asymptotic series of the Mills ratio for large z */
    double iz2 = 1.0 / (z * z);
    double s = 1.0 - iz2 * (1.0 - iz2 * (3.0 - iz2 * (15.0 - iz2 * 105.0)));
    return -0.5 * z * z - log(z) - HALF_LOG_2PI + log(s);
}

/* log P(lo <= Z < hi) for a standard normal Z, lo < hi, either may be infinite */
static double log_bin(double lo, double hi) {
    if (isinf(lo) && lo < 0 && isinf(hi) && hi > 0) return 0.0;
    if (isinf(lo) && lo < 0) return log_q(-hi);
    if (isinf(hi) && hi > 0) return log_q(lo);
    if (lo >= 0.0) {
        double a = log_q(lo), b = log_q(hi);
        return a + log1p(-exp(b - a));
    }
    if (hi <= 0.0) {
        double a = log_q(-hi), b = log_q(-lo);
        return a + log1p(-exp(b - a));
    }
    return log(0.5 * (erf(hi * SQRT1_2) + erf(-lo * SQRT1_2)));
}

static double log_add(double a, double b) {
    if (isinf(a) && a < 0) return b;
    if (isinf(b) && b < 0) return a;
    double mx = a > b ? a : b, mn = a > b ? b : a;
    return mx + log1p(exp(mn - mx));
}

static double llr_one(int32_t m, const float *edges, double sigma_n, double x, int32_t j,
                      uint32_t known_mask, uint32_t kappa, double llr_max) {
    const int32_t nb = 1 << m;
    double ln0 = -INFINITY, ln1 = -INFINITY;
    for (int32_t b = 0; b < nb; ++b) {
        uint32_t g = (uint32_t)(b ^ (b >> 1));
        if ((g & known_mask) != (kappa & known_mask)) continue;
        double lo = (b == 0) ? -INFINITY : ((double)edges[b - 1] - x) / sigma_n;
        double hi = (b == nb - 1) ? INFINITY : ((double)edges[b] - x) / sigma_n;
        double lp = log_bin(lo, hi);
        if ((g >> j) & 1u) ln1 = log_add(ln1, lp);
        else ln0 = log_add(ln0, lp);
    }
    if (isinf(ln0) && ln0 < 0) return -llr_max;
    if (isinf(ln1) && ln1 < 0) return llr_max;
    double L = ln0 - ln1;
    if (L > llr_max) L = llr_max;
    if (L < -llr_max) L = -llr_max;
    return L;
}

int orc_llr_slice(int32_t m, const float *edges, double sigma_n, const float *x, int32_t frames,
                  int32_t n, int32_t j, uint32_t known_mask, const uint8_t *known_label,
                  double llr_max, double *llr_out) {
    if (m < 1 || m > 8 || !edges || !x || !llr_out || j < 0 || j >= m || sigma_n <= 0) return ORC_EINVAL;
    if ((known_mask >> j) & 1u) return ORC_EINVAL;
    if (known_mask && !known_label) return ORC_EINVAL;
    const int64_t total = (int64_t)frames * n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < total; ++i) {
        uint32_t kappa = known_mask ? known_label[i] : 0u;
        llr_out[i] = llr_one(m, edges, sigma_n, (double)x[i], j, known_mask, kappa, llr_max);
    }
    return ORC_OK;
}

/* BI-AWGN channel LLR for config C1 (reading A-16): L = clamp(2y/sigma^2). */
int orc_llr_biawgn(const float *y, int64_t count, double sigma2, double llr_max, double *llr_out) {
    if (!y || !llr_out || sigma2 <= 0) return ORC_EINVAL;
    for (int64_t i = 0; i < count; ++i) {
        double L = 2.0 * (double)y[i] / sigma2;
        llr_out[i] = L > llr_max ? llr_max : (L < -llr_max ? -llr_max : L);
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------
 * O5  Syndrome-based flooding sum-product BP ("the well-known
 * Belief Propagation (BP) decoder"; PAPER.md:231 message passing to checks and
 * back; readings A-8 flooding, A-10 V2C clamp, A-12 stopping rule).
 * Per frame:
 *  1. q_e <- clamp(L_v(e), +-Q_MAX); k = 0: xhat = [L < 0]; if H xhat = s stop (D = 0).
 *  2. for k = 1..max_iter:
 *     CN: r_e = (1 - 2 s_c) * BOXPLUS_{e' in row(c), e' != e} q_e'  (fold left to
 *         right in CSR order; empty fold = +Q_MAX)
 *         a [+] b = sgn(a)sgn(b) min(|a|,|b|) + log1p(e^-|a+b|) - log1p(e^-|a-b|)
 *     VN: post_v = L_v + sum_{e in col(v)} r_e; q_e = clamp(post_v - r_e, +-Q_MAX);
 *         xhat_v = [post_v < 0]
 *     check: if H xhat = s stop (converged, D = k)
 *  3. else: xhat of iteration max_iter, not converged, D = max_iter.
 * ---------------------------------------------------------------------- */
static double sgn(double a) { return a < 0.0 ? -1.0 : 1.0; }

static double boxplus(double a, double b) {
    double aa = fabs(a), ab = fabs(b);
    return sgn(a) * sgn(b) * (aa < ab ? aa : ab) + log1p(exp(-fabs(a + b))) - log1p(exp(-fabs(a - b)));
}

static double clampd(double v, double lim) { return v > lim ? lim : (v < -lim ? -lim : v); }

typedef struct {
    int32_t n, M;
    const int32_t *row_ptr, *col_idx;
    /* CSC built by the oracle itself (plain counting sort) */
    int32_t *col_ptr, *col_edge; /* col_edge: CSR edge ids in column order */
} orc_graph;

static int graph_init(orc_graph *g, int32_t n, int32_t M, const int32_t *row_ptr, const int32_t *col_idx) {
    g->n = n; g->M = M; g->row_ptr = row_ptr; g->col_idx = col_idx;
    const int64_t E = row_ptr[M];
    g->col_ptr = (int32_t *)calloc((size_t)n + 1, sizeof(int32_t));
    g->col_edge = (int32_t *)malloc(sizeof(int32_t) * (size_t)(E > 0 ? E : 1));
    if (!g->col_ptr || !g->col_edge) return ORC_EINVAL;
    for (int64_t e = 0; e < E; ++e) {
        if (col_idx[e] < 0 || col_idx[e] >= n) return ORC_EINVAL;
        g->col_ptr[col_idx[e] + 1]++;
    }
    for (int32_t v = 0; v < n; ++v) g->col_ptr[v + 1] += g->col_ptr[v];
    int32_t *fill = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!fill) return ORC_EINVAL;
    memcpy(fill, g->col_ptr, sizeof(int32_t) * (size_t)n);
    for (int64_t e = 0; e < E; ++e) g->col_edge[fill[col_idx[e]]++] = (int32_t)e;
    free(fill);
    return ORC_OK;
}

static void graph_free(orc_graph *g) { free(g->col_ptr); free(g->col_edge); }

static int syndrome_ok(const orc_graph *g, const uint8_t *xhat, const uint32_t *s) {
    for (int32_t c = 0; c < g->M; ++c) {
        int par = 0;
        for (int32_t e = g->row_ptr[c]; e < g->row_ptr[c + 1]; ++e) par ^= xhat[g->col_idx[e]];
        if (par != get_bit(s, c)) return 0;
    }
    return 1;
}

/* one flooding iteration: CN then VN (fills r, q, post, xhat) */
static void bp_iteration(const orc_graph *g, const double *L, const uint32_t *s, double q_max,
                         double *q, double *r, double *post, uint8_t *xhat) {
    for (int32_t c = 0; c < g->M; ++c) {
        const int32_t beg = g->row_ptr[c], end = g->row_ptr[c + 1];
        const double sign_c = get_bit(s, c) ? -1.0 : 1.0;
        for (int32_t e = beg; e < end; ++e) {
            int have = 0;
            double acc = 0.0;
            for (int32_t e2 = beg; e2 < end; ++e2) {
                if (e2 == e) continue;
                acc = have ? boxplus(acc, q[e2]) : q[e2];
                have = 1;
            }
            r[e] = sign_c * (have ? acc : q_max);
        }
    }
    for (int32_t v = 0; v < g->n; ++v) {
        double p = L[v];
        for (int32_t k = g->col_ptr[v]; k < g->col_ptr[v + 1]; ++k) p += r[g->col_edge[k]];
        post[v] = p;
        for (int32_t k = g->col_ptr[v]; k < g->col_ptr[v + 1]; ++k) {
            int32_t e = g->col_edge[k];
            q[e] = clampd(p - r[e], q_max);
        }
        xhat[v] = p < 0.0 ? 1 : 0;
    }
}

static void bp_init(const orc_graph *g, const double *L, double q_max, double *q, uint8_t *xhat) {
    for (int32_t c = 0; c < g->M; ++c)
        for (int32_t e = g->row_ptr[c]; e < g->row_ptr[c + 1]; ++e) q[e] = clampd(L[g->col_idx[e]], q_max);
    for (int32_t v = 0; v < g->n; ++v) xhat[v] = L[v] < 0.0 ? 1 : 0;
}

/* decode one frame; returns D, sets *conv */
static int32_t bp_frame(const orc_graph *g, const double *L, const uint32_t *s, int32_t max_iter,
                        double q_max, uint8_t *xhat, int *conv) {
    const int64_t E = g->row_ptr[g->M];
    double *q = (double *)malloc(sizeof(double) * (size_t)(E + 1));
    double *r = (double *)malloc(sizeof(double) * (size_t)(E + 1));
    double *post = (double *)malloc(sizeof(double) * (size_t)g->n);
    bp_init(g, L, q_max, q, xhat);
    int32_t D = 0;
    *conv = syndrome_ok(g, xhat, s);
    for (int32_t k = 1; k <= max_iter && !*conv; ++k) {
        bp_iteration(g, L, s, q_max, q, r, post, xhat);
        D = k;
        *conv = syndrome_ok(g, xhat, s);
    }
    free(q); free(r); free(post);
    return D;
}

int orc_bp_decode(int32_t n, int32_t n_checks, const int32_t *row_ptr, const int32_t *col_idx,
                  const double *llr, const uint32_t *synd, int32_t frames, int32_t max_iter,
                  double q_max, uint32_t *bits_out, uint8_t *converged_out, int32_t *iters_out) {
    if (n <= 0 || n_checks <= 0 || !row_ptr || !col_idx || !llr || !synd || max_iter < 0) return ORC_EINVAL;
    orc_graph g;
    if (graph_init(&g, n, n_checks, row_ptr, col_idx) != ORC_OK) { graph_free(&g); return ORC_EINVAL; }
    const int32_t Wn = words_of(n), Wm = words_of(n_checks);
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t f = 0; f < frames; ++f) {
        uint8_t *xhat = (uint8_t *)malloc((size_t)n);
        int conv = 0;
        int32_t D = bp_frame(&g, llr + (int64_t)f * n, synd + (int64_t)f * Wm, max_iter, q_max, xhat, &conv);
        uint32_t *w = bits_out + (int64_t)f * Wn;
        memset(w, 0, sizeof(uint32_t) * (size_t)Wn);
        for (int32_t v = 0; v < n; ++v) set_bit(w, v, xhat[v]);
        converged_out[f] = (uint8_t)conv;
        iters_out[f] = D;
        free(xhat);
    }
    graph_free(&g);
    return ORC_OK;
}

/* exactly k iterations, no early stop; C2V (CSR edge order) and posteriors of iteration k */
int orc_bp_trace(int32_t n, int32_t n_checks, const int32_t *row_ptr, const int32_t *col_idx,
                 const double *llr, const uint32_t *synd, int32_t frames, int32_t k_iters,
                 double q_max, double *c2v_out, double *post_out) {
    if (n <= 0 || n_checks <= 0 || k_iters < 1) return ORC_EINVAL;
    orc_graph g;
    if (graph_init(&g, n, n_checks, row_ptr, col_idx) != ORC_OK) { graph_free(&g); return ORC_EINVAL; }
    const int64_t E = row_ptr[n_checks];
    const int32_t Wm = words_of(n_checks);
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t f = 0; f < frames; ++f) {
        double *q = (double *)malloc(sizeof(double) * (size_t)(E + 1));
        uint8_t *xhat = (uint8_t *)malloc((size_t)n);
        const double *L = llr + (int64_t)f * n;
        bp_init(&g, L, q_max, q, xhat);
        for (int32_t k = 1; k <= k_iters; ++k)
            bp_iteration(&g, L, synd + (int64_t)f * Wm, q_max, q, c2v_out + (int64_t)f * E,
                         post_out + (int64_t)f * n, xhat);
        free(q); free(xhat);
    }
    graph_free(&g);
    return ORC_OK;
}

/* ------------------------------------------------------------------------
 * O5'  Row-layered schedule (reading R-9; PAPER.md:189 names BP
 * without fixing its schedule).  Same stopping rule, clamps and check rule
 * as O5; only the order of the message updates differs.
 *   Layers: greedy colouring of the checks in index order -- check c takes
 *     the smallest colour not taken by a check c' < c sharing a variable with
 *     it.  Checks of one layer share no variable.
 *   Init: r_e = 0, post_v = L_v, xhat_v = [L_v < 0]; test H xhat = s (D = 0).
 *   Iteration k: for layer l = 0, 1, ...: for every check c of layer l:
 *       q_e = post_v - r_e                       (e = (c, v))
 *       r_e <- (1 - 2 s_c) BOXPLUS_{e' != e} clamp(q_e', +-Q_MAX)
 *       post_v <- q_e + r_e
 *     then xhat_v = [post_v < 0]; test H xhat = s (D = k).
 * ---------------------------------------------------------------------- */
int orc_layers(int32_t n, int32_t n_checks, const int32_t *row_ptr, const int32_t *col_idx, int32_t *colour_out) {
    if (n <= 0 || n_checks <= 0 || !row_ptr || !col_idx || !colour_out) return ORC_EINVAL;
    orc_graph g;
    if (graph_init(&g, n, n_checks, row_ptr, col_idx) != ORC_OK) { graph_free(&g); return ORC_EINVAL; }
    /* the checks sharing a variable with c are the checks of the CSC columns of c's variables */
    int32_t *chk_of_edge = (int32_t *)malloc(sizeof(int32_t) * (size_t)(row_ptr[n_checks] + 1));
    for (int32_t c = 0; c < n_checks; ++c)
        for (int32_t e = row_ptr[c]; e < row_ptr[c + 1]; ++e) chk_of_edge[e] = c;
    int32_t max_colour = 0;
    for (int32_t c = 0; c < n_checks; ++c) {
        int32_t k = 0;
        for (;;) { /* smallest k not taken by an earlier neighbouring check */
            int taken = 0;
            for (int32_t e = row_ptr[c]; e < row_ptr[c + 1] && !taken; ++e) {
                const int32_t v = col_idx[e];
                for (int32_t p = g.col_ptr[v]; p < g.col_ptr[v + 1]; ++p) {
                    const int32_t c2 = chk_of_edge[g.col_edge[p]];
                    if (c2 < c && colour_out[c2] == k) { taken = 1; break; }
                }
            }
            if (!taken) break;
            ++k;
        }
        colour_out[c] = k;
        if (k > max_colour) max_colour = k;
    }
    free(chk_of_edge);
    graph_free(&g);
    return max_colour + 1;
}

static void layered_iteration(const orc_graph *g, const int32_t *colour, int32_t n_layers, const uint32_t *s,
                              double q_max, double *r, double *post, double *q, uint8_t *xhat) {
    for (int32_t l = 0; l < n_layers; ++l) {
        for (int32_t c = 0; c < g->M; ++c) {
            if (colour[c] != l) continue;
            const int32_t beg = g->row_ptr[c], end = g->row_ptr[c + 1];
            const double sign_c = get_bit(s, c) ? -1.0 : 1.0;
            for (int32_t e = beg; e < end; ++e) q[e] = post[g->col_idx[e]] - r[e];
            for (int32_t e = beg; e < end; ++e) {
                int have = 0;
                double acc = 0.0;
                for (int32_t e2 = beg; e2 < end; ++e2) {
                    if (e2 == e) continue;
                    const double qc = clampd(q[e2], q_max);
                    acc = have ? boxplus(acc, qc) : qc;
                    have = 1;
                }
                r[e] = sign_c * (have ? acc : q_max);
            }
            for (int32_t e = beg; e < end; ++e) post[g->col_idx[e]] = q[e] + r[e];
        }
    }
    for (int32_t v = 0; v < g->n; ++v) xhat[v] = post[v] < 0.0 ? 1 : 0;
}

/* One frame of the layered decoder: r (E entries) and post (n) are the frame's state.
 * stop_early = 1: the O5 stopping rule (first k with H xhat = s); 0: exactly max_iter
 * iterations (trace).  Returns D, sets *conv. */
static int32_t bp_frame_layered(const orc_graph *g, const int32_t *colour, int32_t n_layers, const double *L,
                                const uint32_t *s, int32_t max_iter, double q_max, int stop_early, uint8_t *xhat,
                                int *conv, double *r, double *post) {
    const int64_t E = g->row_ptr[g->M];
    double *q = (double *)malloc(sizeof(double) * (size_t)(E + 1));
    for (int64_t e = 0; e < E; ++e) r[e] = 0.0;
    for (int32_t v = 0; v < g->n; ++v) {
        post[v] = L[v];
        xhat[v] = L[v] < 0.0 ? 1 : 0;
    }
    *conv = syndrome_ok(g, xhat, s);
    int32_t D = 0;
    for (int32_t k = 1; k <= max_iter && !(stop_early && *conv); ++k) {
        layered_iteration(g, colour, n_layers, s, q_max, r, post, q, xhat);
        D = k;
        *conv = syndrome_ok(g, xhat, s);
    }
    free(q);
    return D;
}

/* stop_early = 1: decode (O5 stopping rule); 0: exactly max_iter iterations (trace).
 * post_out (nullable): posteriors [frames][n] when the frame stops; r_out (nullable): the
 * check-to-variable messages r_e [frames][E] (CSR edge order) when the frame stops. */
int orc_bp_layered(int32_t n, int32_t n_checks, const int32_t *row_ptr, const int32_t *col_idx,
                   const double *llr, const uint32_t *synd, int32_t frames, int32_t max_iter, double q_max,
                   int stop_early, uint32_t *bits_out, uint8_t *converged_out, int32_t *iters_out,
                   double *post_out, double *r_out) {
    if (n <= 0 || n_checks <= 0 || !row_ptr || !col_idx || !llr || !synd || max_iter < 0) return ORC_EINVAL;
    int32_t *colour = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_checks);
    if (!colour) return ORC_EINVAL;
    const int32_t n_layers = orc_layers(n, n_checks, row_ptr, col_idx, colour);
    orc_graph g;
    if (n_layers <= 0 || graph_init(&g, n, n_checks, row_ptr, col_idx) != ORC_OK) {
        free(colour);
        return ORC_EINVAL;
    }
    const int64_t E = row_ptr[n_checks];
    const int32_t Wn = words_of(n), Wm = words_of(n_checks);
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t f = 0; f < frames; ++f) {
        double *r = (double *)malloc(sizeof(double) * (size_t)(E + 1));
        double *post = (double *)malloc(sizeof(double) * (size_t)n);
        uint8_t *xhat = (uint8_t *)malloc((size_t)n);
        int conv = 0;
        const int32_t D = bp_frame_layered(&g, colour, n_layers, llr + (int64_t)f * n, synd + (int64_t)f * Wm,
                                           max_iter, q_max, stop_early, xhat, &conv, r, post);
        if (bits_out) {
            uint32_t *w = bits_out + (int64_t)f * Wn;
            memset(w, 0, sizeof(uint32_t) * (size_t)Wn);
            for (int32_t v = 0; v < n; ++v) set_bit(w, v, xhat[v]);
        }
        if (converged_out) converged_out[f] = (uint8_t)conv;
        if (iters_out) iters_out[f] = D;
        if (post_out) memcpy(post_out + (int64_t)f * n, post, sizeof(double) * (size_t)n);
        if (r_out) memcpy(r_out + (int64_t)f * E, r, sizeof(double) * (size_t)E);
        free(r); free(post); free(xhat);
    }
    graph_free(&g);
    free(colour);
    return ORC_OK;
}

/* ------------------------------------------------------------------------
 * O6  Multi-stage slice driver (PAPER.md:114 steps 4-6, Fig. 3), per frame:
 *   K = {}; for j in order:
 *     disclosed slice (codes[j] == NULL): Alice's l_j := Bob's l_j (bits passed in
 *       synd[j]), K += {j}
 *     else: L <- O4(x, K); decode with (H_j, s_j) -- O5 flooding (schedule 0) or the
 *       row-layered O5' (schedule 1, reading R-9); Alice's l_j <- xhat;
 *       not converged => frame fails, later slices not attempted (A-13);
 *       else K += {j}.
 * Outputs: Alice's labels, frame_ok, iters[f][j] (= D; 0 disclosed; -1 not attempted).
 * ---------------------------------------------------------------------- */
int orc_reconcile(int32_t m, int32_t n, const int32_t *n_checks, const int32_t *const *row_ptrs,
                  const int32_t *const *col_idxs, const int32_t *order, const float *edges,
                  double sigma_n, const float *x, const uint32_t *const *synd, int32_t frames,
                  int32_t max_iter, double q_max, double llr_max, int32_t schedule, uint8_t *label_out,
                  uint8_t *frame_ok, int32_t *iters) {
    if (m < 1 || m > 8 || n <= 0 || !order || !edges || !x || !synd || !label_out || !frame_ok || !iters)
        return ORC_EINVAL;
    if (schedule != 0 && schedule != 1) return ORC_EINVAL;
    orc_graph g[8];
    int32_t *colour[8];
    int32_t n_layers[8];
    memset(g, 0, sizeof(g));
    memset(colour, 0, sizeof(colour));
    memset(n_layers, 0, sizeof(n_layers));
    for (int32_t j = 0; j < m; ++j) {
        if (!row_ptrs[j]) continue;
        if (graph_init(&g[j], n, n_checks[j], row_ptrs[j], col_idxs[j]) != ORC_OK) return ORC_EINVAL;
        if (schedule == 1) {
            colour[j] = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_checks[j]);
            n_layers[j] = orc_layers(n, n_checks[j], row_ptrs[j], col_idxs[j], colour[j]);
            if (n_layers[j] <= 0) return ORC_EINVAL;
        }
    }
    const int32_t Wn = words_of(n);
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t f = 0; f < frames; ++f) {
        uint8_t *lab = label_out + (int64_t)f * n;
        uint8_t *xhat = (uint8_t *)malloc((size_t)n);
        double *L = (double *)malloc(sizeof(double) * (size_t)n);
        memset(lab, 0, (size_t)n);
        uint32_t known = 0;
        int ok = 1;
        for (int32_t t = 0; t < m; ++t) iters[(int64_t)f * m + t] = -1;
        for (int32_t t = 0; t < m && ok; ++t) {
            const int32_t j = order[t];
            if (!row_ptrs[j]) {
                const uint32_t *bits = synd[j] + (int64_t)f * Wn;
                for (int32_t v = 0; v < n; ++v) lab[v] |= (uint8_t)(get_bit(bits, v) << j);
                iters[(int64_t)f * m + j] = 0;
                known |= 1u << j;
                continue;
            }
            for (int32_t v = 0; v < n; ++v)
                L[v] = llr_one(m, edges, sigma_n, (double)x[(int64_t)f * n + v], j, known, lab[v], llr_max);
            int conv = 0;
            const int32_t Wm = words_of(n_checks[j]);
            const uint32_t *sj = synd[j] + (int64_t)f * Wm;
            int32_t D;
            if (schedule == 1) {
                double *r = (double *)malloc(sizeof(double) * (size_t)(row_ptrs[j][n_checks[j]] + 1));
                double *post = (double *)malloc(sizeof(double) * (size_t)n);
                D = bp_frame_layered(&g[j], colour[j], n_layers[j], L, sj, max_iter, q_max, 1, xhat, &conv, r, post);
                free(r); free(post);
            } else {
                D = bp_frame(&g[j], L, sj, max_iter, q_max, xhat, &conv);
            }
            for (int32_t v = 0; v < n; ++v) lab[v] |= (uint8_t)(xhat[v] << j);
            iters[(int64_t)f * m + j] = D;
            if (!conv) ok = 0;
            else known |= 1u << j;
        }
        frame_ok[f] = (uint8_t)ok;
        free(xhat); free(L);
    }
    for (int32_t j = 0; j < m; ++j) {
        if (row_ptrs[j]) graph_free(&g[j]);
        free(colour[j]);
    }
    return ORC_OK;
}
