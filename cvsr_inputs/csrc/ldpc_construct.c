/*
 * Seeded LDPC parity-check matrix construction (input generator, host only).
 *
 * This file builds the sparse parity-check matrices H_j that both the CUDA
 * path and the oracle consume as INPUT DATA.  It holds none of the method's
 * arithmetic (no quantiser, LLR or decoder): the paper does not specify how
 * its codes are built (PAPER.md:392 cites external degree distributions,
 * PAPER.md:413 mentions trapping-set-aware construction), so SURVEY.md §2.6
 * row 40a fixes the reading used here: a seeded configuration model (random
 * socket matching) for a prescribed variable/check degree sequence, followed
 * by duplicate-edge repair so that H has 0/1 entries, deterministic per seed.
 *
 * Output: CSR by check (row_ptr[M+1], col_idx[E]) with each row's column
 * indices sorted ascending.  G (the paper's number of non-zeros)
 * equals E = row_ptr[M].
 *
 * Degrees may be 0 (used when a structured part is merged in by the caller).
 * Error behaviour: returns 0 on success, -1 on bad arguments (degree sums
 * differ, degree < 0, degree > number of opposite nodes), -2 if duplicate
 * repair did not converge within its attempt budget, -3 on allocation failure.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* splitmix64: counter-based seeding of xoshiro256** */
static uint64_t splitmix64(uint64_t *s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

typedef struct { uint64_t s[4]; } rng_t;

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t rng_next(rng_t *r) {
    uint64_t *s = r->s;
    uint64_t result = rotl(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= t; s[3] = rotl(s[3], 45);
    return result;
}

static void rng_seed(rng_t *r, uint64_t seed) {
    uint64_t sm = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&sm);
}

/* unbiased integer in [0, bound) (Lemire's method) */
static uint64_t rng_below(rng_t *r, uint64_t bound) {
    uint64_t x = rng_next(r);
    __uint128_t m = (__uint128_t)x * bound;
    uint64_t l = (uint64_t)m;
    if (l < bound) {
        uint64_t t = (0 - bound) % bound;
        while (l < t) {
            x = rng_next(r);
            m = (__uint128_t)x * bound;
            l = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* does row [beg,end) of col contain v, ignoring position skip? */
static int row_has(const int32_t *col, int64_t beg, int64_t end, int64_t skip, int32_t v) {
    for (int64_t i = beg; i < end; ++i)
        if (i != skip && col[i] == v) return 1;
    return 0;
}

int ldpc_configuration_model(int32_t n_vars, int32_t n_checks,
                             const int32_t *var_deg, const int32_t *chk_deg,
                             uint64_t seed, int32_t *row_ptr, int32_t *col_idx) {
    if (n_vars <= 0 || n_checks <= 0 || !var_deg || !chk_deg || !row_ptr || !col_idx)
        return -1;
    int64_t ev = 0, ec = 0;
    for (int32_t v = 0; v < n_vars; ++v) {
        if (var_deg[v] < 0 || var_deg[v] > n_checks) return -1;
        ev += var_deg[v];
    }
    for (int32_t c = 0; c < n_checks; ++c) {
        if (chk_deg[c] < 0 || chk_deg[c] > n_vars) return -1;
        ec += chk_deg[c];
    }
    if (ev != ec || ev > INT32_MAX) return -1;
    const int64_t E = ev;

    rng_t rng;
    rng_seed(&rng, seed);

    /* variable sockets, shuffled (Fisher-Yates) */
    int64_t k = 0;
    for (int32_t v = 0; v < n_vars; ++v)
        for (int32_t d = 0; d < var_deg[v]; ++d) col_idx[k++] = v;
    for (int64_t i = E - 1; i > 0; --i) {
        int64_t j = (int64_t)rng_below(&rng, (uint64_t)(i + 1));
        int32_t t = col_idx[i]; col_idx[i] = col_idx[j]; col_idx[j] = t;
    }
    row_ptr[0] = 0;
    for (int32_t c = 0; c < n_checks; ++c) row_ptr[c + 1] = row_ptr[c] + chk_deg[c];

    /* row id of each edge position (for swap partner lookup) */
    int32_t *row_of = (int32_t *)malloc(sizeof(int32_t) * (size_t)E);
    if (!row_of) return -3;
    for (int32_t c = 0; c < n_checks; ++c)
        for (int32_t i = row_ptr[c]; i < row_ptr[c + 1]; ++i) row_of[i] = c;

    /* duplicate repair: swap a duplicated socket with a random socket of
       another row such that neither row ends up with a duplicate */
    int status = 0;
    for (int32_t c = 0; c < n_checks && status == 0; ++c) {
        int64_t beg = row_ptr[c], end = row_ptr[c + 1];
        for (int64_t i = beg; i < end; ++i) {
            int tries = 0;
            while (row_has(col_idx, beg, i, -1, col_idx[i])) {
                if (++tries > 100000) { status = -2; break; }
                int64_t p = (int64_t)rng_below(&rng, (uint64_t)E);
                int32_t c2 = row_of[p];
                if (c2 == c) continue;
                int32_t a = col_idx[i], b = col_idx[p];
                if (a == b) continue;
                /* after swap: row c holds b at i, row c2 holds a at p */
                if (row_has(col_idx, beg, end, i, b)) continue;
                if (row_has(col_idx, row_ptr[c2], row_ptr[c2 + 1], p, a)) continue;
                col_idx[i] = b; col_idx[p] = a;
            }
            if (status) break;
        }
    }
    free(row_of);
    if (status) return status;
    for (int32_t c = 0; c < n_checks; ++c)
        qsort(col_idx + row_ptr[c], (size_t)(row_ptr[c + 1] - row_ptr[c]), sizeof(int32_t), cmp_i32);
    return 0;
}

/* seeded Fisher-Yates permutation of [0, n) (used to scatter degree classes) */
int ldpc_permutation(int32_t n, uint64_t seed, int32_t *perm) {
    if (n <= 0 || !perm) return -1;
    rng_t rng;
    rng_seed(&rng, seed);
    for (int32_t i = 0; i < n; ++i) perm[i] = i;
    for (int32_t i = n - 1; i > 0; --i) {
        int32_t j = (int32_t)rng_below(&rng, (uint64_t)(i + 1));
        int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
    return 0;
}

/* ---------------------------------------------------------------- PEG (progressive edge growth)
 * Hu, Eleftheriou, Arnold: edges are placed one at a time, variables in order of increasing
 * degree; the k-th edge of v goes to a check outside the depth-limited BFS tree of v (so no
 * cycle shorter than 2 (depth + 2) is closed), else to a check on the deepest level, with the
 * lowest current degree among those (ties broken by the seed).  Check degrees follow the target
 * sequence chk_deg as capacities.  depth = number of check levels explored (e.g. 4).
 * Host-side input construction only (no method arithmetic).  Returns 0, or <0 on error. */
typedef struct {
    int32_t *items, *pos, *cnt, *start; /* bucket d = items[start[d] .. start[d] + cnt[d]) */
} buckets_t;

int ldpc_peg(int32_t n_vars, int32_t n_checks, const int32_t *var_deg, const int32_t *chk_deg, uint64_t seed,
             int32_t depth, int32_t *row_ptr, int32_t *col_idx) {
    if (n_vars <= 0 || n_checks <= 0 || !var_deg || !chk_deg || !row_ptr || !col_idx || depth < 1) return -1;
    int64_t E = 0, Ec = 0;
    int32_t maxcap = 0;
    for (int32_t v = 0; v < n_vars; ++v) E += var_deg[v];
    for (int32_t c = 0; c < n_checks; ++c) {
        Ec += chk_deg[c];
        if (chk_deg[c] > maxcap) maxcap = chk_deg[c];
    }
    if (E != Ec || E > INT32_MAX) return -1;
    rng_t rng;
    rng_seed(&rng, seed);
    /* adjacency with slack: checks may exceed their target by a few edges in the rare stuck case */
    const int32_t slack = 8;
    int32_t *var_off = (int32_t *)malloc(sizeof(int32_t) * ((size_t)n_vars + 1));
    int32_t *var_adj = (int32_t *)malloc(sizeof(int32_t) * (size_t)E);
    int32_t *var_cnt = (int32_t *)calloc((size_t)n_vars, sizeof(int32_t));
    int32_t *chk_off = (int32_t *)malloc(sizeof(int32_t) * ((size_t)n_checks + 1));
    int32_t *chk_adj = (int32_t *)malloc(sizeof(int32_t) * ((size_t)E + (size_t)n_checks * slack));
    int32_t *cur = (int32_t *)calloc((size_t)n_checks, sizeof(int32_t));
    int32_t *cstamp = (int32_t *)calloc((size_t)n_checks, sizeof(int32_t));
    int32_t *vstamp = (int32_t *)calloc((size_t)n_vars, sizeof(int32_t));
    int32_t *front = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_checks);
    int32_t *next = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_checks);
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_vars);
    /* buckets of checks with spare capacity, by current degree (0 .. maxcap - 1) */
    int32_t *b_items = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_checks * (size_t)maxcap);
    int32_t *b_cnt = (int32_t *)calloc((size_t)maxcap + 1, sizeof(int32_t));
    int32_t *b_pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_checks);
    int status = 0;
    if (!var_off || !var_adj || !var_cnt || !chk_off || !chk_adj || !cur || !cstamp || !vstamp || !front || !next ||
        !order || !b_items || !b_cnt || !b_pos) {
        status = -3;
        goto done;
    }
    var_off[0] = 0;
    for (int32_t v = 0; v < n_vars; ++v) var_off[v + 1] = var_off[v] + var_deg[v];
    chk_off[0] = 0;
    for (int32_t c = 0; c < n_checks; ++c) chk_off[c + 1] = chk_off[c] + chk_deg[c] + slack;
    /* bucket d holds checks of current degree d with cur < cap; stored in a [maxcap][n_checks] grid */
    for (int32_t c = 0; c < n_checks; ++c)
        if (chk_deg[c] > 0) {
            b_pos[c] = b_cnt[0];
            b_items[b_cnt[0]++] = c;
        }
    /* variable order: increasing degree, random within a degree */
    for (int32_t v = 0; v < n_vars; ++v) order[v] = v;
    for (int32_t i = n_vars - 1; i > 0; --i) {
        int32_t j = (int32_t)rng_below(&rng, (uint64_t)i + 1);
        int32_t t = order[i]; order[i] = order[j]; order[j] = t;
    }
    {   /* stable counting sort by degree */
        int32_t maxdv = 0;
        for (int32_t v = 0; v < n_vars; ++v) if (var_deg[v] > maxdv) maxdv = var_deg[v];
        int32_t *cnt = (int32_t *)calloc((size_t)maxdv + 2, sizeof(int32_t));
        int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)n_vars);
        if (!cnt || !tmp) { free(cnt); free(tmp); status = -3; goto done; }
        for (int32_t i = 0; i < n_vars; ++i) cnt[var_deg[order[i]] + 1]++;
        for (int32_t d = 0; d <= maxdv; ++d) cnt[d + 1] += cnt[d];
        for (int32_t i = 0; i < n_vars; ++i) tmp[cnt[var_deg[order[i]]]++] = order[i];
        memcpy(order, tmp, sizeof(int32_t) * (size_t)n_vars);
        free(cnt);
        free(tmp);
    }
    int32_t gen = 0;
    for (int32_t oi = 0; oi < n_vars && status == 0; ++oi) {
        const int32_t v = order[oi];
        for (int32_t k = 0; k < var_deg[v]; ++k) {
            ++gen;
            vstamp[v] = gen;
            int32_t nf = 0, reached = 0;
            for (int32_t i = 0; i < var_cnt[v]; ++i) {
                const int32_t c = var_adj[var_off[v] + i];
                if (cstamp[c] != gen) { cstamp[c] = gen; front[nf++] = c; ++reached; }
            }
            int32_t last_n = nf;
            int32_t *last = front;
            int32_t avail_total = 0;
            for (int32_t d = 0; d < maxcap; ++d) avail_total += b_cnt[d];
            for (int32_t lev = 1; lev < depth && nf > 0; ++lev) {
                int32_t nn = 0;
                for (int32_t i = 0; i < nf; ++i) {
                    const int32_t c = front[i];
                    for (int32_t p = chk_off[c]; p < chk_off[c] + cur[c]; ++p) {
                        const int32_t u = chk_adj[p];
                        if (vstamp[u] == gen) continue;
                        vstamp[u] = gen;
                        for (int32_t q = 0; q < var_cnt[u]; ++q) {
                            const int32_t c2 = var_adj[var_off[u] + q];
                            if (cstamp[c2] != gen) { cstamp[c2] = gen; next[nn++] = c2; ++reached; }
                        }
                    }
                }
                if (nn == 0) break;
                int32_t *t = front; front = next; next = t;
                nf = nn;
                last = front;
                last_n = nn;
            }
            (void)reached;
            /* lowest-degree available check outside the tree (random start within a bucket) */
            int32_t chosen = -1;
            for (int32_t d = 0; d < maxcap && chosen < 0; ++d) {
                const int32_t m = b_cnt[d];
                if (m == 0) continue;
                const int32_t *items = b_items + (size_t)d * n_checks;
                const int32_t s0 = (int32_t)rng_below(&rng, (uint64_t)m);
                for (int32_t i = 0; i < m; ++i) {
                    const int32_t c = items[(s0 + i) % m];
                    if (cstamp[c] != gen) { chosen = c; break; }
                }
            }
            if (chosen < 0) {
                /* every available check is in the tree: lowest-degree available check on the last
                   level that is not yet adjacent to v, else any non-adjacent check (exceeds target) */
                int32_t best = -1;
                for (int32_t i = 0; i < last_n; ++i) {
                    const int32_t c = last[i];
                    if (cur[c] >= chk_deg[c]) continue;
                    int adj = 0;
                    for (int32_t q = 0; q < var_cnt[v]; ++q) if (var_adj[var_off[v] + q] == c) { adj = 1; break; }
                    if (adj) continue;
                    if (best < 0 || cur[c] < cur[best]) best = c;
                }
                if (best < 0) {
                    for (int32_t c = 0; c < n_checks; ++c) {
                        if (cur[c] >= chk_deg[c] + slack) continue;
                        int adj = 0;
                        for (int32_t q = 0; q < var_cnt[v]; ++q) if (var_adj[var_off[v] + q] == c) { adj = 1; break; }
                        if (adj) continue;
                        if (best < 0 || cur[c] < cur[best]) best = c;
                    }
                }
                if (best < 0) { status = -2; break; }
                chosen = best;
            }
            (void)avail_total;
            /* add edge (v, chosen) */
            var_adj[var_off[v] + var_cnt[v]++] = chosen;
            chk_adj[chk_off[chosen] + cur[chosen]] = v;
            const int32_t d0 = cur[chosen];
            if (d0 < chk_deg[chosen]) {  /* remove from bucket d0 (swap-remove) */
                int32_t *items = b_items + (size_t)d0 * n_checks;
                const int32_t p = b_pos[chosen], lastc = items[--b_cnt[d0]];
                items[p] = lastc;
                b_pos[lastc] = p;
            }
            cur[chosen] = d0 + 1;
            if (cur[chosen] < chk_deg[chosen]) {
                int32_t *items = b_items + (size_t)cur[chosen] * n_checks;
                b_pos[chosen] = b_cnt[cur[chosen]];
                items[b_cnt[cur[chosen]]++] = chosen;
            }
        }
    }
    if (status == 0) {
        row_ptr[0] = 0;
        for (int32_t c = 0; c < n_checks; ++c) row_ptr[c + 1] = row_ptr[c] + cur[c];
        if ((int64_t)row_ptr[n_checks] != E) { status = -4; goto done; }
        for (int32_t c = 0; c < n_checks; ++c) {
            memcpy(col_idx + row_ptr[c], chk_adj + chk_off[c], sizeof(int32_t) * (size_t)cur[c]);
            qsort(col_idx + row_ptr[c], (size_t)cur[c], sizeof(int32_t), cmp_i32);
        }
    }
done:
    free(var_off); free(var_adj); free(var_cnt); free(chk_off); free(chk_adj); free(cur); free(cstamp);
    free(vstamp); free(front); free(next); free(order); free(b_items); free(b_cnt); free(b_pos);
    return status;
}
