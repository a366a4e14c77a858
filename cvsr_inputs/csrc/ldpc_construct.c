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
