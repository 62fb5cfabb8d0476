/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Never linked into the product path.
 *
 * CPU restatement of the reference's fleet-feasibility predicate
 * (reference pkg/src/carbon_sched/mig.py:144-181, MigTopology._partition_search /
 * is_feasible_fleet): a slice-count vector is feasible on n GPUs iff it is the sum
 * of exactly n partition-table rows.  The reference decides this by memoised
 * backtracking; this file decides the same predicate by the sum-set dynamic
 * programme T_N = U_k (T_{N-1} + row_k) over the rows without a 7g slice, with
 * the 7g count handled separately (a 7g slice fills a whole GPU, so it only
 * occurs in the single-slice row {7g}).  Equivalence with the reference is
 * pinned exhaustively for n <= 6 by tests/test_oracle_feasibility.py against
 * /root/reference (and by the committed golden counts |F_n|).
 *
 * Layout (deliberately different from the device tables): for each N, keys
 * (b, c, d) = (#4g, #3g, #2g) with 4b+3c+2d <= 7N are numbered in lexicographic
 * order; each key owns W_N = ceil((7N+1)/64) uint64 words, bit e = #1g.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int nmax;
    int nrows;
    int rows[32][4];          /* (b, c, d, e) of the non-7g rows */
    int has7g;
    int64_t *bc_first[129];   /* per N: first key index of (b, c), dense [b][c] */
    int bdim[129], cdim[129];
    int64_t nkeys[129];
    int words[129];
    uint64_t *bits[129];
} feas_t;

static int64_t key_of(const feas_t *f, int N, int b, int c, int d) {
    if (b < 0 || c < 0 || d < 0) return -1;
    if (4 * b + 3 * c + 2 * d > 7 * N) return -1;
    return f->bc_first[N][b * f->cdim[N] + c] + d;
}

static int test_bit(const feas_t *f, int N, int b, int c, int d, int e) {
    if (e < 0) return 0;
    int64_t k = key_of(f, N, b, c, d);
    if (k < 0) return 0;
    if (4 * b + 3 * c + 2 * d + e > 7 * N) return 0;
    const uint64_t *w = f->bits[N] + k * f->words[N];
    return (int)((w[e >> 6] >> (e & 63)) & 1u);
}

void feas_free(void *h) {
    feas_t *f = (feas_t *)h;
    if (!f) return;
    for (int N = 0; N <= f->nmax; ++N) { free(f->bc_first[N]); free(f->bits[N]); }
    free(f);
}

/* rows5: K x 5 slice-count rows (7g,4g,3g,2g,1g).  Returns NULL on bad input. */
void *feas_build(const int *rows5, int K, int nmax) {
    if (nmax < 0 || nmax > 128 || K < 1 || K > 64) return NULL;
    feas_t *f = (feas_t *)calloc(1, sizeof(feas_t));
    f->nmax = nmax;
    for (int k = 0; k < K; ++k) {
        const int *r = rows5 + 5 * k;
        if (r[0] > 0) { f->has7g = 1; continue; }   /* {7g} row: handled by the 7g count */
        int dup = 0;
        for (int j = 0; j < f->nrows; ++j)
            if (!memcmp(f->rows[j], r + 1, 4 * sizeof(int))) dup = 1;
        if (dup) continue;
        if (f->nrows >= 32) { feas_free(f); return NULL; }
        memcpy(f->rows[f->nrows++], r + 1, 4 * sizeof(int));
    }
    for (int N = 0; N <= nmax; ++N) {
        int cap = 7 * N;
        f->bdim[N] = cap / 4 + 1;
        f->cdim[N] = cap / 3 + 1;
        f->bc_first[N] = (int64_t *)malloc(sizeof(int64_t) * f->bdim[N] * f->cdim[N]);
        int64_t nk = 0;
        for (int b = 0; b < f->bdim[N]; ++b)
            for (int c = 0; c < f->cdim[N]; ++c) {
                f->bc_first[N][b * f->cdim[N] + c] = nk;
                int rem = cap - 4 * b - 3 * c;
                if (rem >= 0) nk += rem / 2 + 1;
            }
        f->nkeys[N] = nk;
        f->words[N] = (cap + 1 + 63) / 64;
        f->bits[N] = (uint64_t *)calloc((size_t)nk * f->words[N], sizeof(uint64_t));
        if (!f->bits[N]) { feas_free(f); return NULL; }
        if (N == 0) { f->bits[0][0] = 1u; continue; }
        /* T_N(b,c,d,e) = OR_k T_{N-1}(b-rb, c-rc, d-rd, e-re) */
        for (int b = 0; b < f->bdim[N]; ++b)
            for (int c = 0; c < f->cdim[N]; ++c) {
                int rem = cap - 4 * b - 3 * c;
                if (rem < 0) continue;
                for (int d = 0; d <= rem / 2; ++d) {
                    uint64_t *out = f->bits[N] + (f->bc_first[N][b * f->cdim[N] + c] + d) * f->words[N];
                    int emax = rem - 2 * d;
                    for (int k = 0; k < f->nrows; ++k) {
                        const int *r = f->rows[k];
                        int64_t sk = key_of(f, N - 1, b - r[0], c - r[1], d - r[2]);
                        if (sk < 0) continue;
                        const uint64_t *src = f->bits[N - 1] + sk * f->words[N - 1];
                        int sw = f->words[N - 1];
                        /* out bit e <- src bit (e - re), word by word */
                        int re = r[3];
                        for (int w = 0; w < f->words[N]; ++w) {
                            int lo = w * 64 - re;
                            uint64_t v;
                            if (lo < 0) {
                                v = src[0] << re;
                            } else {
                                int q = lo / 64, sh = lo % 64;
                                uint64_t a = q < sw ? src[q] : 0;
                                uint64_t nx = q + 1 < sw ? src[q + 1] : 0;
                                v = sh ? ((a >> sh) | (nx << (64 - sh))) : a;
                            }
                            out[w] |= v;
                        }
                    }
                    /* clear bits beyond the valid e range */
                    for (int w = 0; w < f->words[N]; ++w) {
                        int first = w * 64;
                        if (first > emax) out[w] = 0;
                        else if (emax - first < 63) out[w] &= (2ull << (emax - first)) - 1;
                    }
                }
            }
    }
    return f;
}

int feas_nmax(void *h) { return ((feas_t *)h)->nmax; }

/* vector (a,b,c,d,e) on exactly n GPUs */
int feas_query(void *h, int n, int a, int b, int c, int d, int e) {
    feas_t *f = (feas_t *)h;
    if (n < 1 || a < 0 || a > n) return 0;
    if (a > 0 && !f->has7g) return 0;
    int N = n - a;
    if (N > f->nmax) return -1;
    return test_bit(f, N, b, c, d, e);
}

void feas_query_batch(void *h, int n, const int32_t *vec5, int64_t count, uint8_t *out) {
    for (int64_t i = 0; i < count; ++i) {
        const int32_t *v = vec5 + 5 * i;
        int r = feas_query(h, n, v[0], v[1], v[2], v[3], v[4]);
        out[i] = (uint8_t)(r > 0);
    }
}

/* |{(b,c,d,e) in T_N}| and |F_n| = sum over a of |T_{n-a}| (the golden counts) */
int64_t feas_count_T(void *h, int N) {
    feas_t *f = (feas_t *)h;
    int64_t total = 0;
    for (int64_t i = 0; i < f->nkeys[N] * f->words[N]; ++i)
        total += __builtin_popcountll(f->bits[N][i]);
    return total;
}
