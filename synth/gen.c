/*
 * synth/gen.c -- seeded synthetic inputs for the SpMxV hot path.
 *
 * This module is the ONLY code shared by the oracle side (oracle/, tests/) and
 * the product side (bench.py driving paper_1203_2739_b200): it produces
 * inputs (matrices, permutations, splittings, vectors) and holds none of the
 * method's arithmetic (no products, no sums of a_ij*x_j, no permuting of a
 * matrix into reordered space -- it *constructs* a reordered matrix and hides
 * it under a permutation, which is how the workloads of BASELINE.json are
 * defined).
 *
 * Workload recipes (SURVEY.md §8(d) and readings
 * A13-A18, A24):
 *   kind 1 UNIFORM   C1: m x n, row length U{lo..hi}, distinct uniform columns.
 *   kind 2 SB        C2/C5: K-way singly-bordered block-diagonal form, Eq.(1)
 *                    of PAPER.md §3.1; interior U{int_lo..int_hi}
 *                    from the block's Ci columns, border U{bord_lo..bord_hi}
 *                    from the |C_B| = K*Bs border columns.  Optional hidden
 *                    owner-aligned permutation (reading A17/A18).
 *   kind 3 DB        C3: doubly-bordered form, Eq.(5), and the
 *                    2D-block split of reading A13 (part ids).
 *   kind 4 POWERLAW  C4: Zipf-Mandelbrot(alpha=2,q) row lengths on [1,Lmax]
 *                    (reading A14), columns band_frac within +-band of the row
 *                    index, the rest uniform (A15).
 *
 * Randomness is counter-based (SplitMix64 keyed by (seed, stream, row, draw)),
 * so output is independent of the number of OpenMP threads.
 *
 * Value variants: 0 real U(-1,1); 1 integer {-4..4}\{0} (x in {-4..4});
 * 2 dyadic round(U(-1,1)*1024)/1024.  Variants 1 and 2 make every partial sum
 * of a row exact in fp64, so any summation order gives the same bits.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { K_UNIFORM = 1, K_SB = 2, K_DB = 3, K_POWERLAW = 4 };
enum { S_LEN = 1, S_COLI = 2, S_COLB = 3, S_VAL = 4, S_X = 5, S_PERM = 6, S_PERMC = 7 };

typedef struct {
    int32_t kind;
    int32_t variant;
    int32_t scramble;     /* 0: identity perms; 1: hidden permutation */
    int32_t pad0;
    int64_t m, n;
    uint64_t seed;
    /* UNIFORM */
    int64_t lo, hi;
    /* SB / DB */
    int64_t K, Rb, Ci, Bs;          /* SB: rows/blk, interior cols/blk, border cols owned per blk */
    int64_t int_lo, int_hi, bord_lo, bord_hi;
    int64_t RB, CB;                 /* DB: border rows, border cols */
    int64_t brow_lo, brow_hi;       /* DB: border-row lengths */
    /* POWERLAW */
    double q;
    int64_t Lmax;
    int64_t band;
    double band_frac;
} synth_params;

static inline uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t rng(uint64_t seed, uint64_t stream, uint64_t row, uint64_t k) {
    uint64_t h = splitmix64(seed * 0xD1342543DE82EF95ULL + stream);
    h = splitmix64(h ^ row);
    return splitmix64(h ^ (k * 0xA24BAED4963EE407ULL));
}
/* uniform integer in [0, range) (range <= 2^32 here; bias < 2^-32, immaterial) */
static inline uint64_t rint_(uint64_t r, uint64_t range) {
    return (uint64_t)(((unsigned __int128)(r >> 32) * range) >> 32);
}
static inline double u01(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }
static inline double uval(uint64_t r) { return 2.0 * u01(r) - 1.0; }

static inline double value_of(int variant, uint64_t r) {
    if (variant == 1) {
        int v = (int)(r % 8);                 /* 0..7 -> -4..-1, 1..4 */
        return (double)(v < 4 ? v - 4 : v - 3);
    }
    if (variant == 2) return nearbyint(uval(r) * 1024.0) / 1024.0;
    return uval(r);
}
static inline double xvalue_of(int variant, uint64_t r) {
    if (variant == 1) return (double)((int)(r % 9) - 4);
    if (variant == 2) return nearbyint(uval(r) * 1024.0) / 1024.0;
    return uval(r);
}

/* ---------------- small open-addressing hash set (per thread) ---------------- */
typedef struct { int64_t* key; int64_t cap; int64_t* used; int64_t nused; } hset;
static void hs_init(hset* s, int64_t maxn) {
    int64_t cap = 64;
    while (cap < 2 * maxn + 2) cap <<= 1;
    s->cap = cap;
    s->key = (int64_t*)malloc(sizeof(int64_t) * cap);
    s->used = (int64_t*)malloc(sizeof(int64_t) * (maxn + 2));
    for (int64_t i = 0; i < cap; ++i) s->key[i] = -1;
    s->nused = 0;
}
static void hs_free(hset* s) { free(s->key); free(s->used); }
static void hs_clear(hset* s) {
    for (int64_t i = 0; i < s->nused; ++i) s->key[s->used[i]] = -1;
    s->nused = 0;
}
/* returns 1 if inserted, 0 if already present */
static int hs_insert(hset* s, int64_t k) {
    uint64_t h = splitmix64((uint64_t)k) & (uint64_t)(s->cap - 1);
    while (s->key[h] != -1) {
        if (s->key[h] == k) return 0;
        h = (h + 1) & (uint64_t)(s->cap - 1);
    }
    s->key[h] = k;
    s->used[s->nused++] = (int64_t)h;
    return 1;
}
static int hs_has(const hset* s, int64_t k) {
    uint64_t h = splitmix64((uint64_t)k) & (uint64_t)(s->cap - 1);
    while (s->key[h] != -1) {
        if (s->key[h] == k) return 1;
        h = (h + 1) & (uint64_t)(s->cap - 1);
    }
    return 0;
}

/* Floyd's algorithm: b distinct integers from [0, W), offset by `off`,
 * appended to out; draws keyed by (stream, row, *k). */
static int64_t floyd(const synth_params* P, uint64_t stream, int64_t row, uint64_t* k,
                     hset* s, int64_t W, int64_t b, int64_t off, int64_t* out) {
    int64_t cnt = 0;
    if (b > W) b = W;
    if (b < 0) b = 0;
    for (int64_t j = W - b; j < W; ++j) {
        int64_t t = (int64_t)rint_(rng(P->seed, stream, (uint64_t)row, (*k)++), (uint64_t)(j + 1));
        if (hs_insert(s, off + t)) out[cnt++] = off + t;
        else { hs_insert(s, off + j); out[cnt++] = off + j; }
    }
    return cnt;
}

/* ---------------- row-length model (permuted-row index p) ---------------- */
static double* zm_cdf = NULL;   /* Zipf-Mandelbrot CDF table, built once per call */

static void build_zm(const synth_params* P) {
    free(zm_cdf);
    zm_cdf = (double*)malloc(sizeof(double) * (size_t)P->Lmax);
    long double acc = 0.0L;
    for (int64_t k = 1; k <= P->Lmax; ++k) acc += powl((long double)k + P->q, -2.0L);
    long double c = 0.0L;
    for (int64_t k = 1; k <= P->Lmax; ++k) {
        c += powl((long double)k + P->q, -2.0L);
        zm_cdf[k - 1] = (double)(c / acc);
    }
    zm_cdf[P->Lmax - 1] = 1.0;
}

static inline int64_t ulen(const synth_params* P, int64_t p, uint64_t k, int64_t lo, int64_t hi) {
    return lo + (int64_t)rint_(rng(P->seed, S_LEN, (uint64_t)p, k), (uint64_t)(hi - lo + 1));
}

/* block of permuted row p for SB/DB (K = border row for DB) */
static inline int64_t row_block(const synth_params* P, int64_t p) {
    int64_t b = p / P->Rb;
    return b < P->K ? b : P->K;
}

static int64_t row_length(const synth_params* P, int64_t p) {
    switch (P->kind) {
    case K_UNIFORM: return ulen(P, p, 0, P->lo, P->hi);
    case K_SB: return ulen(P, p, 0, P->int_lo, P->int_hi) + ulen(P, p, 1, P->bord_lo, P->bord_hi);
    case K_DB:
        if (row_block(P, p) < P->K)
            return ulen(P, p, 0, P->int_lo, P->int_hi) + ulen(P, p, 1, P->bord_lo, P->bord_hi);
        return ulen(P, p, 0, P->brow_lo, P->brow_hi);
    case K_POWERLAW: {
        double u = u01(rng(P->seed, S_LEN, (uint64_t)p, 0));
        int64_t lo = 0, hi = P->Lmax - 1;       /* smallest k with cdf[k] >= u */
        while (lo < hi) { int64_t mid = (lo + hi) / 2; if (zm_cdf[mid] >= u) hi = mid; else lo = mid + 1; }
        int64_t L = lo + 1;
        return L > P->n ? P->n : L;
    }
    }
    return 0;
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* Generate permuted row p: sorted permuted column ids into cols; returns L. */
static int64_t gen_row_cols(const synth_params* P, int64_t p, hset* s, int64_t* cols) {
    hs_clear(s);
    uint64_t k = 0;
    int64_t L = 0;
    switch (P->kind) {
    case K_UNIFORM:
        L = floyd(P, S_COLI, p, &k, s, P->n, ulen(P, p, 0, P->lo, P->hi), 0, cols);
        break;
    case K_SB:
    case K_DB: {
        int64_t blk = row_block(P, p);
        if (blk < P->K) {
            int64_t li = ulen(P, p, 0, P->int_lo, P->int_hi);
            int64_t lb = ulen(P, p, 1, P->bord_lo, P->bord_hi);
            int64_t CBtot = (P->kind == K_SB) ? P->K * P->Bs : P->CB;
            L = floyd(P, S_COLI, p, &k, s, P->Ci, li, blk * P->Ci, cols);
            uint64_t kb = 0;
            L += floyd(P, S_COLB, p, &kb, s, CBtot, lb, P->K * P->Ci, cols + L);
        } else {
            L = floyd(P, S_COLI, p, &k, s, P->n, ulen(P, p, 0, P->brow_lo, P->brow_hi), 0, cols);
        }
        break;
    }
    case K_POWERLAW: {
        int64_t Lr = row_length(P, p);
        int64_t w0 = p - P->band < 0 ? 0 : p - P->band;
        int64_t w1 = p + P->band > P->n - 1 ? P->n - 1 : p + P->band;
        int64_t W = w1 - w0 + 1;
        int64_t b = (int64_t)nearbyint(P->band_frac * (double)Lr);
        if (b > W) b = W;
        L = floyd(P, S_COLI, p, &k, s, W, b, w0, cols);
        uint64_t ku = 0;
        while (L < Lr) {
            int64_t c = (int64_t)rint_(rng(P->seed, S_COLB, (uint64_t)p, ku++), (uint64_t)P->n);
            if (hs_insert(s, c)) cols[L++] = c;
        }
        break;
    }
    }
    qsort(cols, (size_t)L, sizeof(int64_t), cmp_i64);
    return L;
}

/* DB split part of permuted nonzero (i, j), reading A13 */
static inline int32_t db_part(const synth_params* P, int64_t i, int64_t j) {
    int64_t bi = row_block(P, i);
    if (bi < P->K) return (int32_t)bi;
    if (j < P->K * P->Ci) return (int32_t)(j / P->Ci);
    int64_t slice = P->RB / P->K;
    int64_t s = (i - P->K * P->Rb) / slice;
    return (int32_t)(s < P->K ? s : P->K - 1);
}

/* ---------------- owner-aligned hidden permutation (A17/A18) ---------------- */
/* r(c): permuted column -> permuted row of the same owner block (SB only). */
static inline int64_t sb_r(const synth_params* P, int64_t c) {
    int64_t KCi = P->K * P->Ci;
    if (c < KCi) { int64_t b = c / P->Ci; return b * P->Rb + (c - b * P->Ci); }
    int64_t t = c - KCi; int64_t b = t / P->Bs;
    return b * P->Rb + P->Ci + (t - b * P->Bs);
}
static inline int64_t sb_rinv(const synth_params* P, int64_t p) {
    int64_t b = p / P->Rb, l = p - b * P->Rb;
    if (l < P->Ci) return b * P->Ci + l;
    return P->K * P->Ci + b * P->Bs + (l - P->Ci);
}

/* Public: validate parameters; returns 0 or a negative error. */
int synth_check(const synth_params* P) {
    if (P->m <= 0 || P->n <= 0) return -1;
    if (P->kind == K_UNIFORM && (P->lo < 0 || P->hi < P->lo || P->hi > P->n)) return -8;
    if ((P->kind == K_SB || P->kind == K_DB) &&
        (P->int_lo < 0 || P->int_hi < P->int_lo || P->int_hi > P->Ci || P->bord_lo < 0 ||
         P->bord_hi < P->bord_lo || P->bord_hi > (P->kind == K_SB ? P->K * P->Bs : P->CB)))
        return -9;
    if (P->kind == K_DB && (P->brow_lo < 0 || P->brow_hi < P->brow_lo || P->brow_hi > P->n || P->RB < P->K))
        return -10;
    if (P->kind == K_POWERLAW && (P->Lmax < 1 || 2 * P->Lmax > P->n)) return -11;
    if (P->kind == K_SB) {
        if (P->Rb != P->Ci + P->Bs && P->scramble) return -2;
        if (P->m != P->K * P->Rb || P->n != P->K * P->Ci + P->K * P->Bs) return -3;
    }
    if (P->kind == K_DB) {
        if (P->m != P->K * P->Rb + P->RB || P->n != P->K * P->Ci + P->CB) return -4;
        if (P->scramble) return -5;
    }
    if (P->kind == K_POWERLAW && (P->scramble || P->m != P->n)) return -6;
    if (P->kind == K_UNIFORM && P->scramble) return -7;
    return 0;
}

/* Public: permutations (old->new arrays; identity if !scramble) and original
 * row lengths.  row_perm[m], col_perm[n], row_len[m]. */
int synth_structure(const synth_params* P, int32_t* row_perm, int32_t* col_perm, int64_t* row_len) {
    int rc = synth_check(P);
    if (rc) return rc;
    if (P->kind == K_POWERLAW) build_zm(P);
    if (!P->scramble) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < P->m; ++i) row_perm[i] = (int32_t)i;
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < P->n; ++j) col_perm[j] = (int32_t)j;
    } else {
        /* pi: permuted row -> original row id (Fisher-Yates, sequential) */
        int32_t* pi = (int32_t*)malloc(sizeof(int32_t) * (size_t)P->m);
        for (int64_t i = 0; i < P->m; ++i) pi[i] = (int32_t)i;
        for (int64_t i = P->m - 1; i > 0; --i) {
            int64_t j = (int64_t)rint_(rng(P->seed, S_PERM, 0, (uint64_t)i), (uint64_t)(i + 1));
            int32_t t = pi[i]; pi[i] = pi[j]; pi[j] = t;
        }
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < P->m; ++p) row_perm[pi[p]] = (int32_t)p;       /* row_perm = pi^-1 */
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < P->n; ++j) col_perm[j] = (int32_t)sb_rinv(P, row_perm[j]);
        free(pi);
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < P->m; ++i) row_len[i] = row_length(P, row_perm[i]);
    return 0;
}

typedef struct { int64_t c; double v; int32_t part; int32_t pad; } ent;
static int cmp_ent(const void* a, const void* b) {
    int64_t x = ((const ent*)a)->c, y = ((const ent*)b)->c;
    return (x > y) - (x < y);
}

/* Public: fill the ORIGINAL-space CSR (rows sorted by original column).
 * row_ptr (int64, m+1) must already hold the prefix sum of row_len.
 * col_inv: inverse of col_perm (new->old), n entries (ignored if !scramble).
 * part (may be NULL): DB split part id per nonzero, canonical order. */
int synth_fill(const synth_params* P, const int32_t* row_perm, const int32_t* col_inv,
               const int64_t* row_ptr, int32_t* col, double* val, int32_t* part) {
    int rc = synth_check(P);
    if (rc) return rc;
    if (P->kind == K_POWERLAW) build_zm(P);
    int64_t maxL = 0;
    switch (P->kind) {
    case K_UNIFORM: maxL = P->hi; break;
    case K_SB: maxL = P->int_hi + P->bord_hi; break;
    case K_DB: maxL = (P->int_hi + P->bord_hi > P->brow_hi) ? P->int_hi + P->bord_hi : P->brow_hi; break;
    case K_POWERLAW: maxL = P->Lmax; break;
    }
#pragma omp parallel
    {
        hset s; hs_init(&s, maxL);
        int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)(maxL + 1));
        ent* e = (ent*)malloc(sizeof(ent) * (size_t)(maxL + 1));
#pragma omp for schedule(dynamic, 1024)
        for (int64_t i = 0; i < P->m; ++i) {
            int64_t p = row_perm[i];
            int64_t L = gen_row_cols(P, p, &s, cols);
            for (int64_t t = 0; t < L; ++t) {
                e[t].v = value_of(P->variant, rng(P->seed, S_VAL, (uint64_t)p, (uint64_t)t));
                e[t].part = (P->kind == K_DB) ? db_part(P, p, cols[t]) : 0;
                e[t].c = P->scramble ? (int64_t)col_inv[cols[t]] : cols[t];
            }
            if (P->scramble) qsort(e, (size_t)L, sizeof(ent), cmp_ent);
            int64_t base = row_ptr[i];
            for (int64_t t = 0; t < L; ++t) {
                col[base + t] = (int32_t)e[t].c;
                val[base + t] = e[t].v;
                if (part) part[base + t] = e[t].part;
            }
        }
        free(cols); free(e); hs_free(&s);
    }
    return 0;
}

/* Public: dense vector of n entries (original space), stream S_X. */
void synth_vector(int64_t n, uint64_t seed, uint64_t stream, int32_t variant, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) out[j] = xvalue_of(variant, rng(seed, S_X + 16 * stream, 0, (uint64_t)j));
}

/* Public: owner map r as an array (SB only): r[c] = permuted row owning
 * permuted column c.  Used by the power-iteration glue x^_{t+1}[c] = y^_t[r(c)]/m. */
int synth_sb_owner(const synth_params* P, int32_t* r) {
    if (P->kind != K_SB || P->Rb != P->Ci + P->Bs) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < P->n; ++c) r[c] = (int32_t)sb_r(P, c);
    return 0;
}

int synth_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
