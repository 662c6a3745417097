/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU oracle for the SpMxV
 * hot path of Akbudak, Kayaaslan & Aykanat, "Analyzing and enhancing OSKI for
 * sparse matrix-vector multiplication" (arXiv 1203.2739; /root/reference/PAPER.md
 * cited as P:Lnn).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this.  It shares no
 * code, header, table or helper with the CUDA path (paper_1203_2739_b200/),
 * and neither side includes or imports the other.
 *
 * Build: gcc -O3 -ffp-contract=off (no -ffast-math): every multiply and every
 * add rounds separately, in the order written, IEEE round-to-nearest (A21).
 *
 * What it computes:
 *   - the plain product y = A x on the ORIGINAL matrix: the reordered product
 *     y^ = A^ x^ with A^ = P_r A P_c, x^ = x P_c, y^ = P_r y and the
 *     split product y = sum_k A^k x both equal it in exact
 *     arithmetic;
 *   - the literal multiple-SpMxV sequence y <- y + A^k x, k = 1..K;
 *   - the permutation of a CSR matrix and of vectors, used to check ingest;
 *   - validation, the per-entry tolerance scale S_i = sum_j |a_ij x_j|
 *     (north_star), and the power-iteration glue x_{t+1} = y_t/||y_t||_inf;
 *   - the connectivity statistics lambda(c_j) of Eq.(3) and
 *     lambda(r_i), lambda(c_j) of Theorem 3.
 *
 * Pins (tests/test_oracle_*.py, `-m "not gpu"`): brute-force dense matvec
 * (bitwise, same order), hand examples, the 6x6 worked example
 * (tests/golden/), closed forms (identity, diagonal, permutation matrix,
 * rank-1), integer/dyadic exactness, scipy.sparse as an independent library.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* Validation (a1): row_ptr[0] = 0, nondecreasing, row_ptr[m] =
 * nnz; 0 <= col < n; no duplicate (i, j) (reading A3).
 * Returns 0 ok, 1 bad row_ptr, 2 column out of range, 3 duplicate entry.     */
int oracle_validate_csr(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                        const int32_t* col) {
    if (m < 0 || n < 0 || nnz < 0) return 1;
    if (row_ptr[0] != 0 || row_ptr[m] != nnz) return 1;
    for (int64_t i = 0; i < m; ++i)
        if (row_ptr[i + 1] < row_ptr[i]) return 1;
    for (int64_t t = 0; t < nnz; ++t)
        if (col[t] < 0 || (int64_t)col[t] >= n) return 2;
    /* duplicates: stamp array over columns, stamped with the row number + 1 */
    int64_t* stamp = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
    int rc = 0;
    for (int64_t i = 0; i < m && !rc; ++i)
        for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) {
            if (stamp[col[t]] == i + 1) { rc = 3; break; }
            stamp[col[t]] = i + 1;
        }
    free(stamp);
    return rc;
}

/* A permutation given as an old->new array must be a bijection on [0, n)
 * (S:L39-42).  Returns 0 ok, 1 not a bijection.                              */
int oracle_validate_perm(int64_t n, const int32_t* perm) {
    char* seen = (char*)calloc((size_t)(n > 0 ? n : 1), 1);
    int rc = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (perm[i] < 0 || (int64_t)perm[i] >= n || seen[perm[i]]) { rc = 1; break; }
        seen[perm[i]] = 1;
    }
    free(seen);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Permute (§8(c) step 2; "A^ = P_r A P_c"): nonzero (i, j, v) goes to
 * (row_perm[i], col_perm[j], v); rows are counting-sorted by new row index,
 * then each row is sorted by new column (qsort, a library primitive).  With
 * duplicates rejected the result is unique.  part_in/part_out (may be NULL)
 * carry split part ids along.  Output arrays are caller-allocated (m+1, nnz). */
typedef struct { int32_t c; int32_t part; double v; } oent;
static int cmp_oent(const void* a, const void* b) {
    int32_t x = ((const oent*)a)->c, y = ((const oent*)b)->c;
    return (x > y) - (x < y);
}
void oracle_permute(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col,
                    const double* val, const int32_t* row_perm, const int32_t* col_perm,
                    const int32_t* part_in, int64_t* out_row_ptr, int32_t* out_col,
                    double* out_val, int32_t* out_part) {
    (void)n;
    /* new row lengths: new row row_perm[i] has the length of old row i */
    for (int64_t p = 0; p <= m; ++p) out_row_ptr[p] = 0;
    for (int64_t i = 0; i < m; ++i) out_row_ptr[row_perm[i] + 1] = row_ptr[i + 1] - row_ptr[i];
    for (int64_t p = 0; p < m; ++p) out_row_ptr[p + 1] += out_row_ptr[p];
    int64_t maxlen = 0;
    for (int64_t i = 0; i < m; ++i)
        if (row_ptr[i + 1] - row_ptr[i] > maxlen) maxlen = row_ptr[i + 1] - row_ptr[i];
    oent* buf = (oent*)malloc(sizeof(oent) * (size_t)(maxlen > 0 ? maxlen : 1));
    for (int64_t i = 0; i < m; ++i) {
        int64_t L = row_ptr[i + 1] - row_ptr[i];
        for (int64_t t = 0; t < L; ++t) {
            buf[t].c = col_perm[col[row_ptr[i] + t]];
            buf[t].v = val[row_ptr[i] + t];
            buf[t].part = part_in ? part_in[row_ptr[i] + t] : 0;
        }
        qsort(buf, (size_t)L, sizeof(oent), cmp_oent);
        int64_t base = out_row_ptr[row_perm[i]];
        for (int64_t t = 0; t < L; ++t) {
            out_col[base + t] = buf[t].c;
            out_val[base + t] = buf[t].v;
            if (out_part) out_part[base + t] = buf[t].part;
        }
    }
    free(buf);
}

/* Vector maps: x^[col_perm[j]] = x[j] ;  y[i] = y^[row_perm[i]].     */
void oracle_permute_x(int64_t n, const int32_t* col_perm, const double* x, double* xhat) {
    for (int64_t j = 0; j < n; ++j) xhat[col_perm[j]] = x[j];
}
void oracle_unpermute_y(int64_t m, const int32_t* row_perm, const double* yhat, double* y) {
    for (int64_t i = 0; i < m; ++i) y[i] = yhat[row_perm[i]];
}

/* ------------------------------------------------------------------------ */
/* SpMxV (§8(c) step 3): for each row a scalar temporary
 * accumulates val[t]*x[col[t]] in CSR order, then one store y[i] = s.
 * S[i] = sum |val[t]*x[col[t]]| is the per-entry tolerance scale (may be NULL).
 * nthreads > 1 splits ROWS over OpenMP threads; the per-row arithmetic is
 * unchanged, so the result does not depend on nthreads.                     */
void oracle_spmv(int64_t m, const int64_t* row_ptr, const int32_t* col, const double* val,
                 const double* x, double* y, double* S, int32_t nthreads) {
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 4096) num_threads(nthreads > 0 ? nthreads : 1)
#endif
    for (int64_t i = 0; i < m; ++i) {
        double s = 0.0, a = 0.0;
        for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) {
            double prod = val[t] * x[col[t]];
            s = s + prod;
            a = a + fabs(prod);
        }
        y[i] = s;
        if (S) S[i] = a;
    }
}

/* Same, for a list of rows only (sampled parity at full size).               */
void oracle_spmv_rows(int64_t nrows, const int64_t* rows, const int64_t* row_ptr,
                      const int32_t* col, const double* val, const double* x,
                      double* y_out, double* S_out) {
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        double s = 0.0, a = 0.0;
        for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) {
            double prod = val[t] * x[col[t]];
            s = s + prod;
            a = a + fabs(prod);
        }
        y_out[r] = s;
        if (S_out) S_out[r] = a;
    }
}

/* ------------------------------------------------------------------------ */
/* Multiple-SpMxV (§8(c) step 4): y = 0 (reading A9), then for
 * k = 0..K-1 in ascending order (A8): for each row i holding part-k nonzeros,
 * tmp = sum of its part-k products in canonical order, y[i] = y[i] + tmp
 * (A7: "accumulated in the output vector y on the fly").  Literal O(K nnz).
 * Returns 0, or 1 if a part id lies outside [0, K).                          */
int oracle_split(int64_t m, const int64_t* row_ptr, const int32_t* col, const double* val,
                 const int32_t* part, int32_t K, const double* x, double* y) {
    for (int64_t t = 0; t < row_ptr[m]; ++t)
        if (part[t] < 0 || part[t] >= K) return 1;
    for (int64_t i = 0; i < m; ++i) y[i] = 0.0;
    for (int32_t k = 0; k < K; ++k) {
        for (int64_t i = 0; i < m; ++i) {
            double tmp = 0.0;
            int has = 0;
            for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t)
                if (part[t] == k) {
                    double prod = val[t] * x[col[t]];
                    tmp = tmp + prod;
                    has = 1;
                }
            if (has) y[i] = y[i] + tmp;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Power-iteration glue (§8(c) step 5; BJ.c4/c5; "repeatedly
 * performed"): m_t = max_i |y_t[i]|; x_{t+1}[j] = y_t[j] / m_t (square A).   */
double oracle_maxabs(int64_t m, const double* y) {
    double mx = 0.0;
    for (int64_t i = 0; i < m; ++i)
        if (fabs(y[i]) > mx) mx = fabs(y[i]);
    return mx;
}
void oracle_scale(int64_t n, const double* y, double mt, double* xnext) {
    for (int64_t j = 0; j < n; ++j) xnext[j] = y[j] / mt;
}

/* ------------------------------------------------------------------------ */
/* Comparator (§8(c) step 6; north_star "|y - y_ref| <= 1e-12 * sum|a_ij x_j|"):
 * pass iff for every i |y[i] - yref[i]| <= tol * S[i]; S[i] == 0 requires
 * y[i] == +-0; any NaN/Inf fails.  Returns the number of failing entries;
 * *worst = max |d|/S over entries with S > 0, *first_bad = first failing i. */
int64_t oracle_check(int64_t m, const double* y, const double* yref, const double* S, double tol,
                     double* worst, int64_t* first_bad) {
    int64_t bad = 0;
    double w = 0.0;
    *first_bad = -1;
    for (int64_t i = 0; i < m; ++i) {
        int ok;
        if (isnan(y[i]) || isinf(y[i]) || isnan(yref[i]) || isinf(yref[i])) ok = 0;
        else if (S[i] == 0.0) ok = (y[i] == 0.0);
        else {
            double d = fabs(y[i] - yref[i]);
            double r = d / S[i];
            if (r > w) w = r;
            ok = (d <= tol * S[i]);
        }
        if (!ok) { if (bad == 0) *first_bad = i; ++bad; }
    }
    *worst = w;
    return bad;
}

/* ------------------------------------------------------------------------ */
/* Connectivity statistics.
 * Eq.(3): lambda(c_j) = |{R_k : c_j in R_k}|, with R_k the k-th row
 * slice; row_block[i] in [0, K) gives R_k of row i (rows with row_block < 0,
 * e.g. the DB row border R_B, are skipped: that is lambda' of P:L95).
 * Returns sum_j lambda(c_j) (Theorem 1's bound, Eq.(4)); lam_out may be NULL. */
int64_t oracle_sb_lambda(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col,
                         const int32_t* row_block, int32_t* lam_out) {
    int32_t* last = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t* lam = lam_out ? lam_out : (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t j = 0; j < n; ++j) { last[j] = -1; lam[j] = 0; }
    /* count distinct blocks per column; a set per column via a K-bit scan */
    int32_t K = 0;
    for (int64_t i = 0; i < m; ++i) if (row_block[i] + 1 > K) K = row_block[i] + 1;
    for (int32_t k = 0; k < K; ++k) {
        for (int64_t i = 0; i < m; ++i) {
            if (row_block[i] != k) continue;
            for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t)
                if (last[col[t]] != k) { last[col[t]] = k; lam[col[t]] += 1; }
        }
    }
    int64_t sum = 0;
    for (int64_t j = 0; j < n; ++j) sum += lam[j];
    free(last);
    if (!lam_out) free(lam);
    return sum;
}

/* Theorem 3: lambda(r_i) = |{A^k : r_i in A^k}|, lambda(c_j) likewise.
 * Writes sum_i lambda(r_i) and sum_j lambda(c_j) (Corollary 4's bound, Eq.(7)). */
void oracle_split_lambda(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col,
                         const int32_t* part, int32_t K, int64_t* sum_lr, int64_t* sum_lc) {
    int64_t sr = 0, sc = 0;
    char* seen = (char*)calloc((size_t)(n > 0 ? n : 1), 1);
    for (int32_t k = 0; k < K; ++k) {
        memset(seen, 0, (size_t)(n > 0 ? n : 1));
        for (int64_t i = 0; i < m; ++i) {
            int has = 0;
            for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t)
                if (part[t] == k) { has = 1; if (!seen[col[t]]) { seen[col[t]] = 1; ++sc; } }
            sr += has;
        }
    }
    free(seen);
    *sum_lr = sr;
    *sum_lc = sc;
}

/* ------------------------------------------------------------------------ */
/* sBFS ordering (section 5.1): "we apply BFS on the
 * bipartite graph representation of the matrix, so that the resulting BFS
 * orders on the row and column vertices determine row and column
 * reorderings, respectively."  Reading R5 fixes what the paper
 * leaves open, as the textbook queue BFS:
 *   - vertices: rows r_0..r_{m-1} and columns c_0..c_{n-1}; edge (r_i, c_j)
 *     for every stored entry a_ij;
 *   - the root is the lowest-numbered unvisited row; a popped vertex appends
 *     its unvisited neighbours in ascending number; when the queue empties the
 *     next root is again the lowest-numbered unvisited row; columns no row
 *     touches come last, ascending;
 *   - new row number = position among the rows in visiting order; columns
 *     likewise.  row_perm / col_perm are old -> new (reading A1).
 * Then the SB extraction (Eq.(1)) with K blocks (reading R5):
 *   - new row r goes to block min(K-1, floor(K * P(r) / nnz)), P(r) = stored
 *     entries of the rows numbered below r (floor(K * r / m) when nnz = 0);
 *   - a column all of whose rows lie in one block k is interior to block k,
 *     any other column (two or more blocks, or none) is a border column;
 *   - columns are renumbered: block 0's interior columns, ..., block K-1's,
 *     then the border columns C_B, each group in BFS column order.
 * Outputs row_perm[m], col_perm[n] (the SB order, old -> new),
 * row_block_ptr[K+2] (R_B empty), col_block_ptr[K+2] (the last range is C_B),
 * and bfs_row[m], bfs_col[n]: the plain BFS numbers before the extraction.
 * Returns 0, or 1 on bad arguments. */
int oracle_sbfs(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, int32_t K,
                int32_t* row_perm, int32_t* col_perm, int64_t* row_block_ptr, int64_t* col_block_ptr,
                int32_t* bfs_row, int32_t* bfs_col) {
    if (m < 0 || n < 0 || K < 1) return 1;
    const int64_t nnz = row_ptr[m];
    /* row adjacency sorted ascending (input rows may be unsorted) */
    int32_t* radj = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    memcpy(radj, col, sizeof(int32_t) * (size_t)nnz);
    for (int64_t i = 0; i < m; ++i) {   /* insertion sort per row: plain and obviously correct */
        for (int64_t t = row_ptr[i] + 1; t < row_ptr[i + 1]; ++t) {
            int32_t v = radj[t];
            int64_t u = t - 1;
            while (u >= row_ptr[i] && radj[u] > v) { radj[u + 1] = radj[u]; --u; }
            radj[u + 1] = v;
        }
    }
    /* column adjacency: rows in ascending order (counting pass over rows in order) */
    int64_t* cptr = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t t = 0; t < nnz; ++t) cptr[col[t] + 1] += 1;
    for (int64_t j = 0; j < n; ++j) cptr[j + 1] += cptr[j];
    int32_t* cadj = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t j = 0; j < n; ++j) fill[j] = cptr[j];
    for (int64_t i = 0; i < m; ++i)
        for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) cadj[fill[col[t]]++] = (int32_t)i;
    /* queue BFS; queue entries: v >= 0 row v, v < 0 column -v-1 */
    int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + n > 0 ? m + n : 1));
    for (int64_t i = 0; i < m; ++i) bfs_row[i] = -1;
    for (int64_t j = 0; j < n; ++j) bfs_col[j] = -1;
    int64_t head = 0, tail = 0, nr = 0, nc = 0, next_root = 0;
    while (nr < m) {
        while (bfs_row[next_root] >= 0) ++next_root;      /* lowest unvisited row */
        bfs_row[next_root] = (int32_t)nr++;
        queue[tail++] = next_root;
        while (head < tail) {
            const int64_t u = queue[head++];
            if (u >= 0) {
                for (int64_t t = row_ptr[u]; t < row_ptr[u + 1]; ++t) {
                    const int32_t j = radj[t];
                    if (bfs_col[j] < 0) { bfs_col[j] = (int32_t)nc++; queue[tail++] = -(int64_t)j - 1; }
                }
            } else {
                const int64_t j = -u - 1;
                for (int64_t t = cptr[j]; t < cptr[j + 1]; ++t) {
                    const int32_t i = cadj[t];
                    if (bfs_row[i] < 0) { bfs_row[i] = (int32_t)nr++; queue[tail++] = i; }
                }
            }
        }
    }
    for (int64_t j = 0; j < n; ++j)
        if (bfs_col[j] < 0) bfs_col[j] = (int32_t)nc++;   /* untouched columns, ascending */
    /* SB extraction: blocks of the BFS row order by nonzero prefix */
    int64_t* len_new = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    for (int64_t i = 0; i < m; ++i) len_new[bfs_row[i]] = row_ptr[i + 1] - row_ptr[i];
    int32_t* blk_new = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int64_t P = 0;
    for (int64_t r = 0; r < m; ++r) {
        int64_t b = nnz > 0 ? (int64_t)(((__int128)K * P) / nnz) : (K * r) / (m > 0 ? m : 1);
        if (b > K - 1) b = K - 1;
        blk_new[r] = (int32_t)b;
        P += len_new[r];
    }
    for (int32_t k = 0; k <= K + 1; ++k) row_block_ptr[k] = m;
    for (int64_t r = m - 1; r >= 0; --r) row_block_ptr[blk_new[r]] = r;
    for (int32_t k = K - 1; k >= 0; --k)          /* empty blocks start where the next one does */
        if (row_block_ptr[k] > row_block_ptr[k + 1]) row_block_ptr[k] = row_block_ptr[k + 1];
    row_block_ptr[0] = 0;
    /* column classes: -1 none yet, k one block, K two or more / none */
    int32_t* cls = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t j = 0; j < n; ++j) cls[j] = -1;
    for (int64_t i = 0; i < m; ++i) {
        const int32_t b = blk_new[bfs_row[i]];
        for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) {
            const int32_t j = col[t];
            if (cls[j] == -1) cls[j] = b;
            else if (cls[j] != b) cls[j] = K;
        }
    }
    for (int64_t j = 0; j < n; ++j) if (cls[j] == -1) cls[j] = K;
    /* column numbering: by (class, BFS column number) */
    int32_t* by_bfs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t j = 0; j < n; ++j) by_bfs[bfs_col[j]] = (int32_t)j;
    int64_t q = 0;
    for (int32_t k = 0; k <= K; ++k) {
        col_block_ptr[k] = q;
        for (int64_t c = 0; c < n; ++c) {
            const int32_t j = by_bfs[c];
            if (cls[j] == k) col_perm[j] = (int32_t)q++;
        }
    }
    col_block_ptr[K + 1] = n;
    for (int64_t i = 0; i < m; ++i) row_perm[i] = bfs_row[i];
    free(radj); free(cptr); free(cadj); free(fill); free(queue); free(len_new); free(blk_new); free(cls);
    free(by_bfs);
    return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
