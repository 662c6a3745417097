/*
 * spmv.h -- C ABI of the B200-native SpMxV library (libspmv_b200.so).
 *
 * Method: Akbudak, Kayaaslan & Aykanat, "Analyzing and enhancing OSKI for
 * sparse matrix-vector multiplication", arXiv 1203.2739.  P:Lnn cites
 * /root/reference/PAPER.md line nn.
 *
 * The problem statement: y <- A x is computed repeatedly with the same
 * sparse A.  The single-SpMxV framework computes it as y^ <- A^ x^ with
 * A^ = P_r A P_c, x^ = x P_c, y^ = P_r y, where A^ is in singly- (SB,
 * Eq.(1)) or doubly-bordered (DB, Eq.(5)) block-diagonal
 * form.  The multiple-SpMxV framework computes it as y <- y + A^k x for
 * k = 1..K over a nonzero-disjoint split A = A^1 + ... + A^K.
 *
 * Conventions (every call):
 *   - Every call returns spmv_status_t; no C++ exception crosses the ABI.
 *   - Host arrays are only read during the call (spmv_create deep-copies them).
 *   - Device pointers are plain CUDA device addresses on the handle's device.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Permutations are old->new arrays: A^[row_perm[i], col_perm[j]] = A[i, j],
 *     x^[col_perm[j]] = x[j], y^[row_perm[i]] = y[i] (SURVEY reading A1).
 *   - Values are fp64 ("double precision"), column indices int32,
 *     row pointers int64 at the ABI (reading A11).
 *   - One host thread uses a handle at a time; distinct handles are independent.
 */
#ifndef SPMV_B200_H
#define SPMV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct spmv_plan_s* spmv_handle_t;

typedef enum {
    SPMV_OK = 0,
    SPMV_ERR_USAGE = 1,        /* null/invalid handle or pointer, bad flag, x == y, misalignment   */
    SPMV_ERR_DATA = 2,         /* invalid CSR, non-bijective permutation, duplicate (i,j), nonzero  */
                               /* outside the SB/DB envelope, part id outside [0,K), x_len/y_len    */
                               /* not matching the handle ("dimension mismatch")            */
    SPMV_ERR_INTERNAL = 3,     /* CUDA / NCCL / out-of-memory failure (sticky async errors surface  */
                               /* on the next call)                                                */
    SPMV_ERR_UNSUPPORTED = 4   /* split_apply without a split; a shard beyond int32 limits;         */
                               /* ORIGINAL index space with world > 1; DB or no blocks with world>1 */
} spmv_status_t;

/* Block descriptor of the reordered matrix, in PERMUTED index space.
 * kind SPMV_SB: K-way columnwise SB form, Eq.(1): rows of block k
 *   are [row_block_ptr[k], row_block_ptr[k+1]); its interior columns C_k are
 *   [col_block_ptr[k], col_block_ptr[k+1]); the column border C_B is
 *   [col_block_ptr[K], col_block_ptr[K+1]); R_B = [row_block_ptr[K],
 *   row_block_ptr[K+1]) must be empty.
 * kind SPMV_DB: Eq.(5); R_B is the row border (any columns).
 * Envelope: a nonzero of a row in block k must lie in C_k or C_B (Eq.(1)),
 * else spmv_create returns SPMV_ERR_DATA.
 * border_owner_ptr (optional, K+1 entries, may be NULL): block k owns border
 *   columns [border_owner_ptr[k], border_owner_ptr[k+1]) (absolute permuted
 *   column ids inside C_B) for the multi-GPU x layout; NULL = K equal slices
 *   C_B.start + floor(k |C_B| / K). */
enum { SPMV_SB = 1, SPMV_DB = 2 };
typedef struct {
    int32_t kind;
    int32_t K;
    const int64_t* row_block_ptr;     /* K+2 */
    const int64_t* col_block_ptr;     /* K+2 */
    const int64_t* border_owner_ptr;  /* K+1 or NULL */
} spmv_blocks_t;

/* Multi-GPU bootstrap: one process per GPU; every rank calls spmv_create with
 * the same full ORIGINAL-space CSR and the same 128-byte NCCL unique id
 * (made by spmv_nccl_unique_id on one rank and broadcast by the caller).
 * Rank g owns the contiguous diagonal blocks [floor(K g / world),
 * floor(K (g+1) / world)), their rows, their interior columns and their owned
 * border slices (spmv_shard_plan).  This is the row-slice decomposition
 * y_k <- R_k x of P:L79. */
typedef struct {
    int32_t rank;
    int32_t world;
    int32_t device;                   /* CUDA device ordinal of this rank */
    int32_t reserved;
    const void* nccl_unique_id;       /* 128 bytes (ncclUniqueId) */
} spmv_dist_t;

/* apply flags */
enum {
    SPMV_VEC_PERMUTED = 0,     /* x^, y^ in the reordered space; the hot path                */
    SPMV_VEC_ORIGINAL = 1,     /* x, y in the user's order: adds a gather and a scatter (1 GPU only) */
    SPMV_FUSE_MAXABS = 2,      /* also fold max_i |y_i| into the handle's max-abs accumulator         */
    SPMV_SPLIT_LITERAL = 4     /* split_apply only: K separate passes y <- y + A^k x (the unfused    */
                               /* literal sequence of P:L109), instead of the fused pass            */
};

/* spmv_create -- ingest, validate, permute and plan (once; not per SpMxV).
 *   m, n, nnz     : matrix dimensions and nonzero count (m, n >= 0; nnz >= 0)
 *   row_ptr       : host int64[m+1], ORIGINAL space CSR, row_ptr[0]=0, nondecreasing, row_ptr[m]=nnz
 *   col_idx       : host int32[nnz], 0 <= col < n; rows need not be sorted; duplicates rejected (A3)
 *   val           : host double[nnz]; explicit zeros are kept as structural nonzeros (A4)
 *   row_perm      : host int32[m] old->new, or NULL = identity
 *   col_perm      : host int32[n] old->new, or NULL = identity
 *   blocks        : SB/DB descriptor in permuted space, or NULL (generic reordered CSR)
 *   n_parts       : K of the split Pi, 0 = no split
 *   part_of_nnz   : host int32[nnz], part id of each nonzero in the ORIGINAL input
 *                   order (canonical order), or NULL when n_parts == 0
 *   dist          : NULL = 1 GPU (current device), else multi-GPU bootstrap
 *   out           : receives the handle; *out = NULL on any failure (all-or-nothing)
 * Errors: SPMV_ERR_USAGE (null out / bad sizes), SPMV_ERR_DATA (see enum),
 *         SPMV_ERR_UNSUPPORTED, SPMV_ERR_INTERNAL. */
spmv_status_t spmv_create(int64_t m, int64_t n, int64_t nnz,
                          const int64_t* row_ptr, const int32_t* col_idx, const double* val,
                          const int32_t* row_perm, const int32_t* col_perm,
                          const spmv_blocks_t* blocks,
                          int32_t n_parts, const int32_t* part_of_nnz,
                          const spmv_dist_t* dist,
                          spmv_handle_t* out);

/* spmv_apply -- single-SpMxV y^ <- A^ x^, asynchronous on `stream`.
 *   x : device double[x_len]; PERMUTED: x^ (1 GPU: n entries; world > 1: the
 *       rank's owned x, see spmv_info_t); ORIGINAL: x in the user's order
 *   y : device double[y_len]; overwritten (not accumulated); must not alias x
 *   Both must be 8-byte aligned.  No host synchronisation, no allocation:
 *   CUDA-graph capturable (1 GPU).  With world > 1 the border-column x
 *   entries are exchanged with NCCL over NVLink before the local SpMxV.
 * Errors: SPMV_ERR_USAGE, SPMV_ERR_DATA (length mismatch), SPMV_ERR_UNSUPPORTED,
 *         SPMV_ERR_INTERNAL. */
spmv_status_t spmv_apply(spmv_handle_t h, const double* x, int64_t x_len,
                         double* y, int64_t y_len, uint32_t flags, void* stream);

/* spmv_split_apply -- multiple-SpMxV y = 0; y <- y + A^k x, k = 1..K
 * (P:L107-109), in PERMUTED space (or ORIGINAL with the flag).  Default: one
 * fused pass that walks every row tile's part segments in part order and
 * keeps y on chip; SPMV_SPLIT_LITERAL: K passes, y read-modify-written in
 * global memory.  Errors as spmv_apply, plus SPMV_ERR_UNSUPPORTED when the
 * handle has no split. */
spmv_status_t spmv_split_apply(spmv_handle_t h, const double* x, int64_t x_len,
                               double* y, int64_t y_len, uint32_t flags, void* stream);

/* spmv_destroy -- frees all device memory and the NCCL communicator the
 * handle owns.  NULL -> SPMV_OK.  Synchronises the handle's device. */
spmv_status_t spmv_destroy(spmv_handle_t h);

/* ---------------------------------------------------------------------- */
/* Helpers outside the four-call contract.                                 */

typedef struct {
    int64_t m, n, nnz;            /* global (whole matrix) */
    int64_t m_local, nnz_local;   /* this rank's rows / nonzeros (== global at world 1) */
    int64_t row_begin;            /* first global permuted row owned by this rank */
    int64_t x_local_len;          /* length of x passed to apply on this rank (PERMUTED) */
    int64_t x_interior_begin;     /* global permuted column of x_local[0] */
    int64_t x_interior_len;       /* interior columns at the front of x_local */
    int64_t x_border_begin;       /* global permuted column of the owned border slice */
    int64_t x_border_len;         /* owned border slice length (tail of x_local) */
    int64_t border_total;         /* |C_B| */
    int64_t n_tiles;              /* row tiles of the SpMxV kernel */
    int64_t n_long_rows;          /* rows handled by the long-row path */
    int64_t bytes_alg;            /* 12 nnz + 4 (m+1) + 8 m + 8 n_touched, local */
    int64_t bytes_alg_split;      /* same for the fused split pass (0 without a split) */
    int64_t split_segments;       /* (row, part) segments of the split layout */
    int64_t xs_panels;            /* panel kernels (7, 6): panels (0 when the row-tile kernel is used) */
    int64_t xs_groups;            /* panel kernels: 32-entry groups */
    int64_t xs_pad_slots;         /* panel kernels: padding slots among them */
    int64_t bytes_stream;         /* device bytes the apply kernel actually reads + writes (no x reuse) */
    int32_t n_parts, rank, world, kind;
    int32_t has_owner_map;        /* spmv_normalize is available */
    int32_t kernel;               /* single-SpMxV kernel: 7 column-sorted panels (default: SB handles at
                                     any world size, any matrix at world 1, when the plan pads < 25 %),
                                     0 row-tile (otherwise); the others are measurement variants
                                     (SPMV_KERNEL environment variable at create) */
    int32_t split_kernel;         /* fused multiple-SpMxV kernel: 7 column-sorted panels with one y slot
                                     per (row, part) segment (default), 3 row-major part segments,
                                     1 part-major tiles; 0 without a split */
    int32_t reserved;
    int64_t gather_sectors;       /* panel kernel (7): distinct 32-byte x sectors its gathers request per
                                     launch (counted at plan time); with bytes_stream, the bytes that cross
                                     L2 -> SM per launch (the kernel's second roofline) */
} spmv_info_t;

spmv_status_t spmv_get_info(spmv_handle_t h, spmv_info_t* info);

/* Shard plan of the multi-GPU SB layout (host-only, no GPU needed; the same
 * routine spmv_create uses).  Rank `rank` of `world` owns blocks
 * [block_begin, block_end) = [floor(K r / world), floor(K (r+1) / world)),
 * rows [row_begin, row_end), x_local = [interior columns
 * x_interior_begin .. +x_interior_len | owned border slice x_border_begin ..
 * +x_border_len] (all PERMUTED global ids).  world == 1: the whole matrix. */
typedef struct {
    int64_t block_begin, block_end;
    int64_t row_begin, row_end;
    int64_t x_interior_begin, x_interior_len;
    int64_t x_border_begin, x_border_len;
    int64_t x_local_len;
    int64_t border_begin, border_total;   /* C_B */
} spmv_shard_t;

spmv_status_t spmv_shard_plan(const spmv_blocks_t* blocks, int64_t m, int64_t n, int32_t rank, int32_t world,
                              spmv_shard_t* out);

/* Power-iteration glue (BJ configs C4/C5; "repeatedly performed"):
 * spmv_maxabs writes max_i |y_i| over the rows of the last SPMV_FUSE_MAXABS
 * apply (all ranks: NCCL max all-reduce) into the device scalar *m_dev;
 * spmv_normalize computes x^_{t+1}[c] = y^_t[r(c)] / *m_dev where r is the
 * column->row identity map of the square matrix in permuted space
 * (r(c) = row_perm[col_perm^-1[c]]); with world > 1 every owned column's row
 * must be owned by the same rank (owner-aligned layout, SURVEY reading A17),
 * else SPMV_ERR_UNSUPPORTED.  x_next has x_local_len entries. */
spmv_status_t spmv_maxabs(spmv_handle_t h, double* m_dev, void* stream);
spmv_status_t spmv_normalize(spmv_handle_t h, const double* y, const double* m_dev,
                             double* x_next, void* stream);

/* Debug hook: copies the device copy of the PERMUTED local CSR back to host
 * (row_ptr as int64[m_local+1] relative to the rank's first nonzero,
 * col as GLOBAL permuted column ids int32[nnz_local], val double[nnz_local]).
 * Synchronous.  Used by tests to check the ingest bit-exactly. */
spmv_status_t spmv_debug_copy_csr(spmv_handle_t h, int64_t* row_ptr, int32_t* col, double* val);

/* Diagnostics for the measurement harness: roofline
 * microkernels, asynchronous on `stream`, results written to *out_dev only to
 * keep the loads alive.  They bound what the SpMxV kernel can reach:
 *   spmv_diag_read   : 128-bit read stream over `bytes` of device memory (HBM read peak)
 *   spmv_diag_gather : `count` random 8-byte gathers from x[0..n) (x-gather rate)
 *   spmv_diag_csr    : over the handle's device CSR (world 1): mode 0 streams
 *                      col/val only; mode 1 also gathers x[col] (no row sums);
 *                      mode 2 gathers x[col mod 2^20] (8 MB window); mode 3
 *                      gathers independent of col (no load-to-load dependency). */
spmv_status_t spmv_diag_read(const void* buf, int64_t bytes, int32_t blocks_per_sm, double* out_dev, void* stream);
spmv_status_t spmv_diag_gather(const double* x, int64_t n, int64_t count, double* out_dev, void* stream);
spmv_status_t spmv_diag_gather_mode(const double* x, int64_t n, int64_t count, int32_t mode, int32_t blocks_per_sm,
                                    double* out_dev, void* stream);   /* gather flavours 0..7, see diag.cu */
spmv_status_t spmv_diag_csr(spmv_handle_t h, const double* x, int32_t mode, double* out_dev, void* stream);
/* Host-only test hook of the x-staged kernel's planner (plan_xs.cpp): packs a
 * PERMUTED CSR (rows sorted by column, world-1 column ids) with an SB
 * descriptor into panels/groups exactly as spmv_create does, decodes the
 * packed streams again and compares them with the CSR bit for bit (and the
 * format's invariants).  stats[6] = panels, interior groups, border groups,
 * interior padding slots, border padding slots, nonzeros packed.  OK when the
 * round trip is exact; INTERNAL (message in spmv_last_error) when not;
 * UNSUPPORTED when the matrix does not fit the format. */
spmv_status_t spmv_xs_plan_check(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                                 const spmv_blocks_t* blocks, int64_t rows_target, int64_t* stats);

/* Host-only test hook of the column-sorted panel kernel's planner
 * (plan_panel.cpp): packs a PERMUTED CSR (world-1 column ids) into panels
 * (the row ranges of `blocks`, or the whole matrix when blocks is NULL) of
 * about rows_target rows, decodes the groups again and compares them with the
 * CSR bit for bit, checking that no row repeats within an epoch.
 * stats[8] = panels, groups, padding slots, deferred nonzeros, epochs,
 * nonzeros packed, and 1000 x the mean predicted shared-memory wavefronts of
 * a group's y access with natural / bank-coloured y slots.  OK on an exact
 * round trip; INTERNAL otherwise. */
spmv_status_t spmv_pn_plan_check(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                                 const spmv_blocks_t* blocks, int64_t rows_target, int64_t* stats);

/* Host-only test hook of the multi-GPU determinism of the panel plan (SURVEY
 * 8(e)): for each rank of `world`, builds that rank's local CSR of a PERMUTED
 * SB matrix (its blocks' rows; columns in the rank's x layout [interior |
 * C_B]), plans its panels exactly as spmv_create does (sms = the SM count the
 * whole-wave rule assumes) and hashes, per block, the panels' row ranges and
 * every group's (global row, virtual-row rank, global column, value bits) in
 * issue order.  out[r * K + k] = rank r's hash of block k, 0 for blocks it
 * does not own.  Equal hashes at world 1 and world G mean equal summation
 * orders, so y is bit-identical across GPU counts.  USAGE / DATA on bad
 * arguments (blocks must be SB). */
spmv_status_t spmv_pn_shard_hash(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                                 const spmv_blocks_t* blocks, int32_t world, int32_t sms, int64_t* out);

/* Test hook of the multi-GPU path on one GPU.  With SPMV_TEST_RANKS_NO_NCCL
 * set in the environment, spmv_create accepts a dist descriptor whose
 * nccl_unique_id is NULL: the handle is rank `rank` of `world` (its shard,
 * local CSR, x layout and panel plan exactly as on a real multi-GPU run) but
 * has no communicator; its apply skips the border all-gather, and the test
 * supplies the full x(C_B) the all-gather would deliver through this call
 * (`x_border`: device pointer, `len` = |C_B| doubles, copied; the apply still
 * writes the rank's own slice into place first).  USAGE on a handle that is
 * not such a test rank or on a length mismatch. */
spmv_status_t spmv_test_set_border(spmv_handle_t h, const double* x_border, int64_t len);

/* Design microbenchmarks (diag2.cu): kind 1 L2->SM LDG.128 bandwidth over the
 * L2-resident `buf` (`bytes` long, `count` bytes read in total); kind 2 bulk-copy
 * L2->shared bandwidth, param = cluster size 1/2/4/8 (multicast when > 1),
 * `count` bytes delivered per launch over all CTAs; kind 3 shared-memory
 * y[r] += v*x[c] updates (`buf` unused, `count` updates, param 0 random /
 * 1 conflict-free); kind 4 L2 gathers with `param` lanes per 128-byte line
 * (`buf` = x of `bytes`, `count` gathers).  USAGE on bad arguments. */
spmv_status_t spmv_diag_micro(int32_t kind, int32_t param, const void* buf, int64_t bytes, int64_t count,
                              double* out_dev, void* stream);

/* Writes a fresh 128-byte NCCL unique id into out (len >= 128). */
spmv_status_t spmv_nccl_unique_id(void* out, size_t len);

/* Static description of a status code. */
const char* spmv_status_string(spmv_status_t s);

/* Last error message recorded on this thread (for diagnostics). */
const char* spmv_last_error(void);

/* Library version (major*10000 + minor*100 + patch). */
int32_t spmv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPMV_B200_H */
