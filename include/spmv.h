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
 *   C_B.start + floor(k |C_B| / K).  row_border_owner_ptr: the same for the
 *   DB row border R_B (multi-GPU y layout of DB handles). */
enum { SPMV_SB = 1, SPMV_DB = 2 };
typedef struct {
    int32_t kind;
    int32_t K;
    const int64_t* row_block_ptr;     /* K+2 */
    const int64_t* col_block_ptr;     /* K+2 */
    const int64_t* border_owner_ptr;  /* K+1 or NULL */
    const int64_t* row_border_owner_ptr;  /* DB only, K+1 or NULL: block k owns border rows
                                             [p[k], p[k+1]) of R_B for the multi-GPU y layout;
                                             NULL = K equal slices R_B.start + floor(k |R_B| / K) */
} spmv_blocks_t;

/* Multi-GPU bootstrap: one process per GPU; every rank calls spmv_create with
 * the same full ORIGINAL-space CSR and the same 128-byte NCCL unique id
 * (made by spmv_nccl_unique_id on one rank and broadcast by the caller).
 * Rank g owns the contiguous diagonal blocks [floor(K g / world),
 * floor(K (g+1) / world)), their rows, their interior columns and their owned
 * border slices (spmv_shard_plan).
 *   SB (Eq.(1)): the row-slice decomposition y_k <- R_k x of P:L79; the only
 *   exchange is the border x(C_B) (all-gathered every apply).
 *   DB (Eq.(5)) -- the multiple-SpMxV across GPUs (f1): part k of
 *   the split is block k's diagonal block plus its border slices (n_parts == K,
 *   or n_parts == 0: the 2D block assignment -- a nonzero of block row i goes
 *   to i's block, of a border row to its interior column's block, border x
 *   border to the row's border slice); rank g computes its parts' products,
 *   the border rows' per-part temporaries travel to the owner of the row,
 *   which folds them in part order.
 * All ranks must issue the same sequence of apply calls (collective). */
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

/* Create-time options (spmv_create_ex; NULL = all defaults).  Zero means
 * "automatic" in every field. */
enum { SPMV_KERNEL_AUTO = 0, SPMV_KERNEL_PANEL = 1, SPMV_KERNEL_ROWTILE = 2, SPMV_KERNEL_XSTAGED = 3 };
enum { SPMV_SPLIT_AUTO = 0, SPMV_SPLIT_PANEL = 1, SPMV_SPLIT_ROWS = 2 };
enum { SPMV_EXCHANGE_AUTO = 0, SPMV_EXCHANGE_NCCL = 1, SPMV_EXCHANGE_P2P = 2 };
typedef struct {
    int32_t struct_size;     /* sizeof(spmv_options_t) (forward compatibility), or 0 */
    int32_t kernel;          /* single SpMxV: AUTO = column-sorted panels unless their plan pads > 25 %
                                (then row tiles); PANEL forces the panels (whatever the padding);
                                ROWTILE forces row tiles; XSTAGED (1 GPU, SB): each CTA stages its
                                block's x(C_k) and x(C_B) in shared memory once and gathers from
                                there (the cache-fit rule of P:L61) -- UNSUPPORTED when a block's x
                                does not fit; not chosen by AUTO (slower than row tiles on C2) */
    int32_t panel_rows;      /* y slots per panel; 0 = automatic (whole waves of ~16 K-slot panels) */
    int32_t split_kernel;    /* fused multiple-SpMxV: AUTO / PANEL (a y slot per (row, part) segment) /
                                ROWS (row-major part segments, row tiles) */
    int32_t exchange;        /* world > 1: AUTO = P2P when every GPU pair has peer access and stream
                                memory operations are available, else NCCL.  P2P: copy-engine pushes of
                                the border slices into the peers' buffers (CUDA IPC) with device flags,
                                overlapped with the interior epochs of the kernel (a4, f2).  NCCL:
                                ncclAllGather / grouped send-recv on a comm stream, joined before
                                the kernel */
    int32_t index16;         /* f3 (ICSR-style index compression): AUTO (0) = row-tile handles
                                stream 16-bit tile-local column ids (10 B per nonzero instead of 12)
                                whenever every row tile's columns fit two 65,536-id windows (an SB
                                block tile: C_k and C_B, Eq.(1)); 1 = off (32-bit ids) */
    int32_t debug_checks;    /* 1 = run the checked variant of the panel kernel (compute-sanitizer is
                                not available on this GPU pool): every y slot and x column it touches is
                                bounds-checked, and every y update stamps its slot with the epoch in
                                shared memory (atomicExch), so a row updated twice within one epoch --
                                a violation of the planner's race-freedom invariant -- is counted;
                                counts in spmv_info_t.debug_violations.  Slower; for tests */
    int32_t retain_csr;      /* 1 = keep the device copy of the permuted CSR even when the panel kernel
                                does not read it (for spmv_debug_copy_csr); 0 (default) = a panel
                                handle frees it after planning (C5: 13.7 GB less per GPU) */
    int32_t reserved[8];
} spmv_options_t;

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

/* spmv_create_ex -- spmv_create with options (NULL = spmv_create). */
spmv_status_t spmv_create_ex(int64_t m, int64_t n, int64_t nnz,
                             const int64_t* row_ptr, const int32_t* col_idx, const double* val,
                             const int32_t* row_perm, const int32_t* col_perm,
                             const spmv_blocks_t* blocks,
                             int32_t n_parts, const int32_t* part_of_nnz,
                             const spmv_dist_t* dist, const spmv_options_t* options,
                             spmv_handle_t* out);

/* spmv_apply -- single-SpMxV y^ <- A^ x^, asynchronous on `stream`.
 *   x : device double[x_len]; PERMUTED: x^ (1 GPU: n entries; world > 1: the
 *       rank's owned x, see spmv_info_t); ORIGINAL: x in the user's order
 *   y : device double[y_len]; overwritten (not accumulated); must not alias x
 *       (world > 1: the rank's owned rows, y_local_len entries)
 *   Both must be 8-byte aligned.  No host synchronisation, no allocation:
 *   CUDA-graph capturable (1 GPU).  With world > 1 the border-column x
 *   entries are exchanged over NVLink (P2P copy engines or NCCL); on a DB
 *   handle the border rows' per-part temporaries are exchanged and folded in
 *   part order too (the multiple-SpMxV across GPUs).  x must not
 *   change until the call's work on `stream` has completed.
 * Errors: SPMV_ERR_USAGE, SPMV_ERR_DATA (length mismatch), SPMV_ERR_UNSUPPORTED,
 *         SPMV_ERR_INTERNAL. */
spmv_status_t spmv_apply(spmv_handle_t h, const double* x, int64_t x_len,
                         double* y, int64_t y_len, uint32_t flags, void* stream);

/* spmv_split_apply -- multiple-SpMxV y = 0; y <- y + A^k x, k = 1..K
 * (P:L107-109), in PERMUTED space (or ORIGINAL with the flag).  Default: one
 * fused pass that keeps every (row, part) temporary on chip and adds them to
 * y in part order, one y store per row; SPMV_SPLIT_LITERAL: K passes, y
 * read-modify-written in global memory (world 1).  Errors as spmv_apply, plus
 * SPMV_ERR_UNSUPPORTED when the handle has no split. */
spmv_status_t spmv_split_apply(spmv_handle_t h, const double* x, int64_t x_len,
                               double* y, int64_t y_len, uint32_t flags, void* stream);

/* spmv_destroy -- frees all device memory and the NCCL communicator the
 * handle owns.  NULL -> SPMV_OK.  Synchronises the handle's device. */
spmv_status_t spmv_destroy(spmv_handle_t h);

/* ---------------------------------------------------------------------- */
/* Helpers outside the four-call contract.                                 */

typedef struct {
    int64_t m, n, nnz;            /* global (whole matrix) */
    int64_t m_local, nnz_local;   /* this rank's compute rows / nonzeros (== global at world 1) */
    int64_t row_begin;            /* first global permuted row of the rank's blocks */
    int64_t x_local_len;          /* length of x passed to apply on this rank (PERMUTED) */
    int64_t x_interior_begin;     /* global permuted column of x_local[0] */
    int64_t x_interior_len;       /* interior columns at the front of x_local */
    int64_t x_border_begin;       /* global permuted column of the owned border slice */
    int64_t x_border_len;         /* owned border slice length (tail of x_local) */
    int64_t border_total;         /* |C_B| */
    int64_t n_tiles;              /* row tiles (row-tile kernel) */
    int64_t n_long_rows;          /* rows longer than a tile */
    int64_t bytes_alg;            /* 12 nnz + 4 (m+1) + 8 m + 8 n_touched, local */
    int64_t bytes_alg_split;      /* same for the fused split pass (0 without a split) */
    int64_t split_segments;       /* (row, part) segments of the split layout */
    int64_t panels;               /* panel kernel: panels (0 when the row-tile kernel is used) */
    int64_t groups;               /* panel kernel: 32-entry groups */
    int64_t pad_slots;            /* panel kernel: padding slots among them */
    int64_t bytes_stream;         /* device bytes the apply kernel actually reads + writes (no x reuse) */
    int32_t n_parts, rank, world, kind;
    int32_t has_owner_map;        /* spmv_normalize is available */
    int32_t kernel;               /* single-SpMxV kernel: 7 column-sorted panels, 0 row tiles,
                                     8 x-staged (SB blocks' x in shared memory) */
    int32_t split_kernel;         /* fused multiple-SpMxV: 7 panels with one y slot per (row, part)
                                     segment, 3 row-major part segments; 0 without a split */
    int32_t exchange;             /* world > 1: 1 NCCL, 2 P2P copy engines (overlapped), 3 loopback (test) */
    int64_t gather_sectors;       /* panel kernel: distinct 32-byte x sectors its gathers request per
                                     launch (plan time); with bytes_stream, the bytes that cross L2 -> SM */
    int64_t y_local_len;          /* length of y passed to apply on this rank */
    int64_t y_border_begin;       /* DB world > 1: global permuted row of the owned border-row slice */
    int64_t y_border_len;         /*   (tail of y_local) */
    int64_t deferred;             /* panel kernel: nonzeros deferred to a later epoch (repeated row) */
    int64_t y_wavefronts_x1000;   /* panel kernel: predicted shared-memory wavefronts per y access x 1000 */
    int64_t exchange_timeouts;    /* world > 1 P2P: device-side flag waits that timed out (should be 0;
                                     reading it synchronises the device) */
    int64_t index_bytes;          /* row-tile kernel: bytes per column id it streams (2 with the f3
                                     16-bit tile-local ids, else 4) */
    int64_t debug_violations[3];  /* debug_checks: y slots out of bounds, x columns out of bounds, rows
                                     updated twice in one epoch (all 0 on a correct plan; reading them
                                     synchronises the device) */
    double create_s[6];           /* spmv_create's wall time by phase (s): validation + descriptor +
                                     shard; permutation of the rows; tiles + CSR upload; split layouts;
                                     panel plans + upload; maps and buffers (the ingest cost of Table 3's
                                     amortization) */
    int64_t far_nonzeros;         /* panel kernel: nonzeros summed in the barrier-free far phase (those
                                     still deferred when a panel's column sweep ends) */
    int64_t owner_runs;           /* spmv_normalize: > 0 when the column -> row owner map is held as this
                                     many runs of consecutive rows (no per-column map is read), 0 when it
                                     is a per-column array */
} spmv_info_t;

spmv_status_t spmv_get_info(spmv_handle_t h, spmv_info_t* info);

/* Shard plan of the multi-GPU layout (host-only, no GPU needed; the same
 * routine spmv_create uses).  Rank `rank` of `world` owns blocks
 * [block_begin, block_end) = [floor(K r / world), floor(K (r+1) / world)),
 * rows [row_begin, row_end) (+ DB: border rows [y_border_begin, +y_border_len)),
 * x_local = [interior columns x_interior_begin .. +x_interior_len | owned
 * border slice x_border_begin .. +x_border_len] (all PERMUTED global ids).
 * world == 1: the whole matrix. */
typedef struct {
    int64_t block_begin, block_end;
    int64_t row_begin, row_end;
    int64_t x_interior_begin, x_interior_len;
    int64_t x_border_begin, x_border_len;
    int64_t x_local_len;
    int64_t border_begin, border_total;   /* C_B */
    int64_t y_border_begin, y_border_len; /* DB: owned slice of R_B */
    int64_t y_local_len;
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

/* ---------------------------------------------------------------------- */
/* Producing the reordering.                               */

/* spmv_order_sbfs -- the sBFS ordering of P:L134 (section 5.1: BFS on the
 * bipartite graph of A, whose row and column visiting orders give the row
 * and column reorderings) computed on the current CUDA device, followed by
 * the extraction of a K-way SB form (Eq.(1)), so the outputs feed
 * spmv_create directly (kind SPMV_SB).  Definition (reading R5):
 *   - the BFS root is the lowest-numbered unvisited row; a visited vertex
 *     enqueues its unvisited neighbours in ascending number; when the queue
 *     empties the next root is the lowest unvisited row; columns no row
 *     touches are numbered last, ascending;
 *   - new row r joins block min(K-1, floor(K * P(r) / nnz)), P(r) = stored
 *     entries of the rows numbered below r (rows split by nonzeros);
 *   - a column all of whose rows lie in block k is interior to block k;
 *     every other column (two or more blocks, or none) is a border column;
 *     columns are numbered block by block, then C_B, each in BFS order.
 * Arguments (all HOST arrays; synchronous; the device work is this call's):
 *   m, n, nnz, row_ptr[m+1] (int64), col_idx[nnz]: the ORIGINAL-space CSR
 *     (rows need not be sorted; validated: DATA on a bad row_ptr / column);
 *   K >= 1: number of SB diagonal blocks;
 *   row_perm[m], col_perm[n]: receive the old->new permutations (A1);
 *   row_block_ptr[K+2], col_block_ptr[K+2]: receive the block descriptor in
 *     permuted space (R_B empty; [col_block_ptr[K], n) is C_B);
 *   info: optional timings and statistics (NULL allowed).
 * Errors: USAGE (bad arguments), DATA (invalid CSR), UNSUPPORTED (m or n
 * beyond int32), INTERNAL (CUDA / out of device memory). */
typedef struct {
    double bfs_ms;           /* device time of the CSC build and the BFS (CUDA events) */
    double extract_ms;       /* device time of the SB extraction */
    int64_t levels;          /* BFS levels expanded (row and column levels) */
    int64_t components;      /* BFS roots with entries */
    int64_t border_cols;     /* |C_B| of the extracted SB form */
} spmv_order_info_t;

spmv_status_t spmv_order_sbfs(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                              int32_t K, int32_t* row_perm, int32_t* col_perm,
                              int64_t* row_block_ptr, int64_t* col_block_ptr, spmv_order_info_t* info);

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
