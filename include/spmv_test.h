/*
 * spmv_test.h -- test and debug hooks of libspmv_b200.so.  NOT part of the
 * user-facing ABI (include/spmv.h): the parity tests use them to read the
 * library's internal state back and to run the multi-GPU path on one GPU.
 * They never change what spmv_create / spmv_apply compute for a handle made
 * through include/spmv.h.
 */
#ifndef SPMV_B200_TEST_H
#define SPMV_B200_TEST_H

#include "spmv.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Copies the device copy of the PERMUTED local CSR back to host (row_ptr as
 * int64[m_local+1] relative to the rank's first nonzero, col as GLOBAL
 * permuted column ids int32[nnz_local], val double[nnz_local]).  Synchronous.
 * World > 1 DB handles: the local compute rows (block rows, then the
 * border-row temporaries' segments).  Checks the ingest (a1) bit-exactly.
 * A panel-kernel handle keeps the device CSR only when created with
 * spmv_options_t.retain_csr (else UNSUPPORTED). */
spmv_status_t spmv_debug_copy_csr(spmv_handle_t h, int64_t* row_ptr, int32_t* col, double* val);

/* Host-only round trip of the column-sorted panel kernel's planner
 * (plan_panel.cpp): packs a PERMUTED CSR (world-1 column ids) into panels
 * (the row ranges of `blocks`, or the whole matrix when blocks is NULL) of
 * about rows_target rows, decodes the groups again and compares them with the
 * CSR bit for bit, checking that no row repeats within an epoch, that groups
 * never mix interior and border columns, that border groups come last and
 * that every panel fits shared memory.  stats[15] = panels, groups, padding
 * slots, deferred nonzeros, epochs, nonzeros packed, 1000 x the mean predicted
 * shared-memory wavefronts of a group's y access with natural / bank-coloured
 * y slots, the largest panel's shared memory bytes, panels with border
 * groups, distinct 32-byte x sectors over all groups' gathers, padding slots
 * and epochs of the drain (epochs that start after the panel's column sweep
 * has handed out its last nonzero: only deferred ones are left), nonzeros in
 * the far stream, and its steps per warp summed over the panels.  OK on an
 * exact round trip; INTERNAL otherwise. */
spmv_status_t spmv_pn_plan_check(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                                 const spmv_blocks_t* blocks, int64_t rows_target, int64_t* stats);

/* Host-only check of the multi-GPU determinism of the SB panel plan (SURVEY
 * 8(e)): for each rank of `world`, builds that rank's local CSR of a PERMUTED
 * SB matrix (its blocks' rows; columns in the rank's x layout [interior |
 * C_B]), plans its panels exactly as spmv_create does (sms = the SM count the
 * whole-wave rule assumes) and hashes, per block, the panels' row ranges and
 * every group's (global row, virtual-row rank, global column, value bits) in
 * issue order.  out[r * K + k] = rank r's hash of block k, 0 for blocks it
 * does not own.  Equal hashes at world 1 and world G mean equal summation
 * orders, so y is bit-identical across GPU counts. */
spmv_status_t spmv_pn_shard_hash(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                                 const spmv_blocks_t* blocks, int32_t world, int32_t sms, int64_t* out);

/* Rank `rank` of `world` of the multi-GPU path, built on the current device
 * WITHOUT a communicator (shard, local CSR, x / y layouts, plans exactly as a
 * real multi-GPU rank), for the loopback fake of SURVEY §4: create all
 * `world` ranks in one process, then link them with spmv_test_loopback_link.
 * dist->nccl_unique_id is ignored. */
spmv_status_t spmv_test_create_rank(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                                     const double* val, const int32_t* row_perm, const int32_t* col_perm,
                                     const spmv_blocks_t* blocks, int32_t n_parts, const int32_t* part_of_nnz,
                                     const spmv_dist_t* dist, const spmv_options_t* options, spmv_handle_t* out);

/* Links `world` test ranks (handles[r] is rank r) into one loopback group:
 * every rank's exchange then runs the P2P protocol of the multi-GPU path --
 * copy-engine pushes of its border slices (and DB temporaries) into the
 * other ranks' buffers, stream-memory-operation flags, the kernel's device
 * wait before its first border epoch -- with the peers' buffers on the same
 * GPU.  Each rank must then be applied on its own stream, ranks in any order
 * (the same number of applies per rank).  USAGE when a handle is not a test
 * rank of that world or the ranks disagree; UNSUPPORTED without stream
 * memory operations. */
spmv_status_t spmv_test_loopback_link(spmv_handle_t* handles, int32_t world);

/* Test of the debug checks (spmv_options_t.debug_checks): corrupts the panel
 * plan of a panel handle on the device -- kind 1: a warp-1 entry of panel 0's
 * first epoch takes the y slot of a warp-0 entry (a row updated twice in one
 * epoch); 2: a y slot beyond the panel's shared memory; 3: a column delta
 * beyond x for a matrix whose columns are fewer than the group base + 2^17.
 * The handle's results are wrong afterwards; USAGE / UNSUPPORTED otherwise. */
spmv_status_t spmv_test_corrupt_panel(spmv_handle_t h, int32_t kind);

/* The apply stream of a linked loopback test rank (created by
 * spmv_test_loopback_link right after the rank's comm stream, so the ranks'
 * streams do not share the GPU's hardware work queues when
 * CUDA_DEVICE_MAX_CONNECTIONS >= 2 * world): a rank's apply blocks its stream
 * until the peers' pushes land, and a peer's push queued behind that wait on
 * a shared queue would never run.  USAGE for a handle that is not a linked
 * test rank. */
spmv_status_t spmv_test_rank_stream(spmv_handle_t h, void** stream);

/* Per-CTA timeline of the panel kernel (a measurement hook): mode 1 arms the
 * handle -- its next panel-kernel launches record, per CTA (panel), 8 words:
 * SM id, %globaltimer (ns) at start and end, clock64 at start, after the
 * prologue (y zeroed, fold lists copied), after the far phase (and the
 * epilogue's first slot loads), at the end (the end adds one barrier per
 * CTA), after the epochs; mode 0 copies the last launch's records into
 * out[0 .. 8 * panels) (cap words at most; synchronises the device) and
 * disarms.  UNSUPPORTED for a handle without a panel plan. */
spmv_status_t spmv_test_panel_stamps(spmv_handle_t h, int32_t mode, uint64_t* out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* SPMV_B200_TEST_H */
