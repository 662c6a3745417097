/*
 * spmv_diag.h -- C ABI of libspmv_diag.so: measurement microkernels for the
 * benchmark harness.  NOT part of the SpMxV library
 * (include/spmv.h) and never called on the SpMxV path: they measure the
 * bounds the SpMxV kernels are judged against (HBM read stream, L2 -> SM
 * stream, random x gathers), live in the same run as the kernel timing.
 *
 * All calls are asynchronous on `stream` (a cudaStream_t as void*, NULL =
 * legacy default stream) on the current device; results are written to
 * *out_dev only to keep the loads alive.  Return 0 ok, 1 bad arguments,
 * 3 CUDA launch error.
 */
#ifndef SPMV_DIAG_H
#define SPMV_DIAG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 128-bit read stream over `bytes` of device memory `buf` (the HBM read peak
 * when buf is much larger than L2); blocks_per_sm CTAs of 256 threads per SM. */
int32_t spmv_diag_read(const void* buf, int64_t bytes, int32_t blocks_per_sm, double* out_dev, void* stream);

/* `count` random 8-byte gathers from x[0..n) (the x-gather rate of a
 * row-ordered CSR kernel when x is L2-resident). */
int32_t spmv_diag_gather(const double* x, int64_t n, int64_t count, double* out_dev, void* stream);

/* Gather flavours 0..8 (cache hints, lanes per line, bulk, shared memory);
 * n is rounded down to a power of two (address mask). */
int32_t spmv_diag_gather_mode(const double* x, int64_t n, int64_t count, int32_t mode, int32_t blocks_per_sm,
                              double* out_dev, void* stream);

/* Design microbenchmarks: kind 1 L2 -> SM LDG.128 bandwidth over the
 * L2-resident `buf` (`bytes` long, `count` bytes read in total); kind 2
 * bulk-copy L2 -> shared bandwidth, param = cluster size 1/2/4/8 (multicast
 * when > 1), `count` bytes delivered; kind 3 shared-memory y[r] += v*x[c]
 * updates (buf unused, `count` updates, param 0 random / 1 conflict-free);
 * kind 4 L2 gathers with `param` lanes per 128-byte line (buf = x). */
int32_t spmv_diag_micro(int32_t kind, int32_t param, const void* buf, int64_t bytes, int64_t count,
                        double* out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPMV_DIAG_H */
