// diag.h -- measurement microkernels (libspmv_diag.so), NOT part of the SpMxV
// library: they measure the bounds the SpMxV kernels are judged against
// (SURVEY 8(d)); the C ABI is include/spmv_diag.h.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spmvb {
cudaError_t diag_read(const void* buf, int64_t bytes, double* out, int blocks_per_sm, cudaStream_t s);
cudaError_t diag_gather(const double* x, int64_t n, int64_t count, double* out, cudaStream_t s);
cudaError_t diag_gather_mode(const double* x, int64_t n, int64_t count, int mode, int blocks_per_sm, double* out,
                             cudaStream_t s);
cudaError_t diag_micro(int kind, int param, const void* buf, int64_t bytes, int64_t count, double* out,
                       cudaStream_t s);
}  // namespace spmvb
