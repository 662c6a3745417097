// api.cu -- C ABI of the measurement microkernels (include/spmv_diag.h).
#include "../../include/spmv_diag.h"
#include "diag.h"

extern "C" {

int32_t spmv_diag_read(const void* buf, int64_t bytes, int32_t blocks_per_sm, double* out_dev, void* stream) {
    if (!buf || bytes < 16 || !out_dev || blocks_per_sm < 1) return 1;
    return spmvb::diag_read(buf, bytes, out_dev, blocks_per_sm, (cudaStream_t)stream) == cudaSuccess ? 0 : 3;
}

int32_t spmv_diag_gather(const double* x, int64_t n, int64_t count, double* out_dev, void* stream) {
    if (!x || n < 1 || count < 1 || !out_dev) return 1;
    return spmvb::diag_gather(x, n, count, out_dev, (cudaStream_t)stream) == cudaSuccess ? 0 : 3;
}

int32_t spmv_diag_gather_mode(const double* x, int64_t n, int64_t count, int32_t mode, int32_t blocks_per_sm,
                              double* out_dev, void* stream) {
    if (!x || n < 2 || count < 1 || !out_dev || blocks_per_sm < 1) return 1;
    return spmvb::diag_gather_mode(x, n, count, mode, blocks_per_sm, out_dev, (cudaStream_t)stream) == cudaSuccess
               ? 0 : 3;
}

int32_t spmv_diag_micro(int32_t kind, int32_t param, const void* buf, int64_t bytes, int64_t count, double* out_dev,
                        void* stream) {
    if (!out_dev || count < 1 || (kind != 3 && (!buf || bytes < 16))) return 1;
    return spmvb::diag_micro(kind, param, buf, bytes, count, out_dev, (cudaStream_t)stream) == cudaSuccess ? 0 : 3;
}

}  // extern "C"
