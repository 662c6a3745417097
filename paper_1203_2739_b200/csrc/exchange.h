// exchange.h -- the world > 1 exchange (a4, f1, f2); see exchange.cpp.
#pragma once
#include "handle.h"

namespace spmvb {

// What the SpMxV kernel of one apply reads: x_hi (the exchanged x(C_B)) for
// local columns >= x_split, and -- P2P / loopback -- the ready flags it waits
// on before its first border epoch.
struct XView {
    const double* x_hi = nullptr;
    int32_t x_split = INT32_MAX;
    const int32_t* ready = nullptr;
    int32_t seq = 0;
    int32_t* err = nullptr;
    int32_t* herr = nullptr;   // host-mapped sticky flag (set on a timed-out wait)
};

spmv_status_t xchg_alloc(spmv_plan_s* h);                                        // create: buffers
spmv_status_t xchg_agree(spmv_plan_s* h, spmv_status_t local, spmv_status_t* agreed);   // create: all ranks agree
spmv_status_t xchg_connect(spmv_plan_s* h);                                      // create: P2P handles or NCCL
spmv_status_t xchg_pre(spmv_plan_s* h, const double* x, cudaStream_t st, XView& v);     // apply: before the kernel
spmv_status_t xchg_post(spmv_plan_s* h, double* y, unsigned long long* slots, cudaStream_t st);   // after it
spmv_status_t xchg_allreduce_max(spmv_plan_s* h, double* m_dev, cudaStream_t st);
int64_t xchg_timeouts(spmv_plan_s* h);
bool xchg_failed(const spmv_plan_s* h);   // a device-side exchange wait timed out (no synchronisation)
void xchg_release(spmv_plan_s* h);
spmv_status_t xchg_loopback_link(spmv_plan_s** hs, int world);
bool stream_memops_available();

}  // namespace spmvb
