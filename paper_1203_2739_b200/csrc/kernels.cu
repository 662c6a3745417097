// kernels.cu -- small sm_100a kernels around the SpMxV (P:Lnn = PAPER.md line):
//   * ORIGINAL-mode vector maps x^[c] = x[col_perm^-1[c]], y[i] = y^[row_perm[i]]
//     (a3, a7);
//   * the power-iteration glue (a9; "repeatedly performed"): the final
//     fold of the per-warp max |y| slots and x_{t+1} = y_t / m_t.
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace spmvb {

namespace {

__global__ void gather_kernel(const double* __restrict__ src, const int32_t* __restrict__ idx,
                              double* __restrict__ dst, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __ldg(src + idx[i]);
}

// One thread per slot (a single load each, then a warp and a CTA fold): the
// step's serial tail, so it is latency, not bytes (a one-warp loop over the
// 1,024 slots measured 6.8 us under ncu).
__global__ void __launch_bounds__(kMaxSlots) maxabs_finish_kernel(const unsigned long long* __restrict__ slots,
                                                                  double* out) {
    __shared__ unsigned long long wm[kMaxSlots / 32];
    unsigned long long m = slots[threadIdx.x * kSlotStride];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, m, off);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = wm[threadIdx.x];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long o = __shfl_xor_sync(0xffffffffu, m, off);
            m = o > m ? o : m;
        }
        if (threadIdx.x == 0) *out = __longlong_as_double((long long)m);
    }
}

// x_next[c] = y[owner[c]] / m, four columns per thread step: one 128-bit load
// of owner, two 128-bit stores of x (IEEE division: bit-exact with the oracle).
__global__ void __launch_bounds__(256) normalize_kernel(const double* __restrict__ y, const int32_t* __restrict__ owner,
                                                        const double* __restrict__ m, double* __restrict__ x, int64_t n) {
    const double mt = *m;
    const int64_t n4 = n >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int4* o4 = reinterpret_cast<const int4*>(owner);
    double2* x2 = reinterpret_cast<double2*>(x);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4; q += stride) {
        int4 o;
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(o.x), "=r"(o.y), "=r"(o.z), "=r"(o.w) : "l"(o4 + q));
        const double a = __ldg(y + o.x), b = __ldg(y + o.y), c = __ldg(y + o.z), d = __ldg(y + o.w);
        x2[2 * q] = make_double2(a / mt, b / mt);
        x2[2 * q + 1] = make_double2(c / mt, d / mt);
    }
    for (int64_t c = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += stride)
        x[c] = __ldg(y + owner[c]) / mt;
}

// The same update with the owner map stored as runs (create: consecutive local
// columns whose rows are consecutive too, A17's owner-aligned layout: C5 has
// 128 runs for 64 M columns): x_next[l] = y[tgt[r] + l - start[r]] for the run
// r holding l.  No 4-byte map per column is read (16 instead of 20 bytes per
// column of HBM traffic).  Tiles of 1,024 columns; a tile inside one run has its
// offset tgt[r] - start[r] precomputed at create (tdelta), loaded one tile ahead
// so the y loads never wait on it; a tile that straddles runs (kNoDelta) finds
// each column's run by binary search over the (few, L1-resident) run starts.
constexpr int kNormTile = (int)kNormTileCols;
__global__ void __launch_bounds__(256) normalize_runs_kernel(const double* __restrict__ y,
                                                             const int64_t* __restrict__ tdelta,
                                                             const int64_t* __restrict__ start,
                                                             const int32_t* __restrict__ tgt, int64_t R,
                                                             const double* __restrict__ m, double* __restrict__ x,
                                                             int64_t n) {
    const double mt = *m;
    const int64_t T = (n + kNormTile - 1) / kNormTile;
    int64_t t = blockIdx.x;
    int64_t dnext = t < T ? __ldg(tdelta + t) : 0;
    for (; t < T; t += gridDim.x) {
        const int64_t delta = dnext;
        if (t + gridDim.x < T) dnext = __ldg(tdelta + t + gridDim.x);
        const int64_t t0 = t * kNormTile + threadIdx.x;
        double v[4];
        if (delta != kNoDelta && t0 + 3 * 256 < n) {
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = __ldg(y + t0 + k * 256 + delta);
#pragma unroll
            for (int k = 0; k < 4; ++k) x[t0 + k * 256] = v[k] / mt;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t l = t0 + k * 256;
                if (l >= n) break;
                int64_t lo = 0, hi = R - 1;   // last run with start <= l
                while (lo < hi) {
                    const int64_t mid = (lo + hi + 1) >> 1;
                    if (__ldg(start + mid) <= l) lo = mid; else hi = mid - 1;
                }
                x[l] = __ldg(y + __ldg(tgt + lo) + (l - __ldg(start + lo))) / mt;
            }
        }
    }
}

__global__ void normalize_scalar_kernel(const double* __restrict__ y, const int32_t* __restrict__ owner,
                                        const double* __restrict__ m, double* __restrict__ x, int64_t n) {
    const double mt = *m;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
        x[c] = __ldg(y + owner[c]) / mt;
}

// DB split across GPUs (f1): y_i = 0, then y_i <- y_i + tmp_k for
// the row's received per-part temporaries in part order (fold lists built at
// create), one thread per owned border row; max |y| folded like the SpMxV's.
// P2P exchange (ready != nullptr): the peers' temporaries arrive over NVLink
// while earlier work runs; every CTA first waits (thread 0, acquire loads,
// bounded: a timeout counts in *err) until ready[q] - seq >= 0 for every peer
// q -- a device-side wait, so no stream ever blocks on a peer (a blocked
// stream can hold up unrelated work queued behind it) -- and then reads tin
// through L2 (ld.cg: written by the peers' copy engines).
__global__ void __launch_bounds__(256) fold_kernel(const double* tin, const int32_t* __restrict__ fptr,
                                                   const int32_t* __restrict__ fpos, double* __restrict__ y,
                                                   int64_t n, unsigned long long* slots, FoldWait w) {
    if (w.ready) {
        if (threadIdx.x == 0)
            for (int q = 0; q < w.world; ++q) {
                if (q == w.self) continue;
                uint32_t it = 0;
                for (;;) {
                    int32_t v;
                    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(w.ready + q) : "memory");
                    if (v - w.seq >= 0) break;
                    __nanosleep(256);
                    if (++it > (1u << 24)) {   // ~ seconds: the peer is gone
                        atomicAdd(w.err, 1);
                        if (w.herr) *reinterpret_cast<volatile int32_t*>(w.herr) = 1;
                        break;
                    }
                }
            }
        __syncthreads();
    }
    double mx = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double v = 0.0;
        for (int32_t j = fptr[i]; j < fptr[i + 1]; ++j) v = v + __ldcg(tin + fpos[j]);
        y[i] = v;
        mx = fmax(mx, fabs(v));
    }
    if (slots) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if ((threadIdx.x & 31) == 0 && mx > 0.0)
            atomicMax(slots + ((blockIdx.x * 8 + (threadIdx.x >> 5) + 512) & (kMaxSlots - 1)) * kSlotStride,
                      (unsigned long long)__double_as_longlong(mx));
    }
}

int grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    const int64_t cap = (int64_t)kernel_num_sms() * 8;
    if (g > cap) g = cap;
    return (int)(g > 0 ? g : 1);
}

}  // namespace

int kernel_num_sms() {   // per device (a process may hold handles on several GPUs)
    static std::atomic<int> cache[kMaxDevices];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
    if (dev >= kMaxDevices) dev = kMaxDevices - 1;
    int n = cache[dev].load(std::memory_order_relaxed);
    if (n <= 0) {
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

cudaError_t launch_gather(const double* src, const int32_t* idx, double* dst, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    gather_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, idx, dst, n);
    return cudaGetLastError();
}

cudaError_t launch_fold(const double* tin, const int32_t* fptr, const int32_t* fpos, double* y, int64_t n, FoldWait w,
                        unsigned long long* slots, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    fold_kernel<<<grid_for(n, 256), 256, 0, s>>>(tin, fptr, fpos, y, n, slots, w);
    return cudaGetLastError();
}

cudaError_t launch_maxabs_finish(const unsigned long long* slots, double* out, cudaStream_t s) {
    maxabs_finish_kernel<<<1, kMaxSlots, 0, s>>>(slots, out);
    return cudaGetLastError();
}

cudaError_t launch_normalize(const double* y, const int32_t* owner, const double* m, double* x_next,
                             int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (((uintptr_t)x_next & 15) || ((uintptr_t)owner & 15)) {   // vector path needs 16-byte alignment
        normalize_scalar_kernel<<<grid_for(n, 256), 256, 0, s>>>(y, owner, m, x_next, n);
    } else {
        normalize_kernel<<<grid_for((n + 3) / 4, 256), 256, 0, s>>>(y, owner, m, x_next, n);
    }
    return cudaGetLastError();
}

cudaError_t launch_normalize_runs(const double* y, const int64_t* tdelta, const int64_t* start, const int32_t* tgt,
                                  int64_t runs, const double* m, double* x_next, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    normalize_runs_kernel<<<grid_for((n + kNormTile - 1) / kNormTile, 1), 256, 0, s>>>(y, tdelta, start, tgt, runs,
                                                                                       m, x_next, n);
    return cudaGetLastError();
}


// Loads this file's kernels now (cudaFuncGetAttributes forces the lazy loader):
// a kernel first launched while a peer rank's kernel spins on an exchange flag
// would otherwise load its module then, and a module load can wait for the
// running kernels -- the spinning one included (see host.cpp preload_kernels).
cudaError_t preload_kernels_misc() {
    cudaFuncAttributes fa;
    for (const void* k : {(const void*)gather_kernel, (const void*)maxabs_finish_kernel, (const void*)normalize_kernel,
                          (const void*)normalize_runs_kernel,
                          (const void*)normalize_scalar_kernel, (const void*)fold_kernel}) {
        const cudaError_t e = cudaFuncGetAttributes(&fa, k);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace spmvb
