// diag.cu -- roofline microkernels for the measurement harness (SURVEY §8(d)
// "N13"): they bound what the SpMxV kernel can reach on this matrix.
//   read    : a pure 128-bit read stream (HBM read peak; SpMxV is ~95% reads)
//   gather  : random 8-byte gathers from an L2-resident vector (x-gather rate)
#include <cstdint>
#include <cuda_runtime.h>

#include "diag.h"

namespace spmvb {
namespace {

__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int4 ldv4(const void* ptr, uint64_t pol) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr), "l"(pol));
    return r;
}

__global__ void __launch_bounds__(256) read_kernel(const int4* __restrict__ p, int64_t n16, double* out) {
    const uint64_t pol = pol_first();
    int acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        const int4 a = ldv4(p + i, pol), b = ldv4(p + i + stride, pol);
        const int4 c = ldv4(p + i + 2 * stride, pol), d = ldv4(p + i + 3 * stride, pol);
        acc ^= a.x ^ b.y ^ c.z ^ d.w;
    }
    for (; i < n16; i += stride) acc ^= ldv4(p + i, pol).x;
    if (acc == 0x7fffffff) out[0] = acc;   // keep the loads alive
}

__global__ void __launch_bounds__(256) gather_rand_kernel(const double* __restrict__ x, int64_t n, int64_t per_thread,
                                                          double* out) {
    uint64_t s = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ULL + 1;
    double acc = 0.0;
    for (int64_t k = 0; k < per_thread; k += 8) {
        int64_t idx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            idx[u] = (int64_t)(s % (uint64_t)n);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += __ldg(x + idx[u]);
    }
    if (acc == 1.2345) out[0] = acc;
}

// Gather flavours (mode): 0 ld.global.nc (LDG.CONSTANT), 1 ld.global (ca), 2 ld.global.cg,
// 3 ld.global.nc.L1::no_allocate, 4 pairs of lanes share a 16-byte line chunk,
// 5 16-byte gathers (double2), 6 8-lane groups share one 128-byte line,
// 7 cp.async.bulk 16-byte copies into shared memory (TMA unit, no L1 tag lookups)
__device__ __forceinline__ double gload(const double* p, int mode) {
    double v;
    switch (mode) {
    case 1: asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p)); break;
    case 2: asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p)); break;
    case 3: asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p)); break;
    default: v = __ldg(p);
    }
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(256) gather_mode_kernel(const double* __restrict__ x, int64_t n, int64_t per_thread,
                                                          double* out) {
    // n is rounded down to a power of two; 32-bit LCG per thread: ~3 integer ops per index
    uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
    const uint32_t mask = (uint32_t)(n - 1);
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    for (int64_t k = 0; k < per_thread; k += 8) {
        uint32_t idx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s = s * 1664525u + 1013904223u;
            uint32_t r = (s >> 7) & mask;
            if (MODE == 4) r = (r & ~1u) | (lane & 1);
            if (MODE == 6) r = (r & ~15u) | (lane & 7);
            if (MODE == 5) r &= ~1u;
            idx[u] = r;
        }
        if (MODE == 5) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(x + idx[u]));
                acc += v.x + v.y;
            }
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += gload(x + idx[u], MODE == 4 || MODE == 6 ? 0 : MODE);
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

// TMA (bulk-copy engine) gathers: each thread issues 8 x 16-byte bulk copies
// of x into its shared-memory slots, completion tracked by one mbarrier per warp.
__global__ void __launch_bounds__(256) gather_bulk_kernel(const double* __restrict__ x, int64_t n, int64_t per_thread,
                                                          double* out) {
    __shared__ __align__(16) double buf[256 * 16];
    __shared__ __align__(8) uint64_t bar[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar[warp]);
    if (lane == 0) asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(mb), "r"(1));
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;");
    uint64_t s = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ULL + 1;
    double acc = 0.0;
    uint32_t phase = 0;
    for (int64_t k = 0; k < per_thread; k += 8) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(32 * 8 * 16));
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            const int64_t r = (int64_t)(s % (uint64_t)n) & ~1LL;
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&buf[(threadIdx.x * 8 + u) * 2]);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
                         :: "r"(dst), "l"(x + r), "r"(mb) : "memory");
        }
        asm volatile(
            "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}"
            :: "r"(mb), "r"(phase) : "memory");
        phase ^= 1;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += buf[(threadIdx.x * 8 + u) * 2];
        __syncwarp();
    }
    if (acc == 1.2345) out[0] = acc;
}

// Random 8-byte gathers from a 96 KB shared-memory copy (the smem-staged x of C2).
__global__ void __launch_bounds__(256) gather_smem_kernel(const double* __restrict__ x, int64_t per_thread, double* out) {
    extern __shared__ double xs[];
    constexpr int N = 12288;
    for (int i = threadIdx.x; i < N; i += blockDim.x) xs[i] = x[i];
    __syncthreads();
    uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 1;
    double acc = 0.0;
    for (int64_t k = 0; k < per_thread; k += 8) {
        int idx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s = s * 1664525u + 1013904223u;
            idx[u] = (int)((s >> 9) & 8191u);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += xs[idx[u]];
    }
    if (acc == 1.2345) out[0] = acc;
}


int sms() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

}  // namespace

cudaError_t diag_read(const void* buf, int64_t bytes, double* out, int blocks_per_sm, cudaStream_t s) {
    read_kernel<<<sms() * blocks_per_sm, 256, 0, s>>>(static_cast<const int4*>(buf), bytes / 16, out);
    return cudaGetLastError();
}

cudaError_t diag_gather(const double* x, int64_t n, int64_t count, double* out, cudaStream_t s) {
    const int grid = sms() * 8;
    const int64_t per = (count + (int64_t)grid * 256 - 1) / ((int64_t)grid * 256);
    gather_rand_kernel<<<grid, 256, 0, s>>>(x, n, ((per + 7) / 8) * 8, out);
    return cudaGetLastError();
}

cudaError_t diag_gather_mode(const double* x, int64_t n, int64_t count, int mode, int blocks_per_sm, double* out,
                             cudaStream_t s) {
    const int grid = sms() * blocks_per_sm;
    const int64_t per = (count + (int64_t)grid * 256 - 1) / ((int64_t)grid * 256);
    const int64_t pt = ((per + 7) / 8) * 8;
    while (n & (n - 1)) n &= n - 1;   // power of two for the mask
    switch (mode) {
    case 0: gather_mode_kernel<0><<<grid, 256, 0, s>>>(x, n, pt, out); break;
    case 1: gather_mode_kernel<1><<<grid, 256, 0, s>>>(x, n, pt, out); break;
    case 2: gather_mode_kernel<2><<<grid, 256, 0, s>>>(x, n, pt, out); break;
    case 3: gather_mode_kernel<3><<<grid, 256, 0, s>>>(x, n, pt, out); break;
    case 4: gather_mode_kernel<4><<<grid, 256, 0, s>>>(x, n, pt, out); break;
    case 5: gather_mode_kernel<5><<<grid, 256, 0, s>>>(x, n, pt, out); break;
    case 6: gather_mode_kernel<6><<<grid, 256, 0, s>>>(x, n, pt, out); break;
    case 7: gather_bulk_kernel<<<grid, 256, 0, s>>>(x, n, pt, out); break;
    case 8:
        if (n < 12288) return cudaErrorInvalidValue;
        cudaFuncSetAttribute(gather_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 12288 * 8);
        gather_smem_kernel<<<grid, 256, 12288 * 8, s>>>(x, pt, out);
        break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace spmvb
