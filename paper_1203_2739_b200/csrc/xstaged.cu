// xstaged.cu -- the x-staged SB kernel: each CTA copies its SB block's x(C_k)
// and the border x(C_B) into shared memory once, then streams row tiles of
// that block and gathers x from shared memory (P:Lnn = PAPER.md line).
//
// This is the paper's cache-fit rule (a part's x must fit the
// cache; Theorem 1: then x is loaded once per part) with one SM's
// shared memory as the cache, for SB matrices whose blocks are small enough
// (x(C_k) + x(C_B) <= ~24 K entries, e.g. C2: 11,875 + 10,000).  Eq.(1)
// guarantees that the rows of block k touch only C_k and C_B, so
// the staged slice serves every gather of the CTA: a random 8-byte gather
// from shared memory costs about one wavefront per distinct bank instead of
// one L1TEX wavefront per 128-byte line from L2.  Column ids are 16-bit
// block-local (u < |C_k|: C_k[u], else C_B[u - |C_k|]) -- the staged slice's
// own index -- so the stream is 10 B per nonzero (the ICSR idea of P:L43).
//
// Per CTA (1024 threads, one per SM, a run of rowtile.cu's tiles of one
// block): stage x, then every warp sums its share of the rows, one y store
// per row, max |y| folded.  Not the default: on C2 the row-tile
// kernel's L2 gathers are faster (34.8 vs 36.9 us, L2 flushed) -- x is
// L2-resident there anyway and the staging copy is a serial phase
// (DESIGN §5.6).
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace spmvb {
namespace {

constexpr int NT = 512;

__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// No product staging and no CTA barrier after the x copy: each of the CTA's
// 32 warps walks its own contiguous share of the CTA's rows, V lanes per row
// (c.pad, planned from the mean row length), loads (id, value) of its rows
// and gathers from the staged x; fixed lane assignment and xor tree per row
// (deterministic).  Measured on C2 (`profiles/r02_ab_xstaged.txt`): a
// 512-thread form that staged each row tile's products in shared memory (two
// barriers per tile) took 41.0 us, this one 36.9 us, 512 threads 59.4 us,
// border x gathered from L2 with two CTAs per SM 53.3 us.
constexpr int NTW = 1024;
__global__ void __launch_bounds__(NTW, 1) spmv_xstaged_warp_kernel(const XsArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* xs = reinterpret_cast<double*>(smem_raw);
    const XsCta c = A.cta[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < c.nk; i += NTW) xs[i] = __ldg(A.x + c.q0 + i);
    for (int i = tid; i < c.nB; i += NTW) xs[c.nk + i] = __ldg(A.x + c.qB + i);
    const uint64_t pol = pol_evict_first();
    __syncthreads();
    const int R0 = A.tile_row[c.t0], R1 = A.tile_row[c.t1];
    const int V = c.pad, rpw = 32 / V;
    const int w0 = R0 + (int)((int64_t)(R1 - R0) * warp / (NTW / 32));
    const int w1 = R0 + (int)((int64_t)(R1 - R0) * (warp + 1) / (NTW / 32));
    const int j = lane % V;
    double mx = 0.0;
    for (int rb = w0; rb < w1; rb += rpw) {
        const int r = rb + lane / V;
        double acc = 0.0;
        if (r < w1) {
            const int a = A.rowptr[r], b = A.rowptr[r + 1];
#pragma unroll 4
            for (int t = a + j; t < b; t += V) {
                unsigned short u;
                double v;
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(u) : "l"(A.colx + t), "l"(pol));
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(A.val + t), "l"(pol));
                acc = fma(v, xs[u], acc);
            }
        }
        for (int off = V >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (r < w1 && j == 0) {
            A.y[r] = acc;
            mx = fmax(mx, fabs(acc));
        }
    }
    if (A.maxabs_slots) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if (lane == 0 && mx > 0.0)
            atomicMax(A.maxabs_slots + ((blockIdx.x * (NTW / 32) + warp) & (kMaxSlots - 1)) * kSlotStride,
                      (unsigned long long)__double_as_longlong(mx));
    }
}

}  // namespace

int64_t xstaged_smem_bytes(int64_t x_entries) { return 8 * x_entries; }

cudaError_t launch_xstaged(const XsArgs& a, cudaStream_t s) {
    if (a.n_cta <= 0) return cudaSuccess;
    const int64_t smem = xstaged_smem_bytes(a.max_x);
    if (smem > kPnSmemMax) return cudaErrorInvalidValue;   // the planner never selects such a matrix
    static std::atomic<int> ready[kMaxDevices];
    int dev = 0;
    cudaError_t r = cudaGetDevice(&dev);
    if (r != cudaSuccess) return r;
    const int di = dev < kMaxDevices ? dev : kMaxDevices - 1;
    if (!ready[di].load(std::memory_order_acquire) || dev >= kMaxDevices) {
        if ((r = cudaFuncSetAttribute(spmv_xstaged_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kPnSmemMax)) != cudaSuccess)
            return r;
        ready[di].store(1, std::memory_order_release);
    }
    spmv_xstaged_warp_kernel<<<a.n_cta, NTW, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t preload_kernels_xstaged() {
    cudaFuncAttributes fa;
    return cudaFuncGetAttributes(&fa, spmv_xstaged_warp_kernel);
}

}  // namespace spmvb
