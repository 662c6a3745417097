// diag2.cu -- microbenchmarks that decide the x-staging design:
//   kind 1  L2 -> SM read bandwidth: LDG.128 sweeps over an L2-resident buffer
//   kind 2  L2 -> shared memory by the bulk-copy engine (cp.async.bulk), one CTA
//           per SM, a 4-stage mbarrier ring; param = cluster size (1, 2, 4, 8);
//           param > 1 multicasts each chunk to every CTA of the cluster
//   kind 3  shared-memory y[row] += v * x[col] (the chunked-x update), 512
//           threads, y 16 K rows and x 12 K columns resident; param 0 random
//           rows/columns per lane, 1 conflict-free (consecutive per lane)
//   kind 4  L2 gathers where groups of `param` lanes share one 128-byte line
//           (does the LSU cost scale with lanes or with lines per request?)
// None of these touch the SpMxV data structures; they only bound them.
#include <cstdint>
#include <cuda_runtime.h>

#include "diag.h"

namespace spmvb {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---------------------------------------------------------------- kind 1
__global__ void __launch_bounds__(512) l2read_kernel(const int4* __restrict__ buf, int64_t n16, int64_t per_cta,
                                                     double* out) {
    int acc = 0;
    const int64_t base = ((int64_t)blockIdx.x * 7919 * 512) % n16;
    for (int64_t k = threadIdx.x; k < per_cta; k += 4 * 512) {
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int64_t i = (base + k + u * 512) % n16;
            asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(buf + i));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x7fffffff) out[0] = acc;
}

// ---------------------------------------------------------------- kind 2
constexpr int kStages = 4;
constexpr int kChunk = 32768;   // bytes per stage

template <int CL>
__global__ void __launch_bounds__(64, 1) tma_l2_kernel(const char* __restrict__ src, int64_t src_bytes, int64_t chunks,
                                                       double* out) {
    extern __shared__ __align__(128) char smem[];
    char* stage = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kChunk);
    uint64_t* empty = full + kStages;
    uint32_t rank = 0;
    if (CL > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(CL));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (CL > 1) {
        asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        __syncthreads();
    }
    const int64_t cluster_id = blockIdx.x / CL;
    const int64_t n_src_chunks = src_bytes / kChunk;
    double acc = 0.0;
    if (warp == 0) {
        // producer: this CTA issues slice `rank` of every chunk, multicast to the cluster
        if (lane == 0) {
            for (int64_t i = 0; i < chunks; ++i) {
                const int s = (int)(i % kStages);
                const uint32_t ph = (uint32_t)((i / kStages) & 1);
                if (i >= kStages) {
                    asm volatile("{\n.reg .pred p;\nW1: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}"
                                 ::"r"(smem_u32(&empty[s])), "r"(ph ^ 1) : "memory");
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                             "r"(kChunk));
                const int64_t c = (cluster_id * 977 + i) % n_src_chunks;
                const char* g = src + c * kChunk + rank * (kChunk / CL);
                const uint32_t dst = smem_u32(stage + s * kChunk + rank * (kChunk / CL));
                if (CL == 1) {
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(dst), "l"(g), "r"(kChunk), "r"(smem_u32(&full[s])) : "memory");
                } else {
                    const uint16_t mask = (uint16_t)((1u << CL) - 1);
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                                 " [%0], [%1], %2, [%3], %4;"
                                 ::"r"(dst), "l"(g), "r"(kChunk / CL), "r"(smem_u32(&full[s])), "h"(mask) : "memory");
                }
            }
        }
    } else {
        // consumer: wait for the chunk, touch it, release the stage in every CTA of the cluster
        for (int64_t i = 0; i < chunks; ++i) {
            const int s = (int)(i % kStages);
            const uint32_t ph = (uint32_t)((i / kStages) & 1);
            asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}"
                         ::"r"(smem_u32(&full[s])), "r"(ph) : "memory");
            const double* d = reinterpret_cast<const double*>(stage + s * kChunk);
#pragma unroll 4
            for (int k = lane; k < kChunk / 8; k += 32 * 8) acc += d[k];
            __syncwarp();
            if (lane < CL) {
                const uint32_t local = smem_u32(&empty[s]);
                if (CL == 1) {
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(local) : "memory");
                } else {
                    uint32_t remote;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(lane));
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
                }
            }
        }
    }
    if (CL > 1) {
        asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (acc == 1.2345) out[0] = acc;
}

// ---------------------------------------------------------------- kind 3
template <int MODE>
__global__ void __launch_bounds__(512, 1) smem_rmw_kernel(int64_t per_thread, double* out) {
    extern __shared__ __align__(16) double sm[];
    double* y = sm;             // 16384
    double* x = sm + 16384;     // 12288
    for (int i = threadIdx.x; i < 16384; i += 512) y[i] = 0.0;
    for (int i = threadIdx.x; i < 12288; i += 512) x[i] = 1.0 + i;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t s = (blockIdx.x * 512 + threadIdx.x) * 2654435761u + 7u;
    uint32_t sw = (blockIdx.x * 16 + warp) * 2246822519u + 3u;
    const double v = 0.5;
    for (int64_t k = 0; k < per_thread; k += 4) {
        int r[4], c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (MODE == 0) {
                s = s * 1664525u + 1013904223u;
                r[u] = warp * 1024 + ((s >> 8) & 1023);
                s = s * 1664525u + 1013904223u;
                c[u] = (int)((s >> 8) % 12288u);
            } else {
                sw = sw * 1664525u + 1013904223u;
                r[u] = warp * 1024 + ((((sw >> 8) & 31) * 32 + lane) & 1023);
                c[u] = (int)((((sw >> 13) & 255) * 32 + lane) % 12288u);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            y[r[u]] += v * x[c[u]];
            __syncwarp();
        }
    }
    __syncthreads();
    if (y[threadIdx.x] == 1.2345) out[0] = y[threadIdx.x];
}

// ---------------------------------------------------------------- kind 4
template <int G>
__global__ void __launch_bounds__(256) line_gather_kernel(const double* __restrict__ x, int64_t n, int64_t per_thread,
                                                          double* out) {
    uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
    const uint32_t lines = (uint32_t)(n / 16);
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    for (int64_t k = 0; k < per_thread; k += 8) {
        uint32_t idx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s = s * 1664525u + 1013904223u;
            uint32_t line = (s >> 5) % lines;
            line = __shfl_sync(0xffffffffu, line, lane & ~(G - 1));   // group leader's line
            idx[u] = line * 16 + ((lane % G) * (16 / (G > 16 ? 16 : G))) % 16;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += __ldg(x + idx[u]);
    }
    if (acc == 1.2345) out[0] = acc;
}

int n_sms() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

template <int CL>
cudaError_t launch_tma(const char* src, int64_t bytes, int64_t count, double* out, cudaStream_t st) {
    const int sms = n_sms();
    const int grid = (sms / CL) * CL;
    const size_t smem = kStages * kChunk + 2 * kStages * sizeof(uint64_t);
    cudaError_t e = cudaFuncSetAttribute(tma_l2_kernel<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t chunks = count / ((int64_t)grid * kChunk);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, tma_l2_kernel<CL>, src, bytes, chunks, out);
}

}  // namespace

cudaError_t diag_micro(int kind, int param, const void* buf, int64_t bytes, int64_t count, double* out,
                       cudaStream_t st) {
    const int sms = n_sms();
    switch (kind) {
    case 1: {
        const int grid = sms * 4;
        l2read_kernel<<<grid, 512, 0, st>>>(static_cast<const int4*>(buf), bytes / 16, count / 16 / grid, out);
        return cudaGetLastError();
    }
    case 2: {
        const char* src = static_cast<const char*>(buf);
        if (bytes < kChunk) return cudaErrorInvalidValue;
        if (param == 1) return launch_tma<1>(src, bytes, count, out, st);
        if (param == 2) return launch_tma<2>(src, bytes, count, out, st);
        if (param == 4) return launch_tma<4>(src, bytes, count, out, st);
        if (param == 8) return launch_tma<8>(src, bytes, count, out, st);
        return cudaErrorInvalidValue;
    }
    case 3: {
        const size_t smem = (16384 + 12288) * sizeof(double);
        const int64_t per = count / ((int64_t)sms * 512);
        if (param == 0) {
            cudaFuncSetAttribute(smem_rmw_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            smem_rmw_kernel<0><<<sms, 512, smem, st>>>(per, out);
        } else {
            cudaFuncSetAttribute(smem_rmw_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            smem_rmw_kernel<1><<<sms, 512, smem, st>>>(per, out);
        }
        return cudaGetLastError();
    }
    case 4: {
        const double* x = static_cast<const double*>(buf);
        const int64_t n = bytes / 8;
        const int grid = sms * 8;
        const int64_t per = ((count / ((int64_t)grid * 256) + 7) / 8) * 8;
        switch (param) {
        case 1: line_gather_kernel<1><<<grid, 256, 0, st>>>(x, n, per, out); break;
        case 2: line_gather_kernel<2><<<grid, 256, 0, st>>>(x, n, per, out); break;
        case 4: line_gather_kernel<4><<<grid, 256, 0, st>>>(x, n, per, out); break;
        case 8: line_gather_kernel<8><<<grid, 256, 0, st>>>(x, n, per, out); break;
        case 16: line_gather_kernel<16><<<grid, 256, 0, st>>>(x, n, per, out); break;
        case 32: line_gather_kernel<32><<<grid, 256, 0, st>>>(x, n, per, out); break;
        default: return cudaErrorInvalidValue;
        }
        return cudaGetLastError();
    }
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace spmvb
