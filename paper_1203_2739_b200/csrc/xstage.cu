// xstage.cu -- x-staged single-SpMxV y^ = A^ x^ for SB-form matrices
// (Eq.(1)): the default kernel of SB handles on sm_100a.
//
// Why (measured on B200, profiles/r01_micro.json): a random 8-byte x gather
// from L2 costs one L1TEX wavefront per distinct 128-byte line, ~1 per SM
// clock (280 G/s chip-wide), which caps a gather-per-nonzero kernel at ~4.5 ms
// on C5 against a 2.2 ms HBM floor.  Shared-memory updates y[r] += v*x[c]
// run at 1.5 T/s when bank-conflict-free, and the bulk-copy engine moves
// L2-resident data into shared memory at ~20 TB/s.  So the x entries the
// reordering makes reusable -- one SB block's interior columns C_k, the
// paper's "fits into the cache" unit -- are streamed through
// shared memory, and only the coupling columns C_B are gathered
// from L2.
//
// One CTA per panel (a run of <= kXsRowsMax rows of one block), 16 consumer
// warps + 1 producer warp, 1 CTA per SM (~225 KB shared memory):
//   producer : streams x(C_k) in chunks of kXsW columns into a 3-stage ring
//              with cp.async.bulk (TMA), full/empty mbarriers;
//   consumers: warp w owns panel rows [w*rw, (w+1)*rw) and walks its packed
//              nonzero groups (plan_xs.cpp): first the border groups (x from
//              L2, gathers issued 4 groups ahead), then the interior groups
//              in chunk order, each lane doing y_s[r] += v * x_s[c];
//              group data are prefetched 16 groups ahead (L1 no-allocate, L2
//              evict-first: the matrix is read once);
//   epilogue : y_s is written to HBM once per row, max |y| folded.
// The per-row order of products is fixed by the plan: deterministic.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace spmvb {
namespace {

constexpr int NW = kXsWarps;
constexpr int NS = kXsStages;
constexpr int SS = kXsStageStride;
constexpr int kT = (NW + 1) * 32;
constexpr int kD = 16;    // groups in flight per warp
constexpr int kGD = 4;    // border gathers issued this many groups ahead

__device__ __forceinline__ uint32_t sptr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nXW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra XW;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_val(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ld_idx(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

__global__ void __launch_bounds__(kT, 1) spmv_xstage_kernel(const XsArgs A) {
    extern __shared__ __align__(128) unsigned char smraw[];
    double* ys = reinterpret_cast<double*>(smraw);
    double* xs = ys + kXsRowsMax;
    uint64_t* full = reinterpret_cast<uint64_t*>(xs + NS * SS);
    uint64_t* empty = full + NS;

    const int p = blockIdx.x;
    const XsPanel d = A.panel[p];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(sptr(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(sptr(&empty[s])), "r"(NW));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    for (int i = tid; i < d.nrows; i += kT) ys[i] = 0.0;
    __syncthreads();

    // physical chunk start is 16-byte aligned: shift = 1 when x + col0 is not
    const int shift = (int)((reinterpret_cast<uintptr_t>(A.x + d.col0) >> 3) & 1);

    if (warp == NW) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            for (int j = 0; j < d.nch; ++j) {
                const int s = j % NS;
                if (j >= NS) mbar_wait(sptr(&empty[s]), (uint32_t)(((j / NS) - 1) & 1));
                const int lo = d.col0 + j * kXsW - shift;
                const int hi = min(d.col0 + (j + 1) * kXsW, d.col_end);
                const int n = hi - lo, n2 = n & ~1;
                double* dst = xs + s * SS;
                if (n & 1) dst[n - 1] = __ldg(A.x + lo + n - 1);   // odd tail: plain copy
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(&full[s])),
                             "r"(n2 * 8)
                             : "memory");
                if (n2)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            sptr(dst)),
                        "l"(A.x + lo), "r"(n2 * 8), "r"(sptr(&full[s]))
                        : "memory");
            }
        }
    } else {
        // ----------------------------------------------------------- consumers
        const uint64_t pol = pol_evict_first();
        const int wi = p * NW + warp;
        const int b0 = A.wb[wi], nb = A.wb[wi + 1] - b0;
        const int g0 = A.wg[wi], ni = A.wg[wi + 1] - g0;
        const int nq = nb + ni;
        const int rw0 = warp * d.rw;
        const uint32_t cmask = (A.cbits >= 32) ? 0xFFFFFFFFu : ((1u << A.cbits) - 1u);
        const int nch = d.nch;
        const int32_t* U = A.U + d.u_base + warp * nch;
        int jcur = 0, jw = 0, jr = 0;
        int nextU = nch > 1 ? __ldg(U + 1) : 0x7fffffff;

        auto release = [&](int j) {
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sptr(&empty[j % NS])) : "memory");
        };
        double rv[kD];
        uint32_t ri[kD];
        double rx[kGD];
        auto load = [&](int q, double& v, uint32_t& i) {
            if (q < nb) {
                const int64_t o = (int64_t)(b0 + q) * 32 + lane;
                v = ld_val(A.bval + o, pol);
                i = ld_idx(A.bidx + o, pol);
            } else if (q < nq) {
                const int64_t o = (int64_t)(g0 + q - nb) * 32 + lane;
                v = ld_val(A.gval + o, pol);
                i = ld_idx(A.gidx + o, pol);
            }
        };
#pragma unroll
        for (int u = 0; u < kD; ++u) load(u, rv[u], ri[u]);
#pragma unroll
        for (int u = 0; u < kGD; ++u)
            if (u < nb && ri[u] != kXsDummy) rx[u] = __ldg(A.xg + (ri[u] & cmask));

        for (int q0 = 0; q0 < nq; q0 += kD) {
#pragma unroll
            for (int u = 0; u < kD; ++u) {
                const int q = q0 + u;
                if (q >= nq) break;
                const uint32_t i = ri[u];
                if (q < nb) {
                    if (i != kXsDummy) {
                        const int r = rw0 + (int)(i >> A.cbits);
                        ys[r] = fma(rv[u], rx[u % kGD], ys[r]);
                    }
                } else {
                    const int gq = q - nb;
                    while (gq >= nextU) {
                        ++jcur;
                        nextU = (jcur + 1 < nch) ? __ldg(U + jcur + 1) : 0x7fffffff;
                    }
                    // release chunks this warp is done with before waiting for
                    // new ones (the producer refills a stage only after every
                    // warp has released it)
                    const int need = min(jcur + 1, nch - 1);
                    if (jr < jcur || jw <= need) {
                        __syncwarp();
                        while (jw <= need) {
                            while (jr < jcur && jr < jw) release(jr++);
                            mbar_wait(sptr(&full[jw % NS]), (uint32_t)((jw / NS) & 1));
                            ++jw;
                        }
                        while (jr < jcur) release(jr++);
                    }
                    if (i != kXsDummy) {
                        const int r = (int)(i >> 16);
                        int off = (int)(i & 0xFFFFu);
                        int st = jcur;
                        if (off >= kXsW) {
                            off -= kXsW;
                            ++st;
                        }
                        const double xv = xs[(st % NS) * SS + shift + off];
                        ys[r] = fma(rv[u], xv, ys[r]);
                    }
                }
                __syncwarp();
                // refill: group q + kD into this slot; border gather for q + kGD
                load(q + kD, rv[u], ri[u]);
                const int qg = q + kGD;
                if (qg < nb) {
                    const uint32_t ig = ri[(u + kGD) % kD];
                    if (ig != kXsDummy) rx[u % kGD] = __ldg(A.xg + (ig & cmask));
                }
            }
        }
        // every chunk is waited for and released exactly once per warp, in order
        __syncwarp();
        while (jr < nch) {
            if (jr < jw) {
                release(jr++);
            } else {
                mbar_wait(sptr(&full[jw % NS]), (uint32_t)((jw / NS) & 1));
                ++jw;
            }
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- epilogue
    double mx = 0.0;
    for (int i = tid; i < d.nrows; i += kT) {
        const double v = ys[i];
        A.y[d.row0 + i] = v;
        mx = fmax(mx, fabs(v));
    }
    if (A.maxabs_slots) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if (lane == 0 && mx > 0.0)
            atomicMax(A.maxabs_slots + ((p * (NW + 1) + warp) & (kMaxSlots - 1)) * kSlotStride,
                      (unsigned long long)__double_as_longlong(mx));
    }
}

}  // namespace

size_t xstage_smem_bytes() {
    return (size_t)kXsRowsMax * 8 + (size_t)NS * SS * 8 + 2 * NS * sizeof(uint64_t);
}

cudaError_t launch_xstage(const XsArgs& a, cudaStream_t s) {
    if (a.n_panels <= 0) return cudaSuccess;
    static bool attr_done = false;
    const size_t smem = xstage_smem_bytes();
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(spmv_xstage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    spmv_xstage_kernel<<<a.n_panels, kT, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace spmvb
