// panel.cu -- column-sorted panel SpMxV y^ = A^ x^ for SB-form
// matrices (Eq.(1)): the default single-SpMxV kernel of SB handles.
//
// Why (measured on B200, profiles/r01_micro.json): an x gather
// costs one L1TEX wavefront per distinct 128-byte line it touches, ~1 line per
// SM clock.  Row-ordered CSR pays one line per nonzero (C5's columns are
// random inside a 7.8 MB block of x), capping it at ~4.5 ms on C5 against a
// 2.2 ms HBM floor.  Here a CTA owns a panel of up to 28,672 rows of one SB
// block -- the rows that share x(C_k), the block's reused part of x
// -- keeps their y in shared memory, and walks the panel's nonzeros sorted by
// column (plan_panel.cpp), so a warp's 32 gathers hit only a few lines.
//
// One CTA of 16 warps per panel (224 KB of shared memory, 1 CTA per SM).
// Warp w processes groups g0 + 16 t + w, t = 0, 1, ...; every kPnB steps is an
// epoch boundary (__syncthreads): within an epoch all rows are distinct, so
// the shared-memory read-modify-writes y_s[r] += v * x[c] never race.
// Per warp, a register ring keeps kD groups of (value, index, base) in
// flight (L1 no-allocate, L2 evict-first: the matrix is read once) and
// issues the x gathers kGD steps ahead of their use.  The epilogue writes y
// once per row and folds max |y|.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace spmvb {
namespace {

constexpr int NW = kPnWarps;
constexpr int kT = NW * 32;
constexpr int kD = 16;    // groups in flight per warp
constexpr int kGD = 8;    // gathers issued this many steps ahead
static_assert(kD % kPnB == 0 && kD % kGD == 0, "ring geometry");
constexpr uint32_t kDeltaMask = (1u << kPnDeltaBits) - 1u;

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
__device__ __forceinline__ uint32_t ld_u32(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int32_t ld_base(const int32_t* p) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__global__ void __launch_bounds__(kT, 1) spmv_panel_kernel(const PnArgs A) {
    extern __shared__ __align__(16) double ys[];
    const int p = blockIdx.x;
    const PnPanel d = A.panel[p];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < d.nrows; i += kT) ys[i] = 0.0;
    __syncthreads();

    const uint64_t pol = pol_evict_first();
    const int T = d.ne * kPnB;                       // steps per warp
    const int64_t gw = (int64_t)d.g0 + warp;         // group of step t: gw + 16 t

    double rv[kD];
    uint32_t ri[kD];
    int32_t rb[kD];
    double rx[kGD];
    auto load = [&](int t, double& v, uint32_t& i, int32_t& b) {
        const int64_t g = gw + 16 * (int64_t)t;
        v = ld_val(A.gval + g * 32 + lane, pol);
        i = ld_u32(A.gidx + g * 32 + lane, pol);
        b = ld_base(A.gbase + g);
    };
    auto gather = [&](uint32_t i, int32_t b) -> double {
        if (i == kPnDummy) return 0.0;
        const double* xp = b < A.x_split ? A.x_lo + b : A.x_hi + (b - A.x_split);
        return __ldg(xp + (i & kDeltaMask));
    };
#pragma unroll
    for (int u = 0; u < kD; ++u)
        if (u < T) load(u, rv[u], ri[u], rb[u]);
#pragma unroll
    for (int u = 0; u < kGD; ++u)
        if (u < T) rx[u] = gather(ri[u], rb[u]);

    for (int t0 = 0; t0 < T; t0 += kD) {
#pragma unroll
        for (int u = 0; u < kD; ++u) {
            const int t = t0 + u;
            if (t >= T) break;
            const uint32_t i = ri[u];
            if (i != kPnDummy) {
                const int r = (int)(i >> kPnDeltaBits);
                ys[r] = fma(rv[u], rx[u % kGD], ys[r]);
            }
            if (t + kD < T) load(t + kD, rv[u], ri[u], rb[u]);
            if (t + kGD < T) rx[u % kGD] = gather(ri[(u + kGD) % kD], rb[(u + kGD) % kD]);
            if (u % kPnB == kPnB - 1) __syncthreads();   // epoch boundary (T is a multiple of kPnB)
        }
    }
    __syncthreads();

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
            atomicMax(A.maxabs_slots + ((p * NW + warp) & (kMaxSlots - 1)) * kSlotStride,
                      (unsigned long long)__double_as_longlong(mx));
    }
}

}  // namespace

cudaError_t launch_panel(const PnArgs& a, cudaStream_t s) {
    if (a.n_panels <= 0) return cudaSuccess;
    static bool attr_done = false;
    const size_t smem = (size_t)kPnRowsMax * sizeof(double);
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(spmv_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    spmv_panel_kernel<<<a.n_panels, kT, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace spmvb
