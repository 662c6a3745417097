// rowtile.cu -- the default single-SpMxV kernel y^ = A^ x^: one CTA
// of 512 threads per row tile of <= 2048 nonzeros, launched in tile order.
//
// Why this shape (measured on B200): the x gathers are the
// binding limit (~1 lane-request per clock per SM through the LSU,
// scripts/gather_modes.py), so the kernel maximises independent gathers in
// flight: 3 CTAs x 512 threads per SM, one 128-bit quad of (col, val) per
// thread, no per-tile pipeline barriers beyond one __syncthreads.  The
// hardware block scheduler issues tiles in order, so all SMs sweep the rows
// together and the live x footprint is one SB block's x(C_k) + x(C_B)
// (Eq.(1)) -- L2-resident, the paper's "fits into the cache"
// condition with the 126 MB L2 as the cache.  (A persistent schedule
// with static tile strides let CTAs drift and overflowed L2: 4.7x the
// algorithmic DRAM bytes on C5.)
//
// Per tile:
//   1. thread q loads quad q of the tile's col/val (positions 4q..4q+3 from
//      the 16-byte aligned a & ~3), L1 no-allocate + L2 evict-first (the
//      matrix is read once), gathers x[col] through the read-only path
//      (x is the reused operand) and stages the products in shared
//      memory; the tile's row pointers are staged alongside;
//   2. tiles whose rows all have <= 32 nonzeros: vector-per-row, V lanes per
//      row (V = 1..32 chosen per tile at plan time so that rows x V fills the
//      CTA; V = 1 is the paper's serial per-row temporary); lane j
//      sums positions j, j+V, ... of its row, then a fixed xor-shuffle tree;
//      other tiles: thread-per-row for rows <= 32, warp-per-row (fixed lane
//      assignment and tree) for longer rows;
//   3. y is stored coalesced; max |y| is folded per CTA (one atomicMax).
// Rows longer than a tile get a tile of their own: all 512 threads stream
// the row with a fixed assignment and a fixed tree.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace spmvb {
namespace {

constexpr int kRT = 512;                 // threads per tile CTA (one quad each)
static_assert(kRT * 4 == kTileNnz, "one quad per thread");

__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int4 ld_v4(const int32_t* ptr, uint64_t pol) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ double2 ld_v2d(const double* ptr, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(ptr), "l"(pol));
    return r;
}

template <bool XSPLIT>
__device__ __forceinline__ double ldx(const RowTileArgs& A, int c) {
    if (XSPLIT) return c < A.x_split ? __ldg(A.x_lo + c) : __ldg(A.x_hi + (c - A.x_split));
    return __ldg(A.x_lo + c);
}

struct RTSmem {
    double prod[kTileNnz];          // product of position p (nonzero a4 + p)
    int32_t so[kTileRows + 1];      // row_ptr[r0 + j] - a4
    int32_t longrows[kTileRows];    // general tiles: rows with > 32 nonzeros
    int32_t nlong;
    double red[kRT / 32];
};

template <bool XSPLIT>
__global__ void __launch_bounds__(kRT, 3) spmv_rowtile_kernel(const RowTileArgs A) {
    __shared__ __align__(16) RTSmem sm;
    const int t = blockIdx.x;
    const int tid = threadIdx.x;
    const int r0 = A.tile_row[t], r1 = A.tile_row[t + 1];
    const int a = A.tile_nnz[t], b = A.tile_nnz[t + 1];
    const int cls = A.tile_cls[t];
    const int nr = r1 - r0;
    const int a4 = a & ~3;
    const uint64_t pol = pol_evict_first();
    double mx = 0.0;

    if (b - a4 > kTileNnz) {
        // ------------------------------------------- one long row (> a tile)
        const int64_t qa = a >> 2, qb = ((int64_t)b + 3) >> 2;
        double acc = 0.0;
        for (int64_t q = qa + tid; q < qb; q += kRT) {
            const int4 c = ld_v4(A.col + 4 * q, pol);
            const double2 v0 = ld_v2d(A.val + 4 * q, pol);
            const double2 v1 = ld_v2d(A.val + 4 * q + 2, pol);
            const int64_t g = 4 * q;
            if (g + 0 >= a && g + 0 < b) acc += v0.x * ldx<XSPLIT>(A, c.x);
            if (g + 1 >= a && g + 1 < b) acc += v0.y * ldx<XSPLIT>(A, c.y);
            if (g + 2 >= a && g + 2 < b) acc += v1.x * ldx<XSPLIT>(A, c.z);
            if (g + 3 >= a && g + 3 < b) acc += v1.y * ldx<XSPLIT>(A, c.w);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if ((tid & 31) == 0) sm.red[tid >> 5] = acc;
        __syncthreads();
        if (tid == 0) {
            double tot = 0.0;
            for (int w = 0; w < kRT / 32; ++w) tot += sm.red[w];
            A.y[r0] = tot;
            if (A.maxabs_slots && tot != 0.0)
                atomicMax(A.maxabs_slots + (t & (kMaxSlots - 1)) * kSlotStride,
                          (unsigned long long)__double_as_longlong(fabs(tot)));
        }
        return;
    }

    // ------------------------------------------------ stage products, so[]
    for (int j = tid; j <= nr; j += kRT) sm.so[j] = A.rowptr[r0 + j] - a4;
    if (tid == 0) sm.nlong = 0;
    {
        const int q = tid;                               // quad of positions 4q..4q+3
        const int p = 4 * q;
        if (a4 + p < b) {
            const int4 c = ld_v4(A.col + a4 + p, pol);
            const double2 v0 = ld_v2d(A.val + a4 + p, pol);
            const double2 v1 = ld_v2d(A.val + a4 + p + 2, pol);
            const int lo = a - a4, hi = b - a4;
            const double x0 = (p + 0 >= lo && p + 0 < hi) ? ldx<XSPLIT>(A, c.x) : 0.0;
            const double x1 = (p + 1 >= lo && p + 1 < hi) ? ldx<XSPLIT>(A, c.y) : 0.0;
            const double x2 = (p + 2 >= lo && p + 2 < hi) ? ldx<XSPLIT>(A, c.z) : 0.0;
            const double x3 = (p + 3 >= lo && p + 3 < hi) ? ldx<XSPLIT>(A, c.w) : 0.0;
            double2 w0, w1;
            w0.x = v0.x * x0; w0.y = v0.y * x1;
            w1.x = v1.x * x2; w1.y = v1.y * x3;
            *reinterpret_cast<double2*>(&sm.prod[p]) = w0;
            *reinterpret_cast<double2*>(&sm.prod[p + 2]) = w1;
        }
    }
    __syncthreads();

    // ------------------------------------------------------- row sums
    if (cls >= kTileShort) {
        // every row <= 32 nonzeros: V = cls lanes per row (vector-per-row,
        // V chosen at plan time so nr*V <= 512); lane j sums positions
        // p0+j, p0+j+V, ... serially, then a fixed xor-shuffle tree.
        const int V = cls;
        const int r = tid / V;
        const int j = tid - r * V;
        double acc = 0.0;
        if (r < nr) {
            const int p1 = sm.so[r + 1];
            for (int p = sm.so[r] + j; p < p1; p += V) acc += sm.prod[p];
        }
        for (int off = V >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (r < nr && j == 0) {
            A.y[r0 + r] = acc;
            mx = acc < 0 ? -acc : acc;
        }
    } else {
        // short rows: one thread each; long rows: listed, then one warp each
        for (int r = tid; r < nr; r += kRT) {
            const int p0 = sm.so[r], p1 = sm.so[r + 1];
            if (p1 - p0 <= kShortRow) {
                double acc = 0.0;
                for (int p = p0; p < p1; ++p) acc += sm.prod[p];
                A.y[r0 + r] = acc;
                mx = fmax(mx, fabs(acc));
            } else {
                sm.longrows[atomicAdd(&sm.nlong, 1)] = r;    // order irrelevant: each row is summed
            }                                                // by one warp in a fixed order
        }
        __syncthreads();
        const int warp = tid >> 5, lane = tid & 31;
        for (int k = warp; k < sm.nlong; k += kRT / 32) {
            const int r = sm.longrows[k];
            const int p0 = sm.so[r], p1 = sm.so[r + 1];
            double acc = 0.0;
            for (int p = p0 + lane; p < p1; p += 32) acc += sm.prod[p];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) {
                A.y[r0 + r] = acc;
                mx = fmax(mx, fabs(acc));
            }
        }
    }
    if (A.maxabs_slots) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        __syncthreads();
        if ((tid & 31) == 0) sm.red[tid >> 5] = mx;
        __syncthreads();
        if (tid == 0) {
            double m = 0.0;
            for (int w = 0; w < kRT / 32; ++w) m = fmax(m, sm.red[w]);
            if (m > 0.0)
                atomicMax(A.maxabs_slots + (t & (kMaxSlots - 1)) * kSlotStride,
                          (unsigned long long)__double_as_longlong(m));
        }
    }
}

}  // namespace

cudaError_t launch_rowtile(const RowTileArgs& a, bool xsplit, cudaStream_t s) {
    if (a.n_tiles <= 0) return cudaSuccess;
    if (xsplit) spmv_rowtile_kernel<true><<<a.n_tiles, kRT, 0, s>>>(a);
    else spmv_rowtile_kernel<false><<<a.n_tiles, kRT, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace spmvb
