// split.cu -- multiple-SpMxV y = 0; y <- y + A^k x, k = 1..K,
// fused per row tile, sm_100a.
//
// Layout (host.cpp, "split layout"): within each row tile the nonzeros are
// regrouped part-major -- for k = 0..K-1 the part-k runs ("segments") of the
// tile's rows, in row order.  That is the access order the splitting Pi
// defines, executed tile by tile: the whole GPU sweeps the tiles in
// order, and inside a tile the parts are visited in order.
//
// One CTA of 512 threads per tile (same geometry as rowtile.cu):
//   1. one 128-bit quad of the tile's part-major (col, val) stream per
//      thread, L2 evict-first; x gathered through the read-only path; products
//      staged in shared memory; the tile's segment offsets and rows alongside;
//   2. for k = 0..K-1: every part-k segment of <= 32 nonzeros is summed
//      serially by one thread (the per-(row, part) temporary), longer ones by
//      a warp with a fixed tree; then ysum[row] += tmp -- y accumulated on
//      chip "on the fly" in part order, one y store per row.
//      Short segments reproduce the oracle's order bit for bit.
// Literal mode (SPMV_SPLIT_LITERAL) runs the same kernel once per part with
// ysum initialised from y: the unfused sequence of K passes.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace spmvb {
namespace {

constexpr int kST = 512;
static_assert(kST * 4 == kTileNnz, "one quad per thread");

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
__device__ __forceinline__ double ldx(const TileArgs& A, int c) {
    if (XSPLIT) return c < A.x_split ? __ldg(A.x_lo + c) : __ldg(A.x_hi + (c - A.x_split));
    return __ldg(A.x_lo + c);
}

struct SplitSmem {
    double prod[kTileNnz];
    double ysum[kTileRows];
    int32_t so[kTileNnz + 1];       // segment offsets (positions from a4), all parts of the tile
    int32_t srow[kTileNnz];         // tile-local row of each segment
    int32_t kseg[65];               // first segment of part k (relative), K <= 64
    int32_t longsegs[kTileNnz];
    int32_t nlong;
    double red[kST / 32];
};

// sum of positions [p0, p1) of a long segment by one warp (fixed order)
__device__ __forceinline__ double warp_sum(const SplitSmem& sm, int p0, int p1, int lane) {
    double acc = 0.0;
    for (int p = p0 + lane; p < p1; p += 32) acc += sm.prod[p];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    return acc;
}

template <bool XSPLIT>
__global__ void __launch_bounds__(kST, 2) spmv_split_kernel(const TileArgs A) {
    __shared__ __align__(16) SplitSmem sm;
    const int t = blockIdx.x;
    const int tid = threadIdx.x;
    const int K = A.K;
    const int kb = A.k_begin, ke = A.k_end;
    const int s_lo = A.tile_seg[t * K + kb], s_hi = A.tile_seg[t * K + ke];
    if (A.accumulate && s_lo == s_hi) return;           // literal pass: no part-k rows here
    const int r0 = A.tile_row[t];
    const int nr = A.tile_row[t + 1] - r0;
    const int a = A.seg_ptr[s_lo], b = A.seg_ptr[s_hi];
    const int a4 = a & ~3;
    const uint64_t pol = pol_evict_first();

    for (int j = tid; j < nr; j += kST) sm.ysum[j] = A.accumulate ? A.y[r0 + j] : 0.0;

    if (b - a + 3 > kTileNnz) {   // long row: planned as one (host plan_tiles, alignment-free test)
        // one long row (the tile is a single row): per part, fixed-assignment
        // partials + fixed block tree, accumulated in part order
        __syncthreads();
        for (int k = kb; k < ke; ++k) {
            const int s0 = A.tile_seg[t * K + k], s1 = A.tile_seg[t * K + k + 1];
            if (s0 == s1) continue;
            const int64_t pa = A.seg_ptr[s0], pb = A.seg_ptr[s1];
            double acc = 0.0;
            for (int64_t q = (pa >> 2) + tid; q < ((pb + 3) >> 2); q += kST) {
                const int4 c = ld_v4(A.col + 4 * q, pol);
                const double2 v0 = ld_v2d(A.val + 4 * q, pol);
                const double2 v1 = ld_v2d(A.val + 4 * q + 2, pol);
                const int64_t g = 4 * q;
                if (g + 0 >= pa && g + 0 < pb) acc += v0.x * ldx<XSPLIT>(A, c.x);
                if (g + 1 >= pa && g + 1 < pb) acc += v0.y * ldx<XSPLIT>(A, c.y);
                if (g + 2 >= pa && g + 2 < pb) acc += v1.x * ldx<XSPLIT>(A, c.z);
                if (g + 3 >= pa && g + 3 < pb) acc += v1.y * ldx<XSPLIT>(A, c.w);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if ((tid & 31) == 0) sm.red[tid >> 5] = acc;
            __syncthreads();
            if (tid == 0) {
                double tot = 0.0;
                for (int w = 0; w < kST / 32; ++w) tot += sm.red[w];
                sm.ysum[0] += tot;
            }
            __syncthreads();
        }
    } else {
        // ------------------------------------------- stage products, segments
        const int nseg = s_hi - s_lo;
        for (int j = tid; j <= nseg; j += kST) sm.so[j] = A.seg_ptr[s_lo + j] - a4;
        for (int j = tid; j < nseg; j += kST) sm.srow[j] = A.seg_row[s_lo + j];
        for (int k = kb + tid; k <= ke; k += kST) sm.kseg[k - kb] = A.tile_seg[t * K + k] - s_lo;
        if (tid == 0) sm.nlong = 0;
        {
            // branch-free: loads clamped to a valid quad, products masked
            const int p = 4 * tid;
            const int pq = (a4 + p < b) ? p : 0;
            const int4 c = ld_v4(A.col + a4 + pq, pol);
            const double2 v0 = ld_v2d(A.val + a4 + pq, pol);
            const double2 v1 = ld_v2d(A.val + a4 + pq + 2, pol);
            const int lo = a - a4, hi = b - a4;
            const double x0 = ldx<XSPLIT>(A, c.x), x1 = ldx<XSPLIT>(A, c.y);
            const double x2 = ldx<XSPLIT>(A, c.z), x3 = ldx<XSPLIT>(A, c.w);
            double2 w0, w1;
            w0.x = (p + 0 >= lo && p + 0 < hi) ? v0.x * x0 : 0.0;
            w0.y = (p + 1 >= lo && p + 1 < hi) ? v0.y * x1 : 0.0;
            w1.x = (p + 2 >= lo && p + 2 < hi) ? v1.x * x2 : 0.0;
            w1.y = (p + 3 >= lo && p + 3 < hi) ? v1.y * x3 : 0.0;
            if (a4 + p < b) {
                *reinterpret_cast<double2*>(&sm.prod[p]) = w0;
                *reinterpret_cast<double2*>(&sm.prod[p + 2]) = w1;
            }
        }
        __syncthreads();
        // ------------------------------------------- parts in order
        const int warp = tid >> 5, lane = tid & 31;
        for (int k = 0; k < ke - kb; ++k) {
            const int j0 = sm.kseg[k], j1 = sm.kseg[k + 1];
            if (j0 == j1) continue;                                 // CTA-uniform
            bool any_long = false;
            for (int j = j0 + tid; j < j1; j += kST) {
                const int p0 = sm.so[j], p1 = sm.so[j + 1];
                if (p1 - p0 <= kShortRow) {
                    double tmp = 0.0;
                    for (int p = p0; p < p1; ++p) tmp += sm.prod[p];
                    sm.ysum[sm.srow[j]] += tmp;                     // one segment per row per part
                } else {
                    sm.longsegs[atomicAdd(&sm.nlong, 1)] = j;
                    any_long = true;
                }
            }
            if (__syncthreads_or(any_long)) {
                for (int i = warp; i < sm.nlong; i += kST / 32) {
                    const int j = sm.longsegs[i];
                    const double tmp = warp_sum(sm, sm.so[j], sm.so[j + 1], lane);
                    if (lane == 0) sm.ysum[sm.srow[j]] += tmp;
                }
                __syncthreads();
                if (tid == 0) sm.nlong = 0;
            }
            __syncthreads();
        }
    }

    double mx = 0.0;
    for (int j = tid; j < nr; j += kST) {
        const double v = sm.ysum[j];
        A.y[r0 + j] = v;
        mx = fmax(mx, fabs(v));
    }
    if (A.maxabs_slots) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if ((tid & 31) == 0 && mx > 0.0)
            atomicMax(A.maxabs_slots + (t & (kMaxSlots - 1)) * kSlotStride,
                      (unsigned long long)__double_as_longlong(mx));
    }
}

}  // namespace

cudaError_t launch_split(const TileArgs& a, bool xsplit, cudaStream_t s) {
    if (a.n_tiles <= 0) return cudaSuccess;
    if (a.K > 64) return cudaErrorInvalidValue;
    if (xsplit) spmv_split_kernel<true><<<a.n_tiles, kST, 0, s>>>(a);
    else spmv_split_kernel<false><<<a.n_tiles, kST, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace spmvb

// ---------------------------------------------------------------------------
// spmv_split_rows_kernel: fused multiple-SpMxV over the row-major segment
// layout (host.cpp): row r's nonzeros are grouped by part, its segments are
// [row_seg[r], row_seg[r+1]) in part order, segment s covers stream
// positions [seg_ptr[s], seg_ptr[s+1]).  Same tiles and streaming as the
// row-tile kernel (rowtile.cu); the reduction walks each row's segments in
// part order, each into its own temporary, y_r += tmp (reading
// A7) -- so no per-part CTA barriers are needed: the per-row order is the
// whole ordering constraint.  Segments of <= 32 nonzeros are summed serially
// (the oracle's order); rows with a longer segment go to a warp (fixed tree).
namespace spmvb {
namespace {

constexpr int kSR = 256;                      // threads per tile CTA
constexpr int kSRQ = kTileNnz / (4 * kSR);    // quads per thread

__device__ __forceinline__ double ldx_r(const RowTileArgs& A, int c, uint64_t pl) {
    const double* p = c < A.x_split ? A.x_lo + c : A.x_hi + (c - A.x_split);
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pl));
    return v;
}

struct SplitRowsSmem {
    double prod[kTileNnz];
    int32_t sp[kTileNnz + 1];       // seg_ptr[s] - a4 for the tile's segments (each has >= 1 nonzero)
    int32_t rs[kTileRows + 1];      // row_seg[r0 + j] - row_seg[r0]
    int32_t longrows[kTileRows];
    int32_t nlong;
    double red[kSR / 32];
};

template <bool XSPLIT>
__global__ void __launch_bounds__(kSR, 4) spmv_split_rows_kernel(const RowTileArgs A, const int32_t* __restrict__ row_seg,
                                                               const int32_t* __restrict__ seg_ptr) {
    __shared__ __align__(16) SplitRowsSmem sm;
    const int t = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r0 = A.tile_row[t], r1 = A.tile_row[t + 1];
    const int a = A.tile_nnz[t], b = A.tile_nnz[t + 1];
    const int nr = r1 - r0;
    const int a4 = a & ~3;
    const uint64_t pol = pol_evict_first();
    uint64_t pl;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
    double mx = 0.0;

    if (b - a + 3 > kTileNnz) {   // long row: planned as one (host plan_tiles, alignment-free test)
        // one long row: per segment (part order), fixed-assignment partials +
        // fixed block tree, accumulated in part order
        double yr = 0.0;
        const int s0 = row_seg[r0], s1 = row_seg[r0 + 1];
        for (int sg = s0; sg < s1; ++sg) {
            const int pa = seg_ptr[sg], pb = seg_ptr[sg + 1];
            double acc = 0.0;
            for (int e = pa + tid; e < pb; e += kSR) {
                int32_t c;
                double v;
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(c) : "l"(A.col + e), "l"(pol));
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(A.val + e), "l"(pol));
                acc += v * (XSPLIT ? ldx_r(A, c, pl) : ldx_r(A, c, pl));
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) sm.red[warp] = acc;
            __syncthreads();
            if (tid == 0) {
                double tot = 0.0;
                for (int w = 0; w < kSR / 32; ++w) tot += sm.red[w];
                yr += tot;
            }
            __syncthreads();
        }
        if (tid == 0) {
            A.y[r0] = yr;
            if (A.maxabs_slots && yr != 0.0)
                atomicMax(A.maxabs_slots + (t & (kMaxSlots - 1)) * kSlotStride,
                          (unsigned long long)__double_as_longlong(fabs(yr)));
        }
        return;
    }

    // ------------------------------------------------ stage products
    const int sbase = row_seg[r0];
    for (int j = tid; j <= nr; j += kSR) sm.rs[j] = row_seg[r0 + j] - sbase;
    {
        const int ns = row_seg[r1] - sbase;
        for (int j = tid; j <= ns; j += kSR) sm.sp[j] = seg_ptr[sbase + j] - a4;
    }
    if (tid == 0) sm.nlong = 0;
    {
        const int lo = a - a4, hi = b - a4;
        int4 c[kSRQ];
        double2 v0[kSRQ], v1[kSRQ];
#pragma unroll
        for (int k = 0; k < kSRQ; ++k) {   // branch-free: clamped loads, unconditional gathers
            const int p = 4 * (tid + k * kSR);
            const int pq = (a4 + p < b) ? p : 0;
            c[k] = ld_v4(A.col + a4 + pq, pol);
            v0[k] = ld_v2d(A.val + a4 + pq, pol);
            v1[k] = ld_v2d(A.val + a4 + pq + 2, pol);
        }
        double xv[kSRQ][4];
#pragma unroll
        for (int k = 0; k < kSRQ; ++k) {
            xv[k][0] = ldx_r(A, c[k].x, pl);
            xv[k][1] = ldx_r(A, c[k].y, pl);
            xv[k][2] = ldx_r(A, c[k].z, pl);
            xv[k][3] = ldx_r(A, c[k].w, pl);
        }
#pragma unroll
        for (int k = 0; k < kSRQ; ++k) {
            const int p = 4 * (tid + k * kSR);
            double2 w0, w1;
            w0.x = (p + 0 >= lo && p + 0 < hi) ? v0[k].x * xv[k][0] : 0.0;
            w0.y = (p + 1 >= lo && p + 1 < hi) ? v0[k].y * xv[k][1] : 0.0;
            w1.x = (p + 2 >= lo && p + 2 < hi) ? v1[k].x * xv[k][2] : 0.0;
            w1.y = (p + 3 >= lo && p + 3 < hi) ? v1[k].y * xv[k][3] : 0.0;
            if (a4 + p < b) {
                *reinterpret_cast<double2*>(&sm.prod[p]) = w0;
                *reinterpret_cast<double2*>(&sm.prod[p + 2]) = w1;
            }
        }
    }
    __syncthreads();

    // ------------------------------------------------ rows: segments in part order
    for (int r = tid; r < nr; r += kSR) {
        const int s0 = sm.rs[r], s1 = sm.rs[r + 1];
        bool lng = false;
        for (int sg = s0; sg < s1; ++sg) lng |= sm.sp[sg + 1] - sm.sp[sg] > kShortRow;
        if (lng) {
            sm.longrows[atomicAdd(&sm.nlong, 1)] = r;   // summed by one warp below (order irrelevant)
            continue;
        }
        double yr = 0.0;
        for (int sg = s0; sg < s1; ++sg) {
            const int p1 = sm.sp[sg + 1];
            double tmp = 0.0;
            for (int p = sm.sp[sg]; p < p1; ++p) tmp += sm.prod[p];
            yr += tmp;
        }
        A.y[r0 + r] = yr;
        mx = fmax(mx, fabs(yr));
    }
    __syncthreads();
    for (int k = warp; k < sm.nlong; k += kSR / 32) {
        const int r = sm.longrows[k];
        double yr = 0.0;
        for (int sg = sm.rs[r]; sg < sm.rs[r + 1]; ++sg) {
            const int p0 = sm.sp[sg], p1 = sm.sp[sg + 1];
            double tmp = 0.0;
            if (p1 - p0 <= kShortRow) {
                if (lane == 0)
                    for (int p = p0; p < p1; ++p) tmp += sm.prod[p];
            } else {
                for (int p = p0 + lane; p < p1; p += 32) tmp += sm.prod[p];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) tmp += __shfl_xor_sync(0xffffffffu, tmp, off);
            }
            yr += tmp;   // lane 0's copy is the row's value
        }
        if (lane == 0) {
            A.y[r0 + r] = yr;
            mx = fmax(mx, fabs(yr));
        }
    }
    if (A.maxabs_slots) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if (lane == 0 && mx > 0.0)
            atomicMax(A.maxabs_slots + ((t * (kSR / 32) + warp) & (kMaxSlots - 1)) * kSlotStride,
                      (unsigned long long)__double_as_longlong(mx));
    }
}

}  // namespace

cudaError_t launch_split_rows(const RowTileArgs& a, const int32_t* row_seg, const int32_t* seg_ptr, bool xsplit,
                              cudaStream_t s) {
    if (a.n_tiles <= 0) return cudaSuccess;
    if (xsplit) spmv_split_rows_kernel<true><<<a.n_tiles, kSR, 0, s>>>(a, row_seg, seg_ptr);
    else spmv_split_rows_kernel<false><<<a.n_tiles, kSR, 0, s>>>(a, row_seg, seg_ptr);
    return cudaGetLastError();
}


// Loads this file's kernels now (cudaFuncGetAttributes forces the lazy loader):
// a kernel first launched while a peer rank's kernel spins on an exchange flag
// would otherwise load its module then, and a module load can wait for the
// running kernels -- the spinning one included (see host.cpp preload_kernels).
cudaError_t preload_kernels_split() {
    cudaFuncAttributes fa;
    for (const void* k : {(const void*)spmv_split_kernel<false>, (const void*)spmv_split_kernel<true>,
                          (const void*)spmv_split_rows_kernel<false>, (const void*)spmv_split_rows_kernel<true>}) {
        const cudaError_t e = cudaFuncGetAttributes(&fa, k);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace spmvb
