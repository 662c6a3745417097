// rowtile.cu -- the row-tile single-SpMxV kernel y^ = A^ x^: the
// default for matrices without an SB descriptor (C1, C4) and the fallback
// when the panel plan pads too much (panel.cu is the SB default).  One CTA
// of 256 threads per row tile of <= 2048 nonzeros, launched in tile order.
//
// Why this shape (measured on B200): row-ordered x gathers
// cost one L1TEX wavefront per nonzero (~1 line per SM clock), so the kernel
// keeps as many independent gathers in flight as it can: 6 CTAs x 256
// threads per SM, 2 quads of (col, val) per thread, all loads and gathers
// issued without branches, one __syncthreads per tile.  The hardware block
// scheduler issues tiles in order, so all SMs sweep the rows together and the
// live x footprint is one SB block's x(C_k) + x(C_B) (Eq.(1)) --
// L2-resident, the paper's "fits into the cache" condition with the
// 126 MB L2 as the cache.
//
// Per tile:
//   1. each thread loads 128-bit quads of the tile's col/val (positions from
//      the 16-byte aligned a & ~3; quads past the tile end clamped to a valid
//      one), L1 no-allocate + L2 evict-first (the matrix is read once,
//      P:L47); gathers x[col] L1-allocating + L2 evict-last (x is the
//      reused operand); masks the products outside the tile and
//      stages them in shared memory; the tile's row pointers alongside;
//   2. tiles whose rows all have <= 32 nonzeros: vector-per-row, V lanes per
//      row (V = 1..32 chosen per tile at plan time; V = 1 is the paper's
//      serial per-row temporary); lane j sums positions j, j+V, ...
//      of its row, then a fixed xor-shuffle tree; other tiles: thread-per-row
//      for rows <= 32, warp-per-row (fixed lane assignment and tree) for
//      longer rows;
//   3. y is stored coalesced; max |y| is folded per warp (one atomicMax).
// f3 (C16): with 16-bit tile-local column ids the stream is 10 B per nonzero
// (an 8-byte quad of ids + two 16-byte value pairs per four nonzeros).
// Rows longer than a tile get a tile of their own (CTA-per-row class): all
// threads stream the row with a fixed assignment and a fixed tree.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace spmvb {
namespace {

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
// f3: four 16-bit tile-local column ids (8 bytes), decoded with the tile's
// two windows: u + (u < split ? lo : hi), capped at the tile's largest column
// (the quads at a tile's ends also hold a neighbour tile's ids, whose
// products are masked; the cap keeps their gathers inside x)
__device__ __forceinline__ int4 ld_v4c16(const uint16_t* ptr, uint64_t pol, const int4 tb) {
    unsigned short u0, u1, u2, u3;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u16 {%0,%1,%2,%3}, [%4], %5;"
                 : "=h"(u0), "=h"(u1), "=h"(u2), "=h"(u3)
                 : "l"(ptr), "l"(pol));
    auto dec = [&](int u) { return min(u + (u < tb.z ? tb.x : tb.y), tb.w); };
    return make_int4(dec(u0), dec(u1), dec(u2), dec(u3));
}
__device__ __forceinline__ double2 ld_v2d(const double* ptr, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(ptr), "l"(pol));
    return r;
}

// fixed gather flavour of the default path (no run-time switch, no branch):
// L1-allocating -- the tiles an SM runs back to back belong to one SB block,
// whose x(C_k) + x(C_B) (C2: 175 KB) largely stays in L1 between them (C2
// 34.8 -> 31.8 us with L2 flushed, the C4 row-tile fallback 0.250 -> 0.228 ms;
// L1 no-allocate before) -- and L2 evict-last (x is the reused operand)
template <bool XSPLIT>
__device__ __forceinline__ double ldx2(const RowTileArgs& A, int c) {
    uint64_t pl;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
    const double* p = A.x_lo + c;
    if (XSPLIT) p = c < A.x_split ? A.x_lo + c : A.x_hi + (c - A.x_split);
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pl));
    return v;
}

constexpr int NT = 256;                  // threads per tile CTA
constexpr int kNT = NT;
struct RTSmem {
    double prod[kTileNnz];          // product of position p (nonzero a4 + p)
    int32_t so[kTileRows + 1];      // row_ptr[r0 + j] - a4
    int32_t longrows[kTileRows];    // general tiles: rows with > 32 nonzeros
    int32_t nlong;
    double red[NT / 32];
};

// NT threads per tile CTA; each thread streams QPT = 512/NT quads.
// C16: the column ids are the f3 16-bit tile-local ids (col16 + tile_base).
template <bool XSPLIT, bool C16>
__global__ void __launch_bounds__(NT, 6) spmv_rowtile_kernel(const RowTileArgs A) {
    constexpr int QPT = 512 / NT;
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
    const int4 tb = C16 ? A.tile_base[t] : make_int4(0, 0, 0, 0);
    auto cols4 = [&](int64_t pos) { return C16 ? ld_v4c16(A.col16 + pos, pol, tb) : ld_v4(A.col + pos, pol); };

    if (b - a + 3 > kTileNnz) {   // long row: planned as one (host plan_tiles, alignment-free test)
        // ------------------------------------------- one long row (> a tile)
        const int64_t qa = a >> 2, qb = ((int64_t)b + 3) >> 2;
        double acc = 0.0;
        for (int64_t q = qa + tid; q < qb; q += NT) {
            // all four gathers unconditional (the quad's columns are valid), products masked
            const int4 c = cols4(4 * q);
            const double2 v0 = ld_v2d(A.val + 4 * q, pol);
            const double2 v1 = ld_v2d(A.val + 4 * q + 2, pol);
            const double x0 = ldx2<XSPLIT>(A, c.x), x1 = ldx2<XSPLIT>(A, c.y);
            const double x2 = ldx2<XSPLIT>(A, c.z), x3 = ldx2<XSPLIT>(A, c.w);
            const int64_t g = 4 * q;
            acc += (g + 0 >= a && g + 0 < b) ? v0.x * x0 : 0.0;
            acc += (g + 1 >= a && g + 1 < b) ? v0.y * x1 : 0.0;
            acc += (g + 2 >= a && g + 2 < b) ? v1.x * x2 : 0.0;
            acc += (g + 3 >= a && g + 3 < b) ? v1.y * x3 : 0.0;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if ((tid & 31) == 0) sm.red[tid >> 5] = acc;
        __syncthreads();
        if (tid == 0) {
            double tot = 0.0;
            for (int w = 0; w < NT / 32; ++w) tot += sm.red[w];
            A.y[r0] = tot;
            if (A.maxabs_slots && tot != 0.0)
                atomicMax(A.maxabs_slots + (t & (kMaxSlots - 1)) * kSlotStride,
                          (unsigned long long)__double_as_longlong(fabs(tot)));
        }
        return;
    }

    // ------------------------------------------------ stage products, so[]
    for (int j = tid; j <= nr; j += NT) sm.so[j] = A.rowptr[r0 + j] - a4;
    if (tid == 0) sm.nlong = 0;
    {
        // Branch-free staging: every thread loads its QPT quads and gathers all
        // 4 x values unconditionally -- quads past the tile end are clamped to
        // the tile's first quad (a valid address), positions outside
        // [lo, hi) have their product masked to 0 afterwards.  (A gather
        // behind a per-lane branch made the warp wait for it at the
        // reconvergence point: measured on the panel kernel.)
        const int lo = a - a4, hi = b - a4;
        int4 c[QPT];
        double2 v0[QPT], v1[QPT];
#pragma unroll
        for (int k = 0; k < QPT; ++k) {
            const int p = 4 * (tid + k * NT);
            const int pq = (a4 + p < b) ? p : 0;
            c[k] = cols4(a4 + pq);
            v0[k] = ld_v2d(A.val + a4 + pq, pol);
            v1[k] = ld_v2d(A.val + a4 + pq + 2, pol);
        }
        double xv[QPT][4];
#pragma unroll
        for (int k = 0; k < QPT; ++k) {
            xv[k][0] = ldx2<XSPLIT>(A, c[k].x);
            xv[k][1] = ldx2<XSPLIT>(A, c[k].y);
            xv[k][2] = ldx2<XSPLIT>(A, c[k].z);
            xv[k][3] = ldx2<XSPLIT>(A, c[k].w);
        }
#pragma unroll
        for (int k = 0; k < QPT; ++k) {
            const int p = 4 * (tid + k * NT);
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

    // ------------------------------------------------------- row sums
    if (cls >= kTileShort) {
        // every row <= 32 nonzeros: V lanes per row (vector-per-row, V chosen
        // at plan time for 512 threads; halved per halving of NT, >= 1).
        int V = cls * NT / 512;
        if (V < 1) V = 1;
        for (int rb = 0; rb < nr; rb += NT / V) {
            const int r = rb + tid / V;
            const int j = tid % V;
            double acc = 0.0;
            if (r < nr) {
                const int p1 = sm.so[r + 1];
                for (int p = sm.so[r] + j; p < p1; p += V) acc += sm.prod[p];
            }
            for (int off = V >> 1; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (r < nr && j == 0) {
                A.y[r0 + r] = acc;
                mx = fmax(mx, fabs(acc));
            }
        }
    } else {
        // short rows: one thread each; long rows: listed, then one warp each
        for (int r = tid; r < nr; r += NT) {
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
        for (int k = warp; k < sm.nlong; k += NT / 32) {
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
    if (A.maxabs_slots) {   // one atomicMax per warp, no extra barrier
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if ((tid & 31) == 0 && mx > 0.0)
            atomicMax(A.maxabs_slots + ((t * (NT / 32) + (tid >> 5)) & (kMaxSlots - 1)) * kSlotStride,
                      (unsigned long long)__double_as_longlong(mx));
    }
}

}  // namespace

cudaError_t launch_rowtile(const RowTileArgs& a, bool xsplit, cudaStream_t s) {
    if (a.n_tiles <= 0) return cudaSuccess;
    const bool c16 = a.col16 != nullptr;
    if (xsplit) {
        if (c16) spmv_rowtile_kernel<true, true><<<a.n_tiles, kNT, 0, s>>>(a);
        else spmv_rowtile_kernel<true, false><<<a.n_tiles, kNT, 0, s>>>(a);
    } else {
        if (c16) spmv_rowtile_kernel<false, true><<<a.n_tiles, kNT, 0, s>>>(a);
        else spmv_rowtile_kernel<false, false><<<a.n_tiles, kNT, 0, s>>>(a);
    }
    return cudaGetLastError();
}


// Loads this file's kernels now (cudaFuncGetAttributes forces the lazy loader):
// a kernel first launched while a peer rank's kernel spins on an exchange flag
// would otherwise load its module then, and a module load can wait for the
// running kernels -- the spinning one included (see host.cpp preload_kernels).
cudaError_t preload_kernels_rowtile() {
    cudaFuncAttributes fa;
    for (const void* k : {(const void*)spmv_rowtile_kernel<false, false>, (const void*)spmv_rowtile_kernel<false, true>,
                          (const void*)spmv_rowtile_kernel<true, false>, (const void*)spmv_rowtile_kernel<true, true>}) {
        const cudaError_t e = cudaFuncGetAttributes(&fa, k);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace spmvb
