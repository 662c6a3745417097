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
//      P:L47); gathers x[col] with L1 no-allocate + L2 evict-last (x is the
//      reused operand); masks the products outside the tile and
//      stages them in shared memory; the tile's row pointers alongside;
//   2. tiles whose rows all have <= 32 nonzeros: vector-per-row, V lanes per
//      row (V = 1..32 chosen per tile at plan time; V = 1 is the paper's
//      serial per-row temporary); lane j sums positions j, j+V, ...
//      of its row, then a fixed xor-shuffle tree; other tiles: thread-per-row
//      for rows <= 32, warp-per-row (fixed lane assignment and tree) for
//      longer rows;
//   3. y is stored coalesced; max |y| is folded per warp (one atomicMax).
// Rows longer than a tile get a tile of their own (CTA-per-row class): all
// threads stream the row with a fixed assignment and a fixed tree.
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

__device__ __forceinline__ double gx(const double* p, int gmode, uint64_t pl) {
    double v;
    if (gmode == 1) {
        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pl));
    } else if (gmode == 2) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pl));
    } else {
        v = __ldg(p);
    }
    return v;
}

template <bool XSPLIT>
__device__ __forceinline__ double ldx(const RowTileArgs& A, int c) {
    uint64_t pl = 0;
    if (A.gmode) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
    if (XSPLIT) return c < A.x_split ? gx(A.x_lo + c, A.gmode, pl) : gx(A.x_hi + (c - A.x_split), A.gmode, pl);
    return gx(A.x_lo + c, A.gmode, pl);
}



// fixed gather flavour of the default path (no run-time switch, no branch):
// L1 no-allocate (a gathered line is not reused inside a tile) and L2
// evict-last (x is the reused operand)
template <bool XSPLIT>
__device__ __forceinline__ double ldx2(const RowTileArgs& A, int c) {
    uint64_t pl;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
    const double* p = A.x_lo + c;
    if (XSPLIT) p = c < A.x_split ? A.x_lo + c : A.x_hi + (c - A.x_split);
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pl));
    return v;
}

template <int NT>
struct RTSmemT {
    double prod[kTileNnz];          // product of position p (nonzero a4 + p)
    int32_t so[kTileRows + 1];      // row_ptr[r0 + j] - a4
    int32_t longrows[kTileRows];    // general tiles: rows with > 32 nonzeros
    int32_t nlong;
    double red[NT / 32];
};

__device__ __forceinline__ int32_t ld_s32(const int32_t* ptr, uint64_t pol) {
    int32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_f64(const double* ptr, uint64_t pol) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(ptr), "l"(pol));
    return r;
}

// NT threads per tile CTA; each thread streams QPT = 512/NT quads.
// LIN: lane-consecutive positions instead of quads (thread t takes positions
// t, t+NT, ...): the same coalesced stream, but the 32 gathers of one warp
// instruction are for 32 consecutive nonzeros, so sorted columns of a long
// row share 128-byte lines (C4's banded rows).
template <bool XSPLIT, int NT, bool LIN>
__global__ void __launch_bounds__(NT, (NT == 512 ? 3 : NT == 256 ? 6 : 8)) spmv_rowtile_kernel(const RowTileArgs A) {
    constexpr int QPT = 512 / NT;
    __shared__ __align__(16) RTSmemT<NT> sm;
    const int t = blockIdx.x;
    const int tid = threadIdx.x;
    const int r0 = A.tile_row[t], r1 = A.tile_row[t + 1];
    const int a = A.tile_nnz[t], b = A.tile_nnz[t + 1];
    const int cls = A.tile_cls[t];
    const int nr = r1 - r0;
    const int a4 = a & ~3;
    const uint64_t pol = pol_evict_first();
    double mx = 0.0;

    if (b - a + 3 > kTileNnz) {   // long row: planned as one (host plan_tiles, alignment-free test)
        // ------------------------------------------- one long row (> a tile)
        if (A.long_tiles) return;                   // done by spmv_longrow_kernel
        const int64_t qa = a >> 2, qb = ((int64_t)b + 3) >> 2;
        double acc = 0.0;
        if (LIN) {
            for (int64_t e = a + tid; e < b; e += 4 * NT) {
                double v[4], xv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t f = e + u * NT;
                    v[u] = 0.0;
                    if (f < b) {
                        v[u] = ld_f64(A.val + f, pol);
                        xv[u] = ldx<XSPLIT>(A, ld_s32(A.col + f, pol));
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (e + u * NT < b) acc += v[u] * xv[u];
            }
        }
        for (int64_t q = qa + tid; !LIN && q < qb; q += NT) {
            // all four gathers unconditional (the quad's columns are valid), products masked
            const int4 c = ld_v4(A.col + 4 * q, pol);
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
    if (LIN) {
        const int lo = a - a4, hi = b - a4;
        constexpr int PPT = kTileNnz / NT;   // positions per thread
        int32_t c[PPT];
        double v[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const int p = tid + k * NT;
            if (p >= lo && p < hi) {
                c[k] = ld_s32(A.col + a4 + p, pol);
                v[k] = ld_f64(A.val + a4 + p, pol);
            }
        }
        double xv[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const int p = tid + k * NT;
            if (p >= lo && p < hi) xv[k] = ldx<XSPLIT>(A, c[k]);
        }
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const int p = tid + k * NT;
            if (p >= lo && p < hi) sm.prod[p] = v[k] * xv[k];
        }
    } else {
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
            c[k] = ld_v4(A.col + a4 + pq, pol);
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

// ---------------------------------------------------------------------------
// spmv_rowseg_kernel: same tile geometry and streaming as above, but the
// products never touch shared memory (the L1TEX pipe is shared by the x
// gathers and shared-memory wavefronts; ncu: 69 % busy on C5 with staging).
// Thread q keeps the products of positions 4q..4q+3 in registers and walks
// them against the tile's row offsets: rows that start and end inside its
// quad are stored at once; a row running across threads is completed with a
// segmented inclusive scan over the threads (warp shuffles, then one carry
// per warp through shared memory), in a fixed order -- deterministic.
// ---------------------------------------------------------------------------
struct SegSmem {
    int32_t so[kTileRows + 1];
    double wv[kRT / 32];            // per warp: scan value at lane 31
    int32_t wf[kRT / 32];           // per warp: a chain reset happened in the warp
    int32_t wh[kRT / 32];           // per warp: lane 31 carries a row into the next warp
    double red[kRT / 32];
};

template <bool XSPLIT>
__global__ void __launch_bounds__(kRT, 3) spmv_rowseg_kernel(const RowTileArgs A) {
    __shared__ __align__(16) SegSmem sm;
    const int t = blockIdx.x;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int r0 = A.tile_row[t], r1 = A.tile_row[t + 1];
    const int a = A.tile_nnz[t], b = A.tile_nnz[t + 1];
    const int nr = r1 - r0;
    const int a4 = a & ~3;
    const uint64_t pol = pol_evict_first();
    double mx = 0.0;

    if (b - a + 3 > kTileNnz) {   // long row: planned as one (host plan_tiles, alignment-free test)
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
        if (lane == 0) sm.red[warp] = acc;
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

    // -------------------------------------------- stream, gather, products
    for (int j = tid; j <= nr; j += kRT) sm.so[j] = A.rowptr[r0 + j] - a4;
    const int pq = 4 * tid;
    const int lo = a - a4, hi = b - a4;
    const int e_lo = max(pq, lo), e_hi = min(pq + 4, hi);
    const bool act = e_lo < e_hi;
    double pv[4] = {0.0, 0.0, 0.0, 0.0};
    if (a4 + pq < b) {
        const int4 c = ld_v4(A.col + a4 + pq, pol);
        const double2 v0 = ld_v2d(A.val + a4 + pq, pol);
        const double2 v1 = ld_v2d(A.val + a4 + pq + 2, pol);
        const double x0 = (pq + 0 >= lo && pq + 0 < hi) ? ldx<XSPLIT>(A, c.x) : 0.0;
        const double x1 = (pq + 1 >= lo && pq + 1 < hi) ? ldx<XSPLIT>(A, c.y) : 0.0;
        const double x2 = (pq + 2 >= lo && pq + 2 < hi) ? ldx<XSPLIT>(A, c.z) : 0.0;
        const double x3 = (pq + 3 >= lo && pq + 3 < hi) ? ldx<XSPLIT>(A, c.w) : 0.0;
        pv[0] = v0.x * x0; pv[1] = v0.y * x1; pv[2] = v1.x * x2; pv[3] = v1.y * x3;
    }
    __syncthreads();                                     // so[] staged

    for (int r = tid; r < nr; r += kRT)                  // empty rows: y = +0 (A5)
        if (sm.so[r] == sm.so[r + 1]) A.y[r0 + r] = 0.0;

    // ------------------------------------------------ walk the quad
    double v = 0.0;          // scan input: chain value leaving this thread
    bool f = true;           // chain reset at this thread
    bool carry = false;      // this thread's last row continues in the next thread
    int head_row = -1;
    double head_sum = 0.0;
    bool head_ends = false;
    if (act) {
        int lo_r = 0, hi_r = nr - 1;                     // last row with so(r) <= e_lo
        while (lo_r < hi_r) {
            const int mid = (lo_r + hi_r + 1) >> 1;
            if (sm.so[mid] <= e_lo) lo_r = mid; else hi_r = mid - 1;
        }
        int row = lo_r;
        int end = sm.so[row + 1];
        head_row = row;
        bool in_head = true;
        double cur = 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int p = pq + u;
            if (p >= e_lo && p < e_hi) {
                while (p >= end) {
                    if (in_head) { head_sum = cur; head_ends = true; in_head = false; }
                    else { A.y[r0 + row] = cur; mx = fmax(mx, fabs(cur)); }   // row inside the quad
                    cur = 0.0;
                    ++row;
                    end = sm.so[row + 1];
                }
                cur += pv[u];
            }
        }
        if (in_head) {                                   // one row covers the whole quad
            head_sum = cur;
            if (end <= e_hi) head_ends = true;           // ... and ends here
            else { f = false; carry = true; v = cur; }   // ... and runs on: pass the chain
        } else if (end <= e_hi) {                        // last row also ends here
            A.y[r0 + row] = cur;
            mx = fmax(mx, fabs(cur));
        } else {                                         // last row runs on: start a chain
            carry = true;
            v = cur;
        }
    }

    // -------------------------- segmented inclusive scan of chain values
    double S = v;
    bool F = f;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double Su = __shfl_up_sync(0xffffffffu, S, d);
        const bool Fu = __shfl_up_sync(0xffffffffu, F ? 1 : 0, d) != 0;
        if (lane >= d) {
            if (!F) S = Su + S;
            F = F || Fu;
        }
    }
    if (lane == 31) {
        sm.wv[warp] = S;
        sm.wf[warp] = F ? 1 : 0;
        sm.wh[warp] = carry ? 1 : 0;
    }
    __syncthreads();
    // carry into this warp's lane 0: out_k = wf[k] ? wv[k] : c + wv[k],
    // c = wh[k] ? out_k : 0, over earlier warps in order (fixed order)
    double cin = 0.0;
    for (int k = 0; k < warp; ++k) {
        const double out = sm.wf[k] ? sm.wv[k] : cin + sm.wv[k];
        cin = sm.wh[k] ? out : 0.0;
    }
    const double Sfull = F ? S : cin + S;
    const double Sprev = __shfl_up_sync(0xffffffffu, Sfull, 1);
    const bool cprev = __shfl_up_sync(0xffffffffu, carry ? 1 : 0, 1) != 0;
    const double carry_in = (lane == 0) ? cin : (cprev ? Sprev : 0.0);
    if (act && head_ends) {
        const double tot = carry_in + head_sum;
        A.y[r0 + head_row] = tot;
        mx = fmax(mx, fabs(tot));
    }
    if (A.maxabs_slots) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if (lane == 0 && mx > 0.0)
            atomicMax(A.maxabs_slots + ((t * (kRT / 32) + warp) & (kMaxSlots - 1)) * kSlotStride,
                      (unsigned long long)__double_as_longlong(mx));
    }
}

// ---------------------------------------------------------------------------
// spmv_longrow_kernel: rows longer than a tile (CTA-per-row class), one CTA
// each, launched over the list of long tiles.  Each thread keeps LQ quads of
// the row in flight (all stream loads, then all gathers), which the tile
// kernel's register budget (6 CTAs/SM) cannot afford; fixed assignment and
// fixed block tree (deterministic).
template <bool XSPLIT>
__global__ void __launch_bounds__(256, 2) spmv_longrow_kernel(const RowTileArgs A) {
    constexpr int NT = 256, LQ = 4;
    __shared__ double red[NT / 32];
    const int t = A.long_tiles[blockIdx.x];
    const int tid = threadIdx.x;
    const int r0 = A.tile_row[t];
    const int a = A.tile_nnz[t], b = A.tile_nnz[t + 1];
    const uint64_t pol = pol_evict_first();
    const int64_t qa = a >> 2, qb = ((int64_t)b + 3) >> 2;
    double acc = 0.0;
    for (int64_t q0 = qa + tid; q0 < qb; q0 += (int64_t)LQ * NT) {
        int4 c[LQ];
        double2 v0[LQ], v1[LQ];
#pragma unroll
        for (int u = 0; u < LQ; ++u) {
            const int64_t q = q0 + (int64_t)u * NT;
            if (q < qb) {
                c[u] = ld_v4(A.col + 4 * q, pol);
                v0[u] = ld_v2d(A.val + 4 * q, pol);
                v1[u] = ld_v2d(A.val + 4 * q + 2, pol);
            }
        }
        double xv[LQ][4];
#pragma unroll
        for (int u = 0; u < LQ; ++u) {
            const int64_t g = 4 * (q0 + (int64_t)u * NT);
            if (q0 + (int64_t)u * NT < qb) {
                (void)g;
                xv[u][0] = ldx2<XSPLIT>(A, c[u].x);
                xv[u][1] = ldx2<XSPLIT>(A, c[u].y);
                xv[u][2] = ldx2<XSPLIT>(A, c[u].z);
                xv[u][3] = ldx2<XSPLIT>(A, c[u].w);
            }
        }
#pragma unroll
        for (int u = 0; u < LQ; ++u) {
            const int64_t g = 4 * (q0 + (int64_t)u * NT);
            if (q0 + (int64_t)u * NT < qb) {
                if (g + 0 >= a && g + 0 < b) acc += v0[u].x * xv[u][0];
                if (g + 1 >= a && g + 1 < b) acc += v0[u].y * xv[u][1];
                if (g + 2 >= a && g + 2 < b) acc += v1[u].x * xv[u][2];
                if (g + 3 >= a && g + 3 < b) acc += v1[u].y * xv[u][3];
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
        double tot = 0.0;
        for (int w = 0; w < NT / 32; ++w) tot += red[w];
        A.y[r0] = tot;
        if (A.maxabs_slots && tot != 0.0)
            atomicMax(A.maxabs_slots + (t & (kMaxSlots - 1)) * kSlotStride,
                      (unsigned long long)__double_as_longlong(fabs(tot)));
    }
}

}  // namespace

cudaError_t launch_longrows(const RowTileArgs& a, int32_t n_long, bool xsplit, cudaStream_t s) {
    if (n_long <= 0 || !a.long_tiles) return cudaSuccess;
    if (xsplit) spmv_longrow_kernel<true><<<n_long, 256, 0, s>>>(a);
    else spmv_longrow_kernel<false><<<n_long, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_rowtile(const RowTileArgs& a, bool xsplit, int nt, cudaStream_t s, bool lin) {
    if (a.n_tiles <= 0) return cudaSuccess;
    if (lin) {
        if (xsplit) spmv_rowtile_kernel<true, 256, true><<<a.n_tiles, 256, 0, s>>>(a);
        else spmv_rowtile_kernel<false, 256, true><<<a.n_tiles, 256, 0, s>>>(a);
    } else if (nt == 256) {
        if (xsplit) spmv_rowtile_kernel<true, 256, false><<<a.n_tiles, 256, 0, s>>>(a);
        else spmv_rowtile_kernel<false, 256, false><<<a.n_tiles, 256, 0, s>>>(a);
    } else if (nt == 128) {
        if (xsplit) spmv_rowtile_kernel<true, 128, false><<<a.n_tiles, 128, 0, s>>>(a);
        else spmv_rowtile_kernel<false, 128, false><<<a.n_tiles, 128, 0, s>>>(a);
    } else {
        if (xsplit) spmv_rowtile_kernel<true, 512, false><<<a.n_tiles, 512, 0, s>>>(a);
        else spmv_rowtile_kernel<false, 512, false><<<a.n_tiles, 512, 0, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_rowseg(const RowTileArgs& a, bool xsplit, cudaStream_t s) {
    if (a.n_tiles <= 0) return cudaSuccess;
    if (xsplit) spmv_rowseg_kernel<true><<<a.n_tiles, kRT, 0, s>>>(a);
    else spmv_rowseg_kernel<false><<<a.n_tiles, kRT, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace spmvb
