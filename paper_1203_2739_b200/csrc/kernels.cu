// kernels.cu -- sm_100a SpMxV kernels for the reordered (SB/DB) matrix and the
// fused multiple-SpMxV pass.
//
// Paper: Akbudak, Kayaaslan & Aykanat, arXiv 1203.2739 (P:Lnn = PAPER.md line).
//   * CSR SpMxV with a per-row temporary and a single y store.
//   * The reordered product y^ = A^ x^ streams A^ once; the locality
//     the reordering creates is in x: consecutive row tiles of one SB
//     block touch only x(C_k) and x(C_B) (Eq.(1)), so when every
//     CTA sweeps the tiles in order the live x footprint is one block's.
//   * Multiple-SpMxV y <- y + A^k x, k = 1..K: the fused pass
//     walks each row tile's part segments in part order and accumulates y on
//     chip ("on the fly"), writing y once.
//
// Design: one CTA per row tile of <= kTileNnz nonzeros.
//   1. stream: the tile's col/val with 128-bit loads (4 nonzeros per thread
//      step: one v4.s32 + two v2.f64), L1 no-allocate + L2 evict-first, so the
//      matrix stream does not displace x in L2;
//   2. gather x[col] (read-only path, L1-cached: x is what the reordering
//      makes reusable), multiply, stage the products in shared memory;
//   3. merge-path segmented reduction: thread t sums the products
//      [t*E, (t+1)*E) serially, splitting at row (segment) boundaries; a row
//      spanning threads is finished by its first thread adding the following
//      threads' partials in thread order -> deterministic, no fp atomics;
//   4. one coalesced store of the tile's y.
// Rows longer than kTileNnz get their own tile and a block-wide reduction.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace spmvb {

namespace {

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ int4 ld_stream_v4(const int32_t* ptr, uint64_t pol) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ double2 ld_stream_v2d(const double* ptr, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(ptr), "l"(pol));
    return r;
}

template <bool XSPLIT>
__device__ __forceinline__ double ldx(const TileArgs& a, int c) {
    if (XSPLIT) return c < a.x_split ? __ldg(a.x_lo + c) : __ldg(a.x_hi + (c - a.x_split));
    return __ldg(a.x_lo + c);
}

struct Smem {
    double prod[kTileNnz];
    double ysum[kTileRows];
    double head_val[kThreads];
    int32_t so[kTileRows + 1];
    int32_t srow[kTileRows];
    int32_t head_seg[kThreads];
    double red[kThreads / 32];
};

// Products of nonzeros [a, b) (b - a <= kTileNnz) into sm.prod[0 .. b-a).
template <bool XSPLIT>
__device__ __forceinline__ void stage_products(const TileArgs& A, Smem& sm, int a, int b, uint64_t pol) {
    constexpr int kQ = (kTileNnz / 4 + 2 + kThreads - 1) / kThreads;   // quads per thread
    const int qa = a >> 2, qb = (b + 3) >> 2;
    int4 c4[kQ];
    double2 v0[kQ], v1[kQ];
#pragma unroll
    for (int j = 0; j < kQ; ++j) {
        const int q = qa + threadIdx.x + j * kThreads;
        if (q < qb) {
            c4[j] = ld_stream_v4(A.col + 4 * (int64_t)q, pol);
            v0[j] = ld_stream_v2d(A.val + 4 * (int64_t)q, pol);
            v1[j] = ld_stream_v2d(A.val + 4 * (int64_t)q + 2, pol);
        }
    }
    double xv[kQ][4];
#pragma unroll
    for (int j = 0; j < kQ; ++j) {
        const int q = qa + threadIdx.x + j * kThreads;
        if (q < qb) {
            const int g = 4 * q;
            xv[j][0] = (g + 0 >= a && g + 0 < b) ? ldx<XSPLIT>(A, c4[j].x) : 0.0;
            xv[j][1] = (g + 1 >= a && g + 1 < b) ? ldx<XSPLIT>(A, c4[j].y) : 0.0;
            xv[j][2] = (g + 2 >= a && g + 2 < b) ? ldx<XSPLIT>(A, c4[j].z) : 0.0;
            xv[j][3] = (g + 3 >= a && g + 3 < b) ? ldx<XSPLIT>(A, c4[j].w) : 0.0;
        }
    }
#pragma unroll
    for (int j = 0; j < kQ; ++j) {
        const int q = qa + threadIdx.x + j * kThreads;
        if (q < qb) {
            const int g = 4 * q;
            if (g + 0 >= a && g + 0 < b) sm.prod[g + 0 - a] = v0[j].x * xv[j][0];
            if (g + 1 >= a && g + 1 < b) sm.prod[g + 1 - a] = v0[j].y * xv[j][1];
            if (g + 2 >= a && g + 2 < b) sm.prod[g + 2 - a] = v1[j].x * xv[j][2];
            if (g + 3 >= a && g + 3 < b) sm.prod[g + 3 - a] = v1[j].y * xv[j][3];
        }
    }
}

template <bool SPLIT>
__device__ __forceinline__ void emit(Smem& sm, int s, double v) {
    if (SPLIT) sm.ysum[sm.srow[s]] += v;   // one segment per row per part: no race
    else sm.ysum[s] = v;
}

// Merge-path segmented reduction of sm.prod[0..n) over segments
// sm.so[0..nseg] (so[0] = 0, so[nseg] = n).  Ends with __syncthreads().
template <bool SPLIT>
__device__ __forceinline__ void segmented_reduce(Smem& sm, int n, int nseg) {
    constexpr int E = kTileNnz / kThreads;
    const int tid = threadIdx.x;
    const int e0 = tid * E;
    const int e1 = min(e0 + E, n);
    bool pending = false;
    double own = 0.0;
    int own_s = -1;
    sm.head_seg[tid] = -1;
    if (e0 < n) {
        int lo = 0, hi = nseg - 1;            // last segment with so[s] <= e0
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (sm.so[mid] <= e0) lo = mid; else hi = mid - 1;
        }
        int s = lo;
        int e = e0;
        bool head = sm.so[s] < e0;
        while (true) {
            const int se = sm.so[s + 1];
            const int stop = min(se, e1);
            double acc = 0.0;
            for (; e < stop; ++e) acc += sm.prod[e];
            if (se <= e1) {
                if (head) { sm.head_val[tid] = acc; sm.head_seg[tid] = s; head = false; }
                else emit<SPLIT>(sm, s, acc);
                if (se == e1) break;
                ++s;
                while (sm.so[s + 1] == se) ++s;  // skip empty segments
            } else {
                if (head) { sm.head_val[tid] = acc; sm.head_seg[tid] = s; }
                else { pending = true; own = acc; own_s = s; }
                break;
            }
        }
    }
    __syncthreads();
    if (pending) {
        for (int u = tid + 1; u < kThreads && sm.head_seg[u] == own_s; ++u) own += sm.head_val[u];
        emit<SPLIT>(sm, own_s, own);
    }
    __syncthreads();
}

// Long segment [a, b) (> kTileNnz nonzeros, single row): per-thread partials
// over a fixed quad assignment, then a fixed-order block tree.  Returns the
// sum in thread 0.  Ends with __syncthreads().
template <bool XSPLIT>
__device__ __forceinline__ double long_segment(const TileArgs& A, Smem& sm, int64_t a, int64_t b,
                                               uint64_t pol) {
    const int64_t qa = a >> 2, qb = (b + 3) >> 2;
    double acc = 0.0;
    for (int64_t q = qa + threadIdx.x; q < qb; q += kThreads) {
        const int4 c = ld_stream_v4(A.col + 4 * q, pol);
        const double2 v0 = ld_stream_v2d(A.val + 4 * q, pol);
        const double2 v1 = ld_stream_v2d(A.val + 4 * q + 2, pol);
        const int64_t g = 4 * q;
        if (g + 0 >= a && g + 0 < b) acc += v0.x * ldx<XSPLIT>(A, c.x);
        if (g + 1 >= a && g + 1 < b) acc += v0.y * ldx<XSPLIT>(A, c.y);
        if (g + 2 >= a && g + 2 < b) acc += v1.x * ldx<XSPLIT>(A, c.z);
        if (g + 3 >= a && g + 3 < b) acc += v1.y * ldx<XSPLIT>(A, c.w);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = acc;
    __syncthreads();
    double tot = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kThreads / 32; ++w) tot += sm.red[w];
    __syncthreads();
    return tot;
}

template <bool SPLIT, bool XSPLIT>
__global__ void __launch_bounds__(kThreads) spmv_tile_kernel(const TileArgs A) {
    __shared__ Smem sm;
    const int t = blockIdx.x;
    const int tid = threadIdx.x;
    const int r0 = A.tile_row[t];
    const int nr = A.tile_row[t + 1] - r0;
    const uint64_t pol = policy_evict_first();
    if (SPLIT && A.accumulate && A.tile_seg[t * A.K + A.k_begin] == A.tile_seg[t * A.K + A.k_end])
        return;                                            // literal pass: tile has no part-k rows

    for (int k = tid; k < nr; k += kThreads) sm.ysum[k] = A.accumulate ? A.y[r0 + k] : 0.0;

    const int kb = SPLIT ? A.k_begin : 0;
    const int ke = SPLIT ? A.k_end : 1;
    for (int k = kb; k < ke; ++k) {
        int s0, s1;
        if (SPLIT) { s0 = A.tile_seg[t * A.K + k]; s1 = A.tile_seg[t * A.K + k + 1]; }
        else { s0 = r0; s1 = r0 + nr; }
        const int nseg = s1 - s0;
        if (nseg == 0) continue;                           // CTA-uniform
        const int a = A.seg_ptr[s0];
        const int b = A.seg_ptr[s1];
        const int n = b - a;
        if (n == 0) continue;
        if (n > kTileNnz) {                                // single long row
            __syncthreads();
            const double v = long_segment<XSPLIT>(A, sm, a, b, pol);
            if (tid == 0) {
                if (SPLIT) sm.ysum[A.seg_row[s0]] += v; else sm.ysum[0] = v;
            }
            __syncthreads();
            continue;
        }
        for (int j = tid; j <= nseg; j += kThreads) {
            sm.so[j] = A.seg_ptr[s0 + j] - a;
            if (SPLIT && j < nseg) sm.srow[j] = A.seg_row[s0 + j];
        }
        stage_products<XSPLIT>(A, sm, a, b, pol);
        __syncthreads();
        segmented_reduce<SPLIT>(sm, n, nseg);
    }
    __syncthreads();

    double mx = 0.0;
    for (int k = tid; k < nr; k += kThreads) {
        const double v = sm.ysum[k];
        A.y[r0 + k] = v;
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

__global__ void gather_kernel(const double* __restrict__ src, const int32_t* __restrict__ idx,
                              double* __restrict__ dst, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __ldg(src + idx[i]);
}

__global__ void maxabs_finish_kernel(const unsigned long long* __restrict__ slots, double* out) {
    unsigned long long m = 0;
    for (int i = threadIdx.x; i < kMaxSlots; i += blockDim.x) {
        const unsigned long long v = slots[i * kSlotStride];
        m = v > m ? v : m;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, m, off);
        m = o > m ? o : m;
    }
    if (threadIdx.x == 0) *out = __longlong_as_double((long long)m);
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

__global__ void normalize_scalar_kernel(const double* __restrict__ y, const int32_t* __restrict__ owner,
                                        const double* __restrict__ m, double* __restrict__ x, int64_t n) {
    const double mt = *m;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
        x[c] = __ldg(y + owner[c]) / mt;
}

int grid_for(int64_t n, int threads) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    int64_t g = (n + threads - 1) / threads;
    int64_t cap = (int64_t)sms * 8;
    if (g > cap) g = cap;
    return (int)(g > 0 ? g : 1);
}

}  // namespace

int kernel_num_sms() { return grid_for(1LL << 40, 1) / 8; }

cudaError_t launch_tiles(const TileArgs& a, bool split, bool xsplit, cudaStream_t s) {
    if (a.n_tiles <= 0) return cudaSuccess;
    dim3 grid(a.n_tiles), block(kThreads);
    if (split) {
        if (xsplit) spmv_tile_kernel<true, true><<<grid, block, 0, s>>>(a);
        else spmv_tile_kernel<true, false><<<grid, block, 0, s>>>(a);
    } else {
        if (xsplit) spmv_tile_kernel<false, true><<<grid, block, 0, s>>>(a);
        else spmv_tile_kernel<false, false><<<grid, block, 0, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_gather(const double* src, const int32_t* idx, double* dst, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    gather_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, idx, dst, n);
    return cudaGetLastError();
}

cudaError_t launch_maxabs_finish(const unsigned long long* slots, double* out, cudaStream_t s) {
    maxabs_finish_kernel<<<1, 32, 0, s>>>(slots, out);
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

}  // namespace spmvb
