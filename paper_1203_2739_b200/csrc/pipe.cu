// pipe.cu -- the single-SpMxV kernel y^ = A^ x^ (per-row temporary and
// one y store), persistent and warp-specialised for sm_100a.
//
//   * grid = 2 CTAs per SM; the producer warps claim row tiles in order from a
//     global counter (4 at a time), so all CTAs sweep the tiles together and
//     the live x footprint is one SB block's x(C_k) plus x(C_B) (Eq.(1),
//     P:L65-79) -- the paper's "fits into the cache" condition with
//     the 126 MB L2 as the cache;
//   * a producer warp streams each tile's col/val/row-pointer slices into a
//     3-stage shared-memory ring with 1-D bulk async copies (TMA engine,
//     `cp.async.bulk`, SASS UBLKCP) that complete on mbarriers; the matrix is
//     read exactly once with an L2 evict-first policy (no temporal
//     locality in the matrix), leaving the LSU pipe to the x gathers;
//   * 8 consumer warps: thread t takes tile positions t + 256u (conflict-free
//     shared loads), gathers x[col] through the read-only path and stages the
//     products in a swizzled shared buffer; tiles whose rows all have <= 32
//     nonzeros (the common case: 12..23) are reduced one
//     thread per row in CSR order (the paper's per-row temporary), others by a
//     deterministic merge-path segmented sum (a row's sum = its first
//     thread's serial partial, then the later threads' partials in order);
//   * the gathers of tile i+1 are issued before tile i is reduced, so the x
//     gathers -- the binding limit, ~1 lane-request per clock per SM on B200
//     (scripts/gather_modes.py) -- stay in flight across the reduction;
//   * y is stored once per row, coalesced; max |y| for the power iteration is
//     folded per warp, one atomicMax per warp per launch.
// Rows longer than a tile take a direct-load path in the same kernel.
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace spmvb {
namespace {

constexpr int kStages = 3;
constexpr int kCons = kThreads;              // consumer threads (8 warps)
constexpr int kPipeThreads = kCons + 32;     // + one producer warp
constexpr int kE = kTileNnz / kCons;         // positions per consumer thread (8)
constexpr int kSoElems = kTileRows + 4;      // rows+1, <= 3 in front
constexpr int kClaim = 4;                    // tiles claimed per atomic

struct __align__(16) StageHdr {
    int32_t r0, r1, a, b;      // rows [r0, r1), nonzeros [a, b); r0 < 0: end of work
    int32_t cls, pad0, pad1, pad2;   // tile class (internal.h kTileShort / kTileGeneral)
};

struct __align__(16) PipeSmem {
    double val[kStages][kTileNnz];           // positions [0, kTileNnz) from a & ~3
    int32_t col[kStages][kTileNnz];
    int32_t so[kStages][kSoElems];
    StageHdr hdr[kStages];
    double prod[kTileNnz];                   // products, swizzled (swz)
    int32_t so_priv[2][kSoElems];            // consumers' copy of a tile's row pointers
    double ysum[2][kTileRows];
    double head_val[kCons];
    int32_t head_seg[kCons];
    double red[kCons / 32];
    uint64_t full[kStages];
    uint64_t empty[kStages];
};
static_assert(sizeof(int32_t) * kSoElems % 16 == 0, "stage alignment");
static_assert(kE == 8, "consumer layout assumes 8 positions per thread");

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(b)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory"); }

__device__ __forceinline__ uint64_t policy(bool first) {
    uint64_t p;
    if (first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

template <bool XSPLIT>
__device__ __forceinline__ double ldx(const PipeArgs& A, int c) {
    if (XSPLIT) return c < A.x_split ? __ldg(A.x_lo + c) : __ldg(A.x_hi + (c - A.x_split));
    return __ldg(A.x_lo + c);
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

// bank-conflict-free product slot: thread t writes slots t + 256u (products)
// and merge-path thread t reads 8t..8t+7; XOR of bits 4..6 into bits 0..2.
__device__ __forceinline__ int swz(int p) { return p ^ ((p >> 4) & 7); }

// One consumer thread's share of a tile: positions p = tid + 256u of the
// stage buffers (position p holds nonzero a4 + p), values and gathered x.
struct Slice {
    StageHdr h;
    int st;
    bool big;            // long row: direct-load path
    double v[kE];
    double x[kE];
};

// Waits for stage it % kStages, takes this thread's col/val share into
// registers, issues its x gathers, copies the row pointers into so_priv[it&1]
// and releases the stage at once (one arrive per warp), so the producer can
// run a full ring ahead of the consumers.
template <bool XSPLIT>
__device__ __forceinline__ void fetch(const PipeArgs& A, PipeSmem& sm, int it, Slice& S) {
    const int tid = threadIdx.x;
    S.st = it % kStages;
    mbar_wait(&sm.full[S.st], (uint32_t)(it / kStages) & 1);
    S.h = sm.hdr[S.st];
    S.big = false;
    if (S.h.r0 < 0) return;                     // sentinel: no more tiles (stage never released)
    const int off = S.h.a & 3;
    const int n = S.h.b - S.h.a;
    S.big = n + 3 > kTileNnz;   // plan_tiles' alignment-free test (off <= 3)
    int c[kE];
    if (!S.big) {
#pragma unroll
        for (int u = 0; u < kE; ++u) {
            const int p = tid + u * kCons;
            c[u] = sm.col[S.st][p];
            S.v[u] = sm.val[S.st][p];
        }
        const int nso = S.h.r1 - S.h.r0 + 1;
        const int32_t* src = sm.so[S.st] + (S.h.r0 & 3);
        for (int j = tid; j < nso; j += kCons) sm.so_priv[it & 1][j] = src[j];
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&sm.empty[S.st]);
    if (S.big) return;
    const int lo = off, hi = off + n;
#pragma unroll
    for (int u = 0; u < kE; ++u) {
        const int p = tid + u * kCons;
        S.x[u] = (p >= lo && p < hi) ? ldx<XSPLIT>(A, c[u]) : 0.0;
    }
}

template <bool XSPLIT>
__global__ void __launch_bounds__(kPipeThreads, 2) spmv_pipe_kernel(const PipeArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PipeSmem& sm = *reinterpret_cast<PipeSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const int T = A.n_tiles;

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], kCons / 32);   // one arrive per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (tid >= kCons) {
        // ------------------------------------------------------- producer warp
        // Tiles are claimed in order from a global counter, kClaim at a time,
        // so all CTAs stay inside a narrow band of rows: the live x window is
        // one SB block (plus C_B), which stays L2-resident.  A statically
        // strided persistent schedule lets CTAs drift apart and the x window
        // overflows L2 (measured on C5: 4.7x the algorithmic DRAM bytes).
        const int lane = tid & 31;
        const uint64_t pol_first = policy(true);
        const uint64_t pol_norm = policy(false);
        int it = 0;
        int batch = 0;
        if (lane == 0) batch = atomicAdd(A.tile_counter, kClaim);
        batch = __shfl_sync(0xffffffffu, batch, 0);
        while (batch < T) {
            const int tj = batch + lane;
            int m_r0 = 0, m_r1 = 0, m_a = 0, m_b = 0, m_c = 0;
            if (lane < kClaim && tj < T) {
                m_r0 = A.tile_row[tj];
                m_r1 = A.tile_row[tj + 1];
                m_a = A.tile_nnz[tj];
                m_b = A.tile_nnz[tj + 1];
                m_c = A.tile_cls[tj];
            }
            int next = 0;
            if (lane == 0) next = atomicAdd(A.tile_counter, kClaim);   // claim ahead: latency overlaps
            next = __shfl_sync(0xffffffffu, next, 0);
            const int cnt = min(kClaim, T - batch);
            for (int j = 0; j < cnt; ++j, ++it) {
                const int r0 = __shfl_sync(0xffffffffu, m_r0, j);
                const int r1 = __shfl_sync(0xffffffffu, m_r1, j);
                const int a = __shfl_sync(0xffffffffu, m_a, j);
                const int b = __shfl_sync(0xffffffffu, m_b, j);
                const int cls = __shfl_sync(0xffffffffu, m_c, j);
                const int st = it % kStages;
                const uint32_t k = (uint32_t)(it / kStages);
                if (lane == 0) {
                    if (k > 0) mbar_wait(&sm.empty[st], (k - 1) & 1);
                    sm.hdr[st] = StageHdr{r0, r1, a, b, cls, 0, 0, 0};
                    const int a4 = a & ~3;
                    if (b - a + 3 > kTileNnz) {   // long row (plan_tiles' alignment-free test)
                        mbar_arrive(&sm.full[st]);           // long row: consumers load directly
                    } else {
                        const int r4 = r0 & ~3;
                        const uint32_t cb = (uint32_t)(((b - a4) * 4 + 15) & ~15);
                        const uint32_t vb = (uint32_t)((b - a4) * 8 + 15) & ~15u;
                        const uint32_t sb = (uint32_t)(((r1 + 1 - r4) * 4 + 15) & ~15);
                        mbar_arrive_tx(&sm.full[st], cb + vb + sb);
                        if (cb) {
                            bulk_g2s(sm.col[st], A.col + a4, cb, &sm.full[st], pol_first);
                            bulk_g2s(sm.val[st], A.val + a4, vb, &sm.full[st], pol_first);
                        }
                        bulk_g2s(sm.so[st], A.rowptr + r4, sb, &sm.full[st], pol_norm);
                    }
                }
                __syncwarp();
            }
            batch = next;
        }
        // end-of-work sentinel
        if (lane == 0) {
            const int st = it % kStages;
            const uint32_t k = (uint32_t)(it / kStages);
            if (k > 0) mbar_wait(&sm.empty[st], (k - 1) & 1);
            sm.hdr[st] = StageHdr{-1, -1, 0, 0, 0, 0, 0, 0};
            mbar_arrive(&sm.full[st]);
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    const uint64_t pol_first = policy(true);
    double mx = 0.0;
    int it = 0;
    Slice cur, nxt;
    fetch<XSPLIT>(A, sm, 0, cur);
    for (; cur.h.r0 >= 0; ++it) {
        fetch<XSPLIT>(A, sm, it + 1, nxt);                // next tile's gathers in flight
        const StageHdr h = cur.h;
        const int nr = h.r1 - h.r0;
        double* ysum = sm.ysum[it & 1];

        if (cur.big) {
            // single long row: direct 128-bit loads, fixed assignment, fixed tree
            const int64_t qa = h.a >> 2, qb = ((int64_t)h.b + 3) >> 2;
            double acc = 0.0;
            for (int64_t q = qa + tid; q < qb; q += kCons) {
                const int4 c = ld_stream_v4(A.col + 4 * q, pol_first);
                const double2 v0 = ld_stream_v2d(A.val + 4 * q, pol_first);
                const double2 v1 = ld_stream_v2d(A.val + 4 * q + 2, pol_first);
                const int64_t g = 4 * q;
                if (g + 0 >= h.a && g + 0 < h.b) acc += v0.x * ldx<XSPLIT>(A, c.x);
                if (g + 1 >= h.a && g + 1 < h.b) acc += v0.y * ldx<XSPLIT>(A, c.y);
                if (g + 2 >= h.a && g + 2 < h.b) acc += v1.x * ldx<XSPLIT>(A, c.z);
                if (g + 3 >= h.a && g + 3 < h.b) acc += v1.y * ldx<XSPLIT>(A, c.w);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if ((tid & 31) == 0) sm.red[tid >> 5] = acc;
            cons_sync();
            if (tid == 0) {
                double tot = 0.0;
                for (int w = 0; w < kCons / 32; ++w) tot += sm.red[w];
                A.y[h.r0] = tot;
                mx = fmax(mx, fabs(tot));
            }
            cons_sync();
        } else {
            const int off = h.a & 3;
            const int n = h.b - h.a;
            const int a4 = h.a & ~3;
            // so(j) = row_ptr[r0 + j] - a4: row j occupies positions [so(j), so(j+1))
            const int32_t* so = sm.so_priv[it & 1];
#pragma unroll
            for (int u = 0; u < kE; ++u) {
                const int p = tid + u * kCons;
                if (p >= off && p < off + n) sm.prod[swz(p)] = cur.v[u] * cur.x[u];
            }
            if (h.cls >= kTileShort) {
                // rows of <= 32 nonzeros: one thread per row, serial sum in CSR
                // order (the paper's per-row temporary), one y store
                cons_sync();
                for (int r = tid; r < nr; r += kCons) {
                    const int p1 = so[r + 1] - a4;
                    double acc = 0.0;
                    for (int p = so[r] - a4; p < p1; ++p) acc += sm.prod[swz(p)];
                    A.y[h.r0 + r] = acc;
                    mx = fmax(mx, fabs(acc));
                }
                cons_sync();
            } else {
                // general tile: merge-path segmented reduction
                for (int j = tid; j < nr; j += kCons) ysum[j] = 0.0;
                sm.head_seg[tid] = -1;
                cons_sync();    // products staged, ysum zeroed, head_seg reset
                const int e_lo = max(tid * kE, off);
                const int e_hi = min(tid * kE + kE, off + n);
                bool pending = false;
                double own = 0.0;
                int own_s = -1;
                if (e_lo < e_hi) {
                    int lo = 0, hi = nr - 1;              // last row with so(s) <= e_lo
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (so[mid] - a4 <= e_lo) lo = mid; else hi = mid - 1;
                    }
                    int s = lo;
                    int nb = so[s + 1] - a4;              // end of row s
                    bool head = so[s] - a4 < e_lo;        // row began in an earlier thread
                    double acc = 0.0;
                    for (int p = e_lo; p < e_hi; ++p) {
                        while (p >= nb) {                 // close row s (and skip empty rows)
                            if (head) { sm.head_val[tid] = acc; sm.head_seg[tid] = s; head = false; }
                            else if (so[s] - a4 < nb) ysum[s] = acc;
                            acc = 0.0;
                            ++s;
                            nb = so[s + 1] - a4;
                        }
                        acc += sm.prod[swz(p)];
                    }
                    if (nb <= e_hi) {                     // row s ends exactly at e_hi
                        if (head) { sm.head_val[tid] = acc; sm.head_seg[tid] = s; }
                        else ysum[s] = acc;
                    } else {                              // row s continues in later threads
                        if (head) { sm.head_val[tid] = acc; sm.head_seg[tid] = s; }
                        else { pending = true; own = acc; own_s = s; }
                    }
                }
                cons_sync();
                if (pending) {
                    for (int u = tid + 1; u < kCons && sm.head_seg[u] == own_s; ++u) own += sm.head_val[u];
                    ysum[own_s] = own;
                }
                cons_sync();
                for (int j = tid; j < nr; j += kCons) {
                    const double v = ysum[j];
                    A.y[h.r0 + j] = v;
                    mx = fmax(mx, fabs(v));
                }
            }
        }
        cur = nxt;
    }
    if (A.maxabs_slots) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if ((tid & 31) == 0 && mx > 0.0)
            atomicMax(A.maxabs_slots + ((blockIdx.x * 8 + (tid >> 5)) & (kMaxSlots - 1)) * kSlotStride,
                      (unsigned long long)__double_as_longlong(mx));
    }
}

int g_sms = 0;

}  // namespace

cudaError_t launch_pipe(const PipeArgs& a, bool xsplit, cudaStream_t s) {
    if (a.n_tiles <= 0) return cudaSuccess;
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
        cudaFuncSetAttribute(spmv_pipe_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(PipeSmem));
        cudaFuncSetAttribute(spmv_pipe_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(PipeSmem));
    }
    const int grid = 2 * g_sms;
    cudaError_t e = cudaMemsetAsync(a.tile_counter, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
    if (xsplit) spmv_pipe_kernel<true><<<grid, kPipeThreads, sizeof(PipeSmem), s>>>(a);
    else spmv_pipe_kernel<false><<<grid, kPipeThreads, sizeof(PipeSmem), s>>>(a);
    return cudaGetLastError();
}

size_t pipe_smem_bytes() { return sizeof(PipeSmem); }

}  // namespace spmvb
