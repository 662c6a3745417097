// pipe.cu -- the single-SpMxV kernel y^ = A^ x^ (per-row temporary and
// one y store), persistent and warp-specialised for sm_100a.
//
//   * grid = 2 CTAs per SM, row tiles dealt round-robin (t = blockIdx.x +
//     i*grid): all CTAs sweep the tiles in order, so the live x footprint is
//     one SB block's x(C_k) plus x(C_B) (Eq.(1)) -- the paper's
//     "fits into the cache" condition with the 126 MB L2 as the cache;
//   * a producer warp streams each tile's col/val/row-pointer slices into a
//     3-stage shared-memory ring with 1-D bulk async copies (TMA engine,
//     `cp.async.bulk`, SASS UBLKCP) that complete on mbarriers; the matrix is
//     read exactly once with an L2 evict-first policy (no temporal
//     locality in the matrix), leaving the LSU pipe to the x gathers;
//   * 8 consumer warps: thread t owns tile positions [8t, 8t+8) (two LDS.128
//     of columns, four of values), gathers x[col] through the read-only path,
//     keeps the products in registers and reduces them with a deterministic
//     merge-path segmented sum (a row's sum = its first thread's serial
//     partial, then the later threads' partials in thread order);
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

struct __align__(16) StageHdr {
    int32_t r0, r1, a, b;
};

struct __align__(16) PipeSmem {
    double val[kStages][kTileNnz];           // positions [0, kTileNnz) from a & ~3
    int32_t col[kStages][kTileNnz];
    int32_t so[kStages][kSoElems];
    StageHdr hdr[kStages];
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

// One consumer thread's slice of a tile: positions [8t, 8t+8) of the stage
// buffers (position p holds nonzero a4 + p), its values and gathered x.
struct Slice {
    StageHdr h;
    int st;
    bool big;            // long row: direct-load path
    double v[kE];
    double x[kE];
};

template <bool XSPLIT>
__device__ __forceinline__ void fetch(const PipeArgs& A, PipeSmem& sm, int it, Slice& S) {
    const int tid = threadIdx.x;
    S.st = it % kStages;
    mbar_wait(&sm.full[S.st], (uint32_t)(it / kStages) & 1);
    S.h = sm.hdr[S.st];
    const int off = S.h.a & 3;
    const int n = S.h.b - S.h.a;
    S.big = off + n > kTileNnz;
    if (S.big) return;
    const int lo = off, hi = off + n;
    const int p0 = tid * kE;
    const int4 c0 = *reinterpret_cast<const int4*>(&sm.col[S.st][p0]);
    const int4 c1 = *reinterpret_cast<const int4*>(&sm.col[S.st][p0 + 4]);
    const double2* vp = reinterpret_cast<const double2*>(&sm.val[S.st][p0]);
    const double2 v0 = vp[0], v1 = vp[1], v2 = vp[2], v3 = vp[3];
    const int c[kE] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    S.v[0] = v0.x; S.v[1] = v0.y; S.v[2] = v1.x; S.v[3] = v1.y;
    S.v[4] = v2.x; S.v[5] = v2.y; S.v[6] = v3.x; S.v[7] = v3.y;
#pragma unroll
    for (int u = 0; u < kE; ++u) {
        const int p = p0 + u;
        S.x[u] = (p >= lo && p < hi) ? ldx<XSPLIT>(A, c[u]) : 0.0;
    }
}

template <bool XSPLIT>
__global__ void __launch_bounds__(kPipeThreads, 2) spmv_pipe_kernel(const PipeArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PipeSmem& sm = *reinterpret_cast<PipeSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const int T = A.n_tiles;
    const int G = gridDim.x;

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (tid >= kCons) {
        // ------------------------------------------------------- producer warp
        const int lane = tid & 31;
        const uint64_t pol_first = policy(true);
        const uint64_t pol_norm = policy(false);
        int it = 0;
        for (int base = blockIdx.x; base < T; base += 32 * G) {
            const int tj = base + lane * G;
            int m_r0 = 0, m_r1 = 0, m_a = 0, m_b = 0;
            if (tj < T) {
                m_r0 = A.tile_row[tj];
                m_r1 = A.tile_row[tj + 1];
                m_a = A.tile_nnz[tj];
                m_b = A.tile_nnz[tj + 1];
            }
            const int cnt = min(32, (T - base + G - 1) / G);
            for (int j = 0; j < cnt; ++j, ++it) {
                const int r0 = __shfl_sync(0xffffffffu, m_r0, j);
                const int r1 = __shfl_sync(0xffffffffu, m_r1, j);
                const int a = __shfl_sync(0xffffffffu, m_a, j);
                const int b = __shfl_sync(0xffffffffu, m_b, j);
                const int st = it % kStages;
                const uint32_t k = (uint32_t)(it / kStages);
                if (lane == 0) {
                    if (k > 0) mbar_wait(&sm.empty[st], (k - 1) & 1);
                    sm.hdr[st] = StageHdr{r0, r1, a, b};
                    const int a4 = a & ~3;
                    if (b - a4 > kTileNnz) {
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
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    const uint64_t pol_first = policy(true);
    double mx = 0.0;
    int it = 0;
    int t = blockIdx.x;
    Slice cur, nxt;
    if (t < T) fetch<XSPLIT>(A, sm, 0, cur);
    for (; t < T; t += G, ++it) {
        if (t + G < T) fetch<XSPLIT>(A, sm, it + 1, nxt);   // next tile's gathers in flight
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
                mbar_arrive(&sm.empty[cur.st]);
            }
            cons_sync();
        } else {
            for (int j = tid; j < nr; j += kCons) ysum[j] = 0.0;
            const int off = h.a & 3;
            const int n = h.b - h.a;
            // so(j) = row_ptr[r0 + j] - a4: row j occupies positions [so(j), so(j+1))
            const int32_t* so = sm.so[cur.st] + (h.r0 & 3);
            const int a4 = h.a & ~3;
            const int e_lo = max(tid * kE, off);
            const int e_hi = min(tid * kE + kE, off + n);
            bool pending = false;
            double own = 0.0;
            int own_s = -1;
            sm.head_seg[tid] = -1;
            cons_sync();    // ysum zeroed, head_seg reset before any emit
            if (e_lo < e_hi) {
                int lo = 0, hi = nr - 1;                  // last row with so(s) <= e_lo
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (so[mid] - a4 <= e_lo) lo = mid; else hi = mid - 1;
                }
                int s = lo;
                int nb = so[s + 1] - a4;                  // end of row s
                bool head = so[s] - a4 < e_lo;            // row began in an earlier thread
                double acc = 0.0;
#pragma unroll
                for (int u = 0; u < kE; ++u) {
                    const int p = tid * kE + u;
                    if (p >= e_lo && p < e_hi) {
                        while (p >= nb) {                 // close row s (and skip empty rows)
                            if (head) { sm.head_val[tid] = acc; sm.head_seg[tid] = s; head = false; }
                            else if (so[s] - a4 < nb) ysum[s] = acc;
                            acc = 0.0;
                            ++s;
                            nb = so[s + 1] - a4;
                        }
                        acc += cur.v[u] * cur.x[u];
                    }
                }
                if (nb <= e_hi) {                         // row s ends exactly at e_hi
                    if (head) { sm.head_val[tid] = acc; sm.head_seg[tid] = s; }
                    else ysum[s] = acc;
                } else {                                  // row s continues in later threads
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
            if (tid == 0) mbar_arrive(&sm.empty[cur.st]);   // stage consumed
            for (int j = tid; j < nr; j += kCons) {
                const double v = ysum[j];
                A.y[h.r0 + j] = v;
                mx = fmax(mx, fabs(v));
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
    const int grid = a.n_tiles < 2 * g_sms ? a.n_tiles : 2 * g_sms;
    if (xsplit) spmv_pipe_kernel<true><<<grid, kPipeThreads, sizeof(PipeSmem), s>>>(a);
    else spmv_pipe_kernel<false><<<grid, kPipeThreads, sizeof(PipeSmem), s>>>(a);
    return cudaGetLastError();
}

size_t pipe_smem_bytes() { return sizeof(PipeSmem); }

}  // namespace spmvb
