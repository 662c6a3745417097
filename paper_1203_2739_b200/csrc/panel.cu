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
#include <algorithm>
#include <cstdlib>
#include <cuda_runtime.h>

#include "internal.h"

namespace spmvb {
namespace {

constexpr int NW = kPnWarps;
constexpr int kT = NW * 32;
constexpr int kD = 16;    // groups in flight per warp (template default)
constexpr int kDefD = kPnB == 8 ? 16 : 12;   // the launch default
constexpr int kPF = 8;    // default: epochs of the group stream prefetched into L2 ahead
static_assert(kD % kPnB == 0, "ring geometry");
constexpr uint32_t kDeltaMask = (1u << kPnDeltaBits) - 1u;

__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_x(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
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

// MODE (ablation, measurements only; 0 = the kernel): 1 no x gathers (x = 1),
// 2 no shared-memory y update (register sum), 3 no epoch barriers (racy),
// 4 no L2 prefetch of the group stream, 5 gathers 4 steps ahead (not 8),
// 6 gathers of a fixed 2 MB window (no dependence on the loaded indices' values)
template <int MODE, int KD_ = kD, int KGD_ = 8>
__global__ void __launch_bounds__(kT, 1) spmv_panel_kernel(const PnArgs A) {
    constexpr bool kMain = MODE == 0 || MODE == 24;      // the kernel (24: without the next-panel prefetch)
    constexpr int kD = KD_;                              // groups in flight per warp
    constexpr int kGD = MODE == 5 ? 4 : KGD_;            // gathers issued this many steps ahead
    static_assert(kD % kGD == 0 && kD % kPnB == 0, "ring geometry");
    extern __shared__ __align__(16) double ys[];
    const int p = blockIdx.x;
    const PnPanel d = A.panel[p];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < ((d.nslots + 15) & ~15); i += kT) ys[i] = 0.0;   // the panel's y slots
    // virtual-row slot lists of the panel's split rows, copied to shared memory
    // once (the epilogue folds them by warps)
    uint16_t* ssl = reinterpret_cast<uint16_t*>(ys + A.max_rows + 1);
    int32_t* sdesc = reinterpret_cast<int32_t*>(ssl + ((A.max_sslots + 7) & ~7));   // (first, count, row) per split row
    {
        for (int i = tid; i < d.sslot_n; i += kT) ssl[i] = A.split_slots[d.sslot0 + i];
        for (int i = tid; i < d.split_n; i += kT) {
            const int e = d.split_off + i;
            sdesc[3 * i] = A.split_first[e] - d.sslot0;
            sdesc[3 * i + 1] = A.split_cnt[e];
            sdesc[3 * i + 2] = A.split_row[e];
        }
    }
    __syncthreads();

    const uint64_t pol = pol_evict_first();
    const uint64_t polx = pol_evict_last();   // x is the reused operand
    const int PF = A.pf_epochs > 0 ? A.pf_epochs : kPF;
    const int T = d.ne * kPnB;                       // steps per warp
    const int scratch = A.max_rows;                  // y slot of the padding lanes
    const int64_t gw = (int64_t)d.g0 + warp;         // group of step t: gw + 16 t

    double rv[kD];
    uint32_t ri[kD];
    int32_t rb[kD];
    double rx[kGD];
    // one 16-byte load per epoch gives the warp the bases of its kPnB groups
    // (slots u..u+3 of the ring; the bases of u+1..u+3 it replaces were last
    // used by gathers issued >= 1 step earlier, since kGD >= kPnB)
    static_assert(!kMain || kGD >= 4, "base quad overwrites bases still needed");
    static_assert(kPnB % 4 == 0, "bases are loaded four at a time");
    const int4* gb4 = reinterpret_cast<const int4*>(A.gbase4 + d.g0);
    auto load = [&](int t, double& v, uint32_t& i, int32_t& b) {
        const int64_t g = gw + 16 * (int64_t)t;
        v = ld_val(A.gval + g * 32 + lane, pol);
        i = ld_u32(A.gidx + g * 32 + lane, pol);
        if (!kMain) b = ld_base(A.gbase + g);
    };
    auto load_b4 = [&](int t, int32_t& b0, int32_t& b1, int32_t& b2, int32_t& b3) {   // t % 4 == 0
        int4 q;
        const int64_t o = ((int64_t)(t / kPnB) * kPnWarps + warp) * (kPnB / 4) + (t % kPnB) / 4;
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "l"(gb4 + o));
        b0 = q.x; b1 = q.y; b2 = q.z; b3 = q.w;
    };
    double racc = 0.0;
    auto gather = [&](uint32_t i, int32_t b) -> double {
        if (MODE == 1) return 1.0;
        if (MODE == 6) return __ldg(A.x_lo + ((b + (int)(i & 0xFFF)) & 0x3FFFF));
        if (MODE == 15) {
            if (i == kPnDummy) return 0.0;
            const double* xp = b < A.x_split ? A.x_lo + b : A.x_hi + (b - A.x_split);
            return __ldg(xp + (i & kDeltaMask));
        }
        if (MODE == 16) return ld_x(A.x_lo + ((b + (int)(i & 0xFFF)) & 0x3FFFF), polx);
        if (MODE == 13) return i == kPnDummy ? 0.0 : ld_x(A.x_lo + ((b + (int)(i & kDeltaMask)) & 0x3FFFF), polx);
        if (MODE == 14) return i == kPnDummy ? 0.0 : ld_x(A.x_lo + ((b & 0x3FFFF) + (int)(i & kDeltaMask)), polx);
        // unconditional: a padding lane reads x[base] (valid) and adds 0 * x into
        // the scratch y slot -- a predicated-off load behind a branch made the
        // warp wait for the gather at the branch (measured 1.6x slower)
        const double* xp = b < A.x_split ? A.x_lo + b : A.x_hi + (b - A.x_split);
        return ld_x(xp + (i & kDeltaMask), polx);
    };
    // L2 prefetch of the panel's group stream kPF epochs ahead (one bulk
    // prefetch per array per epoch, issued by thread 0): the register ring
    // then waits for L2, not HBM, latency -- the x gathers depend on the
    // loaded indices, so their distance is what bounds the pipeline.
    // Past the panel's last epoch it prefetches the first epochs of panel
    // p + gridDim.x -- about the panel the block scheduler starts next, on
    // whichever SM frees first -- so a new CTA's ring does not fill from HBM.
    int nx_g0 = 0, nx_ne = 0;
    if (tid == 0 && MODE != 24 && p + (int)gridDim.x < A.n_panels) {
        nx_g0 = A.panel[p + gridDim.x].g0;
        nx_ne = A.panel[p + gridDim.x].ne;
    }
    auto prefetch_epoch = [&](int e) {
        if (tid == 0 && e >= d.ne && e - d.ne < nx_ne) {
            const int64_t g = (int64_t)nx_g0 + (int64_t)(e - d.ne) * kPnEpoch;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gval + g * 32), "r"(kPnEpoch * 32 * 8)
                         : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gidx + g * 32), "r"(kPnEpoch * 32 * 4)
                         : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((kMain ? A.gbase4 : A.gbase) + g),
                         "r"(kPnEpoch * 4) : "memory");
        } else if (tid == 0 && e < d.ne) {
            const int64_t g = (int64_t)d.g0 + (int64_t)e * kPnEpoch;
            // normal priority: an evict_first prefetch is the first victim of the next one
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gval + g * 32), "r"(kPnEpoch * 32 * 8)
                         : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gidx + g * 32), "r"(kPnEpoch * 32 * 4)
                         : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((kMain ? A.gbase4 : A.gbase) + g),
                         "r"(kPnEpoch * 4) : "memory");
        }
    };
    if (MODE != 4) {
        for (int e = 0; e < PF; ++e) prefetch_epoch(e);
        // this panel's slice of the next SB block's x(C_k), kept in L2 (evict_last)
        if (tid == 32 && d.pf_len > 0) {
            const uint64_t pl = pol_evict_last();
            // 16-byte aligned start and length (bulk prefetch granularity)
            const uintptr_t a0 = reinterpret_cast<uintptr_t>(A.x_lo + d.pf_col) & ~uintptr_t(15);
            const uintptr_t a1 = reinterpret_cast<uintptr_t>(A.x_lo + d.pf_col + d.pf_len) & ~uintptr_t(15);
            for (uintptr_t a = a0; a < a1; a += 32768) {
                const uint32_t n = (uint32_t)(a1 - a < 32768 ? a1 - a : 32768);
                asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a), "r"(n), "l"(pl)
                             : "memory");
            }
        }
    }
#pragma unroll
    for (int u = 0; u < kD; ++u) {
        if (u < T) load(u, rv[u], ri[u], rb[u]);
        if (kMain && u % 4 == 0 && u < T) load_b4(u, rb[u], rb[u + 1], rb[u + 2], rb[u + 3]);
    }
#pragma unroll
    for (int u = 0; u < kGD; ++u)
        if (u < T) rx[u] = gather(ri[u], rb[u]);

    for (int t0 = 0; t0 < T; t0 += kD) {
#pragma unroll
        for (int u = 0; u < kD; ++u) {
            const int t = t0 + u;
            if (t >= T) break;
            const uint32_t i = ri[u];
            if (MODE == 2) {
                racc = fma(rv[u], rx[u % kGD], racc);
            } else {
                int r = (int)(i >> kPnDeltaBits);
                r = r == (int)(kPnDummy >> kPnDeltaBits) ? scratch : r;
                ys[r] = fma(rv[u], rx[u % kGD], ys[r]);
            }
            if (t + kD < T) {
                load(t + kD, rv[u], ri[u], rb[u]);
                if (kMain && u % 4 == 0)
                    load_b4(t + kD, rb[u], rb[(u + 1) % kD], rb[(u + 2) % kD], rb[(u + 3) % kD]);
            }
            if (t + kGD < T) rx[u % kGD] = gather(ri[(u + kGD) % kD], rb[(u + kGD) % kD]);
            if (u % kPnB == kPnB - 1) {                  // epoch boundary (T is a multiple of kPnB)
                if (MODE != 3) __syncthreads();
                if (MODE != 4) prefetch_epoch(t / kPnB + PF);
            }
        }
    }
    if (MODE == 2 && racc == 1.2345) ys[0] = racc;
    // epilogue: y[row] = ys[slot(row)].  The slot loads are batched 16 per
    // thread (clamped addresses, no branch) and the first batch is issued
    // before the barrier, so their latency is not paid once per row.
    constexpr int EB = 16;
    uint16_t sl[EB];
    const uint16_t* r2s = A.row2slot + d.row0;
    const int nrl = d.nrows;
    auto load_slots = [&](int i0) {
#pragma unroll
        for (int k = 0; k < EB; ++k) sl[k] = r2s[min(i0 + k * kT, nrl - 1)];
    };
    load_slots(tid);
    __syncthreads();

    double mx = 0.0;
    for (int i0 = tid; i0 < nrl; i0 += EB * kT) {
        if (i0 != tid) load_slots(i0);
#pragma unroll
        for (int k = 0; k < EB; ++k) {
            const int i = i0 + k * kT;
            if (i < nrl && sl[k] < 0x8000) {        // split rows: below
                const double v = ys[sl[k]];
                A.y[d.row0 + i] = v;
                mx = fmax(mx, fabs(v));
            }
        }
    }
    // rows split into virtual rows (long rows; a split handle's (row, part)
    // segments): up to kPnFoldSeq slots, one thread per row adds them in fold
    // order (part order); longer rows one warp each, lanes sum strided
    // slots, fixed xor tree.  Both orders are fixed by the plan (deterministic).
    for (int k = tid; k < d.split_short; k += kT) {
        const int f = sdesc[3 * k], c = sdesc[3 * k + 1];
        double v = ys[ssl[f]];
        for (int j = 1; j < c; ++j) v += ys[ssl[f + j]];
        A.y[d.row0 + sdesc[3 * k + 2]] = v;
        mx = fmax(mx, fabs(v));
    }
    for (int k = d.split_short + warp; k < d.split_n; k += NW) {
        const int f = sdesc[3 * k], c = sdesc[3 * k + 1];
        double v = 0.0;
        for (int j = lane; j < c; j += 32) v += ys[ssl[f + j]];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) {
            A.y[d.row0 + sdesc[3 * k + 2]] = v;
            mx = fmax(mx, fabs(v));
        }
    }
    if (A.maxabs_slots) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if (lane == 0 && mx > 0.0)
            atomicMax(A.maxabs_slots + ((p * NW + warp) & (kMaxSlots - 1)) * kSlotStride,
                      (unsigned long long)__double_as_longlong(mx));
    }
}

// ---------------------------------------------------------------------------
// Variant with the x gathers going to shared memory (cp.async, no register
// cost per gather in flight): G steps of gathers in flight per warp.
template <int G>
__global__ void __launch_bounds__(kT, 1) spmv_panel2_kernel(const PnArgs A) {
    constexpr int kD2 = 24;   // groups of (value, index, base) in flight per warp (registers)
    static_assert(kD2 % kPnB == 0 && kD2 % G == 0 && G >= 2 && G < kD2, "ring geometry");
    extern __shared__ __align__(16) double sm2[];
    double* ys = sm2;
    const int p = blockIdx.x;
    const PnPanel d = A.panel[p];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    double* gr = sm2 + ((A.max_rows + 2) & ~1) + warp * G * 32;
    const uint32_t gr_s = (uint32_t)__cvta_generic_to_shared(gr) + lane * 8;
    for (int i = tid; i < ((d.nslots + 15) & ~15); i += kT) ys[i] = 0.0;   // the panel's y slots
    __syncthreads();

    const uint64_t pol = pol_evict_first();
    const uint64_t polx = pol_evict_last();
    const int PF = A.pf_epochs > 0 ? A.pf_epochs : kPF;
    const int T = d.ne * kPnB;
    const int64_t gw = (int64_t)d.g0 + warp;

    double rv[kD2];
    uint32_t ri[kD2];
    int32_t rb[kD2];
    auto load = [&](int t, double& v, uint32_t& i, int32_t& b) {
        const int64_t g = gw + 16 * (int64_t)t;
        v = ld_val(A.gval + g * 32 + lane, pol);
        i = ld_u32(A.gidx + g * 32 + lane, pol);
        b = ld_base(A.gbase + g);
    };
    auto issue = [&](int slot, uint32_t i, int32_t b) {
        if (i != kPnDummy) {
            const double* xp = (b < A.x_split ? A.x_lo + b : A.x_hi + (b - A.x_split)) + (i & kDeltaMask);
            asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(gr_s + slot * 256),
                         "l"(xp), "l"(polx) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto prefetch_epoch = [&](int e) {
        if (tid == 0 && e < d.ne) {
            const int64_t g = (int64_t)d.g0 + (int64_t)e * kPnEpoch;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gval + g * 32), "r"(kPnEpoch * 32 * 8)
                         : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gidx + g * 32), "r"(kPnEpoch * 32 * 4)
                         : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gbase + g), "r"(kPnEpoch * 4)
                         : "memory");
        }
    };
    for (int e = 0; e < PF; ++e) prefetch_epoch(e);
    if (tid == 32 && d.pf_len > 0) {
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(A.x_lo + d.pf_col) & ~uintptr_t(15);
        const uintptr_t a1 = reinterpret_cast<uintptr_t>(A.x_lo + d.pf_col + d.pf_len) & ~uintptr_t(15);
        for (uintptr_t a = a0; a < a1; a += 32768) {
            const uint32_t n = (uint32_t)(a1 - a < 32768 ? a1 - a : 32768);
            asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a), "r"(n), "l"(polx)
                         : "memory");
        }
    }
#pragma unroll
    for (int u = 0; u < kD2; ++u)
        if (u < T) load(u, rv[u], ri[u], rb[u]);
#pragma unroll
    for (int u = 0; u < G - 1; ++u) {
        if (u < T) issue(u, ri[u], rb[u]);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }

    for (int t0 = 0; t0 < T; t0 += kD2) {
#pragma unroll
        for (int u = 0; u < kD2; ++u) {
            const int t = t0 + u;
            if (t >= T) break;
            // gathers of step t + G - 1 into ring slot (t + G - 1) % G (consumed at step t - 1)
            if (t + G - 1 < T) issue((u + G - 1) % G, ri[(u + G - 1) % kD2], rb[(u + G - 1) % kD2]);
            else asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group %0;" ::"n"(G - 1) : "memory");
            const uint32_t i = ri[u];
            if (i != kPnDummy) {
                const int r = (int)(i >> kPnDeltaBits);
                ys[r] = fma(rv[u], gr[(u % G) * 32 + lane], ys[r]);
            }
            if (t + kD2 < T) load(t + kD2, rv[u], ri[u], rb[u]);
            if (u % kPnB == kPnB - 1) {
                __syncthreads();
                prefetch_epoch(t / kPnB + PF);
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();

    double mx = 0.0;
    for (int i = tid; i < d.nrows; i += kT) {
        const uint16_t q = A.row2slot[d.row0 + i];
        double v = 0.0;
        if (q < 0x8000) {
            v = ys[q];
        } else {
            const int k = d.split_off + (q & 0x7FFF);
            for (int j = 0; j < A.split_cnt[k]; ++j) v += ys[A.split_slots[A.split_first[k] + j]];
        }
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

// ---------------------------------------------------------------------------
// Variant 3: the group stream goes HBM -> L2 (bulk prefetch) -> shared memory
// (bulk copies, one per array per epoch, mbarrier-tracked) instead of
// through registers, so the LSU queue carries only the x gathers (L2 hits)
// and the shared-memory traffic.  NS epochs of stream staged, G steps of
// gathers in flight per warp.
constexpr int kStage3 = kPnEpoch * 32 * 8 + kPnEpoch * 32 * 4 + kPnEpoch * 4;   // 24,832 B per epoch

template <int NS, int G>
__global__ void __launch_bounds__(kT, 1) spmv_panel3_kernel(const PnArgs A) {
    static_assert(G % kPnB == 0 && G / kPnB <= NS - 1, "gathers read stages loaded ahead");
    constexpr int U = G;   // unroll (multiple of kPnB)
    extern __shared__ __align__(128) unsigned char sm3[];
    const int p = blockIdx.x;
    const PnPanel d = A.panel[p];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int yb = (((A.max_rows + 1) * 8 + 127) / 128) * 128;
    double* ys = reinterpret_cast<double*>(sm3);
    unsigned char* st = sm3 + yb;
    uint64_t* full = reinterpret_cast<uint64_t*>(st + NS * kStage3);
    auto sval = [&](int e) { return reinterpret_cast<const double*>(st + (e % NS) * kStage3); };
    auto sidx = [&](int e) { return reinterpret_cast<const uint32_t*>(st + (e % NS) * kStage3 + kPnEpoch * 32 * 8); };
    auto sbase = [&](int e) { return reinterpret_cast<const int32_t*>(st + (e % NS) * kStage3 + kPnEpoch * 32 * 12); };

    const uint64_t polx = pol_evict_last();
    const uint64_t pol = pol_evict_first();
    const int PF = A.pf_epochs > 0 ? A.pf_epochs : kPF;
    const int ne = d.ne, T = ne * kPnB;
    auto bulk = [&](void* dst, const void* src, int bytes, uint64_t* bar) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                     "r"((uint32_t)__cvta_generic_to_shared(bar)), "l"(pol) : "memory");
    };
    auto load_epoch = [&](int e) {   // thread 0 only
        if (e >= ne) return;
        uint64_t* bar = &full[e % NS];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                     "r"(kStage3) : "memory");
        const int64_t g = (int64_t)d.g0 + (int64_t)e * kPnEpoch;
        unsigned char* dst = st + (e % NS) * kStage3;
        bulk(dst, A.gval + g * 32, kPnEpoch * 32 * 8, bar);
        bulk(dst + kPnEpoch * 32 * 8, A.gidx + g * 32, kPnEpoch * 32 * 4, bar);
        bulk(dst + kPnEpoch * 32 * 12, A.gbase + g, kPnEpoch * 4, bar);
    };
    auto prefetch_epoch = [&](int e) {   // thread 0 only
        if (e >= ne) return;
        const int64_t g = (int64_t)d.g0 + (int64_t)e * kPnEpoch;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gval + g * 32), "r"(kPnEpoch * 32 * 8) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gidx + g * 32), "r"(kPnEpoch * 32 * 4) : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gbase + g), "r"(kPnEpoch * 4) : "memory");
    };
    auto wait_epoch = [&](int e) {
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&full[e % NS]);
        const uint32_t par = (uint32_t)((e / NS) & 1);
        asm volatile("{\n.reg .pred q;\nW3: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W3;\n}"
                     ::"r"(bar), "r"(par) : "memory");
    };

    if (tid == 0) {
        for (int s = 0; s < NS; ++s)
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    for (int i = tid; i < ((d.nslots + 15) & ~15); i += kT) ys[i] = 0.0;   // the panel's y slots
    __syncthreads();
    if (tid == 0) {
        for (int e = 0; e < NS; ++e) load_epoch(e);
        for (int e = NS; e < NS + PF; ++e) prefetch_epoch(e);
    }
    if (tid == 32 && d.pf_len > 0) {
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(A.x_lo + d.pf_col) & ~uintptr_t(15);
        const uintptr_t a1 = reinterpret_cast<uintptr_t>(A.x_lo + d.pf_col + d.pf_len) & ~uintptr_t(15);
        for (uintptr_t a = a0; a < a1; a += 32768) {
            const uint32_t n = (uint32_t)(a1 - a < 32768 ? a1 - a : 32768);
            asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(a), "r"(n), "l"(polx)
                         : "memory");
        }
    }

    double rx[G];
    uint32_t ri[G];
    // gather of step t: group k = (t % kPnB) * 16 + warp of epoch t / kPnB
    auto issue = [&](int t, double& xv, uint32_t& iv) {
        const int e = t / kPnB, k = (t % kPnB) * NW + warp;
        const uint32_t i = sidx(e)[k * 32 + lane];
        const int32_t b = sbase(e)[k];
        iv = i;
        const double* xp = b < A.x_split ? A.x_lo + b : A.x_hi + (b - A.x_split);
        xv = ld_x(xp + (i & kDeltaMask), polx);   // padding lanes: x[base], added 0 * x into the scratch slot
    };
    for (int e = 0; e < G / kPnB && e < ne; ++e) wait_epoch(e);
#pragma unroll
    for (int u = 0; u < G; ++u)
        if (u < T) issue(u, rx[u], ri[u]);

    for (int t0 = 0; t0 < T; t0 += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = t0 + u;
            if (t >= T) break;
            const int e = t / kPnB, k = (u % kPnB) * NW + warp;
            const uint32_t i = ri[u];
            {
                int r = (int)(i >> kPnDeltaBits);
                r = r == (int)(kPnDummy >> kPnDeltaBits) ? A.max_rows : r;
                ys[r] = fma(sval(e)[k * 32 + lane], rx[u], ys[r]);
            }
            const int tn = t + G;
            if (tn < T) {
                if (u % kPnB == 0) wait_epoch(tn / kPnB);
                issue(tn, rx[u], ri[u]);
            }
            if (u % kPnB == kPnB - 1) {   // end of epoch e: its stage is free for epoch e + NS
                __syncthreads();
                if (tid == 0) {
                    load_epoch(e + NS);
                    prefetch_epoch(e + NS + PF);
                }
            }
        }
    }
    __syncthreads();

    double mx = 0.0;
    for (int i = tid; i < d.nrows; i += kT) {
        const uint16_t q = A.row2slot[d.row0 + i];
        double v = 0.0;
        if (q < 0x8000) {
            v = ys[q];
        } else {
            const int k = d.split_off + (q & 0x7FFF);
            for (int j = 0; j < A.split_cnt[k]; ++j) v += ys[A.split_slots[A.split_first[k] + j]];
        }
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
    static int mode = -1, pf_env = 0;
    // only the panel's y in shared memory: the rest of the 256 KB L1/shared
    // array stays L1, which holds the global loads in flight
    const size_t smem = (size_t)(a.max_rows + 1) * sizeof(double)     // + the padding lanes' scratch slot
                        + (size_t)((a.max_sslots + 7) & ~7) * 2           // split rows' slot lists
                        + (size_t)a.max_split_n * 12;                     // and their (first, count, row)
    if (mode < 0) {
        const char* e = getenv("SPMV_PN_MODE");   // ablations for measurements only
        mode = e ? atoi(e) : 0;
        const char* f = getenv("SPMV_PN_PF");
        pf_env = f ? atoi(f) : 0;
        cudaError_t r = cudaSuccess;
        const int smax = 227 * 1024;
        r = cudaFuncSetAttribute(spmv_panel_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
#if SPMV_PN_B == 4
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<0, 24, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
#endif
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<0, 16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<0, kDefD, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<0, 8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<24, kDefD, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
#if SPMV_PN_B == 4
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<0, 20, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
#endif
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<15>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<13>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<14>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel2_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel2_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel3_kernel<4, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel3_kernel<3, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
#if SPMV_PN_B == 4
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel3_kernel<4, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
#endif
#if SPMV_PN_B == 4
        if (r == cudaSuccess) r = cudaFuncSetAttribute(spmv_panel3_kernel<5, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
#endif
        if (r != cudaSuccess) return r;
    }
    PnArgs b = a;
    auto smem3 = [&](int NS) { return (size_t)((((a.max_rows + 1) * 8 + 127) / 128) * 128) + (size_t)NS * kStage3 + 64; };
    auto smem2 = [&](int G) { return (size_t)((a.max_rows + 2) & ~1) * 8 + (size_t)NW * G * 256; };
    if (pf_env > 0) b.pf_epochs = pf_env;
    switch (mode) {
    case 1: spmv_panel_kernel<1><<<b.n_panels, kT, smem, s>>>(b); break;
    case 2: spmv_panel_kernel<2><<<b.n_panels, kT, smem, s>>>(b); break;
    case 3: spmv_panel_kernel<3><<<b.n_panels, kT, smem, s>>>(b); break;
    case 4: spmv_panel_kernel<4><<<b.n_panels, kT, smem, s>>>(b); break;
#if SPMV_PN_B == 4
    case 17: spmv_panel_kernel<0, 24, 8><<<b.n_panels, kT, smem, s>>>(b); break;
#endif
    case 18: spmv_panel_kernel<0, 16, 4><<<b.n_panels, kT, smem, s>>>(b); break;
#if SPMV_PN_B == 4
    case 19: spmv_panel_kernel<0, 12, 4><<<b.n_panels, kT, smem, s>>>(b); break;
#endif
#if SPMV_PN_B == 4
    case 20: spmv_panel_kernel<0, 20, 4><<<b.n_panels, kT, smem, s>>>(b); break;
#endif
    case 15: spmv_panel_kernel<15><<<b.n_panels, kT, smem, s>>>(b); break;
    case 16: spmv_panel_kernel<16><<<b.n_panels, kT, smem, s>>>(b); break;
    case 13: spmv_panel_kernel<13><<<b.n_panels, kT, smem, s>>>(b); break;
    case 14: spmv_panel_kernel<14><<<b.n_panels, kT, smem, s>>>(b); break;
    case 6: spmv_panel_kernel<6><<<b.n_panels, kT, smem, s>>>(b); break;
    case 5: spmv_panel_kernel<5><<<b.n_panels, kT, smem, s>>>(b); break;
    case 9: spmv_panel3_kernel<4, 8><<<b.n_panels, kT, smem3(4), s>>>(b); break;
    case 10: spmv_panel3_kernel<3, 8><<<b.n_panels, kT, smem3(3), s>>>(b); break;
#if SPMV_PN_B == 4
    case 11: spmv_panel3_kernel<4, 12><<<b.n_panels, kT, smem3(4), s>>>(b); break;
#endif
#if SPMV_PN_B == 4
    case 12: spmv_panel3_kernel<5, 16><<<b.n_panels, kT, smem3(5), s>>>(b); break;
#endif
    case 7: spmv_panel2_kernel<8><<<b.n_panels, kT, smem2(8), s>>>(b); break;
    case 8: spmv_panel2_kernel<12><<<b.n_panels, kT, smem2(12), s>>>(b); break;
    case 21: spmv_panel_kernel<0><<<b.n_panels, kT, smem, s>>>(b); break;   // previous default (16, 8)
    case 22: spmv_panel_kernel<0, 8, 4><<<b.n_panels, kT, smem, s>>>(b); break;
    case 24: spmv_panel_kernel<24, kDefD, 4><<<b.n_panels, kT, smem, s>>>(b); break;   // no next-panel prefetch
    default: spmv_panel_kernel<0, kDefD, 4><<<b.n_panels, kT, smem, s>>>(b);
    }
    return cudaGetLastError();
}

}  // namespace spmvb
