// panel.cu -- column-sorted panel SpMxV y^ = A^ x^: the default
// kernel at world 1 (and of SB-form handles, Eq.(1), at any world
// size), and of the fused multiple-SpMxV, whose (row, part)
// segments are planned as virtual rows of their own.
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
// One CTA of 16 warps per panel (y of up to 28,672 slots in shared memory,
// about 16 K by default so the rest of the L1 holds the loads in flight; 1
// CTA per SM; panel counts sum to whole waves).
// Warp w processes groups g0 + 16 t + w, t = 0, 1, ...; every kPnB steps is an
// epoch boundary (__syncthreads): within an epoch all rows are distinct, so
// the shared-memory read-modify-writes y_s[r] += v * x[c] never race.
// Per warp, a register ring keeps kD (8) groups of (value, index, base) in
// flight (L1 no-allocate, L2 evict-first: the matrix is read once) and
// issues the x gathers kGD steps ahead of their use.  The epilogue writes y
// once per row and folds max |y|.
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace spmvb {
namespace {

constexpr int NW = kPnWarps;
constexpr int kT = NW * 32;
constexpr int kDefD = 8;    // steps (groups) in flight per warp, the launch default (8 beat 12 and 16 on C5
                            // by 2.5 % / 1 %, interleaved A/B; equal on C4 and C3)
constexpr int kPF = 4;    // default: epochs of the group stream prefetched into L2 ahead (with the 8-deep
                          // ring: 4 beat 2, 3, 5, 6, 8, 12 -- C5 -3.8 %, C4 -2.2 % vs 8, interleaved A/B;
                          // re-checked late round 2 under the power cap: 2 / 3 / 6 vs 4
                          // = +9 / +1 / 0 %, profiles/r02_ab_stream_prefetch.txt)
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
__device__ __forceinline__ double ld_x_na(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_x(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
// world > 1: the border buffer is written by the exchange while the kernel
// runs (before the CTA's border epochs), so its reads are coherent weak loads,
// not the read-only (.nc) path, and never allocate in L1
__device__ __forceinline__ double ld_x_co(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int32_t ld_acquire_sys(const int32_t* p) {
    int32_t v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Group stream layout (host.cpp upload_panel_stream): the kPnB = 4 groups a
// warp runs in one epoch form a 128-entry block, (epoch e, warp w) at
// g0 * 32 + (e * 16 + w) * 128: values as two (step, lane, step & 1) pairs
// -- one 16-byte load per lane covers two steps -- and indices as (lane,
// step) quads -- one 16-byte load per lane covers the four steps.  A warp
// issues 4 stream loads per epoch (2 value, 1 index, 1 base quad) instead of
// 9, so fewer L1 requests carry the same bytes.
//
// NA: x gathers L1::no_allocate (SB handles: a panel's gathers rarely revisit
// a line across groups); XS: x split over two buffers at x_split (world > 1:
// interior | gathered border).
// CHK (spmv_options_t.debug_checks): every y slot and x column is bounds-
// checked and every y update stamps its slot with the epoch (atomicExch in
// shared memory), counting a row updated twice within one epoch -- the
// planner's race-freedom invariant -- into A.dbg (compute-sanitizer is not
// available on this GPU pool).
template <bool NA, bool XS, bool CHK>
__global__ void __launch_bounds__(kT, 1) spmv_panel_kernel(const PnArgs A) {
    {   // one panel per CTA
        const int p = blockIdx.x;
        constexpr int kD = kDefD;                            // steps (groups) in flight per warp
        constexpr int kGD = 4;                               // gathers issued this many steps ahead
        // the ring is refilled four slots at a time after the last step of a warp's
        // epoch, so kD - 3..kD steps are loaded ahead; a gather needs its step's
        // index loaded: kGD <= kD - 4
        static_assert(kPnB == 4 && kD % 4 == 0 && kGD >= 1 && kGD <= kD - 4, "ring geometry");
        extern __shared__ __align__(16) double ys[];
        const PnPanel d = A.panel[p];
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        unsigned long long* const stp = A.stamps ? A.stamps + (int64_t)p * 8 : nullptr;
        if (stp && tid == 0) {
            uint32_t sm;
            unsigned long long gt;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
            stp[0] = sm;
            stp[1] = gt;
            stp[3] = clock64();
        }
        const uint64_t pol = pol_evict_first();
        const uint64_t polx = pol_evict_last();   // x is the reused operand
        constexpr int PF = kPF;
        const int T = d.ne * kPnB;                       // steps per warp

        double rv[kD];
        uint32_t ri[kD];
        int32_t rb[kD];
        double rx[kGD];
        // running stream pointers: the warp's block of the next epoch to load
        // (the stream is padded by kPnPadGroups groups, so the ring may read
        // ahead past the panel's last epoch without bounds checks)
        const int64_t blk0 = (int64_t)d.g0 * 32 + warp * 128;
        const double* vp = A.gval + blk0 + lane * 2;
        const uint32_t* ip = A.gidx + blk0 + lane * 4;
        const int4* bp = reinterpret_cast<const int4*>(A.gbase4 + d.g0) + warp;
        auto load4 = [&](int u) {   // the next epoch's four steps into ring slots u..u+3
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                         : "=d"(rv[u]), "=d"(rv[u + 1]) : "l"(vp), "l"(pol));
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                         : "=d"(rv[u + 2]), "=d"(rv[u + 3]) : "l"(vp + 64), "l"(pol));
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                         : "=r"(ri[u]), "=r"(ri[u + 1]), "=r"(ri[u + 2]), "=r"(ri[u + 3]) : "l"(ip), "l"(pol));
            asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(rb[u]), "=r"(rb[u + 1]), "=r"(rb[u + 2]), "=r"(rb[u + 3]) : "l"(bp));
            vp += kPnWarps * 128;
            ip += kPnWarps * 128;
            bp += kPnWarps;
        };
        auto gather_col = [&](uint32_t c) -> double {
            if (CHK && (int64_t)c >= A.x_cols) {
                atomicAdd(A.dbg + 1, 1ull);
                c = 0;
            }
            const double* xa = !XS ? A.x_lo + c
                                   : (int32_t)c < A.x_split ? A.x_lo + c : A.x_hi + (c - (uint32_t)A.x_split);
            return XS ? ld_x_co(xa, polx) : NA ? ld_x_na(xa, polx) : ld_x(xa, polx);
        };
        auto gather = [&](uint32_t i, int32_t b) -> double {
            // unconditional: a padding lane reads x[base] (valid) and adds 0 * x into
            // the scratch y slot -- a predicated-off load behind a branch made the
            // warp wait for the gather at the branch (measured 1.6x slower)
            // XS: x is split at x_split between two buffers (world > 1: interior |
            // gathered border); world 1 reads one vector (no select per gather)
            // column = base + delta (non-negative, < 2^31): one unsigned 32-bit add
            // and one wide multiply-add form the address
            return gather_col((uint32_t)b + (i & kDeltaMask));
        };
        // a4 (world > 1, P2P exchange): the border x(C_B) of this apply may
        // still be in flight over NVLink while the interior epochs run.  A
        // gather is issued one epoch ahead of its step, so the CTA waits for
        // every peer's ready flag at the end of epoch bepoch - 2 (before the
        // first border gather), thread 0 polling with acquire loads, the rest
        // at the epoch barrier.  Bounded: a timeout counts in *err, no hang.
        const bool must_wait = XS && A.ready != nullptr && d.bepoch < d.ne;
        auto border_wait = [&]() {
            if (tid == 0) {
                for (int q = 0; q < A.world; ++q) {
                    if (q == A.self) continue;
                    uint32_t it = 0;
                    while ((int32_t)(ld_acquire_sys(A.ready + q) - A.seq) < 0) {
                        __nanosleep(128);
                        if (++it > (1u << 25)) {   // ~ seconds: the peer is gone
                            atomicAdd(A.err, 1);
                            if (A.herr) *reinterpret_cast<volatile int32_t*>(A.herr) = 1;
                            break;
                        }
                    }
                }
            }
        };
        // L2 prefetch of the panel's group stream kPF epochs ahead (one bulk
        // prefetch per array per epoch, issued by thread 0): the register ring
        // then waits for L2, not HBM, latency -- the x gathers depend on the
        // loaded indices, so their distance is what bounds the pipeline.
        // Past the panel's last epoch it prefetches the head of the panel's far
        // stream (the phase after the epochs).
        auto prefetch_far = [&](int s0) {   // far steps [s0, s0 + kPnFarRing) into L2
            if (tid != 0 || s0 >= d.fs) return;
            const int64_t b = ((int64_t)d.fb + (int64_t)s0 * NW) * 32;
            constexpr uint32_t n = kPnFarRing * NW * 32;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.fval + b), "r"(n * 8) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.fcol + b), "r"(n * 4) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.fslot + b), "r"(n * 2) : "memory");
        };
        auto prefetch_epoch = [&](int e) {
            if (tid != 0) return;
            if (e >= d.ne) {
                if (e == d.ne) {   // the epilogue's slot map of the panel's rows (16-byte granules)
                    const uintptr_t a0 = reinterpret_cast<uintptr_t>(A.row2slot + d.row0) & ~uintptr_t(15);
                    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(A.row2slot + d.row0 + d.nrows) + 15) & ~uintptr_t(15);
                    if (a1 > a0)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
                }
                if (e - d.ne < 2) prefetch_far((e - d.ne) * kPnFarRing);
                return;
            }
            const int64_t g = (int64_t)d.g0 + (int64_t)e * kPnEpoch;
            // normal priority: an evict_first prefetch is the first victim of the next one
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gval + g * 32), "r"(kPnEpoch * 32 * 8)
                         : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gidx + g * 32), "r"(kPnEpoch * 32 * 4)
                         : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.gbase4 + g), "r"(kPnEpoch * 4) : "memory");
        };
        {
            for (int e = 0; e < PF; ++e) prefetch_epoch(e);
        }
    #pragma unroll
        for (int u = 0; u < kD; u += 4) load4(u);
        // the ring's first loads are in flight while the CTA zeroes its y slots
        // and copies the fold lists (C4: the prologue was 3.9 % of a CTA's clocks)
        for (int i = tid; i < ((d.nslots + 15) & ~15); i += kT) ys[i] = 0.0;   // the panel's y slots
        // virtual-row slot lists of the panel's split rows, copied to shared memory
        // once (the epilogue folds them)
        uint16_t* ssl = reinterpret_cast<uint16_t*>(ys + A.max_rows + 16);
        int32_t* sdesc = reinterpret_cast<int32_t*>(ssl + ((A.max_sslots + 7) & ~7));   // (first, count, row) per split row
        for (int i = tid; i < d.sslot_n; i += kT) ssl[i] = A.split_slots[d.sslot0 + i];
        for (int i = tid; i < d.split_n; i += kT) {
            const int e = d.split_off + i;
            sdesc[3 * i] = A.split_first[e] - d.sslot0;
            sdesc[3 * i + 1] = A.split_cnt[e];
            sdesc[3 * i + 2] = A.split_row[e];
        }
        int32_t* stamp = sdesc + 3 * A.max_split_n;   // CHK only: epoch + 1 of each slot's last update
        if (CHK)
            for (int i = tid; i < A.max_rows + 16; i += kT) stamp[i] = 0;
        __syncthreads();
        if (stp && tid == 0) stp[4] = clock64();

        if (must_wait && d.bepoch == 0) {
            border_wait();
            __syncthreads();
        }
    #pragma unroll
        for (int u = 0; u < kGD; ++u) rx[u] = gather(ri[u], rb[u]);
        if (must_wait && d.bepoch == 1) {
            border_wait();
            __syncthreads();
        }

        auto step = [&](int u, int t) {   // consume ring slot u (compile-time) of step t
            const uint32_t i = ri[u];
            // padding lanes carry the scratch slot (host upload), value 0
            const int r = (int)(i >> kPnDeltaBits);
            if (CHK) {
                if (r >= A.max_rows + 16) {
                    atomicAdd(A.dbg + 0, 1ull);
                    return;
                }
                if (r < A.max_rows) {
                    const int ep = t / kPnB + 1;
                    if (atomicExch(stamp + r, ep) == ep) atomicAdd(A.dbg + 2, 1ull);
                }
            }
            ys[r] = fma(rv[u], rx[u % kGD], ys[r]);
        };
        auto epoch_end = [&](int t) {
            if (must_wait && t / kPnB + 2 == d.bepoch) border_wait();
            __syncthreads();
            prefetch_epoch(t / kPnB + PF);
        };
        // whole ring turns without bounds checks: loads and gathers past the
        // panel's end read the next panel's (or the pad's) valid stream
        int t0 = 0;
        for (; t0 + kD <= T; t0 += kD) {
    #pragma unroll
            for (int u = 0; u < kD; ++u) {
                step(u, t0 + u);
                // after the warp's last step of an epoch: refill its four slots with
                // the steps kD later
                if (u % 4 == 3) load4(u - 3);
                rx[u % kGD] = gather(ri[(u + kGD) % kD], rb[(u + kGD) % kD]);
                if (u % kPnB == kPnB - 1) epoch_end(t0 + u);   // epoch boundary
            }
        }
        // the last T - t0 (0, 4 or 8) steps are already in the ring
    #pragma unroll
        for (int u = 0; u < kD - 4; ++u) {
            if (t0 + u >= T) break;
            step(u, t0 + u);
            if (u + kGD < kD) rx[u % kGD] = gather(ri[(u + kGD) % kD], rb[(u + kGD) % kD]);
            if (u % kPnB == kPnB - 1) epoch_end(t0 + u);
        }
        // far phase (plan_panel.cpp): each lane sums its runs of far nonzeros in a
        // register and adds a run's sum to its y slot at the run's last entry.
        // A slot belongs to one lane and every epoch is done (the last epoch
        // barrier), so nothing races and no barrier is needed until the
        // epilogue's.  Loads kPnFarRing steps ahead, gathers kFG ahead.
        if (stp && tid == 0) stp[7] = clock64();
        if (d.fs > 0) {
            if (XS && A.ready != nullptr && d.bepoch >= d.ne) {   // no border epoch waited for the exchange
                border_wait();
                __syncthreads();
            }
            constexpr int FR = kPnFarRing, kFG = 4;
            static_assert(kFG < FR, "far ring geometry");
            const int64_t fstep = (int64_t)NW * 32;
            const int64_t f0 = ((int64_t)d.fb + warp) * 32 + lane;
            double fv[FR], fx[kFG];
            uint32_t fc[FR], fsl[FR];
            auto fload = [&](int u, int st) {
                const int64_t at = f0 + (int64_t)st * fstep;
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                             : "=d"(fv[u]) : "l"(A.fval + at), "l"(pol));
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                             : "=r"(fc[u]) : "l"(A.fcol + at), "l"(pol));
                asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;"
                             : "=r"(fsl[u]) : "l"(A.fslot + at), "l"(pol));
            };
    #pragma unroll
            for (int u = 0; u < FR; ++u) fload(u, u);
    #pragma unroll
            for (int u = 0; u < kFG; ++u) fx[u] = gather_col(fc[u]);
            double acc = 0.0;
            for (int s0 = 0; s0 < d.fs; s0 += FR) {
                prefetch_far(s0 + 2 * FR);
    #pragma unroll
                for (int u = 0; u < FR; ++u) {
                    acc = fma(fv[u], fx[u % kFG], acc);
                    const uint32_t sl = fsl[u];
                    if (sl & kPnFarLast) {
                        const int r = (int)(sl & (kPnFarLast - 1));
                        if (CHK && r >= A.max_rows) {
                            atomicAdd(A.dbg + 0, 1ull);
                        } else {
                            ys[r] += acc;
                        }
                        acc = 0.0;
                    }
                    fload(u, s0 + u + FR);
                    fx[u % kFG] = gather_col(fc[(u + kFG) % FR]);
                }
            }
        }
        // epilogue: y[row] = ys[slot(row)].  The slot loads are batched 16 per
        // thread (clamped addresses, no branch) and the first batch is issued
        // before the barrier, so their latency is not paid once per row.
        constexpr int EB = 32;   // slot loads per thread and batch: panels of <= 16 K rows in one batch
        uint16_t sl[EB];
        const uint16_t* r2s = A.row2slot + d.row0;
        const int nrl = d.nrows;
        auto load_slots = [&](int i0) {
    #pragma unroll
            for (int k = 0; k < EB; ++k) sl[k] = r2s[min(i0 + k * kT, nrl - 1)];
        };
        load_slots(tid);
        __syncthreads();
        if (stp && tid == 0) stp[5] = clock64();

        // DB across GPUs: a panel of border-row temporaries writes them to y_hi
        const bool tpanel = d.row0 >= A.y_split;
        double* const yb = tpanel ? A.y_hi - A.y_split : A.y;
        double mx = 0.0;
        for (int i0 = tid; i0 < nrl; i0 += EB * kT) {
            if (i0 != tid) load_slots(i0);
    #pragma unroll
            for (int k = 0; k < EB; ++k) {
                const int i = i0 + k * kT;
                if (i < nrl && sl[k] < 0x8000) {        // split rows: below
                    if (CHK && sl[k] >= A.max_rows) {
                        atomicAdd(A.dbg + 0, 1ull);
                        continue;
                    }
                    const double v = ys[sl[k]];
                    yb[d.row0 + i] = v;
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
            yb[d.row0 + sdesc[3 * k + 2]] = v;
            mx = fmax(mx, fabs(v));
        }
        for (int k = d.split_short + warp; k < d.split_n; k += NW) {
            const int f = sdesc[3 * k], c = sdesc[3 * k + 1];
            double v = 0.0;
            for (int j = lane; j < c; j += 32) v += ys[ssl[f + j]];
    #pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane == 0) {
                yb[d.row0 + sdesc[3 * k + 2]] = v;
                mx = fmax(mx, fabs(v));
            }
        }
        if (A.maxabs_slots && !tpanel) {
    #pragma unroll
            for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            if (lane == 0 && mx > 0.0)
                atomicMax(A.maxabs_slots + ((p * NW + warp) & (kMaxSlots - 1)) * kSlotStride,
                          (unsigned long long)__double_as_longlong(mx));
        }
        if (stp) {
            __syncthreads();
            if (tid == 0) {
                unsigned long long gt;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
                stp[6] = clock64();
                stp[2] = gt;
            }
        }
    }
}

}  // namespace

namespace {

template <bool CHK>
cudaError_t launch_panel_t(const PnArgs& a, cudaStream_t s, int64_t smem) {
    // the opt-in shared-memory limit is a per-device function attribute: set
    // it once per device (a process may hold handles on several GPUs)
    static std::atomic<int> ready[kMaxDevices];
    int dev = 0;
    cudaError_t r = cudaGetDevice(&dev);
    if (r != cudaSuccess) return r;
    const int di = dev < kMaxDevices ? dev : kMaxDevices - 1;
    if (!ready[di].load(std::memory_order_acquire) || dev >= kMaxDevices) {
        const int smax = (int)kPnSmemMax;
        for (const void* k : {(const void*)spmv_panel_kernel<false, false, CHK>, (const void*)spmv_panel_kernel<false, true, CHK>,
                              (const void*)spmv_panel_kernel<true, false, CHK>, (const void*)spmv_panel_kernel<true, true, CHK>})
        {
            if ((r = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smax)) != cudaSuccess)
                return r;
#ifdef SPMV_PN_CARVEOUT   // build-time experiment: shared-memory carveout hint (% of the maximum)
            if ((r = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, SPMV_PN_CARVEOUT)) !=
                cudaSuccess)
                return r;
#endif
        }
        ready[di].store(1, std::memory_order_release);
    }
    const bool xs = a.x_split != INT32_MAX;
    if (a.gather_na) {
        if (xs) spmv_panel_kernel<true, true, CHK><<<a.n_panels, kT, smem, s>>>(a);
        else spmv_panel_kernel<true, false, CHK><<<a.n_panels, kT, smem, s>>>(a);
    } else {
        if (xs) spmv_panel_kernel<false, true, CHK><<<a.n_panels, kT, smem, s>>>(a);
        else spmv_panel_kernel<false, false, CHK><<<a.n_panels, kT, smem, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_panel(const PnArgs& a, cudaStream_t s) {
    if (a.n_panels <= 0) return cudaSuccess;
    // only the panel's y (and split-row fold lists) in shared memory: the rest
    // of the 256 KB L1/shared array stays L1, which holds the loads in flight
    int64_t smem = panel_smem_bytes(a.max_rows, a.max_sslots, a.max_split_n);
    if (a.dbg) smem += 4 * (int64_t)(a.max_rows + 16);   // the checked variant's epoch stamps
    if (smem > kPnSmemMax) return cudaErrorInvalidValue;   // the planner never builds such a panel
    return a.dbg ? launch_panel_t<true>(a, s, smem) : launch_panel_t<false>(a, s, smem);
}

// Loads this file's kernels now (cudaFuncGetAttributes forces the lazy loader):
// a kernel first launched while a peer rank's kernel spins on an exchange flag
// would otherwise load its module then, and a module load can wait for the
// running kernels -- the spinning one included (see host.cpp).
cudaError_t preload_kernels_panel() {
    cudaFuncAttributes fa;
    for (const void* k : {(const void*)spmv_panel_kernel<false, false, false>, (const void*)spmv_panel_kernel<false, true, false>,
                          (const void*)spmv_panel_kernel<true, false, false>, (const void*)spmv_panel_kernel<true, true, false>,
                          (const void*)spmv_panel_kernel<false, false, true>, (const void*)spmv_panel_kernel<false, true, true>,
                          (const void*)spmv_panel_kernel<true, false, true>, (const void*)spmv_panel_kernel<true, true, true>}) {
        const cudaError_t e = cudaFuncGetAttributes(&fa, k);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace spmvb
