// host.cpp -- the C ABI of include/spmv.h: ingest, validation, permutation,
// planning, device upload and apply orchestration.  The world > 1 exchange
// lives in exchange.cpp, the test hooks of include/spmv_test.h in
// test_hooks.cpp.
//
// Paper: Akbudak, Kayaaslan & Aykanat, arXiv 1203.2739 (P:Lnn = PAPER.md line).
//   a1 ingest  : A^ = P_r A P_c, old->new arrays
//   a2 plan    : SB/DB envelope of Eq.(1)/(5); panels / row
//                tiles; split segments of Pi; shard of the row-slice
//                decomposition y_k <- R_k x and, for DB, of the split
//                (part k = block k's products)
//   a3/a4      : x preparation; border-x exchange (coupling columns are the only
//                input shared between row slices) -- exchange.cpp
//   a5-a7      : one SpMxV kernel launch (panel.cu; rowtile.cu fallback)
//   a8         : fused multiple-SpMxV
//   a9         : max-abs and x-update glue for the power iterations
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>
#include <omp.h>

#include "exchange.h"
#include "handle.h"

namespace spmvb {

thread_local std::string g_last_error;

spmv_status_t fail(spmv_status_t s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

template <class T>
spmv_status_t dalloc(spmv_plan_s* h, T** out, size_t count) {
    void* p = nullptr;
    size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(SPMV_ERR_INTERNAL, "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
    }
    h->allocs.push_back(p);
    *out = static_cast<T*>(p);
    return SPMV_OK;
}

template <class T>
spmv_status_t upload(spmv_plan_s* h, T** out, const T* src, size_t count, size_t alloc_count) {
    spmv_status_t s = dalloc(h, out, std::max(count, alloc_count));
    if (s) return s;
    if (alloc_count > count) CUDA_TRY(cudaMemset(*out, 0, std::max(count, alloc_count) * sizeof(T)));
    if (count) CUDA_TRY(cudaMemcpy(*out, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return SPMV_OK;
}
void dfree(spmv_plan_s* h, void* p) {
    if (!p) return;
    for (size_t i = 0; i < h->allocs.size(); ++i)
        if (h->allocs[i] == p) {
            cudaFree(p);
            h->allocs.erase(h->allocs.begin() + (int64_t)i);
            return;
        }
}
template spmv_status_t dalloc<double>(spmv_plan_s*, double**, size_t);
template spmv_status_t dalloc<int32_t>(spmv_plan_s*, int32_t**, size_t);
template spmv_status_t dalloc<char>(spmv_plan_s*, char**, size_t);
template spmv_status_t dalloc<unsigned long long>(spmv_plan_s*, unsigned long long**, size_t);
template spmv_status_t upload<int32_t>(spmv_plan_s*, int32_t**, const int32_t*, size_t, size_t);
template spmv_status_t upload<uint16_t>(spmv_plan_s*, uint16_t**, const uint16_t*, size_t, size_t);
template spmv_status_t upload<int4>(spmv_plan_s*, int4**, const int4*, size_t, size_t);
template spmv_status_t upload<XsCta>(spmv_plan_s*, XsCta**, const XsCta*, size_t, size_t);

void free_plan(spmv_plan_s* h) {
    if (!h) return;
    DeviceGuard g(h->device);
    cudaDeviceSynchronize();
    xchg_release(h);
    for (void* p : h->allocs) cudaFree(p);
    h->allocs.clear();
    if (h->d_stamps) cudaFree(h->d_stamps);
    if (h->comm) ncclCommDestroy(h->comm);
    h->comm = nullptr;
    h->magic = 0;
    delete h;
}

bool valid(spmv_handle_t h) { return h && h->magic == kMagic; }

}  // namespace spmvb

using namespace spmvb;

namespace {

// Row-tile plan (rowtile.cu): greedy over rows; a tile holds whole rows with
// <= kTileNnz nonzeros and <= kTileRows rows; a longer row is a tile of its
// own (CTA-per-row).  Tiles never cross an SB block boundary (cuts), and the
// capacity test assumes the worst 16-byte alignment of the tile's first
// nonzero, so tiles -- and every row's summation order -- do not depend on
// where the rank's local CSR starts (identical at every world size).
void plan_tiles(const std::vector<int64_t>& rp, int64_t m_loc, const std::vector<int64_t>& cuts,
                std::vector<int32_t>& tile_row, int64_t& n_long) {
    tile_row.clear();
    n_long = 0;
    size_t ci = 0;
    int64_t r = 0;
    tile_row.push_back(0);
    while (r < m_loc) {
        while (ci < cuts.size() && cuts[ci] <= r) ++ci;
        const int64_t lim = ci < cuts.size() ? std::min<int64_t>(cuts[ci], m_loc) : m_loc;
        const int64_t a0 = rp[r];
        if (rp[r + 1] - a0 + 3 > kTileNnz) {
            ++r;
            ++n_long;
        } else {
            int64_t e = r;
            while (e < lim && e - r < kTileRows && rp[e + 1] - a0 + 3 <= kTileNnz) ++e;
            r = e;
        }
        tile_row.push_back((int32_t)r);
    }
}

spmv_options_t default_options() {
    spmv_options_t o;
    memset(&o, 0, sizeof o);
    o.struct_size = (int32_t)sizeof o;
    return o;
}

}  // namespace

namespace spmvb {

// The panel plan's layout decisions for one rank (pure host logic, shared by
// plan_pn and the spmv_pn_shard_hash test hook): its row ranges (SB/DB
// blocks, else all rows), their interior column ranges (rotation, x
// prefetch), the panel size target and whole-wave count, the x split, and --
// for SB handles without a split -- each range's panel count from the global
// per-block slot counts, so a block's panels do not depend on the GPU count.
PnSetup pn_setup(int kind, int world, int64_t row_begin, int64_t m_blk, int64_t m_loc, int64_t x_int_begin,
                 int64_t x_int_len, int64_t n, const std::vector<int64_t>& rbp, const std::vector<int64_t>& cbp,
                 const std::vector<int64_t>& blk_slots, const std::vector<int64_t>& rp,
                 const std::vector<int32_t>* part, int64_t sms, int64_t rows_opt) {
    PnSetup S;
    S.sms = sms;
    const int K = (int)rbp.size() - 2;
    const int64_t R0 = row_begin, R1 = row_begin + m_blk;
    const int64_t q0 = world > 1 ? x_int_begin : 0;
    if (kind == SPMV_SB || (kind == SPMV_DB && world > 1)) {
        for (int k = 0; k < K; ++k) {
            const int64_t a = std::max(rbp[k], R0), b = std::min(rbp[k + 1], R1);
            if (b > a) {
                S.ranges.push_back({a - R0, b - R0});
                S.xcols.push_back({cbp[k] - q0, cbp[k + 1] - q0});
            }
        }
        if (m_loc > m_blk) {   // DB world > 1: the border-row temporaries' rows
            S.ranges.push_back({m_blk, m_loc});
            S.xcols.push_back({0, std::max<int64_t>(x_int_len, 1)});
        }
    } else {   // no SB structure (or DB at world 1): panels of consecutive rows, no x prefetch
        S.ranges.push_back({0, m_loc});
    }
    // the global per-block counts (SB, no split) decide the cuts, else this rank's rows
    S.global = kind == SPMV_SB && !part && K > 0 && (int)blk_slots.size() == K;
    int64_t total_slots = 0;
    if (S.global)
        for (int64_t v : blk_slots) total_slots += v;
    else
        total_slots = panel_total_slots(rp, m_loc, part);
    // panels: about kPnRowsTarget slots, their count a multiple of the SM
    // count when possible (whole waves of one CTA per SM)
    S.target = kPnRowsTarget;
    for (int64_t k = 1; k <= 4096; ++k) {
        const int64_t r = (total_slots + sms * k - 1) / (sms * k);
        if (r <= kPnRowsTarget) {
            S.target = r;
            S.waves = k;
            break;
        }
    }
    if (S.target < 1024) {
        S.target = 1024;
        S.waves = 0;
    }
    if (rows_opt > 0) {   // spmv_options_t.panel_rows
        S.target = rows_opt;
        S.waves = 0;
    }
    // groups never mix interior and border columns at world > 1 (two x
    // buffers); SB plans keep the same rule at world 1 (C_B starts at
    // cbp[K]) so the groups -- and every row's summation order -- are the
    // same on any number of GPUs
    S.xs = world > 1 ? x_int_len : (kind == SPMV_SB ? cbp[K] : INT32_MAX);
    if (S.global) {
        const std::vector<int64_t> np_all = panel_counts(blk_slots, S.target, S.waves * sms);
        for (int k = 0; k < K; ++k)
            if (std::min(rbp[k + 1], R1) > std::max(rbp[k], R0)) S.range_panels.push_back(np_all[k]);
    }
    return S;
}

}  // namespace spmvb

namespace {

// Builds and uploads the column-sorted panel kernel's plan (plan_panel.cpp).
// Leaves the plan empty (the caller falls back to row tiles) when it would be
// poor (> 25 % padding, unless forced) or cannot be built.
spmv_status_t plan_pn(spmv_plan_s* h, PanelPlan& pl, const std::vector<int64_t>& rp, const std::vector<int32_t>& pcol,
                      const std::vector<double>& pval, const std::vector<int64_t>& rbp,
                      const std::vector<int64_t>& cbp, const std::vector<int32_t>* part, bool forced,
                      std::string* why_out = nullptr) {
    const PnSetup S = pn_setup(h->kind, h->world, h->row_begin, h->m_blk, h->m_loc, h->x_int_begin, h->x_int_len, h->n,
                               rbp, cbp, h->blk_slots, rp, part, kernel_num_sms(), h->opt.panel_rows);
    std::vector<PnPanelData> pd;
    PnPlanStats st;
    std::string why;
    if (!plan_panel(rp, pcol, pval, S.ranges, S.xs, S.target, pd, st, why, S.xcols.empty() ? nullptr : &S.xcols,
                    S.sms, part, S.waves * S.sms, S.global ? &S.range_panels : nullptr)) {
        if (why_out) *why_out = why;
        return SPMV_OK;
    }
    if (st.entries != h->nnz_loc)
        return fail(SPMV_ERR_INTERNAL, "panel plan lost nonzeros (%lld of %lld)", (long long)st.entries,
                    (long long)h->nnz_loc);
    if (!forced && st.pads > st.entries / 4) {   // > 25 % padding: the row-tile kernel is cheaper
        if (why_out) *why_out = "padding above 25 %";
        return SPMV_OK;
    }
    const int64_t P = (int64_t)pd.size(), G = st.groups;
    std::vector<PnPanel> desc(P);
    int32_t max_rows = 0, max_ss = 0, max_sn = 0;
    int64_t FB = 0;   // far-stream blocks (32 entries) of all panels
    for (int64_t p = 0; p < P; ++p) {
        pd[p].desc.fb = (int32_t)FB;
        FB += (int64_t)pd[p].desc.fs * kPnWarps;
        if (FB >= INT32_MAX / 64) {
            if (why_out) *why_out = "far stream beyond int32 blocks";
            return SPMV_OK;
        }
        desc[p] = pd[p].desc;
        max_rows = std::max(max_rows, (pd[p].nslots + 15) & ~15);
        max_ss = std::max(max_ss, (int32_t)pd[p].split_slots.size());
        max_sn = std::max(max_sn, (int32_t)pd[p].split_first.size());
    }
    // the launch reserves the largest of each shared-memory component (panel.cu)
    if (panel_smem_bytes(max_rows, max_ss, max_sn) > kPnSmemMax) {
        if (why_out) *why_out = "panels' shared memory beyond 227 KB";
        return SPMV_OK;
    }
    spmv_status_t s;
    if ((s = upload(h, &pl.d_panel, desc.data(), P))) return s;
    // + kPnPadGroups zero groups: the kernel's register ring reads ahead past
    // the last panel's last epoch without bounds checks
    const int64_t Gp = G + kPnPadGroups;
    if ((s = dalloc(h, &pl.d_gval, Gp * 32))) return s;
    if ((s = dalloc(h, &pl.d_gidx, Gp * 32))) return s;
    if ((s = dalloc(h, &pl.d_gbase4, Gp))) return s;
    CUDA_TRY(cudaMemset(pl.d_gval + G * 32, 0, kPnPadGroups * 32 * sizeof(double)));
    CUDA_TRY(cudaMemset(pl.d_gidx + G * 32, 0, kPnPadGroups * 32 * sizeof(uint32_t)));
    CUDA_TRY(cudaMemset(pl.d_gbase4 + G, 0, kPnPadGroups * sizeof(int32_t)));
    {
        std::vector<uint16_t> r2s(std::max<int64_t>(h->m_loc, 1), 0);
        std::vector<int32_t> sf, sc, sr;
        std::vector<uint16_t> ss;
        for (int64_t p = 0; p < P; ++p) {
            std::copy(pd[p].row2slot.begin(), pd[p].row2slot.end(), r2s.begin() + pd[p].desc.row0);
            desc[p].split_off = (int32_t)sf.size();
            desc[p].nslots = pd[p].nslots;
            const int32_t base = (int32_t)ss.size();
            desc[p].split_n = (int32_t)pd[p].split_first.size();
            desc[p].split_short = pd[p].split_short;
            desc[p].sslot0 = base;
            desc[p].sslot_n = (int32_t)pd[p].split_slots.size();
            for (size_t k = 0; k < pd[p].split_first.size(); ++k) {
                sf.push_back(base + pd[p].split_first[k]);   // absolute index into split_slots
                sc.push_back(pd[p].split_cnt[k]);
                sr.push_back(pd[p].split_row[k]);
            }
            ss.insert(ss.end(), pd[p].split_slots.begin(), pd[p].split_slots.end());
        }
        if ((s = upload(h, &pl.d_r2s, r2s.data(), r2s.size()))) return s;
        if (sf.empty()) {
            sf.push_back(0);
            sc.push_back(0);
            sr.push_back(0);
            ss.push_back(0);
        }
        if ((s = upload(h, &pl.d_split_row, sr.data(), sr.size()))) return s;
        if ((s = upload(h, &pl.d_split_first, sf.data(), sf.size()))) return s;
        if ((s = upload(h, &pl.d_split_cnt, sc.data(), sc.size()))) return s;
        if ((s = upload(h, &pl.d_split_slots, ss.data(), ss.size()))) return s;
        CUDA_TRY(cudaMemcpy(pl.d_panel, desc.data(), P * sizeof(PnPanel), cudaMemcpyHostToDevice));
    }
    pl.max_rows = max_rows;
    pl.max_sslots = max_ss;
    pl.max_split_n = max_sn;
    // padding lanes: the planner's dummy index of bank b becomes the scratch
    // y slot max_rows + b (delta 0: a valid x read, times the value 0)
    const uint32_t dummy_dev = (uint32_t)pl.max_rows << kPnDeltaBits;
    // device layout of the group stream (panel.cu): per (epoch, warp) a
    // 128-entry block; values as (step pair, lane, step & 1), indices as
    // (lane, step), so 16-byte loads cover 2 / 4 of a warp's steps.  Built for
    // batches of consecutive panels in parallel (their groups are contiguous
    // on the device), one copy per batch and array.
    std::vector<double> tv;
    std::vector<uint32_t> ti;
    std::vector<int32_t> tb;
    for (int64_t p0 = 0; p0 < P;) {
        int64_t p1 = p0, ng = 0;
        while (p1 < P && (ng == 0 || ng + (int64_t)pd[p1].gbase.size() <= (int64_t(1) << 20))) ng += (int64_t)pd[p1++].gbase.size();
        const int64_t gb = pd[p0].desc.g0;
        tv.resize(ng * 32);
        ti.resize(ng * 32);
        tb.resize(ng);
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t p = p0; p < p1; ++p) {
            PnPanelData& D = pd[p];
            const int64_t off = (int64_t)D.desc.g0 - gb, n = (int64_t)D.gbase.size();
            for (int64_t g = 0; g < n; ++g) {
                const int64_t q = g / kPnWarps, w = g % kPnWarps;   // g = (e * 4 + b) * 16 + w
                const int64_t e = q / kPnB, b = q % kPnB;
                const int64_t blk = (off + (e * kPnWarps + w) * kPnB) * 32;
                for (int l = 0; l < 32; ++l) {
                    tv[blk + (b / 2) * 64 + l * 2 + (b & 1)] = D.gval[g * 32 + l];
                    const uint32_t i = D.gidx[g * 32 + l];
                    ti[blk + l * 4 + b] =
                        pn_is_dummy(i) ? dummy_dev + (((i >> kPnDeltaBits) - kPnDummyRow) << kPnDeltaBits) : i;
                }
            }
            std::copy(D.gbase4.begin(), D.gbase4.end(), tb.begin() + off);
            std::vector<double>().swap(D.gval);
            std::vector<uint32_t>().swap(D.gidx);
            std::vector<int32_t>().swap(D.gbase);
            std::vector<int32_t>().swap(D.gbase4);
        }
        if (ng) {
            CUDA_TRY(cudaMemcpy(pl.d_gval + gb * 32, tv.data(), ng * 32 * 8, cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(pl.d_gidx + gb * 32, ti.data(), ng * 32 * 4, cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(pl.d_gbase4 + gb, tb.data(), ng * 4, cudaMemcpyHostToDevice));
        }
        p0 = p1;
    }
    {   // far stream, + one ring turn of padding blocks (read-ahead past the last panel)
        const int64_t FBp = FB + (int64_t)kPnFarRing * kPnWarps;
        if ((s = dalloc(h, &pl.d_fval, FBp * 32))) return s;
        if ((s = dalloc(h, &pl.d_fcol, FBp * 32))) return s;
        if ((s = dalloc(h, &pl.d_fslot, FBp * 32))) return s;
        CUDA_TRY(cudaMemset(pl.d_fval + FB * 32, 0, kPnFarRing * kPnWarps * 32 * sizeof(double)));
        CUDA_TRY(cudaMemset(pl.d_fcol + FB * 32, 0, kPnFarRing * kPnWarps * 32 * sizeof(uint32_t)));
        CUDA_TRY(cudaMemset(pl.d_fslot + FB * 32, 0, kPnFarRing * kPnWarps * 32 * sizeof(uint16_t)));
        std::vector<uint32_t> fc;
        for (int64_t p = 0; p < P; ++p) {
            PnPanelData& D = pd[p];
            const int64_t at = (int64_t)D.desc.fb * 32, ne = (int64_t)D.fval.size();
            if (!ne) continue;
            fc.assign(D.fcol.begin(), D.fcol.end());
            CUDA_TRY(cudaMemcpy(pl.d_fval + at, D.fval.data(), ne * 8, cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(pl.d_fcol + at, fc.data(), ne * 4, cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(pl.d_fslot + at, D.fslot.data(), ne * 2, cudaMemcpyHostToDevice));
            std::vector<double>().swap(D.fval);
            std::vector<int32_t>().swap(D.fcol);
            std::vector<uint16_t>().swap(D.fslot);
        }
        pl.far = st.far;
        pl.far_blocks = FB;
    }
    pl.panels = P;
    pl.groups = G;
    pl.pad = st.pads;
    pl.gsectors = st.gsectors;
    pl.deferred = st.deferred;
    pl.ywf = st.ywf1;
    // SB/DB blocks: a panel's gathers rarely revisit an x line across groups,
    // and skipping the L1 allocation leaves the L1 to the loads in flight
    // (interleaved A/B on C5: -0.9 %); matrices without blocks (C4: band
    // columns revisited) keep allocating (+8 % without); world > 1 always
    // bypasses L1 (the border buffer is rewritten by the exchange)
    pl.gather_na = (h->kind != 0 || h->world > 1) ? 1 : 0;
    return SPMV_OK;
}

}  // namespace

extern "C" {

const char* spmv_status_string(spmv_status_t s) {
    switch (s) {
    case SPMV_OK: return "ok";
    case SPMV_ERR_USAGE: return "usage error";
    case SPMV_ERR_DATA: return "data error";
    case SPMV_ERR_INTERNAL: return "internal error";
    case SPMV_ERR_UNSUPPORTED: return "unsupported";
    }
    return "unknown status";
}

const char* spmv_last_error(void) { return g_last_error.c_str(); }

int32_t spmv_version(void) { return 20000; }

spmv_status_t spmv_nccl_unique_id(void* out, size_t len) {
    if (!out || len < sizeof(ncclUniqueId)) return fail(SPMV_ERR_USAGE, "nccl_unique_id: buffer too small");
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    memcpy(out, &id, sizeof id);
    return SPMV_OK;
}

spmv_status_t spmv_shard_plan(const spmv_blocks_t* blocks, int64_t m, int64_t n, int32_t rank, int32_t world,
                              spmv_shard_t* out) {
    if (!blocks || !out || world < 1 || rank < 0 || rank >= world) return fail(SPMV_ERR_USAGE, "shard_plan: bad arguments");
    const int K = blocks->K;
    if (K < 1 || !blocks->row_block_ptr || !blocks->col_block_ptr) return fail(SPMV_ERR_USAGE, "shard_plan: bad blocks");
    if (world > K) return fail(SPMV_ERR_UNSUPPORTED, "fewer blocks than ranks");
    const int64_t* rbp = blocks->row_block_ptr;
    const int64_t* cbp = blocks->col_block_ptr;
    if (rbp[K + 1] != m || cbp[K + 1] != n) return fail(SPMV_ERR_DATA, "block descriptor does not cover the matrix");
    const bool db = blocks->kind == SPMV_DB;
    const int64_t CB = cbp[K + 1] - cbp[K], RB = rbp[K + 1] - rbp[K];
    auto bo = [&](int k) -> int64_t {
        return blocks->border_owner_ptr ? blocks->border_owner_ptr[k] : cbp[K] + (CB * k) / K;
    };
    auto ro = [&](int k) -> int64_t {
        return blocks->row_border_owner_ptr ? blocks->row_border_owner_ptr[k] : rbp[K] + (RB * k) / K;
    };
    auto first_block = [&](int r) { return (int)((int64_t)K * r / world); };
    memset(out, 0, sizeof *out);
    out->border_begin = cbp[K];
    out->border_total = CB;
    if (world == 1) {
        out->row_begin = 0;
        out->row_end = m;
        out->x_interior_begin = 0;
        out->x_interior_len = n;
        out->x_border_begin = cbp[K];
        out->x_border_len = 0;
        out->x_local_len = n;
        out->block_begin = 0;
        out->block_end = K;
        out->y_border_begin = rbp[K];
        out->y_border_len = 0;
        out->y_local_len = m;
        return SPMV_OK;
    }
    const int b0 = first_block(rank), b1 = first_block(rank + 1);
    out->block_begin = b0;
    out->block_end = b1;
    out->row_begin = rbp[b0];
    out->row_end = rbp[b1];
    out->x_interior_begin = cbp[b0];
    out->x_interior_len = cbp[b1] - cbp[b0];
    out->x_border_begin = bo(b0);
    out->x_border_len = bo(b1) - bo(b0);
    out->x_local_len = out->x_interior_len + out->x_border_len;
    out->y_border_begin = db ? ro(b0) : rbp[K];
    out->y_border_len = db ? ro(b1) - ro(b0) : 0;
    out->y_local_len = (out->row_end - out->row_begin) + out->y_border_len;
    return SPMV_OK;
}

}  // extern "C"

namespace spmvb {

spmv_status_t create_impl(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                          const double* val, const int32_t* row_perm, const int32_t* col_perm,
                          const spmv_blocks_t* blocks, int32_t n_parts, const int32_t* part_of_nnz,
                          const spmv_dist_t* dist, const spmv_options_t* options, bool test_rank, spmv_plan_s* h) {
    // create phases (spmv_info_t.create_s): wall seconds since the previous mark
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](int k) {
        const auto now = std::chrono::steady_clock::now();
        h->create_s[k] += std::chrono::duration<double>(now - t_last).count();
        t_last = now;
    };
    // ---------------------------------------------------------- arguments
    h->opt = default_options();
    if (options) {
        const size_t sz = options->struct_size > 0 ? std::min<size_t>(options->struct_size, sizeof(spmv_options_t))
                                                   : sizeof(spmv_options_t);
        memcpy(&h->opt, options, sz);
        h->opt.struct_size = (int32_t)sizeof(spmv_options_t);
    }
    const spmv_options_t& O = h->opt;
    if (O.kernel < 0 || O.kernel > 3 || O.split_kernel < 0 || O.split_kernel > 2 || O.exchange < 0 ||
        O.exchange > 2 || O.panel_rows < 0 || O.index16 < 0 || O.index16 > 1 || O.debug_checks < 0 ||
        O.debug_checks > 1 || O.retain_csr < 0 || O.retain_csr > 1)
        return fail(SPMV_ERR_USAGE, "bad options");
    if (m < 0 || n < 0 || nnz < 0) return fail(SPMV_ERR_USAGE, "negative dimension");
    if (!row_ptr) return fail(SPMV_ERR_USAGE, "row_ptr is NULL");
    if (nnz > 0 && (!col_idx || !val)) return fail(SPMV_ERR_USAGE, "col_idx/val is NULL");
    if (n_parts < 0 || (n_parts > 0 && !part_of_nnz)) return fail(SPMV_ERR_USAGE, "bad split arguments");
    if (n_parts > kMaxParts) return fail(SPMV_ERR_UNSUPPORTED, "more than %d split parts", kMaxParts);
    if (m > INT32_MAX - 1 || n > INT32_MAX - 1) return fail(SPMV_ERR_UNSUPPORTED, "dimension beyond int32");
    const int world = dist ? dist->world : 1;
    const int rank = dist ? dist->rank : 0;
    if (dist && (world < 1 || rank < 0 || rank >= world || (!test_rank && world > 1 && !dist->nccl_unique_id)))
        return fail(SPMV_ERR_USAGE, "bad dist descriptor");
    h->test_rank = test_rank;
    if (world > 1 && (!blocks || (blocks->kind != SPMV_SB && blocks->kind != SPMV_DB)))
        return fail(SPMV_ERR_UNSUPPORTED, "world > 1 needs an SB or DB block descriptor");
    if (world > 1 && blocks->kind == SPMV_DB && n_parts != 0 && n_parts != blocks->K)
        return fail(SPMV_ERR_UNSUPPORTED, "DB across GPUs: the split must have one part per block (n_parts == K)");
    h->rank = rank;
    h->world = world;
    h->m = m; h->n = n; h->nnz = nnz;
    h->n_parts = n_parts;
    h->has_perm = row_perm || col_perm;
    if (dist) {
        h->device = dist->device;
    } else if (cudaGetDevice(&h->device) != cudaSuccess) {   // no GPU: the host-side validation still runs,
        cudaGetLastError();                                  // the first CUDA call fails (INTERNAL)
        h->device = -1;
    }

    // ------------------------------------------------ CSR structure (a1)
    if (row_ptr[0] != 0 || row_ptr[m] != nnz) return fail(SPMV_ERR_DATA, "row_ptr[0] != 0 or row_ptr[m] != nnz");
    {
        std::atomic<int> bad{0};
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < m; ++i)
            if (row_ptr[i + 1] < row_ptr[i]) bad = 1;
        if (bad) return fail(SPMV_ERR_DATA, "row_ptr not nondecreasing");
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < nnz; ++t)
            if (col_idx[t] < 0 || (int64_t)col_idx[t] >= n) bad = 2;
        if (bad) return fail(SPMV_ERR_DATA, "column index out of range");
        if (n_parts > 0) {
#pragma omp parallel for schedule(static)
            for (int64_t t = 0; t < nnz; ++t)
                if (part_of_nnz[t] < 0 || part_of_nnz[t] >= n_parts) bad = 3;
            if (bad) return fail(SPMV_ERR_DATA, "part id outside [0, K)");
        }
    }
    // permutations must be bijections
    std::vector<int32_t> row_inv(m), col_inv(n);
    for (int pass = 0; pass < 2; ++pass) {
        const int32_t* p = pass ? col_perm : row_perm;
        const int64_t len = pass ? n : m;
        std::vector<int32_t>& inv = pass ? col_inv : row_inv;
        if (!p) {
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < len; ++i) inv[i] = (int32_t)i;
            continue;
        }
        std::fill(inv.begin(), inv.end(), -1);
        for (int64_t i = 0; i < len; ++i) {
            if (p[i] < 0 || (int64_t)p[i] >= len || inv[p[i]] != -1)
                return fail(SPMV_ERR_DATA, "%s permutation is not a bijection", pass ? "column" : "row");
            inv[p[i]] = (int32_t)i;
        }
    }

    // ------------------------------------------------ block descriptor (a2)
    int K = 0;
    std::vector<int64_t> rbp, cbp;
    if (blocks) {
        K = blocks->K;
        if ((blocks->kind != SPMV_SB && blocks->kind != SPMV_DB) || K < 1 || !blocks->row_block_ptr ||
            !blocks->col_block_ptr)
            return fail(SPMV_ERR_USAGE, "bad block descriptor");
        rbp.assign(blocks->row_block_ptr, blocks->row_block_ptr + K + 2);
        cbp.assign(blocks->col_block_ptr, blocks->col_block_ptr + K + 2);
        if (rbp[0] != 0 || rbp[K + 1] != m || cbp[0] != 0 || cbp[K + 1] != n)
            return fail(SPMV_ERR_DATA, "block descriptor does not cover the matrix");
        for (int k = 0; k <= K; ++k)
            if (rbp[k + 1] < rbp[k] || cbp[k + 1] < cbp[k])
                return fail(SPMV_ERR_DATA, "block descriptor not nondecreasing");
        if (blocks->kind == SPMV_SB && rbp[K] != rbp[K + 1])
            return fail(SPMV_ERR_DATA, "SB form with a non-empty row border");
        h->kind = blocks->kind;
        h->border_begin = cbp[K];
        h->border_total = cbp[K + 1] - cbp[K];
        for (int pass = 0; pass < 2; ++pass) {
            const int64_t* q = pass ? blocks->row_border_owner_ptr : blocks->border_owner_ptr;
            if (!q) continue;
            const int64_t lo = pass ? rbp[K] : cbp[K], hi = pass ? rbp[K + 1] : cbp[K + 1];
            if (q[0] != lo || q[K] != hi) return fail(SPMV_ERR_DATA, "border owner pointers do not cover the border");
            for (int k = 0; k < K; ++k)
                if (q[k + 1] < q[k]) return fail(SPMV_ERR_DATA, "border owner pointers not nondecreasing");
        }
    }
    const bool db_dist = world > 1 && h->kind == SPMV_DB;

    // --------------------------------------------------- shard
    spmv_shard_t sh;
    if (blocks) {
        spmv_status_t ss = spmv_shard_plan(blocks, m, n, rank, world, &sh);
        if (ss) return ss;
    } else {
        memset(&sh, 0, sizeof sh);
        sh.row_end = m;
        sh.x_interior_len = n;
        sh.x_local_len = n;
        sh.y_local_len = m;
    }
    if (world > 1) {
        h->bord_off.resize(world);
        h->bord_cnt.resize(world);
        for (int r = 0; r < world; ++r) {
            spmv_shard_t o;
            spmv_shard_plan(blocks, m, n, r, world, &o);
            h->bord_off[r] = o.x_border_begin - o.border_begin;
            h->bord_cnt[r] = o.x_border_len;
            if (h->bord_cnt[r] != h->bord_cnt[0]) h->equal_slices = false;
        }
    }
    const int64_t R0 = sh.row_begin, R1 = sh.row_end;
    h->row_begin = R0;
    h->m_blk = R1 - R0;
    h->x_int_begin = sh.x_interior_begin;
    h->x_int_len = sh.x_interior_len;
    h->x_bord_begin = sh.x_border_begin;
    h->x_bord_len = sh.x_border_len;
    h->x_local_len = sh.x_local_len;
    h->y_bord_begin = sh.y_border_begin;
    h->y_bord_len = sh.y_border_len;
    h->m_out = sh.y_local_len;

    // block of each permuted row / column (DB across GPUs: the part rule)
    auto row_block = [&](int64_t r) -> int {
        return (int)(std::upper_bound(rbp.begin(), rbp.begin() + K + 1, r) - rbp.begin()) - 1;
    };
    auto col_block = [&](int64_t c) -> int {
        return (int)(std::upper_bound(cbp.begin(), cbp.begin() + K + 1, c) - cbp.begin()) - 1;
    };
    // owner block of a border row's slice (DB)
    std::vector<int64_t> rop;
    if (h->kind == SPMV_DB) {
        rop.resize(K + 1);
        const int64_t RB = rbp[K + 1] - rbp[K];
        for (int k = 0; k <= K; ++k)
            rop[k] = blocks->row_border_owner_ptr ? blocks->row_border_owner_ptr[k] : rbp[K] + (RB * k) / K;
    }
    auto rslice_block = [&](int64_t r) -> int {
        return (int)(std::upper_bound(rop.begin(), rop.end(), r) - rop.begin()) - 1;
    };
    auto block_rank = [&](int k) -> int {   // rank owning block k: blocks [floor(K g / G), floor(K (g+1) / G))
        int g = (int)(((int64_t)k * world) / K);
        while (g + 1 < world && (int64_t)K * (g + 1) / world <= k) ++g;
        while (g > 0 && (int64_t)K * g / world > k) --g;
        return g;
    };
    const int b0 = blocks ? (int)sh.block_begin : 0, b1 = blocks ? (int)sh.block_end : 0;

    DeviceGuard dg(h->device);
    if (!dg.ok()) return fail(SPMV_ERR_INTERNAL, "cannot select device %d", h->device);
    // ---------------------------------------------- NCCL bootstrap (a4)
    if (world > 1 && !test_rank) {
        ncclUniqueId id;
        memcpy(&id, dist->nccl_unique_id, sizeof id);
        NCCL_TRY(ncclCommInitRank(&h->comm, world, id, rank));
    }

    // From here on every failure is local to this rank: it is recorded in
    // local_status and all ranks agree on the outcome at the end.
    spmv_status_t local_status = SPMV_OK;
    mark(0);   // validation, block descriptor, shard, communicator
    auto run_local = [&]() -> spmv_status_t {
        // --------------------------------------- permute the local rows (a1)
        // new row p has the entries of old row row_inv[p], columns mapped
        // through col_perm, sorted by new column; duplicates rejected (A3).
        // DB across GPUs: after the rank's block rows come its border-row
        // temporaries -- one compute row per (destination rank, own part,
        // border row) with that part's nonzeros of the row.
        const int64_t m_blk = h->m_blk;
        std::vector<int64_t> rrow;   // global permuted row of each compute row
        std::vector<int32_t> rpart;  // DB across GPUs: part of each temporary row (-1: block row)
        rrow.reserve(m_blk);
        for (int64_t p = 0; p < m_blk; ++p) rrow.push_back(R0 + p);
        // part of nonzero t (original input index) in permuted row gp, new column c
        auto part_of = [&](int64_t t, int64_t gp, int64_t c) -> int {
            if (n_parts) return part_of_nnz[t];
            const int kb = row_block(gp);
            if (kb < K) return kb;                              // block row: its block
            const int kc = c < cbp[K] ? col_block(c) : K;
            return kc < K ? kc : rslice_block(gp);              // border row: column block, else row slice
        };
        std::vector<int64_t> brow_len;   // DB: per border row and own part: nonzero count
        const int nown = b1 - b0;
        const int64_t RBn = db_dist ? rbp[K + 1] - rbp[K] : 0;
        std::atomic<int> bad_part{0};
        if (db_dist) {
            // which (border row, own part) segments exist and how long they are
            brow_len.assign(RBn * nown, 0);
#pragma omp parallel for schedule(dynamic, 256)
            for (int64_t q = 0; q < RBn; ++q) {
                const int64_t gp = rbp[K] + q, i = row_inv[gp];
                for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) {
                    const int64_t c = col_perm ? col_perm[col_idx[t]] : col_idx[t];
                    const int k = part_of(t, gp, c);
                    if (c < cbp[K] && col_block(c) != k) bad_part = 1;   // interior column of another block
                    if (k >= b0 && k < b1) brow_len[q * nown + (k - b0)]++;
                }
            }
            if (bad_part)
                return fail(SPMV_ERR_UNSUPPORTED,
                            "DB across GPUs: a border-row nonzero's part is not its interior column's block");
            // temporaries ordered (destination rank, part, row): each destination's run is contiguous
            for (int r = 0; r < world; ++r)
                for (int k = b0; k < b1; ++k)
                    for (int64_t q = 0; q < RBn; ++q) {
                        const int64_t gp = rbp[K] + q;
                        if (block_rank(rslice_block(gp)) != r || brow_len[q * nown + (k - b0)] == 0) continue;
                        rrow.push_back(gp);
                        rpart.push_back(k);
                    }
        }
        const int64_t m_loc = (int64_t)rrow.size();
        h->m_loc = m_loc;
        h->n_T = m_loc - m_blk;
        std::vector<int64_t> rp(m_loc + 1);
        rp[0] = 0;
        // row lengths in parallel (row_inv and row_ptr are random reads under a
        // hidden permutation), then the running sum
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < m_loc; ++p) {
            const int64_t i = row_inv[rrow[p]];
            rp[p + 1] = p < m_blk ? row_ptr[i + 1] - row_ptr[i]
                                  : brow_len[(rrow[p] - rbp[K]) * nown + (rpart[p - m_blk] - b0)];
        }
        for (int64_t p = 0; p < m_loc; ++p) rp[p + 1] += rp[p];
        const int64_t nnz_loc = rp[m_loc];
        h->nnz_loc = nnz_loc;
        if (nnz_loc + kPad >= INT32_MAX) return fail(SPMV_ERR_UNSUPPORTED, "shard nnz beyond int32");

        std::vector<int32_t> pcol(nnz_loc);
        std::vector<double> pval(nnz_loc);
        std::vector<int32_t> ppart;
        if (n_parts && !db_dist) ppart.resize(nnz_loc);
        {
            std::atomic<int> dup{0}, env{0};
            const bool sb_env = blocks != nullptr;
#pragma omp parallel
            {
                std::vector<int64_t> idx;
                std::vector<int32_t> key;
#pragma omp for schedule(dynamic, 2048)
                for (int64_t p = 0; p < m_loc; ++p) {
                    // A hidden permutation makes every step of row_inv -> row_ptr ->
                    // (col_idx, val) -> col_perm a cache miss (C5: 9 s of create on
                    // 16 cores): software-prefetch the chain kPfD rows apart per level
                    constexpr int64_t kPfD = 4;
                    if (p + 4 * kPfD < m_blk) __builtin_prefetch(&row_inv[rrow[p + 4 * kPfD]]);
                    if (p + 3 * kPfD < m_blk) __builtin_prefetch(&row_ptr[row_inv[rrow[p + 3 * kPfD]]]);
                    if (p + 2 * kPfD < m_blk) {
                        const int64_t i2 = row_inv[rrow[p + 2 * kPfD]];
                        const int64_t a2 = row_ptr[i2], e2 = std::min(row_ptr[i2 + 1], a2 + 64);
                        for (int64_t t = a2; t < e2; t += 16) __builtin_prefetch(&col_idx[t]);
                        for (int64_t t = a2; t < e2; t += 8) __builtin_prefetch(&val[t]);
                    }
                    if (col_perm && p + kPfD < m_blk) {
                        const int64_t i1 = row_inv[rrow[p + kPfD]];
                        const int64_t a1 = row_ptr[i1], e1 = std::min(row_ptr[i1 + 1], a1 + 64);
                        for (int64_t t = a1; t < e1; ++t) __builtin_prefetch(&col_perm[col_idx[t]]);
                    }
                    const int64_t gp = rrow[p];
                    const int64_t i = row_inv[gp];
                    const int64_t a = row_ptr[i], L = row_ptr[i + 1] - a;
                    const int64_t o = rp[p];
                    key.resize(L);
                    idx.resize(L);
                    for (int64_t t = 0; t < L; ++t) {
                        key[t] = col_perm ? col_perm[col_idx[a + t]] : col_idx[a + t];
                        idx[t] = t;
                    }
                    bool sorted = true;
                    for (int64_t t = 1; t < L; ++t)
                        if (key[t] < key[t - 1]) { sorted = false; break; }
                    if (!sorted) {
                        if (L <= 32) {   // insertion sort (stable)
                            for (int64_t t = 1; t < L; ++t) {
                                int64_t j = t;
                                const int64_t v = idx[t];
                                while (j > 0 && key[idx[j - 1]] > key[v]) { idx[j] = idx[j - 1]; --j; }
                                idx[j] = v;
                            }
                        } else {
                            std::stable_sort(idx.begin(), idx.end(),
                                             [&](int64_t u, int64_t v) { return key[u] < key[v]; });
                        }
                    }
                    for (int64_t t = 1; t < L; ++t)
                        if (key[idx[t]] == key[idx[t - 1]]) dup = 1;
                    const int kb = blocks ? row_block(gp) : 0;
                    int64_t w = o;
                    for (int64_t t = 0; t < L; ++t) {
                        const int64_t s = idx[t];
                        if (p >= m_blk) {   // a border-row temporary: only its part's nonzeros
                            if (part_of(a + s, gp, key[s]) != rpart[p - m_blk]) continue;
                        } else if (db_dist && n_parts && part_of_nnz[a + s] != kb) {
                            env = 2;        // a block row's nonzero outside its block's part
                        }
                        pcol[w] = key[s];
                        pval[w] = val[a + s];
                        if (!ppart.empty()) ppart[w] = part_of_nnz[a + s];
                        ++w;
                    }
                    if (sb_env && p < m_blk && kb < K) {   // envelope of Eq.(1)/(5)
                        for (int64_t t = 0; t < L; ++t) {
                            const int64_t c = key[t];
                            if (!((c >= cbp[kb] && c < cbp[kb + 1]) || c >= cbp[K])) { env = 1; break; }
                        }
                    }
                }
            }
            if (dup) return fail(SPMV_ERR_DATA, "duplicate (i, j) entry");
            if (env == 1) return fail(SPMV_ERR_DATA, "nonzero outside the SB/DB envelope");
            if (env == 2) return fail(SPMV_ERR_UNSUPPORTED, "DB across GPUs: part k must hold block k's rows");
        }

        mark(1);   // permutation of the local rows
        // -------------------------------------- local column ids (x layout)
        // world 1: global permuted ids.  world > 1: [interior | full C_B]: the
        // kernel reads c < x_int_len from the user's x, the rest from the
        // exchanged border buffer.
        if (world > 1) {
            const int64_t Q0 = h->x_int_begin, B0 = h->border_begin, nint = h->x_int_len;
            std::atomic<int> outside{0};
#pragma omp parallel for schedule(static)
            for (int64_t t = 0; t < nnz_loc; ++t) {
                const int64_t c = pcol[t];
                if (c < B0 && (c < Q0 || c >= Q0 + nint)) outside = 1;
                pcol[t] = (int32_t)(c >= B0 ? nint + (c - B0) : c - Q0);
            }
            if (outside) return fail(SPMV_ERR_INTERNAL, "local column outside the rank's x layout");
        }

        // ------------------------------------------------------ tiles (a2)
        std::vector<int64_t> cuts;
        if (blocks)
            for (int k = 1; k <= K; ++k)
                if (rbp[k] > R0 && rbp[k] < R1) cuts.push_back(rbp[k] - R0);
        if (m_loc > m_blk) cuts.push_back(m_blk);
        std::vector<int32_t> tile_row;
        plan_tiles(rp, m_loc, cuts, tile_row, h->n_long);
        const int64_t T = (int64_t)tile_row.size() - 1;
        h->n_tiles = T;
        if (T >= INT32_MAX) return fail(SPMV_ERR_UNSUPPORTED, "too many tiles");

        // algorithmic bytes: 12 nnz + 4 (m+1) + 8 m + 8 n_touched
        {
            const int64_t xl = world > 1 ? h->x_int_len + h->border_total : n;
            std::vector<char> touched(std::max<int64_t>(xl, 1), 0);
#pragma omp parallel for schedule(static)
            for (int64_t t = 0; t < nnz_loc; ++t) touched[pcol[t]] = 1;
            int64_t nt = 0;
#pragma omp parallel for reduction(+ : nt)
            for (int64_t c = 0; c < xl; ++c) nt += touched[c];
            h->bytes_alg = 12 * nnz_loc + 4 * (m_loc + 1) + 8 * m_loc + 8 * nt;
            h->bytes_alg_split = 0;
            if (n_parts) h->bytes_alg_split = 12 * nnz_loc + 8 * m_loc + 8 * nt;   // + segment metadata below
        }

        // Every kernel of the apply path is loaded now, not at its first launch
        // (CUDA's lazy loading): on a multi-GPU run a rank's kernel spins on a
        // peer's exchange flag, and a module load can wait for the kernels
        // running on the device -- a peer's first launch of, e.g., the DB fold
        // kernel would then stall the exchange until the device-side waits time
        // out (found by the loopback tests).
        {
            static std::atomic<int> loaded[kMaxDevices];
            const int di = h->device >= 0 && h->device < kMaxDevices ? h->device : kMaxDevices - 1;
            if (!loaded[di].load(std::memory_order_acquire)) {
                for (cudaError_t (*f)() : {preload_kernels_misc, preload_kernels_panel, preload_kernels_rowtile,
                                           preload_kernels_split, preload_kernels_xstaged}) {
                    const cudaError_t e = f();
                    if (e != cudaSuccess) return fail(SPMV_ERR_INTERNAL, "kernel preload: %s", cudaGetErrorString(e));
                }
                loaded[di].store(1, std::memory_order_release);
            }
        }

        // ------------------------------------------------ device upload
        std::vector<int32_t> rp32(m_loc + 1);
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p <= m_loc; ++p) rp32[p] = (int32_t)rp[p];
        spmv_status_t s;
        if ((s = upload(h, &h->d_rowptr, rp32.data(), m_loc + 1, m_loc + 1 + kPad))) return s;
        if ((s = upload(h, &h->d_col, pcol.data(), nnz_loc, nnz_loc + kPad))) return s;
        if ((s = upload(h, &h->d_val, pval.data(), nnz_loc, nnz_loc + kPad))) return s;
        if ((s = upload(h, &h->d_tile_row, tile_row.data(), T + 1))) return s;
        {
            std::vector<int32_t> tile_nnz(T + 1);
            for (int64_t t = 0; t <= T; ++t) tile_nnz[t] = (int32_t)rp[tile_row[t]];
            if ((s = upload(h, &h->d_tile_nnz, tile_nnz.data(), T + 1))) return s;
            std::vector<int32_t> tile_cls(std::max<int64_t>(T, 1), kTileGeneral);
#pragma omp parallel for schedule(static)
            for (int64_t t = 0; t < T; ++t) {
                int64_t mx = 0;
                for (int64_t r = tile_row[t]; r < tile_row[t + 1]; ++r) mx = std::max(mx, rp[r + 1] - rp[r]);
                // short tiles: lanes per row V = largest power of two with
                // rows * V <= 512, capped at 32 and at the longest row rounded
                // up to a power of two (rowtile.cu halves it for 256 threads)
                int32_t cls = kTileGeneral;
                if (mx <= kShortRow) {
                    const int64_t nr = tile_row[t + 1] - tile_row[t];
                    int32_t V = 1;
                    while (V < 32 && nr * (2 * V) <= 512 && V < mx) V *= 2;
                    cls = V;
                }
                tile_cls[t] = cls;
            }
            if ((s = upload(h, &h->d_tile_cls, tile_cls.data(), T))) return s;
        }
        h->bytes_stream = 12 * nnz_loc + 4 * (m_loc + 1) + 8 * m_loc;

        // ------------------- f3: 16-bit tile-local column ids (row tiles)
        // The ICSR idea of P:L43 (fewer index bytes per nonzero) in the form
        // the SB layout allows: a row tile never crosses an SB block, so its
        // columns lie in its block's interior C_k and the border C_B (Eq.(1))
        // -- two windows.  Per tile, the windows are cut at the largest gap
        // between its distinct columns; id u = c - lo for c in the low window,
        // split + (c - hi_start) in the high one, decoded on the device as
        // u + (u < split ? lo : hi) with hi = hi_start - split.  Used when
        // every tile's windows fit 65,536 ids together (C1, C2): the kernel
        // then streams 2 + 8 bytes per nonzero instead of 4 + 8.  Integer
        // decoding: the same columns, the same summation order (bit-identical).
        h->index_bytes = 4;
        if (h->opt.index16 == 0 && T > 0 && nnz_loc > 0) {
            std::vector<uint16_t> c16(nnz_loc + kPad, 0);
            std::vector<int4> tb(T);
            std::atomic<int> fits{1};
#pragma omp parallel
            {
                std::vector<int32_t> cs;
#pragma omp for schedule(dynamic, 16)
                for (int64_t t = 0; t < T; ++t) {
                    if (!fits.load(std::memory_order_relaxed)) continue;
                    const int64_t a = rp[tile_row[t]], b = rp[tile_row[t + 1]];
                    cs.assign(pcol.begin() + a, pcol.begin() + b);
                    std::sort(cs.begin(), cs.end());
                    cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
                    int32_t lo = cs.empty() ? 0 : cs.front(), split = 65536, hi = lo;
                    if (!cs.empty() && (int64_t)cs.back() - lo >= 65536) {
                        size_t g = 0;   // largest gap: between cs[g] and cs[g + 1]
                        for (size_t q = 1; q + 1 < cs.size(); ++q)
                            if (cs[q + 1] - cs[q] > cs[g + 1] - cs[g]) g = q;
                        const int64_t lenA = (int64_t)cs[g] - lo + 1, lenB = (int64_t)cs.back() - cs[g + 1] + 1;
                        if (lenA + lenB > 65536) {
                            fits = 0;
                            continue;
                        }
                        split = (int32_t)lenA;
                        hi = cs[g + 1] - split;
                    }
                    tb[t] = make_int4(lo, hi, split, cs.empty() ? 0 : cs.back());
                    for (int64_t e = a; e < b; ++e) {
                        const int32_t c = pcol[e];
                        c16[e] = (uint16_t)(c - lo < split ? c - lo : c - hi);
                    }
                }
            }
            if (fits) {
                if ((s = upload(h, &h->d_col16, c16.data(), nnz_loc + kPad))) return s;
                if ((s = upload(h, &h->d_tile_base, tb.data(), T))) return s;
                h->index_bytes = 2;
                h->bytes_stream -= 2 * nnz_loc;
            }
        }

        mark(2);   // tiles, CSR upload, f3 ids
        // -------------------------------------------- split layout (a8)
        // Within each row tile the nonzeros are regrouped part-major: for k =
        // 0..K-1, the tile's rows' part-k runs ("segments") in row order --
        // the access order Pi defines, executed tile by tile (the
        // literal K-pass sequence); and row-major: each row's segments in part
        // order (the fused fallback).  DB across GPUs: the split is the ranks'
        // parts, folded after the exchange (exchange.cpp).
        if (n_parts && !db_dist) {
            const int KP = n_parts;
            std::vector<int64_t> seg_cnt(T * KP, 0), nz_cnt(T * KP, 0);
#pragma omp parallel for schedule(dynamic, 64)
            for (int64_t t = 0; t < T; ++t) {
                std::vector<int64_t> stamp(KP, -1);
                for (int64_t r = tile_row[t]; r < tile_row[t + 1]; ++r) {
                    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
                        const int k = ppart[e];
                        nz_cnt[t * KP + k]++;
                        if (stamp[k] != r) { stamp[k] = r; seg_cnt[t * KP + k]++; }
                    }
                }
            }
            std::vector<int32_t> tile_seg(T * KP + 1);
            std::vector<int64_t> seg_off(T * KP + 1), nz_off(T * KP + 1);
            seg_off[0] = 0;
            nz_off[0] = 0;
            for (int64_t q = 0; q < T * KP; ++q) {
                seg_off[q + 1] = seg_off[q] + seg_cnt[q];
                nz_off[q + 1] = nz_off[q] + nz_cnt[q];
            }
            const int64_t S = seg_off[T * KP];
            if (S >= INT32_MAX) return fail(SPMV_ERR_UNSUPPORTED, "too many split segments");
            h->n_seg = S;
            for (int64_t q = 0; q <= T * KP; ++q) tile_seg[q] = (int32_t)seg_off[q];
            std::vector<int32_t> seg_ptr(S + 1), seg_row(std::max<int64_t>(S, 1)), scol(nnz_loc);
            std::vector<double> sval(nnz_loc);
            seg_ptr[S] = (int32_t)nnz_loc;
#pragma omp parallel for schedule(dynamic, 64)
            for (int64_t t = 0; t < T; ++t) {
                for (int k = 0; k < KP; ++k) {
                    int64_t sg = seg_off[t * KP + k];
                    int64_t nz = nz_off[t * KP + k];
                    for (int64_t r = tile_row[t]; r < tile_row[t + 1]; ++r) {
                        bool has = false;
                        for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
                            if (ppart[e] != k) continue;
                            if (!has) {
                                seg_ptr[sg] = (int32_t)nz;
                                seg_row[sg] = (int32_t)(r - tile_row[t]);
                                ++sg;
                                has = true;
                            }
                            scol[nz] = pcol[e];
                            sval[nz] = pval[e];
                            ++nz;
                        }
                    }
                }
            }
            h->bytes_alg_split += 8 * S + 4 * (T * KP + 1);
            {
                std::vector<int32_t> fcol(nnz_loc), frowseg(m_loc + 1), fsegptr(S + 1);
                std::vector<double> fval(nnz_loc);
                std::vector<int32_t> rcnt(m_loc);
#pragma omp parallel for schedule(dynamic, 4096)
                for (int64_t r = 0; r < m_loc; ++r) {
                    std::vector<int32_t> cnt(KP, 0);
                    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) cnt[ppart[e]]++;
                    int32_t c = 0;
                    for (int k = 0; k < KP; ++k) c += cnt[k] > 0;
                    rcnt[r] = c;
                }
                frowseg[0] = 0;
                for (int64_t r = 0; r < m_loc; ++r) frowseg[r + 1] = frowseg[r] + rcnt[r];
                if (frowseg[m_loc] != S) return fail(SPMV_ERR_INTERNAL, "split layout: segment count mismatch");
#pragma omp parallel for schedule(dynamic, 4096)
                for (int64_t r = 0; r < m_loc; ++r) {
                    std::vector<int32_t> cnt(KP, 0), off(KP + 1, 0);
                    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) cnt[ppart[e]]++;
                    for (int k = 0; k < KP; ++k) off[k + 1] = off[k] + cnt[k];
                    int32_t sg = frowseg[r];
                    for (int k = 0; k < KP; ++k)
                        if (cnt[k]) fsegptr[sg++] = (int32_t)(rp[r] + off[k]);
                    std::vector<int32_t> pos(off.begin(), off.end() - 1);
                    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
                        const int64_t q = rp[r] + pos[ppart[e]]++;
                        fcol[q] = pcol[e];
                        fval[q] = pval[e];
                    }
                }
                fsegptr[S] = (int32_t)nnz_loc;
                if ((s = upload(h, &h->d_fcol, fcol.data(), nnz_loc, nnz_loc + kPad))) return s;
                if ((s = upload(h, &h->d_fval, fval.data(), nnz_loc, nnz_loc + kPad))) return s;
                if ((s = upload(h, &h->d_frowseg, frowseg.data(), m_loc + 1))) return s;
                if ((s = upload(h, &h->d_fsegptr, fsegptr.data(), S + 1))) return s;
            }
            if ((s = upload(h, &h->d_tile_seg, tile_seg.data(), T * KP + 1))) return s;
            if ((s = upload(h, &h->d_seg_ptr, seg_ptr.data(), S + 1))) return s;
            if ((s = upload(h, &h->d_seg_row, seg_row.data(), S))) return s;
            if ((s = upload(h, &h->d_scol, scol.data(), nnz_loc, nnz_loc + kPad))) return s;
            if ((s = upload(h, &h->d_sval, sval.data(), nnz_loc, nnz_loc + kPad))) return s;
        }

        // global per-block y-slot counts (SB): every rank cuts its blocks into
        // the same panels as a single GPU would, so the summation order of a
        // row -- and y -- does not depend on the number of GPUs
        if (blocks && h->kind == SPMV_SB && nnz_loc > 0) {
            std::vector<int64_t> loc(K, 0);
            for (int64_t i = 0; i < m; ++i) {
                const int64_t nr = row_perm ? row_perm[i] : i;
                const int k = row_block(nr);
                if (k >= 0 && k < K) loc[k] += row_slots(row_ptr[i + 1] - row_ptr[i]);
            }
            h->blk_slots = loc;
        }

        mark(3);   // split layouts
        // ---------------- fused multiple-SpMxV on panels (a8): (row, part) virtual rows
        if (n_parts && !db_dist && nnz_loc > 0 && O.split_kernel != SPMV_SPLIT_ROWS) {
            if ((s = plan_pn(h, h->pns, rp, pcol, pval, rbp, cbp, &ppart,
                             O.split_kernel == SPMV_SPLIT_PANEL || world > 1)))
                return s;
            if (world > 1 && !h->pns.ok())
                return fail(SPMV_ERR_UNSUPPORTED, "world > 1: the split's panel plan cannot be built");
        }
        // ------------------ single SpMxV: x-staged SB blocks (Eq.(1))
        // world 1, SB: when every block's x(C_k) + x(C_B) fits one SM's shared
        // memory beside the tile buffers, each CTA stages its block's slice
        // once and gathers from shared memory (C2: 11,875 + 10,000 entries)
        h->kernel = 0;
        // (measured slower than the row tiles on C2, so only on request)
        const bool xs_try = world == 1 && h->kind == SPMV_SB && nnz_loc > 0 && T > 0 &&
                            O.kernel == SPMV_KERNEL_XSTAGED;
        if (xs_try) {
            const int64_t nB = cbp[K + 1] - cbp[K];
            int64_t max_x = 0;
            for (int k = 0; k < K; ++k) max_x = std::max<int64_t>(max_x, cbp[k + 1] - cbp[k] + nB);
            const bool fits = xstaged_smem_bytes(max_x) <= kPnSmemMax && max_x <= 65536;
            if (!fits && O.kernel == SPMV_KERNEL_XSTAGED)
                return fail(SPMV_ERR_UNSUPPORTED, "x-staged kernel: a block's x(C_k) + x(C_B) (%lld entries) "
                                                  "does not fit shared memory", (long long)max_x);
            if (fits) {
                // tiles of each block (tiles never cross a block: cuts at rbp)
                std::vector<int32_t> tile_blk(T);
                for (int64_t t = 0; t < T; ++t) tile_blk[t] = row_block(R0 + tile_row[t]);
                bool ok = true;
                for (int64_t t = 0; t < T && ok; ++t) ok = tile_blk[t] < K;
                if (ok) {
                    // block-local ids
                    std::vector<uint16_t> cx(nnz_loc + kPad, 0);
#pragma omp parallel for schedule(dynamic, 64)
                    for (int64_t t = 0; t < T; ++t) {
                        const int k = tile_blk[t];
                        const int64_t q0 = cbp[k], nk = cbp[k + 1] - cbp[k];
                        for (int64_t e = rp[tile_row[t]]; e < rp[tile_row[t + 1]]; ++e) {
                            const int64_t c = pcol[e];
                            cx[e] = (uint16_t)(c < cbp[K] ? c - q0 : nk + (c - cbp[K]));
                        }
                    }
                    // CTAs: about one per SM, shared among the blocks by nonzeros,
                    // each a contiguous run of its block's tiles balanced by nonzeros
                    const int64_t sms = kernel_num_sms();
                    std::vector<XsCta> ctas;
                    int64_t t = 0;
                    for (int k = 0; k < K; ++k) {
                        const int64_t ta = t;
                        while (t < T && tile_blk[t] == k) ++t;
                        if (t == ta) continue;
                        const int64_t za = rp[tile_row[ta]], zb = rp[tile_row[t]];
                        const int64_t nc = std::max<int64_t>(1, std::min<int64_t>(t - ta,
                                               (sms * (zb - za) + nnz_loc / 2) / std::max<int64_t>(nnz_loc, 1)));
                        int64_t u = ta;
                        for (int64_t j = 0; j < nc; ++j) {
                            const int64_t target = za + (zb - za) * (j + 1) / nc;
                            int64_t v = u + 1;
                            while (v < t && rp[tile_row[v]] < target) ++v;
                            if (j == nc - 1) v = t;
                            if (v <= u) continue;
                            XsCta c{};
                            c.t0 = (int32_t)u;
                            c.t1 = (int32_t)v;
                            c.q0 = (int32_t)cbp[k];
                            c.nk = (int32_t)(cbp[k + 1] - cbp[k]);
                            c.qB = (int32_t)cbp[K];
                            c.nB = (int32_t)nB;
                            c.k = k;
                            {   // lanes per row for the warp-independent form: ~ mean row length / 3
                                const int64_t rows = tile_row[v] - tile_row[u];
                                const int64_t nz = rp[tile_row[v]] - rp[tile_row[u]];
                                int32_t V = 1;
                                while (V < 32 && V * 3 < (rows ? nz / rows : 1)) V *= 2;
                                c.pad = V;
                            }
                            ctas.push_back(c);
                            u = v;
                        }
                    }
                    if ((s = upload(h, &h->d_colx, cx.data(), nnz_loc + kPad))) return s;
                    if ((s = upload(h, &h->d_xcta, ctas.data(), ctas.size()))) return s;
                    h->xs_ncta = (int32_t)ctas.size();
                    h->xs_max_x = (int32_t)max_x;
                    h->kernel = 8;
                    h->bytes_stream = 10 * nnz_loc + 4 * (m_loc + 1) + 8 * m_loc;
                }
            }
        }
        // ------------------------------ single SpMxV: column-sorted panels (a5-a7)
        // any matrix at world 1 (C4: 0.18 vs 0.26 ms for the row-tile kernel);
        // small matrices fall back to row tiles through the padding test; at
        // world > 1 the panel kernel is the only one with the border wait
        if (h->kernel == 0 && nnz_loc > 0 && O.kernel != SPMV_KERNEL_ROWTILE && O.kernel != SPMV_KERNEL_XSTAGED) {
            std::string why;
            if ((s = plan_pn(h, h->pn, rp, pcol, pval, rbp, cbp, nullptr, O.kernel == SPMV_KERNEL_PANEL || world > 1,
                             &why)))
                return s;
            if (h->pn.ok()) {
                h->kernel = 7;
                h->bytes_stream = (12 * 32 + 4) * h->pn.groups + 14 * 32 * h->pn.far_blocks + 8 * h->m_loc;
                // the panel kernel reads only its group stream: the device CSR
                // copy (and the row tiles' 16-bit ids) would double the
                // handle's memory (C5: 13.7 GB) -- released unless asked for
                if (!O.retain_csr) {
                    dfree(h, h->d_col);
                    dfree(h, h->d_val);
                    dfree(h, h->d_col16);
                    dfree(h, h->d_tile_base);
                    h->d_col = nullptr;
                    h->d_val = nullptr;
                    h->d_col16 = nullptr;
                    h->d_tile_base = nullptr;
                }
            } else if (world > 1) {
                return fail(SPMV_ERR_UNSUPPORTED, "world > 1: the panel plan cannot be built (%s)", why.c_str());
            }
        } else if (world > 1 && nnz_loc > 0) {
            return fail(SPMV_ERR_UNSUPPORTED, "world > 1 runs the panel kernel");
        }

        mark(4);   // panel plans and their upload
        // -------------------------------------- ORIGINAL-mode maps (a3, a7)
        if (world == 1 && h->has_perm) {
            if ((s = upload(h, &h->d_colinv, col_inv.data(), n))) return s;
            std::vector<int32_t> rperm(m);
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < m; ++i) rperm[i] = row_perm ? row_perm[i] : (int32_t)i;
            if ((s = upload(h, &h->d_rowperm, rperm.data(), m))) return s;
            if ((s = dalloc(h, &h->d_xhat, n))) return s;
            if ((s = dalloc(h, &h->d_yhat, m))) return s;
        }

        // ------------------------------- owner map r(c) for the x-update (a9)
        // Square A: column c (new) is old column j = col_inv[c]; as a row, old
        // j is new row row_perm[j]; its place in y_local is its offset in the
        // rank's block rows, or (DB across GPUs) in its owned border-row slice.
        if (m == n && m > 0) {
            std::vector<int32_t> owner(h->x_local_len);
            std::atomic<int> outside{0};
            const int64_t YB0 = h->y_bord_begin, YBL = h->y_bord_len;
#pragma omp parallel for schedule(static)
            for (int64_t l = 0; l < h->x_local_len; ++l) {
                const int64_t c = (world > 1) ? (l < h->x_int_len ? h->x_int_begin + l
                                                                  : h->x_bord_begin + (l - h->x_int_len))
                                              : l;
                const int64_t j = col_inv[c];
                const int64_t r = row_perm ? row_perm[j] : j;
                if (r >= R0 && r < R1) owner[l] = (int32_t)(r - R0);
                else if (YBL > 0 && r >= YB0 && r < YB0 + YBL) owner[l] = (int32_t)(m_blk + (r - YB0));
                else { outside = 1; owner[l] = 0; }
            }
            if (!outside) {
                // runs of consecutive rows (A17's owner-aligned layout: one per block's interior
                // columns and one per owned border slice): the x-update then reads no map per column
                std::vector<int64_t> rs;
                std::vector<int32_t> rt;
                for (int64_t l = 0; l < h->x_local_len; ++l)
                    if (l == 0 || owner[l] != owner[l - 1] + 1) {
                        rs.push_back(l);
                        rt.push_back(owner[l]);
                        if ((int64_t)rs.size() * kOwnerRunMin > h->x_local_len) break;
                    }
                if ((int64_t)rs.size() * kOwnerRunMin <= h->x_local_len) {
                    h->owner_runs = (int64_t)rs.size();
                    rs.push_back(h->x_local_len);
                    const int64_t T = (h->x_local_len + kNormTileCols - 1) / kNormTileCols;
                    std::vector<int64_t> td(T);
                    for (int64_t t = 0, r = 0; t < T; ++t) {   // r: run of the tile's first column
                        const int64_t a = t * kNormTileCols, b = std::min(a + kNormTileCols, h->x_local_len);
                        while (rs[r + 1] <= a) ++r;
                        td[t] = rs[r + 1] >= b ? (int64_t)rt[r] - rs[r] : kNoDelta;
                    }
                    if ((s = upload(h, &h->d_own_start, rs.data(), rs.size()))) return s;
                    if ((s = upload(h, &h->d_own_tgt, rt.data(), rt.size()))) return s;
                    if ((s = upload(h, &h->d_own_tdelta, td.data(), td.size()))) return s;
                } else if ((s = upload(h, &h->d_owner, owner.data(), h->x_local_len))) {
                    return s;
                }
                h->has_owner = true;
            }
        }

        // ------------------------------------------------- misc buffers
        if ((s = dalloc(h, &h->d_slots, kMaxSlots * kSlotStride))) return s;
        if (h->opt.debug_checks) {   // the checked panel kernel's violation counters
            if ((s = dalloc(h, &h->d_dbg, 3))) return s;
            CUDA_TRY(cudaMemset(h->d_dbg, 0, 3 * sizeof(unsigned long long)));
        }
        CUDA_TRY(cudaMemset(h->d_slots, 0, kMaxSlots * kSlotStride * sizeof(unsigned long long)));

        // ---------------- DB across GPUs: temporaries and their fold lists (f1)
        if (db_dist) {
            if ((s = dalloc(h, &h->d_T, std::max<int64_t>(h->n_T, 1)))) return s;
            // counts cnt[p][r] of temporaries rank p sends to rank r: every rank
            // derives them from the full input (same on all ranks)
            std::vector<int64_t> cnt((size_t)world * world, 0);
            // per border row q and part k: segment exists
            std::vector<uint8_t> has((size_t)RBn * K, 0);
#pragma omp parallel for schedule(dynamic, 256)
            for (int64_t q = 0; q < RBn; ++q) {
                const int64_t gp = rbp[K] + q, i = row_inv[gp];
                for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) {
                    const int64_t c = col_perm ? col_perm[col_idx[t]] : col_idx[t];
                    has[q * K + part_of(t, gp, c)] = 1;
                }
            }
            for (int64_t q = 0; q < RBn; ++q) {
                const int dst = block_rank(rslice_block(rbp[K] + q));
                for (int k = 0; k < K; ++k)
                    if (has[q * K + k]) cnt[(size_t)block_rank(k) * world + dst]++;
            }
            h->t_send_off.assign(world, 0);
            h->t_send_cnt.assign(world, 0);
            h->t_recv_off.assign(world, 0);
            h->t_recv_cnt.assign(world, 0);
            int64_t so = 0;
            for (int r = 0; r < world; ++r) {
                h->t_send_off[r] = so;
                h->t_send_cnt[r] = cnt[(size_t)rank * world + r];
                so += h->t_send_cnt[r];
            }
            if (so != h->n_T) return fail(SPMV_ERR_INTERNAL, "DB temporaries: count mismatch (%lld vs %lld)",
                                          (long long)so, (long long)h->n_T);
            int64_t tmax = 0;
            for (int r = 0; r < world; ++r) {
                int64_t ro_ = 0;
                for (int p = 0; p < world; ++p) ro_ += cnt[(size_t)p * world + r];
                tmax = std::max(tmax, ro_);
            }
            int64_t ro = 0;
            for (int p = 0; p < world; ++p) {
                h->t_recv_off[p] = ro;
                h->t_recv_cnt[p] = cnt[(size_t)p * world + rank];
                ro += h->t_recv_cnt[p];
            }
            h->t_recv_total = ro;
            h->t_recv_max = tmax;
            h->t_dst_off.assign(world, 0);
            for (int r = 0; r < world; ++r)
                for (int p = 0; p < rank; ++p) h->t_dst_off[r] += cnt[(size_t)p * world + r];
            // fold lists: for each owned border row, its temporaries' positions
            // in the received buffer, in part order (sources are ranks in order,
            // each sending its parts in order, then rows in order)
            const int64_t YB0 = h->y_bord_begin, YBL = h->y_bord_len;
            std::vector<int32_t> fptr(YBL + 1, 0), fpos;
            std::vector<std::vector<int32_t>> lists(YBL);
            int64_t pos = 0;
            for (int k = 0; k < K; ++k)
                for (int64_t q = YB0 - rbp[K]; q < YB0 - rbp[K] + YBL; ++q)
                    if (has[q * K + k]) lists[q - (YB0 - rbp[K])].push_back((int32_t)pos++);
            if (pos != ro) return fail(SPMV_ERR_INTERNAL, "DB temporaries: receive count mismatch");
            for (int64_t i = 0; i < YBL; ++i) {
                fptr[i + 1] = fptr[i] + (int32_t)lists[i].size();
                fpos.insert(fpos.end(), lists[i].begin(), lists[i].end());
            }
            if ((s = upload(h, &h->d_fold_ptr, fptr.data(), YBL + 1))) return s;
            if (fpos.empty()) fpos.push_back(0);
            if ((s = upload(h, &h->d_fold_pos, fpos.data(), fpos.size()))) return s;
        }
        // ---------------- world > 1: exchange buffers (a4 / f2)
        if (world > 1) {
            if ((s = xchg_alloc(h))) return s;
        }
        CUDA_TRY(cudaDeviceSynchronize());
        return SPMV_OK;
    };
    local_status = run_local();
    mark(5);   // maps, buffers, exchange allocation
    if (world > 1 && !test_rank) {   // every rank returns the same status (after all planning)
        spmv_status_t agreed = SPMV_OK;
        spmv_status_t r = xchg_agree(h, local_status, &agreed);
        if (r != SPMV_OK) return r;
        if (agreed != SPMV_OK) {
            if (local_status == SPMV_OK) return fail(agreed, "create failed on another rank");
            return local_status;
        }
        if ((r = xchg_connect(h)) != SPMV_OK) return r;   // P2P handles (all ranks agree inside), else NCCL
    }
    return local_status;
}

}  // namespace spmvb

extern "C" {

spmv_status_t spmv_create_ex(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                             const double* val, const int32_t* row_perm, const int32_t* col_perm,
                             const spmv_blocks_t* blocks, int32_t n_parts, const int32_t* part_of_nnz,
                             const spmv_dist_t* dist, const spmv_options_t* options, spmv_handle_t* out) {
    return create_common(m, n, nnz, row_ptr, col_idx, val, row_perm, col_perm, blocks, n_parts, part_of_nnz, dist,
                         options, false, out);
}

spmv_status_t spmv_create(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                          const double* val, const int32_t* row_perm, const int32_t* col_perm,
                          const spmv_blocks_t* blocks, int32_t n_parts, const int32_t* part_of_nnz,
                          const spmv_dist_t* dist, spmv_handle_t* out) {
    return create_common(m, n, nnz, row_ptr, col_idx, val, row_perm, col_perm, blocks, n_parts, part_of_nnz, dist,
                         nullptr, false, out);
}

spmv_status_t spmv_destroy(spmv_handle_t h) {
    if (!h) return SPMV_OK;
    if (!valid(h)) return fail(SPMV_ERR_USAGE, "invalid handle");
    free_plan(h);
    return SPMV_OK;
}

}  // extern "C"

namespace spmvb {

spmv_status_t create_common(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                            const double* val, const int32_t* row_perm, const int32_t* col_perm,
                            const spmv_blocks_t* blocks, int32_t n_parts, const int32_t* part_of_nnz,
                            const spmv_dist_t* dist, const spmv_options_t* options, bool test_rank,
                            spmv_handle_t* out) {
    if (!out) return fail(SPMV_ERR_USAGE, "out is NULL");
    *out = nullptr;
    spmv_plan_s* h = new (std::nothrow) spmv_plan_s();
    if (!h) return fail(SPMV_ERR_INTERNAL, "out of host memory");
    spmv_status_t s;
    try {
        s = create_impl(m, n, nnz, row_ptr, col_idx, val, row_perm, col_perm, blocks, n_parts, part_of_nnz, dist,
                        options, test_rank, h);
    } catch (const std::bad_alloc&) {
        s = fail(SPMV_ERR_INTERNAL, "out of host memory");
    } catch (...) {
        s = fail(SPMV_ERR_INTERNAL, "unexpected exception");
    }
    if (s != SPMV_OK) {
        free_plan(h);
        return s;
    }
    *out = h;
    return SPMV_OK;
}

}  // namespace spmvb

// --------------------------------------------------------------- apply
namespace {

spmv_status_t check_vectors(spmv_handle_t h, const double* x, int64_t x_len, double* y, int64_t y_len,
                            uint32_t flags) {
    if (!valid(h)) return fail(SPMV_ERR_USAGE, "invalid handle");
    if (flags & ~(uint32_t)(SPMV_VEC_ORIGINAL | SPMV_FUSE_MAXABS | SPMV_SPLIT_LITERAL))
        return fail(SPMV_ERR_USAGE, "unknown flag");
    if ((!x && x_len) || (!y && y_len)) return fail(SPMV_ERR_USAGE, "NULL vector");
    if ((const void*)x == (const void*)y && x) return fail(SPMV_ERR_USAGE, "x and y alias");
    if (((uintptr_t)x & 7) || ((uintptr_t)y & 7)) return fail(SPMV_ERR_USAGE, "x/y not 8-byte aligned");
    const bool orig = flags & SPMV_VEC_ORIGINAL;
    if (orig && h->world > 1) return fail(SPMV_ERR_UNSUPPORTED, "ORIGINAL index space with world > 1");
    const int64_t xl = orig ? h->n : h->x_local_len;
    const int64_t yl = orig ? h->m : h->m_out;
    if (x_len != xl || y_len != yl)
        return fail(SPMV_ERR_DATA, "dimension mismatch: x_len %lld (want %lld), y_len %lld (want %lld)",
                    (long long)x_len, (long long)xl, (long long)y_len, (long long)yl);
    return SPMV_OK;
}

void fill_pn_args(const PanelPlan& pl, PnArgs& X) {
    X.panel = pl.d_panel;
    X.n_panels = (int32_t)pl.panels;
    X.gval = pl.d_gval;
    X.gidx = pl.d_gidx;
    X.gbase4 = pl.d_gbase4;
    X.max_rows = pl.max_rows;
    X.row2slot = pl.d_r2s;
    X.split_first = pl.d_split_first;
    X.split_cnt = pl.d_split_cnt;
    X.split_slots = pl.d_split_slots;
    X.split_row = pl.d_split_row;
    X.max_sslots = pl.max_sslots;
    X.max_split_n = pl.max_split_n;
    X.gather_na = pl.gather_na;
    X.fval = pl.d_fval;
    X.fcol = pl.d_fcol;
    X.fslot = pl.d_fslot;
}

spmv_status_t run(spmv_handle_t h, const double* x, double* y, uint32_t flags, cudaStream_t st, bool split) {
    DeviceGuard dg(h->device);
    if (!dg.ok()) return fail(SPMV_ERR_INTERNAL, "cannot select device %d", h->device);
    const bool orig = (flags & SPMV_VEC_ORIGINAL) && h->has_perm;
    const double* xk = x;
    double* yk = y;
    if (orig) {   // a3: x^[c] = x[col_inv[c]]
        CUDA_TRY(launch_gather(x, h->d_colinv, h->d_xhat, h->n, st));
        xk = h->d_xhat;
        yk = h->d_yhat;
    }
    unsigned long long* slots = nullptr;
    if (flags & SPMV_FUSE_MAXABS) {
        CUDA_TRY(cudaMemsetAsync(h->d_slots, 0, kMaxSlots * kSlotStride * sizeof(unsigned long long), st));
        slots = h->d_slots;
    }
    // a4: world > 1 -- the border x(C_B) this apply reads (exchange.cpp)
    XView xv;
    xv.x_hi = xk;
    xv.x_split = INT32_MAX;
    if (h->world > 1 && xchg_failed(h))   // sticky: a peer stopped answering in an earlier apply
        return fail(SPMV_ERR_INTERNAL, "a border exchange timed out in an earlier apply (a peer is gone); "
                                       "its results were invalid");
    if (h->world > 1) {
        spmv_status_t s = xchg_pre(h, xk, st, xv);
        if (s) return s;
    }
    const bool xsplit = xv.x_split != INT32_MAX;
    // DB across GPUs: the split is the ranks' parts (exchange.cpp folds them)
    const bool db_dist = h->world > 1 && h->kind == SPMV_DB;
    if (split && !db_dist && (flags & SPMV_SPLIT_LITERAL)) {
        if (h->world > 1) return fail(SPMV_ERR_UNSUPPORTED, "SPLIT_LITERAL with world > 1");
        // y = 0; y <- y + A^k x, one pass per k
        TileArgs A{};
        A.tile_row = h->d_tile_row;
        A.n_tiles = (int32_t)h->n_tiles;
        A.y = yk;
        A.x_lo = xk;
        A.x_hi = xk;
        A.x_split = INT32_MAX;
        A.tile_seg = h->d_tile_seg;
        A.seg_ptr = h->d_seg_ptr;
        A.seg_row = h->d_seg_row;
        A.col = h->d_scol;
        A.val = h->d_sval;
        A.K = h->n_parts;
        CUDA_TRY(cudaMemsetAsync(yk, 0, h->m_loc * sizeof(double), st));
        for (int k = 0; k < h->n_parts; ++k) {
            TileArgs B = A;
            B.k_begin = k;
            B.k_end = k + 1;
            B.accumulate = 1;
            B.maxabs_slots = k == h->n_parts - 1 ? slots : nullptr;
            CUDA_TRY(launch_split(B, false, st));
        }
    } else if ((!split || db_dist) ? h->kernel == 7 : h->pns.ok()) {
        PnArgs X{};
        fill_pn_args((!split || db_dist) ? h->pn : h->pns, X);
        X.x_lo = xk;
        X.x_hi = xv.x_hi;
        X.x_split = xv.x_split;
        X.y = yk;
        X.y_hi = db_dist ? h->d_T : nullptr;   // DB across GPUs: temporaries' rows -> d_T
        X.y_split = db_dist ? (int32_t)h->m_blk : INT32_MAX;
        X.maxabs_slots = slots;
        X.ready = xv.ready;
        X.world = h->world;
        X.self = h->rank;
        X.seq = xv.seq;
        X.err = xv.err;
        X.herr = xv.herr;
        X.dbg = h->d_dbg;
        X.stamps = h->d_stamps;
        X.x_cols = h->world > 1 ? h->x_int_len + h->border_total : h->n;
        CUDA_TRY(launch_panel(X, st));
    } else if (!split && h->kernel == 8) {
        XsArgs Q{};
        Q.cta = h->d_xcta;
        Q.n_cta = h->xs_ncta;
        Q.max_x = h->xs_max_x;
        Q.tile_row = h->d_tile_row;
        Q.tile_nnz = h->d_tile_nnz;
        Q.tile_cls = h->d_tile_cls;
        Q.rowptr = h->d_rowptr;
        Q.colx = h->d_colx;
        Q.val = h->d_val;
        Q.x = xk;
        Q.y = yk;
        Q.maxabs_slots = slots;
        CUDA_TRY(launch_xstaged(Q, st));
    } else if (!split) {
        RowTileArgs P{};
        P.tile_row = h->d_tile_row;
        P.tile_nnz = h->d_tile_nnz;
        P.tile_cls = h->d_tile_cls;
        P.rowptr = h->d_rowptr;
        P.col = h->d_col;
        P.col16 = h->d_col16;
        P.tile_base = h->d_tile_base;
        P.val = h->d_val;
        P.x_lo = xk;
        P.x_hi = xv.x_hi;
        P.x_split = xv.x_split;
        P.n_tiles = (int32_t)h->n_tiles;
        P.y = yk;
        P.maxabs_slots = slots;
        CUDA_TRY(launch_rowtile(P, xsplit, st));
    } else {
        // fused multiple-SpMxV, row-major segments (split.cu spmv_split_rows_kernel)
        RowTileArgs R{};
        R.tile_row = h->d_tile_row;
        R.tile_nnz = h->d_tile_nnz;
        R.tile_cls = h->d_tile_cls;
        R.rowptr = h->d_rowptr;
        R.col = h->d_fcol;
        R.val = h->d_fval;
        R.x_lo = xk;
        R.x_hi = xv.x_hi;
        R.x_split = xv.x_split;
        R.n_tiles = (int32_t)h->n_tiles;
        R.y = yk;
        R.maxabs_slots = slots;
        CUDA_TRY(launch_split_rows(R, h->d_frowseg, h->d_fsegptr, xsplit, st));
    }
    if (h->world > 1) {
        spmv_status_t s = xchg_post(h, yk, slots, st);
        if (s) return s;
    }
    if (orig)   // a7: y[i] = y^[row_perm[i]]
        CUDA_TRY(launch_gather(h->d_yhat, h->d_rowperm, y, h->m, st));
    return SPMV_OK;
}

}  // namespace

extern "C" {

spmv_status_t spmv_apply(spmv_handle_t h, const double* x, int64_t x_len, double* y, int64_t y_len, uint32_t flags,
                         void* stream) {
    spmv_status_t s = check_vectors(h, x, x_len, y, y_len, flags);
    if (s) return s;
    if (flags & SPMV_SPLIT_LITERAL) return fail(SPMV_ERR_USAGE, "SPLIT_LITERAL is a split_apply flag");
    return run(h, x, y, flags, (cudaStream_t)stream, false);
}

spmv_status_t spmv_split_apply(spmv_handle_t h, const double* x, int64_t x_len, double* y, int64_t y_len,
                               uint32_t flags, void* stream) {
    spmv_status_t s = check_vectors(h, x, x_len, y, y_len, flags);
    if (s) return s;
    if (!h->n_parts && !(h->world > 1 && h->kind == SPMV_DB)) return fail(SPMV_ERR_UNSUPPORTED, "handle has no split");
    return run(h, x, y, flags, (cudaStream_t)stream, true);
}

spmv_status_t spmv_get_info(spmv_handle_t h, spmv_info_t* info) {
    if (!valid(h) || !info) return fail(SPMV_ERR_USAGE, "invalid handle or info");
    memset(info, 0, sizeof *info);
    info->m = h->m; info->n = h->n; info->nnz = h->nnz;
    info->m_local = h->m_loc; info->nnz_local = h->nnz_loc; info->row_begin = h->row_begin;
    info->x_local_len = h->x_local_len;
    info->x_interior_begin = h->x_int_begin; info->x_interior_len = h->x_int_len;
    info->x_border_begin = h->x_bord_begin; info->x_border_len = h->x_bord_len;
    info->border_total = h->border_total;
    info->n_tiles = h->n_tiles; info->n_long_rows = h->n_long;
    info->bytes_alg = h->bytes_alg; info->bytes_alg_split = h->bytes_alg_split;
    info->split_segments = h->n_seg;
    info->n_parts = h->n_parts; info->rank = h->rank; info->world = h->world; info->kind = h->kind;
    info->has_owner_map = h->has_owner ? 1 : 0;
    info->owner_runs = h->owner_runs;
    info->panels = h->kernel == 7 ? h->pn.panels : 0;
    info->groups = h->kernel == 7 ? h->pn.groups : 0;
    info->far_nonzeros = h->kernel == 7 ? h->pn.far : 0;
    info->pad_slots = h->kernel == 7 ? h->pn.pad : 0;
    info->deferred = h->kernel == 7 ? h->pn.deferred : 0;
    info->y_wavefronts_x1000 = h->kernel == 7 ? (int64_t)(h->pn.ywf * 1000.0) : 0;
    info->bytes_stream = h->bytes_stream;
    info->kernel = h->kernel;
    info->gather_sectors = h->kernel == 7 ? h->pn.gsectors : 0;
    info->split_kernel = h->n_parts == 0 ? 0 : h->pns.ok() ? 7 : (h->world > 1 && h->kind == SPMV_DB) ? 7 : 3;
    info->exchange = h->xmode;
    info->y_local_len = h->m_out;
    info->y_border_begin = h->y_bord_begin;
    info->y_border_len = h->y_bord_len;
    info->exchange_timeouts = xchg_timeouts(h);
    info->index_bytes = h->index_bytes;
    for (int k = 0; k < 6; ++k) info->create_s[k] = h->create_s[k];
    for (int k = 0; k < 3; ++k) info->debug_violations[k] = 0;
    if (h->d_dbg) {
        DeviceGuard g(h->device);
        unsigned long long v[3] = {0, 0, 0};
        if (cudaDeviceSynchronize() == cudaSuccess &&
            cudaMemcpy(v, h->d_dbg, sizeof v, cudaMemcpyDeviceToHost) == cudaSuccess)
            for (int k = 0; k < 3; ++k) info->debug_violations[k] = (int64_t)v[k];
        else
            cudaGetLastError();
    }
    return SPMV_OK;
}

spmv_status_t spmv_maxabs(spmv_handle_t h, double* m_dev, void* stream) {
    if (!valid(h) || !m_dev) return fail(SPMV_ERR_USAGE, "invalid handle or pointer");
    cudaStream_t st = (cudaStream_t)stream;
    DeviceGuard dg(h->device);
    CUDA_TRY(launch_maxabs_finish(h->d_slots, m_dev, st));
    if (h->world > 1) {
        spmv_status_t s = xchg_allreduce_max(h, m_dev, st);
        if (s) return s;
    }
    return SPMV_OK;
}

spmv_status_t spmv_normalize(spmv_handle_t h, const double* y, const double* m_dev, double* x_next, void* stream) {
    if (!valid(h) || !y || !m_dev || !x_next) return fail(SPMV_ERR_USAGE, "invalid handle or pointer");
    if (!h->has_owner) return fail(SPMV_ERR_UNSUPPORTED, "no owner-aligned column->row map (A17)");
    DeviceGuard dg(h->device);
    if (h->owner_runs > 0)
        CUDA_TRY(launch_normalize_runs(y, h->d_own_tdelta, h->d_own_start, h->d_own_tgt, h->owner_runs, m_dev, x_next,
                                       h->x_local_len, (cudaStream_t)stream));
    else
        CUDA_TRY(launch_normalize(y, h->d_owner, m_dev, x_next, h->x_local_len, (cudaStream_t)stream));
    return SPMV_OK;
}

}  // extern "C"
