// host.cpp -- the C ABI of include/spmv.h: ingest, validation, permutation,
// planning, device upload, apply orchestration and the NCCL border exchange.
//
// Paper: Akbudak, Kayaaslan & Aykanat, arXiv 1203.2739 (P:Lnn = PAPER.md line).
//   a1 ingest  : A^ = P_r A P_c, old->new arrays
//   a2 plan    : SB/DB envelope of Eq.(1)/(5); row tiles;
//                split segments of Pi; shard of the row-slice
//                decomposition y_k <- R_k x
//   a3/a4      : x preparation; border-x exchange over NCCL (coupling columns
//                are the only input shared between row slices)
//   a5-a7      : one tile-kernel launch (kernels.cu)
//   a8         : fused multiple-SpMxV
//   a9         : max-abs and x-update glue for the power iterations
#include <algorithm>
#include <atomic>
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

#include "../../include/spmv.h"
#include "internal.h"
#include "plan_xs.h"
#include "plan_panel.h"

using spmvb::kTileNnz;
using spmvb::kTileRows;

namespace {

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

#define CUDA_TRY(expr)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(SPMV_ERR_INTERNAL, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),  \
                        __FILE__, __LINE__);                                                  \
    } while (0)

#define NCCL_TRY(expr)                                                                        \
    do {                                                                                      \
        ncclResult_t r_ = (expr);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return fail(SPMV_ERR_INTERNAL, "%s: %s (%s:%d)", #expr, ncclGetErrorString(r_),   \
                        __FILE__, __LINE__);                                                  \
    } while (0)

constexpr uint32_t kMagic = 0x53504d56u;   // "SPMV"
constexpr int64_t kPad = 8;                // col/val padding (128-bit quad loads past the end)

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

}  // namespace

struct PanelPlan {
    spmvb::PnPanel* d_panel = nullptr;
    double* d_gval = nullptr;
    uint32_t* d_gidx = nullptr;
    int32_t* d_gbase4 = nullptr;
    uint16_t* d_r2s = nullptr;        // [m_loc] y slot of each row in its panel (or split entry)
    int32_t* d_split_first = nullptr;
    int32_t* d_split_cnt = nullptr;
    uint16_t* d_split_slots = nullptr;
    int32_t* d_split_row = nullptr;
    int32_t max_sslots = 0, max_split_n = 0;
    int64_t panels = 0, groups = 0, pad = 0, gsectors = 0;
    int32_t max_rows = 0;
    int32_t gather_na = 0;            // x gathers bypass L1 allocation (SPMV_PN_GATHER_NA at create)
    int32_t ring = 0;                 // register-ring depth (SPMV_PN_RING at create; 0 = default)
    int32_t pf = 0;                   // L2 prefetch distance in epochs (SPMV_PN_PF at create; 0 = default)
    int32_t persist = 0;              // persistent CTAs (SPMV_PN_PERSIST at create)
    bool ok() const { return panels > 0; }
};

struct spmv_plan_s {
    uint32_t magic = kMagic;
    int device = 0;
    int rank = 0, world = 1;
    int kind = 0;                     // 0 none, 1 SB, 2 DB
    int64_t m = 0, n = 0, nnz = 0;    // global
    int64_t m_loc = 0, nnz_loc = 0, row_begin = 0;
    int64_t x_int_begin = 0, x_int_len = 0;     // interior columns (global permuted range)
    int64_t x_bord_begin = 0, x_bord_len = 0;   // owned border slice (global permuted)
    int64_t border_begin = 0, border_total = 0; // C_B
    int64_t x_local_len = 0;
    int64_t n_tiles = 0, n_long = 0;
    int32_t n_parts = 0;
    int64_t n_seg = 0;
    int64_t bytes_alg = 0, bytes_alg_split = 0;
    bool has_perm = false;
    bool has_owner = false;

    // device arrays (one allocation each)
    int32_t* d_rowptr = nullptr;      // [m_loc+1]
    int32_t* d_col = nullptr;         // [nnz_loc + pad] local column ids
    double* d_val = nullptr;          // [nnz_loc + pad]
    int32_t* d_tile_row = nullptr;    // [T+1]
    int32_t* d_tile_nnz = nullptr;    // [T+1] row_ptr[tile_row[t]]
    int* d_counter = nullptr;         // tile-claim counter of the pipe kernel
    int32_t* d_tile_cls = nullptr;    // [T] tile class (internal.h)
    int32_t* d_long_tiles = nullptr;  // [n_long] tiles holding one long row
    cudaStream_t side = nullptr;      // long-row kernel stream (forked from / joined to the caller's)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int kernel = 0;                   // 0 rowtile/256, 1 pipe, 2 tile, 3 rowtile/512, 4 rowseg, 5 rowtile/128,
                                      // 6 x-staged, 7 column-sorted panels (default for SB handles)
    // x-staged kernel (xstage.cu)
    spmvb::XsPanel* d_xs_panel = nullptr;
    int32_t* d_xs_wg = nullptr;
    int32_t* d_xs_wb = nullptr;
    int32_t* d_xs_U = nullptr;
    double* d_xs_gval = nullptr;
    uint32_t* d_xs_gidx = nullptr;
    double* d_xs_bval = nullptr;
    uint32_t* d_xs_bidx = nullptr;
    int32_t xs_cbits = 0;
    int64_t xs_panels = 0, xs_groups = 0, xs_pad = 0, xs_gb = 0;
    int64_t bytes_stream = 0;
    // column-sorted panel kernel (panel.cu): single SpMxV, and the fused
    // multiple-SpMxV over (row, part) virtual rows
    PanelPlan pn, pns;
    int32_t* d_tile_seg = nullptr;    // [T*K+1]
    int32_t* d_seg_ptr = nullptr;     // [S+1]
    int32_t* d_seg_row = nullptr;     // [S]
    int32_t* d_scol = nullptr;        // [nnz_loc + pad] split stream
    double* d_sval = nullptr;
    // fused split, row-major: each row's part segments in part order (P:L109 per row)
    int32_t* d_fcol = nullptr;        // [nnz_loc + pad]
    double* d_fval = nullptr;
    int32_t* d_frowseg = nullptr;     // [m_loc+1] first segment of each row
    int32_t* d_fsegptr = nullptr;     // [S+1] segment start positions (same positions as the CSR rows)
    bool split_rowmajor = true;
    std::vector<int64_t> blk_slots;   // SB: y slots per block over the whole matrix (panel cuts)
    bool test_nocomm = false;         // a test rank without a communicator (spmv_test_set_border)
    int64_t xs_test = 0;              // SPMV_PN_XS_TEST at create (SB, world 1): run the kernel's x-split
                                      // path with x_hi = x + C_B start (same values, two pointers)
    int32_t* d_colinv = nullptr;      // ORIGINAL mode: x^[c] = x[colinv[c]]
    int32_t* d_rowperm = nullptr;     // ORIGINAL mode: y[i] = y^[row_perm[i]]
    double* d_xhat = nullptr;
    double* d_yhat = nullptr;
    int32_t* d_owner = nullptr;       // [x_local_len] local col -> local row
    unsigned long long* d_slots = nullptr;
    double* d_xborder = nullptr;      // [border_total] gathered x(C_B) (world > 1)
    double* d_mscratch = nullptr;

    // exchange
    ncclComm_t comm = nullptr;
    std::vector<int64_t> bord_off, bord_cnt;   // per rank, offsets inside C_B
    bool equal_slices = true;
    std::vector<void*> allocs;
};

namespace {

template <class T>
spmv_status_t dalloc(spmv_plan_s* h, T** out, size_t count) {
    void* p = nullptr;
    size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess)
        return fail(SPMV_ERR_INTERNAL, "cudaMalloc(%zu bytes): %s", bytes, cudaGetErrorString(e));
    h->allocs.push_back(p);
    *out = static_cast<T*>(p);
    return SPMV_OK;
}

template <class T>
spmv_status_t upload(spmv_plan_s* h, T** out, const T* src, size_t count, size_t alloc_count = 0) {
    spmv_status_t s = dalloc(h, out, std::max(count, alloc_count));
    if (s) return s;
    if (alloc_count > count) CUDA_TRY(cudaMemset(*out, 0, std::max(count, alloc_count) * sizeof(T)));
    if (count) CUDA_TRY(cudaMemcpy(*out, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return SPMV_OK;
}

void free_plan(spmv_plan_s* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    for (void* p : h->allocs) cudaFree(p);
    h->allocs.clear();
    if (h->comm) ncclCommDestroy(h->comm);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    h->comm = nullptr;
    h->magic = 0;
    delete h;
}

bool valid(spmv_handle_t h) { return h && h->magic == kMagic; }

// Row-tile plan: greedy over rows; a tile holds whole
// rows with <= kTileNnz nonzeros and <= kTileRows rows; a longer row is a tile
// of its own (long-row path).  Tiles never cross an SB block boundary
// (block_row_ptr), so tiles are identical at every world size.
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
        // a tile's nonzeros sit at positions [(a & 3), (a & 3) + n) of a
        // 16-byte aligned kTileNnz-slot stage buffer (pipe.cu); the capacity
        // test assumes the worst alignment (3), so the cuts do not depend on
        // where the rank's local CSR starts -- tiles, and so every row's
        // summation order, are the same at every world size
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

int32_t spmv_version(void) { return 100; }

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
    const int64_t CB = cbp[K + 1] - cbp[K];
    auto bo = [&](int k) -> int64_t {
        return blocks->border_owner_ptr ? blocks->border_owner_ptr[k] : cbp[K] + (CB * k) / K;
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
    return SPMV_OK;
}

// Builds and uploads the x-staged kernel's panels (plan_xs.cpp).  Leaves the
// handle on the row-tile kernel when the matrix does not fit the format.
static spmv_status_t plan_xs(spmv_plan_s* h, const std::vector<int64_t>& rp, const std::vector<int32_t>& pcol,
                             const std::vector<double>& pval, const std::vector<int64_t>& rbp,
                             const std::vector<int64_t>& cbp) {
    const int K = (int)rbp.size() - 2;
    const int64_t R0 = h->row_begin, R1 = h->row_begin + h->m_loc;
    std::vector<spmvb::XsBlockIn> bl;
    for (int k = 0; k < K; ++k) {
        if (rbp[k + 1] <= R0 || rbp[k] >= R1) continue;
        spmvb::XsBlockIn b;
        b.r0 = rbp[k] - R0;
        b.r1 = rbp[k + 1] - R0;
        const int64_t q0 = h->world > 1 ? h->x_int_begin : 0;
        b.c0 = cbp[k] - q0;
        b.c1 = cbp[k + 1] - q0;
        bl.push_back(b);
    }
    const int64_t gb = h->world > 1 ? h->x_int_len : cbp[K];
    h->xs_gb = gb;
    const int64_t target = std::min<int64_t>(spmvb::kXsRowsMax,
                                             std::max<int64_t>(256, h->m / (3 * (int64_t)spmvb::kernel_num_sms())));
    std::vector<spmvb::XsPanelData> pd;
    spmvb::XsPlanStats st;
    std::string why;
    int cbits = 0;
    if (!spmvb::plan_xstage(rp, pcol, pval, bl, gb, h->border_total, target, pd, cbits, st, why)) return SPMV_OK;
    if (st.entries != h->nnz_loc) return fail(SPMV_ERR_INTERNAL, "x-staged plan lost nonzeros (%lld of %lld)",
                                              (long long)st.entries, (long long)h->nnz_loc);
    const int NW = spmvb::kXsWarps;
    const int64_t P = (int64_t)pd.size();
    std::vector<spmvb::XsPanel> desc(P);
    std::vector<int32_t> wg(P * NW + 1), wb(P * NW + 1);
    int64_t gi = 0, gbn = 0, nu = 0;
    for (int64_t p = 0; p < P; ++p) {
        desc[p] = pd[p].desc;
        for (int w = 0; w < NW; ++w) {
            wg[p * NW + w] = (int32_t)gi;
            wb[p * NW + w] = (int32_t)gbn;
            gi += pd[p].g_cnt[w];
            gbn += pd[p].b_cnt[w];
        }
        nu += (int64_t)NW * pd[p].desc.nch;
    }
    wg[P * NW] = (int32_t)gi;
    wb[P * NW] = (int32_t)gbn;
    spmv_status_t s;
    if ((s = upload(h, &h->d_xs_panel, desc.data(), P))) return s;
    if ((s = upload(h, &h->d_xs_wg, wg.data(), P * NW + 1))) return s;
    if ((s = upload(h, &h->d_xs_wb, wb.data(), P * NW + 1))) return s;
    if ((s = dalloc(h, &h->d_xs_U, std::max<int64_t>(nu, 1)))) return s;
    if ((s = dalloc(h, &h->d_xs_gval, gi * 32))) return s;
    if ((s = dalloc(h, &h->d_xs_gidx, gi * 32))) return s;
    if ((s = dalloc(h, &h->d_xs_bval, gbn * 32))) return s;
    if ((s = dalloc(h, &h->d_xs_bidx, gbn * 32))) return s;
    for (int64_t p = 0; p < P; ++p) {
        spmvb::XsPanelData& D = pd[p];
        const int64_t go = wg[p * NW], bo = wb[p * NW];
        if (!D.u_rel.empty() && D.desc.nch)
            CUDA_TRY(cudaMemcpy(h->d_xs_U + D.desc.u_base, D.u_rel.data(), (size_t)NW * D.desc.nch * 4,
                                cudaMemcpyHostToDevice));
        if (!D.gval.empty()) {
            CUDA_TRY(cudaMemcpy(h->d_xs_gval + go * 32, D.gval.data(), D.gval.size() * 8, cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(h->d_xs_gidx + go * 32, D.gidx.data(), D.gidx.size() * 4, cudaMemcpyHostToDevice));
        }
        if (!D.bval.empty()) {
            CUDA_TRY(cudaMemcpy(h->d_xs_bval + bo * 32, D.bval.data(), D.bval.size() * 8, cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(h->d_xs_bidx + bo * 32, D.bidx.data(), D.bidx.size() * 4, cudaMemcpyHostToDevice));
        }
        std::vector<double>().swap(D.gval);
        std::vector<uint32_t>().swap(D.gidx);
        std::vector<double>().swap(D.bval);
        std::vector<uint32_t>().swap(D.bidx);
    }
    h->xs_cbits = cbits;
    h->xs_panels = P;
    h->xs_groups = gi + gbn;
    h->xs_pad = st.pad_i + st.pad_b;
    h->bytes_stream = 12 * 32 * (gi + gbn) + 8 * (P * NW + 1) * 2 + 4 * nu + 8 * h->m_loc;
    h->kernel = 6;
    return SPMV_OK;
}

// The panel plan's layout decisions for one rank (pure host logic, shared by
// plan_pn and the spmv_pn_shard_hash test hook): its row ranges (SB blocks,
// else all rows), their interior column ranges (rotation, x prefetch), the
// panel size target and whole-wave count, the x split, and -- for SB
// handles without a split -- each range's panel count from the global
// per-block slot counts, so a block's panels do not depend on the GPU count.
struct PnSetup {
    std::vector<std::pair<int64_t, int64_t>> ranges, xcols;
    std::vector<int64_t> range_panels;
    int64_t target = 0, waves = 0, xs = INT32_MAX, sms = 148;
    bool global = false;
};

static PnSetup pn_setup(int kind, int world, int64_t row_begin, int64_t m_loc, int64_t x_int_begin, int64_t x_int_len,
                        int64_t n, const std::vector<int64_t>& rbp, const std::vector<int64_t>& cbp,
                        const std::vector<int64_t>& blk_slots, const std::vector<int64_t>& rp,
                        const std::vector<int32_t>* part, int64_t sms) {
    PnSetup S;
    S.sms = sms;
    const int K = (int)rbp.size() - 2;
    const int64_t R0 = row_begin, R1 = row_begin + m_loc;
    const int64_t q0 = world > 1 ? x_int_begin : 0;
    if (kind == SPMV_SB) {
        for (int k = 0; k < K; ++k) {
            const int64_t a = std::max(rbp[k], R0), b = std::min(rbp[k + 1], R1);
            if (b > a) {
                S.ranges.push_back({a - R0, b - R0});
                S.xcols.push_back({cbp[k] - q0, cbp[k + 1] - q0});
            }
        }
    } else {   // no SB structure: panels of consecutive rows, no x prefetch
        S.ranges.push_back({0, m_loc});
        if (getenv("SPMV_PN_ROT_GENERIC")) S.xcols.push_back({0, n});   // measurement: rotated sweeps
    }
    // the global per-block counts (SB, no split) decide the cuts, else this rank's rows
    S.global = kind == SPMV_SB && !part && K > 0 && (int)blk_slots.size() == K;
    int64_t total_slots = 0;
    if (S.global)
        for (int64_t v : blk_slots) total_slots += v;
    else
        total_slots = spmvb::panel_total_slots(rp, m_loc, part);
    // panels: about kPnRowsTarget slots, their count a multiple of the SM
    // count when possible (whole waves of one CTA per SM)
    S.target = spmvb::kPnRowsTarget;
    for (int64_t k = 1; k <= 4096; ++k) {
        const int64_t r = (total_slots + sms * k - 1) / (sms * k);
        if (r <= spmvb::kPnRowsTarget) {
            S.target = r;
            S.waves = k;
            break;
        }
    }
    if (S.target < 1024) {
        S.target = 1024;
        S.waves = 0;
    }
    if (const char* e = getenv("SPMV_PN_ROWS")) {   // tests / measurements
        S.target = std::max<int64_t>(1, atoll(e));
        S.waves = 0;
    }
    if (getenv("SPMV_PN_NOWAVES")) S.waves = 0;   // measurement: per-range ceil(slots / target)
    // groups never mix interior and border columns at world > 1 (two x
    // buffers); SB plans keep the same rule at world 1 (C_B starts at
    // cbp[K]) so the groups -- and every row's summation order -- are the
    // same on any number of GPUs
    S.xs = world > 1 ? x_int_len : (kind == SPMV_SB ? cbp[K] : INT32_MAX);
    if (S.global) {
        const std::vector<int64_t> np_all = spmvb::panel_counts(blk_slots, S.target, S.waves * sms);
        for (int k = 0; k < K; ++k)
            if (std::min(rbp[k + 1], R1) > std::max(rbp[k], R0)) S.range_panels.push_back(np_all[k]);
    }
    return S;
}

// Builds and uploads the column-sorted panel kernel's plan (plan_panel.cpp).
// Leaves the handle on the row-tile kernel when the plan would be poor.
static spmv_status_t plan_pn(spmv_plan_s* h, PanelPlan& pl, const std::vector<int64_t>& rp,
                             const std::vector<int32_t>& pcol, const std::vector<double>& pval,
                             const std::vector<int64_t>& rbp, const std::vector<int64_t>& cbp,
                             const std::vector<int32_t>* part) {
    if (const char* e = getenv("SPMV_L2_PERSIST_MB")) {   // measurements: L2 set-aside for evict_last lines
        CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)atoll(e) << 20));
    }
    const PnSetup S = pn_setup(h->kind, h->world, h->row_begin, h->m_loc, h->x_int_begin, h->x_int_len, h->n, rbp, cbp,
                               h->blk_slots, rp, part, spmvb::kernel_num_sms());
    std::vector<spmvb::PnPanelData> pd;
    spmvb::PnPlanStats st;
    std::string why;
    if (!spmvb::plan_panel(rp, pcol, pval, S.ranges, S.xs, S.target, pd, st, why, S.xcols.empty() ? nullptr : &S.xcols,
                           S.sms, part, S.waves * S.sms, S.global ? &S.range_panels : nullptr))
        return SPMV_OK;
    if (st.entries != h->nnz_loc)
        return fail(SPMV_ERR_INTERNAL, "panel plan lost nonzeros (%lld of %lld)", (long long)st.entries,
                    (long long)h->nnz_loc);
    const char* kenv = getenv("SPMV_KERNEL");
    const bool forced = kenv && strcmp(kenv, "panel") == 0;
    if (!forced && st.pads > st.entries / 4) return SPMV_OK;   // > 25 % padding: the row-tile kernel is cheaper
    const int64_t P = (int64_t)pd.size(), G = st.groups;
    std::vector<spmvb::PnPanel> desc(P);
    for (int64_t p = 0; p < P; ++p) desc[p] = pd[p].desc;
    spmv_status_t s;
    if ((s = upload(h, &pl.d_panel, desc.data(), P))) return s;
    // + kPnPadGroups zero groups: the kernel's register ring reads ahead past
    // the last panel's last epoch without bounds checks
    const int64_t Gp = G + spmvb::kPnPadGroups;
    if ((s = dalloc(h, &pl.d_gval, Gp * 32))) return s;
    if ((s = dalloc(h, &pl.d_gidx, Gp * 32))) return s;
    if ((s = dalloc(h, &pl.d_gbase4, Gp))) return s;
    CUDA_TRY(cudaMemset(pl.d_gval + G * 32, 0, spmvb::kPnPadGroups * 32 * sizeof(double)));
    CUDA_TRY(cudaMemset(pl.d_gidx + G * 32, 0, spmvb::kPnPadGroups * 32 * sizeof(uint32_t)));
    CUDA_TRY(cudaMemset(pl.d_gbase4 + G, 0, spmvb::kPnPadGroups * sizeof(int32_t)));
    {
        std::vector<uint16_t> r2s(std::max<int64_t>(h->m_loc, 1), 0);
        std::vector<int32_t> sf, sc, sr;
        std::vector<uint16_t> ss;
        pl.max_sslots = 0;
        pl.max_split_n = 0;
        for (int64_t p = 0; p < P; ++p) {
            std::copy(pd[p].row2slot.begin(), pd[p].row2slot.end(), r2s.begin() + pd[p].desc.row0);
            desc[p].split_off = (int32_t)sf.size();
            desc[p].nslots = pd[p].nslots;
            const int32_t base = (int32_t)ss.size();
            desc[p].split_n = (int32_t)pd[p].split_first.size();
            desc[p].split_short = pd[p].split_short;
            desc[p].sslot0 = base;
            desc[p].sslot_n = (int32_t)pd[p].split_slots.size();
            pl.max_sslots = std::max(pl.max_sslots, desc[p].sslot_n);
            pl.max_split_n = std::max(pl.max_split_n, desc[p].split_n);
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
        CUDA_TRY(cudaMemcpy(pl.d_panel, desc.data(), P * sizeof(spmvb::PnPanel), cudaMemcpyHostToDevice));
    }
    pl.max_rows = 0;
    for (int64_t p = 0; p < P; ++p) pl.max_rows = std::max(pl.max_rows, (pd[p].nslots + 15) & ~15);
    // padding lanes: the planner's dummy index becomes the scratch y slot
    // max_rows (delta 0: a valid x read, times the value 0)
    const uint32_t dummy_dev = (uint32_t)pl.max_rows << spmvb::kPnDeltaBits;
    std::vector<double> tv;
    std::vector<uint32_t> ti;
    for (int64_t p = 0; p < P; ++p) {
        spmvb::PnPanelData& D = pd[p];
        const int64_t g0 = D.desc.g0, ng = (int64_t)D.gbase.size();
        if (ng) {
            // device layout of the group stream (panel.cu): per (epoch, warp) a
            // 128-entry block; values as (step pair, lane, step & 1), indices as
            // (lane, step), so 16-byte loads cover 2 / 4 of a warp's steps
            tv.resize(ng * 32);
            ti.resize(ng * 32);
            for (int64_t g = 0; g < ng; ++g) {
                const int64_t q = g / spmvb::kPnWarps, w = g % spmvb::kPnWarps;   // g = (e * 4 + b) * 16 + w
                const int64_t e = q / spmvb::kPnB, b = q % spmvb::kPnB;
                const int64_t blk = (e * spmvb::kPnWarps + w) * 128;
                for (int l = 0; l < 32; ++l) {
                    tv[blk + (b / 2) * 64 + l * 2 + (b & 1)] = D.gval[g * 32 + l];
                    const uint32_t i = D.gidx[g * 32 + l];
                    ti[blk + l * 4 + b] = i == spmvb::kPnDummy ? dummy_dev : i;
                }
            }
            CUDA_TRY(cudaMemcpy(pl.d_gval + g0 * 32, tv.data(), ng * 32 * 8, cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(pl.d_gidx + g0 * 32, ti.data(), ng * 32 * 4, cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(pl.d_gbase4 + g0, D.gbase4.data(), ng * 4, cudaMemcpyHostToDevice));
        }
        std::vector<double>().swap(D.gval);
        std::vector<uint32_t>().swap(D.gidx);
        std::vector<int32_t>().swap(D.gbase);
        std::vector<int32_t>().swap(D.gbase4);
    }
    pl.panels = P;
    pl.groups = G;
    pl.pad = st.pads;
    pl.gsectors = st.gsectors;
    // SB blocks: a panel's gathers rarely revisit an x line across groups, and
    // skipping the L1 allocation leaves the L1 to the loads in flight
    // (interleaved A/B on C5: -0.9 %, 5 of 6 rounds); matrices without blocks
    // (C4: band columns revisited) keep allocating (+8 % without)
    pl.gather_na = h->kind == SPMV_SB ? 1 : 0;
    if (const char* e = getenv("SPMV_PN_GATHER_NA")) pl.gather_na = atoi(e);
    if (const char* e = getenv("SPMV_PN_RING")) pl.ring = atoi(e);   // measurements: 8, 12 or 16
    if (const char* e = getenv("SPMV_PN_PF")) pl.pf = atoi(e);       // measurements: epochs ahead
    if (const char* e = getenv("SPMV_PN_PERSIST")) pl.persist = atoi(e);
    if (!part) {
        h->bytes_stream = (12 * 32 + 4) * G + 8 * h->m_loc;
        h->kernel = 7;
    }
    return SPMV_OK;
}

static spmv_status_t create_impl(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                                 const int32_t* col_idx, const double* val, const int32_t* row_perm,
                                 const int32_t* col_perm, const spmv_blocks_t* blocks, int32_t n_parts,
                                 const int32_t* part_of_nnz, const spmv_dist_t* dist, spmv_plan_s* h) {
    // ---------------------------------------------------------- arguments
    if (m < 0 || n < 0 || nnz < 0) return fail(SPMV_ERR_USAGE, "negative dimension");
    if (!row_ptr) return fail(SPMV_ERR_USAGE, "row_ptr is NULL");
    if (nnz > 0 && (!col_idx || !val)) return fail(SPMV_ERR_USAGE, "col_idx/val is NULL");
    if (n_parts < 0 || (n_parts > 0 && !part_of_nnz)) return fail(SPMV_ERR_USAGE, "bad split arguments");
    if (n_parts > spmvb::kMaxParts) return fail(SPMV_ERR_UNSUPPORTED, "more than %d split parts", spmvb::kMaxParts);
    if (m > INT32_MAX - 1 || n > INT32_MAX - 1) return fail(SPMV_ERR_UNSUPPORTED, "dimension beyond int32");
    const int world = dist ? dist->world : 1;
    const int rank = dist ? dist->rank : 0;
    // test rank (spmv_test_set_border): a multi-GPU shard without a communicator
    const bool test_nocomm = dist && world > 1 && !dist->nccl_unique_id && getenv("SPMV_TEST_RANKS_NO_NCCL");
    if (dist && (world < 1 || rank < 0 || rank >= world || (!dist->nccl_unique_id && !test_nocomm)))
        return fail(SPMV_ERR_USAGE, "bad dist descriptor");
    h->test_nocomm = test_nocomm;
    if (world > 1 && (!blocks || blocks->kind != SPMV_SB))
        return fail(SPMV_ERR_UNSUPPORTED, "world > 1 needs an SB block descriptor (DB split sharding is NEXT f1)");
    h->rank = rank;
    h->world = world;
    h->m = m; h->n = n; h->nnz = nnz;
    h->n_parts = n_parts;
    h->has_perm = row_perm || col_perm;

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
    std::vector<int64_t> rbp, cbp, bop;
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
        bop.resize(K + 1);
        if (blocks->border_owner_ptr) {
            for (int k = 0; k <= K; ++k) bop[k] = blocks->border_owner_ptr[k];
            if (bop[0] != cbp[K] || bop[K] != cbp[K + 1])
                return fail(SPMV_ERR_DATA, "border_owner_ptr does not cover C_B");
            for (int k = 0; k < K; ++k)
                if (bop[k + 1] < bop[k]) return fail(SPMV_ERR_DATA, "border_owner_ptr not nondecreasing");
        } else {
            for (int k = 0; k <= K; ++k) bop[k] = cbp[K] + (h->border_total * k) / K;
        }
    }

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
    h->m_loc = R1 - R0;
    h->x_int_begin = sh.x_interior_begin;
    h->x_int_len = sh.x_interior_len;
    h->x_bord_begin = sh.x_border_begin;
    h->x_bord_len = sh.x_border_len;
    h->x_local_len = sh.x_local_len;

    // ---------------------------------------------- NCCL bootstrap (a4)
    if (world > 1) {
        h->device = dist->device;
        CUDA_TRY(cudaSetDevice(h->device));
        if (!test_nocomm) {
            ncclUniqueId id;
            memcpy(&id, dist->nccl_unique_id, sizeof id);
            NCCL_TRY(ncclCommInitRank(&h->comm, world, id, rank));
        }
    }

    // --------------------------------------- permute the local rows (a1)
    // new row p has the entries of old row row_inv[p], columns mapped through
    // col_perm, sorted by new column; duplicates rejected (reading A3).
    const int64_t m_loc = h->m_loc;
    std::vector<int64_t> rp(m_loc + 1);
    rp[0] = 0;
    for (int64_t p = 0; p < m_loc; ++p) {
        const int64_t i = row_inv[R0 + p];
        rp[p + 1] = rp[p] + (row_ptr[i + 1] - row_ptr[i]);
    }
    const int64_t nnz_loc = rp[m_loc];
    h->nnz_loc = nnz_loc;
    spmv_status_t local_status = SPMV_OK;
    if (nnz_loc + kPad >= INT32_MAX) local_status = fail(SPMV_ERR_UNSUPPORTED, "shard nnz beyond int32");

    std::vector<int32_t> pcol, lcol;
    std::vector<double> pval;
    std::vector<int32_t> ppart;
    std::vector<int64_t> n_long_rows;
    if (local_status == SPMV_OK) {
        pcol.resize(nnz_loc);
        pval.resize(nnz_loc);
        if (n_parts) ppart.resize(nnz_loc);
        std::atomic<int> dup{0}, env{0};
        const bool sb_env = blocks != nullptr;
#pragma omp parallel
        {
            std::vector<int64_t> idx;
            std::vector<int32_t> key;
#pragma omp for schedule(dynamic, 2048)
            for (int64_t p = 0; p < m_loc; ++p) {
                const int64_t i = row_inv[R0 + p];
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
                for (int64_t t = 0; t < L; ++t) {
                    const int64_t s = idx[t];
                    pcol[o + t] = key[s];
                    pval[o + t] = val[a + s];
                    if (n_parts) ppart[o + t] = part_of_nnz[a + s];
                    if (t && pcol[o + t] == pcol[o + t - 1]) dup = 1;
                }
                if (sb_env) {   // envelope of Eq.(1)/(5)
                    const int64_t gp = R0 + p;
                    const int64_t k = std::upper_bound(rbp.begin(), rbp.begin() + K + 1, gp) - rbp.begin() - 1;
                    if (k < K) {
                        for (int64_t t = 0; t < L; ++t) {
                            const int64_t c = pcol[o + t];
                            if (!((c >= cbp[k] && c < cbp[k + 1]) || c >= cbp[K])) { env = 1; break; }
                        }
                    }
                }
            }
        }
        if (dup) local_status = fail(SPMV_ERR_DATA, "duplicate (i, j) entry");
        else if (env) local_status = fail(SPMV_ERR_DATA, "nonzero outside the SB/DB envelope");
    }
    if (world > 1 && !test_nocomm) {   // every rank returns the same status
        int* d_st = nullptr;
        int st = (int)local_status;
        CUDA_TRY(cudaMalloc(&d_st, sizeof(int)));
        CUDA_TRY(cudaMemcpy(d_st, &st, sizeof(int), cudaMemcpyHostToDevice));
        NCCL_TRY(ncclAllReduce(d_st, d_st, 1, ncclInt32, ncclMax, h->comm, 0));
        CUDA_TRY(cudaMemcpy(&st, d_st, sizeof(int), cudaMemcpyDeviceToHost));
        cudaFree(d_st);
        if (st != SPMV_OK && local_status == SPMV_OK)
            local_status = fail((spmv_status_t)st, "create failed on another rank");
    }
    if (local_status != SPMV_OK) return local_status;
    if (world == 1) {
        if (dist) h->device = dist->device;
        else CUDA_TRY(cudaGetDevice(&h->device));
        CUDA_TRY(cudaSetDevice(h->device));
    }

    // -------------------------------------- local column ids (x layout)
    // world 1: global permuted ids.  world > 1: [interior | full C_B] where
    // the kernel reads c < x_int_len from the user's x and the rest from the
    // gathered border buffer.
    if (world > 1) {
        const int64_t Q0 = h->x_int_begin, B0 = h->border_begin, nint = h->x_int_len;
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < nnz_loc; ++t) {
            const int64_t c = pcol[t];
            pcol[t] = (int32_t)(c >= B0 ? nint + (c - B0) : c - Q0);
        }
    }

    // ------------------------------------------------------ tiles (a2)
    std::vector<int64_t> cuts;
    if (blocks)
        for (int k = 1; k <= K; ++k)
            if (rbp[k] > R0 && rbp[k] < R1) cuts.push_back(rbp[k] - R0);
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
        std::vector<int32_t> tile_cls(std::max<int64_t>(T, 1), spmvb::kTileGeneral);
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < T; ++t) {
            int64_t mx = 0;
            for (int64_t r = tile_row[t]; r < tile_row[t + 1]; ++r) mx = std::max(mx, rp[r + 1] - rp[r]);
            // short tiles: lanes per row V = largest power of two with
            // rows * V <= 512 (rowtile.cu CTA), capped at 32 and at the
            // longest row rounded up to a power of two
            int32_t cls = spmvb::kTileGeneral;
            if (mx <= spmvb::kShortRow) {
                const int64_t nr = tile_row[t + 1] - tile_row[t];
                int32_t V = 1;
                while (V < 32 && nr * (2 * V) <= 512 && V < mx) V *= 2;
                cls = V;
            }
            tile_cls[t] = cls;
        }
        if ((s = upload(h, &h->d_tile_cls, tile_cls.data(), T))) return s;
        {
            std::vector<int32_t> lt;
            for (int64_t t = 0; t < T; ++t)
                if (rp[tile_row[t + 1]] - rp[tile_row[t]] + 3 > kTileNnz) lt.push_back((int32_t)t);
            if (!lt.empty() && (s = upload(h, &h->d_long_tiles, lt.data(), lt.size()))) return s;
            h->n_long = (int64_t)lt.size();
        }
        const char* kenv = getenv("SPMV_KERNEL");   // A/B switch for measurements only
        h->kernel = 0;
        if (kenv && strcmp(kenv, "pipe") == 0) h->kernel = 1;
        if (kenv && strcmp(kenv, "tile") == 0) h->kernel = 2;
        if (kenv && strcmp(kenv, "rowtile512") == 0) h->kernel = 3;
        if (kenv && strcmp(kenv, "rowseg") == 0) h->kernel = 4;
        if (kenv && strcmp(kenv, "rowtile128") == 0) h->kernel = 5;
        if (kenv && strcmp(kenv, "rowlin") == 0) h->kernel = 8;
    }
    h->bytes_stream = 12 * nnz_loc + 4 * (m_loc + 1) + 8 * m_loc;

    // -------------------------------------------- split layout (a8)
    // Within each row tile the nonzeros are regrouped part-major: for k = 0..K-1,
    // the tile's rows' part-k runs ("segments") in row order.  This is the
    // access order that Pi defines, executed tile by tile.
    if (n_parts) {
        const int KP = n_parts;
        std::vector<int64_t> seg_cnt(T * KP, 0), nz_cnt(T * KP, 0);
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t t = 0; t < T; ++t) {
            std::vector<int64_t> stamp(KP, -1);   // last row that opened a part-k segment
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
        std::vector<int32_t> seg_ptr(S + 1), seg_row(S), scol(nnz_loc);
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
        // row-major fused layout: row r's entries regrouped by part (stable in
        // column order inside a part); segments in part order per row
        {
            std::vector<int32_t> fcol(nnz_loc), frowseg(m_loc + 1), fsegptr(S + 1);
            std::vector<double> fval(nnz_loc);
            std::vector<int32_t> rcnt(m_loc);
#pragma omp parallel for schedule(dynamic, 4096)
            for (int64_t r = 0; r < m_loc; ++r) {
                // distinct parts of the row = its segments
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

    // ---------------- fused multiple-SpMxV on panels (a8): (row, part) virtual rows
    if (n_parts && world == 1 && nnz_loc > 0 && !getenv("SPMV_SPLIT_ROWTILE")) {
        if ((s = plan_pn(h, h->pns, rp, pcol, pval, rbp, cbp, &ppart))) return s;
    }

    if (blocks && h->kind == SPMV_SB && world == 1 && getenv("SPMV_PN_XS_TEST") && cbp.size() >= 2)
        h->xs_test = cbp[cbp.size() - 2];   // C_B's first column: the plan's group split (pn_setup)
    // global per-block y-slot counts (SB): every rank cuts its blocks into the
    // same panels as a single GPU would, so the summation order of a row --
    // and y -- does not depend on the number of GPUs
    if (blocks && h->kind == SPMV_SB && nnz_loc > 0) {
        const int K = (int)rbp.size() - 2;
        h->blk_slots.assign(K, 0);
        std::vector<int64_t> loc(K, 0);
        for (int64_t i = 0; i < m; ++i) {
            const int64_t nr = row_perm ? row_perm[i] : i;
            const int k = (int)(std::upper_bound(rbp.begin(), rbp.begin() + K + 1, nr) - rbp.begin()) - 1;
            if (k >= 0 && k < K) loc[k] += spmvb::row_slots(row_ptr[i + 1] - row_ptr[i]);
        }
        h->blk_slots = loc;
    }

    // ------------------------------------ x-staged plan (SB handles, a5/a6)
    {
        const char* kenv = getenv("SPMV_KERNEL");
        const bool sb = blocks && h->kind == SPMV_SB && nnz_loc > 0;
        // any matrix at world 1: panels of consecutive rows (C4: 0.231 vs 0.259 ms for the
        // row-tile kernel); small matrices fall back to row tiles through the padding test
        const bool generic = nnz_loc > 0 && world == 1;
        if (sb && kenv && strcmp(kenv, "xstage") == 0) {
            if ((s = plan_xs(h, rp, pcol, pval, rbp, cbp))) return s;
        } else if ((sb || generic) && (!kenv || strcmp(kenv, "panel") == 0)) {
            if ((s = plan_pn(h, h->pn, rp, pcol, pval, rbp, cbp, nullptr))) return s;
        }
    }

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
    // Square A: column c (new) is old column j = col_inv[c]; as a row, old j
    // is new row row_perm[j].  x^_{t+1}[c] = y^_t[row_perm[col_inv[c]]] / m.
    if (m == n && m > 0) {
        std::vector<int32_t> owner(h->x_local_len);
        std::atomic<int> outside{0};
#pragma omp parallel for schedule(static)
        for (int64_t l = 0; l < h->x_local_len; ++l) {
            const int64_t c = (world > 1) ? (l < h->x_int_len ? h->x_int_begin + l
                                                              : h->x_bord_begin + (l - h->x_int_len))
                                          : l;
            const int64_t j = col_inv[c];
            const int64_t r = row_perm ? row_perm[j] : j;
            if (r < R0 || r >= R1) { outside = 1; owner[l] = 0; }
            else owner[l] = (int32_t)(r - R0);
        }
        if (!outside) {
            if ((s = upload(h, &h->d_owner, owner.data(), h->x_local_len))) return s;
            h->has_owner = true;
        }
    }

    // ------------------------------------------------- misc buffers
    if ((s = dalloc(h, &h->d_slots, spmvb::kMaxSlots * spmvb::kSlotStride))) return s;
    CUDA_TRY(cudaMemset(h->d_slots, 0, spmvb::kMaxSlots * spmvb::kSlotStride * sizeof(unsigned long long)));
    if ((s = dalloc(h, &h->d_mscratch, 2))) return s;
    if ((s = dalloc(h, &h->d_counter, 4))) return s;
    if (world > 1) {
        if ((s = dalloc(h, &h->d_xborder, h->border_total))) return s;
        CUDA_TRY(cudaMemset(h->d_xborder, 0, std::max<int64_t>(h->border_total, 1) * sizeof(double)));
    }
    CUDA_TRY(cudaDeviceSynchronize());
    return SPMV_OK;
}

spmv_status_t spmv_create(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                          const double* val, const int32_t* row_perm, const int32_t* col_perm,
                          const spmv_blocks_t* blocks, int32_t n_parts, const int32_t* part_of_nnz,
                          const spmv_dist_t* dist, spmv_handle_t* out) {
    if (!out) return fail(SPMV_ERR_USAGE, "out is NULL");
    *out = nullptr;
    spmv_plan_s* h = new (std::nothrow) spmv_plan_s();
    if (!h) return fail(SPMV_ERR_INTERNAL, "out of host memory");
    spmv_status_t s;
    try {
        s = create_impl(m, n, nnz, row_ptr, col_idx, val, row_perm, col_perm, blocks, n_parts, part_of_nnz,
                        dist, h);
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

spmv_status_t spmv_destroy(spmv_handle_t h) {
    if (!h) return SPMV_OK;
    if (!valid(h)) return fail(SPMV_ERR_USAGE, "invalid handle");
    free_plan(h);
    return SPMV_OK;
}

// --------------------------------------------------------------- apply
static spmv_status_t check_vectors(spmv_handle_t h, const double* x, int64_t x_len, double* y, int64_t y_len,
                                   uint32_t flags) {
    if (!valid(h)) return fail(SPMV_ERR_USAGE, "invalid handle");
    if (flags & ~(uint32_t)(SPMV_VEC_ORIGINAL | SPMV_FUSE_MAXABS | SPMV_SPLIT_LITERAL))
        return fail(SPMV_ERR_USAGE, "unknown flag");
    if ((!x && x_len) || (!y && y_len)) return fail(SPMV_ERR_USAGE, "NULL vector");
    if ((const void*)x == (const void*)y && x) return fail(SPMV_ERR_USAGE, "x and y alias");
    if (((uintptr_t)x & 7) || ((uintptr_t)y & 7)) return fail(SPMV_ERR_USAGE, "x/y not 8-byte aligned");
    if (h->kernel == 6 && !(flags & SPMV_VEC_ORIGINAL) && ((uintptr_t)x & 15))
        return fail(SPMV_ERR_USAGE, "x not 16-byte aligned (the x-staged kernel bulk-copies x)");
    const bool orig = flags & SPMV_VEC_ORIGINAL;
    if (orig && h->world > 1) return fail(SPMV_ERR_UNSUPPORTED, "ORIGINAL index space with world > 1");
    const int64_t xl = orig ? h->n : h->x_local_len;
    const int64_t yl = orig ? h->m : h->m_loc;
    if (x_len != xl || y_len != yl)
        return fail(SPMV_ERR_DATA, "dimension mismatch: x_len %lld (want %lld), y_len %lld (want %lld)",
                    (long long)x_len, (long long)xl, (long long)y_len, (long long)yl);
    return SPMV_OK;
}

static void fill_pn_args(const PanelPlan& pl, spmvb::PnArgs& X) {
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
    X.ring = pl.ring;
    X.pf_epochs = pl.pf;
    X.persist = pl.persist;
}

static spmv_status_t run(spmv_handle_t h, const double* x, double* y, uint32_t flags, cudaStream_t st,
                         bool split) {
    CUDA_TRY(cudaSetDevice(h->device));
    const bool orig = (flags & SPMV_VEC_ORIGINAL) && h->has_perm;
    const double* xk = x;
    double* yk = y;
    if (orig) {   // a3: x^[c] = x[col_inv[c]]
        CUDA_TRY(spmvb::launch_gather(x, h->d_colinv, h->d_xhat, h->n, st));
        xk = h->d_xhat;
        yk = h->d_yhat;
    }
    spmvb::TileArgs A{};
    A.tile_row = h->d_tile_row;
    A.n_tiles = (int32_t)h->n_tiles;
    A.y = yk;
    A.x_lo = xk;
    A.x_hi = xk;
    A.x_split = INT32_MAX;
    bool xsplit = false;
    if (h->world > 1) {   // a4: border-x exchange over NCCL
        if (h->x_bord_len)
            CUDA_TRY(cudaMemcpyAsync(h->d_xborder + h->bord_off[h->rank], x + h->x_int_len,
                                     h->x_bord_len * sizeof(double), cudaMemcpyDeviceToDevice, st));
        if (h->test_nocomm) {
            // test rank: the other slices were supplied by spmv_test_set_border
        } else if (h->equal_slices) {
            NCCL_TRY(ncclAllGather(h->d_xborder + h->bord_off[h->rank], h->d_xborder, h->bord_cnt[0], ncclFloat64,
                                   h->comm, st));
        } else {
            NCCL_TRY(ncclGroupStart());
            for (int r = 0; r < h->world; ++r)
                if (h->bord_cnt[r])
                    NCCL_TRY(ncclBroadcast(h->d_xborder + h->bord_off[r], h->d_xborder + h->bord_off[r],
                                           h->bord_cnt[r], ncclFloat64, r, h->comm, st));
            NCCL_TRY(ncclGroupEnd());
        }
        A.x_hi = h->d_xborder;
        A.x_split = (int32_t)h->x_int_len;
        xsplit = true;
    }
    if (flags & SPMV_FUSE_MAXABS) {
        CUDA_TRY(cudaMemsetAsync(h->d_slots, 0,
                                 spmvb::kMaxSlots * spmvb::kSlotStride * sizeof(unsigned long long), st));
        A.maxabs_slots = h->d_slots;
    }
    if (!split && h->kernel == 7) {
        spmvb::PnArgs X{};
        fill_pn_args(h->pn, X);
        X.x_split = A.x_split;
        X.x_lo = A.x_lo;
        X.x_hi = A.x_hi;
        if (h->xs_test > 0 && h->world == 1) {   // test: the world > 1 two-buffer x path on one GPU
            X.x_split = (int32_t)h->xs_test;
            X.x_hi = A.x_lo + h->xs_test;
        }
        X.y = yk;
        X.maxabs_slots = A.maxabs_slots;
        CUDA_TRY(spmvb::launch_panel(X, st));
    } else if (!split && h->kernel == 6) {
        spmvb::XsArgs X{};
        X.panel = h->d_xs_panel;
        X.n_panels = (int32_t)h->xs_panels;
        X.cbits = h->xs_cbits;
        X.wg = h->d_xs_wg;
        X.wb = h->d_xs_wb;
        X.U = h->d_xs_U;
        X.gval = h->d_xs_gval;
        X.gidx = h->d_xs_gidx;
        X.bval = h->d_xs_bval;
        X.bidx = h->d_xs_bidx;
        X.x = xk;
        X.xg = xsplit ? A.x_hi : xk + h->xs_gb;
        X.y = yk;
        X.maxabs_slots = A.maxabs_slots;
        CUDA_TRY(spmvb::launch_xstage(X, st));
    } else if (!split && h->kernel != 2) {
        spmvb::PipeArgs P{};
        P.tile_row = h->d_tile_row;
        P.tile_nnz = h->d_tile_nnz;
        P.tile_cls = h->d_tile_cls;
        P.rowptr = h->d_rowptr;
        P.col = h->d_col;
        P.val = h->d_val;
        P.x_lo = A.x_lo;
        P.x_hi = A.x_hi;
        P.x_split = A.x_split;
        P.n_tiles = A.n_tiles;
        P.y = A.y;
        P.maxabs_slots = A.maxabs_slots;
        P.tile_counter = h->d_counter;
        // x gathers: L1 no-allocate (a gathered line is not reused by the tile) and
        // L2 evict-last (x is the reused operand; the matrix streams evict-first)
        P.gmode = 2;
        if (const char* g = getenv("SPMV_RT_GMODE")) P.gmode = atoi(g);   // measurements only
        const bool rowtile_family = h->kernel == 0 || h->kernel == 3 || h->kernel == 5 || h->kernel == 8;
        const char* lenv = getenv("SPMV_LONG");   // measurements: "separate" / "side" stream; default inline
        if (rowtile_family && h->d_long_tiles && lenv) P.long_tiles = h->d_long_tiles;
        const bool side = P.long_tiles && strcmp(lenv, "side") == 0;
        if (side) {
            if (!h->side) {
                CUDA_TRY(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
                CUDA_TRY(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
                CUDA_TRY(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
            }
            CUDA_TRY(cudaEventRecord(h->ev_fork, st));
            CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
            CUDA_TRY(spmvb::launch_longrows(P, (int32_t)h->n_long, xsplit, h->side));
            CUDA_TRY(cudaEventRecord(h->ev_join, h->side));
        }
        if (h->kernel == 1) CUDA_TRY(spmvb::launch_pipe(P, xsplit, st));
        else if (h->kernel == 3) CUDA_TRY(spmvb::launch_rowtile(P, xsplit, 512, st));
        else if (h->kernel == 4) CUDA_TRY(spmvb::launch_rowseg(P, xsplit, st));
        else if (h->kernel == 5) CUDA_TRY(spmvb::launch_rowtile(P, xsplit, 128, st));
        else if (h->kernel == 8) CUDA_TRY(spmvb::launch_rowtile(P, xsplit, 256, st, true));
        else CUDA_TRY(spmvb::launch_rowtile(P, xsplit, 256, st));
        if (side) CUDA_TRY(cudaStreamWaitEvent(st, h->ev_join, 0));
        else if (P.long_tiles) CUDA_TRY(spmvb::launch_longrows(P, (int32_t)h->n_long, xsplit, st));
    } else if (!split) {
        A.tile_seg = h->d_tile_row;
        A.seg_ptr = h->d_rowptr;
        A.seg_row = nullptr;
        A.col = h->d_col;
        A.val = h->d_val;
        A.K = 1; A.k_begin = 0; A.k_end = 1;
        CUDA_TRY(spmvb::launch_tiles(A, false, xsplit, st));
    } else {
        A.tile_seg = h->d_tile_seg;
        A.seg_ptr = h->d_seg_ptr;
        A.seg_row = h->d_seg_row;
        A.col = h->d_scol;
        A.val = h->d_sval;
        A.K = h->n_parts;
        if (flags & SPMV_SPLIT_LITERAL) {   // y = 0; y <- y + A^k x, one pass per k
            CUDA_TRY(cudaMemsetAsync(yk, 0, h->m_loc * sizeof(double), st));
            for (int k = 0; k < h->n_parts; ++k) {
                spmvb::TileArgs B = A;
                B.k_begin = k; B.k_end = k + 1;
                B.accumulate = 1;
                if (k != h->n_parts - 1) B.maxabs_slots = nullptr;
                if (h->kernel == 2) CUDA_TRY(spmvb::launch_tiles(B, true, xsplit, st));
                else CUDA_TRY(spmvb::launch_split(B, xsplit, st));
            }
        } else if (h->pns.ok() && h->kernel != 2) {
            // fused multiple-SpMxV on column-sorted panels: each (row, part)
            // segment accumulates in its own y slot, folded per row
            spmvb::PnArgs X{};
            fill_pn_args(h->pns, X);
            X.x_split = A.x_split;
            X.x_lo = A.x_lo;
            X.x_hi = A.x_hi;
            X.y = yk;
            X.maxabs_slots = A.maxabs_slots;
            CUDA_TRY(spmvb::launch_panel(X, st));
        } else if (h->split_rowmajor && h->kernel != 2 && !getenv("SPMV_SPLIT_PARTMAJOR")) {
            // fused multiple-SpMxV, row-major segments (split.cu spmv_split_rows_kernel)
            spmvb::RowTileArgs R{};
            R.tile_row = h->d_tile_row;
            R.tile_nnz = h->d_tile_nnz;
            R.tile_cls = h->d_tile_cls;
            R.rowptr = h->d_rowptr;
            R.col = h->d_fcol;
            R.val = h->d_fval;
            R.x_lo = A.x_lo;
            R.x_hi = A.x_hi;
            R.x_split = A.x_split;
            R.n_tiles = A.n_tiles;
            R.y = yk;
            R.maxabs_slots = A.maxabs_slots;
            R.gmode = 2;
            CUDA_TRY(spmvb::launch_split_rows(R, h->d_frowseg, h->d_fsegptr, xsplit, st));
        } else {
            A.k_begin = 0; A.k_end = h->n_parts;
            if (h->kernel == 2) CUDA_TRY(spmvb::launch_tiles(A, true, xsplit, st));
            else CUDA_TRY(spmvb::launch_split(A, xsplit, st));
        }
    }
    if (orig)   // a7: y[i] = y^[row_perm[i]]
        CUDA_TRY(spmvb::launch_gather(h->d_yhat, h->d_rowperm, y, h->m, st));
    return SPMV_OK;
}

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
    if (!h->n_parts) return fail(SPMV_ERR_UNSUPPORTED, "handle has no split");
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
    info->xs_panels = h->kernel == 7 ? h->pn.panels : h->xs_panels;
    info->xs_groups = h->kernel == 7 ? h->pn.groups : h->xs_groups;
    info->xs_pad_slots = h->kernel == 7 ? h->pn.pad : h->xs_pad;
    info->bytes_stream = h->bytes_stream;
    info->kernel = h->kernel;
    info->gather_sectors = h->kernel == 7 ? h->pn.gsectors : 0;
    info->split_kernel = h->n_parts == 0 ? 0
                         : (h->pns.ok() && h->kernel != 2) ? 7
                         : (h->split_rowmajor && h->kernel != 2 && !getenv("SPMV_SPLIT_PARTMAJOR")) ? 3 : 1;
    return SPMV_OK;
}

spmv_status_t spmv_maxabs(spmv_handle_t h, double* m_dev, void* stream) {
    if (!valid(h) || !m_dev) return fail(SPMV_ERR_USAGE, "invalid handle or pointer");
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaSetDevice(h->device));
    CUDA_TRY(spmvb::launch_maxabs_finish(h->d_slots, m_dev, st));
    if (h->world > 1 && h->comm) NCCL_TRY(ncclAllReduce(m_dev, m_dev, 1, ncclFloat64, ncclMax, h->comm, st));
    return SPMV_OK;
}

spmv_status_t spmv_normalize(spmv_handle_t h, const double* y, const double* m_dev, double* x_next, void* stream) {
    if (!valid(h) || !y || !m_dev || !x_next) return fail(SPMV_ERR_USAGE, "invalid handle or pointer");
    if (!h->has_owner) return fail(SPMV_ERR_UNSUPPORTED, "no owner-aligned column->row map (A17)");
    CUDA_TRY(cudaSetDevice(h->device));
    CUDA_TRY(spmvb::launch_normalize(y, h->d_owner, m_dev, x_next, h->x_local_len, (cudaStream_t)stream));
    return SPMV_OK;
}

spmv_status_t spmv_debug_copy_csr(spmv_handle_t h, int64_t* row_ptr, int32_t* col, double* val) {
    if (!valid(h) || !row_ptr || (h->nnz_loc && (!col || !val))) return fail(SPMV_ERR_USAGE, "bad arguments");
    CUDA_TRY(cudaSetDevice(h->device));
    CUDA_TRY(cudaDeviceSynchronize());
    std::vector<int32_t> rp(h->m_loc + 1);
    CUDA_TRY(cudaMemcpy(rp.data(), h->d_rowptr, rp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < rp.size(); ++i) row_ptr[i] = rp[i];
    if (h->nnz_loc) {
        CUDA_TRY(cudaMemcpy(col, h->d_col, h->nnz_loc * sizeof(int32_t), cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(val, h->d_val, h->nnz_loc * sizeof(double), cudaMemcpyDeviceToHost));
        if (h->world > 1) {   // back to global permuted ids
            const int64_t Q0 = h->x_int_begin, B0 = h->border_begin, nint = h->x_int_len;
            for (int64_t t = 0; t < h->nnz_loc; ++t)
                col[t] = (int32_t)(col[t] >= nint ? B0 + (col[t] - nint) : Q0 + col[t]);
        }
    }
    return SPMV_OK;
}

// ------------------------------------------------------------ diagnostics
spmv_status_t spmv_diag_read(const void* buf, int64_t bytes, int32_t blocks_per_sm, double* out_dev, void* stream) {
    if (!buf || bytes < 16 || !out_dev || blocks_per_sm < 1) return fail(SPMV_ERR_USAGE, "diag_read: bad arguments");
    CUDA_TRY(spmvb::diag_read(buf, bytes, out_dev, blocks_per_sm, (cudaStream_t)stream));
    return SPMV_OK;
}

spmv_status_t spmv_diag_gather(const double* x, int64_t n, int64_t count, double* out_dev, void* stream) {
    if (!x || n < 1 || count < 1 || !out_dev) return fail(SPMV_ERR_USAGE, "diag_gather: bad arguments");
    CUDA_TRY(spmvb::diag_gather(x, n, count, out_dev, (cudaStream_t)stream));
    return SPMV_OK;
}

spmv_status_t spmv_diag_gather_mode(const double* x, int64_t n, int64_t count, int32_t mode, int32_t blocks_per_sm,
                                    double* out_dev, void* stream) {
    if (!x || n < 2 || count < 1 || !out_dev || blocks_per_sm < 1) return fail(SPMV_ERR_USAGE, "diag_gather_mode: bad arguments");
    CUDA_TRY(spmvb::diag_gather_mode(x, n, count, mode, blocks_per_sm, out_dev, (cudaStream_t)stream));
    return SPMV_OK;
}

spmv_status_t spmv_diag_csr(spmv_handle_t h, const double* x, int32_t mode, double* out_dev, void* stream) {
    if (!valid(h) || !out_dev || (mode >= 1 && !x) || mode < 0 || mode > 3)
        return fail(SPMV_ERR_USAGE, "diag_csr: bad arguments");
    if (h->world > 1) return fail(SPMV_ERR_UNSUPPORTED, "diag_csr: world 1 only");
    CUDA_TRY(cudaSetDevice(h->device));
    CUDA_TRY(spmvb::diag_csr(h->d_col, h->d_val, x, h->nnz_loc, mode, out_dev, (cudaStream_t)stream));
    return SPMV_OK;
}

spmv_status_t spmv_xs_plan_check(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                                 const spmv_blocks_t* blocks, int64_t rows_target, int64_t* stats) {
    if (m < 0 || n < 0 || !row_ptr || !blocks || !stats || blocks->kind != SPMV_SB || blocks->K < 1 ||
        !blocks->row_block_ptr || !blocks->col_block_ptr)
        return fail(SPMV_ERR_USAGE, "xs_plan_check: bad arguments");
    const int K = blocks->K;
    const int64_t nnz = row_ptr[m];
    if (nnz > 0 && (!col || !val)) return fail(SPMV_ERR_USAGE, "xs_plan_check: NULL col/val");
    try {
        std::vector<int64_t> rp(row_ptr, row_ptr + m + 1);
        std::vector<int32_t> c(col, col + nnz);
        std::vector<double> v(val, val + nnz);
        std::vector<spmvb::XsBlockIn> bl;
        for (int k = 0; k < K; ++k)
            bl.push_back({blocks->row_block_ptr[k], blocks->row_block_ptr[k + 1], blocks->col_block_ptr[k],
                          blocks->col_block_ptr[k + 1]});
        const int64_t gb = blocks->col_block_ptr[K];
        const int64_t glen = blocks->col_block_ptr[K + 1] - gb;
        std::vector<spmvb::XsPanelData> pd;
        spmvb::XsPlanStats st;
        std::string why;
        int cbits = 0;
        if (!spmvb::plan_xstage(rp, c, v, bl, gb, glen, rows_target, pd, cbits, st, why))
            return fail(SPMV_ERR_UNSUPPORTED, "xs_plan_check: %s", why.c_str());
        stats[0] = st.panels; stats[1] = st.groups_i; stats[2] = st.groups_b;
        stats[3] = st.pad_i; stats[4] = st.pad_b; stats[5] = st.entries;
        if (st.entries != nnz) return fail(SPMV_ERR_INTERNAL, "xs_plan_check: plan holds %lld of %lld nonzeros",
                                           (long long)st.entries, (long long)nnz);
        if (!spmvb::verify_xstage(rp, c, v, gb, cbits, pd, why))
            return fail(SPMV_ERR_INTERNAL, "xs_plan_check: %s", why.c_str());
    } catch (const std::bad_alloc&) {
        return fail(SPMV_ERR_INTERNAL, "out of host memory");
    }
    return SPMV_OK;
}

spmv_status_t spmv_pn_plan_check(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                                 const spmv_blocks_t* blocks, int64_t rows_target, int64_t* stats) {
    if (m < 0 || n < 0 || !row_ptr || !stats) return fail(SPMV_ERR_USAGE, "pn_plan_check: bad arguments");
    const int64_t nnz = row_ptr[m];
    if (nnz > 0 && (!col || !val)) return fail(SPMV_ERR_USAGE, "pn_plan_check: NULL col/val");
    try {
        std::vector<int64_t> rp(row_ptr, row_ptr + m + 1);
        std::vector<int32_t> c(col, col + nnz);
        std::vector<double> v(val, val + nnz);
        std::vector<std::pair<int64_t, int64_t>> ranges;
        if (blocks && blocks->K > 0 && blocks->row_block_ptr) {
            for (int k = 0; k <= blocks->K; ++k)
                if (blocks->row_block_ptr[k + 1] > blocks->row_block_ptr[k])
                    ranges.push_back({blocks->row_block_ptr[k], blocks->row_block_ptr[k + 1]});
        } else {
            ranges.push_back({0, m});
        }
        std::vector<spmvb::PnPanelData> pd;
        spmvb::PnPlanStats st;
        std::string why;
        // SB: columns >= C_B's start come from the second x pointer (the border
        // exchange buffer at world > 1); groups must not mix the two sides
        const int64_t xs = (blocks && blocks->K > 0 && blocks->col_block_ptr) ? blocks->col_block_ptr[blocks->K]
                                                                            : (int64_t)INT32_MAX;
        if (!spmvb::plan_panel(rp, c, v, ranges, xs, rows_target, pd, st, why))
            return fail(SPMV_ERR_UNSUPPORTED, "pn_plan_check: %s", why.c_str());
        stats[0] = st.panels; stats[1] = st.groups; stats[2] = st.pads;
        stats[3] = st.deferred; stats[4] = st.epochs; stats[5] = st.entries;
        stats[6] = (int64_t)(st.ywf0 * 1000.0); stats[7] = (int64_t)(st.ywf1 * 1000.0);
        if (st.entries != nnz) return fail(SPMV_ERR_INTERNAL, "pn_plan_check: plan holds %lld of %lld nonzeros",
                                           (long long)st.entries, (long long)nnz);
        if (!spmvb::verify_panel(rp, c, v, xs, pd, why))
            return fail(SPMV_ERR_INTERNAL, "pn_plan_check: %s", why.c_str());
    } catch (const std::bad_alloc&) {
        return fail(SPMV_ERR_INTERNAL, "out of host memory");
    }
    return SPMV_OK;
}

spmv_status_t spmv_pn_shard_hash(int64_t m, int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                                 const spmv_blocks_t* blocks, int32_t world, int32_t sms, int64_t* out) {
    if (m < 0 || n < 0 || !row_ptr || !out || !blocks || world < 1 || sms < 1)
        return fail(SPMV_ERR_USAGE, "pn_shard_hash: bad arguments");
    if (blocks->kind != SPMV_SB || blocks->K < 1 || !blocks->row_block_ptr || !blocks->col_block_ptr)
        return fail(SPMV_ERR_DATA, "pn_shard_hash: needs an SB block descriptor");
    const int K = blocks->K;
    const int64_t nnz = row_ptr[m];
    if (nnz > 0 && (!col || !val)) return fail(SPMV_ERR_USAGE, "pn_shard_hash: NULL col/val");
    try {
        std::vector<int64_t> rbp(blocks->row_block_ptr, blocks->row_block_ptr + K + 2);
        std::vector<int64_t> cbp(blocks->col_block_ptr, blocks->col_block_ptr + K + 2);
        std::vector<int64_t> blk(K, 0);   // global per-block slots, as spmv_create counts them
        for (int k = 0; k < K; ++k)
            for (int64_t i = rbp[k]; i < rbp[k + 1]; ++i) blk[k] += spmvb::row_slots(row_ptr[i + 1] - row_ptr[i]);
        for (int64_t i = 0; i < (int64_t)world * K; ++i) out[i] = 0;
        for (int r = 0; r < world; ++r) {
            spmv_shard_t sh;
            spmv_status_t s = spmv_shard_plan(blocks, m, n, r, world, &sh);
            if (s != SPMV_OK) return s;
            const int64_t R0 = sh.row_begin, ml = sh.row_end - sh.row_begin;
            // local CSR in the rank's x layout (create_impl's: interior columns
            // shifted to 0, then the full C_B)
            std::vector<int64_t> rp(ml + 1, 0);
            std::vector<int32_t> c;
            std::vector<double> v;
            for (int64_t i = 0; i < ml; ++i) {
                for (int64_t t = row_ptr[R0 + i]; t < row_ptr[R0 + i + 1]; ++t) {
                    const int64_t g = col[t];
                    int64_t l = g;
                    if (world > 1)
                        l = g >= cbp[K] ? sh.x_interior_len + (g - cbp[K]) : g - sh.x_interior_begin;
                    c.push_back((int32_t)l);
                    v.push_back(val[t]);
                }
                rp[i + 1] = (int64_t)c.size();
            }
            const PnSetup S = pn_setup(SPMV_SB, world, R0, ml, sh.x_interior_begin, sh.x_interior_len, n, rbp, cbp, blk,
                                       rp, nullptr, sms);
            std::vector<spmvb::PnPanelData> pd;
            spmvb::PnPlanStats st;
            std::string why;
            if (!spmvb::plan_panel(rp, c, v, S.ranges, S.xs, S.target, pd, st, why,
                                   S.xcols.empty() ? nullptr : &S.xcols, S.sms, nullptr, S.waves * S.sms,
                                   S.global ? &S.range_panels : nullptr))
                return fail(SPMV_ERR_UNSUPPORTED, "pn_shard_hash: %s", why.c_str());
            for (const auto& P : pd) {
                const int64_t row0 = R0 + P.desc.row0;
                const int k = (int)(std::upper_bound(rbp.begin(), rbp.begin() + K + 1, row0) - rbp.begin()) - 1;
                // slot -> (panel row, virtual-row rank)
                const int32_t nsl = ((P.nslots + 15) / 16) * 16;
                std::vector<int32_t> srow(nsl, -1), svr(nsl, 0);
                for (int32_t i = 0; i < P.desc.nrows; ++i) {
                    const int32_t sl = P.row2slot[i];
                    if (sl < 0x8000) {
                        srow[sl] = i;
                    } else {
                        const int32_t q = sl & 0x7FFF;
                        for (int32_t j = 0; j < P.split_cnt[q]; ++j) {
                            srow[P.split_slots[P.split_first[q] + j]] = i;
                            svr[P.split_slots[P.split_first[q] + j]] = j;
                        }
                    }
                }
                uint64_t hsh = (uint64_t)out[(int64_t)r * K + k] ^ 0xcbf29ce484222325ull;
                auto mix = [&](uint64_t x) { hsh = (hsh ^ x) * 0x100000001b3ull; };
                mix((uint64_t)row0);
                mix((uint64_t)P.desc.nrows);
                const int64_t G = (int64_t)P.gbase.size();
                for (int64_t g = 0; g < G; ++g)
                    for (int l = 0; l < 32; ++l) {
                        const uint32_t i = P.gidx[g * 32 + l];
                        if (i == spmvb::kPnDummy) continue;
                        const int32_t sl = (int32_t)(i >> spmvb::kPnDeltaBits);
                        const int64_t lc = (int64_t)P.gbase[g] + (i & ((1u << spmvb::kPnDeltaBits) - 1));
                        int64_t gc = lc;
                        if (world > 1) gc = lc >= sh.x_interior_len ? cbp[K] + (lc - sh.x_interior_len) : lc + sh.x_interior_begin;
                        uint64_t vb;
                        memcpy(&vb, &P.gval[g * 32 + l], 8);
                        mix((uint64_t)(R0 + P.desc.row0 + (sl < nsl ? srow[sl] : -1)));
                        mix((uint64_t)(sl < nsl ? svr[sl] : -1));
                        mix((uint64_t)gc);
                        mix(vb);
                    }
                out[(int64_t)r * K + k] = (int64_t)hsh;
            }
        }
    } catch (const std::bad_alloc&) {
        return fail(SPMV_ERR_INTERNAL, "out of host memory");
    }
    return SPMV_OK;
}

spmv_status_t spmv_test_set_border(spmv_handle_t h, const double* x_border, int64_t len) {
    if (!valid(h) || !h->test_nocomm || !x_border) return fail(SPMV_ERR_USAGE, "test_set_border: not a test rank");
    if (len != h->border_total) return fail(SPMV_ERR_USAGE, "test_set_border: length %lld != |C_B| %lld",
                                            (long long)len, (long long)h->border_total);
    CUDA_TRY(cudaSetDevice(h->device));
    if (len) CUDA_TRY(cudaMemcpy(h->d_xborder, x_border, len * sizeof(double), cudaMemcpyDeviceToDevice));
    return SPMV_OK;
}

spmv_status_t spmv_diag_micro(int32_t kind, int32_t param, const void* buf, int64_t bytes, int64_t count,
                              double* out_dev, void* stream) {
    if (!out_dev || count < 1 || (kind != 3 && (!buf || bytes < 16))) return fail(SPMV_ERR_USAGE, "diag_micro: bad arguments");
    CUDA_TRY(spmvb::diag_micro(kind, param, buf, bytes, count, out_dev, (cudaStream_t)stream));
    return SPMV_OK;
}

}  // extern "C"
