// handle.h -- the library's handle (spmv_plan_s) and the pieces host.cpp,
// exchange.cpp and test_hooks.cpp share.  Not part of the ABI.
#pragma once
#include <cstdarg>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/spmv.h"
#include "internal.h"
#include "plan_panel.h"

namespace spmvb {

spmv_status_t fail(spmv_status_t s, const char* fmt, ...);

#define CUDA_TRY(expr)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (expr);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return ::spmvb::fail(SPMV_ERR_INTERNAL, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                                 __FILE__, __LINE__);                                               \
    } while (0)

#define NCCL_TRY(expr)                                                                              \
    do {                                                                                            \
        ncclResult_t r_ = (expr);                                                                   \
        if (r_ != ncclSuccess)                                                                      \
            return ::spmvb::fail(SPMV_ERR_INTERNAL, "%s: %s (%s:%d)", #expr, ncclGetErrorString(r_), \
                                 __FILE__, __LINE__);                                               \
    } while (0)

constexpr uint32_t kMagic = 0x53504d56u;   // "SPMV"
constexpr int64_t kPad = 8;                // col/val padding (128-bit quad loads past the end)

// Restores the caller's current device on scope exit (the library
// must not leave PyTorch's current device changed).
class DeviceGuard {
  public:
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&old_) != cudaSuccess) old_ = -1;
        if (dev >= 0 && dev != old_) {
            ok_ = cudaSetDevice(dev) == cudaSuccess;
            changed_ = true;
        }
    }
    ~DeviceGuard() {
        if (changed_ && old_ >= 0) cudaSetDevice(old_);
    }
    bool ok() const { return ok_; }

  private:
    int old_ = -1;
    bool changed_ = false, ok_ = true;
};

struct PanelPlan {
    PnPanel* d_panel = nullptr;
    double* d_gval = nullptr;
    uint32_t* d_gidx = nullptr;
    int32_t* d_gbase4 = nullptr;
    uint16_t* d_r2s = nullptr;        // [rows] y slot of each row in its panel (or split entry)
    int32_t* d_split_first = nullptr;
    int32_t* d_split_cnt = nullptr;
    uint16_t* d_split_slots = nullptr;
    int32_t* d_split_row = nullptr;
    double* d_fval = nullptr;         // far stream (PnPanel::fs / fb)
    uint32_t* d_fcol = nullptr;
    uint16_t* d_fslot = nullptr;
    int64_t far = 0, far_blocks = 0;
    int32_t max_sslots = 0, max_split_n = 0;
    int64_t panels = 0, groups = 0, pad = 0, gsectors = 0, deferred = 0;
    int32_t max_rows = 0;
    int32_t gather_na = 0;            // x gathers bypass L1 allocation (SB handles)
    double ywf = 0;                   // predicted y wavefronts per group access (planner statistics)
    bool ok() const { return panels > 0; }
};

// World > 1 exchange modes (spmv_info_t.exchange).
enum XMode : int32_t {
    kXNone = 0,      // world 1
    kXNccl = 1,      // NCCL all-gather / grouped send-recv on a comm stream, joined before the kernel
    kXP2P = 2,       // copy-engine pushes into the peers' buffers (CUDA IPC), device flags; the kernel's
                     // interior epochs overlap the exchange (a4, f2)
    kXLoopback = 3,  // test: kXP2P between handles of one process on one GPU (SURVEY §4 loopback fake)
};

// Symmetric per-rank exchange buffers, one allocation (identical layout on
// every rank, so a peer's buffer is its base + the same offsets).
struct XBufs {
    void* base = nullptr;
    size_t bytes = 0;
    double* xb[2] = {nullptr, nullptr};   // x(C_B), all slices, by apply parity
    double* tin[2] = {nullptr, nullptr};  // DB split: received border-row temporaries, by parity
    int32_t* ready = nullptr;             // [world] ready[q] = seq: rank q's border-x slice of apply seq landed
    int32_t* done = nullptr;              // [world] done[q] = seq: rank q finished reading its buffers of apply seq
    int32_t* tready = nullptr;            // [world] tready[q] = seq: rank q's border-row temporaries landed
    int32_t* tdone = nullptr;             // [world] tdone[q] = seq: rank q folded its temporaries of apply seq
    int32_t* err = nullptr;               // [1] device-side wait timeouts
    int32_t* herr = nullptr;              // host-mapped flag (device address) set by a timed-out wait: the
                                          // next apply reports it without a synchronisation (sticky error)
    int32_t* herr_host = nullptr;         // the same flag's host address (cudaHostAlloc, mapped)
};

}  // namespace spmvb

struct spmv_plan_s {
    uint32_t magic = spmvb::kMagic;
    int device = 0;
    int rank = 0, world = 1;
    int kind = 0;                     // 0 none, 1 SB, 2 DB
    spmv_options_t opt{};
    int64_t m = 0, n = 0, nnz = 0;    // global
    // local compute rows: [rows of the rank's blocks (y_local head) | DB world > 1: one row per
    // (own part, border row) segment -- the border-row temporaries T]
    int64_t m_loc = 0, nnz_loc = 0, row_begin = 0;
    int64_t m_out = 0;                // y_local length: block rows + owned border-row slice (DB world > 1)
    int64_t m_blk = 0;                // block rows of the rank (y_local head)
    int64_t y_bord_begin = 0, y_bord_len = 0;   // owned border-row slice (DB world > 1)
    int64_t n_T = 0;                  // DB world > 1: border-row temporaries this rank computes
    int64_t x_int_begin = 0, x_int_len = 0;     // interior columns (global permuted range)
    int64_t x_bord_begin = 0, x_bord_len = 0;   // owned border slice (global permuted)
    int64_t border_begin = 0, border_total = 0; // C_B
    int64_t x_local_len = 0;
    int64_t n_tiles = 0, n_long = 0;
    int32_t n_parts = 0;
    int64_t n_seg = 0;
    int64_t bytes_alg = 0, bytes_alg_split = 0, bytes_stream = 0;
    int64_t index_bytes = 4;          // row-tile column ids: 4, or 2 with the f3 16-bit ids
    double create_s[6] = {0, 0, 0, 0, 0, 0};   // spmv_info_t.create_s
    bool has_perm = false;
    bool has_owner = false;
    int kernel = 0;                   // 7 column-sorted panels, 0 row tiles

    // device arrays (one allocation each)
    int32_t* d_rowptr = nullptr;      // [m_loc+1]
    int32_t* d_col = nullptr;         // [nnz_loc + pad] local column ids
    unsigned long long* d_dbg = nullptr;   // debug_checks: violation counters [3]
    unsigned long long* d_stamps = nullptr;   // test hook spmv_test_panel_stamps: [panels * 8] or nullptr
    uint16_t* d_col16 = nullptr;      // f3: [nnz_loc + pad] 16-bit tile-local column ids (or nullptr)
    uint16_t* d_colx = nullptr;       // x-staged kernel: [nnz_loc + pad] 16-bit block-local ids
    spmvb::XsCta* d_xcta = nullptr;   // x-staged kernel: per CTA its tiles and x slices
    int32_t xs_ncta = 0, xs_max_x = 0;
    int4* d_tile_base = nullptr;      // f3: [T] per tile (lo, hi, split, largest column)
    double* d_val = nullptr;          // [nnz_loc + pad]
    int32_t* d_tile_row = nullptr;    // [T+1]
    int32_t* d_tile_nnz = nullptr;    // [T+1] row_ptr[tile_row[t]]
    int32_t* d_tile_cls = nullptr;    // [T] tile class (internal.h)
    // column-sorted panel kernel (panel.cu): single SpMxV, and the fused
    // multiple-SpMxV over (row, part) virtual rows
    spmvb::PanelPlan pn, pns;
    // split layouts (a8): part-major tiles (literal K-pass sequence) and
    // row-major segments (fused fallback when the panel plan is rejected)
    int32_t* d_tile_seg = nullptr;    // [T*K+1]
    int32_t* d_seg_ptr = nullptr;     // [S+1]
    int32_t* d_seg_row = nullptr;     // [S]
    int32_t* d_scol = nullptr;        // [nnz_loc + pad] split stream
    double* d_sval = nullptr;
    int32_t* d_fcol = nullptr;        // [nnz_loc + pad]
    double* d_fval = nullptr;
    int32_t* d_frowseg = nullptr;     // [m_loc+1] first segment of each row
    int32_t* d_fsegptr = nullptr;     // [S+1]
    std::vector<int64_t> blk_slots;   // SB: y slots per block over the whole matrix (panel cuts)
    int32_t* d_colinv = nullptr;      // ORIGINAL mode: x^[c] = x[colinv[c]]
    int32_t* d_rowperm = nullptr;     // ORIGINAL mode: y[i] = y^[row_perm[i]]
    double* d_xhat = nullptr;
    double* d_yhat = nullptr;
    int32_t* d_owner = nullptr;       // [x_local_len] local col -> local y row (when not as runs)
    int64_t owner_runs = 0;           // > 0: the owner map as runs of consecutive rows instead
    int64_t* d_own_start = nullptr;   // [owner_runs + 1] first local column of each run (last = x_local_len)
    int32_t* d_own_tgt = nullptr;     // [owner_runs] its local y row
    int64_t* d_own_tdelta = nullptr;  // [tiles of kNormTileCols] tgt - start of the tile's run, or kNoDelta
    unsigned long long* d_slots = nullptr;

    // ---------------- world > 1
    int32_t xmode = spmvb::kXNone;
    ncclComm_t comm = nullptr;
    bool test_rank = false;           // created by spmv_test_create_rank (no communicator)
    cudaStream_t comm_stream = nullptr;
    cudaStream_t test_stream = nullptr;   // loopback test ranks: the apply stream the test uses (own queue)
    cudaEvent_t ev_x = nullptr, ev_comm = nullptr, ev_kernel = nullptr;
    int32_t seq = 0;                  // applies issued (all ranks issue the same sequence)
    std::vector<int64_t> bord_off, bord_cnt;   // per rank: owned C_B slice (offset inside C_B, length)
    bool equal_slices = true;
    spmvb::XBufs xb;                  // this rank's symmetric buffers
    std::vector<spmvb::XBufs> peer;   // every rank's buffers as mapped here (P2P / loopback)
    std::vector<void*> ipc_opened;    // peer bases opened with cudaIpcOpenMemHandle
    // DB split across ranks (f1): border-row temporaries
    double* d_T = nullptr;            // [n_T] this rank's temporaries, ordered (dest rank, part, row)
    std::vector<int64_t> t_send_off, t_send_cnt;   // per dest rank, in d_T
    std::vector<int64_t> t_recv_off, t_recv_cnt;   // per source rank, in tin
    std::vector<int64_t> t_dst_off;   // per dest rank: where this rank's run lands in that rank's tin
    int64_t t_recv_total = 0, t_recv_max = 0;
    int32_t* d_fold_ptr = nullptr;    // [y_bord_len + 1] per owned border row: its temporaries in tin
    int32_t* d_fold_pos = nullptr;    // positions in tin, part order

    std::vector<void*> allocs;
};

namespace spmvb {

template <class T>
spmv_status_t dalloc(spmv_plan_s* h, T** out, size_t count);
template <class T>
spmv_status_t upload(spmv_plan_s* h, T** out, const T* src, size_t count, size_t alloc_count = 0);
void dfree(spmv_plan_s* h, void* p);   // frees one of the handle's allocations early
void free_plan(spmv_plan_s* h);
bool valid(spmv_handle_t h);

// creation shared by spmv_create(_ex) and spmv_test_create_rank
spmv_status_t create_common(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                            const double* val, const int32_t* row_perm, const int32_t* col_perm,
                            const spmv_blocks_t* blocks, int32_t n_parts, const int32_t* part_of_nnz,
                            const spmv_dist_t* dist, const spmv_options_t* options, bool test_rank,
                            spmv_handle_t* out);

// The panel plan's layout decisions for one rank (host.cpp pn_setup).
struct PnSetup {
    std::vector<std::pair<int64_t, int64_t>> ranges, xcols;
    std::vector<int64_t> range_panels;
    int64_t target = 0, waves = 0, xs = INT32_MAX, sms = 148;
    bool global = false;
};
PnSetup pn_setup(int kind, int world, int64_t row_begin, int64_t m_blk, int64_t m_loc, int64_t x_int_begin,
                 int64_t x_int_len, int64_t n, const std::vector<int64_t>& rbp, const std::vector<int64_t>& cbp,
                 const std::vector<int64_t>& blk_slots, const std::vector<int64_t>& rp,
                 const std::vector<int32_t>* part, int64_t sms, int64_t rows_opt);

}  // namespace spmvb
