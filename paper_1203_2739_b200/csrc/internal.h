// internal.h -- shared between the host library (host.cpp) and the kernels
// (kernels.cu, rowtile.cu, split.cu, panel.cu).  Not part of the ABI
// (include/spmv.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spmvb {

// Row-tile geometry of the SpMxV kernels.
//   kThreads : threads per CTA
//   kTileNnz : max nonzeros of a multi-row tile; rows longer than this get a
//              tile of their own and take the long-row path
//   kTileRows: max rows of a tile (bounds the shared-memory row arrays)
constexpr int kThreads = 256;
constexpr int kTileNnz = 2048;
constexpr int kTileRows = 512;
constexpr int kTileShort = 1;      // >= 1: every row has <= kShortRow nonzeros; value = lanes per row
constexpr int kTileGeneral = 0;
constexpr int kShortRow = 32;
constexpr int kMaxDevices = 64;     // per-device caches (SM count, kernel attributes)
constexpr int64_t kOwnerRunMin = 64;   // owner map kept as runs when they average >= this many columns
constexpr int kMaxSlots = 1024;      // max-abs accumulator slots (spread atomics)
constexpr int kSlotStride = 16;    // 16 x 8 B = 128 B apart

// A "segment" is the run of nonzeros of one row inside one split part
// (P:L107): with no split, segments are the rows.  Tile t covers local rows
// [tile_row[t], tile_row[t+1]); its part-k segments are
// [tile_seg[t*K+k], tile_seg[t*K+k+1]) with nonzeros [seg_ptr[s], seg_ptr[s+1]).
struct TileArgs {
    const int32_t* tile_row;   // [T+1]
    const int32_t* tile_seg;   // [T*K+1]  (plain: == tile_row, K = 1)
    const int32_t* seg_ptr;    // [S+1]    (plain: row_ptr)
    const int32_t* seg_row;    // [S] tile-local row of each segment (plain: unused)
    const int32_t* col;        // [nnz + pad] local column ids
    const double* val;         // [nnz + pad]
    const double* x_lo;        // x for columns < x_split
    const double* x_hi;        // x_hi[c - x_split] for columns >= x_split
    int32_t x_split;
    int32_t n_tiles;
    double* y;                 // local rows
    int32_t K, k_begin, k_end; // parts processed in this pass
    int32_t accumulate;        // 1: y <- y + (sum over parts) (literal split pass)
    unsigned long long* maxabs_slots;   // nullptr or kMaxSlots*kSlotStride
};

// Row-tile single-SpMxV kernel (rowtile.cu): one 256-thread CTA per row tile
// (the fallback when the panel plan is rejected, and the row-major fused
// split, split.cu).
struct RowTileArgs {
    const int32_t* tile_row;   // [T+1]
    const int32_t* tile_nnz;   // [T+1] = row_ptr[tile_row[t]]
    const int32_t* tile_cls;   // [T] kTileShort.. (lanes per row) / kTileGeneral
    const int32_t* rowptr;     // [m+1+pad]
    const int32_t* col;        // [nnz+pad]
    const double* val;         // [nnz+pad]
    const double* x_lo;
    const double* x_hi;
    int32_t x_split;
    int32_t n_tiles;
    double* y;
    unsigned long long* maxabs_slots;
    // f3: 16-bit tile-local column ids (nullptr: col is used).  Tile t's id u
    // decodes to min(u + (u < tile_base[t].z ? tile_base[t].x : tile_base[t].y), tile_base[t].w)
    const uint16_t* col16;     // [nnz+pad]
    const int4* tile_base;     // [T] (lo, hi, split, largest column of the tile)
};
cudaError_t launch_rowtile(const RowTileArgs& a, bool xsplit, cudaStream_t s);

// x-staged SB kernel (xstaged.cu): one CTA per range of row tiles of one SB
// block, x(C_k) and x(C_B) staged in shared memory, 16-bit block-local ids.
struct XsCta {
    int32_t t0, t1;    // its row tiles [t0, t1) (all of one block)
    int32_t q0, nk;    // x(C_k) = x[q0, q0 + nk)
    int32_t qB, nB;    // x(C_B) = x[qB, qB + nB)
    int32_t k, pad;    // pad: lanes per row of the warp-independent form
};
struct XsArgs {
    const XsCta* cta;
    int32_t n_cta;
    int32_t max_x;             // largest nk + nB (shared memory)
    const int32_t* tile_row;   // rowtile.cu's tiles
    const int32_t* tile_nnz;
    const int32_t* tile_cls;   // lanes per row for 512 threads (kTileShort..32) / kTileGeneral
    const int32_t* rowptr;
    const uint16_t* colx;      // [nnz+pad] block-local ids: u < nk -> C_k[u], else C_B[u - nk]
    const double* val;
    const double* x;
    double* y;
    unsigned long long* maxabs_slots;
};
int64_t xstaged_smem_bytes(int64_t x_entries);
cudaError_t launch_xstaged(const XsArgs& a, cudaStream_t s);
cudaError_t preload_kernels_xstaged();
// Fused / literal multiple-SpMxV kernel (split.cu), K <= 64 parts.
constexpr int kMaxParts = 64;
cudaError_t launch_split(const TileArgs& a, bool xsplit, cudaStream_t s);
// Fused multiple-SpMxV over the row-major segment layout: per row, the part
// segments in part order, each summed into its own temporary (split.cu).
cudaError_t launch_split_rows(const RowTileArgs& a, const int32_t* row_seg, const int32_t* seg_ptr, bool xsplit,
                              cudaStream_t s);
// x^[c] = x[colinv[c]]   (ORIGINAL-mode x preparation, a3)
cudaError_t launch_gather(const double* src, const int32_t* idx, double* dst, int64_t n, cudaStream_t s);
// DB split across GPUs: y[i] = fold of tin[fpos[fptr[i]..fptr[i+1])] in order (f1).  With
// w.ready set (P2P exchange) the kernel first waits on the device until
// ready[q] - seq >= 0 for every peer q != self (bounded; a timeout adds 1 to *err).
struct FoldWait {
    const int32_t* ready = nullptr;
    int32_t world = 1, self = 0, seq = 0;
    int32_t* err = nullptr;
    int32_t* herr = nullptr;   // host-mapped sticky flag, also set on a timeout
};
cudaError_t launch_fold(const double* tin, const int32_t* fptr, const int32_t* fpos, double* y, int64_t n, FoldWait w,
                        unsigned long long* slots, cudaStream_t s);
// max over slots -> *out
cudaError_t launch_maxabs_finish(const unsigned long long* slots, double* out, cudaStream_t s);
// x_next[c] = y[owner[c]] / *m   (power-iteration glue, a9)
cudaError_t launch_normalize(const double* y, const int32_t* owner, const double* m, double* x_next,
                             int64_t n, cudaStream_t s);
// the same with the owner map as runs: x_next[l] = y[tgt[r] + l - start[r]], start[r] <= l < start[r+1];
// tdelta[t] = tgt[r] - start[r] when tile t (kNormTileCols columns) lies in one run r, else kNoDelta
constexpr int64_t kNormTileCols = 1024;
constexpr int64_t kNoDelta = INT64_MIN;
cudaError_t launch_normalize_runs(const double* y, const int64_t* tdelta, const int64_t* start, const int32_t* tgt,
                                  int64_t runs, const double* m, double* x_next, int64_t n, cudaStream_t s);
int kernel_num_sms();   // SMs of the current device
// Eager loading of every SpMxV-path kernel on the current device (per .cu file)
cudaError_t preload_kernels_misc();
cudaError_t preload_kernels_panel();
cudaError_t preload_kernels_rowtile();
cudaError_t preload_kernels_split();

// ---------------------------------------------------------------------------
// Column-sorted panel SpMxV (panel.cu, plan_panel.cpp): the
// default kernel of SB handles.  A panel is a run of <= kPnRowsMax rows of one
// SB block whose y lives in shared memory.  Its nonzeros are sorted by column
// and cut into 32-entry groups, so one warp-wide x gather touches few 128-byte
// lines (the L1TEX cost is per line, not per lane).  Groups are issued in
// epochs of kPnB groups per warp; the rows of an epoch are distinct, so the
// shared-memory y updates of one epoch never race, and a CTA barrier
// separates epochs.
#ifndef SPMV_PN_WARPS
#define SPMV_PN_WARPS 16
#endif
constexpr int kPnWarps = SPMV_PN_WARPS;      // warps per panel CTA
constexpr int kPnB = 4;                      // groups per warp per epoch (4 beat 8)
constexpr int kPnEpoch = kPnWarps * kPnB;    // groups per epoch
constexpr int kPnPadGroups = 4 * kPnEpoch;  // zero groups after the stream (ring read-ahead, <= 16 steps)
constexpr int kPnRowsMax = 28672;            // y rows per panel (224 KB of shared memory)
constexpr int kPnRowsTarget = 16384;         // default panel size: 128 KB of y, the rest of the
                                             // 256 KB L1/shared array stays L1 (measured best, §5.3)
constexpr int kPnRowBits = 15;               // idx = (row_in_panel << 17) | (col - group base)
constexpr int kPnDeltaBits = 17;
// Padding lanes run the same code branch-free: their index holds delta 0 (a
// valid x address, times the value 0) and a row field 0x7FF0 + b, which the
// upload maps to scratch y slot max_rows + b -- the planner picks b among the
// 8-byte banks its half-warp leaves free, so padding never adds a y bank
// conflict.
constexpr uint32_t kPnDummyRow = 0x7FF0;
constexpr uint32_t pn_dummy(int bank) { return (kPnDummyRow + (uint32_t)bank) << 17; }
constexpr bool pn_is_dummy(uint32_t i) { return (i >> 17) >= kPnDummyRow; }

struct PnPanel {
    int32_t row0;      // first local row
    int32_t nrows;     // rows (<= kPnRowsMax)
    int32_t g0;        // first group of the panel (groups of epoch e, step b, warp w: g0 + (e*kPnB + b)*16 + w)
    int32_t ne;        // epochs
    int32_t split_off; // first entry of this panel in PnArgs::split_first / split_cnt / split_row
    int32_t nslots;    // y slots (virtual rows) of the panel
    int32_t split_n;   // rows of the panel split into virtual rows
    int32_t sslot0;    // their virtual rows' slots: split_slots[sslot0, sslot0 + sslot_n)
    int32_t sslot_n;
    int32_t split_short; // split rows [0, split_short) have <= kPnFoldSeq virtual rows (folded by one thread)
    int32_t fs;        // far-stream steps per warp (a multiple of kPnFarRing)
    int32_t fb;        // first 32-entry block of the panel's far stream
    int32_t bepoch;    // first epoch with a border-column (x_split side) group; ne if none.  Interior
                       // groups come first (the planner's column order), so at world > 1 the border-x
                       // exchange overlaps epochs [0, bepoch) (a4)
};
constexpr int kPnFoldSeq = 32;               // virtual rows a thread folds sequentially
// Far phase (plan_panel.cpp build_panel, panel.cu): the nonzeros still
// deferred when a panel's column sweep ends are summed by one lane per y slot
// after the epochs, barrier-free.
constexpr int kPnFarRing = 8;                // far steps per ring turn (the stream is padded to whole turns)
constexpr uint16_t kPnFarLast = 0x8000;      // fslot flag: the run's last entry (add the run's sum to y)
constexpr uint16_t kPnFarPad = 0x7FFF;       // fslot of a padding entry (value 0, never stored)
#ifndef SPMV_PN_PEND
#define SPMV_PN_PEND 32
#endif
constexpr int kPnPend = SPMV_PN_PEND;        // planner: bank-blocked nonzeros an epoch keeps pending before
                                             // it closes a group early (y bank conflicts vs padding)
#ifndef SPMV_PN_VMAX
#define SPMV_PN_VMAX 32
#endif
constexpr int kPnSplitAt = SPMV_PN_VMAX;     // a row with more nonzeros is split into interleaved
constexpr int kPnVMax = SPMV_PN_VMAX;        // virtual rows of <= kPnVMax nonzeros (own y slots,
                                             // folded in order in the epilogue)

struct PnArgs {
    const PnPanel* panel;
    int32_t n_panels;
    int32_t x_split;          // columns >= x_split read x_hi[c - x_split]
    const double* gval;       // [groups*32] per (epoch, warp) blocks of 128: (step pair, lane, step & 1)
    const uint32_t* gidx;     // [groups*32] per (epoch, warp) blocks of 128: (lane, step)
    const int32_t* gbase4;    // [groups] same, (epoch, warp, step) order (16-byte loads)
    const double* x_lo;
    const double* x_hi;
    double* y;
    unsigned long long* maxabs_slots;
    int32_t max_rows;         // largest panel's y slots (a multiple of 16); slots max_rows + 0..15 are the
                              // padding lanes' scratch (one per bank); shared memory = panel_smem_bytes
    const uint16_t* row2slot; // [local rows] y slot of each row within its panel (bank colouring), or
                              // 0x8000 | k: row split into virtual rows, see split_*
    const int32_t* split_first;   // [split rows] first entry in split_slots (absolute)
    const int32_t* split_cnt;     // [split rows] virtual rows of the row
    const uint16_t* split_slots;  // slots of the virtual rows, in fold order
    const int32_t* split_row;     // [split rows] panel-local row
    int32_t max_sslots;           // largest sslot_n over the panels (shared-memory copy)
    int32_t max_split_n;          // largest split_n over the panels (shared-memory copy of the descriptors)
    int32_t gather_na;        // x gathers L1::no_allocate (plan choice: SB handles; 0 = allocate)
    // DB across GPUs: rows >= y_split are the border-row temporaries, written to y_hi[row - y_split]
    // (and left out of the max-abs fold)
    double* y_hi;
    int32_t y_split;
    // world > 1 with the P2P exchange (a4): before its first border epoch a CTA waits until
    // ready[q] - seq >= 0 (wrap-safe) for every rank q != self; a wait that times out adds 1 to
    // *err and goes on (no hang).  ready == nullptr: no wait (world 1, or the exchange completed
    // before the launch)
    const int32_t* ready;
    int32_t world, self, seq;
    int32_t* err;
    int32_t* herr;            // host-mapped sticky flag, also set on a timeout (the next apply reports it)
    // debug_checks (spmv_options_t): the checked kernel variant counts y slots out of bounds, x
    // columns >= x_cols and rows updated twice in one epoch into dbg[0..2]
    unsigned long long* dbg;
    int64_t x_cols;
    // test hook spmv_test_panel_stamps: per CTA 8 words (SM id, globaltimer at start and end,
    // clock64 at start, after the prologue, after the epochs, at the end), or nullptr
    unsigned long long* stamps;
    // far stream (PnPanel::fs / fb): [blocks * 32] (step, warp, lane) order
    const double* fval;
    const uint32_t* fcol;
    const uint16_t* fslot;
};
// Dynamic shared memory of a panel CTA: its y slots (+ the padding lanes'
// 16 scratch slots), the split rows' slot lists (u16) and their (first, count,
// row) descriptors.  The planner caps every panel at kPnSmemMax (ADVICE r1:
// split rows add bytes beyond the slots) and the launch re-checks it.
constexpr int64_t kPnSmemMax = 227 * 1024;
inline int64_t panel_smem_bytes(int64_t slots16, int64_t sslots, int64_t split_n) {
    return (slots16 + 16) * 8 + ((sslots + 7) & ~int64_t(7)) * 2 + split_n * 12;
}
cudaError_t launch_panel(const PnArgs& a, cudaStream_t s);   // a.dbg != nullptr: the checked variant

}  // namespace spmvb
