// internal.h -- shared between the host library (host.cpp) and the kernels
// (kernels.cu).  Not part of the ABI (include/spmv.h is).
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

cudaError_t launch_tiles(const TileArgs& a, bool split, bool xsplit, cudaStream_t s);

// Persistent warp-specialised single-SpMxV kernel (pipe.cu).
struct PipeArgs {
    const int32_t* tile_row;   // [T+1]
    const int32_t* tile_nnz;   // [T+1] = row_ptr[tile_row[t]]
    const int32_t* tile_cls;   // [T] kTileShort / kTileGeneral
    const int32_t* rowptr;     // [m+1+4]
    const int32_t* col;        // [nnz+pad]
    const double* val;         // [nnz+pad]
    const double* x_lo;
    const double* x_hi;
    int32_t x_split;
    int32_t n_tiles;
    double* y;
    unsigned long long* maxabs_slots;
    int* tile_counter;         // zeroed by launch_pipe before every launch
    int32_t gmode;             // x gather flavour (measurements): 0 ld.global.nc, 1 + L2 evict_last,
                               // 2 + L1 no_allocate and L2 evict_last
    const int32_t* long_tiles; // tiles holding one row longer than a tile (run by launch_longrows), or
                               // nullptr: the tile kernel runs them itself
};
cudaError_t launch_longrows(const PipeArgs& a, int32_t n_long, bool xsplit, cudaStream_t s);
cudaError_t launch_pipe(const PipeArgs& a, bool xsplit, cudaStream_t s);
// Default single-SpMxV kernel (rowtile.cu): one 512-thread CTA per row tile.
using RowTileArgs = PipeArgs;
cudaError_t launch_rowtile(const RowTileArgs& a, bool xsplit, int threads, cudaStream_t s, bool lin = false);
cudaError_t launch_rowseg(const RowTileArgs& a, bool xsplit, cudaStream_t s);
// Fused / literal multiple-SpMxV kernel (split.cu), K <= 64 parts.
constexpr int kMaxParts = 64;
cudaError_t launch_split(const TileArgs& a, bool xsplit, cudaStream_t s);
// Fused multiple-SpMxV over the row-major segment layout: per row, the part
// segments in part order, each summed into its own temporary (split.cu).
cudaError_t launch_split_rows(const RowTileArgs& a, const int32_t* row_seg, const int32_t* seg_ptr, bool xsplit,
                              cudaStream_t s);
size_t pipe_smem_bytes();
// x^[c] = x[colinv[c]]   (ORIGINAL-mode x preparation, a3)
cudaError_t launch_gather(const double* src, const int32_t* idx, double* dst, int64_t n, cudaStream_t s);
// max over slots -> *out
cudaError_t launch_maxabs_finish(const unsigned long long* slots, double* out, cudaStream_t s);
// x_next[c] = y[owner[c]] / *m   (power-iteration glue, a9)
cudaError_t launch_normalize(const double* y, const int32_t* owner, const double* m, double* x_next,
                             int64_t n, cudaStream_t s);
int kernel_num_sms();

// ---------------------------------------------------------------------------
// x-staged single-SpMxV (xstage.cu, plan_xs.cpp).  A panel is a
// run of rows of one SB block; its interior columns C_k are streamed through
// shared memory in chunks of kXsW columns by the bulk-copy engine, its y rows
// live in shared memory, and its nonzeros are pre-packed into 32-entry groups
// (one per lane) with distinct rows and spread shared-memory banks.  Border
// (C_B) nonzeros are gathered from L2.
constexpr int kXsWarps = 16;                 // consumer warps; each owns a row range
constexpr int kXsStages = 3;                 // x chunk ring
constexpr int kXsW = 2048;                   // columns per chunk (multiple of 16)
constexpr int kXsStageStride = kXsW + 16;    // doubles per stage buffer
constexpr int kXsRowsMax = 22528;            // y rows per panel (shared memory)
constexpr uint32_t kXsDummy = 0xFFFFFFFFu;   // padding slot
static_assert(kXsW % 16 == 0, "chunk width must keep the bank map shift-invariant");

struct XsPanel {
    int32_t row0;      // first local row
    int32_t nrows;     // rows in the panel (<= kXsRowsMax)
    int32_t col0;      // first interior column (local id); chunk j starts at col0 + j*kXsW
    int32_t col_end;   // one past the last interior column
    int32_t nch;       // chunks
    int32_t u_base;    // offset of this panel's per-warp chunk tables in XsArgs::U
    int32_t rw;        // rows per warp (warp w owns [w*rw, min((w+1)*rw, nrows)))
    int32_t pad;
};

struct XsArgs {
    const XsPanel* panel;
    int32_t n_panels;
    int32_t cbits;            // border index: (row_in_warp << cbits) | border column
    const int32_t* wg;        // [P*NW+1] interior groups of (panel, warp), contiguous
    const int32_t* wb;        // [P*NW+1] border groups of (panel, warp)
    const int32_t* U;         // per (panel, warp): nch entries, U[j] = first group with min chunk >= j
    const double* gval;       // [groups*32]
    const uint32_t* gidx;     // [groups*32] (row_in_panel << 16) | offset from its group's first chunk
    const double* bval;
    const uint32_t* bidx;
    const double* x;          // interior columns: x[col]
    const double* xg;         // border columns: xg[border column]
    double* y;                // local rows
    unsigned long long* maxabs_slots;
};
cudaError_t launch_xstage(const XsArgs& a, cudaStream_t s);
size_t xstage_smem_bytes();

// ---------------------------------------------------------------------------
// Column-sorted panel SpMxV (panel.cu, plan_panel.cpp): the
// default kernel of SB handles.  A panel is a run of <= kPnRowsMax rows of one
// SB block whose y lives in shared memory.  Its nonzeros are sorted by column
// and cut into 32-entry groups, so one warp-wide x gather touches few 128-byte
// lines (the L1TEX cost is per line, not per lane).  Groups are issued in
// epochs of kPnB groups per warp; the rows of an epoch are distinct, so the
// shared-memory y updates of one epoch never race, and a CTA barrier
// separates epochs.
constexpr int kPnWarps = 16;                 // warps per panel CTA
#ifndef SPMV_PN_B
#define SPMV_PN_B 4
#endif
constexpr int kPnB = SPMV_PN_B;              // groups per warp per epoch
constexpr int kPnEpoch = kPnWarps * kPnB;    // groups per epoch
constexpr int kPnPadGroups = 4 * kPnEpoch;  // zero groups after the stream (ring read-ahead, <= 16 steps)
constexpr int kPnRowsMax = 28672;            // y rows per panel (224 KB of shared memory)
constexpr int kPnRowsTarget = 16384;         // default panel size: 128 KB of y, the rest of the
                                             // 256 KB L1/shared array stays L1 (measured best, §5.3)
constexpr int kPnRowBits = 15;               // idx = (row_in_panel << 17) | (col - group base)
constexpr int kPnDeltaBits = 17;
constexpr uint32_t kPnDummy = 0xFFFE0000u;   // row field 0x7FFF (-> scratch y slot), delta 0 (a valid x
                                             // address): padding lanes run the same code branch-free

struct PnPanel {
    int32_t row0;      // first local row
    int32_t nrows;     // rows (<= kPnRowsMax)
    int32_t g0;        // first group of the panel (groups of epoch e, step b, warp w: g0 + (e*kPnB + b)*16 + w)
    int32_t ne;        // epochs
    int32_t pf_col;    // x_lo[pf_col, pf_col + pf_len) is prefetched into L2 at panel start
    int32_t pf_len;    //   (a slice of the next block's interior columns, SB Eq.(1))
    int32_t split_off; // first entry of this panel in PnArgs::split_first / split_cnt / split_row
    int32_t nslots;    // y slots (virtual rows) of the panel
    int32_t split_n;   // rows of the panel split into virtual rows
    int32_t sslot0;    // their virtual rows' slots: split_slots[sslot0, sslot0 + sslot_n)
    int32_t sslot_n;
    int32_t split_short; // split rows [0, split_short) have <= kPnFoldSeq virtual rows (folded by one thread)
};
#ifndef SPMV_PN_FOLDSEQ
#define SPMV_PN_FOLDSEQ 32
#endif
constexpr int kPnFoldSeq = SPMV_PN_FOLDSEQ;   // virtual rows a thread folds sequentially
#ifndef SPMV_PN_VMAX
#define SPMV_PN_VMAX 32
#endif
constexpr int kPnSplitAt = 32;               // a row with more nonzeros is split into interleaved
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
    int32_t max_rows;         // largest panel's y slots (a multiple of 16); slot max_rows is the padding
                              // lanes' scratch; shared memory = 8 * (max_rows + 1) bytes (the rest stays L1)
    const uint16_t* row2slot; // [local rows] y slot of each row within its panel (bank colouring), or
                              // 0x8000 | k: row split into virtual rows, see split_*
    const int32_t* split_first;   // [split rows] first entry in split_slots (absolute)
    const int32_t* split_cnt;     // [split rows] virtual rows of the row
    const uint16_t* split_slots;  // slots of the virtual rows, in fold order
    const int32_t* split_row;     // [split rows] panel-local row
    int32_t max_sslots;           // largest sslot_n over the panels (shared-memory copy)
    int32_t max_split_n;          // largest split_n over the panels (shared-memory copy of the descriptors)
    int32_t pf_epochs;        // epochs of the group stream prefetched into L2 ahead (0 = default)
    int32_t gather_na;        // x gathers L1::no_allocate (plan choice; 0 = allocate)
    int32_t ring;             // register-ring depth in steps (8, 12 or 16; 0 = default)
    int32_t persist;          // 1: one CTA per SM walks the panels (measurement switch)
};
cudaError_t launch_panel(const PnArgs& a, cudaStream_t s);

// roofline microkernels (diag.cu)
cudaError_t diag_read(const void* buf, int64_t bytes, double* out, int blocks_per_sm, cudaStream_t s);
cudaError_t diag_gather(const double* x, int64_t n, int64_t count, double* out, cudaStream_t s);
cudaError_t diag_gather_mode(const double* x, int64_t n, int64_t count, int mode, int blocks_per_sm, double* out,
                             cudaStream_t s);
cudaError_t diag_csr(const int32_t* col, const double* val, const double* x, int64_t nnz, int mode, double* out,
                     cudaStream_t s);
cudaError_t diag_micro(int kind, int param, const void* buf, int64_t bytes, int64_t count, double* out,
                       cudaStream_t s);

}  // namespace spmvb
