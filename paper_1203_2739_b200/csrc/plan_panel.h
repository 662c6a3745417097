// plan_panel.h -- host planner of the column-sorted panel kernel (panel.cu).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "internal.h"

namespace spmvb {

struct PnPanelData {
    PnPanel desc{};
    std::vector<double> gval;      // [groups*32]
    std::vector<uint32_t> gidx;    // [groups*32]
    std::vector<int32_t> gbase;    // [groups]
    std::vector<int32_t> gbase4;   // [groups] the same bases in (epoch, warp, step) order: one 16-byte
                                   // load gives a warp the bases of its kPnB groups of an epoch
    std::vector<uint16_t> row2slot; // [nrows] y slot of each panel row (bank colouring), or 0x8000 | k for a
                                    // row split into virtual rows: split_* entry k of this panel
    std::vector<int32_t> split_first, split_cnt;   // per split row: its virtual rows' slots in split_slots
    std::vector<int32_t> split_row;                // per split row: its panel-local row
    std::vector<uint16_t> split_slots;
    int32_t split_short = 0;        // split rows [0, split_short) have <= kPnFoldSeq virtual rows
    int32_t nslots = 0;             // y slots used (virtual rows), before rounding to 16
    int64_t entries = 0, pads = 0, deferred = 0;
    int64_t pads_drain = 0, epochs_drain = 0;   // padding / epochs after the sweep's last nonzero
    int64_t far = 0;                // nonzeros in the far stream
    std::vector<double> fval;       // [fs * kPnWarps * 32] far stream, (step, warp, lane) order
    std::vector<int32_t> fcol;      //   column (the handle's local column ids)
    std::vector<uint16_t> fslot;    //   y slot | kPnFarLast at a run's last entry
    int64_t gsectors = 0;          // distinct 32-byte x sectors over the groups' gathers
    int32_t rot = 0;               // the column sweep starts at this column (wraps around)
    double ywf0 = 0, ywf1 = 0;     // predicted y wavefronts per group access: natural slots / coloured
};

struct PnPlanStats {
    int64_t panels = 0, groups = 0, entries = 0, pads = 0, deferred = 0, epochs = 0, gsectors = 0;
    int64_t pads_drain = 0, epochs_drain = 0;
    int64_t far = 0, far_steps = 0;   // far-stream nonzeros, sum over panels of its steps per warp
    double ywf0 = 0, ywf1 = 0;     // mean predicted y wavefronts per group access, before / after colouring
};

// Row ranges [r0, r1) (local rows; e.g. the SB blocks of this rank) are cut
// into panels of about rows_target rows.  Columns >= x_split come from the
// second x pointer; a group never mixes the two sides.  Returns false (and
// why) when the plan would be poor (caller falls back to the row-tile kernel).
// xcols (optional, one per range): the range's interior columns [c0, c1) --
// the panels of range k start their column sweeps spread over them.  pf_sms
// is unused (the next block's x was once prefetched into L2 ahead of its
// panels: measured 0.5 GB more DRAM reads per C5 launch, removed).
// part (optional, per CSR nonzero): plan the multiple-SpMxV -- each (row,
// part) segment gets its own virtual rows, folded in part order.
// total_panels (optional): split the ranges into this many panels in all
// (proportional to their slots), e.g. whole waves of one CTA per SM.
// range_panels (optional): the panel count of each range, fixed by the caller.
bool plan_panel(const std::vector<int64_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
                const std::vector<std::pair<int64_t, int64_t>>& ranges, int64_t x_split, int64_t rows_target,
                std::vector<PnPanelData>& out, PnPlanStats& st, std::string& why,
                const std::vector<std::pair<int64_t, int64_t>>* xcols = nullptr, int64_t pf_sms = 148,
                const std::vector<int32_t>* part = nullptr, int64_t total_panels = 0,
                const std::vector<int64_t>* range_panels = nullptr);

// y slots of a row of L nonzeros without a split (its virtual rows).
int64_t row_slots(int64_t L);

// Panels per range from the ranges' slot counts: ceil(S_k / R), or shares of
// `total` (> 0) proportional to S_k (largest remainder), never fewer than
// the slot cap allows.  Depends only on (S, R, total), so a multi-GPU rank
// that passes the global per-block counts gets the same cuts as world 1.
std::vector<int64_t> panel_counts(const std::vector<int64_t>& Sk, int64_t R, int64_t total);

// y slots (virtual rows) the plan needs for local rows [0, m) (panel sizing).
int64_t panel_total_slots(const std::vector<int64_t>& rp, int64_t m, const std::vector<int32_t>* part = nullptr);

// Test hook: decode the groups back into (row, column, value) and compare with
// the CSR bit for bit; checks the epoch invariant (distinct rows per epoch).
bool verify_panel(const std::vector<int64_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
                  int64_t x_split, const std::vector<PnPanelData>& pd, std::string& why);

}  // namespace spmvb
