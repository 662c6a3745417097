// plan_xs.h -- host planner of the x-staged SpMxV kernel (xstage.cu).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "internal.h"

namespace spmvb {

struct XsBlockIn {
    int64_t r0, r1;   // local rows of the SB block
    int64_t c0, c1;   // its interior columns (local ids)
};

// One panel's packed streams (warps in order).
struct XsPanelData {
    XsPanel desc{};
    std::vector<int32_t> g_cnt;     // [NW] interior groups per warp
    std::vector<int32_t> u_rel;     // [NW*nch] U[j] relative to the warp's first group
    std::vector<double> gval;
    std::vector<uint32_t> gidx;
    std::vector<int32_t> b_cnt;     // [NW] border groups per warp
    std::vector<double> bval;
    std::vector<uint32_t> bidx;
    int64_t entries = 0, pad_i = 0, pad_b = 0;
};

struct XsPlanStats {
    int64_t panels = 0, groups_i = 0, groups_b = 0, entries = 0, pad_i = 0, pad_b = 0;
};

// Packs the local CSR (rows sorted by column) into panels.  gb = first border
// column (local id); border columns are [gb, gb + g_len).  rows_target = rows
// per panel to aim for.  Returns false (and why) when the matrix does not fit
// the format (caller falls back to the row-tile kernel).
bool plan_xstage(const std::vector<int64_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
                 const std::vector<XsBlockIn>& blocks, int64_t gb, int64_t g_len, int64_t rows_target,
                 std::vector<XsPanelData>& out, int& cbits, XsPlanStats& st, std::string& why);

// Test hook: decode the packed streams and compare with the CSR bit for bit.
bool verify_xstage(const std::vector<int64_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
                   int64_t gb, int cbits, const std::vector<XsPanelData>& pd, std::string& why);

}  // namespace spmvb
