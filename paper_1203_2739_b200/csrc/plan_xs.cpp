// plan_xs.cpp -- host planner of the x-staged SpMxV kernel (xstage.cu).
//
// What it builds ("x-staged kernel"): for every SB block
// (Eq.(1)) the rows are cut into panels; a panel's y rows sit in
// shared memory and its interior x columns C_k stream through a shared-memory
// ring chunk by chunk.  This is the paper's "fits into the cache" condition
// made explicit on B200: the part of x that a group of rows
// reuses is staged on chip; only the coupling columns C_B are read
// from L2.  Each warp of the panel's CTA owns a contiguous range of the panel
// rows (so y updates never race between warps) and walks its nonzeros in
// chunk order, 32 at a time (one per lane).  The planner packs each warp's
// nonzeros into such 32-entry groups:
//   * the rows in a group are distinct (the y update is a plain
//     read-modify-write in shared memory);
//   * within each half-warp, the y rows and x columns fall into distinct
//     8-byte shared-memory banks where the greedy can arrange it (measured:
//     conflict-free updates run 2.5x faster than random ones, profiles/);
//   * a group holds nonzeros of at most two consecutive chunks, so only the
//     last group of a warp's panel carries padding.
// Padding slots are kXsDummy (the lane does nothing).  The order of a row's
// products is chunk order, i.e. ascending column blocks; any order is within
// the oracle tolerance (reading A6), and the plan is deterministic.
#include "plan_xs.h"

#include <algorithm>
#include <cstring>
#include <deque>
#include <omp.h>

namespace spmvb {
namespace {

constexpr int kMaxOpen = 24;     // non-full groups a new entry may be placed into
constexpr size_t kMaxDeque = 256; // groups waiting for emission

struct Grp {
    uint32_t idx[32];
    double val[32];
    int32_t row[32];
    uint8_t xc[2][16], yc[2][16];   // entries per 8-byte bank, per half-warp
    int8_t fill[2];
    int32_t minc;
    bool closed;
    bool full() const { return fill[0] == 16 && fill[1] == 16; }
    bool has_row(int32_t r) const {
        for (int h = 0; h < 2; ++h)
            for (int s = 0; s < fill[h]; ++s)
                if (row[h * 16 + s] == r) return true;
        return false;
    }
};

// Greedy packer of one warp's stream.  An entry goes to the oldest open group
// with a half-warp where its y bank and x bank are still free (conflict
// degree 1); failing that, to the oldest where both stay <= 2; failing that,
// to a new group.  Rows within a group are always distinct.
class Packer {
  public:
    Packer(bool interior, std::vector<double>& val, std::vector<uint32_t>& idx, std::vector<int32_t>* minc)
        : interior_(interior), oval_(val), oidx_(idx), ominc_(minc) {}

    // interior: a = column offset from the panel's col0, chunk = a / kXsW
    // border  : a unused for banks, chunk = 0
    void place(int32_t r, int32_t a, int32_t chunk, double v, uint32_t border_idx) {
        const int yb = r & 15, xb = a & 15;
        for (int cap = 1; cap <= 3; ++cap) {
            for (size_t gi = 0; gi < q_.size(); ++gi) {
                Grp& g = q_[gi];
                if (g.closed || g.full()) continue;
                for (int h = 0; h < 2; ++h) {
                    if (g.fill[h] == 16 || g.yc[h][yb] >= cap) continue;
                    if (interior_ && g.xc[h][xb] >= cap) continue;
                    if (g.has_row(r)) break;
                    put(g, h, r, a, v, border_idx, yb, xb);
                    if (g.full()) --open_;
                    flush();
                    return;
                }
            }
        }
        q_.emplace_back();
        Grp& g = q_.back();
        std::memset(g.xc, 0, sizeof g.xc);
        std::memset(g.yc, 0, sizeof g.yc);
        g.fill[0] = g.fill[1] = 0;
        g.minc = chunk;
        g.closed = false;
        ++open_;
        put(g, 0, r, a, v, border_idx, yb, xb);
        if (open_ > kMaxOpen || q_.size() > kMaxDeque) close_oldest();
        flush();
    }

    // before entries of chunk j: groups whose first chunk is < j-1 cannot take more
    void begin_chunk(int32_t j) {
        for (Grp& g : q_)
            if (!g.closed && !g.full() && g.minc < j - 1) {
                g.closed = true;
                --open_;
            }
        flush();
    }

    void finish() {
        for (Grp& g : q_)
            if (!g.closed && !g.full()) {
                g.closed = true;
                --open_;
            }
        flush();
    }

    int64_t groups = 0, pads = 0;

  private:
    void put(Grp& g, int h, int32_t r, int32_t a, double v, uint32_t border_idx, int yb, int xb) {
        const int lane = h * 16 + g.fill[h]++;
        g.idx[lane] = interior_ ? ((uint32_t)r << 16) | (uint32_t)(a - g.minc * kXsW) : border_idx;
        g.val[lane] = v;
        g.row[lane] = r;
        g.yc[h][yb]++;
        if (interior_) g.xc[h][xb]++;
    }
    void close_oldest() {
        for (Grp& g : q_)
            if (!g.closed && !g.full()) {
                g.closed = true;
                --open_;
                return;
            }
    }
    void flush() {
        while (!q_.empty() && (q_.front().closed || q_.front().full())) {
            Grp& g = q_.front();
            // lanes: half h slots [h*16, h*16 + fill[h]); the rest padding
            for (int h = 0; h < 2; ++h)
                for (int s = g.fill[h]; s < 16; ++s) {
                    g.idx[h * 16 + s] = kXsDummy;
                    g.val[h * 16 + s] = 0.0;
                    ++pads;
                }
            oval_.insert(oval_.end(), g.val, g.val + 32);
            oidx_.insert(oidx_.end(), g.idx, g.idx + 32);
            if (ominc_) ominc_->push_back(g.minc);
            ++groups;
            q_.pop_front();
        }
    }

    bool interior_;
    std::vector<double>& oval_;
    std::vector<uint32_t>& oidx_;
    std::vector<int32_t>* ominc_;
    std::deque<Grp> q_;
    int open_ = 0;
};

void pack_panel(const std::vector<int64_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
                int64_t gb, int cbits, XsPanelData& P) {
    const XsPanel& d = P.desc;
    const int NW = kXsWarps;
    P.g_cnt.assign(NW, 0);
    P.b_cnt.assign(NW, 0);
    P.u_rel.assign((size_t)NW * std::max(d.nch, 1), 0);
    std::vector<int32_t> cnt(d.nch + 1), minc;
    std::vector<int32_t> er, ea;     // bucketed entries: row, window column
    std::vector<double> ev;
    std::vector<int64_t> eorder;
    for (int w = 0; w < NW; ++w) {
        const int64_t ra = (int64_t)d.row0 + (int64_t)w * d.rw;
        const int64_t rb = std::max(ra, std::min<int64_t>(ra + d.rw, (int64_t)d.row0 + d.nrows));
        // ---- interior entries, bucketed by chunk (stable: row order, then column)
        std::fill(cnt.begin(), cnt.end(), 0);
        int64_t ni = 0;
        for (int64_t r = ra; r < rb; ++r)
            for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
                const int64_t c = col[e];
                if (c >= d.col0 && c < d.col_end) {
                    ++cnt[(c - d.col0) / kXsW + 1];
                    ++ni;
                }
            }
        for (int j = 0; j < d.nch; ++j) cnt[j + 1] += cnt[j];
        er.resize(ni);
        ea.resize(ni);
        ev.resize(ni);
        {
            // within a chunk, entries go round-robin over the rows (the k-th
            // entry of every row, then the (k+1)-th ...): consecutive entries
            // then have distinct rows and consecutive y banks
            std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
            std::vector<int64_t> cur(rb - ra);
            for (int64_t r = ra; r < rb; ++r) cur[r - ra] = rp[r];
            bool more = true;
            while (more) {
                more = false;
                for (int64_t r = ra; r < rb; ++r) {
                    int64_t& e = cur[r - ra];
                    // next interior entry of row r (skip border entries)
                    while (e < rp[r + 1] && !(col[e] >= d.col0 && col[e] < d.col_end)) ++e;
                    if (e >= rp[r + 1]) continue;
                    more = true;
                    const int32_t a = (int32_t)(col[e] - d.col0);
                    const int32_t k = pos[a / kXsW]++;
                    er[k] = (int32_t)(r - d.row0);
                    ea[k] = a;
                    ev[k] = val[e];
                    ++e;
                }
            }
        }
        minc.clear();
        Packer pi(true, P.gval, P.gidx, &minc);
        for (int j = 0; j < d.nch; ++j) {
            pi.begin_chunk(j);
            for (int32_t k = cnt[j]; k < cnt[j + 1]; ++k) pi.place(er[k], ea[k], j, ev[k], 0);
        }
        pi.finish();
        P.g_cnt[w] = (int32_t)pi.groups;
        P.pad_i += pi.pads;
        P.entries += ni;
        // U[j] = first group (relative) whose first chunk is >= j
        {
            size_t g = 0;
            for (int j = 0; j < d.nch; ++j) {
                while (g < minc.size() && minc[g] < j) ++g;
                P.u_rel[(size_t)w * d.nch + j] = (int32_t)g;
            }
        }
        // ---- border entries (columns >= gb), gathered from L2 by the kernel
        Packer pb(false, P.bval, P.bidx, nullptr);
        int64_t nb = 0;
        for (int64_t r = ra; r < rb; ++r)
            for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
                const int64_t c = col[e];
                if (c >= gb) {
                    const uint32_t bidx = ((uint32_t)(r - ra) << cbits) | (uint32_t)(c - gb);
                    pb.place((int32_t)(r - d.row0), 0, 0, val[e], bidx);
                    ++nb;
                }
            }
        pb.finish();
        P.b_cnt[w] = (int32_t)pb.groups;
        P.pad_b += pb.pads;
        P.entries += nb;
    }
}

}  // namespace

bool plan_xstage(const std::vector<int64_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
                 const std::vector<XsBlockIn>& blocks, int64_t gb, int64_t g_len, int64_t rows_target,
                 std::vector<XsPanelData>& out, int& cbits, XsPlanStats& st, std::string& why) {
    out.clear();
    st = XsPlanStats{};
    cbits = 1;
    while (cbits < 31 && (int64_t(1) << cbits) < std::max<int64_t>(g_len, 1)) ++cbits;
    const int64_t rw_max = (int64_t(1) << (32 - cbits)) - 1;   // rows per warp the border index can address
    int64_t R = std::min<int64_t>(std::max<int64_t>(rows_target, kXsWarps), kXsRowsMax);
    R = std::min<int64_t>(R, rw_max * kXsWarps);
    if (R < kXsWarps) {
        why = "border too wide for the packed border index";
        return false;
    }
    // panels: block k's rows cut into ceil(L / R) near-equal panels
    std::vector<XsPanel> descs;
    for (const XsBlockIn& b : blocks) {
        const int64_t L = b.r1 - b.r0;
        if (L <= 0) continue;
        if (b.c1 - b.c0 > (int64_t)INT32_MAX / 2) {
            why = "block interior too wide";
            return false;
        }
        const int64_t np = (L + R - 1) / R;
        for (int64_t p = 0; p < np; ++p) {
            const int64_t a = b.r0 + L * p / np, e = b.r0 + L * (p + 1) / np;
            XsPanel d{};
            d.row0 = (int32_t)a;
            d.nrows = (int32_t)(e - a);
            d.col0 = (int32_t)b.c0;
            d.col_end = (int32_t)b.c1;
            d.nch = (int32_t)((b.c1 - b.c0 + kXsW - 1) / kXsW);
            d.rw = (d.nrows + kXsWarps - 1) / kXsWarps;
            descs.push_back(d);
        }
    }
    out.resize(descs.size());
    for (size_t p = 0; p < descs.size(); ++p) out[p].desc = descs[p];
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < (int64_t)out.size(); ++p) pack_panel(rp, col, val, gb, cbits, out[p]);
    int64_t u = 0;
    for (XsPanelData& P : out) {
        P.desc.u_base = (int32_t)u;
        u += (int64_t)kXsWarps * P.desc.nch;
        if (u > INT32_MAX) {
            why = "chunk tables beyond int32";
            return false;
        }
        st.panels++;
        st.groups_i += (int64_t)P.gidx.size() / 32;
        st.groups_b += (int64_t)P.bidx.size() / 32;
        st.entries += P.entries;
        st.pad_i += P.pad_i;
        st.pad_b += P.pad_b;
    }
    if ((st.groups_i + 1) * 32 > INT32_MAX || (st.groups_b + 1) * 32 > INT32_MAX) {
        why = "too many groups for int32 group ids";
        return false;
    }
    return true;
}

}  // namespace spmvb

namespace spmvb {

// Test hook: decodes the packed streams back into (row, column, value)
// triples and checks them against the CSR bit for bit, together with the
// format's invariants (distinct rows per group, at most two consecutive
// chunks per group, dummy slots carry 0).  Host only.
bool verify_xstage(const std::vector<int64_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
                   int64_t gb, int cbits, const std::vector<XsPanelData>& pd, std::string& why) {
    const int NW = kXsWarps;
    const uint32_t cmask = (1u << cbits) - 1u;
    bool ok = true;
    std::string err;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < (int64_t)pd.size(); ++p) {
        const XsPanelData& P = pd[p];
        const XsPanel& d = P.desc;
        std::vector<std::vector<std::pair<int64_t, double>>> got(d.nrows);
        std::string e;
        int64_t go = 0, bo = 0;
        for (int w = 0; w < NW && e.empty(); ++w) {
            const int64_t lo = (int64_t)w * d.rw, hi = std::min<int64_t>(lo + d.rw, d.nrows);
            for (int64_t q = 0; q < P.g_cnt[w] && e.empty(); ++q) {
                int j = 0;
                while (j + 1 < d.nch && P.u_rel[(size_t)w * d.nch + j + 1] <= q) ++j;
                std::vector<int64_t> rows;
                for (int l = 0; l < 32; ++l) {
                    const uint32_t i = P.gidx[(go + q) * 32 + l];
                    const double v = P.gval[(go + q) * 32 + l];
                    if (i == kXsDummy) {
                        if (v != 0.0) e = "dummy slot with a value";
                        continue;
                    }
                    const int64_t r = i >> 16, off = i & 0xFFFF;
                    const int64_t c = (int64_t)d.col0 + (int64_t)j * kXsW + off;
                    if (r < lo || r >= hi) e = "interior row outside the warp's range";
                    else if (off >= 2 * kXsW || c >= d.col_end) e = "interior column outside the window";
                    else if ((c - d.col0) / kXsW != j && (c - d.col0) / kXsW != j + 1) e = "group spans > 2 chunks";
                    else {
                        got[r].push_back({c, v});
                        rows.push_back(r);
                    }
                }
                std::sort(rows.begin(), rows.end());
                if (std::adjacent_find(rows.begin(), rows.end()) != rows.end()) e = "repeated row in a group";
            }
            for (int64_t q = 0; q < P.b_cnt[w] && e.empty(); ++q) {
                std::vector<int64_t> rows;
                for (int l = 0; l < 32; ++l) {
                    const uint32_t i = P.bidx[(bo + q) * 32 + l];
                    const double v = P.bval[(bo + q) * 32 + l];
                    if (i == kXsDummy) {
                        if (v != 0.0) e = "dummy slot with a value";
                        continue;
                    }
                    const int64_t r = lo + (int64_t)(i >> cbits), c = gb + (int64_t)(i & cmask);
                    if (r >= hi) e = "border row outside the warp's range";
                    else {
                        got[r].push_back({c, v});
                        rows.push_back(r);
                    }
                }
                std::sort(rows.begin(), rows.end());
                if (std::adjacent_find(rows.begin(), rows.end()) != rows.end()) e = "repeated row in a border group";
            }
            go += P.g_cnt[w];
            bo += P.b_cnt[w];
        }
        for (int64_t r = 0; r < d.nrows && e.empty(); ++r) {
            auto& g = got[r];
            std::sort(g.begin(), g.end(), [](const std::pair<int64_t, double>& a, const std::pair<int64_t, double>& b) {
                return a.first < b.first;
            });
            const int64_t R = d.row0 + r;
            if ((int64_t)g.size() != rp[R + 1] - rp[R]) {
                e = "row nonzero count differs";
                break;
            }
            for (int64_t t = 0; t < (int64_t)g.size(); ++t)
                if (g[t].first != col[rp[R] + t] || std::memcmp(&g[t].second, &val[rp[R] + t], 8) != 0) {
                    e = "decoded (column, value) differs from the CSR";
                    break;
                }
        }
        if (!e.empty()) {
#pragma omp critical
            {
                ok = false;
                err = e + " (panel " + std::to_string(p) + ")";
            }
        }
    }
    if (!ok) why = err;
    return ok;
}

}  // namespace spmvb
