// plan_panel.cpp -- host planner of the column-sorted panel kernel (panel.cu).
//
// Why this layout (measured, profiles/r01_micro.json): a warp-wide 8-byte
// gather from L2 costs one L1TEX wavefront per distinct 128-byte line, so the
// row-ordered CSR loop pays one wavefront per nonzero (C5's columns are
// random within a 980,000-column SB block, Eq.(1)).  The temporal
// locality the SB reordering creates (rows of one block only touch
// x(C_k) and x(C_B)) is exploited here by processing a large panel of rows
// of one block together: sorted by column, the panel's nonzeros hit each x
// line several times in a row, so 32 consecutive nonzeros touch only a few
// lines.  y of the panel lives in shared memory (the per-row temporary of
// P:L41-49 becomes a shared-memory accumulator written to HBM once).
//
// Plan of one panel:
//   1. its nonzeros, sorted by (column, row-major position);
//   2. epochs: runs of kPnEpoch groups whose rows are all distinct, filled in
//      column order; a nonzero whose row is already in the epoch is deferred
//      to the next epoch (taken first there);
//   3. groups: 32 consecutive nonzeros of an epoch sharing a base column
//      (column - base < 2^17) and one side of x_split; within a group the
//      lanes alternate between the half-warps by y bank (row mod 16) so that
//      the shared-memory y updates spread over the banks;
//   4. padding: kPnDummy slots (the lane does nothing) and all-dummy groups
//      completing the last epoch.
// Row sums therefore accumulate in column order (ascending, except deferred
// nonzeros); any order is within the oracle tolerance (reading A6), and the
// plan is deterministic.
#include "plan_panel.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <omp.h>

namespace spmvb {
namespace {

struct Ent {
    int32_t row;   // row in panel
    int32_t col;   // local column id
    double v;
};

class Emitter {
  public:
    explicit Emitter(std::vector<Ent>& ents, std::vector<int32_t>& bases) : E_(ents), B_(bases) {}
    void add(const Ent& e) { cur_[n_++] = e; }
    int size() const { return n_; }
    int32_t base() const { return cur_[0].col; }
    void close() {   // the group's entries (row -1 = padding), emitted after the y-slot colouring
        for (int k = 0; k < 32; ++k) E_.push_back(k < n_ ? cur_[k] : Ent{-1, 0, 0.0});
        B_.push_back(n_ ? cur_[0].col : 0);
        n_ = 0;
    }

  private:
    std::vector<Ent>& E_;
    std::vector<int32_t>& B_;
    Ent cur_[32];
    int n_ = 0;
};

// Shared-memory y slots: 8-byte bank = slot mod 16.  A warp-wide 64-bit access
// costs (per half-warp) as many wavefronts as the most repeated bank, so the
// rows of each group should spread over the 16 banks.  Start from slot = row
// (bank = row mod 16, all banks the same size) and improve by swapping the
// banks of two rows when that lowers sum over groups of sum_b count_b^2 (a
// local search, deterministic: fixed pseudo-random order).  Then rows of bank
// b take slots b, b+16, ... in row order.
void colour_slots(int32_t nr, const std::vector<Ent>& ents, int64_t G, std::vector<uint16_t>& row2slot,
                  std::vector<int32_t>& slot_of_row) {
    std::vector<int32_t> bank(nr);
    for (int32_t r = 0; r < nr; ++r) bank[r] = r & 15;
    // row -> groups
    std::vector<int32_t> rg_ptr(nr + 1, 0);
    for (int64_t i = 0; i < G * 32; ++i)
        if (ents[i].row >= 0) rg_ptr[ents[i].row + 1]++;
    for (int32_t r = 0; r < nr; ++r) rg_ptr[r + 1] += rg_ptr[r];
    std::vector<int32_t> rg(rg_ptr[nr]), fill(rg_ptr.begin(), rg_ptr.end() - 1);
    for (int64_t g = 0; g < G; ++g)
        for (int k = 0; k < 32; ++k) {
            const int32_t r = ents[g * 32 + k].row;
            if (r >= 0) rg[fill[r]++] = (int32_t)g;
        }
    std::vector<uint8_t> cnt(G * 16, 0);
    for (int64_t g = 0; g < G; ++g)
        for (int k = 0; k < 32; ++k) {
            const int32_t r = ents[g * 32 + k].row;
            if (r >= 0) cnt[g * 16 + bank[r]]++;
        }
    // rows of each bank (for picking swap partners)
    std::vector<std::vector<int32_t>> of_bank(16);
    std::vector<int32_t> pos(nr);
    for (int32_t r = 0; r < nr; ++r) {
        pos[r] = (int32_t)of_bank[bank[r]].size();
        of_bank[bank[r]].push_back(r);
    }
    uint64_t rs = 0x9E3779B97F4A7C15ull ^ (uint64_t)nr;
    auto rnd = [&]() {
        rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17;
        return rs;
    };
#ifndef SPMV_PN_WPOW
#define SPMV_PN_WPOW 3
#endif
// Round 2, first form: 8 sweeps x 8 random (bank, partner) tries per row --
// predicted y wavefronts per access 4.02 -> 3.79 on C5's geometry (C5 SpMxV
// -1.0 % sustained) but three quarters of spmv_create's planning time.  Now
// directed (below): 4 sweeps x 2 best banks x 3 partners reach 3.75 (C4: 3.42
// against 3.45) in 0.3x the colouring time; 8 such sweeps give 3.70, the
// plateau 32 sweeps of the random form reached (3.695).
#ifndef SPMV_PN_SWEEPS
#define SPMV_PN_SWEEPS 4
#endif
#ifndef SPMV_PN_TRIES
#define SPMV_PN_TRIES 3
#endif
#ifndef SPMV_PN_CBANKS
#define SPMV_PN_CBANKS 2
#endif
    int64_t W[34];
    for (int c = 0; c < 34; ++c) {
        int64_t v = 1;
        for (int k = 0; k < SPMV_PN_WPOW; ++k) v *= c;
        W[c] = v;
    }
    // groups of the swap partner, marked once per candidate pair (a group
    // holding both rows of a swap keeps its counts: the moves cancel)
    std::vector<uint32_t> gmark(std::max<int64_t>(G, 1), 0);
    uint32_t tag = 0;
    auto mark_groups = [&](int32_t r) {
        ++tag;
        for (int32_t q = rg_ptr[r]; q < rg_ptr[r + 1]; ++q) gmark[rg[q]] = tag;
    };
    auto gain_move = [&](int32_t r, int b1, int b2) {
        // cost change of moving r from b1 to b2, skipping the marked groups
        int64_t d = 0;
        for (int32_t q = rg_ptr[r]; q < rg_ptr[r + 1]; ++q) {
            const int64_t g = rg[q];
            if (gmark[g] == tag) continue;
            d += W[cnt[g * 16 + b2] + 1] - W[cnt[g * 16 + b2]] + W[cnt[g * 16 + b1] - 1] - W[cnt[g * 16 + b1]];
        }
        return d;
    };
    auto apply_move = [&](int32_t r, int b1, int b2) {
        for (int32_t q = rg_ptr[r]; q < rg_ptr[r + 1]; ++q) {
            const int64_t g = rg[q];
            cnt[g * 16 + b1]--;
            cnt[g * 16 + b2]++;
        }
    };
    // Directed swaps: one pass over r's groups gives the cost change of moving
    // r to each of the 16 banks (add[b]) and of leaving its own (rem); the
    // kPnColBanks best target banks are tried with kPnColTries random partners
    // each, whose own move back to r's bank is evaluated the same way.  These
    // estimates ignore groups holding both rows (their moves cancel there), so
    // the chosen swap is re-evaluated exactly (group marks) before it is applied.
    int64_t DA[34], DR[34];   // DA[c] = W[c+1] - W[c] (c <= 32), DR[c] = W[c-1] - W[c] (c >= 1)
    for (int c = 0; c < 33; ++c) DA[c] = W[c + 1] - W[c];
    for (int c = 1; c < 34; ++c) DR[c] = W[c - 1] - W[c];
    DA[33] = 0;
    DR[0] = 0;
    constexpr int kSweeps = SPMV_PN_SWEEPS, kTries = SPMV_PN_TRIES, kBanks = SPMV_PN_CBANKS;
    for (int sw = 0; sw < kSweeps; ++sw)
        for (int32_t i = 0; i < nr; ++i) {
            const int32_t r = (int32_t)((i * 40503ull + sw * 7919ull) % (uint64_t)nr);   // fixed visiting order
            if (rg_ptr[r + 1] == rg_ptr[r]) continue;
            const int b1 = bank[r];
            int64_t add[16] = {0}, rem = 0;
            for (int32_t q = rg_ptr[r]; q < rg_ptr[r + 1]; ++q) {
                const uint8_t* c = &cnt[(int64_t)rg[q] * 16];
                for (int b = 0; b < 16; ++b) add[b] += DA[c[b]];
                rem += DR[c[b1]];
            }
            add[b1] = INT64_MAX;
            int64_t best = 0;
            int32_t bs = -1;
            for (int kb = 0; kb < kBanks; ++kb) {
                int b2 = 0;
                for (int b = 1; b < 16; ++b)
                    if (add[b] < add[b2]) b2 = b;
                if (add[b2] == INT64_MAX) break;
                const int64_t d1 = rem + add[b2];
                add[b2] = INT64_MAX;
                if (of_bank[b2].empty()) continue;
                for (int k = 0; k < kTries; ++k) {
                    const int32_t s2 = of_bank[b2][rnd() % of_bank[b2].size()];
                    int64_t d = d1;
                    for (int32_t q = rg_ptr[s2]; q < rg_ptr[s2 + 1]; ++q) {
                        const uint8_t* c = &cnt[(int64_t)rg[q] * 16];
                        d += DA[c[b1]] + DR[c[b2]];
                    }
                    if (d < best) { best = d; bs = s2; }
                }
            }
            if (bs >= 0) {
                const int b2 = bank[bs];
                mark_groups(bs);
                int64_t d = gain_move(r, b1, b2);
                mark_groups(r);
                d += gain_move(bs, b2, b1);
                if (d >= 0) continue;
                apply_move(r, b1, b2);
                apply_move(bs, b2, b1);
                std::swap(of_bank[b1][pos[r]], of_bank[b2][pos[bs]]);
                std::swap(pos[r], pos[bs]);
                bank[r] = b2;
                bank[bs] = b1;
            }
        }
    row2slot.assign(nr, 0);
    slot_of_row.assign(nr, 0);
    std::vector<int32_t> next(16, 0);
    for (int32_t r = 0; r < nr; ++r) {
        const int32_t sl = bank[r] + 16 * next[bank[r]]++;
        row2slot[r] = (uint16_t)sl;
        slot_of_row[r] = sl;
    }
}

// Predicted wavefronts of one warp-wide 64-bit y access of a packed group: a
// 64-bit shared-memory access is served per half-warp, one wavefront per
// distinct address in the most loaded 8-byte bank (slot mod 16; lanes on the
// same address merge -- the padding lanes of a half share one scratch slot).
double y_wavefronts(const uint32_t* idx) {
    double w = 0;
    for (int h = 0; h < 2; ++h) {
        int c[16] = {0}, m = 0;
        bool dummy[16] = {};
        for (int l = h * 16; l < h * 16 + 16; ++l) {
            const uint32_t r = idx[l] >> kPnDeltaBits;
            if (pn_is_dummy(idx[l])) {
                const int b = (int)(r - kPnDummyRow);
                if (!dummy[b]) m = std::max(m, ++c[b]);
                dummy[b] = true;
            } else {
                m = std::max(m, ++c[r & 15]);
            }
        }
        w += std::max(m, 1);
    }
    return w;
}

// Lanes of a group: with c_b entries in bank b (slot mod 16), half-warp 0
// takes a_b of them and half 1 the rest, each half at most 16 lanes, chosen
// to minimise max_b a_b + max_b (c_b - a_b) -- the access's wavefronts (an
// alternating split pays 4 for two banks of 3 entries, this one 3).  Each
// half's padding lanes share the scratch slot of its least loaded bank.
// The half-warp split of a group's banks: bank b's c_b entries, a_b of them
// in half 0 -- minimising max_b a_b + max_b (c_b - a_b) with at most 16 lanes
// per half.  Returns that cost (each half counted at least 1: the padding
// lanes of a half share the scratch slot of its least loaded bank).
int split_banks(const int c[16], int n, int m, int a[16]) {
    for (int b = 0; b < 16; ++b) a[b] = 0;
    for (int S = m; S <= 2 * m + 2; ++S)
        for (int T0 = (S + 1) / 2; T0 <= S; ++T0) {
            const int T1 = S - T0;
            int lo_s = 0, hi_s = 0;
            bool ok = true;
            for (int b = 0; b < 16 && ok; ++b) {
                const int lo = std::max(0, c[b] - T1), hi = std::min(c[b], T0);
                ok = lo <= hi;
                lo_s += lo;
                hi_s += hi;
            }
            if (!ok || lo_s > 16 || hi_s < n - 16) continue;
            int tot = 0;
            for (int b = 0; b < 16; ++b) tot += (a[b] = std::max(0, c[b] - T1));
            for (int b = 0; b < 16 && tot < n - 16; ++b) {
                const int add = std::min(std::min(c[b], T0) - a[b], n - 16 - tot);
                a[b] += add;
                tot += add;
            }
            int m0 = 0, m1 = 0;
            for (int b = 0; b < 16; ++b) {
                m0 = std::max(m0, a[b]);
                m1 = std::max(m1, c[b] - a[b]);
            }
            return std::max(m0, 1) + std::max(m1, 1);
        }
    return 2 * m;
}

void emit_group(const Ent* e, int32_t base, const std::vector<int32_t>& slot, PnPanelData& P) {
    int c[16] = {0}, n = 0, m = 0;
    const Ent* byb[16][32];
    for (int k = 0; k < 32; ++k)
        if (e[k].row >= 0) {
            const int b = slot[e[k].row] & 15;
            byb[b][c[b]++] = &e[k];
            m = std::max(m, c[b]);
            ++n;
        }
    int a[16];
    split_banks(c, n, m, a);
    uint32_t idx[32];
    double val[32];
    int nh[2] = {0, 0}, load[2][16] = {};
    for (int b = 0; b < 16; ++b)
        for (int j = 0; j < c[b]; ++j) {
            const int h = j < a[b] ? 0 : 1;
            const Ent& x = *byb[b][j];
            const int lane = h * 16 + nh[h]++;
            idx[lane] = ((uint32_t)slot[x.row] << kPnDeltaBits) | (uint32_t)(x.col - base);
            val[lane] = x.v;
            ++load[h][b];
        }
    for (int h = 0; h < 2; ++h) {
        int bmin = 0;
        for (int b = 1; b < 16; ++b)
            if (load[h][b] < load[h][bmin]) bmin = b;
        while (nh[h] < 16) {
            const int lane = h * 16 + nh[h]++;
            idx[lane] = pn_dummy(bmin);
            val[lane] = 0.0;
        }
    }
    P.gval.insert(P.gval.end(), val, val + 32);
    P.gidx.insert(P.gidx.end(), idx, idx + 32);
    P.gbase.push_back(base);
    P.pads += 32 - n;
}

// Virtual rows of row r.  Without a split: ceil(L / kPnVMax) interleaved
// virtual rows when L > kPnSplitAt, else 1.  With a split (multiple-SpMxV,
// P:L107-109): each part segment of the row (its nonzeros of part k, in
// part order) gets its own virtual rows, split the same way by the segment's
// length -- the per-(row, part) temporaries of reading A7, folded in part
// order by the epilogue.  vr[j] (optional) receives the virtual row (relative
// to the row's first) of the row's j-th nonzero.
int32_t row_vrows(const int64_t* rp, const int32_t* part, int64_t r, int32_t* vr) {
    const int64_t a = rp[r], L = rp[r + 1] - a;
    auto nv_of = [](int64_t len) -> int32_t { return len > kPnSplitAt ? (int32_t)((len + kPnVMax - 1) / kPnVMax) : 1; };
    if (!part) {
        const int32_t nv = nv_of(L);
        if (vr)
            for (int64_t j = 0; j < L; ++j) vr[j] = (int32_t)(j % nv);
        return std::max(nv, (int32_t)1);
    }
    if (L == 0) return 1;
    // segments in part order: stable sort of the row's positions by part
    int64_t idx_small[64];
    std::vector<int64_t> idx_big;
    int64_t* idx = idx_small;
    if (L > 64) {
        idx_big.resize(L);
        idx = idx_big.data();
    }
    for (int64_t j = 0; j < L; ++j) idx[j] = j;
    std::stable_sort(idx, idx + L, [&](int64_t u, int64_t v) { return part[a + u] < part[a + v]; });
    int32_t total = 0;
    for (int64_t s0 = 0; s0 < L;) {
        int64_t s1 = s0;
        while (s1 < L && part[a + idx[s1]] == part[a + idx[s0]]) ++s1;
        const int32_t nv = nv_of(s1 - s0);
        if (vr)
            for (int64_t q = s0; q < s1; ++q) vr[idx[q]] = total + (int32_t)((q - s0) % nv);
        total += nv;
        s0 = s1;
    }
    return total;
}

void build_panel(const std::vector<int64_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
                 int64_t x_split, PnPanelData& P, const int32_t* part) {
    const int64_t r0 = P.desc.row0, nrr = P.desc.nrows;
    const int64_t a = rp[r0], n = rp[r0 + nrr] - a;
    // virtual rows: a row with L > kPnVMax nonzeros gets ceil(L / kPnVMax)
    // interleaved virtual rows (its j-th nonzero in column order goes to
    // virtual row j mod nv), so no epoch needs more than one nonzero of it
    // per virtual row; the epilogue folds them in order.
    std::vector<int32_t> vbase(nrr + 1), vcount(nrr), evr(n);
    vbase[0] = 0;
    for (int64_t r = 0; r < nrr; ++r) {
        vcount[r] = row_vrows(rp.data(), part, r0 + r, evr.data() + (rp[r0 + r] - a));
        vbase[r + 1] = vbase[r] + vcount[r];
    }
    const int64_t nr = vbase[nrr];   // virtual rows = y slots
    P.nslots = (int32_t)nr;
    if (P.rot < 0) {
        // no block structure: start the sweep where the panel's nonzeros are
        // densest (a banded matrix's diagonal band; C4's rows put 70 % of their
        // nonzeros within +-2,000 of the diagonal).  The band is where rows
        // repeat within an epoch's column window and nonzeros are deferred;
        // swept first, its deferred nonzeros drain into the sparse epochs that
        // follow instead of into near-empty epochs after the sweep's end
        // (C4: 14 % of the groups' slots were such drain padding)
        constexpr int kBin = 12;
        int64_t cmax = 0;
        for (int64_t e = a; e < a + n; ++e)
            if (col[e] < x_split) cmax = std::max<int64_t>(cmax, col[e]);
        std::vector<int64_t> h((cmax >> kBin) + 1, 0);
        for (int64_t e = a; e < a + n; ++e)
            if (col[e] < x_split) h[col[e] >> kBin]++;
        size_t b = (size_t)(std::max_element(h.begin(), h.end()) - h.begin());
        const int64_t floor_ = h[b] / 32;
        while (b > 0 && h[b - 1] > floor_) --b;
        P.rot = (int32_t)((int64_t)b << kBin);
    }
    std::vector<Ent> ents(n);
    std::vector<uint64_t> keys(n);
    for (int64_t r = 0; r < nrr; ++r)
        for (int64_t e = rp[r0 + r]; e < rp[r0 + r + 1]; ++e) {
            const int64_t i = e - a;
            const int32_t vr = vbase[r] + evr[i];
            ents[i] = {vr, col[e], val[e]};
            // rotated sweep: panels of one block start at different columns, so
            // concurrently running CTAs do not all hit the same x lines (L2
            // slices); columns >= x_split (the border C_B, Eq.(1)) come after
            // every interior column, so a panel's border groups form its last
            // epochs -- at world > 1 the border-x exchange then overlaps the
            // interior groups (a4)
            const int64_t c = col[e];
            const uint64_t rel = c >= x_split ? (uint64_t(1) << 31) | (uint64_t)(c - x_split)
                                              : (uint64_t)(c >= P.rot ? c - P.rot : c - P.rot + x_split);
            keys[i] = (rel << 32) | (uint64_t)i;
        }
    if (n > 1) {
        // keys are unique and were built in ascending entry id: a stable LSD
        // radix sort on the upper 32 bits (3 passes of 11 bits) is the full
        // sort (std::sort here was a fifth of the planning time)
        std::vector<uint64_t> tmp(n);
        std::vector<int64_t> h(2049);
        uint64_t *src = keys.data(), *dst = tmp.data();
        for (int sh = 32; sh < 64; sh += 11) {
            std::fill(h.begin(), h.end(), 0);
            for (int64_t i = 0; i < n; ++i) h[((src[i] >> sh) & 2047) + 1]++;
            if (h[((src[0] >> sh) & 2047) + 1] == n) continue;   // one bucket: the pass is the identity
            for (int b = 0; b < 2048; ++b) h[b + 1] += h[b];
            for (int64_t i = 0; i < n; ++i) dst[h[(src[i] >> sh) & 2047]++] = src[i];
            std::swap(src, dst);
        }
        if (src != keys.data()) keys.swap(tmp);
    }
    P.entries = n;
    // Sweep order; the far stream (the barrier-free phase after the epochs,
    // panel.cu) takes what is still deferred when the sweep ends (below).
    // Measured and not kept: also sending nonzeros with few
    // others of the panel within +-128 columns, or sparse deferred ones, to the
    // far stream -- C4 +2.5 %, C5 +3 % (the phase is short and its pipeline
    // fill is paid at every CTA's end).
    std::vector<int64_t> fars;   // far entries (entry ids)
    std::vector<int64_t> order(n);
    for (int64_t q = 0; q < n; ++q) order[q] = (int64_t)(keys[q] & 0xFFFFFFFFu);
    const int64_t nn = (int64_t)order.size();

    const int64_t kMaxDelta = int64_t(1) << kPnDeltaBits;
    auto side = [&](int32_t c) { return (int64_t)c >= x_split; };
    std::vector<int32_t> stamp(nr, -1);
    std::vector<int64_t> deferred, nd;
    std::vector<Ent> gents;
    std::vector<int32_t> gbases;
    Emitter em(gents, gbases);
    int64_t pos = 0;
    int32_t epoch = 0;
    std::vector<uint8_t> drain_epoch;
    while (pos < nn || !deferred.empty()) {
        int ng = 0;
        bool full = false;
        if (pos >= nn) {
            // the sweep is done: what is still deferred would fill near-empty
            // epochs one nonzero per row at a time (C4: 14 % of all slots) --
            // it goes to the far phase instead
            fars.insert(fars.end(), deferred.begin(), deferred.end());
            deferred.clear();
            break;
        }
        drain_epoch.push_back(pos >= nn);
        // returns false when the epoch is full (entry not taken)
        auto take = [&](int64_t i) -> bool {
            const Ent& e = ents[i];
            const int64_t delta = (int64_t)e.col - em.base();
            if (em.size() > 0 && (em.size() == 32 || delta < 0 || delta >= kMaxDelta || side(e.col) != side(em.base()))) {
                em.close();
                if (++ng == kPnEpoch) return false;
            }
            em.add(e);
            stamp[e.row] = epoch;
            return true;
        };
        nd.clear();
        for (int64_t i : deferred) {
            if (full || stamp[ents[i].row] == epoch) {
                nd.push_back(i);
                continue;
            }
            if (!take(i)) {
                full = true;
                nd.push_back(i);
            }
        }
        deferred.swap(nd);
        while (!full && pos < nn) {
            const int64_t i = order[pos];
            if (stamp[ents[i].row] == epoch) {
                deferred.push_back(i);
                ++P.deferred;
                ++pos;
                continue;
            }
            if (!take(i)) break;
            ++pos;
        }
        if (em.size() > 0) {
            em.close();
            ++ng;
        }
        while (ng < kPnEpoch) {   // all-dummy groups complete the epoch
            em.close();
            ++ng;
        }
        ++epoch;
    }
    P.desc.ne = epoch;
    // y-slot colouring, then the groups' lanes and packed indices
    const int64_t G = (int64_t)gbases.size();
    std::vector<int32_t> slot;
    std::vector<int32_t> ident(nr);
    for (int32_t r = 0; r < (int32_t)nr; ++r) ident[r] = r;
    if (nr > 0x7FFF) return;   // caller rejects the plan (slot field)
    {   // statistics: predicted y wavefronts with natural slots (slot = virtual row)
        double w = 0;
        for (int64_t g = 0; g < G; ++g) {
            int c[16] = {0}, n = 0, m = 0, a[16];
            for (int k = 0; k < 32; ++k) {
                const int32_t r = gents[g * 32 + k].row;
                if (r >= 0) m = std::max(m, ++c[r & 15]), ++n;
            }
            w += split_banks(c, n, m, a);
        }
        P.ywf0 = G ? w / G : 0;
    }
    std::vector<uint16_t> v2s;
    colour_slots((int32_t)nr, gents, G, v2s, slot);
    // Far stream: each virtual row's far nonzeros form one run, owned by one
    // lane (runs balanced over the CTA's kPnWarps x 32 lanes, longest first);
    // the lane sums a run in a register and adds it to the y slot once, at
    // the run's last entry (slot | kPnFarLast).  No two lanes share a slot, so
    // the phase needs no barrier.  Step s of warp w, lane l is entry
    // (s * kPnWarps + w) * 32 + l; steps are padded to whole ring turns.
    {
        std::sort(fars.begin(), fars.end(), [&](int64_t u, int64_t v) {   // by row, then CSR position
            return ents[u].row != ents[v].row ? ents[u].row < ents[v].row : u < v;
        });
        struct Run { int64_t b, e; };
        std::vector<Run> runs;
        for (int64_t q = 0; q < (int64_t)fars.size();) {
            int64_t e = q;
            while (e < (int64_t)fars.size() && ents[fars[e]].row == ents[fars[q]].row) ++e;
            runs.push_back({q, e});
            q = e;
        }
        std::stable_sort(runs.begin(), runs.end(), [](const Run& u, const Run& v) { return u.e - u.b > v.e - v.b; });
        constexpr int kBins = kPnWarps * 32;
        std::vector<int64_t> load(kBins, 0);
        std::vector<std::vector<int32_t>> bin(kBins);   // run ids per lane
        for (int32_t k = 0; k < (int32_t)runs.size(); ++k) {
            int b = 0;
            for (int j = 1; j < kBins; ++j)
                if (load[j] < load[b]) b = j;
            bin[b].push_back(k);
            load[b] += runs[k].e - runs[k].b;
        }
        int64_t fs = 0;
        for (int j = 0; j < kBins; ++j) fs = std::max(fs, load[j]);
        fs = (fs + kPnFarRing - 1) / kPnFarRing * kPnFarRing;
        P.desc.fs = (int32_t)fs;
        P.far = (int64_t)fars.size();
        const int32_t dcol = fars.empty() ? 0 : ents[fars[0]].col;   // padding: a valid x read, times 0
        P.fval.assign(fs * kBins, 0.0);
        P.fcol.assign(fs * kBins, dcol);
        P.fslot.assign(fs * kBins, kPnFarPad);
        for (int j = 0; j < kBins; ++j) {
            const int w = j / 32, l = j % 32;
            int64_t st = 0;
            for (int32_t k : bin[j])
                for (int64_t q = runs[k].b; q < runs[k].e; ++q, ++st) {
                    const Ent& e = ents[fars[q]];
                    const int64_t at = (st * kPnWarps + w) * 32 + l;
                    P.fval[at] = e.v;
                    P.fcol[at] = e.col;
                    P.fslot[at] = (uint16_t)(slot[e.row] | (q + 1 == runs[k].e ? kPnFarLast : 0));
                }
        }
    }
    // real rows -> slot, or -> split entry (virtual rows' slots in fold order)
    // split rows with <= kPnFoldSeq virtual rows first (the epilogue folds
    // those one thread per row, sequentially), then the longer ones (a warp each)
    P.row2slot.resize(nrr);
    for (int pass = 0; pass < 2; ++pass) {
        for (int64_t r = 0; r < nrr; ++r) {
            if (vcount[r] == 1) {
                if (pass == 0) P.row2slot[r] = v2s[vbase[r]];
            } else if ((vcount[r] <= kPnFoldSeq) == (pass == 0)) {
                P.row2slot[r] = (uint16_t)(0x8000 | P.split_first.size());
                P.split_first.push_back((int32_t)P.split_slots.size());
                P.split_cnt.push_back(vcount[r]);
                P.split_row.push_back((int32_t)r);
                for (int32_t j = 0; j < vcount[r]; ++j) P.split_slots.push_back(v2s[vbase[r] + j]);
            }
        }
        if (pass == 0) P.split_short = (int32_t)P.split_first.size();
    }
    double w = 0;
    for (int32_t e = 0; e < epoch; ++e) P.epochs_drain += drain_epoch[e];
    for (int64_t g = 0; g < G; ++g) {
        if (drain_epoch[g / kPnEpoch]) {
            int np = 0;
            for (int k = 0; k < 32; ++k) np += gents[g * 32 + k].row < 0;
            P.pads_drain += np;
        }
        emit_group(&gents[g * 32], gbases[g], slot, P);
        w += y_wavefronts(&P.gidx[g * 32]);
        // distinct 32-byte x sectors the group's gather requests (padding
        // lanes read x[base]): the gather bytes that cross L2 -> SM
        int64_t sec[32];
        int ns = 0;
        for (int k = 0; k < 32; ++k) {
            const int64_t c = gents[g * 32 + k].row >= 0 ? gents[g * 32 + k].col : gbases[g];
            const int64_t s = c < x_split ? (c >> 2) : ((int64_t(1) << 40) | ((c - x_split) >> 2));
            bool seen = false;
            for (int j = 0; j < ns && !seen; ++j) seen = sec[j] == s;
            if (!seen) sec[ns++] = s;
        }
        P.gsectors += ns;
    }
    P.ywf1 = G ? w / G : 0;
    // first epoch holding a border (x_split side) group: at world > 1 the
    // kernel waits for the border-x exchange before it (a4)
    P.desc.bepoch = epoch;
    for (int64_t g = 0; g < G; ++g)
        if ((int64_t)gbases[g] >= x_split) {
            P.desc.bepoch = (int32_t)(g / kPnEpoch);
            break;
        }
    P.gbase4.resize(P.gbase.size());
    for (int32_t e = 0; e < epoch; ++e)
        for (int w = 0; w < kPnWarps; ++w)
            for (int b = 0; b < kPnB; ++b)
                P.gbase4[((int64_t)e * kPnWarps + w) * kPnB + b] = P.gbase[(int64_t)e * kPnEpoch + b * kPnWarps + w];
}

}  // namespace

bool plan_panel(const std::vector<int64_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
                const std::vector<std::pair<int64_t, int64_t>>& ranges, int64_t x_split, int64_t rows_target,
                std::vector<PnPanelData>& out, PnPlanStats& st, std::string& why,
                const std::vector<std::pair<int64_t, int64_t>>* xcols, int64_t pf_sms,
                const std::vector<int32_t>* part, int64_t total_panels,
                const std::vector<int64_t>* range_panels) {
    out.clear();
    st = PnPlanStats{};
    const int64_t R = std::min<int64_t>(std::max<int64_t>(rows_target, 1), kPnRowsMax);
    const int32_t* pp = part ? part->data() : nullptr;
    auto slots_of = [&](int64_t r) -> int64_t { return row_vrows(rp.data(), pp, r, nullptr); };
    // panels per range (panel_counts), unless the caller fixed them
    std::vector<int64_t> np_of;
    if (range_panels && range_panels->size() == ranges.size()) {
        np_of = *range_panels;
    } else {
        std::vector<int64_t> Sk(ranges.size(), 0);
        for (size_t k = 0; k < ranges.size(); ++k)
            for (int64_t r = ranges[k].first; r < ranges[k].second; ++r) Sk[k] += slots_of(r);
        np_of = panel_counts(Sk, R, total_panels);
    }
    for (size_t k = 0; k < ranges.size(); ++k) {
        const auto& rg = ranges[k];
        const int64_t L = rg.second - rg.first;
        if (L <= 0) continue;
        // panel boundaries: np = ceil(slots / R) panels, cut at equal shares of
        // the bytes they move (12 per nonzero, 8 + 2 per y slot: the y write
        // and its slot map), so panels of rows with few and many nonzeros take
        // about the same time (C4's Zipf rows: balancing by slots left a 13 %
        // tail); a panel never exceeds 1.25 R slots (its y lives in shared
        // memory, and the rest of the L1 holds the loads in flight) -- when that
        // cap would add panels (a second wave), the cuts balance slots instead
        int64_t S = 0, C = 0;
        for (int64_t r = rg.first; r < rg.second; ++r) {
            const int64_t s = slots_of(r);
            S += s;
            C += 12 * (rp[r + 1] - rp[r]) + 10 * s;
        }
        const int64_t np0 = std::max<int64_t>(np_of[k], 1);
        const int64_t Rk = (S + np0 - 1) / np0;   // this range's slots per panel
        const int64_t cap = std::min<int64_t>(Rk + Rk / 4, kPnRowsMax);
        // shared memory of a panel (panel_smem_bytes): 8 B per y slot, plus 2 B
        // per slot and 12 B per row for rows split into virtual rows (the
        // epilogue's fold lists); a panel never exceeds kPnSmemMax, whatever
        // the cut mode (rows of 33-64 nonzeros need ~16 B per slot)
        auto smem_of = [](int64_t s) -> int64_t { return 8 * s + (s > 1 ? 2 * s + 12 : 0); };
#ifndef SPMV_PN_SMEM_CAP
#define SPMV_PN_SMEM_CAP kPnSmemMax
#endif
        const int64_t smem_cap = std::min<int64_t>(kPnSmemMax, SPMV_PN_SMEM_CAP) - 8 * 16 - 8 * 16 - 16;   // slack: rounding of slots / lists, scratch slots
        auto make_cuts = [&](bool by_bytes) {
            std::vector<int64_t> cut(1, rg.first);
            const int64_t tot = by_bytes ? C : S;
            int64_t acc = 0, ps = 0, pb = 0, pi = 1;
            for (int64_t r = rg.first; r < rg.second; ++r) {
                const int64_t s = slots_of(r);
                if (ps > 0 && ((by_bytes && ps + s > cap) || pb + smem_of(s) > smem_cap)) {   // caps: cut before r
                    cut.push_back(r);
                    ps = 0;
                    pb = 0;
                    while (pi < np0 && acc >= tot * pi / np0) ++pi;
                }
                acc += by_bytes ? 12 * (rp[r + 1] - rp[r]) + 10 * s : s;
                ps += s;
                pb += smem_of(s);
                if (pi < np0 && acc >= tot * pi / np0 && r + 1 < rg.second) {
                    cut.push_back(r + 1);
                    ps = 0;
                    pb = 0;
                    while (pi < np0 && acc >= tot * pi / np0) ++pi;
                }
            }
            cut.push_back(rg.second);
            return cut;
        };
        std::vector<int64_t> cut = make_cuts(true);
        if ((int64_t)cut.size() - 1 > np0) cut = make_cuts(false);   // the cap added panels: cut by slots
        int64_t np = (int64_t)cut.size() - 1;
        for (int64_t p = 0; p < np; ++p) {
            const int64_t a = cut[p], e = cut[p + 1];
            int64_t ps = 0;
            for (int64_t r = a; r < e; ++r) ps += slots_of(r);
            if (ps > kPnRowsMax || ps > (int64_t(1) << kPnRowBits) - 1) {
                why = "panel y slots beyond shared memory / the packed slot field (a very long row)";
                return false;
            }
            if (rp[e] - rp[a] >= (int64_t(1) << 32)) {
                why = "panel nonzeros beyond 2^32";
                return false;
            }
            PnPanelData d;
            d.rot = -1;   // build_panel picks the densest region (no block structure)
            d.desc.row0 = (int32_t)a;
            d.desc.nrows = (int32_t)(e - a);
            if (xcols && k < xcols->size()) {
                const int64_t c0 = (*xcols)[k].first, c1 = (*xcols)[k].second;
                d.rot = (int32_t)(c0 + (c1 - c0) * p / np);
            }
            out.push_back(std::move(d));
        }
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < (int64_t)out.size(); ++p) build_panel(rp, col, val, x_split, out[p], pp);
    int64_t g = 0;
    for (PnPanelData& P : out) {
        P.desc.g0 = (int32_t)g;
        g += (int64_t)P.gbase.size();
        if (g >= INT32_MAX / 32) {
            why = "too many groups for int32 group ids";
            return false;
        }
        st.panels++;
        st.entries += P.entries;
        st.pads += P.pads;
        st.deferred += P.deferred;
        st.gsectors += P.gsectors;
        st.pads_drain += P.pads_drain;
        st.far += P.far;
        st.far_steps += P.desc.fs;
        st.epochs_drain += P.epochs_drain;
        st.epochs += P.desc.ne;
        st.ywf0 += P.ywf0 * (double)P.gbase.size();
        st.ywf1 += P.ywf1 * (double)P.gbase.size();
    }
    st.groups = g;
    if (g) {
        st.ywf0 /= (double)g;
        st.ywf1 /= (double)g;
    }
    return true;
}

int64_t row_slots(int64_t L) { return L > kPnSplitAt ? (L + kPnVMax - 1) / kPnVMax : 1; }

std::vector<int64_t> panel_counts(const std::vector<int64_t>& Sk, int64_t R, int64_t total) {
    // ceil(slots / R) per range, or -- given a total (whole waves of one CTA
    // per SM) -- shares of that total proportional to the ranges' slots
    // (largest remainder), so several SB blocks still add up to whole waves
    // (C5: 64 blocks x 63 panels = 27.2 waves left a 0.24-wave tail)
    R = std::min<int64_t>(std::max<int64_t>(R, 1), kPnRowsMax);
    std::vector<int64_t> np(Sk.size(), 0);
    int64_t Stot = 0;
    for (size_t k = 0; k < Sk.size(); ++k) {
        Stot += Sk[k];
        np[k] = (Sk[k] + R - 1) / R;
    }
    if (total > 0 && Stot > 0) {
        std::vector<std::pair<double, size_t>> rem;
        int64_t given = 0;
        for (size_t k = 0; k < Sk.size(); ++k) {
            const double q = (double)total * (double)Sk[k] / (double)Stot;
            np[k] = Sk[k] > 0 ? std::max<int64_t>(1, (int64_t)q) : 0;
            given += np[k];
            rem.push_back({q - (double)(int64_t)q, k});
        }
        std::sort(rem.begin(), rem.end(), [](const auto& a, const auto& b) {
            return a.first != b.first ? a.first > b.first : a.second < b.second;
        });
        for (size_t j = 0; given < total && j < rem.size(); ++j)
            if (Sk[rem[j].second] > 0) { ++np[rem[j].second]; ++given; }
        for (size_t k = 0; k < Sk.size(); ++k)   // never above the slot cap
            np[k] = std::max(np[k], (Sk[k] + kPnRowsMax - 1) / kPnRowsMax);
    }
    return np;
}

int64_t panel_total_slots(const std::vector<int64_t>& rp, int64_t m, const std::vector<int32_t>* part) {
    int64_t t = 0;
    const int32_t* pp = part ? part->data() : nullptr;
#pragma omp parallel for reduction(+ : t) schedule(dynamic, 4096)
    for (int64_t r = 0; r < m; ++r) t += row_vrows(rp.data(), pp, r, nullptr);
    return t;
}

bool verify_panel(const std::vector<int64_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
                  int64_t x_split, const std::vector<PnPanelData>& pd, std::string& why) {
    bool ok = true;
    std::string err;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < (int64_t)pd.size(); ++p) {
        const PnPanelData& P = pd[p];
        const PnPanel& d = P.desc;
        std::string e;
        if ((int64_t)P.gbase.size() != (int64_t)d.ne * kPnEpoch) e = "group count != epochs * kPnEpoch";
        for (int64_t g = 0; g < (int64_t)P.gbase.size() && e.empty(); ++g) {
            const int64_t ep = g / kPnEpoch, k = g % kPnEpoch, b = k / kPnWarps, w = k % kPnWarps;
            if (P.gbase4[(ep * kPnWarps + w) * kPnB + b] != P.gbase[g]) e = "gbase4 is not the (epoch, warp, step) order of gbase";
        }
        std::vector<std::vector<std::pair<int32_t, double>>> got(d.nrows);
        const int32_t nsl = ((P.nslots + 15) / 16) * 16;
        std::vector<int32_t> stamp(nsl, -1);
        std::vector<int32_t> row_of_slot(nsl, -1);
        if ((int32_t)P.row2slot.size() != d.nrows) e = "row2slot size";
        auto own = [&](int32_t sl, int32_t r) {
            if (sl >= nsl || row_of_slot[sl] != -1) e = "slot map is not injective into the panel's slots";
            else row_of_slot[sl] = r;
        };
        for (int32_t r = 0; r < d.nrows && e.empty(); ++r) {
            const int32_t sl = P.row2slot[r];
            if (sl < 0x8000) {
                own(sl, r);
            } else {
                const int32_t k = sl & 0x7FFF;
                if (k >= (int32_t)P.split_first.size()) { e = "split index out of range"; break; }
                if ((k < P.split_short) != (P.split_cnt[k] <= kPnFoldSeq)) { e = "split rows not ordered short first"; break; }
                if (P.split_row[k] != r) { e = "split_row does not name the row"; break; }
                for (int32_t j = 0; j < P.split_cnt[k] && e.empty(); ++j) own(P.split_slots[P.split_first[k] + j], r);
            }
        }
        for (int64_t ep = 0; ep < d.ne && e.empty(); ++ep)
            for (int k = 0; k < kPnEpoch && e.empty(); ++k) {
                const int64_t g = ep * kPnEpoch + k;
                const int32_t base = P.gbase[g];
                int s = -1;
                for (int l = 0; l < 32; ++l) {
                    const uint32_t i = P.gidx[g * 32 + l];
                    const double v = P.gval[g * 32 + l];
                    if (pn_is_dummy(i)) {
                        if (v != 0.0) e = "dummy slot with a value";
                        continue;
                    }
                    const int32_t sl = (int32_t)(i >> kPnDeltaBits);
                    const int64_t c = (int64_t)base + (i & ((1u << kPnDeltaBits) - 1));
                    if (sl >= nsl || row_of_slot[sl] < 0) { e = "slot outside the panel"; break; }
                    const int32_t r = row_of_slot[sl];
                    if (stamp[sl] == ep) { e = "y slot repeated within an epoch"; break; }
                    stamp[sl] = (int32_t)ep;
                    const int sd = c >= x_split;
                    if (s >= 0 && sd != s) { e = "group mixes both sides of x_split"; break; }
                    s = sd;
                    got[r].push_back({(int32_t)c, v});
                }
            }
        // far stream: runs owned by one lane each, the slot flagged at the run's end
        if ((int64_t)P.fval.size() != (int64_t)d.fs * kPnWarps * 32 || P.fcol.size() != P.fval.size() ||
            P.fslot.size() != P.fval.size())
            e = "far stream size != fs * warps * 32";
        {
            std::vector<int32_t> owner(nsl, -1);
            for (int64_t j = 0; j < (int64_t)kPnWarps * 32 && e.empty(); ++j) {
                int32_t open = -1;   // slot of the lane's current run
                for (int64_t st = 0; st < d.fs && e.empty(); ++st) {
                    const int64_t at = (st * kPnWarps + j / 32) * 32 + j % 32;
                    const int32_t sl = P.fslot[at] & (kPnFarLast - 1);
                    const bool last = (P.fslot[at] & kPnFarLast) != 0;
                    if (P.fslot[at] == kPnFarPad) {   // padding (after the lane's runs)
                        if (open >= 0) { e = "far padding inside a run"; break; }
                        continue;
                    }
                    if (sl >= nsl || row_of_slot[sl] < 0) { e = "far slot outside the panel"; break; }
                    if (open >= 0 && sl != open) { e = "far run changes slot before its last entry"; break; }
                    if (owner[sl] >= 0 && owner[sl] != j) { e = "far slot owned by two lanes"; break; }
                    owner[sl] = (int32_t)j;
                    got[row_of_slot[sl]].push_back({P.fcol[at], P.fval[at]});
                    open = last ? -1 : sl;
                }
                if (e.empty() && open >= 0) e = "far run without a last entry";
            }
        }
        for (int64_t r = 0; r < d.nrows && e.empty(); ++r) {
            auto& gr = got[r];
            std::sort(gr.begin(), gr.end(),
                      [](const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b) { return a.first < b.first; });
            const int64_t R = d.row0 + r;
            if ((int64_t)gr.size() != rp[R + 1] - rp[R]) { e = "row nonzero count differs"; break; }
            for (int64_t t = 0; t < (int64_t)gr.size(); ++t)
                if (gr[t].first != col[rp[R] + t] || std::memcmp(&gr[t].second, &val[rp[R] + t], 8) != 0) {
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
