// test_hooks.cpp -- the test and debug hooks of include/spmv_test.h.  They
// read the library's state back or run host-only planner round trips; none
// changes what a handle made through include/spmv.h computes.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/spmv_test.h"
#include "exchange.h"
#include "handle.h"

using namespace spmvb;

extern "C" {

spmv_status_t spmv_debug_copy_csr(spmv_handle_t h, int64_t* row_ptr, int32_t* col, double* val) {
    if (!valid(h) || !row_ptr || (h->nnz_loc && (!col || !val))) return fail(SPMV_ERR_USAGE, "bad arguments");
    if (h->nnz_loc && !h->d_col)
        return fail(SPMV_ERR_UNSUPPORTED, "the device CSR was released (panel kernel); create with retain_csr");
    DeviceGuard g(h->device);
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
        std::vector<PnPanelData> pd;
        PnPlanStats st;
        std::string why;
        // SB: columns >= C_B's start come from the second x pointer (the border
        // exchange buffer at world > 1); groups must not mix the two sides
        const int64_t xs = (blocks && blocks->K > 0 && blocks->col_block_ptr) ? blocks->col_block_ptr[blocks->K]
                                                                            : (int64_t)INT32_MAX;
        if (!plan_panel(rp, c, v, ranges, xs, rows_target, pd, st, why))
            return fail(SPMV_ERR_UNSUPPORTED, "pn_plan_check: %s", why.c_str());
        int64_t smax = 0, with_border = 0;
        for (const auto& P : pd) {
            smax = std::max<int64_t>(smax, panel_smem_bytes((P.nslots + 15) & ~15, (int64_t)P.split_slots.size(),
                                                            (int64_t)P.split_first.size()));
            if (P.desc.bepoch < P.desc.ne) ++with_border;
            for (int64_t g = 0; g < (int64_t)P.desc.bepoch * kPnEpoch && g < (int64_t)P.gbase.size(); ++g)
                if (P.gbase[g] >= xs) return fail(SPMV_ERR_INTERNAL, "pn_plan_check: border group before bepoch");
        }
        stats[0] = st.panels; stats[1] = st.groups; stats[2] = st.pads;
        stats[3] = st.deferred; stats[4] = st.epochs; stats[5] = st.entries;
        stats[6] = (int64_t)(st.ywf0 * 1000.0); stats[7] = (int64_t)(st.ywf1 * 1000.0);
        stats[8] = smax; stats[9] = with_border; stats[10] = st.gsectors;
        stats[11] = st.pads_drain; stats[12] = st.epochs_drain;
        stats[13] = st.far; stats[14] = st.far_steps;
        if (st.entries != nnz) return fail(SPMV_ERR_INTERNAL, "pn_plan_check: plan holds %lld of %lld nonzeros",
                                           (long long)st.entries, (long long)nnz);
        if (smax > kPnSmemMax) return fail(SPMV_ERR_INTERNAL, "pn_plan_check: a panel needs %lld B of shared memory",
                                           (long long)smax);
        if (!verify_panel(rp, c, v, xs, pd, why)) return fail(SPMV_ERR_INTERNAL, "pn_plan_check: %s", why.c_str());
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
            for (int64_t i = rbp[k]; i < rbp[k + 1]; ++i) blk[k] += row_slots(row_ptr[i + 1] - row_ptr[i]);
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
                    if (world > 1) l = g >= cbp[K] ? sh.x_interior_len + (g - cbp[K]) : g - sh.x_interior_begin;
                    c.push_back((int32_t)l);
                    v.push_back(val[t]);
                }
                rp[i + 1] = (int64_t)c.size();
            }
            const PnSetup S = pn_setup(SPMV_SB, world, R0, ml, ml, sh.x_interior_begin, sh.x_interior_len, n, rbp, cbp,
                                       blk, rp, nullptr, sms, 0);
            std::vector<PnPanelData> pd;
            PnPlanStats st;
            std::string why;
            if (!plan_panel(rp, c, v, S.ranges, S.xs, S.target, pd, st, why, S.xcols.empty() ? nullptr : &S.xcols,
                            S.sms, nullptr, S.waves * S.sms, S.global ? &S.range_panels : nullptr))
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
                        if (pn_is_dummy(i)) continue;
                        const int32_t sl = (int32_t)(i >> kPnDeltaBits);
                        const int64_t lc = (int64_t)P.gbase[g] + (i & ((1u << kPnDeltaBits) - 1));
                        int64_t gc = lc;
                        if (world > 1)
                            gc = lc >= sh.x_interior_len ? cbp[K] + (lc - sh.x_interior_len) : lc + sh.x_interior_begin;
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

spmv_status_t spmv_test_create_rank(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                                     const double* val, const int32_t* row_perm, const int32_t* col_perm,
                                     const spmv_blocks_t* blocks, int32_t n_parts, const int32_t* part_of_nnz,
                                     const spmv_dist_t* dist, const spmv_options_t* options, spmv_handle_t* out) {
    if (!dist || dist->world < 2) return fail(SPMV_ERR_USAGE, "test_create_rank: needs a dist with world > 1");
    return create_common(m, n, nnz, row_ptr, col_idx, val, row_perm, col_perm, blocks, n_parts, part_of_nnz, dist,
                         options, true, out);
}

spmv_status_t spmv_test_loopback_link(spmv_handle_t* handles, int32_t world) {
    if (!handles || world < 2) return fail(SPMV_ERR_USAGE, "loopback_link: bad arguments");
    return xchg_loopback_link(handles, world);
}

spmv_status_t spmv_test_corrupt_panel(spmv_handle_t h, int32_t kind) {
    if (!valid(h) || kind < 1 || kind > 3) return fail(SPMV_ERR_USAGE, "corrupt_panel: bad arguments");
    if (h->kernel != 7 || !h->pn.ok()) return fail(SPMV_ERR_UNSUPPORTED, "corrupt_panel: not a panel handle");
    DeviceGuard g(h->device);
    // panel 0, epoch 0: warp 0's and warp 1's 128-entry blocks, (lane, step) -> l * 4 + b
    PnPanel p0;
    CUDA_TRY(cudaMemcpy(&p0, h->pn.d_panel, sizeof p0, cudaMemcpyDeviceToHost));
    uint32_t blk[256];
    uint32_t* dev = h->pn.d_gidx + (int64_t)p0.g0 * 32;
    CUDA_TRY(cudaMemcpy(blk, dev, sizeof blk, cudaMemcpyDeviceToHost));
    const uint32_t mask = (1u << kPnDeltaBits) - 1u;
    int a = -1, b = -1;   // a real entry of warp 0 and one of warp 1
    for (int q = 0; q < 128 && a < 0; ++q)
        if ((blk[q] >> kPnDeltaBits) < (uint32_t)h->pn.max_rows) a = q;
    for (int q = 128; q < 256 && b < 0; ++q)
        if ((blk[q] >> kPnDeltaBits) < (uint32_t)h->pn.max_rows) b = q;
    if (a < 0 || b < 0) return fail(SPMV_ERR_UNSUPPORTED, "corrupt_panel: epoch 0 too sparse");
    if (kind == 1) blk[b] = (blk[a] & ~mask) | (blk[b] & mask);              // warp 1 updates warp 0's row
    if (kind == 2) blk[b] = ((uint32_t)(h->pn.max_rows + 100) << kPnDeltaBits) | (blk[b] & mask);   // slot
    if (kind == 3) blk[b] = (blk[b] & ~mask) | mask;                           // column delta 2^17 - 1
    CUDA_TRY(cudaMemcpy(dev, blk, sizeof blk, cudaMemcpyHostToDevice));
    return SPMV_OK;
}

spmv_status_t spmv_test_panel_stamps(spmv_handle_t h, int32_t mode, uint64_t* out, int64_t cap) {
    if (!valid(h) || mode < 0 || mode > 1 || (mode == 0 && (!out || cap < 0)))
        return fail(SPMV_ERR_USAGE, "panel_stamps: bad arguments");
    if (h->kernel != 7 || !h->pn.ok()) return fail(SPMV_ERR_UNSUPPORTED, "panel_stamps: not a panel handle");
    DeviceGuard g(h->device);
    const int64_t n = (int64_t)h->pn.panels * 8;
    if (mode == 1) {
        if (!h->d_stamps) CUDA_TRY(cudaMalloc(&h->d_stamps, n * sizeof(unsigned long long)));
        CUDA_TRY(cudaMemset(h->d_stamps, 0, n * sizeof(unsigned long long)));
        return SPMV_OK;
    }
    if (!h->d_stamps) return fail(SPMV_ERR_USAGE, "panel_stamps: not armed");
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(out, h->d_stamps, std::min(n, cap) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaFree(h->d_stamps));
    h->d_stamps = nullptr;
    return SPMV_OK;
}

spmv_status_t spmv_test_rank_stream(spmv_handle_t h, void** stream) {
    if (!valid(h) || !stream) return fail(SPMV_ERR_USAGE, "rank_stream: bad arguments");
    if (!h->test_rank || !h->test_stream) return fail(SPMV_ERR_USAGE, "rank_stream: not a linked test rank");
    *stream = (void*)h->test_stream;
    return SPMV_OK;
}

}  // extern "C"
