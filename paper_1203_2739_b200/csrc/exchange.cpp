// exchange.cpp -- the world > 1 exchange of the sharded SpMxV (P:Lnn = PAPER.md).
//
// SB (Eq.(1)): rank g owns the rows of its diagonal blocks; the row
// slices y_k <- R_k x share input only through the coupling columns C_B
// (P:L79), so one exchange per apply gathers every rank's owned slice of
// x(C_B) into every rank's border buffer (a4).
// DB split across ranks (f1): part k = block k's products; the
// border rows' per-part temporaries travel to the rank owning the row, which
// adds them in part order.
//
// Two transports:
//   * P2P (f2, the default when every GPU pair has peer access): each rank's
//     exchange buffers are one allocation mapped into every peer with CUDA
//     IPC.  Per apply seq, on a high-priority comm stream, a rank pushes its
//     slice into every peer's border buffer of parity seq & 1 with the copy
//     engines (no SM is needed, so the pushes cannot deadlock against the
//     SpMxV kernel), then writes ready[me] = seq into the peer with a stream
//     memory operation.  The SpMxV kernel starts at once: its interior epochs
//     need no exchanged data, and each CTA waits for the ready flags only
//     before its first border epoch (panel.cu) -- the exchange overlaps the
//     interior compute.  A push of apply seq waits (stream wait-value) until
//     the peer reported done >= seq - 2, i.e. finished reading that parity.
//     DB: the temporaries are pushed the same way after the kernel, and the
//     fold kernel waits for the peers' tready flags on the device (bounded),
//     so no apply stream ever blocks on a peer's progress.
//   * NCCL: in-place ncclAllGather (grouped broadcasts for unequal slices) and
//     grouped send/recv of the temporaries, on the apply stream before / after
//     the kernel (no overlap: an SpMxV kernel spinning on a flag could keep an
//     NCCL kernel from being scheduled).
// The loopback fake of SURVEY §4 runs the P2P protocol between the G ranks'
// handles of one process on one GPU (spmv_test_loopback_link).
#include <algorithm>
#include <cstring>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include "exchange.h"

namespace spmvb {
namespace {

typedef CUresult (*MemOpFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct MemOps {
    MemOpFn wait = nullptr, write = nullptr;
    bool ok = false;
};

// cuStreamWaitValue32 / cuStreamWriteValue32 through the runtime's driver
// entry points (no link-time dependency on libcuda: the library also loads on
// machines without a driver, for the host-only tests)
const MemOps& memops() {
    static const MemOps m = [] {
        MemOps r;
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            r.wait = (MemOpFn)f;
        f = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            r.write = (MemOpFn)f;
        cudaGetLastError();
        r.ok = r.wait && r.write;
        return r;
    }();
    return m;
}

spmv_status_t wait_geq(cudaStream_t s, const int32_t* addr, int32_t v) {
    const CUresult r = memops().wait((CUstream)s, (CUdeviceptr)addr, (cuuint32_t)v, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(SPMV_ERR_INTERNAL, "cuStreamWaitValue32 failed (%d)", (int)r);
    return SPMV_OK;
}

spmv_status_t write_val(cudaStream_t s, int32_t* addr, int32_t v) {
    const CUresult r = memops().write((CUstream)s, (CUdeviceptr)addr, (cuuint32_t)v, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(SPMV_ERR_INTERNAL, "cuStreamWriteValue32 failed (%d)", (int)r);
    return SPMV_OK;
}

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// Offsets of the symmetric buffer (identical on every rank).
struct XLayout {
    size_t xb[2], tin[2], ready, done, tready, tdone, err, bytes;
};

XLayout layout_of(const spmv_plan_s* h) {
    XLayout L;
    size_t o = 0;
    const size_t xbb = align256((size_t)std::max<int64_t>(h->border_total, 1) * sizeof(double));
    const size_t tb = align256((size_t)std::max<int64_t>(h->t_recv_max, 1) * sizeof(double));
    const size_t fb = align256((size_t)h->world * sizeof(int32_t));
    L.xb[0] = o; o += xbb;
    L.xb[1] = o; o += xbb;
    L.tin[0] = o; o += tb;
    L.tin[1] = o; o += tb;
    L.ready = o; o += fb;
    L.done = o; o += fb;
    L.tready = o; o += fb;
    L.tdone = o; o += fb;
    L.err = o; o += 256;
    L.bytes = o;
    return L;
}

XBufs view_of(void* base, const XLayout& L) {
    XBufs b;
    char* c = static_cast<char*>(base);
    b.base = base;
    b.bytes = L.bytes;
    b.xb[0] = reinterpret_cast<double*>(c + L.xb[0]);
    b.xb[1] = reinterpret_cast<double*>(c + L.xb[1]);
    b.tin[0] = reinterpret_cast<double*>(c + L.tin[0]);
    b.tin[1] = reinterpret_cast<double*>(c + L.tin[1]);
    b.ready = reinterpret_cast<int32_t*>(c + L.ready);
    b.done = reinterpret_cast<int32_t*>(c + L.done);
    b.tready = reinterpret_cast<int32_t*>(c + L.tready);
    b.tdone = reinterpret_cast<int32_t*>(c + L.tdone);
    b.err = reinterpret_cast<int32_t*>(c + L.err);
    return b;
}

spmv_status_t make_streams(spmv_plan_s* h) {
    if (h->comm_stream) return SPMV_OK;
    int lo = 0, hi = 0;
    CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_TRY(cudaStreamCreateWithPriority(&h->comm_stream, cudaStreamNonBlocking, hi));
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_x, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_comm, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&h->ev_kernel, cudaEventDisableTiming));
    return SPMV_OK;
}

// NCCL all-gather of a small host record (create time only)
spmv_status_t allgather_host(spmv_plan_s* h, const void* mine, size_t bytes, std::vector<char>& all) {
    char* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, bytes * h->world));
    spmv_status_t s = SPMV_OK;
    cudaError_t e = cudaMemcpy(d + bytes * h->rank, mine, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) s = fail(SPMV_ERR_INTERNAL, "cudaMemcpy: %s", cudaGetErrorString(e));
    if (!s) {
        ncclResult_t r = ncclAllGather(d + bytes * h->rank, d, bytes, ncclChar, h->comm, 0);
        if (r != ncclSuccess) s = fail(SPMV_ERR_INTERNAL, "ncclAllGather: %s", ncclGetErrorString(r));
    }
    all.resize(bytes * h->world);
    if (!s) {
        e = cudaMemcpy(all.data(), d, bytes * h->world, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) s = fail(SPMV_ERR_INTERNAL, "cudaMemcpy: %s", cudaGetErrorString(e));
    }
    cudaFree(d);
    return s;
}

spmv_status_t allreduce_min_host(spmv_plan_s* h, int32_t v, int32_t* out) {
    std::vector<char> all;
    spmv_status_t s = allgather_host(h, &v, sizeof v, all);
    if (s) return s;
    int32_t m = v;
    for (int r = 0; r < h->world; ++r) {
        int32_t q;
        memcpy(&q, all.data() + r * sizeof q, sizeof q);
        m = std::min(m, q);
    }
    *out = m;
    return SPMV_OK;
}

}  // namespace

bool stream_memops_available() { return memops().ok; }

spmv_status_t xchg_alloc(spmv_plan_s* h) {
    const XLayout L = layout_of(h);
    char* base = nullptr;
    spmv_status_t s = dalloc(h, &base, L.bytes);
    if (s) return s;
    CUDA_TRY(cudaMemset(base, 0, L.bytes));
    h->xb = view_of(base, L);
    void* hp = nullptr;
    CUDA_TRY(cudaHostAlloc(&hp, 64, cudaHostAllocMapped));
    h->xb.herr_host = static_cast<int32_t*>(hp);
    *h->xb.herr_host = 0;
    void* dp = nullptr;
    CUDA_TRY(cudaHostGetDevicePointer(&dp, hp, 0));
    h->xb.herr = static_cast<int32_t*>(dp);
    return SPMV_OK;
}

bool xchg_failed(const spmv_plan_s* h) {
    return h->xb.herr_host && *reinterpret_cast<volatile int32_t*>(h->xb.herr_host) != 0;
}

spmv_status_t xchg_agree(spmv_plan_s* h, spmv_status_t local, spmv_status_t* agreed) {
    if (!h->comm) {
        *agreed = local;
        return SPMV_OK;
    }
    // the worst status: max over ranks (0 = ok); any failure fails every rank
    int32_t neg = -(int32_t)local, m = 0;
    spmv_status_t s = allreduce_min_host(h, neg, &m);
    if (s) return s;
    *agreed = (spmv_status_t)(-m);
    return SPMV_OK;
}

spmv_status_t xchg_connect(spmv_plan_s* h) {
    h->xmode = kXNccl;
    CUDA_TRY(cudaDeviceSynchronize());
    if (h->opt.exchange == SPMV_EXCHANGE_NCCL) return make_streams(h);
    // P2P: every rank's device, IPC handle of its exchange buffer, and whether
    // it can reach every peer
    struct Rec {
        int32_t dev, ok;
        cudaIpcMemHandle_t ipc;
    } mine;
    memset(&mine, 0, sizeof mine);
    mine.dev = h->device;
    mine.ok = stream_memops_available() ? 1 : 0;
    if (mine.ok && cudaIpcGetMemHandle(&mine.ipc, h->xb.base) != cudaSuccess) {
        cudaGetLastError();
        mine.ok = 0;
    }
    std::vector<char> all;
    spmv_status_t s = allgather_host(h, &mine, sizeof mine, all);
    if (s) return s;
    std::vector<Rec> rec(h->world);
    for (int r = 0; r < h->world; ++r) memcpy(&rec[r], all.data() + r * sizeof(Rec), sizeof(Rec));
    int32_t ok = 1;
    for (int r = 0; r < h->world; ++r) {
        if (!rec[r].ok) ok = 0;
        if (r == h->rank) continue;
        int can = 0;
        if (rec[r].dev == h->device || cudaDeviceCanAccessPeer(&can, h->device, rec[r].dev) != cudaSuccess || !can)
            ok = 0;
    }
    int32_t all_ok = 0;
    if ((s = allreduce_min_host(h, ok, &all_ok))) return s;
    if (all_ok) {
        const XLayout L = layout_of(h);
        h->peer.assign(h->world, XBufs{});
        int32_t opened = 1;
        for (int r = 0; r < h->world; ++r) {
            if (r == h->rank) {
                h->peer[r] = h->xb;
                continue;
            }
            void* p = nullptr;
            if (cudaIpcOpenMemHandle(&p, rec[r].ipc, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                opened = 0;
                break;
            }
            h->ipc_opened.push_back(p);
            h->peer[r] = view_of(p, L);
        }
        if ((s = allreduce_min_host(h, opened, &all_ok))) return s;
        if (all_ok) {
            h->xmode = kXP2P;
        } else {
            for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
            h->ipc_opened.clear();
            h->peer.clear();
        }
    }
    if (h->xmode != kXP2P && h->opt.exchange == SPMV_EXCHANGE_P2P)
        return fail(SPMV_ERR_UNSUPPORTED, "P2P exchange requested but not available on every rank");
    return make_streams(h);
}

spmv_status_t xchg_loopback_link(spmv_plan_s** hs, int world) {
    if (!stream_memops_available()) return fail(SPMV_ERR_UNSUPPORTED, "stream memory operations unavailable");
    for (int r = 0; r < world; ++r) {
        spmv_plan_s* h = hs[r];
        if (!valid(h) || !h->test_rank || h->world != world || h->rank != r || h->device != hs[0]->device ||
            h->xb.bytes != hs[0]->xb.bytes)
            return fail(SPMV_ERR_USAGE, "loopback_link: handle %d is not test rank %d of world %d", r, r, world);
    }
    // On one GPU every rank's streams share the device's hardware work
    // queues; a stream blocked in a wait on a peer's flag (DB: the fold waits
    // for the peers' temporaries) would also block whatever else sits in its
    // queue -- possibly the very push it waits for.  Streams are assigned to
    // the queues round-robin in creation order, so each rank's comm stream
    // and an apply stream for the test (spmv_test_rank_stream) are created
    // here back to back: with CUDA_DEVICE_MAX_CONNECTIONS >= 2 * world they
    // get queues of their own (on a real multi-GPU run each rank has its own
    // device and no such aliasing exists).
    for (int r = 0; r < world; ++r) {
        spmv_plan_s* h = hs[r];
        DeviceGuard g(h->device);
        h->peer.assign(world, XBufs{});
        for (int q = 0; q < world; ++q) h->peer[q] = hs[q]->xb;
        h->xmode = kXLoopback;
        if (h->comm_stream) {
            cudaStreamDestroy(h->comm_stream);
            h->comm_stream = nullptr;
        }
        if (h->test_stream) {
            cudaStreamDestroy(h->test_stream);
            h->test_stream = nullptr;
        }
        spmv_status_t s = make_streams(h);
        if (s) return s;
        CUDA_TRY(cudaStreamCreateWithFlags(&h->test_stream, cudaStreamNonBlocking));
    }
    return SPMV_OK;
}

spmv_status_t xchg_pre(spmv_plan_s* h, const double* x, cudaStream_t st, XView& v) {
    const int64_t nint = h->x_int_len, len = h->x_bord_len;
    const int me = h->rank;
    v.x_split = (int32_t)nint;
    if (h->xmode == kXNone) return fail(SPMV_ERR_USAGE, "test rank not linked (spmv_test_loopback_link)");
    if (h->xmode == kXNccl) {
        double* xb = h->xb.xb[0];
        if (len) CUDA_TRY(cudaMemcpyAsync(xb + h->bord_off[me], x + nint, len * sizeof(double),
                                          cudaMemcpyDeviceToDevice, st));
        if (h->border_total) {
            // in place: every rank's slice sits at its own offset of C_B;
            // ncclAllGather's in-place form needs bord_off[r] == r * count
            bool inplace = h->equal_slices;
            for (int r = 0; r < h->world && inplace; ++r) inplace = h->bord_off[r] == (int64_t)r * h->bord_cnt[0];
            if (inplace) {
                NCCL_TRY(ncclAllGather(xb + h->bord_off[me], xb, h->bord_cnt[0], ncclFloat64, h->comm, st));
            } else {
                NCCL_TRY(ncclGroupStart());
                for (int r = 0; r < h->world; ++r)
                    if (h->bord_cnt[r])
                        NCCL_TRY(ncclBroadcast(xb + h->bord_off[r], xb + h->bord_off[r], h->bord_cnt[r], ncclFloat64, r,
                                               h->comm, st));
                NCCL_TRY(ncclGroupEnd());
            }
        }
        v.x_hi = xb;
        return SPMV_OK;
    }
    // P2P / loopback
    const int32_t seq = ++h->seq;
    const int par = seq & 1;
    double* xb = h->xb.xb[par];
    if (len) CUDA_TRY(cudaMemcpyAsync(xb + h->bord_off[me], x + nint, len * sizeof(double), cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaEventRecord(h->ev_x, st));
    CUDA_TRY(cudaStreamWaitEvent(h->comm_stream, h->ev_x, 0));
    spmv_status_t s;
    for (int r = 0; r < h->world; ++r) {
        if (r == me) continue;
        // rank r finished reading its parity-`par` buffer (apply seq - 2)
        if ((s = wait_geq(h->comm_stream, h->xb.done + r, seq - 2))) return s;
        if (len)
            CUDA_TRY(cudaMemcpyAsync(h->peer[r].xb[par] + h->bord_off[me], x + nint, len * sizeof(double),
                                     cudaMemcpyDeviceToDevice, h->comm_stream));
        if ((s = write_val(h->comm_stream, h->peer[r].ready + me, seq))) return s;
    }
    CUDA_TRY(cudaEventRecord(h->ev_comm, h->comm_stream));
    v.x_hi = xb;
    v.ready = h->xb.ready;
    v.seq = seq;
    v.err = h->xb.err;
    v.herr = h->xb.herr;
    return SPMV_OK;
}

spmv_status_t xchg_post(spmv_plan_s* h, double* y, unsigned long long* slots, cudaStream_t st) {
    const int me = h->rank;
    const bool db = h->kind == SPMV_DB;
    if (h->xmode == kXNccl) {
        if (!db) return SPMV_OK;
        double* tin = h->xb.tin[0];
        if (h->t_send_cnt[me])
            CUDA_TRY(cudaMemcpyAsync(tin + h->t_recv_off[me], h->d_T + h->t_send_off[me],
                                     h->t_send_cnt[me] * sizeof(double), cudaMemcpyDeviceToDevice, st));
        NCCL_TRY(ncclGroupStart());
        for (int r = 0; r < h->world; ++r) {
            if (r == me) continue;
            if (h->t_send_cnt[r]) NCCL_TRY(ncclSend(h->d_T + h->t_send_off[r], h->t_send_cnt[r], ncclFloat64, r, h->comm, st));
            if (h->t_recv_cnt[r]) NCCL_TRY(ncclRecv(tin + h->t_recv_off[r], h->t_recv_cnt[r], ncclFloat64, r, h->comm, st));
        }
        NCCL_TRY(ncclGroupEnd());
        CUDA_TRY(launch_fold(tin, h->d_fold_ptr, h->d_fold_pos, y + h->m_blk, h->y_bord_len, FoldWait{}, slots, st));
        return SPMV_OK;
    }
    const int32_t seq = h->seq;
    const int par = seq & 1;
    spmv_status_t s;
    // this rank finished reading its parity-`par` border buffer
    for (int r = 0; r < h->world; ++r)
        if (r != me && (s = write_val(st, h->peer[r].done + me, seq))) return s;
    if (db) {
        double* tin = h->xb.tin[par];
        if (h->t_send_cnt[me])
            CUDA_TRY(cudaMemcpyAsync(tin + h->t_recv_off[me], h->d_T + h->t_send_off[me],
                                     h->t_send_cnt[me] * sizeof(double), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(cudaEventRecord(h->ev_kernel, st));
        CUDA_TRY(cudaStreamWaitEvent(h->comm_stream, h->ev_kernel, 0));
        for (int r = 0; r < h->world; ++r) {
            if (r == me) continue;
            if ((s = wait_geq(h->comm_stream, h->xb.tdone + r, seq - 2))) return s;
            if (h->t_send_cnt[r])
                CUDA_TRY(cudaMemcpyAsync(h->peer[r].tin[par] + h->t_dst_off[r], h->d_T + h->t_send_off[r],
                                         h->t_send_cnt[r] * sizeof(double), cudaMemcpyDeviceToDevice, h->comm_stream));
            if ((s = write_val(h->comm_stream, h->peer[r].tready + me, seq))) return s;
        }
        CUDA_TRY(cudaEventRecord(h->ev_comm, h->comm_stream));
        // the fold kernel waits for the peers' tready flags on the device
        FoldWait fw;
        fw.ready = h->xb.tready;
        fw.world = h->world;
        fw.self = me;
        fw.seq = seq;
        fw.err = h->xb.err;
        fw.herr = h->xb.herr;
        CUDA_TRY(launch_fold(tin, h->d_fold_ptr, h->d_fold_pos, y + h->m_blk, h->y_bord_len, fw, slots, st));
        for (int r = 0; r < h->world; ++r)
            if (r != me && (s = write_val(st, h->peer[r].tdone + me, seq))) return s;
    }
    // the apply completes on `st` only after this rank's pushes (they read x and d_T)
    CUDA_TRY(cudaStreamWaitEvent(st, h->ev_comm, 0));
    return SPMV_OK;
}

spmv_status_t xchg_allreduce_max(spmv_plan_s* h, double* m_dev, cudaStream_t st) {
    if (h->comm) NCCL_TRY(ncclAllReduce(m_dev, m_dev, 1, ncclFloat64, ncclMax, h->comm, st));
    return SPMV_OK;   // test ranks: the rank's own max (the test folds the ranks' maxima)
}

int64_t xchg_timeouts(spmv_plan_s* h) {
    if (!h->xb.err) return 0;
    DeviceGuard g(h->device);
    int32_t v = 0;
    if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpy(&v, h->xb.err, sizeof v, cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return v;
}

void xchg_release(spmv_plan_s* h) {
    if (h->xb.herr_host) cudaFreeHost(h->xb.herr_host);
    h->xb.herr_host = h->xb.herr = nullptr;
    for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
    h->ipc_opened.clear();
    if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
    if (h->test_stream) cudaStreamDestroy(h->test_stream);
    h->test_stream = nullptr;
    if (h->ev_x) cudaEventDestroy(h->ev_x);
    if (h->ev_comm) cudaEventDestroy(h->ev_comm);
    if (h->ev_kernel) cudaEventDestroy(h->ev_kernel);
    h->comm_stream = nullptr;
    h->ev_x = h->ev_comm = h->ev_kernel = nullptr;
}

}  // namespace spmvb
