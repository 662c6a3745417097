// order.cu -- producing the reordering instead of receiving it (SURVEY 8(f)
// f4): the sBFS ordering of P:L134 (section 5.1: "we apply BFS on the
// bipartite graph representation of the matrix, so that the resulting BFS
// orders on the row and column vertices determine row and column
// reorderings") on the GPU, then the extraction of a K-way SB form (Eq.(1),
// P:L65-71) from it, so the result feeds spmv_create directly.
//
// What is computed (reading R5; the oracle's oracle_sbfs is the
// same definition written as a serial queue BFS):
//   * BFS on the bipartite graph (row vertices, column vertices, an edge per
//     stored entry); the root is the lowest-numbered unvisited row; a popped
//     vertex appends its unvisited neighbours in ascending number; the next
//     root when the queue empties is again the lowest unvisited row; columns
//     no row touches come last, ascending.  Rows and columns are numbered in
//     visiting order.
//   * SB extraction: new row r joins block min(K-1, floor(K P(r) / nnz)),
//     P(r) = entries of the rows numbered below r; a column whose rows all lie
//     in block k is interior to block k, every other column is a border
//     column; columns are numbered block by block, C_B last, each group in
//     BFS column order.
//
// GPU form of the queue BFS (level-synchronous, deterministic): the queue
// order inside a level is (position of the first frontier vertex adjacent to
// v, v) -- a popped vertex appends its neighbours in ascending number, and
// the earliest-popped neighbour wins.  Each level: one warp per frontier
// vertex scans its adjacency; an unvisited neighbour takes the atomic minimum
// of the parent positions; first touches are collected (atomic append, order
// irrelevant), then sorted by the 64-bit key (parent position, id) and
// numbered.  The column->row adjacency (CSC) is built on the device by a
// counting pass; its order within a column does not matter (minima).  Sorts
// and scans are CUB library primitives; the BFS, CSC and extraction kernels
// are this file's.
#include <cstdint>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "handle.h"

namespace spmvb {
namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;

__global__ void col_count_kernel(const int32_t* __restrict__ col, int64_t nnz, unsigned long long* __restrict__ cnt) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + col[t], 1ull);
}

// one warp per row: its entries' row id into the CSC
__global__ void csc_fill_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t m,
                                unsigned long long* __restrict__ fill, int32_t* __restrict__ cadj) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < m;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5)
        for (int64_t t = rp[i] + lane; t < rp[i + 1]; t += 32) {
            const unsigned long long p = atomicAdd(fill + col[t], 1ull);
            cadj[p] = (int32_t)i;
        }
}

// One BFS level: frontier vertices (side A) in queue order; their unvisited
// neighbours (side B) take the minimum frontier position; first touches are
// appended to `next`.
__global__ void expand_kernel(const int32_t* __restrict__ front, int64_t nf, const int64_t* __restrict__ ptr,
                              const int32_t* __restrict__ adj, const int32_t* __restrict__ num_b,
                              uint32_t* __restrict__ cand, int32_t* __restrict__ next, unsigned long long* nnext) {
    const int lane = threadIdx.x & 31;
    for (int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; p < nf;
         p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t u = front[p];
        for (int64_t t = ptr[u] + lane; t < ptr[u + 1]; t += 32) {
            const int32_t v = adj[t];
            if (num_b[v] >= 0) continue;
            if (cand[v] <= (uint32_t)p) continue;   // already claimed by an earlier parent
            const uint32_t old = atomicMin(cand + v, (uint32_t)p);
            if (old == kNone) next[atomicAdd(nnext, 1ull)] = v;
        }
    }
}

__global__ void make_keys_kernel(const int32_t* __restrict__ next, int64_t nn, const uint32_t* __restrict__ cand,
                                 unsigned long long* __restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = next[i];
        keys[i] = ((unsigned long long)cand[v] << 32) | (uint32_t)v;
    }
}

__global__ void number_kernel(const unsigned long long* __restrict__ keys, int64_t nn, int64_t base,
                              int32_t* __restrict__ num, int32_t* __restrict__ front) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = (int32_t)(keys[i] & 0xFFFFFFFFull);
        num[v] = (int32_t)(base + i);
        front[i] = v;
    }
}

// lowest row in [a, b) that is unvisited and has entries (atomicMin)
__global__ void find_root_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ num, int64_t a, int64_t b,
                                 unsigned long long* out) {
    for (int64_t i = a + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x)
        if (num[i] < 0 && rp[i + 1] > rp[i]) atomicMin(out, (unsigned long long)i);
}

// rows of [a, b) without entries (never reached by the BFS: each is a root of
// its own) numbered base + (empty rows below it in [a, b)) -- ascending
__global__ void number_empty_kernel(const int64_t* __restrict__ empty_before, int32_t* __restrict__ num,
                                    const int64_t* __restrict__ rp, int64_t a, int64_t b, int64_t base) {
    for (int64_t i = a + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x)
        if (rp[i + 1] == rp[i]) num[i] = (int32_t)(base + empty_before[i] - empty_before[a]);
}

__global__ void empty_flag_kernel(const int64_t* __restrict__ rp, int64_t m, int64_t* __restrict__ f) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        f[i] = rp[i + 1] == rp[i] ? 1 : 0;
}

__global__ void unvisited_flag_kernel(const int32_t* __restrict__ num, int64_t n, int64_t* __restrict__ f) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        f[i] = num[i] < 0 ? 1 : 0;
}

__global__ void number_unvisited_kernel(const int64_t* __restrict__ before, int32_t* __restrict__ num, int64_t n,
                                        int64_t base) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (num[i] < 0) num[i] = (int32_t)(base + before[i]);
}

// ---- SB extraction
__global__ void new_len_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ rnum, int64_t m,
                               int64_t* __restrict__ len_new) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        len_new[rnum[i]] = rp[i + 1] - rp[i];
}

// block of new row r from the entries before it (exclusive prefix P)
__global__ void block_kernel(const int64_t* __restrict__ P, int64_t m, int64_t nnz, int32_t K, int32_t* __restrict__ blk) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t b;
        if (nnz > 0) b = (int64_t)(((unsigned __int128)K * (unsigned __int128)P[r]) / (unsigned __int128)nnz);
        else b = ((int64_t)K * r) / m;
        blk[r] = (int32_t)(b < K - 1 ? b : K - 1);
    }
}

// row_block_ptr[k] = first new row whose block is >= k (blk is nondecreasing)
__global__ void block_ptr_kernel(const int32_t* __restrict__ blk, int64_t m, int32_t K, int64_t* __restrict__ rbp) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k > K + 1) return;
    if (k == 0) { rbp[0] = 0; return; }
    if (k >= K) { rbp[k] = m; return; }
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (blk[mid] >= k) hi = mid;
        else lo = mid + 1;
    }
    rbp[k] = lo;
}

// class of every column: -1 untouched, k one block, K two or more blocks
__global__ void col_class_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                 const int32_t* __restrict__ rnum, const int32_t* __restrict__ blk, int64_t m, int32_t K,
                                 int32_t* __restrict__ cls) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < m;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int32_t b = blk[rnum[i]];
        for (int64_t t = rp[i] + lane; t < rp[i + 1]; t += 32) {
            const int32_t j = col[t];
            const int32_t c = cls[j];
            if (c == b || c == K) continue;
            const int32_t old = atomicCAS(cls + j, -1, b);
            if (old != -1 && old != b) cls[j] = K;
        }
    }
}

// sort key of column j: (class, BFS number); untouched columns are border
__global__ void col_keys_kernel(const int32_t* __restrict__ cls, const int32_t* __restrict__ cnum, int64_t n, int32_t K,
                                unsigned long long* __restrict__ keys, int32_t* __restrict__ ids) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = cls[j] < 0 ? K : cls[j];
        keys[j] = ((unsigned long long)(uint32_t)c << 32) | (uint32_t)cnum[j];
        ids[j] = (int32_t)j;
    }
}

__global__ void col_perm_kernel(const int32_t* __restrict__ ids_sorted, int64_t n, int32_t* __restrict__ col_perm) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
        col_perm[ids_sorted[q]] = (int32_t)q;
}

// col_block_ptr[k] = first sorted column whose class is >= k
__global__ void col_block_ptr_kernel(const unsigned long long* __restrict__ keys, int64_t n, int32_t K,
                                     int64_t* __restrict__ cbp) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k > K + 1) return;
    if (k == K + 1) { cbp[k] = n; return; }
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)(keys[mid] >> 32) >= k) hi = mid;
        else lo = mid + 1;
    }
    cbp[k] = lo;
}

int grid_for(int64_t work, int threads) {
    const int64_t g = (work + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

// device buffers of one ordering call, freed on every exit path
struct Buf {
    std::vector<void*> p;
    template <typename T>
    cudaError_t get(T** out, size_t count) {
        void* q = nullptr;
        const cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
        if (e == cudaSuccess) p.push_back(q);
        *out = static_cast<T*>(q);
        return e;
    }
    ~Buf() {
        for (void* q : p) cudaFree(q);
    }
};

#define OTRY(expr)                                                                                 \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess) return fail(SPMV_ERR_INTERNAL, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

// exclusive prefix sum of int64 (CUB), with a temporary of its own
cudaError_t exclusive_sum(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    size_t tb = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s);
    if (e != cudaSuccess) return e;
    void* t = nullptr;
    if ((e = cudaMalloc(&t, std::max<size_t>(tb, 1))) != cudaSuccess) return e;
    e = cub::DeviceScan::ExclusiveSum(t, tb, in, out, n, s);
    cudaFree(t);
    return e;
}

cudaError_t sort_keys(unsigned long long* keys, unsigned long long* tmp_keys, int64_t n, cudaStream_t s,
                      int32_t** ids = nullptr, int32_t* ids_out = nullptr) {
    size_t tb = 0;
    cudaError_t e;
    if (ids) e = cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, tmp_keys, *ids, ids_out, n, 0, 64, s);
    else e = cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, tmp_keys, n, 0, 64, s);
    if (e != cudaSuccess) return e;
    void* t = nullptr;
    if ((e = cudaMalloc(&t, std::max<size_t>(tb, 1))) != cudaSuccess) return e;
    if (ids) e = cub::DeviceRadixSort::SortPairs(t, tb, keys, tmp_keys, *ids, ids_out, n, 0, 64, s);
    else e = cub::DeviceRadixSort::SortKeys(t, tb, keys, tmp_keys, n, 0, 64, s);
    cudaFree(t);
    return e;
}

spmv_status_t order_impl(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx, int32_t K,
                         int32_t* row_perm, int32_t* col_perm, int64_t* row_block_ptr, int64_t* col_block_ptr,
                         spmv_order_info_t* info) {
    cudaStream_t s = 0;
    Buf B;
    int64_t *rp, *cptr;
    int32_t *col, *cadj, *rnum, *cnum, *fa, *fb;
    uint32_t *rcand, *ccand;
    unsigned long long *ucnt, *keys, *keys2, *dcount;
    OTRY(B.get(&rp, m + 1));
    OTRY(B.get(&col, nnz));
    OTRY(B.get(&cptr, n + 1));
    OTRY(B.get(&cadj, nnz));
    OTRY(B.get(&ucnt, n + 1));
    OTRY(B.get(&rnum, m));
    OTRY(B.get(&cnum, n));
    OTRY(B.get(&rcand, m));
    OTRY(B.get(&ccand, n));
    const int64_t mx = std::max(m, n);
    OTRY(B.get(&fa, mx));
    OTRY(B.get(&fb, mx));
    OTRY(B.get(&keys, mx));
    OTRY(B.get(&keys2, mx));
    OTRY(B.get(&dcount, 2));
    unsigned long long* hcount = nullptr;
    OTRY(cudaMallocHost(&hcount, 2 * sizeof(unsigned long long)));
    struct HostFree {
        void* p;
        ~HostFree() { cudaFreeHost(p); }
    } hf{hcount};
    cudaEvent_t e0, e1, e2;
    OTRY(cudaEventCreate(&e0));
    OTRY(cudaEventCreate(&e1));
    OTRY(cudaEventCreate(&e2));
    struct EvFree {
        cudaEvent_t a, b, c;
        ~EvFree() { cudaEventDestroy(a); cudaEventDestroy(b); cudaEventDestroy(c); }
    } ef{e0, e1, e2};

    OTRY(cudaMemcpy(rp, row_ptr, (m + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    if (nnz) OTRY(cudaMemcpy(col, col_idx, nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
    OTRY(cudaEventRecord(e0, s));
    // CSC (column -> rows)
    OTRY(cudaMemsetAsync(ucnt, 0, (n + 1) * sizeof(unsigned long long), s));
    if (nnz) col_count_kernel<<<grid_for(nnz, 256), 256, 0, s>>>(col, nnz, ucnt);
    OTRY(cudaGetLastError());
    OTRY(exclusive_sum(reinterpret_cast<const int64_t*>(ucnt), cptr, n + 1, s));
    OTRY(cudaMemcpyAsync(ucnt, cptr, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    if (nnz) csc_fill_kernel<<<grid_for(m * 32, 256), 256, 0, s>>>(rp, col, m, ucnt, cadj);
    OTRY(cudaGetLastError());
    OTRY(cudaMemsetAsync(rnum, 0xFF, m * sizeof(int32_t), s));
    OTRY(cudaMemsetAsync(cnum, 0xFF, n * sizeof(int32_t), s));
    OTRY(cudaMemsetAsync(rcand, 0xFF, m * sizeof(uint32_t), s));
    OTRY(cudaMemsetAsync(ccand, 0xFF, n * sizeof(uint32_t), s));
    // empty rows: prefix counts (they are numbered as roots, never reached)
    int64_t *eflag, *ebefore;
    OTRY(B.get(&eflag, m + 1));
    OTRY(B.get(&ebefore, m + 1));
    if (m) empty_flag_kernel<<<grid_for(m, 256), 256, 0, s>>>(rp, m, eflag);
    OTRY(cudaMemsetAsync(eflag + m, 0, sizeof(int64_t), s));
    OTRY(exclusive_sum(eflag, ebefore, m + 1, s));

    int64_t nr = 0, nc = 0, next_root = 0, levels = 0, comps = 0;
    while (nr < m) {
        // the lowest unvisited row with entries at or above next_root; the
        // empty rows below it are roots of their own, numbered first
        int64_t root = m;
        for (int64_t a = next_root, chunk = 1 << 16; a < m; a += chunk, chunk *= 2) {
            const int64_t b = std::min(m, a + chunk);
            OTRY(cudaMemsetAsync(dcount, 0xFF, sizeof(unsigned long long), s));
            find_root_kernel<<<grid_for(b - a, 256), 256, 0, s>>>(rp, rnum, a, b, dcount);
            OTRY(cudaMemcpyAsync(hcount, dcount, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
            OTRY(cudaStreamSynchronize(s));
            if (hcount[0] != ~0ull) {
                root = (int64_t)hcount[0];
                break;
            }
        }
        int64_t ebuf[2] = {0, 0};
        OTRY(cudaMemcpy(&ebuf[0], ebefore + next_root, sizeof(int64_t), cudaMemcpyDeviceToHost));
        OTRY(cudaMemcpy(&ebuf[1], ebefore + root, sizeof(int64_t), cudaMemcpyDeviceToHost));
        if (ebuf[1] > ebuf[0]) {
            number_empty_kernel<<<grid_for(root - next_root, 256), 256, 0, s>>>(ebefore, rnum, rp, next_root, root, nr);
            OTRY(cudaGetLastError());
            nr += ebuf[1] - ebuf[0];
        }
        next_root = root;
        if (root >= m) break;
        // BFS from root: level by level, rows and columns alternating
        const int32_t r32 = (int32_t)root;
        OTRY(cudaMemcpyAsync(fa, &r32, sizeof(int32_t), cudaMemcpyHostToDevice, s));
        OTRY(cudaMemcpyAsync(rnum + root, &nr, sizeof(int32_t), cudaMemcpyHostToDevice, s));   // little endian
        ++nr;
        ++comps;
        int64_t nf = 1;
        bool rows_side = true;   // the frontier holds rows
        while (nf > 0) {
            OTRY(cudaMemsetAsync(dcount, 0, sizeof(unsigned long long), s));
            if (rows_side) expand_kernel<<<grid_for(nf * 32, 256), 256, 0, s>>>(fa, nf, rp, col, cnum, ccand, fb, dcount);
            else expand_kernel<<<grid_for(nf * 32, 256), 256, 0, s>>>(fa, nf, cptr, cadj, rnum, rcand, fb, dcount);
            OTRY(cudaGetLastError());
            OTRY(cudaMemcpyAsync(hcount, dcount, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
            OTRY(cudaStreamSynchronize(s));
            const int64_t nn = (int64_t)hcount[0];
            ++levels;
            if (nn > 0) {
                make_keys_kernel<<<grid_for(nn, 256), 256, 0, s>>>(fb, nn, rows_side ? ccand : rcand, keys);
                OTRY(cudaGetLastError());
                OTRY(sort_keys(keys, keys2, nn, s));
                number_kernel<<<grid_for(nn, 256), 256, 0, s>>>(keys2, nn, rows_side ? nc : nr, rows_side ? cnum : rnum, fa);
                OTRY(cudaGetLastError());
                if (rows_side) nc += nn;
                else nr += nn;
            }
            nf = nn;
            rows_side = !rows_side;
        }
        ++next_root;
    }
    // columns no row touches: after the visited ones, ascending
    if (nc < n) {
        int64_t *uf, *ub;
        OTRY(B.get(&uf, n));
        OTRY(B.get(&ub, n));
        unvisited_flag_kernel<<<grid_for(n, 256), 256, 0, s>>>(cnum, n, uf);
        OTRY(exclusive_sum(uf, ub, n, s));
        number_unvisited_kernel<<<grid_for(n, 256), 256, 0, s>>>(ub, cnum, n, nc);
        OTRY(cudaGetLastError());
    }
    OTRY(cudaEventRecord(e1, s));
    // ---- SB extraction
    int64_t *len_new, *P, *drbp, *dcbp;
    int32_t *blk, *cls, *ids, *ids2;
    OTRY(B.get(&len_new, m));
    OTRY(B.get(&P, m));
    OTRY(B.get(&blk, m));
    OTRY(B.get(&drbp, K + 2));
    OTRY(B.get(&dcbp, K + 2));
    OTRY(B.get(&cls, n));
    OTRY(B.get(&ids, n));
    OTRY(B.get(&ids2, n));
    if (m) {
        new_len_kernel<<<grid_for(m, 256), 256, 0, s>>>(rp, rnum, m, len_new);
        OTRY(exclusive_sum(len_new, P, m, s));
        block_kernel<<<grid_for(m, 256), 256, 0, s>>>(P, m, nnz, K, blk);
    }
    block_ptr_kernel<<<(K + 2 + 127) / 128, 128, 0, s>>>(blk, m, K, drbp);
    OTRY(cudaMemsetAsync(cls, 0xFF, n * sizeof(int32_t), s));
    if (nnz) col_class_kernel<<<grid_for(m * 32, 256), 256, 0, s>>>(rp, col, rnum, blk, m, K, cls);
    if (n) {
        col_keys_kernel<<<grid_for(n, 256), 256, 0, s>>>(cls, cnum, n, K, keys, ids);
        OTRY(sort_keys(keys, keys2, n, s, &ids, ids2));
        col_perm_kernel<<<grid_for(n, 256), 256, 0, s>>>(ids2, n, ids);   // ids now holds col_perm
    }
    col_block_ptr_kernel<<<(K + 2 + 127) / 128, 128, 0, s>>>(keys2, n, K, dcbp);
    OTRY(cudaGetLastError());
    OTRY(cudaEventRecord(e2, s));
    OTRY(cudaMemcpyAsync(row_perm, rnum, m * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    OTRY(cudaMemcpyAsync(col_perm, ids, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    OTRY(cudaMemcpyAsync(row_block_ptr, drbp, (K + 2) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    OTRY(cudaMemcpyAsync(col_block_ptr, dcbp, (K + 2) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    OTRY(cudaStreamSynchronize(s));
    if (info) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, e0, e1);
        cudaEventElapsedTime(&b, e1, e2);
        info->bfs_ms = a;
        info->extract_ms = b;
        info->levels = levels;
        info->components = comps;
        info->border_cols = n - col_block_ptr[K];
    }
    return SPMV_OK;
}

}  // namespace
}  // namespace spmvb

extern "C" spmv_status_t spmv_order_sbfs(int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                                         const int32_t* col_idx, int32_t K, int32_t* row_perm, int32_t* col_perm,
                                         int64_t* row_block_ptr, int64_t* col_block_ptr, spmv_order_info_t* info) {
    using namespace spmvb;
    if (m < 0 || n < 0 || nnz < 0 || K < 1 || !row_ptr || (nnz && !col_idx) || (m && !row_perm) || (n && !col_perm) ||
        !row_block_ptr || !col_block_ptr)
        return fail(SPMV_ERR_USAGE, "spmv_order_sbfs: bad arguments");
    if (m > INT32_MAX || n > INT32_MAX) return fail(SPMV_ERR_UNSUPPORTED, "spmv_order_sbfs: m or n beyond int32");
    if (row_ptr[0] != 0 || row_ptr[m] != nnz) return fail(SPMV_ERR_DATA, "spmv_order_sbfs: bad row_ptr");
    for (int64_t i = 0; i < m; ++i)
        if (row_ptr[i + 1] < row_ptr[i]) return fail(SPMV_ERR_DATA, "spmv_order_sbfs: row_ptr not nondecreasing");
    for (int64_t t = 0; t < nnz; ++t)
        if (col_idx[t] < 0 || (int64_t)col_idx[t] >= n) return fail(SPMV_ERR_DATA, "spmv_order_sbfs: column out of range");
    if (info) std::memset(info, 0, sizeof *info);
    return order_impl(m, n, nnz, row_ptr, col_idx, K, row_perm, col_perm, row_block_ptr, col_block_ptr, info);
}
