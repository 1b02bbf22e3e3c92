// pms8g_kernels.cu — sm_100a kernels of the B200-native PMS8 per-S1-l-mer search.
//
//   K1 encode_kernel     every l-mer of the n sequences -> two bit planes
//                        (replaces PackedSequenceSet, src/packed_seq.cpp:30-81)
//   K2 rowbuild_kernel   per S1 l-mer (anchor): rows of l-mers within 2d, compacted
//                        with warp ballot/popc, rows ordered by size
//                        (replaces PairCompatibilityMatrix src/solver.cpp:25-63 +
//                        the anchor push of run_anchored src/solver.cpp:427-432)
//   K3 taskscan_kernel   exclusive scan of per-anchor task counts (work queue)
//   K4 search_kernel     persistent: one warp = one DFS worker pulling (S1 l-mer,
//                        depth-1 branch) tasks off a global atomic counter; push
//                        filter with the pair + Theorem-1 triple conditions
//                        (MotifSearch::push src/solver.cpp:245-337, recurse :406-419),
//                        common d-neighbourhood enumeration (NeighborhoodEnumerator
//                        src/neighborhood.cpp:164-270, neighborhood.hpp:63-88) and
//                        warp-parallel verification (verify_candidate :344-362)
//   K5 (host, CUB)       device radix sort + unique of packed motif keys
//                        (canonical_motif_set src/solver.cpp:16-21)
//
// All work is integer/bitwise: Hamming distance of two l-mers is
// popc((a.h ^ b.h) | (a.o ^ b.o)) per 32 symbols (1 LOP3-pair + POPC).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "pms8g_device.cuh"
#include "pms8g_common.cuh"
#include "pms8g_launch.h"

namespace pms8g {

using namespace dev;

// ---------------------------------------------------------------------------
// K1: encode
template <int W>
__global__ void encode_kernel(const uint8_t* __restrict__ codes, int n, int m, int l, int w,
                              Lmer<W>* __restrict__ table, int* error_flag) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n * w) return;
    const int r = id / w, off = id - r * w;
    const uint8_t* s = codes + static_cast<size_t>(r) * m + off;
    Lmer<W> x;
#pragma unroll
    for (int i = 0; i < W; ++i) x.h[i] = x.o[i] = 0;
    bool bad = false;
    for (int p = 0; p < l; ++p) {
        const int c = s[p];
        bad |= c > 3;
        set_code<W>(x, p, c & 3);
    }
    if (bad) atomicOr(error_flag, 1);
    table[id] = x;
}

// ---------------------------------------------------------------------------
// K2: row build. One block per anchor (S1 l-mer); warps stride over rows 1..n-1.
// Pass 1 counts survivors (Hd <= 2d) per row, rows are then ordered by size
// (stable, as RowMatrix::sort_rows_by_size src/solver.cpp:205-217), pass 2
// recomputes and writes the compacted entries in that order.
template <int W>
__global__ void rowbuild_kernel(const Lmer<W>* __restrict__ table, int n, int w, int d, int K, int sort_rows,
                                const int32_t* __restrict__ anchor_off, int nanchors,
                                uint32_t* __restrict__ l1_entries, LevelMeta* __restrict__ l1_meta,
                                unsigned long long* counters) {
    __shared__ int cnt[MAXN];
    __shared__ int startp[MAXN];
    __shared__ int posof[MAXN];
    const int ai = blockIdx.x;
    if (ai >= nanchors) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const Lmer<W> A = table[anchor_off[ai]];
    const int cap = 2 * d;
    for (int r = 1 + warp; r < n; r += nw) {
        int c = 0;
        for (int base = 0; base < w; base += 32) {
            const int o = base + lane;
            const bool ok = o < w && dist<W>(A, table[r * w + o]) <= cap;
            c += __popc(__ballot_sync(0xffffffffu, ok));
        }
        if (lane == 0) cnt[r] = c;
    }
    __syncthreads();
    const int nrows = n - 1;
    if (warp == 0) {
        // physical order: ascending count, ties by row index (stable)
        const int r = lane + 1;
        int rank = lane;
        int c = 0;
        if (lane < nrows) {
            c = cnt[r];
            if (sort_rows) {
                rank = 0;
                for (int q = 1; q < n; ++q) {
                    const int cq = cnt[q];
                    rank += (cq < c) || (cq == c && q < r);
                }
            }
            posof[r] = rank;
        }
        __syncwarp();
        // exclusive scan over positions
        int cpos = 0;
        if (lane < nrows) {
            for (int q = 1; q < n; ++q)
                if (posof[q] == lane) cpos = cnt[q];
        }
        int incl = cpos;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, s);
            if (lane >= s) incl += v;
        }
        const int excl = incl - cpos;
        if (lane < nrows) startp[lane] = excl;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        const bool empty = lane < nrows && cpos == 0;
        const bool any_empty = __any_sync(0xffffffffu, empty);
        LevelMeta* M = l1_meta + ai;
        if (lane < nrows) {
            M->start[lane] = static_cast<uint32_t>(excl);
            M->cnt[lane] = static_cast<uint32_t>(cpos);
            int row = 0;
            for (int q = 1; q < n; ++q)
                if (posof[q] == lane) row = q;
            M->order[lane] = static_cast<uint8_t>(row);
        }
        if (lane == 0) {
            M->nrows = nrows;
            M->total = total;
            M->branch = 0;
            M->viable = any_empty ? 0 : 1;
            atomicAdd(counters + C_SLOTS, static_cast<unsigned long long>(nrows) * w);
            atomicAdd(counters + C_PUSHES, 1ull);
            if (!any_empty) atomicAdd(counters + C_VIABLE, 1ull);
        }
    }
    __syncthreads();
    uint32_t* out = l1_entries + static_cast<size_t>(ai) * K;
    for (int r = 1 + warp; r < n; r += nw) {
        int dst = startp[posof[r]];
        for (int base = 0; base < w; base += 32) {
            const int o = base + lane;
            const bool ok = o < w && dist<W>(A, table[r * w + o]) <= cap;
            const unsigned bal = __ballot_sync(0xffffffffu, ok);
            if (ok) out[dst + __popc(bal & lanemask_lt())] = (static_cast<uint32_t>(r) << 24) | (r * w + o);
            dst += __popc(bal);
        }
    }
}

// ---------------------------------------------------------------------------
// K3: task scan (one warp). tasks(a) = cnt[branch] (t >= 2) or 1 (t == 1).
__global__ void taskscan_kernel(const LevelMeta* __restrict__ l1_meta, int nanchors, int t, long long* task_base) {
    const int lane = threadIdx.x & 31;
    long long carry = 0;
    for (int base = 0; base < nanchors; base += 32) {
        const int a = base + lane;
        long long c = 0;
        if (a < nanchors) {
            const LevelMeta& M = l1_meta[a];
            if (M.viable) c = (t == 1) ? 1 : M.cnt[M.branch];
        }
        long long incl = c;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const long long v = __shfl_up_sync(0xffffffffu, incl, s);
            if (lane >= s) incl += v;
        }
        if (a < nanchors) task_base[a] = carry + incl - c;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) task_base[nanchors] = carry;
}

// ---------------------------------------------------------------------------
// Static task order (heaviest first): task idx = (anchor a, depth-1 branch j)
// gets the key dist(anchor, u_j). Closer pairs have far more compatible
// l-mers below them, so sorting by the key front-loads the long tasks and
// leaves the short ones for the end of the queue (less tail for the
// dynamic donation to absorb). Slots past the task count sort last.
template <int W>
__global__ void taskorder_kernel(const Lmer<W>* __restrict__ table, const uint32_t* __restrict__ l1_entries,
                                 const LevelMeta* __restrict__ l1_meta, const int32_t* __restrict__ anchor_off,
                                 const long long* __restrict__ task_base, int nanchors, int K, long long cap,
                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const long long nstatic = task_base[nanchors];
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cap;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        uint32_t key = 0xFFFFFFFFu;
        if (i < nstatic) {
            int lo = 0, hi = nanchors - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (task_base[mid] <= i) lo = mid;
                else hi = mid - 1;
            }
            const LevelMeta& M = l1_meta[lo];
            const int j = static_cast<int>(i - task_base[lo]);
            const uint32_t u = l1_entries[static_cast<size_t>(lo) * K + M.start[M.branch] + j] & ID_MASK;
            const Lmer<W> A = table[anchor_off[lo]], U = table[u];
            int dd = 0;
#pragma unroll
            for (int x = 0; x < W; ++x) dd += __popc((A.h[x] ^ U.h[x]) | (A.o[x] ^ U.o[x]));
            key = static_cast<uint32_t>(dd);
        }
        keys[i] = key;
        vals[i] = static_cast<uint32_t>(i);
    }
}

cudaError_t launch_taskorder(int W, const void* table, const uint32_t* l1_entries, const LevelMeta* l1_meta,
                             const int32_t* anchor_off, const long long* task_base, int nanchors, int K,
                             long long cap, uint32_t* keys, uint32_t* vals, cudaStream_t s) {
    const int blocks = static_cast<int>(std::min<long long>((cap + 255) / 256, 4096));
    if (W == 1)
        taskorder_kernel<1><<<blocks, 256, 0, s>>>(static_cast<const Lmer<1>*>(table), l1_entries, l1_meta,
                                                   anchor_off, task_base, nanchors, K, cap, keys, vals);
    else
        taskorder_kernel<2><<<blocks, 256, 0, s>>>(static_cast<const Lmer<2>*>(table), l1_entries, l1_meta,
                                                   anchor_off, task_base, nanchors, K, cap, keys, vals);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Re-verification of final motifs against every window of every sequence
// (SolverConfig::reverify_against_originals, src/solver.cpp:367-379).
template <int W>
__global__ void reverify_kernel(const Lmer<W>* __restrict__ table, int n, int w, int l, int d,
                                const unsigned long long* __restrict__ keys, long long count, int* fail) {
    const long long i = static_cast<long long>(blockIdx.x);
    if (i >= count) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __shared__ int ok_rows;
    if (threadIdx.x == 0) ok_rows = 0;
    __syncthreads();
    Lmer<W> c;
#pragma unroll
    for (int x = 0; x < W; ++x) c.h[x] = c.o[x] = 0;
    const unsigned long long klo = keys[2 * i], khi = keys[2 * i + 1];
    for (int p = 0; p < l; ++p) {
        const int sh = 2 * (l - 1 - p);
        const int code = static_cast<int>(((sh >= 64) ? (khi >> (sh - 64)) : (klo >> sh)) & 3ull);
        set_code<W>(c, p, code);
    }
    for (int r = warp; r < n; r += nw) {
        bool hit = false;
        for (int base = 0; base < w && !hit; base += 32) {
            const int o = base + lane;
            const bool h = o < w && dist<W>(c, table[r * w + o]) <= d;
            hit = __any_sync(0xffffffffu, h);
        }
        if (hit && lane == 0) atomicAdd(&ok_rows, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0 && ok_rows != n) atomicOr(fail, 1);
}

// ---------------------------------------------------------------------------
// Integer-pipe peak microbenchmark: 8 independent LOP3 chains per thread.
__global__ void intpeak_lop3_kernel(uint32_t seed, int iters, uint32_t* sink) {
    uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, a4 = a0 * 11u, a5 = a0 * 13u,
             a6 = a0 * 17u, a7 = a0 * 19u;
    const uint32_t b = seed * 0x9E3779B9u, c = seed ^ 0x85EBCA6Bu;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a0) : "r"(b), "r"(c));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a1) : "r"(b), "r"(c));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a2) : "r"(b), "r"(c));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a3) : "r"(b), "r"(c));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a4) : "r"(b), "r"(c));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a5) : "r"(b), "r"(c));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a6) : "r"(b), "r"(c));
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a7) : "r"(b), "r"(c));
        }
    }
    const uint32_t r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
    if (r == 0x12345678u) sink[0] = r;
}

__global__ void intpeak_popc_kernel(uint32_t seed, int iters, uint32_t* sink) {
    uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, a4 = a0 * 11u, a5 = a0 * 13u,
             a6 = a0 * 17u, a7 = a0 * 19u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            asm volatile("popc.b32 %0, %0;" : "+r"(a0));
            asm volatile("popc.b32 %0, %0;" : "+r"(a1));
            asm volatile("popc.b32 %0, %0;" : "+r"(a2));
            asm volatile("popc.b32 %0, %0;" : "+r"(a3));
            asm volatile("popc.b32 %0, %0;" : "+r"(a4));
            asm volatile("popc.b32 %0, %0;" : "+r"(a5));
            asm volatile("popc.b32 %0, %0;" : "+r"(a6));
            asm volatile("popc.b32 %0, %0;" : "+r"(a7));
        }
    }
    const uint32_t r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
    if (r == 0x12345678u) sink[0] = r;
}

// ---------------------------------------------------------------------------
// host-side launchers

size_t lmer_bytes(int W) { return W == 1 ? sizeof(Lmer<1>) : sizeof(Lmer<2>); }
cudaError_t launch_encode(int W, const uint8_t* codes, int n, int m, int l, int w, void* table, int* err,
                          cudaStream_t s) {
    const int K = n * w;
    const int threads = 256, blocks = (K + threads - 1) / threads;
    if (W == 1) encode_kernel<1><<<blocks, threads, 0, s>>>(codes, n, m, l, w, static_cast<Lmer<1>*>(table), err);
    else encode_kernel<2><<<blocks, threads, 0, s>>>(codes, n, m, l, w, static_cast<Lmer<2>*>(table), err);
    return cudaGetLastError();
}

cudaError_t launch_rowbuild(int W, const void* table, int n, int w, int d, int K, int sort_rows,
                            const int32_t* anchor_off, int nanchors, uint32_t* l1_entries, LevelMeta* l1_meta,
                            unsigned long long* counters, cudaStream_t s) {
    if (nanchors == 0) return cudaSuccess;
    const int threads = 256;
    if (W == 1)
        rowbuild_kernel<1><<<nanchors, threads, 0, s>>>(static_cast<const Lmer<1>*>(table), n, w, d, K, sort_rows,
                                                         anchor_off, nanchors, l1_entries, l1_meta, counters);
    else
        rowbuild_kernel<2><<<nanchors, threads, 0, s>>>(static_cast<const Lmer<2>*>(table), n, w, d, K, sort_rows,
                                                         anchor_off, nanchors, l1_entries, l1_meta, counters);
    return cudaGetLastError();
}

cudaError_t launch_taskscan(const LevelMeta* l1_meta, int nanchors, int t, long long* task_base, cudaStream_t s) {
    taskscan_kernel<<<1, 32, 0, s>>>(l1_meta, nanchors, t, task_base);
    return cudaGetLastError();
}

cudaError_t launch_reverify(int W, const void* table, int n, int w, int l, int d, const unsigned long long* keys,
                            long long count, int* fail, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    const unsigned blocks = static_cast<unsigned>(count);
    if (W == 1)
        reverify_kernel<1><<<blocks, 256, 0, s>>>(static_cast<const Lmer<1>*>(table), n, w, l, d, keys, count, fail);
    else
        reverify_kernel<2><<<blocks, 256, 0, s>>>(static_cast<const Lmer<2>*>(table), n, w, l, d, keys, count, fail);
    return cudaGetLastError();
}

cudaError_t launch_intpeak(int which, int blocks, int threads, int iters, uint32_t* sink, cudaStream_t s) {
    if (which == 0) intpeak_lop3_kernel<<<blocks, threads, 0, s>>>(0x1234567u, iters, sink);
    else intpeak_popc_kernel<<<blocks, threads, 0, s>>>(0x1234567u, iters, sink);
    return cudaGetLastError();
}

}  // namespace pms8g
