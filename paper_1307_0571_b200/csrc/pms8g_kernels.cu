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

#include <cstdint>

#include "pms8g_device.cuh"
#include "pms8g_launch.h"

namespace pms8g {

namespace {

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <int W>
struct Mask {
    uint32_t w[W];
};

template <int W>
__device__ __forceinline__ Mask<W> mism(const Lmer<W>& a, const Lmer<W>& b) {
    Mask<W> m;
#pragma unroll
    for (int i = 0; i < W; ++i) m.w[i] = (a.h[i] ^ b.h[i]) | (a.o[i] ^ b.o[i]);
    return m;
}

template <int W>
__device__ __forceinline__ int popcm(const Mask<W>& m) {
    int s = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) s += __popc(m.w[i]);
    return s;
}

template <int W>
__device__ __forceinline__ int dist(const Lmer<W>& a, const Lmer<W>& b) {
    return popcm<W>(mism<W>(a, b));
}

template <int W>
__device__ __forceinline__ int popc_and3(const Mask<W>& a, const Mask<W>& b, const Mask<W>& c) {
    int s = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) s += __popc(a.w[i] & b.w[i] & c.w[i]);
    return s;
}

// number of set bits at positions >= p (0 <= p <= 32W)
template <int W>
__device__ __forceinline__ int suffix_popc(const Mask<W>& m, int p) {
    int s = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        const int lo = p - 32 * i;  // bits of word i at index >= lo
        if (lo <= 0) s += __popc(m.w[i]);
        else if (lo < 32) s += __popc(m.w[i] >> lo);
    }
    return s;
}

template <int W>
__device__ __forceinline__ int code_at(const Lmer<W>& x, int p) {
    const int wi = (W == 1) ? 0 : (p >> 5);
    const int b = p & 31;
    uint32_t h, o;
    if (W == 1 || wi == 0) {
        h = x.h[0];
        o = x.o[0];
    } else {
        h = x.h[W - 1];
        o = x.o[W - 1];
    }
    return static_cast<int>((((h >> b) & 1u) << 1) | ((o >> b) & 1u));
}

template <int W>
__device__ __forceinline__ void set_code(Lmer<W>& x, int p, int c) {
    const int b = p & 31;
    if (W == 1 || p < 32) {
        x.h[0] |= static_cast<uint32_t>((c >> 1) & 1) << b;
        x.o[0] |= static_cast<uint32_t>(c & 1) << b;
    } else {
        x.h[W - 1] |= static_cast<uint32_t>((c >> 1) & 1) << b;
        x.o[W - 1] |= static_cast<uint32_t>(c & 1) << b;
    }
}

template <int W>
__device__ __forceinline__ Lmer<W> shfl_lmer(const Lmer<W>& x, int src) {
    Lmer<W> y;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        y.h[i] = __shfl_sync(0xffffffffu, x.h[i], src);
        y.o[i] = __shfl_sync(0xffffffffu, x.o[i], src);
    }
    return y;
}

// 128-bit MSB-first key: symbol 0 in the highest used 2 bits.
template <int W>
__device__ __forceinline__ void make_key(const Lmer<W>& x, int l, unsigned long long& lo, unsigned long long& hi) {
    lo = 0;
    hi = 0;
    for (int p = 0; p < l; ++p) {
        const unsigned long long c = static_cast<unsigned long long>(code_at<W>(x, p));
        const int sh = 2 * (l - 1 - p);
        if (sh >= 64) hi |= c << (sh - 64);
        else lo |= c << sh;
    }
}

}  // namespace

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
            M->start[lane] = static_cast<uint16_t>(excl);
            M->cnt[lane] = static_cast<uint16_t>(cpos);
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
// K4: persistent search kernel

template <int W>
struct Node {
    Lmer<W> c;      // candidate prefix planes
    uint32_t rA;    // budgets of members 0..3, biased by +64, one byte each
    uint32_t rB;    // budgets of members 4..5 (bytes 0,1); prefix length p in byte 3
};

template <int W>
struct WarpShared {
    LevelMeta lev[MAXT + 1];
    int iter[MAXT + 1];
    uint32_t stack_id[MAXT];
    uint16_t cnt_by_row[MAXN];
    uint8_t vorder[MAXN];
    uint32_t eq[64];
    uint8_t thr_pair[65 * NPAIR];
    uint8_t thr_tri[65 * NTRI];
    uint8_t cons[65];
    Lmer<W> cand[CANDCAP];
};

template <int W>
struct SmemLayout {
    static constexpr int NODE_SMEM = (W == 1) ? 128 : 64;
    __host__ __device__ static constexpr size_t warp_bytes() {
        return ((sizeof(WarpShared<W>) + sizeof(Node<W>) * NODE_SMEM) + 15) / 16 * 16;
    }
};

template <int W>
struct WarpCtx {
    const SearchParams* P;
    const Lmer<W>* T;  // table in shared memory
    WarpShared<W>* S;
    Node<W>* node_smem;
    Node<W>* node_glob;
    uint32_t* lvl_glob;  // level buffers (levels 2..t)
    int lane;
    unsigned long long c_push, c_viable, c_slots, c_tuples, c_leaves, c_emit, c_vcmp, c_nodes;
    long long clk_filter, clk_pattern;
};

template <int W>
__device__ __forceinline__ uint32_t* level_entries(WarpCtx<W>& C, int k, const uint32_t* l1) {
    return k == 1 ? const_cast<uint32_t*>(l1) : C.lvl_glob + static_cast<size_t>(k - 2) * C.P->level_cap;
}

// Push of u = stack[k] onto a stack of k members: filter level k (minus its
// branching row) into level k+1. Returns viable (no remaining row emptied).
// Pair rule Hd(v,u) <= 2d, then Theorem 1 with budgets (d,d,d) against every
// older member s_i via Cd3 = (h_vi + h_vu + h_iu + n4)/2 <= 3d, with the
// reference's shortcut: n4 <= min(h) so sum + min <= 6d accepts without n4
// (src/solver.cpp:282-335).
template <int W>
__device__ bool filter_push(WarpCtx<W>& C, int k, const uint32_t* src, uint32_t* dst) {
    const SearchParams& P = *C.P;
    const int lane = C.lane;
    LevelMeta& Ls = C.S->lev[k];
    LevelMeta& Ld = C.S->lev[k + 1];
    const int d = P.d, six_d = 6 * d, two_d = 2 * d;

    const Lmer<W> U = C.T[C.S->stack_id[k] & ID_MASK];
    Lmer<W> Sm[MAXT];
    Mask<W> Miu[MAXT];
    int hs[MAXT];
#pragma unroll
    for (int i = 0; i < MAXT; ++i) {
        if (i < k) {
            Sm[i] = C.T[C.S->stack_id[i] & ID_MASK];
            Miu[i] = mism<W>(Sm[i], U);
            hs[i] = popcm<W>(Miu[i]);
        }
    }
    const int jb = Ls.branch;
    const int bstart = Ls.start[jb], bcnt = Ls.cnt[jb];
    const int n_iter = Ls.total - bcnt;
    const int nrows = Ls.nrows;
    if (lane < MAXN) C.S->cnt_by_row[lane] = 0;
    __syncwarp();
    int out = 0;
    bool dead = false;
    for (int base = 0; base < n_iter; base += 32) {
        const int f = base + lane;
        const bool valid = f < n_iter;
        const int idx = f < bstart ? f : f + bcnt;
        const uint32_t e = valid ? src[idx] : 0xFFFFFFFFu;
        bool keep = false;
        if (valid) {
            const Lmer<W> V = C.T[e & ID_MASK];
            const Mask<W> mu = mism<W>(V, U);
            const int hvu = popcm<W>(mu);
            keep = hvu <= two_d;
#pragma unroll
            for (int i = 0; i < MAXT; ++i) {
                if (i < k && keep) {
                    const Mask<W> mi = mism<W>(V, Sm[i]);
                    const int hvi = popcm<W>(mi);
                    const int sum = hvi + hvu + hs[i];
                    if (sum > six_d) {
                        keep = false;
                    } else {
                        const int mn = min(min(hvi, hvu), hs[i]);
                        if (sum + mn > six_d) keep = sum + popc_and3<W>(mi, mu, Miu[i]) <= six_d;
                    }
                }
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) dst[out + __popc(bal & lanemask_lt())] = e;
        out += __popc(bal);
        // per-row kept counts: rows are contiguous segments of the flat range
        const uint32_t row = e >> 24;
        const uint32_t prow = __shfl_up_sync(0xffffffffu, row, 1);
        const uint32_t nrow = __shfl_down_sync(0xffffffffu, row, 1);
        const bool first = valid && (lane == 0 || prow != row);
        const bool nvalid = (f + 1) < n_iter;
        const bool last = valid && (lane == 31 || !nvalid || nrow != row);
        const unsigned starts = __ballot_sync(0xffffffffu, first);
        bool empty_row = false;
        if (last) {
            const int s0 = 31 - __clz(starts & ((2u << lane) - 1u));
            const unsigned segmask = ((2u << lane) - 1u) & ~((1u << s0) - 1u);
            const int kept = __popc(bal & segmask) + C.S->cnt_by_row[row];
            C.S->cnt_by_row[row] = static_cast<uint16_t>(kept);
            // the row is complete when the next flat entry belongs to another
            // row (known inside the batch) or the range ends
            const bool complete = (lane < 31 && (!nvalid || nrow != row)) || (lane == 31 && !nvalid);
            empty_row = complete && kept == 0;
        }
        __syncwarp();
        if (__any_sync(0xffffffffu, empty_row)) {
            dead = true;
            break;
        }
    }
    C.c_push += 1;
    C.c_slots += static_cast<unsigned long long>(n_iter);
    if (dead) return false;
    // level k+1 row table: level k order without the branching row
    const int nr2 = nrows - 1;
    int c = 0;
    uint8_t row = 0;
    if (lane < nr2) {
        const int j = lane < jb ? lane : lane + 1;
        row = Ls.order[j];
        c = C.S->cnt_by_row[row];
    }
    int incl = c;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, s);
        if (lane >= s) incl += v;
    }
    const bool empty = lane < nr2 && c == 0;
    if (__any_sync(0xffffffffu, empty)) return false;
    // branching row: smallest count, ties by position (or position 0 unsorted)
    int key = lane < nr2 ? (c << 8) | lane : 0x7FFFFFFF;
    if (P.sort_rows) {
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, s));
    } else {
        key = __shfl_sync(0xffffffffu, key, 0);
    }
    if (lane < nr2) {
        Ld.start[lane] = static_cast<uint16_t>(incl - c);
        Ld.cnt[lane] = static_cast<uint16_t>(c);
        Ld.order[lane] = row;
    }
    if (lane == 0) {
        Ld.nrows = nr2;
        Ld.total = out;
        Ld.branch = key & 0xFF;
        Ld.viable = 1;
    }
    __syncwarp();
    C.c_viable += 1;
    return true;
}

// Verify up to 32 buffered candidates (lane i holds cand[i]) against the
// level's rows, smallest row first; a candidate survives a row when some
// surviving l-mer is within d (verify_candidate, src/solver.cpp:344-362).
// Survivors are emitted as packed keys.
template <int W>
__device__ void verify_batch(WarpCtx<W>& C, const LevelMeta& L, const uint32_t* entries, int nb) {
    const SearchParams& P = *C.P;
    const int lane = C.lane;
    bool alive = lane < nb;
    Lmer<W> cand;
    if (alive) cand = C.S->cand[lane];
    const int d = P.d;
    for (int r = 0; r < L.nrows; ++r) {
        const unsigned am = __ballot_sync(0xffffffffu, alive);
        if (am == 0) break;
        const int j = C.S->vorder[r];
        const int st = L.start[j], cnt = L.cnt[j];
        bool hit = false;
        int scanned = 0;
        bool done = false;
        for (int base = 0; base < cnt && !done; base += 32) {
            // one coalesced load of up to 32 row entries, broadcast by shuffle
            const uint32_t mine = base + lane < cnt ? entries[st + base + lane] : 0u;
            const int lim = min(32, cnt - base);
            for (int x = 0; x < lim; ++x) {
                const uint32_t id = __shfl_sync(0xffffffffu, mine, x) & ID_MASK;
                const Lmer<W> V = C.T[id];
                hit |= dist<W>(cand, V) <= d;
                ++scanned;
                if ((x & 7) == 7 && __all_sync(0xffffffffu, hit || !alive)) {
                    done = true;
                    break;
                }
            }
        }
        C.c_vcmp += static_cast<unsigned long long>(__popc(am)) * scanned;
        alive = alive && hit;
    }
    const unsigned em = __ballot_sync(0xffffffffu, alive);
    if (em) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(P.key_count, static_cast<unsigned long long>(__popc(em)));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (alive) {
            const unsigned long long pos = base + __popc(em & lanemask_lt());
            if (static_cast<long long>(pos) < P.key_cap) {
                unsigned long long klo, khi;
                make_key<W>(cand, P.l, klo, khi);
                P.keys[2 * pos] = klo;
                P.keys[2 * pos + 1] = khi;
            }
        }
        C.c_emit += __popc(em);
    }
}

// Common d-neighbourhood of the t-tuple on the stack, enumerated by a
// warp-cooperative DFS: each round pops 8 nodes and evaluates their 4
// children on 32 lanes; children are pruned exactly as
// NeighborhoodEnumerator::prune (src/neighborhood.cpp:228-270: exhausted
// budgets, pair suffix distances, Theorem-1 triples, consensus bound), checked
// only on edges that spent budget (neighborhood.hpp:72). Leaves feed the
// verification buffer.
template <int W>
__device__ void enumerate_verify(WarpCtx<W>& C, int k, const uint32_t* entries) {
    const SearchParams& P = *C.P;
    const int lane = C.lane;
    const int l = P.l, d = P.d;
    const int t = k;  // tuple size
    const LevelMeta& L = C.S->lev[k];
    WarpShared<W>& S = *C.S;
    const long long c0 = clock64();

    Lmer<W> Tm[MAXT];
#pragma unroll
    for (int i = 0; i < MAXT; ++i)
        if (i < t) Tm[i] = C.T[S.stack_id[i] & ID_MASK];

    // --- per-tuple suffix tables (NeighborhoodEnumerator::prepare, :164-226)
    for (int p = lane; p <= l; p += 32) {
        uint32_t e = 0;
        if (p < l) {
#pragma unroll
            for (int i = 0; i < MAXT; ++i)
                if (i < t) e |= 1u << (8 * code_at<W>(Tm[i], p) + i);
            S.eq[p] = e;
        }
#pragma unroll
        for (int j = 1; j < MAXT; ++j)
#pragma unroll
            for (int i = 0; i < j; ++i)
                if (j < t) {
                    const Mask<W> mij = mism<W>(Tm[i], Tm[j]);
                    S.thr_pair[p * NPAIR + j * (j - 1) / 2 + i] = static_cast<uint8_t>(suffix_popc<W>(mij, p));
                }
#pragma unroll
        for (int h = 2; h < MAXT; ++h)
#pragma unroll
            for (int j = 1; j < h; ++j)
#pragma unroll
                for (int i = 0; i < j; ++i)
                    if (h < t) {
                        const Mask<W> mij = mism<W>(Tm[i], Tm[j]);
                        const Mask<W> mih = mism<W>(Tm[i], Tm[h]);
                        const Mask<W> mjh = mism<W>(Tm[j], Tm[h]);
                        Mask<W> n4;
#pragma unroll
                        for (int x = 0; x < W; ++x) n4.w[x] = mij.w[x] & mih.w[x] & mjh.w[x];
                        const int v = (suffix_popc<W>(mij, p) + suffix_popc<W>(mih, p) + suffix_popc<W>(mjh, p) +
                                       suffix_popc<W>(n4, p)) / 2;
                        S.thr_tri[p * NTRI + h * (h - 1) * (h - 2) / 6 + j * (j - 1) / 2 + i] =
                            static_cast<uint8_t>(v);
                    }
    }
    __syncwarp();
    // consensus suffix: sum over columns >= p of (t - max frequency)
    {
        int carry = 0;
        const int nchunk = (l + 32) / 32;  // positions 0..l
        for (int ch = nchunk - 1; ch >= 0; --ch) {
            const int p = ch * 32 + lane;
            int v = 0;
            if (p < l) {
                const uint32_t e = S.eq[p];
                const int best = max(max(__popc(e & 0xFFu), __popc(e & 0xFF00u)),
                                     max(__popc(e & 0xFF0000u), __popc(e & 0xFF000000u)));
                v = t - best;
            }
            // reverse inclusive scan (suffix sum) within the chunk
            int incl = v;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const int x = __shfl_down_sync(0xffffffffu, incl, s);
                if (lane + s < 32) incl += x;
            }
            if (p <= l) S.cons[p] = static_cast<uint8_t>(incl + carry);
            carry += __shfl_sync(0xffffffffu, incl, 0);
        }
    }
    // verification order: rows by ascending count
    if (lane < L.nrows) {
        const int c = L.cnt[lane];
        int rank = 0;
        for (int q = 0; q < L.nrows; ++q) {
            const int cq = L.cnt[q];
            rank += (cq < c) || (cq == c && q < lane);
        }
        S.vorder[rank] = static_cast<uint8_t>(lane);
    }
    __syncwarp();

    // --- DFS
    const int node_smem_cap = SmemLayout<W>::NODE_SMEM;
    auto node_ptr = [&](int idx) -> Node<W>* {
        return idx < node_smem_cap ? C.node_smem + idx : C.node_glob + (idx - node_smem_cap);
    };
    const uint32_t tmask = (1u << t) - 1u;
    int nn = 1, ncand = 0;
    if (lane == 0) {
        Node<W> root;
#pragma unroll
        for (int i = 0; i < W; ++i) root.c.h[i] = root.c.o[i] = 0;
        const uint32_t b = static_cast<uint32_t>(d + 64);
        root.rA = b | (b << 8) | (b << 16) | (b << 24);
        root.rB = b | (b << 8);
        *node_ptr(0) = root;
    }
    __syncwarp();
    const int prune = P.prune;
    const int cap_nodes = node_smem_cap + P.node_cap;
    unsigned long long nodes = 0, leaves = 0;
    while (nn > 0) {
        const int take = min(8, nn);
        const int base = nn - take;
        const int slot = lane >> 2;
        const int c = lane & 3;
        const bool active = slot < take;
        Node<W> nd;
        if (active) nd = *node_ptr(base + slot);
        __syncwarp();
        nodes += take;
        bool ok = false, leaf = false;
        Node<W> ch;
        if (active) {
            const int p = static_cast<int>(nd.rB >> 24);
            const uint32_t em = (S.eq[p] >> (8 * c)) & tmask;  // members matching symbol c
            const uint32_t mm = ~em & tmask;                   // members charged on this edge
            int r[MAXT];
#pragma unroll
            for (int i = 0; i < MAXT; ++i) {
                const uint32_t word = i < 4 ? nd.rA : nd.rB;
                r[i] = static_cast<int>((word >> (8 * (i & 3))) & 0xFFu) - 64 - static_cast<int>((mm >> i) & 1u);
            }
            ch.c = nd.c;
            set_code<W>(ch.c, p, c);
            const int q = p + 1;
            bool neg = false;
#pragma unroll
            for (int i = 0; i < MAXT; ++i)
                if (i < t) neg |= r[i] < 0;
            leaf = q == l;
            if (leaf) {
                ok = !neg;
            } else if (prune == 0 || mm == 0) {
                ok = true;
            } else {
                ok = !neg;
                if (ok) {
#pragma unroll
                    for (int j = 1; j < MAXT; ++j)
#pragma unroll
                        for (int i = 0; i < j; ++i)
                            if (j < t) ok &= S.thr_pair[q * NPAIR + j * (j - 1) / 2 + i] <= r[i] + r[j];
                }
                if (ok && prune == 2) {
#pragma unroll
                    for (int h = 2; h < MAXT; ++h)
#pragma unroll
                        for (int j = 1; j < h; ++j)
#pragma unroll
                            for (int i = 0; i < j; ++i)
                                if (h < t)
                                    ok &= S.thr_tri[q * NTRI + h * (h - 1) * (h - 2) / 6 + j * (j - 1) / 2 + i] <=
                                          r[i] + r[j] + r[h];
                    int sum = 0;
#pragma unroll
                    for (int i = 0; i < MAXT; ++i)
                        if (i < t) sum += r[i];
                    if (t >= 2) ok &= S.cons[q] <= sum;
                }
            }
            uint32_t rA = 0, rB = 0;
#pragma unroll
            for (int i = 0; i < MAXT; ++i) {
                const uint32_t b = static_cast<uint32_t>(r[i] + 64) & 0xFFu;
                if (i < 4) rA |= b << (8 * i);
                else rB |= b << (8 * (i - 4));
            }
            ch.rA = rA;
            ch.rB = rB | (static_cast<uint32_t>(q) << 24);
        }
        const unsigned lb = __ballot_sync(0xffffffffu, ok && leaf);
        const unsigned ib = __ballot_sync(0xffffffffu, ok && !leaf);
        if (ok && leaf) S.cand[ncand + __popc(lb & lanemask_lt())] = ch.c;
        if (ok && !leaf) {
            const int pos = base + __popc(ib & lanemask_lt());
            if (pos < cap_nodes) *node_ptr(pos) = ch;
        }
        ncand += __popc(lb);
        leaves += __popc(lb);
        nn = base + __popc(ib);
        if (nn > cap_nodes) {
            if (lane == 0) atomicOr(P.error_flag, 2);
            nn = 0;
        }
        __syncwarp();
        if (ncand >= 32) {
            verify_batch<W>(C, L, entries, 32);
            __syncwarp();
            const int rest = ncand - 32;
            Lmer<W> tmp;
            if (lane < rest) tmp = S.cand[32 + lane];
            __syncwarp();
            if (lane < rest) S.cand[lane] = tmp;
            __syncwarp();
            ncand = rest;
        }
    }
    if (ncand > 0) {
        verify_batch<W>(C, L, entries, ncand);
        __syncwarp();
    }
    C.c_tuples += 1;
    C.c_leaves += leaves;
    C.c_nodes += nodes;
    C.clk_pattern += clock64() - c0;
}

template <int W>
__global__ void __launch_bounds__(512, 1) search_kernel(SearchParams P) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    Lmer<W>* T = reinterpret_cast<Lmer<W>*>(smem);
    const Lmer<W>* gT = static_cast<const Lmer<W>*>(P.table);
    for (int i = threadIdx.x; i < P.K; i += blockDim.x) T[i] = gT[i];
    const size_t table_bytes = (static_cast<size_t>(P.K) * sizeof(Lmer<W>) + 15) / 16 * 16;
    uint8_t* wbase = smem + table_bytes + SmemLayout<W>::warp_bytes() * warp;
    __syncthreads();

    WarpCtx<W> C;
    C.P = &P;
    C.T = T;
    C.S = reinterpret_cast<WarpShared<W>*>(wbase);
    C.node_smem = reinterpret_cast<Node<W>*>(wbase + sizeof(WarpShared<W>));
    const size_t gw = static_cast<size_t>(blockIdx.x) * nwarps + warp;
    uint32_t* scratch = P.scratch + gw * P.scratch_words;
    C.lvl_glob = scratch;
    C.node_glob = reinterpret_cast<Node<W>*>(scratch + static_cast<size_t>(P.t > 1 ? P.t - 1 : 0) * P.level_cap);
    C.lane = lane;
    C.c_push = C.c_viable = C.c_slots = C.c_tuples = C.c_leaves = C.c_emit = C.c_vcmp = C.c_nodes = 0;
    C.clk_filter = C.clk_pattern = 0;
    WarpShared<W>& S = *C.S;
    const int t = P.t;
    const long long ntasks = P.task_base[P.nanchors];

    for (;;) {
        long long task = 0;
        if (lane == 0) task = static_cast<long long>(atomicAdd(P.task_counter, 1ull));
        task = __shfl_sync(0xffffffffu, task, 0);
        if (task >= ntasks) break;
        // anchor index: last a with task_base[a] <= task
        int lo = 0, hi = P.nanchors - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (P.task_base[mid] <= task) lo = mid;
            else hi = mid - 1;
        }
        const int ai = lo;
        const int j = static_cast<int>(task - P.task_base[ai]);
        const uint32_t* l1 = P.l1_entries + static_cast<size_t>(ai) * P.K;
        // level 1 row table from the row build
        {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(P.l1_meta + ai);
            uint32_t* dstm = reinterpret_cast<uint32_t*>(&S.lev[1]);
            for (int x = lane; x < static_cast<int>(sizeof(LevelMeta) / 4); x += 32) dstm[x] = src[x];
        }
        if (lane == 0) S.stack_id[0] = static_cast<uint32_t>(P.anchor_off[ai]);
        __syncwarp();
        if (t == 1) {
            enumerate_verify<W>(C, 1, l1);
            continue;
        }
        // depth-1 branch: u = j-th entry of the anchor's branching row
        const LevelMeta& L1 = S.lev[1];
        const uint32_t u = l1[L1.start[L1.branch] + j];
        if (lane == 0) S.stack_id[1] = u;
        __syncwarp();
        const long long f0 = clock64();
        bool v = filter_push<W>(C, 1, l1, level_entries<W>(C, 2, l1));
        C.clk_filter += clock64() - f0;
        if (!v) continue;
        if (t == 2) {
            enumerate_verify<W>(C, 2, level_entries<W>(C, 2, l1));
            continue;
        }
        // DFS over levels 2..t-1
        int k = 2;
        if (lane == 0) S.iter[2] = 0;
        __syncwarp();
        while (k >= 2) {
            LevelMeta& L = S.lev[k];
            const int it = S.iter[k];
            if (it >= L.cnt[L.branch]) {
                --k;
                continue;
            }
            uint32_t* ek = level_entries<W>(C, k, l1);
            const uint32_t uu = ek[L.start[L.branch] + it];
            __syncwarp();
            if (lane == 0) {
                S.iter[k] = it + 1;
                S.stack_id[k] = uu;
            }
            __syncwarp();
            const long long f1 = clock64();
            const bool ok = filter_push<W>(C, k, ek, level_entries<W>(C, k + 1, l1));
            C.clk_filter += clock64() - f1;
            if (!ok) continue;
            if (k + 1 == t) {
                enumerate_verify<W>(C, t, level_entries<W>(C, t, l1));
            } else {
                ++k;
                if (lane == 0) S.iter[k] = 0;
                __syncwarp();
            }
        }
    }
    if (lane == 0) {
        atomicAdd(P.counters + C_PUSHES, C.c_push);
        atomicAdd(P.counters + C_VIABLE, C.c_viable);
        atomicAdd(P.counters + C_SLOTS, C.c_slots);
        atomicAdd(P.counters + C_TUPLES, C.c_tuples);
        atomicAdd(P.counters + C_LEAVES, C.c_leaves);
        atomicAdd(P.counters + C_EMITTED, C.c_emit);
        atomicAdd(P.counters + C_VCMP, C.c_vcmp);
        atomicAdd(P.counters + C_NODES, C.c_nodes);
        atomicAdd(P.counters + C_CLK_FILTER, static_cast<unsigned long long>(C.clk_filter));
        atomicAdd(P.counters + C_CLK_PATTERN, static_cast<unsigned long long>(C.clk_pattern));
    }
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

template <int W>
size_t search_smem_bytes(int K, int warps) {
    return (static_cast<size_t>(K) * sizeof(Lmer<W>) + 15) / 16 * 16 + SmemLayout<W>::warp_bytes() * warps;
}

size_t lmer_bytes(int W) { return W == 1 ? sizeof(Lmer<1>) : sizeof(Lmer<2>); }
size_t node_bytes(int W) { return W == 1 ? sizeof(Node<1>) : sizeof(Node<2>); }
size_t search_smem(int W, int K, int warps) {
    return W == 1 ? search_smem_bytes<1>(K, warps) : search_smem_bytes<2>(K, warps);
}
size_t search_warp_smem(int W) { return W == 1 ? SmemLayout<1>::warp_bytes() : SmemLayout<2>::warp_bytes(); }

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

cudaError_t set_search_smem(int W, size_t bytes) {
    if (W == 1)
        return cudaFuncSetAttribute(search_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(bytes));
    return cudaFuncSetAttribute(search_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes));
}

cudaError_t launch_search(int W, const SearchParams& P, int blocks, int warps, size_t smem, cudaStream_t s) {
    if (W == 1) search_kernel<1><<<blocks, warps * 32, smem, s>>>(P);
    else search_kernel<2><<<blocks, warps * 32, smem, s>>>(P);
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
