// pms8g_sigma.cu — the per-S1-l-mer search for alphabets of 5..32 symbols
// (protein: 20), SURVEY.md §8(f) row 4.
//
// The reference packs b = ceil(log2 sigma) bits per symbol (src/alphabet.cpp:
// 41, include/pms8/packed_seq.hpp:86-88); here an l-mer (l <= 32) is B = b bit
// planes of one 32-bit word each: symbol code c at position p sets bit p of
// plane k iff bit k of c is set. Two l-mers mismatch at p iff some plane
// differs there, so Hd = popc(OR_k (x.p[k] ^ y.p[k])) — the same XOR/OR/POPC
// form as the two-plane DNA path, with B planes.
//
//   encode_sigma_kernel    codes -> B planes per l-mer (PackedSequenceSet)
//   rowbuild_sigma_kernel  per S1 l-mer: rows of l-mers within 2d, in the
//                          LevelMeta/entry layout of the DNA path (the task
//                          scan and the static task count are shared)
//   sigma_search_kernel    persistent warps over (S1 l-mer, depth-1 branch)
//                          tasks: DFS pushes that filter every remaining row
//                          with the pair rule and Theorem 1 (MotifSearch::push,
//                          src/solver.cpp:245-337), the branching row being the
//                          smallest (sort_rows_by_size); at the switch depth the
//                          common d-neighbourhood is enumerated sigma-way with
//                          the budget, pair-suffix and consensus-suffix bounds
//                          (NeighborhoodEnumerator::prune, src/neighborhood.cpp:
//                          114-156) and every leaf is verified against the
//                          remaining rows (verify_candidate, src/solver.cpp:
//                          344-362)
//   reverify_sigma_kernel  SolverConfig::reverify_against_originals
// Keys: B bits per symbol, MSB-first (B*l <= 128), sorted/deduplicated by
// the same device radix sort as the DNA path.
#include <cuda_runtime.h>

#include <cstdint>

#include "pms8g_common.cuh"
#include "pms8g_device.cuh"
#include "pms8g_sigma.h"

namespace pms8g {

using namespace dev;

namespace {

template <int B>
struct LmerS {
    uint32_t p[B];
};

template <int B>
__device__ __forceinline__ uint32_t smism(const LmerS<B>& a, const LmerS<B>& b) {
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < B; ++k) m |= a.p[k] ^ b.p[k];
    return m;
}

template <int B>
__device__ __forceinline__ int sdist(const LmerS<B>& a, const LmerS<B>& b) {
    return __popc(smism<B>(a, b));
}

template <int B>
__device__ __forceinline__ int scode(const LmerS<B>& x, int p) {
    int c = 0;
#pragma unroll
    for (int k = 0; k < B; ++k) c |= static_cast<int>((x.p[k] >> p) & 1u) << k;
    return c;
}

template <int B>
__device__ __forceinline__ LmerS<B> ldt(const LmerS<B>* __restrict__ T, uint32_t id) {
    LmerS<B> x;
#pragma unroll
    for (int k = 0; k < B; ++k) x.p[k] = __ldg(&T[id].p[k]);
    return x;
}

template <int B>
__global__ void encode_sigma_kernel(const uint8_t* __restrict__ codes, int n, int m, int l, int w, int sigma,
                                    LmerS<B>* __restrict__ table, int* error_flag) {
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n * w) return;
    const int r = id / w, off = id - r * w;
    const uint8_t* s = codes + static_cast<size_t>(r) * m + off;
    LmerS<B> x;
#pragma unroll
    for (int k = 0; k < B; ++k) x.p[k] = 0u;
    bool bad = false;
    for (int p = 0; p < l; ++p) {
        const int c = s[p];
        bad |= c >= sigma;
#pragma unroll
        for (int k = 0; k < B; ++k) x.p[k] |= static_cast<uint32_t>((c >> k) & 1) << p;
    }
    if (bad) atomicOr(error_flag, 1);
    table[id] = x;
}

// One block per anchor: rows 1..n-1 of l-mers within 2d of the anchor, rows
// ordered by size (RowMatrix::sort_rows_by_size), entry = row << 24 | id.
template <int B>
__global__ void rowbuild_sigma_kernel(const LmerS<B>* __restrict__ table, int n, int w, int d, int K,
                                      const int32_t* __restrict__ anchor_off, int nanchors,
                                      uint32_t* __restrict__ l1_entries, LevelMeta* __restrict__ l1_meta,
                                      unsigned long long* counters) {
    __shared__ int cnt[MAXN], startp[MAXN], posof[MAXN];
    const int ai = blockIdx.x;
    if (ai >= nanchors) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const LmerS<B> A = ldt<B>(table, static_cast<uint32_t>(anchor_off[ai]));
    for (int r = 1 + warp; r < n; r += nw) {
        int c = 0;
        for (int base = 0; base < w; base += 32) {
            const int o = base + lane;
            c += __popc(__ballot_sync(0xffffffffu, o < w && sdist<B>(A, ldt<B>(table, r * w + o)) <= 2 * d));
        }
        if (lane == 0) cnt[r] = c;
    }
    __syncthreads();
    const int nrows = n - 1;
    if (warp == 0) {
        int c = 0, rank = 0;
        if (lane < nrows) {
            c = cnt[lane + 1];
            for (int q = 1; q < n; ++q) rank += (cnt[q] < c) || (cnt[q] == c && q < lane + 1);
            posof[lane + 1] = rank;
        }
        __syncwarp();
        int cpos = 0, row = 0;
        if (lane < nrows)
            for (int q = 1; q < n; ++q)
                if (posof[q] == lane) {
                    cpos = cnt[q];
                    row = q;
                }
        int incl = cpos;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, s);
            if (lane >= s) incl += v;
        }
        if (lane < nrows) startp[lane] = incl - cpos;
        const bool any_empty = __any_sync(0xffffffffu, lane < nrows && cpos == 0);
        LevelMeta* M = l1_meta + ai;
        if (lane < nrows) {
            M->start[lane] = static_cast<uint32_t>(incl - cpos);
            M->cnt[lane] = static_cast<uint32_t>(cpos);
            M->order[lane] = static_cast<uint8_t>(row);
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
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
            const bool ok = o < w && sdist<B>(A, ldt<B>(table, r * w + o)) <= 2 * d;
            const unsigned bal = __ballot_sync(0xffffffffu, ok);
            if (ok) out[dst + __popc(bal & lanemask_lt())] = (static_cast<uint32_t>(r) << 24) | (r * w + o);
            dst += __popc(bal);
        }
    }
}

// Per-warp shared state of the search.
constexpr int SCAND = 32;  // candidates verified per batch (one per lane)

struct SigmaWarp {
    LevelMeta lev[MAXT + 1];
    int iter[MAXT + 1], iter_end[MAXT + 1];
    uint32_t stack_id[MAXT];
    uint32_t cnt_by_row[MAXN];
    uint8_t sym[MAXT][32];           // tuple members' symbols per position
    uint8_t pair_suf[33][NPAIR];     // Hd of members i<j over positions >= q
    uint8_t cons_suf[33];            // consensus cost over positions >= q
    uint32_t cand[SCAND][8];         // leaf planes awaiting verification
    unsigned long long ctr[W_SIGMA_N];
};

struct SigmaNode {
    uint32_t p[5];   // prefix planes (positions < pos)
    uint8_t r[MAXT];  // remaining budgets
    uint8_t pos;
    uint8_t pad;
};

template <int B, int MT>
struct SCtx {
    const SigmaParams* P;
    SigmaWarp* S;
    uint32_t* lvl;     // per-warp level buffers (levels 2..t)
    SigmaNode* nodes;  // per-warp enumeration stack
    const uint32_t* l1;
    int lane;
    __device__ __forceinline__ uint32_t* entries(int k) const {
        return k == 1 ? const_cast<uint32_t*>(l1) : lvl + static_cast<size_t>(k - 2) * P->level_cap;
    }
    __device__ __forceinline__ LmerS<B> lm(uint32_t id) const {
        return ldt<B>(static_cast<const LmerS<B>*>(P->table), id & ID_MASK);
    }
    __device__ __forceinline__ void add(int i, unsigned long long v) {
        if (lane == 0) S->ctr[i] += v;
    }
};

// Push u = stack[k]: filter every remaining row of level k except the
// branching row into level k+1 (pair rule + Theorem 1 for every older
// member); the new branching row is the smallest. Returns viable.
template <int B, int MT>
__device__ __noinline__ bool sigma_push(SCtx<B, MT>& C, int k) {
    const SigmaParams& P = *C.P;
    SigmaWarp& S = *C.S;
    const int lane = C.lane;
    const LevelMeta& Ls = S.lev[k];
    LevelMeta& Ld = S.lev[k + 1];
    const uint32_t* src = C.entries(k);
    uint32_t* dst = C.entries(k + 1);
    const int d = P.d;
    const LmerS<B> U = C.lm(S.stack_id[k]);
    LmerS<B> Sm[MT];
    uint32_t Miu[MT];
    int hs[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i)
        if (i < k) {
            Sm[i] = C.lm(S.stack_id[i]);
            Miu[i] = smism<B>(Sm[i], U);
            hs[i] = __popc(Miu[i]);
        }
    const int jb = Ls.branch;
    if (lane < MAXN) S.cnt_by_row[lane] = 0;
    __syncwarp();
    int out = 0;
    unsigned long long slots = 0;
    for (int j = 0; j < Ls.nrows; ++j) {
        if (j == jb) continue;
        const int st = Ls.start[j], cnt = Ls.cnt[j];
        const int row = Ls.order[j];
        int kept = 0;
        for (int base = 0; base < cnt; base += 32) {
            const int f = base + lane;
            bool keep = false;
            uint32_t e = 0;
            if (f < cnt) {
                e = src[st + f];
                const LmerS<B> V = C.lm(e);
                const uint32_t mu = smism<B>(V, U);
                const int hvu = __popc(mu);
                keep = hvu <= 2 * d;
#pragma unroll
                for (int i = 0; i < MT; ++i)
                    if (i < k && keep) {
                        const uint32_t mi = smism<B>(V, Sm[i]);
                        const int hvi = __popc(mi);
                        const int sum = hvi + hvu + hs[i];
                        // Cd3 = (h_vi + h_vu + h_iu + n4) / 2 <= 3d (all-distinct
                        // columns n4: any alphabet, src/pruning.cpp)
                        keep = sum <= 6 * d && sum + __popc(mi & mu & Miu[i]) <= 6 * d;
                    }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) dst[out + kept + __popc(bal & lanemask_lt())] = e;
            kept += __popc(bal);
        }
        slots += static_cast<unsigned long long>(cnt);
        if (lane == 0) S.cnt_by_row[row] = static_cast<uint32_t>(kept);
        out += kept;
    }
    __syncwarp();
    C.add(W_SIGMA_PUSH, 1);
    C.add(W_SIGMA_SLOTS, slots);
    // level k+1 row table: rows in level-k order minus the branching row
    const int nr2 = Ls.nrows - 1;
    int c = 0, row = 0;
    if (lane < nr2) {
        const int j = lane < jb ? lane : lane + 1;
        row = Ls.order[j];
        c = S.cnt_by_row[row];
    }
    int incl = c;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, s);
        if (lane >= s) incl += v;
    }
    if (__any_sync(0xffffffffu, lane < nr2 && c == 0)) return false;
    int key = lane < nr2 ? (c << 8) | lane : 0x7FFFFFFF;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, s));
    if (lane < nr2) {
        Ld.start[lane] = static_cast<uint32_t>(incl - c);
        Ld.cnt[lane] = static_cast<uint32_t>(c);
        Ld.order[lane] = static_cast<uint8_t>(row);
    }
    if (lane == 0) {
        Ld.nrows = nr2;
        Ld.total = out;
        Ld.branch = key & 0xFF;
        Ld.viable = 1;
    }
    __syncwarp();
    C.add(W_SIGMA_VIABLE, 1);
    return true;
}

// Verify `n` buffered candidates against every row of level t (one lane per
// candidate); survivors become keys.
template <int B, int MT>
__device__ __noinline__ void sigma_verify(SCtx<B, MT>& C, int t, int n) {
    const SigmaParams& P = *C.P;
    SigmaWarp& S = *C.S;
    const int lane = C.lane;
    const LevelMeta& L = S.lev[t];
    const uint32_t* ent = C.entries(t);
    LmerS<B> cd;
#pragma unroll
    for (int k = 0; k < B; ++k) cd.p[k] = lane < n ? S.cand[lane][k] : 0u;
    bool alive = lane < n;
    unsigned long long vcmp = 0;
    for (int j = 0; j < L.nrows && __any_sync(0xffffffffu, alive); ++j) {
        const int st = L.start[j], cnt = L.cnt[j];
        bool hit = false;
        for (int base = 0; base < cnt; base += 32) {
            const int f = base + lane;
            const LmerS<B> mine = C.lm(f < cnt ? ent[st + f] : ent[st]);
            const int lim = min(32, cnt - base);
            for (int x = 0; x < lim; ++x) {
                LmerS<B> v;
#pragma unroll
                for (int k = 0; k < B; ++k) v.p[k] = __shfl_sync(0xffffffffu, mine.p[k], x);
                hit |= sdist<B>(cd, v) <= P.d;
            }
            vcmp += static_cast<unsigned long long>(lim) * __popc(__ballot_sync(0xffffffffu, alive && !hit));
            if (__all_sync(0xffffffffu, !alive || hit)) break;
        }
        alive = alive && hit;
    }
    C.add(W_SIGMA_VCMP, vcmp);
    const unsigned em = __ballot_sync(0xffffffffu, alive);
    if (!em) return;
    unsigned long long pos0 = 0;
    if (lane == 0) pos0 = atomicAdd(P.key_count, static_cast<unsigned long long>(__popc(em)));
    pos0 = __shfl_sync(0xffffffffu, pos0, 0);
    if (alive) {
        const unsigned long long pos = pos0 + __popc(em & lanemask_lt());
        if (static_cast<long long>(pos) < P.key_cap) {
            // B bits per symbol, symbol 0 in the highest used bits
            unsigned long long lo = 0, hi = 0;
            for (int p = 0; p < P.l; ++p) {
                const unsigned long long c = static_cast<unsigned long long>(scode<B>(cd, p));
                const int sh = B * (P.l - 1 - p);
                if (sh >= 64) hi |= c << (sh - 64);
                else {
                    lo |= c << sh;
                    if (sh + B > 64) hi |= c >> (64 - sh);
                }
            }
            P.keys[2 * pos] = lo;
            P.keys[2 * pos + 1] = hi;
        }
    }
    C.add(W_SIGMA_EMIT, static_cast<unsigned long long>(__popc(em)));
}

// Common d-neighbourhood of the t-tuple on the stack, sigma-way DFS; a round
// expands floor(32 / sigma) nodes, one lane per (node, symbol).
template <int B, int MT>
__device__ __noinline__ void sigma_enumerate(SCtx<B, MT>& C, int t) {
    const SigmaParams& P = *C.P;
    SigmaWarp& S = *C.S;
    const int lane = C.lane, l = P.l, sigma = P.sigma, d = P.d;
    // tables: member symbols, pair-suffix distances, consensus-suffix cost
    LmerS<B> Tm[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i)
        if (i < t) Tm[i] = C.lm(S.stack_id[i]);
    if (lane < l) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
            if (i < t) S.sym[i][lane] = static_cast<uint8_t>(scode<B>(Tm[i], lane));
    }
    __syncwarp();
    {
        // consensus cost of column p: t minus the most frequent symbol's count
        int cost = 0;
        if (lane < l) {
            int best = 0;
#pragma unroll
            for (int i = 0; i < MT; ++i)
                if (i < t) {
                    int f = 0;
#pragma unroll
                    for (int j = 0; j < MT; ++j)
                        if (j < t) f += S.sym[j][lane] == S.sym[i][lane];
                    best = max(best, f);
                }
            cost = t - best;
        }
        // suffix sums over positions >= q (reverse inclusive scan)
        int incl = cost;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const int v = __shfl_down_sync(0xffffffffu, incl, s);
            if (lane + s < 32) incl += v;
        }
        if (lane <= l) S.cons_suf[lane] = static_cast<uint8_t>(lane < l ? incl : 0);
#pragma unroll
        for (int j = 1; j < MT; ++j)
#pragma unroll
            for (int i = 0; i < j; ++i)
                if (j < t) {
                    const uint32_t m = smism<B>(Tm[i], Tm[j]);
                    if (lane <= l)
                        S.pair_suf[lane][j * (j - 1) / 2 + i] =
                            static_cast<uint8_t>(lane < 32 ? __popc(lane < l ? (m >> lane) : 0u) : 0);
                }
    }
    __syncwarp();
    C.add(W_SIGMA_TUPLES, 1);
    // DFS over positions; children of a node: every symbol
    SigmaNode* ns = C.nodes;
    int nn = 0;
    if (lane == 0) {
        SigmaNode root;
#pragma unroll
        for (int k = 0; k < 5; ++k) root.p[k] = 0u;
#pragma unroll
        for (int i = 0; i < MAXT; ++i) root.r[i] = static_cast<uint8_t>(d);
        root.pos = 0;
        root.pad = 0;
        ns[0] = root;
    }
    nn = 1;
    __syncwarp();
    const int per = max(1, 32 / sigma);  // nodes per round
    int ncand = 0;
    unsigned long long nodes = 0, leaves = 0;
    const int prune = P.prune;
    while (nn > 0) {
        const int take = min(per, nn);
        const int base = nn - take;
        const int slot = lane / sigma, c = lane - slot * sigma;
        const bool active = slot < take && lane < per * sigma;
        SigmaNode nd{}, ch{};
        bool ok = false, leaf = false;
        if (active) {
            nd = ns[base + slot];
            const int p = nd.pos;
            ok = true;
            int sum = 0;
#pragma unroll
            for (int i = 0; i < MT; ++i)
                if (i < t) {
                    const int r = static_cast<int>(nd.r[i]) - (S.sym[i][p] != c ? 1 : 0);
                    ok &= r >= 0;
                    ch.r[i] = static_cast<uint8_t>(r < 0 ? 0 : r);
                    sum += r;
                }
            ch.pos = static_cast<uint8_t>(p + 1);
#pragma unroll
            for (int k = 0; k < B; ++k) ch.p[k] = nd.p[k] | (static_cast<uint32_t>((c >> k) & 1) << p);
            leaf = p + 1 == l;
            if (ok && !leaf && prune >= 1) {
                const int q = p + 1;
#pragma unroll
                for (int j = 1; j < MT; ++j)
#pragma unroll
                    for (int i = 0; i < j; ++i)
                        if (j < t) ok &= S.pair_suf[q][j * (j - 1) / 2 + i] <= ch.r[i] + ch.r[j];
                if (prune >= 2 && t >= 2) ok &= S.cons_suf[q] <= sum;
            }
        }
        nodes += take;
        __syncwarp();
        const unsigned lb = __ballot_sync(0xffffffffu, ok && leaf);
        const unsigned ib = __ballot_sync(0xffffffffu, ok && !leaf);
        const unsigned lt = lanemask_lt();
        const int nl = __popc(lb);
        // leaves -> candidate buffer (verify when it would overflow)
        if (ncand + nl > SCAND) {
            sigma_verify<B, MT>(C, t, ncand);
            ncand = 0;
            __syncwarp();
        }
        if (ok && leaf) {
#pragma unroll
            for (int k = 0; k < B; ++k) S.cand[ncand + __popc(lb & lt)][k] = ch.p[k];
        }
        ncand += nl;
        leaves += nl;
        if (ok && !leaf) ns[base + __popc(ib & lt)] = ch;
        nn = base + __popc(ib);
        __syncwarp();
        if (nn + 32 > P.node_cap) {
            if (lane == 0) atomicOr(P.error_flag, 2);
            break;
        }
    }
    if (ncand > 0) sigma_verify<B, MT>(C, t, ncand);
    C.add(W_SIGMA_LEAVES, leaves);
    C.add(W_SIGMA_NODES, nodes);
}

template <int B, int MT>
__device__ void sigma_dfs(SCtx<B, MT>& C, int j0) {
    const int t = C.P->t;
    SigmaWarp& S = *C.S;
    if (C.lane == 0) {
        S.iter[1] = j0;
        S.iter_end[1] = j0 + 1;
    }
    __syncwarp();
    int k = 1;
    while (k >= 1) {
        const LevelMeta& L = S.lev[k];
        const int it = S.iter[k];
        if (it >= S.iter_end[k]) {
            --k;
            continue;
        }
        const uint32_t u = C.entries(k)[L.start[L.branch] + it];
        __syncwarp();
        if (C.lane == 0) {
            S.iter[k] = it + 1;
            S.stack_id[k] = u;
        }
        __syncwarp();
        if (!sigma_push<B, MT>(C, k)) continue;
        if (k + 1 == t) {
            sigma_enumerate<B, MT>(C, t);
        } else {
            ++k;
            if (C.lane == 0) {
                S.iter[k] = 0;
                S.iter_end[k] = S.lev[k].cnt[S.lev[k].branch];
            }
            __syncwarp();
        }
    }
}

template <int B, int MT>
__global__ void __launch_bounds__(512, 1) sigma_search_kernel(const __grid_constant__ SigmaParams P) {
    extern __shared__ __align__(16) uint8_t sigma_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    SCtx<B, MT> C;
    C.P = &P;
    C.S = reinterpret_cast<SigmaWarp*>(sigma_smem) + warp;
    C.lane = lane;
    const size_t gw = static_cast<size_t>(blockIdx.x) * nwarps + warp;
    uint32_t* scratch = P.scratch + gw * P.scratch_words;
    C.lvl = scratch;
    C.nodes = reinterpret_cast<SigmaNode*>(scratch + static_cast<size_t>(P.t > 1 ? P.t - 1 : 0) * P.level_cap);
    SigmaWarp& S = *C.S;
    if (lane < W_SIGMA_N) S.ctr[lane] = 0;
    __syncwarp();
    const unsigned long long nstatic = static_cast<unsigned long long>(P.task_base[P.nanchors]);
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(P.next_task, 1ull);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= nstatic) break;
        int lo = 0, hi = P.nanchors - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (static_cast<unsigned long long>(P.task_base[mid]) <= idx) lo = mid;
            else hi = mid - 1;
        }
        C.l1 = P.l1_entries + static_cast<size_t>(lo) * P.K;
        const uint32_t* srcm = reinterpret_cast<const uint32_t*>(P.l1_meta + lo);
        uint32_t* dstm = reinterpret_cast<uint32_t*>(&S.lev[1]);
        for (int x = lane; x < static_cast<int>(sizeof(LevelMeta) / 4); x += 32) dstm[x] = srcm[x];
        if (lane == 0) S.stack_id[0] = static_cast<uint32_t>(P.anchor_off[lo]);
        __syncwarp();
        const int j = static_cast<int>(idx - static_cast<unsigned long long>(P.task_base[lo]));
        if (P.t == 1) {
            if (j == 0) sigma_enumerate<B, MT>(C, 1);
        } else {
            sigma_dfs<B, MT>(C, j);
        }
    }
    __syncwarp();
    if (lane == 0) {
        const int map[W_SIGMA_N] = {C_PUSHES, C_VIABLE, C_SLOTS, C_TUPLES, C_LEAVES, C_EMITTED, C_VCMP, C_NODES};
#pragma unroll
        for (int i = 0; i < W_SIGMA_N; ++i) atomicAdd(P.counters + map[i], S.ctr[i]);
    }
}

template <int B>
__global__ void reverify_sigma_kernel(const LmerS<B>* __restrict__ table, int n, int w, int l, int d,
                                      const unsigned long long* __restrict__ keys, long long count, int* fail) {
    const long long i = blockIdx.x;
    if (i >= count) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __shared__ int ok_rows;
    if (threadIdx.x == 0) ok_rows = 0;
    __syncthreads();
    LmerS<B> c;
#pragma unroll
    for (int k = 0; k < B; ++k) c.p[k] = 0u;
    const unsigned long long klo = keys[2 * i], khi = keys[2 * i + 1];
    for (int p = 0; p < l; ++p) {
        const int sh = B * (l - 1 - p);
        unsigned long long v = sh >= 64 ? (khi >> (sh - 64)) : ((klo >> sh) | (sh + B > 64 ? khi << (64 - sh) : 0ull));
        const int code = static_cast<int>(v & ((1ull << B) - 1));
#pragma unroll
        for (int k = 0; k < B; ++k) c.p[k] |= static_cast<uint32_t>((code >> k) & 1) << p;
    }
    for (int r = warp; r < n; r += nw) {
        bool hit = false;
        for (int base = 0; base < w && !hit; base += 32) {
            const int o = base + lane;
            hit = __any_sync(0xffffffffu, o < w && sdist<B>(c, ldt<B>(table, r * w + o)) <= d);
        }
        if (hit && lane == 0) atomicAdd(&ok_rows, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0 && ok_rows != n) atomicOr(fail, 1);
}

}  // namespace

size_t sigma_lmer_bytes(int B) { return 4u * static_cast<size_t>(B); }
size_t sigma_node_bytes() { return sizeof(SigmaNode); }
size_t sigma_warp_smem() { return (sizeof(SigmaWarp) + 15) / 16 * 16; }

#define PMS8G_SIGMA_B(X) X(3) X(4) X(5)

cudaError_t launch_encode_sigma(int B, const uint8_t* codes, int n, int m, int l, int w, int sigma, void* table,
                                int* err, cudaStream_t s) {
    const int K = n * w;
    const int blocks = (K + 255) / 256;
#define PMS8G_E(BB)                                                                                          \
    if (B == BB) {                                                                                           \
        encode_sigma_kernel<BB><<<blocks, 256, 0, s>>>(codes, n, m, l, w, sigma, static_cast<LmerS<BB>*>(table), \
                                                       err);                                                 \
        return cudaGetLastError();                                                                           \
    }
    PMS8G_SIGMA_B(PMS8G_E)
#undef PMS8G_E
    return cudaErrorInvalidValue;
}

cudaError_t launch_rowbuild_sigma(int B, const void* table, int n, int w, int d, int K, const int32_t* anchor_off,
                                  int nanchors, uint32_t* l1_entries, LevelMeta* l1_meta, unsigned long long* counters,
                                  cudaStream_t s) {
    if (nanchors <= 0) return cudaSuccess;
#define PMS8G_R(BB)                                                                                            \
    if (B == BB) {                                                                                             \
        rowbuild_sigma_kernel<BB><<<nanchors, 256, 0, s>>>(static_cast<const LmerS<BB>*>(table), n, w, d, K,  \
                                                            anchor_off, nanchors, l1_entries, l1_meta, counters); \
        return cudaGetLastError();                                                                             \
    }
    PMS8G_SIGMA_B(PMS8G_R)
#undef PMS8G_R
    return cudaErrorInvalidValue;
}

cudaError_t launch_search_sigma(int B, const SigmaParams& P, int blocks, int warps, cudaStream_t s) {
    const int mt = P.t < 2 ? 2 : P.t;
    const size_t smem = sigma_warp_smem() * warps;
#define PMS8G_S(BB, M)                                                                                      \
    if (B == BB && mt == M) {                                                                               \
        cudaError_t e = cudaFuncSetAttribute(sigma_search_kernel<BB, M>,                                    \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)); \
        if (e != cudaSuccess) return e;                                                                     \
        sigma_search_kernel<BB, M><<<blocks, warps * 32, smem, s>>>(P);                                     \
        return cudaGetLastError();                                                                          \
    }
#define PMS8G_SB(BB) PMS8G_S(BB, 2) PMS8G_S(BB, 3) PMS8G_S(BB, 4) PMS8G_S(BB, 5) PMS8G_S(BB, 6)
    PMS8G_SIGMA_B(PMS8G_SB)
#undef PMS8G_SB
#undef PMS8G_S
    return cudaErrorInvalidValue;
}

cudaError_t launch_reverify_sigma(int B, const void* table, int n, int w, int l, int d,
                                  const unsigned long long* keys, long long count, int* fail, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
#define PMS8G_V(BB)                                                                                             \
    if (B == BB) {                                                                                              \
        reverify_sigma_kernel<BB><<<static_cast<unsigned>(count), 256, 0, s>>>(                                \
            static_cast<const LmerS<BB>*>(table), n, w, l, d, keys, count, fail);                              \
        return cudaGetLastError();                                                                              \
    }
    PMS8G_SIGMA_B(PMS8G_V)
#undef PMS8G_V
    return cudaErrorInvalidValue;
}

}  // namespace pms8g
