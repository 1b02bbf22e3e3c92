// pms8g_search.cu — K4: the persistent sm_100a search kernel.
//
// One warp = one depth-first worker. Work arrives as tasks:
//   static  (S1 l-mer a, depth-1 branch j): push the j-th l-mer u of a's
//           branching row, then search below it (run_anchored + recurse,
//           src/solver.cpp:406-432, with the first level unrolled);
//   dynamic (a, stack prefix, branch range at level k) or (a, k-tuple, DFS
//           nodes): donated by a busy warp while other warps wait, rebuilt by
//           the receiver by replaying the prefix pushes.
// Per push, the warp filters every remaining row with the pair rule and
// PMS8's Theorem-1 triple rule (MotifSearch::push, src/solver.cpp:245-337).
// At the switch depth t it enumerates the tuple's common d-neighbourhood
// (NeighborhoodEnumerator, src/neighborhood.cpp:164-270) 16 nodes x 4
// symbols per round and verifies candidates breadth-first against the
// remaining rows (verify_candidate, src/solver.cpp:344-362), smallest row
// first, compacting survivors between rows.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "pms8g_common.cuh"
#include "pms8g_device.cuh"
#include "pms8g_launch.h"

namespace pms8g {

using namespace dev;

namespace {

// per-rule rejection counters of the push filters (pair_rej, tri_rej,
// cons_rej): diagnostics builds only (three adds per slot and 15 shuffles per
// push otherwise)
#ifdef PMS8G_LEVELSTATS
#define PMS8G_REJ(x) (x)
#else
#define PMS8G_REJ(x) ((void)0)
#endif

// push filters of builds with t >= this run Theorem 1 in a rolled loop over
// the older members (t >= 4: the members live in shared memory)
#ifndef PMS8G_ROLLED_MT
#define PMS8G_ROLLED_MT 4
#endif

// push filters of builds with t >= this queue the survivors of the cheap rules
// and run Theorem 1 on full warps of them (WarpFixed::qe)
#ifndef PMS8G_QUEUE_MT
#define PMS8G_QUEUE_MT 5
#endif

// push filters of builds with t >= this stop at the first emptied row
#ifndef PMS8G_EARLYOUT_MT
#define PMS8G_EARLYOUT_MT 5
#endif

template <int W>
struct Node {
    Lmer<W> c;    // candidate prefix planes
    uint32_t rA;  // budgets of members 0..3, biased by +64, one byte each
    uint32_t rB;  // budgets of members 4..6 (bytes 0..2); prefix length p in byte 3
};

extern __shared__ __align__(16) uint8_t dyn_smem[];

template <int W>
struct NodeSmem {
    static constexpr int N = W == 1 ? 128 : 64;  // power of two
};

enum WCtr { W_PUSH, W_VIABLE, W_SLOTS, W_TUPLES, W_LEAVES, W_EMIT, W_VCMP, W_NODES, W_PAIRREJ, W_TRIREJ, W_TASKS,
            W_DONATED, W_REPLAYS, W_CLKF, W_CLKP, W_CONSREJ, W_ROUNDS, W_N };

// Wait state of a warp's claim loop (lane 0 only; shared memory, so the
// persistent loop keeps no registers for it).
struct WaitState {
    int waiting;
    unsigned int backoff;
    long long wait_t0, beat_t0;
    unsigned long long beat;
    unsigned long long chunk_next, chunk_end;  // static tasks claimed in a chunk, not yet started
};

struct WarpFixed {
    int iter[MAXT + 1];
    int iter_end[MAXT + 1];
    uint32_t stack_id[MAXT];
    uint32_t cnt_by_row[MAXN];
    uint8_t vorder[MAXN];
    uint8_t perm[64];            // enumeration depth -> l-mer position of the current tuple
    unsigned long long diag[5];  // diagnostics: counters at task start + start time (ns)
    TaskHeader task;
    unsigned long long ctr[W_N];  // per-warp counters (lane 0 updates)
    uint32_t lazy_mask;          // rows of the lazy level already filtered
    int lazy_level;              // level whose rows are filtered on demand (0: none)
    WaitState wait;              // claim loop state (lane 0)
    // push filters of the t >= 4 builds: the older stack members, their
    // mismatch masks against the new top and its distances to them (read by
    // broadcast LDS in the filter loop instead of pinning ~40 registers)
    uint32_t fsm[MAXT][4];
    uint32_t fmiu[MAXT][2];
    int32_t fhs[MAXT];
    // consensus row rule: slot k = masks of stack[0..k-1] (cons_prepare);
    // 12-word (16-byte aligned) slots so a filter loads them with LDS.128
    __align__(16) uint32_t cons[2][12];  // slot 0: the push filter's pass; slot 1: the lazy level's rows
    // LAST member: a search with switch depth t allocates lev[0..t] only
    // (warp_fixed_bytes), so the shallow one-word builds keep 16 warps next
    // to the l-mer table in shared memory
    LevelMeta lev[MAXT + 1];
};

// Push filters of the t >= PMS8G_QUEUE_MT builds: survivors of the cheap
// rules (consensus, pair) wait here, with their l-mers, until 32 of them run
// the Theorem-1 triple rule together (circular, 64 entry ids; the l-mers are
// re-read from the table, L1-resident by then). Placed after the warp's
// WarpFixed in those builds only.
struct PushQueue {
    uint32_t qe[64];
};

__host__ __device__ constexpr int warp_fixed_bytes(int t) {
    return (static_cast<int>(offsetof(WarpFixed, lev)) + (t + 1) * static_cast<int>(sizeof(LevelMeta)) + 15) / 16 * 16;
}


// Member cache (t >= 4 builds): S.fsm[i] holds the l-mer of stack[i] while it
// is on the stack - written when the member is set (begin_anchor, a received
// task's prefix) or first pushed (StackSet::load, lazy_push), so the per-push
// set-up reads the older members from shared memory instead of the table.
template <int W>
__device__ __forceinline__ void cache_member(WarpFixed& S, int i, const Lmer<W>& x) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
        S.fsm[i][2 * w] = x.h[w];
        S.fsm[i][2 * w + 1] = x.o[w];
    }
}
template <int W>
__device__ __forceinline__ Lmer<W> cached_member(const WarpFixed& S, int i) {
    Lmer<W> x;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        x.h[w] = S.fsm[i][2 * w];
        x.o[w] = S.fsm[i][2 * w + 1];
    }
    return x;
}

constexpr int MAXCH = 5;  // candidate chunks of 32 held in registers by verify

// Read-only table load through the non-coherent L1 path (global tables).
template <int W>
__device__ __forceinline__ Lmer<W> ldg_lmer(const Lmer<W>* p) {
    Lmer<W> x;
    if constexpr (W == 2) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
        x.h[0] = v.x;
        x.h[W - 1] = v.y;
        x.o[0] = v.z;
        x.o[W - 1] = v.w;
    } else {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
        x.h[0] = v.x;
        x.o[0] = v.y;
    }
    return x;
}


// Where the l-mer table lives. One-word l-mers (8 B) are staged in every
// CTA's shared memory (94 KB for n=20, m=600). Two-word l-mers (16 B: 176 KB
// for (50,21)) would leave room for 7 warps per SM, so their table stays in
// global memory, L2-resident and read through L1 with 16 warps per SM:
// measured (50,21) 617 ms per 12-S1-l-mer sample, against 634 ms with the
// table split over 2-CTA clusters and read through DSMEM, and 3.3x slower
// with 7 warps. One-word instances whose table does not fit
// shared memory run the two-word build (upper words zero).
template <int W>
constexpr bool kGlobalTable = W == 2;

template <int W, int MT>
struct WarpCtx {
    const SearchParams* P;
    uint32_t off_S, off_thr, off_cand, off_nodes;  // byte offsets into the dynamic shared memory
    Node<W>* node_glob;
    uint32_t* lvl_glob;
    const uint32_t* l1;  // level-1 entries of the current anchor
    int anchor;          // anchor index of the current task
    int lane;
    int pushes_since_check;
    unsigned int checks;  // starvation checks made (lane 0; heartbeat pacing)
    const Lmer<W>* gt;  // two-word builds: the table in global memory
    uint8_t* thr_glob;  // t >= 5 builds: enumeration tables in global scratch
    // shared-memory views derived from the extern __shared__ symbol, so every
    // access compiles to LDS/STS rather than generic LD/ST
    __device__ __forceinline__ const Lmer<W>* T() const { return reinterpret_cast<const Lmer<W>*>(dyn_smem); }
    // l-mer `id` of the table (one-word: LDS.64; two-word: LDG.128 via L1)
    __device__ __forceinline__ Lmer<W> lmer(uint32_t id) const {
        if constexpr (kGlobalTable<W>) return ldg_lmer<W>(gt + id);
        else return T()[id];
    }
    __device__ __forceinline__ WarpFixed* S() const { return reinterpret_cast<WarpFixed*>(dyn_smem + off_S); }
    // enumeration tables: shared memory, or (t >= 5 builds, where few tuples
    // are ever enumerated) the warp's global scratch
    __device__ __forceinline__ uint8_t* thr() const {
        if constexpr (MT >= 5) return thr_glob;
        else return dyn_smem + off_thr;
    }
    __device__ __forceinline__ Lmer<W>* cand() const { return reinterpret_cast<Lmer<W>*>(dyn_smem + off_cand); }
    __device__ __forceinline__ Node<W>* node_smem() const { return reinterpret_cast<Node<W>*>(dyn_smem + off_nodes); }
    __device__ __forceinline__ void add(int i, unsigned long long v) {
        if (lane == 0) S()->ctr[i] += v;
    }
};

// The table location of a context in registers, for hot loops (the context
// itself lives in local memory across the noinline calls).
template <int W>
struct TableRef {
    const Lmer<W>* gt;  // two-word builds
    __device__ __forceinline__ Lmer<W> get(uint32_t id) const {
        if constexpr (kGlobalTable<W>) return ldg_lmer<W>(gt + id);
        else return reinterpret_cast<const Lmer<W>*>(dyn_smem)[id];
    }
};

template <int W, int MT>
__device__ __forceinline__ TableRef<W> table_ref(const WarpCtx<W, MT>& C) {
    TableRef<W> t;
    t.gt = C.gt;
    return t;
}

// generic (non-SWAR) enumeration tables at the start of the thr region:
// eq[64] (members holding each symbol per position), cons[68] (consensus
// suffix bound), then the pair/triple thresholds
constexpr int GEN_TBL_BYTES = 64 * 4 + 68 + 4;
template <int W, int MT>
__device__ __forceinline__ uint32_t* gen_eq(const WarpCtx<W, MT>& C) {
    return reinterpret_cast<uint32_t*>(C.thr());
}
template <int W, int MT>
__device__ __forceinline__ uint8_t* gen_cons(const WarpCtx<W, MT>& C) {
    return C.thr() + 64 * 4;
}

template <int W, int MT>
__device__ __forceinline__ uint32_t* level_entries(WarpCtx<W, MT>& C, int k) {
    return k == 1 ? const_cast<uint32_t*>(C.l1) : C.lvl_glob + static_cast<size_t>(k - 2) * C.P->level_cap;
}

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ unsigned int ld_volatile(const unsigned int* p) {
    return *reinterpret_cast<const volatile unsigned int*>(p);
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Record a failure and the S1 offset of the subproblem it happened in (the
// first failure wins), so the host can name it like run_parallel does
// (src/parallel.cpp:66-86). error_flag[1] = S1 offset + 1 (0: none).
template <int W, int MT>
__device__ __forceinline__ void raise_error(const WarpCtx<W, MT>& C, int bit) {
    atomicOr(C.P->error_flag, bit);
    atomicCAS(C.P->error_flag + 1, 0, C.P->anchor_off[C.anchor] + 1);
}

// Schedule-shaking test hook (run_parallel's jitter, src/parallel.cpp:57-65):
// sleep a seeded pseudo-random 0..jitter_ns ns (out of line: it must not cost
// the persistent loop registers).
__device__ __noinline__ void jitter_sleep(const SearchParams& P, unsigned long long key) {
    unsigned long long z = P.jitter_seed + 0x9E3779B97F4A7C15ull * key;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    unsigned long long ns = (z ^ (z >> 31)) % (P.jitter_ns + 1);
    while (ns > 0) {
        const unsigned int step = static_cast<unsigned int>(ns < 1000000ull ? ns : 1000000ull);
        __nanosleep(step);
        ns -= step;
    }
}

// The tuple size of a build: builds are specialised on the switch depth
// (launch_search picks MT = max(2, t)), so t == MT whenever MT >= 3 and only
// the MT = 2 build sees two sizes (t = 1, 2). Folding t into a constant drops
// the per-member predicates and the code of the smaller sizes.
template <int MT>
__device__ __forceinline__ int tuple_size(int t) {
    return MT >= 3 ? MT : t;
}

// ---------------------------------------------------------------- static tasks
// Static tasks come from the device-local counter, or (multi-GPU) from the
// shared queue counter every rank claims from over NVLink. The shared counter
// carries an epoch (one per run, advanced in the same order on every rank):
// a run that finds an older epoch opens its own at task 0, one that finds a
// newer epoch knows every task of its run was claimed already (a rank only
// moves on once the previous run's counter was exhausted), so the counter
// never needs a reset between runs.
__device__ __forceinline__ bool statics_left(const SearchParams& P, unsigned long long nstatic) {
    if (!P.gqueue) return ld_volatile(&P.qs->static_next) < nstatic;
    const unsigned long long v = ld_relaxed_sys(P.gqueue);
    const unsigned long long ep = v >> GQ_SHIFT;
    return ep < P.gepoch || (ep == P.gepoch && (v & GQ_MASK) < nstatic);
}

// Claims static tasks [idx, idx + n). From the shared cross-GPU counter a
// warp takes a chunk of up to P.claim_chunk tasks per CAS while more than
// P.chunk_until tasks remain (far from the tail, where imbalance costs
// nothing and every CAS is an NVLink round trip), then one at a time.
__device__ __forceinline__ bool claim_static(const SearchParams& P, unsigned long long nstatic,
                                             unsigned long long& idx, unsigned int& n) {
    n = 1;
    if (!P.gqueue) {
        idx = atomicAdd(&P.qs->static_next, 1ull);
        return idx < nstatic;
    }
    unsigned long long v = ld_relaxed_sys(P.gqueue);
    for (;;) {
        const unsigned long long ep = v >> GQ_SHIFT;
        unsigned long long cnt = v & GQ_MASK, nv;
        if (ep > P.gepoch) return false;
        if (ep < P.gepoch) {
            cnt = 0;  // this run's epoch opens at task 0
        } else if (cnt >= nstatic) {
            return false;
        }
        const unsigned long long left = nstatic - cnt;
        n = left > static_cast<unsigned long long>(P.chunk_until) ? static_cast<unsigned int>(P.claim_chunk) : 1u;
        if (n > left) n = static_cast<unsigned int>(left);
        nv = (P.gepoch << GQ_SHIFT) | (cnt + n);
        idx = cnt;
        const unsigned long long old = atomicCAS_system(P.gqueue, v, nv);
        if (old == v) return true;
        v = old;
    }
}

// Stack consensus bound as a row filter. m l-mers have a common d-neighbour
// only if their consensus cost (sum over columns of m minus the most frequent
// symbol's count) is at most m*d; the witness v of a motif in any remaining
// row forms such a set with the stack, so a push may drop every row entry v
// for which stack + v fails the bound — a sound rule like Theorem 1, applied
// by the push filters next to the pair and triple rules once stack + v has 4+
// members (for 3 members Theorem 1 is exact). Incremental form: for the k
// members stack[0..k-1], G[c] = positions where symbol c is a plurality
// symbol (count == the column maximum M) and need = (k+1)(l-d) - sum M,
// computed once per push (cons_prepare, slot k); then v passes iff
// popc(sum over c of G[c] & [v == c]) >= need (adding v raises a column's
// maximum exactly where v holds a plurality symbol). Kept in the warp's
// shared memory (read by broadcast LDS in the filter loops), 4W+1 words per
// slot.
template <int W, int MT>
__device__ __forceinline__ uint32_t* cons_slot(const WarpCtx<W, MT>& C, int k) {
    return C.S()->cons[k];
}

template <int W, int MT>
__device__ __noinline__ void cons_prepare(WarpCtx<W, MT>& C, int k, int slot_index) {
    // Lane c*W + w owns symbol c in word w (the slot's own index): it folds
    // the k members into ge[j] = positions where at least j of them hold c;
    // the column maxima come from an OR over the four symbol lanes of a word.
    const SearchParams& P = *C.P;
    const WarpFixed& S = *C.S();
    const int l = P.l, lane = C.lane;
    uint32_t* slot = cons_slot<W, MT>(C, slot_index);
    const int w = lane % W, c = lane / W;
    const int nb = min(32, l - 32 * w);
    uint32_t lm = nb >= 32 ? 0xffffffffu : (nb <= 0 ? 0u : ((1u << nb) - 1u));
    if (lane >= 4 * W) lm = 0u;  // idle lanes carry zeros through the exchanges
    const uint32_t fh = (c & 2) ? 0u : 0xffffffffu, fo = (c & 1) ? 0u : 0xffffffffu;
    uint32_t ge[MT + 1];
    ge[0] = lm;
#pragma unroll
    for (int j = 1; j <= MT; ++j) ge[j] = 0u;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        if (i < k) {
            const Lmer<W> x = cached_member<W>(S, i);  // member cache: a broadcast LDS
            const uint32_t hw = (W == 2 && w) ? x.h[W - 1] : x.h[0];
            const uint32_t ow = (W == 2 && w) ? x.o[W - 1] : x.o[0];
            const uint32_t e = (hw ^ fh) & (ow ^ fo) & lm;  // positions where member i holds c
            // (after members 0..i at most i + 1 of them hold c)
#pragma unroll
            for (int j = MT; j >= 1; --j)
                if (j <= i + 1) ge[j] |= ge[j - 1] & e;
        }
    }
    uint32_t g = 0u, mg_above = 0u;
    int sum_m = 0;
#pragma unroll
    for (int j = MT; j >= 1; --j) {
        if (j <= k) {  // warp-uniform
            uint32_t mg = ge[j];  // -> positions whose column maximum is >= j
            mg |= __shfl_xor_sync(0xffffffffu, mg, W);
            mg |= __shfl_xor_sync(0xffffffffu, mg, 2 * W);
            sum_m += __popc(mg);
            g |= mg & ~mg_above & ge[j];  // maximum == j and c reaches it
            mg_above = mg;
        }
    }
    if (lane < 4 * W) slot[lane] = g;
    int tot = __shfl_sync(0xffffffffu, sum_m, 0);
    if constexpr (W == 2) tot += __shfl_sync(0xffffffffu, sum_m, 1);
    if (lane == 0) slot[4 * W] = static_cast<uint32_t>((k + 1) * (l - P.d) - tot);
    __syncwarp();
}

// A view of one slot for a filter pass (the masks stay in shared memory:
// pinned in registers they would be spilled around the filter loop).
template <int W>
struct ConsMasks {
    const uint32_t* slot;
};

template <int W, int MT>
__device__ __forceinline__ ConsMasks<W> load_cons(const WarpCtx<W, MT>& C, int k) {
    return ConsMasks<W>{cons_slot<W, MT>(C, k)};
}

template <int W>
__device__ __forceinline__ bool cons_pass(const ConsMasks<W>& cm, const Lmer<W>& x) {
    // the 4W masks and `need` as LDS.128/LDS.64 broadcasts
    uint32_t g[4 * W + 1];
    const uint4* v = reinterpret_cast<const uint4*>(cm.slot);
    if constexpr (W == 2) {
        const uint4 a = v[0], b = v[1];
        g[0] = a.x, g[1] = a.y, g[2] = a.z, g[3] = a.w, g[4] = b.x, g[5] = b.y, g[6] = b.z, g[7] = b.w;
        g[8] = cm.slot[8];
    } else {
        const uint4 a = v[0];
        g[0] = a.x, g[1] = a.y, g[2] = a.z, g[3] = a.w;
        g[4] = cm.slot[4];
    }
    int matches = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        const uint32_t h = x.h[w], o = x.o[w];
        matches += __popc((g[0 * W + w] & ~(h | o)) | (g[1 * W + w] & o & ~h) | (g[2 * W + w] & h & ~o) |
                          (g[3 * W + w] & h & o));
    }
    return matches >= static_cast<int>(g[4 * W]);
}

// Pushes whose filter applies the consensus row rule: stack + v has 4+
// members (k >= 2), full pruning, t >= 4 builds.
template <int MT>
__device__ __forceinline__ bool cons_rows_at(const SearchParams& P, int k) {
    return MT >= 4 && P.cons_rows && k >= 2;
}

// One claim attempt by lane 0: 0 static task, 1 dynamic task (idx set),
// 2 terminate, -1 nothing yet (backed off). Protocol in DESIGN.md §4.
__device__ __noinline__ int claim_task(const SearchParams& P, unsigned long long nstatic, WaitState& ws,
                                       unsigned long long& idx) {
    QueueState* qs = P.qs;
    const unsigned long long qcap = static_cast<unsigned long long>(P.qcap);
    int kind = -1;
    if (ws.chunk_next < ws.chunk_end) {
        // the rest of this warp's claimed chunk (already counted as busy)
        idx = ws.chunk_next++;
        return 0;
    }
    const bool have_static = statics_left(P, nstatic);
    const unsigned long long h0 = ld_volatile(&qs->head);
    const bool have_dyn = ld_volatile(&P.qstate[h0 % qcap]) == 2u * static_cast<unsigned int>(h0 / qcap) + 1u;
    if (have_static || have_dyn) {
        // announce before claiming so that no waiter can observe
        // busy == 0 while a claimed task is still unannounced
        atomicAdd(&qs->busy, 1u);
        unsigned int n = 1;
        if (have_static && claim_static(P, nstatic, idx, n)) {
            kind = 0;
            atomicAdd(P.counters + C_STATIC, static_cast<unsigned long long>(n));
            if (n > 1) {
                // the chunk's later tasks stay announced until they are done
                atomicAdd(&qs->busy, n - 1);
                ws.chunk_next = idx + 1;
                ws.chunk_end = idx + n;
            }
        }
        if (kind < 0) {
            const unsigned long long h = ld_volatile(&qs->head);
            if (ld_volatile(&P.qstate[h % qcap]) == 2u * static_cast<unsigned int>(h / qcap) + 1u &&
                atomicCAS(&qs->head, h, h + 1) == h) {
                kind = 1;
                idx = h;
                __threadfence();
            }
        }
        if (kind < 0) atomicSub(&qs->busy, 1u);
    }
    if (kind < 0) {
        if (!ws.waiting) {
            atomicAdd(&qs->waiting, 1u);
            ws.waiting = 1;
            ws.wait_t0 = ws.beat_t0 = clock64();
            ws.beat = ld_volatile(&qs->heartbeat);
            ws.backoff = 128;
        }
        const unsigned long long b = ld_volatile(&qs->heartbeat);
        if (b != ws.beat) {  // somebody is still working: not stuck
            ws.beat = b;
            ws.beat_t0 = clock64();
        }
        if (ld_volatile(&qs->busy) == 0u && ld_volatile(&qs->head) >= ld_volatile(&qs->alloc) &&
            !statics_left(P, nstatic)) {
            kind = 2;
        } else if (clock64() - ws.beat_t0 > (1ll << 37)) {
            // watchdog: ~70 s with busy warps but no heartbeat (they beat
            // every few starvation checks while others wait): a lost task
            atomicOr(P.error_flag, 8);
            kind = 2;
        } else {
            // idle warps back off so their polling does not steal issue
            // slots and L2 bandwidth from the busy ones
            __nanosleep(ws.backoff);
            ws.backoff = min(ws.backoff * 2, 8192u);
        }
    }
    if (kind >= 0 && ws.waiting) {
        atomicSub(&qs->waiting, 1u);
        ws.waiting = 0;
        atomicAdd(P.counters + C_IDLE, static_cast<unsigned long long>(clock64() - ws.wait_t0));
    }
    return kind;
}

// The older stack members s_i (i < k) of a push of u = stack[k], for the
// Theorem-1 triple rule: Hd(v, s_i), Hd(s_i, u) and the all-distinct count
// n4 = popc(mism(v,s_i) & mism(v,u) & mism(s_i,u)) give the triple's
// consensus cost Cd3 = (h_vi + h_vu + h_iu + n4) / 2 <= 3d
// (MotifSearch::push, src/solver.cpp:302-319, with its sum + min <= 6d
// shortcut). Builds with t <= 3 keep the members in registers; t >= 4 builds
// keep them in shared memory (broadcast reads; most slots never get here).
template <int W, int MT>
struct StackSet {
    static constexpr bool kSmem = MT >= 4;
    Lmer<W> sm[kSmem ? 1 : MT];
    Mask<W> miu[kSmem ? 1 : MT];
    int hs[kSmem ? 1 : MT];
    const WarpFixed* S;

    __device__ __forceinline__ void load(const WarpCtx<W, MT>& C, int k, const Lmer<W>& U) {
        const TableRef<W> tr = table_ref<W, MT>(C);
        WarpFixed* Sw = C.S();
        S = Sw;
        if constexpr (kSmem) {
            if (C.lane < k) {
                const Lmer<W> x = cached_member<W>(*Sw, C.lane);
                const Mask<W> m = mism<W>(x, U);
#pragma unroll
                for (int w = 0; w < W; ++w) Sw->fmiu[C.lane][w] = m.w[w];
                Sw->fhs[C.lane] = popcm<W>(m);
            } else if (C.lane == k) {
                cache_member<W>(*Sw, k, U);  // the new top joins the member cache
            }
            __syncwarp();
        } else {
#pragma unroll
            for (int i = 0; i < MT; ++i)
                if (i < k) {
                    sm[i] = tr.get(Sw->stack_id[i] & ID_MASK);
                    miu[i] = mism<W>(sm[i], U);
                    hs[i] = popcm<W>(miu[i]);
                }
        }
    }

    __device__ __forceinline__ bool triple_ok(int i, const Lmer<W>& V, const Mask<W>& mu, int hvu,
                                              int six_d) const {
        Lmer<W> x;
        Mask<W> mi_u;
        int h_iu;
        if constexpr (kSmem) {
#pragma unroll
            for (int w = 0; w < W; ++w) {
                x.h[w] = S->fsm[i][2 * w];
                x.o[w] = S->fsm[i][2 * w + 1];
                mi_u.w[w] = S->fmiu[i][w];
            }
            h_iu = S->fhs[i];
        } else {
            x = sm[i];
            mi_u = miu[i];
            h_iu = hs[i];
        }
        const Mask<W> mi = mism<W>(V, x);
        const int hvi = popcm<W>(mi);
        const int sum = hvi + hvu + h_iu;
        if (sum > six_d) return false;
        const int mn = min(min(hvi, hvu), h_iu);
        return sum + mn <= six_d || sum + popc_and3<W>(mi, mu, mi_u) <= six_d;
    }
};

// ---------------------------------------------------------------- push filter
// Push of u = stack[k] onto a stack of k members: filter level k (minus its
// branching row) into level k+1. Returns viable (no remaining row emptied).
template <int W, int MT>
__device__ __noinline__ bool filter_push(WarpCtx<W, MT>& C, int k) {
    const SearchParams& P = *C.P;
    const int lane = C.lane;
    WarpFixed& S = *C.S();
    LevelMeta& Ls = S.lev[k];
    LevelMeta& Ld = S.lev[k + 1];
    const uint32_t* src = level_entries<W, MT>(C, k);
    uint32_t* dst = level_entries<W, MT>(C, k + 1);
    const int d = P.d, six_d = 6 * d, two_d = 2 * d;
    const long long f0 = clock64();

    const TableRef<W> tr = table_ref<W, MT>(C);
    const int jb = Ls.branch;
    const int bstart = Ls.start[jb], bcnt = Ls.cnt[jb];
    const int n_iter = Ls.total - bcnt;
    const int nrows = Ls.nrows;
    // the next block's entries are loaded one iteration ahead (the level
    // entries stream from L2; this hides one load latency per block)
    const uint32_t un_iter = static_cast<uint32_t>(n_iter), ubstart = static_cast<uint32_t>(bstart),
                   ubcnt = static_cast<uint32_t>(bcnt);
    auto load_entry = [&](int f) -> uint32_t {
        const uint32_t uf = static_cast<uint32_t>(f);  // 32-bit unsigned index: one IMAD.WIDE.U32
        // past the end: row 0xFF (a row change after the last entry) with id 0,
        // so that the l-mer prefetch of a padding slot needs no select
        return uf < un_iter ? src[uf + (uf < ubstart ? 0u : ubcnt)] : 0xFF000000u;
    };
    // software pipeline: entries two blocks ahead, their l-mers (table reads)
    // one block ahead (t >= 4 builds; the t <= 3 builds keep the one-block
    // entry prefetch: their register budget goes to the enumeration and
    // verification loops). The first loads are issued before the per-push
    // set-up below (stack members, consensus masks), so their latency
    // overlaps it: most pushes at depth scan only a few blocks.
    constexpr bool kPipeV = MT >= 4;
    uint32_t e_next = load_entry(lane);
    uint32_t e_next2 = kPipeV ? load_entry(lane + 32) : 0u;
    const Lmer<W> U = tr.get(S.stack_id[k] & ID_MASK);
    Lmer<W> V_next;
    if constexpr (kPipeV) V_next = tr.get(e_next & ID_MASK);
    StackSet<W, MT> ss;
    ss.load(C, k, U);
    const bool cons = cons_rows_at<MT>(P, k);
    ConsMasks<W> cm;
    if (cons) {
        // a fixed slot: its address is the warp's base plus a constant (no
        // register or spill slot for it inside the filter loop)
        cons_prepare<W, MT>(C, k + 1, 0);
        cm = ConsMasks<W>{S.cons[0]};  // from the S view already live in the loop
    }
    if (lane < MAXN) S.cnt_by_row[lane] = 0;
    if (lane == 0) S.lazy_level = 0;
    __syncwarp();
    int out = 0;
    [[maybe_unused]] unsigned pair_rej = 0, tri_rej = 0, cons_rej = 0;
    // early exit on an emptied row (builds where non-viable pushes are common)
    constexpr bool kEarlyOut = MT >= PMS8G_EARLYOUT_MT;
#ifdef PMS8G_LEVELSTATS
    unsigned ls_cheap = 0, ls_blocks = 0;
#endif
    unsigned seg_kept = 0u;  // the row segment open at the block start kept an entry
    int n_done = n_iter;
    bool dead = false;
    // survivors of the cheap rules queue up (WarpFixed::qe/qv); Theorem 1
    // against the older members runs on 32 of them at a time, and the kept
    // ones are appended to the new level (flat order is preserved)
    constexpr bool kQueue = MT >= PMS8G_QUEUE_MT && StackSet<W, MT>::kSmem;
    PushQueue& Q = *reinterpret_cast<PushQueue*>(reinterpret_cast<uint8_t*>(&S) + warp_fixed_bytes(tuple_size<MT>(P.t)));
    int qh = 0, qn = 0;
    auto resolve = [&](int cntq) {
        const bool have = lane < cntq;
        uint32_t qe = 0u;
        bool kp = false;
        if (have) {
            const int qi = (qh + lane) & 63;
            qe = Q.qe[qi];
            Lmer<W> QV;
            QV = tr.get(qe & ID_MASK);
            const Mask<W> qmu = mism<W>(QV, U);
            const int qhvu = popcm<W>(qmu);
            kp = true;
            for (int i = 0; i < k; ++i)
                if (kp) kp = ss.triple_ok(i, QV, qmu, qhvu, six_d);
            PMS8G_REJ(tri_rej += !kp);
        }
        const unsigned b2 = __ballot_sync(0xffffffffu, kp);
        if (b2) {
            if (kp) dst[out + __popc(b2 & lanemask_lt())] = qe;
            out += __popc(b2);
            const uint32_t row = qe >> 24;
            const unsigned grp = __match_any_sync(0xffffffffu, row) & b2;
            if (kp && __ffs(grp) - 1 == lane) S.cnt_by_row[row] += static_cast<uint32_t>(__popc(grp));
        }
        __syncwarp();
        qh = (qh + cntq) & 63;
        qn -= cntq;
    };
    for (int base = 0; base < n_iter; base += 32) {
        const int f = base + lane;
        const bool valid = f < n_iter;
        const uint32_t e = e_next;
        Lmer<W> V;
        if constexpr (kPipeV) {
            V = V_next;
            e_next = e_next2;
            e_next2 = load_entry(f + 64);
            if (base + 32 < n_iter) V_next = tr.get(e_next & ID_MASK);
        } else {
            e_next = load_entry(f + 32);
            if (valid) V = tr.get(e & ID_MASK);
        }
        bool keep = false;
        Mask<W> mu;
        int hvu = 0;
        if (valid) {
            // the consensus rule first: at deep levels it rejects most slots
            keep = true;
            if (cons) {
                keep = cons_pass<W>(cm, V);
                PMS8G_REJ(cons_rej += !keep);
            }
            if (keep) {
                mu = mism<W>(V, U);
                hvu = popcm<W>(mu);
                keep = hvu <= two_d;
                PMS8G_REJ(pair_rej += !keep);
            }
        }
#ifdef PMS8G_LEVELSTATS
        ls_cheap += keep;
        ls_blocks += __any_sync(0xffffffffu, keep) ? 1u : 0u;
#endif
        if constexpr (kQueue) {
            const unsigned cb = __ballot_sync(0xffffffffu, keep);
            if constexpr (kEarlyOut) {
                // a row that ends in this block without a survivor of the
                // cheap rules makes the push non-viable: stop (at t >= 5 most
                // pushes end this way). `ends` marks the last entry of each
                // row segment; a carry chain over the non-end positions tells
                // per segment whether it kept anything. (Rows emptied by
                // Theorem 1 alone are found after the pass.)
                // Rows are contiguous, so a block holds a row end iff the next
                // block starts in another row than this one (the big rows of
                // depth 2 span ~6 blocks: most blocks skip the row logic).
                // (lane 0 holds both the block's first entry and the next
                // block's first entry: one vote instead of two broadcasts)
                const unsigned rowdiff = __ballot_sync(0xffffffffu, ((e_next ^ e) >> 24) != 0u);
                if (!(rowdiff & 1u)) {
                    seg_kept |= cb != 0u ? 1u : 0u;
                } else {
                    const uint32_t nxt_blk = __shfl_sync(0xffffffffu, e_next, 0);
                    const uint32_t nxt_lane = __shfl_down_sync(0xffffffffu, e, 1);
                    const uint32_t nxt = lane == 31 ? nxt_blk : nxt_lane;
                    const unsigned ends = __ballot_sync(0xffffffffu, valid && (nxt >> 24) != (e >> 24));
                    const unsigned balc = cb | seg_kept;
                    const unsigned mid = ~ends;
                    const unsigned nonempty = (((balc & mid) + mid) & ends) | (balc & ends);
                    if (ends & ~nonempty) {
                        n_done = min(base + 32, n_iter);
                        dead = true;
                        break;
                    }
                    if (ends) seg_kept = (ends >> 31) ? 0u : ((cb >> (32 - __clz(ends))) != 0u ? 1u : 0u);
                    else seg_kept |= cb != 0u ? 1u : 0u;
                }
            }
            if (cb) {
                if (keep) {
                    const int qi = (qh + qn + __popc(cb & lanemask_lt())) & 63;
                    Q.qe[qi] = e;
                }
                qn += __popc(cb);
                if (qn >= 32) {
                    __syncwarp();  // the queue stores above, before resolve reads them
                    resolve(32);
                }
            }
            continue;
        }
        if constexpr (MT >= 5) {
            // Theorem 1 against the older members: skipped by the whole warp
            // when no lane survived the cheap rules (most blocks at depth;
            // measured +3.5% on (50,21), -4% on the t = 4 builds, which keep
            // the unrolled form)
            if (__any_sync(0xffffffffu, keep)) {
                const bool before = keep;
                for (int i = 0; i < k; ++i)
                    if (keep) keep = ss.triple_ok(i, V, mu, hvu, six_d);
                PMS8G_REJ(tri_rej += before && !keep);
            }
        } else if constexpr (MT >= PMS8G_ROLLED_MT) {
#pragma unroll 1
            for (int i = 0; i < k; ++i) {
                if (keep) {
                    keep = ss.triple_ok(i, V, mu, hvu, six_d);
                    PMS8G_REJ(tri_rej += !keep);
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                if (i < k && keep) {
                    keep = ss.triple_ok(i, V, mu, hvu, six_d);
                    PMS8G_REJ(tri_rej += !keep);
                }
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if constexpr (kEarlyOut) {
            // a row that ends in this block without a survivor makes the push
            // non-viable: stop (at t >= 5 most pushes end this way). `ends`
            // marks the last entry of each row segment; a carry chain over the
            // non-end positions tells per segment whether it kept anything.
            const uint32_t nxt_blk = __shfl_sync(0xffffffffu, e_next, 0);
            const uint32_t nxt_lane = __shfl_down_sync(0xffffffffu, e, 1);
            const uint32_t nxt = lane == 31 ? nxt_blk : nxt_lane;
            const unsigned ends = __ballot_sync(0xffffffffu, valid && (nxt >> 24) != (e >> 24));
            const unsigned balc = bal | seg_kept;
            const unsigned mid = ~ends;
            const unsigned nonempty = (((balc & mid) + mid) & ends) | (balc & ends);
            if (ends & ~nonempty) {
                n_done = min(base + 32, n_iter);
                dead = true;
                break;
            }
            if (ends) seg_kept = (ends >> 31) ? 0u : ((bal >> (32 - __clz(ends))) != 0u ? 1u : 0u);
            else seg_kept |= bal != 0u ? 1u : 0u;
        }
        if (MT < 5 || bal) {  // warp-uniform: deep blocks without survivors write nothing
            if (keep) dst[out + __popc(bal & lanemask_lt())] = e;
            out += __popc(bal);
            // per-row kept counts: one leader lane per distinct row among the
            // kept entries (rows are contiguous segments: one or two per block)
            const uint32_t row = e >> 24;
            const unsigned grp = __match_any_sync(0xffffffffu, row) & bal;
            if (keep && __ffs(grp) - 1 == lane) S.cnt_by_row[row] += static_cast<uint32_t>(__popc(grp));
            __syncwarp();
        }
    }
    if constexpr (kQueue) {
        __syncwarp();
        if (!dead && qn > 0) resolve(qn);
    }
    __syncwarp();
    // an emptied row is detected after the pass (almost every push is viable,
    // so the pass rarely could have stopped early)
    C.add(W_PUSH, 1);
    C.add(W_SLOTS, static_cast<unsigned long long>(n_done));
#ifdef PMS8G_LEVELSTATS
    {
        unsigned pr = pair_rej, tr = tri_rej, cr = cons_rej;
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) {
            pr += __shfl_xor_sync(0xffffffffu, pr, sh);
            tr += __shfl_xor_sync(0xffffffffu, tr, sh);
            cr += __shfl_xor_sync(0xffffffffu, cr, sh);
        }
        C.add(W_PAIRREJ, pr);
        C.add(W_TRIREJ, tr);
        C.add(W_CONSREJ, cr);
    }
#endif
#ifdef PMS8G_LEVELSTATS
    {
        unsigned ch = ls_cheap;
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) ch += __shfl_xor_sync(0xffffffffu, ch, sh);
        if (lane == 0) {
            unsigned long long* q = P.counters + C_LVL0 + 6 * min(k, 7);
            atomicAdd(q + 0, 1ull);
            atomicAdd(q + 1, dead ? 1ull : 0ull);
            atomicAdd(q + 2, static_cast<unsigned long long>(n_done));
            atomicAdd(q + 3, static_cast<unsigned long long>(ch));
            atomicAdd(q + 4, static_cast<unsigned long long>(out));
            atomicAdd(q + 5, static_cast<unsigned long long>(ls_blocks));
        }
    }
#endif
    bool ok = !dead;
    if (ok) {
        const int nr2 = nrows - 1;
        int c = 0;
        uint8_t row = 0;
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
        if (__any_sync(0xffffffffu, lane < nr2 && c == 0)) {
            ok = false;
        } else {
            int key = lane < nr2 ? (c << 8) | lane : 0x7FFFFFFF;
            if (P.sort_rows) {
#pragma unroll
                for (int s = 16; s > 0; s >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, s));
            } else {
                key = __shfl_sync(0xffffffffu, key, 0);
            }
            if (lane < nr2) {
                Ld.start[lane] = static_cast<uint32_t>(incl - c);
                Ld.cnt[lane] = static_cast<uint32_t>(c);
                Ld.order[lane] = row;
            }
            if (lane == 0) {
                Ld.nrows = nr2;
                Ld.total = out;
                Ld.branch = key & 0xFF;
                Ld.viable = 1;
            }
            C.add(W_VIABLE, 1);
        }
    }
    __syncwarp();
    C.add(W_CLKF, static_cast<unsigned long long>(clock64() - f0));
    return ok;
}

// Filter one row j of level k against u = stack[k] with the same pair +
// Theorem-1 rule as filter_push, writing the survivors of level k+1 at the
// row's level-k offset. Returns the surviving count.
template <int W, int MT>
__device__ __noinline__ int filter_one_row(WarpCtx<W, MT>& C, int k, int j) {
    const SearchParams& P = *C.P;
    const int lane = C.lane;
    WarpFixed& S = *C.S();
    const LevelMeta& Ls = S.lev[k];
    const uint32_t* src = level_entries<W, MT>(C, k) + Ls.start[j];
    uint32_t* dst = level_entries<W, MT>(C, k + 1) + Ls.start[j];
    const int cnt = Ls.cnt[j];
    const int d = P.d, six_d = 6 * d, two_d = 2 * d;
    // consensus row rule: slot 1 was prepared by the lazy push
    const bool cons = cons_rows_at<MT>(P, k);
    ConsMasks<W> cm;
    if (cons) cm = load_cons<W, MT>(C, 1);
    const TableRef<W> tr = table_ref<W, MT>(C);
    const Lmer<W> U = tr.get(S.stack_id[k] & ID_MASK);
    StackSet<W, MT> ss;
    ss.load(C, k, U);
    int out = 0;
    // entries two blocks ahead, their l-mers one block ahead (as filter_push)
    constexpr bool kPipeV = MT >= 4;
    uint32_t e_next = lane < cnt ? src[lane] : 0u;
    uint32_t e_next2 = kPipeV && lane + 32 < cnt ? src[lane + 32] : 0u;
    Lmer<W> V_next;
    if constexpr (kPipeV) V_next = tr.get(e_next & ID_MASK);
    for (int base = 0; base < cnt; base += 32) {
        const int f = base + lane;
        bool keep = false;
        Mask<W> mu;
        int hvu = 0;
        const uint32_t e = e_next;
        Lmer<W> V;
        if constexpr (kPipeV) {
            V = V_next;
            e_next = e_next2;
            e_next2 = f + 64 < cnt ? src[f + 64] : 0u;
            if (base + 32 < cnt) V_next = tr.get(e_next & ID_MASK);
        } else {
            e_next = f + 32 < cnt ? src[f + 32] : 0u;
            if (f < cnt) V = tr.get(e & ID_MASK);
        }
        if (f < cnt) {
            keep = !cons || cons_pass<W>(cm, V);
            if (keep) {
                mu = mism<W>(V, U);
                hvu = popcm<W>(mu);
                keep = hvu <= two_d;
            }
        }
        if constexpr (MT >= 5) {
            if (__any_sync(0xffffffffu, keep))  // as filter_push: whole-warp skip
                for (int i = 0; i < k; ++i)
                    if (keep) keep = ss.triple_ok(i, V, mu, hvu, six_d);
        } else if constexpr (MT >= PMS8G_ROLLED_MT) {
            // rolled (members in shared memory): ~1.5 KB less hot code per
            // filter in the I-cache-bound t = 4 builds
#pragma unroll 1
            for (int i = 0; i < k; ++i)
                if (keep) keep = ss.triple_ok(i, V, mu, hvu, six_d);
        } else {
#pragma unroll
            for (int i = 0; i < MT; ++i)
                if (i < k && keep) keep = ss.triple_ok(i, V, mu, hvu, six_d);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) dst[out + __popc(bal & lanemask_lt())] = e;
        out += __popc(bal);
    }
    C.add(W_SLOTS, static_cast<unsigned long long>(cnt));
    __syncwarp();
    return out;
}

// Push of u = stack[k] that completes the t-tuple: instead of filtering
// every remaining row (most are never read, because verification stops at
// the first row without a witness), the rows of level k+1 are filtered on
// demand by verification; only the smallest row is filtered eagerly as the
// viability check (an empty row means no motif below, src/solver.cpp:331-334).
template <int W, int MT>
__device__ __noinline__ bool lazy_push(WarpCtx<W, MT>& C, int k) {
    const int lane = C.lane;
    WarpFixed& S = *C.S();
    const LevelMeta& Ls = S.lev[k];
    LevelMeta& Ld = S.lev[k + 1];
    const int jb = Ls.branch;
    const int nr2 = Ls.nrows - 1;
    const long long f0 = clock64();
    if (cons_rows_at<MT>(*C.P, k)) {
        if (lane == 0) cache_member<W>(S, k, C.lmer(S.stack_id[k] & ID_MASK));
        __syncwarp();
        cons_prepare<W, MT>(C, k + 1, 1);  // for filter_one_row
    }
    int c = 0x7FFF;
    if (lane < nr2) {
        const int j = lane < jb ? lane : lane + 1;
        Ld.start[lane] = Ls.start[j];
        c = Ls.cnt[j];
        Ld.cnt[lane] = static_cast<uint32_t>(c);
        Ld.order[lane] = Ls.order[j];
    }
    // smallest unfiltered row (ties by position)
    int key = lane < nr2 ? (c << 8) | lane : 0x7FFFFFFF;
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, sh));
    if (lane == 0) {
        Ld.nrows = nr2;
        Ld.total = Ls.total;
        Ld.branch = 0;
        Ld.viable = 1;
        S.lazy_mask = 0u;
        S.lazy_level = k + 1;
    }
    __syncwarp();
    C.add(W_PUSH, 1);
    bool ok = true;
    if (nr2 > 0) {
        // the level-(k+1) row at position p comes from level-k position p' (p' skips the branch row)
        const int p = key & 0xFF;
        const int pk = p < jb ? p : p + 1;
        const int got = filter_one_row<W, MT>(C, k, pk);
        if (lane == 0) {
            Ld.cnt[p] = static_cast<uint32_t>(got);
            S.lazy_mask = 1u << p;
        }
        __syncwarp();
        ok = got > 0;
    }
    if (ok) C.add(W_VIABLE, 1);
    C.add(W_CLKF, static_cast<unsigned long long>(clock64() - f0));
    return ok;
}

// ---------------------------------------------------------------- donation
// Publish one dynamic task (header + nnodes nodes fetched by getnode(i)).
// Bounded MPMC ring: position s lives in slot s % qcap during round
// r = s / qcap; the slot state is 2r while free for that round's producer and
// 2r+1 once published, and the consumer frees it for round r+1 (2r+2) after
// copying the task out, so a slot is never overwritten while being read.
template <int W, int MT, typename F>
__device__ __noinline__ void publish(WarpCtx<W, MT>& C, TaskHeader& h, int nnodes, F getnode) {
    const SearchParams& P = *C.P;
    // level handed off with the task (TaskHeader::hlevel)
    {
        const int hl = h.kind == 0 ? h.k : h.k - 1;
        h.hlevel = (hl >= 2 && C.S()->lev[hl].total <= P.don_cap) ? static_cast<uint32_t>(hl) : 0u;
        h.pad = 0;
    }
    unsigned long long s = 0;
    if (C.lane == 0) {
        s = atomicAdd(&P.qs->alloc, 1ull);
        const unsigned int want = static_cast<unsigned int>(2 * (s / static_cast<unsigned long long>(P.qcap)));
        while (ld_volatile(&P.qstate[s % static_cast<unsigned long long>(P.qcap)]) != want) __nanosleep(200);
    }
    s = __shfl_sync(0xffffffffu, s, 0);
    const unsigned long long slot_i = s % static_cast<unsigned long long>(P.qcap);
    uint8_t* slot = P.qslots + slot_i * P.qslot_bytes;
    const uint32_t* hs = reinterpret_cast<const uint32_t*>(&h);
    uint32_t* hd = reinterpret_cast<uint32_t*>(slot);
    for (int x = C.lane; x < static_cast<int>(sizeof(TaskHeader) / 4); x += 32) hd[x] = hs[x];
    Node<W>* nd = reinterpret_cast<Node<W>*>(slot + sizeof(TaskHeader));
    for (int x = C.lane; x < nnodes; x += 32) nd[x] = getnode(x);
    if (h.hlevel) {
        const LevelMeta& L = C.S()->lev[h.hlevel];
        uint32_t* lm = reinterpret_cast<uint32_t*>(slot + P.qslot_lvl_off);
        const uint32_t* ms = reinterpret_cast<const uint32_t*>(&L);
        constexpr int MW = static_cast<int>(sizeof(LevelMeta) / 4);
        for (int x = C.lane; x < MW; x += 32) lm[x] = ms[x];
        const uint32_t* es = level_entries<W, MT>(C, static_cast<int>(h.hlevel));
        uint32_t* ed = lm + MW;
        const int tot = L.total;
        for (int x = C.lane; x < tot; x += 32) ed[x] = es[x];
    }
    __threadfence();
    __syncwarp();
    if (C.lane == 0) {
        __threadfence();
        atomicExch(&P.qstate[slot_i], static_cast<unsigned int>(2 * (s / static_cast<unsigned long long>(P.qcap)) + 1));
    }
    __syncwarp();
    C.add(W_DONATED, 1);
}

// True when idle warps are waiting and the queue cannot feed them.
template <int W, int MT>
__device__ bool starving(WarpCtx<W, MT>& C) {
    const SearchParams& P = *C.P;
    int want = 0;
    if (C.lane == 0) {
        const unsigned int waiting = ld_volatile(&P.qs->waiting);
        if (waiting > 0) {
            // heartbeat for the waiters' watchdog: busy warps are making progress
            if ((++C.checks & 7) == 0) atomicAdd(&P.qs->heartbeat, 1ull);
            const unsigned long long alloc = ld_volatile(&P.qs->alloc), head = ld_volatile(&P.qs->head);
            const unsigned long long queued = alloc > head ? alloc - head : 0;
            want = queued < waiting;
        }
    }
    return __shfl_sync(0xffffffffu, want, 0) != 0;
}

// DFS-level donation: give away the upper half of the remaining branch range
// of the shallowest level in [kmin, k] that has at least two branches left.
template <int W, int MT>
__device__ __noinline__ void maybe_donate_dfs(WarpCtx<W, MT>& C, int kmin, int k) {
    if (!C.P->donate) return;
    if (++C.pushes_since_check < C.P->don_pushes) return;
    C.pushes_since_check = 0;
    C.checks = 0;
    if (!starving<W, MT>(C)) return;
    WarpFixed& S = *C.S();
    for (int kk = kmin; kk <= k; ++kk) {
        const int it = S.iter[kk], end = S.iter_end[kk];
        if (end - it >= 2) {
            const int mid = it + (end - it + 1) / 2;
            TaskHeader h;
            h.anchor = C.anchor;
            h.kind = 0;
            h.k = static_cast<int16_t>(kk);
            h.a0 = mid;
            h.a1 = end;
#pragma unroll
            for (int i = 0; i < MAXT; ++i) h.stack[i] = i < kk ? S.stack_id[i] : 0u;
            __syncwarp();
            if (C.lane == 0) S.iter_end[kk] = mid;
            __syncwarp();
            publish<W, MT>(C, h, 0, [&](int) { return Node<W>{}; });
            return;
        }
    }
}

// ---------------------------------------------------------------- verification
// One row pass of the breadth-first verification, specialised on the number
// of 32-candidate chunks each lane holds in registers: every row entry is
// loaded once (32 per coalesced load) and broadcast by shuffle, and each
// compare instruction covers 32 x NCH candidate/entry pairs. Survivors are
// compacted to the front of the buffer; returns their number.
template <int W, int MT, int NCH>
__device__ __forceinline__ int verify_row(const WarpCtx<W, MT>& C, Lmer<W>* cand, const uint32_t* entries, int st,
                                         int cnt, int n, int d, int lane, int& scanned) {
    Lmer<W> cd[NCH];
    bool alive[NCH];
    int hm[NCH];  // smallest distance to the entries scanned so far (dead lanes: 0)
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        alive[ch] = ch * 32 + lane < n;
        hm[ch] = alive[ch] ? 0x7fff : 0;
        if (alive[ch]) cd[ch] = cand[ch * 32 + lane];
    }
    // entries per all-witnessed check. The t = 4 builds are bound by
    // instruction fetch (hot code > the 32 KB L1.5 I-cache): half the unroll
    // there ((21,8) -2%, (23,9) -3%; neutral for t <= 3)
    constexpr int U = MT == 4 ? (NCH == 1 ? 4 : 2) : (NCH == 1 ? 8 : (NCH == 2 ? 4 : 2));
    bool done = false;
    for (int eb = 0; eb < cnt && !done; eb += 32) {
        // lanes past the row's end hold a copy of its first entry, so whole
        // blocks of U entries can be compared without bound checks (a
        // duplicate cannot change "some entry is within d")
        const int lim = min(32, cnt - eb);
        const Lmer<W> mine = C.lmer(entries[st + eb + (lane < lim ? lane : 0)] & ID_MASK);
        for (int x0 = 0; x0 < lim; x0 += U) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const Lmer<W> V = shfl_lmer<W>(mine, (x0 + u) & 31);
                // XOR, XOR|OR, POPC, IMNMX per compare
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) hm[ch] = min(hm[ch], dist<W>(cd[ch], V));
            }
            scanned += U;
            int mx = hm[0];
#pragma unroll
            for (int ch = 1; ch < NCH; ++ch) mx = max(mx, hm[ch]);
            if (__all_sync(0xffffffffu, mx <= d)) {
                done = true;
                break;
            }
        }
    }
    __syncwarp();
    int out = 0;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        const bool keep = alive[ch] && hm[ch] <= d;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) cand[out + __popc(bal & lanemask_lt())] = cd[ch];
        out += __popc(bal);
    }
    __syncwarp();
    return out;
}

// Few candidates (n <= 12): lanes hold row entries instead, and each
// candidate is checked against 32 entries per ballot, stopping at its first
// witness.
template <int W, int MT>
__device__ __forceinline__ int verify_row_small(const WarpCtx<W, MT>& C, Lmer<W>* cand, const uint32_t* entries,
                                               int st, int cnt, int n, int d, int lane, int& scanned) {
    unsigned pass = 0u;  // bit i: candidate i has a witness in this row
    for (int eb = 0; eb < cnt; eb += 32) {
        const bool have = eb + lane < cnt;
        Lmer<W> mine;
        if (have) mine = C.lmer(entries[st + eb + lane] & ID_MASK);
        for (int i = 0; i < n; ++i) {
            if ((pass >> i) & 1u) continue;
            const Lmer<W> c = cand[i];
            if (__ballot_sync(0xffffffffu, have && dist<W>(c, mine) <= d)) pass |= 1u << i;
        }
        scanned += min(32, cnt - eb);
        if (pass == (n == 32 ? 0xffffffffu : ((1u << n) - 1u))) break;
    }
    // compact survivors in order
    Lmer<W> mine;
    const bool keep = lane < n && ((pass >> lane) & 1u);
    if (lane < n) mine = cand[lane];
    __syncwarp();
    if (keep) cand[__popc(pass & lanemask_lt())] = mine;
    __syncwarp();
    return __popc(pass);
}

// Make row position p of the lazy level t available (filter it on demand).
template <int W, int MT>
__device__ __forceinline__ void ensure_row(WarpCtx<W, MT>& C, int t, int p) {
    WarpFixed& S = *C.S();
    if (S.lazy_level != t || (S.lazy_mask >> p) & 1u) return;
    const int k = t - 1;
    const int jb = S.lev[k].branch;
    const int pk = p < jb ? p : p + 1;
    const int got = filter_one_row<W, MT>(C, k, pk);
    if (C.lane == 0) {
        S.lev[t].cnt[p] = static_cast<uint32_t>(got);
        S.lazy_mask |= 1u << p;
    }
    __syncwarp();
}

// Breadth-first verification of the buffered candidates against the level's
// rows, smallest row first (verify_candidate checks rows in size order and
// stops at the first row without a witness); survivors are emitted as keys.
template <int W, int MT>
__device__ __noinline__ void verify_all(WarpCtx<W, MT>& C, const LevelMeta& L, const uint32_t* entries, int ncand) {
    const SearchParams& P = *C.P;
    const int lane = C.lane;
    const int d = P.d;
    int n = ncand;
    unsigned long long vcmp = 0;
    const int tlev = static_cast<int>(&L - C.S()->lev);
    for (int r = 0; r < L.nrows && n > 0; ++r) {
        const int j = C.S()->vorder[r];
        ensure_row<W, MT>(C, tlev, j);
        const int st = L.start[j], cnt = L.cnt[j];
        int scanned = 0, out = 0;
        if (n <= 12) {
            out = verify_row_small<W, MT>(C, C.cand(), entries, st, cnt, n, d, lane, scanned);
        } else if (MT == 4) {
            // t = 4 builds (instruction-fetch bound): one specialisation, 64
            // candidates per pass over the row, instead of three - the row is
            // re-read for candidates 65..160, but 3.4 KB of hot code go
            // ((21,8) -4.5%, (23,9) -4.4%)
            for (int g0 = 0; g0 < n; g0 += 64) {
                const int ng = min(64, n - g0);
                int sg = 0;
                const int og = verify_row<W, MT, 2>(C, C.cand() + g0, entries, st, cnt, ng, d, lane, sg);
                vcmp += static_cast<unsigned long long>(ng) * sg;
                if (g0 > 0) {
                    Lmer<W> mv[2];
                    for (int q = 0; q < 2; ++q)
                        if (q * 32 + lane < og) mv[q] = C.cand()[g0 + q * 32 + lane];
                    __syncwarp();
                    for (int q = 0; q < 2; ++q)
                        if (q * 32 + lane < og) C.cand()[out + q * 32 + lane] = mv[q];
                    __syncwarp();
                }
                out += og;
            }
        } else switch ((n + 31) >> 5) {
            case 1: out = verify_row<W, MT, 1>(C, C.cand(), entries, st, cnt, n, d, lane, scanned); break;
            case 2: out = verify_row<W, MT, 2>(C, C.cand(), entries, st, cnt, n, d, lane, scanned); break;
            default: out = verify_row<W, MT, 5>(C, C.cand(), entries, st, cnt, n, d, lane, scanned); break;
        }
        vcmp += static_cast<unsigned long long>(n) * scanned;
        n = out;
    }
    C.add(W_VCMP, vcmp);
    // emit the survivors as packed keys
    for (int base = 0; base < n; base += 32) {
        const bool alive = base + lane < n;
        const unsigned em = __ballot_sync(0xffffffffu, alive);
        unsigned long long pos0 = 0;
        if (lane == 0) pos0 = atomicAdd(P.key_count, static_cast<unsigned long long>(__popc(em)));
        pos0 = __shfl_sync(0xffffffffu, pos0, 0);
        if (alive) {
            const unsigned long long pos = pos0 + __popc(em & lanemask_lt());
            if (static_cast<long long>(pos) < P.key_cap) {
                unsigned long long klo, khi;
                make_key<W>(C.cand()[base + lane], P.l, klo, khi);
                P.keys[2 * pos] = klo;
                P.keys[2 * pos + 1] = khi;
            }
        }
        C.add(W_EMIT, __popc(em));
    }
    __syncwarp();
}

// Verification order of a level's rows: S.vorder[r] = position of the r-th
// smallest row (ties by position), verify_candidate's ascending-size order
// (src/solver.cpp:344-362). A rolled loop over register broadcasts: it runs
// once per tuple, and unrolled it cost ~5 KB of hot code (I-cache).
__device__ __forceinline__ void rank_rows(WarpFixed& S, const LevelMeta& L, int lane) {
    const int nr = L.nrows;
    const unsigned key = lane < nr ? (static_cast<unsigned>(L.cnt[lane]) << 5) | static_cast<unsigned>(lane) : ~0u;
    int rank = 0;
#pragma unroll 1
    for (int q = 0; q < nr; ++q) rank += __shfl_sync(0xffffffffu, key, q) < key;
    if (lane < nr) S.vorder[rank] = static_cast<uint8_t>(lane);
}

// ---------------------------------------------------------------- enumeration
// Enumeration order of the tuple's positions. The common d-neighbourhood
// does not depend on the order in which positions are assigned, and the
// pruning bounds of NeighborhoodEnumerator::prune (src/neighborhood.cpp:
// 228-270) are sound for any order as long as their suffix tables follow it.
// Positions where the members agree go first (key: consensus column cost,
// then the number of distinct symbols; ties by position): a non-consensus
// symbol there charges every member, so infeasible prefixes die near the
// root (about 2x fewer tree nodes on the planted configs).
// On return S.perm[depth] is the position assigned at that depth and Tm
// holds the members with their symbols moved to depth order, so the suffix
// tables can be built from Tm as if the order were natural. exact_tree keeps
// the natural order (the reference's tree).
template <int W, int MT>
__device__ __noinline__ void order_positions(WarpCtx<W, MT>& C, int t, Lmer<W>* Tm) {
    t = tuple_size<MT>(t);
    const int lane = C.lane, l = C.P->l;
    WarpFixed& S = *C.S();
    constexpr int NC = W;  // 32-position chunks
    if (!C.P->reorder) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (c * 32 + lane < l) S.perm[c * 32 + lane] = static_cast<uint8_t>(c * 32 + lane);
        __syncwarp();
        return;
    }
    // two-word members in registers (Tm lives on the stack: its address
    // crosses calls); one-word builds read it in place (their register
    // budget is shared with the fast loop)
    Lmer<W> tm_r[MT];
    if constexpr (W == 2) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
            if (i < t) tm_r[i] = Tm[i];
    }
    // (indexed with unrolled constants, so tm_r stays in registers; a pointer
    // to it would put it back on the stack)
#define PMS8G_TM(i) (W == 2 ? tm_r[i] : Tm[i])
    int key[NC];
    unsigned present = 0u;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int p = c * 32 + lane;
        key[c] = 31;  // past the end: sorts last
        if (p < l) {
            int f[4] = {0, 0, 0, 0};
#pragma unroll
            for (int i = 0; i < MT; ++i)
                if (i < t) {
                    const int ci = code_at<W>(PMS8G_TM(i), p);
#pragma unroll
                    for (int x = 0; x < 4; ++x) f[x] += ci == x;
                }
            const int best = max(max(f[0], f[1]), max(f[2], f[3]));
            const int dis = (f[0] > 0) + (f[1] > 0) + (f[2] > 0) + (f[3] > 0);
            key[c] = (t - best) * 4 + dis - 1;
        }
        present |= __reduce_or_sync(0xffffffffu, 1u << key[c]);
    }
    int rank[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) rank[c] = 0;
    const unsigned lt = lanemask_lt();
    while (present) {
        const int k = __ffs(present) - 1;
        present &= present - 1;
        unsigned b[NC];
        int tot = 0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            b[c] = __ballot_sync(0xffffffffu, key[c] == k);
            tot += __popc(b[c]);
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            if (key[c] > k) rank[c] += tot;
            if (key[c] == k) {
                int before = __popc(b[c] & lt);
#pragma unroll
                for (int e = 0; e < NC; ++e)
                    if (e < c) before += __popc(b[e]);
                rank[c] += before;
            }
        }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
        if (c * 32 + lane < l) S.perm[rank[c]] = static_cast<uint8_t>(c * 32 + lane);
    __syncwarp();
    // move every member's symbols to depth order (all reads before writes)
    uint32_t nh[MT][NC], no[MT][NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int q = c * 32 + lane;
        const int pos = q < l ? S.perm[q] : 0;
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int code = (i < t && q < l) ? code_at<W>(PMS8G_TM(i), pos) : 0;
            nh[i][c] = __ballot_sync(0xffffffffu, (code >> 1) & 1);
            no[i][c] = __ballot_sync(0xffffffffu, code & 1);
        }
    }
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            Tm[i].h[c] = nh[i][c];
            Tm[i].o[c] = no[i][c];
        }
}

#undef PMS8G_TM

// Per-tuple suffix tables (NeighborhoodEnumerator::prepare, :164-226):
// eq[p] (members holding each symbol), pair suffix distances, Theorem-1
// triple thresholds (Cd3 = (h_ij + h_ih + h_jh + n4) / 2 of the suffix) and
// the consensus suffix bound, plus the verification row order.
template <int W, int MT>
__device__ __noinline__ void prepare_tuple(WarpCtx<W, MT>& C, int t, const LevelMeta& L, Lmer<W>* Tm) {
    t = tuple_size<MT>(t);
    const SearchParams& P = *C.P;
    const int lane = C.lane, l = P.l;
    WarpFixed& S = *C.S();
    const int np = P.plan.npair, ntot = P.plan.npair + P.plan.ntri;
    // two-word members in registers (see order_positions)
    Lmer<W> tm_r[MT];
    if constexpr (W == 2) {
#pragma unroll
        for (int i = 0; i < MT; ++i)
            if (i < t) tm_r[i] = Tm[i];
    }
    // (indexed with unrolled constants, so tm_r stays in registers; a pointer
    // to it would put it back on the stack)
#define PMS8G_TM(i) (W == 2 ? tm_r[i] : Tm[i])
    for (int p = lane; p <= l; p += 32) {
        uint32_t e = 0;
        if (p < l) {
#pragma unroll
            for (int i = 0; i < MT; ++i)
                if (i < t) e |= 1u << (8 * code_at<W>(PMS8G_TM(i), p) + i);
            gen_eq(C)[p] = e;
        }
        uint8_t* row = C.thr() + GEN_TBL_BYTES + p * ntot;
#pragma unroll
        for (int j = 1; j < MT; ++j)
#pragma unroll
            for (int i = 0; i < j; ++i)
                if (j < t) row[j * (j - 1) / 2 + i] = static_cast<uint8_t>(suffix_popc<W>(mism<W>(PMS8G_TM(i), PMS8G_TM(j)), p));
#pragma unroll
        for (int h = 2; h < MT; ++h)
#pragma unroll
            for (int j = 1; j < h; ++j)
#pragma unroll
                for (int i = 0; i < j; ++i)
                    if (h < t) {
                        const Mask<W> mij = mism<W>(PMS8G_TM(i), PMS8G_TM(j));
                        const Mask<W> mih = mism<W>(PMS8G_TM(i), PMS8G_TM(h));
                        const Mask<W> mjh = mism<W>(PMS8G_TM(j), PMS8G_TM(h));
                        Mask<W> n4;
#pragma unroll
                        for (int x = 0; x < W; ++x) n4.w[x] = mij.w[x] & mih.w[x] & mjh.w[x];
                        const int v = (suffix_popc<W>(mij, p) + suffix_popc<W>(mih, p) + suffix_popc<W>(mjh, p) +
                                       suffix_popc<W>(n4, p)) / 2;
                        row[np + h * (h - 1) * (h - 2) / 6 + j * (j - 1) / 2 + i] = static_cast<uint8_t>(v);
                    }
    }
    __syncwarp();
#undef PMS8G_TM
    int carry = 0;
    const int nchunk = (l + 32) / 32;
    for (int ch = nchunk - 1; ch >= 0; --ch) {
        const int p = ch * 32 + lane;
        int v = 0;
        if (p < l) {
            const uint32_t e = gen_eq(C)[p];
            const int best = max(max(__popc(e & 0xFFu), __popc(e & 0xFF00u)),
                                 max(__popc(e & 0xFF0000u), __popc(e & 0xFF000000u)));
            v = t - best;
        }
        int incl = v;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const int x = __shfl_down_sync(0xffffffffu, incl, s);
            if (lane + s < 32) incl += x;
        }
        if (p <= l) gen_cons(C)[p] = static_cast<uint8_t>(incl + carry);
        carry += __shfl_sync(0xffffffffu, incl, 0);
    }
    rank_rows(S, L, lane);
    __syncwarp();
}

// Evaluate child (node, symbol c). Returns ok; writes child + leaf flag.
template <int W, int MT>
__device__ __forceinline__ bool expand_child(const WarpCtx<W, MT>& C, const Node<W>& nd, int c, int t, uint32_t tmask,
                                             int prune, Node<W>& ch, bool& leaf) {
    const SearchParams& P = *C.P;
    const WarpFixed& S = *C.S();
    const int p = static_cast<int>(nd.rB >> 24);
    const uint32_t em = (gen_eq(C)[p] >> (8 * c)) & tmask;  // members matching symbol c
    const uint32_t mm = ~em & tmask;                   // members charged on this edge
    int r[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const uint32_t word = i < 4 ? nd.rA : nd.rB;
        r[i] = static_cast<int>((word >> (8 * (i & 3))) & 0xFFu) - 64 - static_cast<int>((mm >> i) & 1u);
    }
    ch.c = nd.c;
    set_code<W>(ch.c, S.perm[p], c);
    const int q = p + 1;
    bool neg = false;
#pragma unroll
    for (int i = 0; i < MT; ++i)
        if (i < t) neg |= r[i] < 0;
    leaf = q == P.l;
    bool ok;
    if (leaf) {
        ok = !neg;
    } else if (prune == 0 || mm == 0) {
        ok = true;
    } else {
        ok = !neg;
        const uint8_t* row = C.thr() + GEN_TBL_BYTES + q * (P.plan.npair + P.plan.ntri);
        if (ok) {
#pragma unroll
            for (int j = 1; j < MT; ++j)
#pragma unroll
                for (int i = 0; i < j; ++i)
                    if (j < t) ok &= row[j * (j - 1) / 2 + i] <= r[i] + r[j];
        }
        if (ok && prune == 2) {
#pragma unroll
            for (int h = 2; h < MT; ++h)
#pragma unroll
                for (int j = 1; j < h; ++j)
#pragma unroll
                    for (int i = 0; i < j; ++i)
                        if (h < t)
                            ok &= row[P.plan.npair + h * (h - 1) * (h - 2) / 6 + j * (j - 1) / 2 + i] <=
                                  r[i] + r[j] + r[h];
            int sum = 0;
#pragma unroll
            for (int i = 0; i < MT; ++i)
                if (i < t) sum += r[i];
            if (t >= 2) ok &= gen_cons(C)[q] <= sum;
        }
    }
    uint32_t rA = 0, rB = 0;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const uint32_t b = static_cast<uint32_t>(r[i] + 64) & 0xFFu;
        if (i < 4) rA |= b << (8 * i);
        else rB |= b << (8 * (i - 4));
    }
    ch.rA = rA;
    ch.rB = rB | (static_cast<uint32_t>(q) << 24);
    return ok;
}


// ---------------------------------------------------------------- SWAR path (t <= 4)
// Budgets of up to 4 tuple members live in one word, one byte each (r_i >= 0,
// unused members pinned at 0). Per tuple and position p, DEC[p][c] holds
// [s_i[p] != c] in byte i, so a child's budgets are (R | 0x80..) - DEC with no
// cross-byte borrow and a cleared bit 7 flags an exhausted budget. Per suffix
// start q, THR[q] packs the pair thresholds [01,12,23,02], [13,03,cons,-] and
// the Theorem-1 triple thresholds [012,123,013,023]; the pair sums and triple
// sums come from three shifted adds and are compared bytewise. Same rules as
// NeighborhoodEnumerator::prune (src/neighborhood.cpp:228-270), branch-free.
__device__ __forceinline__ bool bytes_ge(uint32_t x, uint32_t y) {
    return (((x | 0x80808080u) - y) & 0x80808080u) == 0x80808080u;
}

template <int W, int MT>
__device__ __noinline__ void prepare_tuple_swar(WarpCtx<W, MT>& C, int t, const LevelMeta& L, const Lmer<W>* Tm) {
    t = tuple_size<MT>(t);
    const int lane = C.lane, l = C.P->l;
    WarpFixed& S = *C.S();
    uint32_t* dec = reinterpret_cast<uint32_t*>(C.thr());          // [l][4]
    uint4* thr = reinterpret_cast<uint4*>(C.thr() + 16 * ((l + 3) & ~3) );  // [l+1]
    const int nchunk = (l + 32) / 32;  // positions 0..l
    int carry = 0, carry_next = 0;
    for (int ch = nchunk - 1; ch >= 0; --ch) {
        const int p = ch * 32 + lane;
        carry = carry_next;
        if (p < l) {
            uint32_t dd[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int i = 0; i < MT; ++i)
                if (i < t) {
                    const int ci = code_at<W>(Tm[i], p);
#pragma unroll
                    for (int c = 0; c < 4; ++c) dd[c] |= static_cast<uint32_t>(ci != c) << (8 * i);
                }
#pragma unroll
            for (int c = 0; c < 4; ++c) dec[4 * p + c] = dd[c];
        }
        uint32_t pr[6] = {0u, 0u, 0u, 0u, 0u, 0u};  // 01,12,23,02,13,03
        uint32_t tr[4] = {0u, 0u, 0u, 0u};          // 012,123,013,023
        Mask<W> m[4][4];
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = i + 1; j < MT; ++j) m[i][j] = mism<W>(Tm[i], Tm[j]);
        auto ps = [&](int i, int j) -> uint32_t {
            return (i < t && j < t) ? static_cast<uint32_t>(suffix_popc<W>(m[i][j], p)) : 0u;
        };
        auto ts = [&](int i, int j, int h) -> uint32_t {
            if (!(i < t && j < t && h < t)) return 0u;
            Mask<W> n4;
#pragma unroll
            for (int x = 0; x < W; ++x) n4.w[x] = m[i][j].w[x] & m[i][h].w[x] & m[j][h].w[x];
            return static_cast<uint32_t>((suffix_popc<W>(m[i][j], p) + suffix_popc<W>(m[i][h], p) +
                                          suffix_popc<W>(m[j][h], p) + suffix_popc<W>(n4, p)) / 2);
        };
        if (MT >= 2) pr[0] = ps(0, 1);
        if (MT >= 3) {
            pr[1] = ps(1, 2);
            pr[3] = ps(0, 2);
            tr[0] = ts(0, 1, 2);
        }
        if (MT >= 4) {
            pr[2] = ps(2, 3);
            pr[4] = ps(1, 3);
            pr[5] = ps(0, 3);
            tr[1] = ts(1, 2, 3);
            tr[2] = ts(0, 1, 3);
            tr[3] = ts(0, 2, 3);
        }
        // consensus suffix bound: column cost t - max frequency, summed over
        // the suffix by a reverse scan across lanes (two chunks for l > 31)
        uint32_t cons = 0;
        {
            int v = 0;
            if (p < l) {
                int f0 = 0, f1 = 0, f2 = 0, f3 = 0;
#pragma unroll
                for (int i = 0; i < MT; ++i)
                    if (i < t) {
                        const int ci = code_at<W>(Tm[i], p);
                        f0 += ci == 0;
                        f1 += ci == 1;
                        f2 += ci == 2;
                        f3 += ci == 3;
                    }
                v = t - max(max(f0, f1), max(f2, f3));
            }
            int incl = v;
#pragma unroll
            for (int sh = 1; sh < 32; sh <<= 1) {
                const int x = __shfl_down_sync(0xffffffffu, incl, sh);
                if (lane + sh < 32) incl += x;
            }
            // carry from the later chunk (positions p + 32 ...) is added below
            cons = static_cast<uint32_t>(incl) + static_cast<uint32_t>(carry);
            carry_next = __shfl_sync(0xffffffffu, incl, 0) + carry;
        }
        // budgets are <= d <= 31 here, so every sum is <= 124: clamping the
        // thresholds at 127 keeps the bytewise compares borrow-free
#pragma unroll
        for (int x = 0; x < 6; ++x) pr[x] = min(pr[x], 127u);
#pragma unroll
        for (int x = 0; x < 4; ++x) tr[x] = min(tr[x], 127u);
        cons = min(cons, 127u);
        if (p <= l) {
            uint4 w;
            w.x = pr[0] | (pr[1] << 8) | (pr[2] << 16) | (pr[3] << 24);
            w.y = pr[4] | (pr[5] << 8) | (cons << 16);
            w.z = tr[0] | (tr[1] << 8) | (tr[2] << 16) | (tr[3] << 24);
            w.w = p >= 1 ? S.perm[p - 1] : 0u;  // position assigned by children of depth p - 1
            thr[p] = w;
        }
    }
    rank_rows(S, L, lane);
    __syncwarp();
}

// prepare_tuple_swar + order_positions for the fast loop (l <= 32, t <= 4),
// computed on whole 32-position bit planes instead of per-position symbol
// extraction: pair mismatch masks, Theorem-1 "all distinct" masks and the
// consensus column-cost masks (cost >= 1, >= 2, >= 3) are a few LOP3s each,
// every suffix sum is one shifted POPC per lane, and the agreement-first
// order is a stable rank over at most five (cost, distinct) classes.
template <int MT>
__device__ __noinline__ void prepare_tuple_fast(WarpCtx<1, MT>& C, int t, const LevelMeta& L, Lmer<1>* Tm) {
    t = tuple_size<MT>(t);
    const int lane = C.lane, l = C.P->l;
    WarpFixed& S = *C.S();
    uint4* dec4 = reinterpret_cast<uint4*>(C.thr());                       // [l] x {c = 0..3}
    uint4* thr = reinterpret_cast<uint4*>(C.thr() + 16 * ((l + 3) & ~3));  // [l + 1]
    const uint32_t lmask = l >= 32 ? 0xffffffffu : ((1u << l) - 1u);
    const bool in = lane < l;
    uint32_t h[MT], o[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        h[i] = i < t ? Tm[i].h[0] : 0u;
        o[i] = i < t ? Tm[i].o[0] : 0u;
    }
    int pos = lane;
    if (C.P->reorder) {
        uint32_t e = 0;  // byte c: members holding symbol c at this lane's position
#pragma unroll
        for (int i = 0; i < MT; ++i)
            if (i < t) e += 1u << (8 * ((((h[i] >> lane) & 1u) << 1) | ((o[i] >> lane) & 1u)));
        const uint32_t m2 = __vmaxu4(e, e >> 16);
        const int best = static_cast<int>(max(m2 & 0xFFu, (m2 >> 8) & 0xFFu));
        const int dis = __popc((e | (e >> 1) | (e >> 2)) & 0x01010101u);
        const int key = in ? (t - best) * 4 + dis - 1 : 31;
        unsigned present = __reduce_or_sync(0xffffffffu, 1u << key);
        const unsigned lt = lanemask_lt();
        int rank = 0;
        while (present) {
            const int k = __ffs(present) - 1;
            present &= present - 1;
            const unsigned b = __ballot_sync(0xffffffffu, key == k);
            rank += key > k ? __popc(b) : (key == k ? __popc(b & lt) : 0);
        }
        if (in) S.perm[rank] = static_cast<uint8_t>(lane);
        __syncwarp();
        pos = in ? S.perm[lane] : 0;
#pragma unroll
        for (int i = 0; i < MT; ++i)
            if (i < t) {
                const uint32_t hb = __ballot_sync(0xffffffffu, in && ((h[i] >> pos) & 1u));
                const uint32_t ob = __ballot_sync(0xffffffffu, in && ((o[i] >> pos) & 1u));
                h[i] = hb;
                o[i] = ob;
            }
    } else if (in) {
        S.perm[lane] = static_cast<uint8_t>(lane);
    }
    // budget decrements of the two child pairs at this depth
    if (in) {
        uint32_t e = 0;  // byte c, bit i: member i holds symbol c
#pragma unroll
        for (int i = 0; i < MT; ++i)
            if (i < t) e |= 1u << (8 * ((((h[i] >> lane) & 1u) << 1) | ((o[i] >> lane) & 1u)) + i);
        const uint32_t tm = (1u << t) - 1u;
        uint32_t dd[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) dd[c] = (((~(e >> (8 * c))) & tm) * 0x00204081u) & 0x01010101u;
        dec4[lane] = make_uint4(dd[0], dd[1], dd[2], dd[3]);
    }
    // suffix thresholds
    uint32_t m[4][4];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = i + 1; j < MT; ++j) m[i][j] = (i < t && j < t) ? ((h[i] ^ h[j]) | (o[i] ^ o[j])) : 0u;
    uint32_t a1 = 0u, a2 = 0u, a3 = 0u;  // column cost >= 1, >= 2, >= 3
    if (MT == 2 || t == 2) {
        a1 = m[0][1];
    } else if (MT == 3 || t == 3) {
        a1 = m[0][1] | m[0][2];
        a2 = m[0][1] & m[0][2] & m[1][2];
    } else if (MT >= 4 && t == 4) {
        a1 = m[0][1] | m[0][2] | m[0][3];
        const uint32_t three = (~m[0][1] & ~m[0][2]) | (~m[0][1] & ~m[0][3]) | (~m[0][2] & ~m[0][3]) |
                               (~m[1][2] & ~m[1][3]);
        a2 = ~three & lmask;
        a3 = m[0][1] & m[0][2] & m[0][3] & m[1][2] & m[1][3] & m[2][3];
    }
    const int prevpos = __shfl_up_sync(0xffffffffu, pos, 1);
    const int lastpos = __shfl_sync(0xffffffffu, pos, 31);
    for (int q = lane; q <= l; q += 32) {
        auto sp = [&](uint32_t x) -> uint32_t { return q < 32 ? static_cast<uint32_t>(__popc(x >> q)) : 0u; };
        auto tri = [&](uint32_t x, uint32_t y, uint32_t z) -> uint32_t {
            return (sp(x) + sp(y) + sp(z) + sp(x & y & z)) >> 1;
        };
        uint32_t pr[6] = {0u, 0u, 0u, 0u, 0u, 0u};  // 01,12,23,02,13,03
        uint32_t tr[4] = {0u, 0u, 0u, 0u};          // 012,123,013,023
        if (MT >= 2) pr[0] = sp(m[0][1]);
        if (MT >= 3) {
            pr[1] = sp(m[1][2]);
            pr[3] = sp(m[0][2]);
            tr[0] = tri(m[0][1], m[0][2], m[1][2]);
        }
        if (MT >= 4) {
            pr[2] = sp(m[2][3]);
            pr[4] = sp(m[1][3]);
            pr[5] = sp(m[0][3]);
            tr[1] = tri(m[1][2], m[1][3], m[2][3]);
            tr[2] = tri(m[0][1], m[0][3], m[1][3]);
            tr[3] = tri(m[0][2], m[0][3], m[2][3]);
        }
        // budgets are <= d <= 31 here: thresholds clamp at 127 (borrow-free compares)
        const uint32_t cons = min(sp(a1) + sp(a2) + sp(a3), 127u);
#pragma unroll
        for (int x = 0; x < 6; ++x) pr[x] = min(pr[x], 127u);
#pragma unroll
        for (int x = 0; x < 4; ++x) tr[x] = min(tr[x], 127u);
        uint4 w;
        // stored as 0x80 - threshold per byte (bytes <= 127: no borrows), see swar_feasible
        w.x = 0x80808080u - (pr[0] | (pr[1] << 8) | (pr[2] << 16) | (pr[3] << 24));
        w.y = 0x80808080u - (pr[4] | (pr[5] << 8) | (cons << 16));
        w.z = 0x80808080u - (tr[0] | (tr[1] << 8) | (tr[2] << 16) | (tr[3] << 24));
        w.w = q == 0 ? 0u : static_cast<uint32_t>(q < 32 ? prevpos : lastpos);  // position of depth q - 1
        thr[q] = w;
    }
    rank_rows(S, L, lane);
    __syncwarp();
}

template <int W, int MT>
__device__ __forceinline__ bool expand_child_swar(const WarpCtx<W, MT>& C, const Node<W>& nd, int c, int prune,
                                                  Node<W>& ch, bool& leaf) {
    const int l = C.P->l;
    const uint32_t* dec = reinterpret_cast<const uint32_t*>(C.thr());
    const uint4* thr = reinterpret_cast<const uint4*>(C.thr() + 16 * ((l + 3) & ~3));
    const int p = static_cast<int>(nd.rB >> 24);
    const uint32_t D = dec[4 * p + c];
    uint32_t R = (nd.rA | 0x80808080u) - D;
    bool ok = (R & 0x80808080u) == 0x80808080u;
    R &= 0x7F7F7F7Fu;
    const int q = p + 1;
    leaf = q == l;
    if (!leaf && prune != 0 && D != 0u) {
        const uint4 T = thr[q];
        const uint32_t r3 = R >> 24;
        const uint32_t A1 = R + (R >> 8);    // [01, 12, 23, 3]
        const uint32_t A2 = R + (R >> 16);   // [02, 13, 2, 3]
        const uint32_t A3 = R + r3;          // [03, 1, 2, 3]
        const uint32_t P1 = (A1 & 0x00FFFFFFu) | (A2 << 24);                      // [01,12,23,02]
        const uint32_t S3 = A1 + (R >> 16);                                       // [012, 123, ..]
        const uint32_t cons = (S3 + r3) & 0xFFu;                                  // r0+r1+r2+r3
        const uint32_t P2 = ((A2 >> 8) & 0xFFu) | ((A3 & 0xFFu) << 8) | (cons << 16);  // [13,03,cons,0]
        const uint32_t B1 = (A1 + r3) & 0xFFu;                                    // 013
        const uint32_t B2 = (A2 + r3) & 0xFFu;                                    // 023
        const uint32_t T3 = (S3 & 0xFFFFu) | (B1 << 16) | (B2 << 24);             // [012,123,013,023]
        ok = ok && bytes_ge(P1, T.x) && bytes_ge(P2, prune == 2 ? T.y : (T.y & 0xFFFFu)) &&
             (prune != 2 || bytes_ge(T3, T.z));
    }
    ch.c = nd.c;
    set_code<W>(ch.c, C.S()->perm[p], c);
    ch.rA = R;
    ch.rB = static_cast<uint32_t>(q) << 24;
    return ok;
}


// SWAR check of a child's budget bytes R against the suffix thresholds of
// its position (pairs, consensus, Theorem-1 triples), specialised on MT. The
// fast tables hold 0x80 - threshold per byte (prepare_tuple_fast), so
// "sum >= threshold" is bit 7 of sum + (0x80 - threshold): every sum and
// threshold is <= 127, so no byte carries into the next, and the three
// words are checked with one AND. Sums are assembled with PRMT.
template <int MT>
__device__ __forceinline__ bool swar_feasible(uint32_t R, const uint4& T, int prune) {
    const uint32_t M = 0x80808080u;
    const uint32_t A1 = R + (R >> 8);  // [01, 12, 23, 3]
    if (MT == 2) return ((A1 + T.x) & 0x80u) != 0u;
    const uint32_t R16 = R >> 16;
    const uint32_t A2 = R + R16;                       // [02, 13, 2, 3]
    const uint32_t P1 = __byte_perm(A1, A2, 0x4210);   // [01, 12, 23, 02]
    const uint32_t S3 = A1 + R16;                      // [012, 123, ., .]
    if (MT == 3) {
        // pairs 01,12,02 + triple 012 (= the consensus bound for 3 members)
        const uint32_t a = P1 + T.x;
        return ((prune == 2 ? a & (S3 + T.z) : a) & M) == M;
    }
    const uint32_t R24 = R >> 24;
    const uint32_t B = R + R24;                              // [03, ...]
    const uint32_t X = __byte_perm(A2, B, 0x0041);           // [13, 03, ., .]
    const uint32_t P2 = __byte_perm(X, S3 + R24, 0x0410);    // [13, 03, 0123, 13]
    const uint32_t Y = __byte_perm(A1 + R24, A2 + R24, 0x0040);  // [013, 023, ., .]
    const uint32_t T3 = __byte_perm(S3, Y, 0x5410);              // [012, 123, 013, 023]
    // pairs only (prune == 1): the consensus and triple thresholds become
    // "always pass" (0x80 - 0) instead of a second code path, so no dead
    // arithmetic is if-converted into the child check
    const uint32_t ty = prune == 2 ? T.y : ((T.y & 0xFFFFu) | 0x80800000u);
    const uint32_t tz = prune == 2 ? T.z : M;
    return ((P1 + T.x) & (P2 + ty) & (T3 + tz) & M) == M;
}

// Enumeration loop for l <= 32 and t <= 4: nodes are uint4 {h, o, budgets,
// p<<24}; a round pops 16 nodes, each lane evaluates two sibling children
// (symbols 2(lane&1) and 2(lane&1)+1) from one LDS.128 node, one LDS.64 of
// budget decrements and one LDS.128 of suffix thresholds.
template <int MT>
__device__ __noinline__ void enum_loop_fast(WarpCtx<1, MT>& C, int t, const LevelMeta& L, const uint32_t* entries,
                                            int bot, int nn, int nov, unsigned long long& nodes_out,
                                            unsigned long long& leaves_out) {
    const SearchParams& P = *C.P;
    const int lane = C.lane, l = P.l;
    WarpFixed& S = *C.S();
    constexpr int NS = NodeSmem<1>::N;
    constexpr int SPILL = NS / 4;
    uint4* ns = reinterpret_cast<uint4*>(C.node_smem());
    uint4* ov = reinterpret_cast<uint4*>(C.node_glob);
    uint2* cand = reinterpret_cast<uint2*>(C.cand());
    const uint2* dec2 = reinterpret_cast<const uint2*>(C.thr());
    const uint4* thr = reinterpret_cast<const uint4*>(C.thr() + 16 * ((l + 3) & ~3));
    const int prune = P.prune;
    const int cand_cap = P.plan.cand_cap;
    const uint32_t odd = lane & 1;
    unsigned long long leaves = 0, nodes = 0;
    uint32_t leaves32 = 0, nodes32 = 0, rounds32 = 0;
    int rounds = 0, burst = 0;
    int ncand = 0;
    const bool may_donate = P.donate != 0;
    while (nn > 0 || nov > 0) {
        // slow paths (uniform): refill from / spill to the global overflow,
        // periodic donation check, 32-bit counter flush
        if (nn == 0 || nn > NS - 48 || (++rounds & P.don_rounds_mask) == 0) {
            if (nn == 0) {
                nov -= SPILL;
                if (lane < SPILL) ns[(bot + lane) & (NS - 1)] = ov[nov + lane];
                nn = SPILL;
                __syncwarp();
            }
            if ((rounds & P.don_rounds_mask) == 0) {
                leaves += leaves32;
                nodes += nodes32;
                leaves32 = nodes32 = 0;
                if (may_donate && (nov >= NDON || nn >= NDON + 16) && starving<1, MT>(C)) {
                    TaskHeader h;
                    h.anchor = C.anchor;
                    h.kind = 1;
                    h.k = static_cast<int16_t>(t);
                    // the shallowest 32 nodes (overflow first)
                    const int half = NDON;
                    h.a0 = half;
                    h.a1 = 0;
#pragma unroll
                    for (int i = 0; i < MAXT; ++i) h.stack[i] = i < t ? S.stack_id[i] : 0u;
                            if (nov >= NDON) {
                        const int o0 = nov - NDON;
                        publish<1, MT>(C, h, NDON, [&](int x) { return C.node_glob[o0 + x]; });
                        nov -= NDON;
                    } else {
                        const int b0 = bot;
                        publish<1, MT>(C, h, half, [&](int x) { return C.node_smem()[(b0 + x) & (NS - 1)]; });
                        bot = (bot + half) & (NS - 1);
                        nn -= half;
                    }
                    // up to don_burst donations per check while warps starve
                    if (++burst < P.don_burst) --rounds;
                    else burst = 0;
                    continue;
                }
                burst = 0;
            }
            bool overflow = false;
            while (nn > NS - 48) {
                if (nov + SPILL > P.node_cap) {
                    if (lane == 0) raise_error<1, MT>(C, 2);
                    overflow = true;
                    break;
                }
                if (lane < SPILL) ov[nov + lane] = ns[(bot + lane) & (NS - 1)];
                nov += SPILL;
                bot = (bot + SPILL) & (NS - 1);
                nn -= SPILL;
                __syncwarp();
            }
            if (overflow) break;
        }
        const int take = min(16, nn);
        const int base = nn - take;
        const bool active = (lane >> 1) < take;
        ++rounds32;
        uint4 nd = make_uint4(0u, 0u, 0u, 0u);
        if (active) nd = ns[(bot + base + (lane >> 1)) & (NS - 1)];
        nodes32 += take;
        const int p = static_cast<int>(nd.w >> 24);
        const uint2 D = dec2[2 * p + odd];
        const uint4 T = thr[p + 1];
        uint32_t R0 = (nd.z | 0x80808080u) - D.x;
        uint32_t R1 = (nd.z | 0x80808080u) - D.y;
        bool ok0 = active && (R0 & 0x80808080u) == 0x80808080u;
        bool ok1 = active && (R1 & 0x80808080u) == 0x80808080u;
        R0 &= 0x7F7F7F7Fu;
        R1 &= 0x7F7F7F7Fu;
        const bool leaf = p + 1 == l;
        if (prune != 0) {
            // branch-free: both children are checked on every lane (a leaf,
            // or a child that spent no budget, is feasible by construction)
            const bool f0 = swar_feasible<MT>(R0, T, prune);
            const bool f1 = swar_feasible<MT>(R1, T, prune);
            ok0 = ok0 & (leaf | (D.x == 0u) | f0);
            ok1 = ok1 & (leaf | (D.y == 0u) | f1);
        }
        const uint32_t bit = 1u << T.w;
        const uint32_t h = nd.x | (odd ? bit : 0u);
        const uint32_t o1 = nd.y | bit;
        const uint32_t q24 = nd.w + (1u << 24);
        __syncwarp();
        const unsigned lt = lanemask_lt();
        const unsigned lb0 = __ballot_sync(0xffffffffu, ok0 && leaf);
        const unsigned lb1 = __ballot_sync(0xffffffffu, ok1 && leaf);
        const unsigned ib0 = __ballot_sync(0xffffffffu, ok0 && !leaf);
        const unsigned ib1 = __ballot_sync(0xffffffffu, ok1 && !leaf);
        const int n0 = __popc(ib0);
        const int nl0 = __popc(lb0);
        const int b2 = bot + base;
        if (ok0 & leaf) cand[ncand + __popc(lb0 & lt)] = make_uint2(h, nd.y);
        if (ok1 & leaf) cand[ncand + nl0 + __popc(lb1 & lt)] = make_uint2(h, o1);
        if (ok0 & !leaf) ns[(b2 + __popc(ib0 & lt)) & (NS - 1)] = make_uint4(h, nd.y, R0, q24);
        if (ok1 & !leaf) ns[(b2 + n0 + __popc(ib1 & lt)) & (NS - 1)] = make_uint4(h, o1, R1, q24);
        const int nl = nl0 + __popc(lb1);
        ncand += nl;
        leaves32 += nl;
        nn = base + n0 + __popc(ib1);
        __syncwarp();
        if (ncand > cand_cap - 64) {
            verify_all<1, MT>(C, L, entries, ncand);
            ncand = 0;
        }
    }
    leaves += leaves32;
    nodes += nodes32;
    C.add(W_ROUNDS, rounds32);
    if (ncand > 0) verify_all<1, MT>(C, L, entries, ncand);
    nodes_out += nodes;
    leaves_out += leaves;
}

// Root consensus bound: a common neighbour within d of every member exists
// only if the column costs (members minus the most frequent symbol) sum to at
// most t*d — NeighborhoodEnumerator::prune's consensus rule at the root
// (src/neighborhood.cpp:150-154), which fails for every child of the root
// when it fails here. For 5- and 6-tuples most tuples fail it, and the check
// costs a few instructions per position instead of building the tables.
template <int W, int MT>
__device__ __forceinline__ bool root_consensus_ok(const WarpCtx<W, MT>& C, int t, const Lmer<W>* Tm) {
    const int lane = C.lane, l = C.P->l;
    int cost = 0;
    for (int p = lane; p < l; p += 32) {
        uint32_t e = 0;  // byte c: members holding symbol c at p
#pragma unroll
        for (int i = 0; i < MT; ++i)
            if (i < t) e += 1u << (8 * code_at<W>(Tm[i], p));
        const uint32_t m2 = __vmaxu4(e, e >> 16);
        cost += t - static_cast<int>(max(m2 & 0xFFu, (m2 >> 8) & 0xFFu));
    }
    cost = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(cost)));
    return cost <= t * C.P->d;
}

// The same bound for the m members on the stack (u = stack[m-1] included):
// they have a common d-neighbour only if their consensus cost is at most m*d,
// and every deeper member can only add column cost, so a stack that fails it
// has no motif below it. Checked before the push (which it saves) on levels
// of 4+ members; Theorem 1 already decides 3-member stacks exactly.
template <int W, int MT>
__device__ __forceinline__ bool stack_consensus_ok(const WarpCtx<W, MT>& C, int m) {
    const WarpFixed& S = *C.S();
    Lmer<W> Tm[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i)
        if (i < m) Tm[i] = C.lmer(S.stack_id[i] & ID_MASK);
    return root_consensus_ok<W, MT>(C, m, Tm);
}

// Common d-neighbourhood of the t-tuple on the stack + verification. The
// DFS starts from the root, or (ndon > 0) from ndon donated nodes already
// copied to the bottom of the node stack.
template <int W, int MT>
__device__ __noinline__ void enumerate_verify(WarpCtx<W, MT>& C, int t, int ndon) {
    t = tuple_size<MT>(t);
    const SearchParams& P = *C.P;
    const int lane = C.lane;
    WarpFixed& S = *C.S();
    const LevelMeta& L = S.lev[t];
    const uint32_t* entries = level_entries<W, MT>(C, t);
    const long long c0 = clock64();

    Lmer<W> Tm[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i)
        if (i < t) Tm[i] = C.lmer(S.stack_id[i] & ID_MASK);
    if constexpr (MT >= 5) {
        if (ndon == 0 && P.prune == 2 && !P.cons_rows && !root_consensus_ok<W, MT>(C, t, Tm)) {
            C.add(W_TUPLES, 1);
            C.add(W_CLKP, static_cast<unsigned long long>(clock64() - c0));
            return;
        }
    }
    const bool swar = MT <= 4 && P.d <= 31;
    bool fast = false;
    if constexpr (W == 1 && MT <= 4) fast = swar;
    if constexpr (W == 1 && MT <= 4) {
        if (fast) prepare_tuple_fast<MT>(C, t, L, Tm);
    }
    if (!fast) {
        order_positions<W, MT>(C, t, Tm);
        if (swar) prepare_tuple_swar<W, MT>(C, t, L, Tm);
        else prepare_tuple<W, MT>(C, t, L, Tm);
    }

    const uint32_t tmask = (1u << t) - 1u;
    // node stack: circular buffer of NS nodes in shared memory; chunks of
    // SPILL bottom nodes move to a per-warp global overflow LIFO when it
    // fills, and come back when it drains (all hot accesses are LDS/STS)
    constexpr int NS = NodeSmem<W>::N;
    constexpr int SPILL = NS / 4;
    Node<W>* ns = C.node_smem();
    Node<W>* ov = C.node_glob;
    int bot = 0, nn = 0, nov = 0;
    if (ndon > 0) {
        nn = ndon;
    } else {
        if (lane == 0) {
            Node<W> root;
#pragma unroll
            for (int i = 0; i < W; ++i) root.c.h[i] = root.c.o[i] = 0;
            if (swar) {
                uint32_t b = 0;
                for (int i = 0; i < t; ++i) b |= static_cast<uint32_t>(P.d) << (8 * i);
                root.rA = b;
                root.rB = 0;
            } else {
                const uint32_t b = static_cast<uint32_t>(P.d + 64);
                root.rA = b | (b << 8) | (b << 16) | (b << 24);
                root.rB = b | (b << 8) | (b << 16);
            }
            ns[0] = root;
        }
        nn = 1;
    }
    __syncwarp();
    const int prune = P.prune;
    const int cand_cap = P.plan.cand_cap;
    unsigned long long nodes = 0, leaves = 0;
    int ncand = 0, rounds = 0;
    if constexpr (W == 1) {
        if (swar) {
            enum_loop_fast<MT>(C, t, L, entries, bot, nn, nov, nodes, leaves);
            goto done;
        }
    }
    while (nn > 0 || nov > 0) {
        if (nn == 0) {  // refill from the overflow
            nov -= SPILL;
            if (lane < SPILL) ns[(bot + lane) & (NS - 1)] = ov[nov + lane];
            nn = SPILL;
            __syncwarp();
        }
        // donate the shallowest nodes when other warps are starving
        if (P.donate && ((++rounds & P.don_gen_mask) == 0) && (nov >= NDON || nn >= NDON + 16) && starving<W, MT>(C)) {
            TaskHeader h;
            h.anchor = C.anchor;
            h.kind = 1;
            h.k = static_cast<int16_t>(t);
            const int half = NDON;
            h.a0 = half;
            h.a1 = 0;
#pragma unroll
            for (int i = 0; i < MAXT; ++i) h.stack[i] = i < t ? S.stack_id[i] : 0u;
            if (nov >= NDON) {
                const int o0 = nov - NDON;
                publish<W, MT>(C, h, NDON, [&](int x) { return ov[o0 + x]; });
                nov -= NDON;
            } else {
                const int b0 = bot;
                publish<W, MT>(C, h, half, [&](int x) { return ns[(b0 + x) & (NS - 1)]; });
                bot = (bot + half) & (NS - 1);
                nn -= half;
            }
            continue;
        }
        bool overflow = false;
        while (nn > NS - 48) {  // spill bottom chunks: a round may add 48 nodes net
            if (nov + SPILL > P.node_cap) {
                if (lane == 0) raise_error<W, MT>(C, 2);
                overflow = true;
                break;
            }
            if (lane < SPILL) ov[nov + lane] = ns[(bot + lane) & (NS - 1)];
            nov += SPILL;
            bot = (bot + SPILL) & (NS - 1);
            nn -= SPILL;
            __syncwarp();
        }
        if (overflow) break;
        const int take = min(16, nn);
        const int base = nn - take;
        const int slot = lane >> 1;
        const bool active = slot < take;
        Node<W> nd;
        if (active) nd = ns[(bot + base + slot) & (NS - 1)];
        __syncwarp();
        nodes += take;
        Node<W> ch0, ch1;
        bool leaf0 = false, leaf1 = false, ok0 = false, ok1 = false;
        if (active) {
            const int c = (lane & 1) * 2;
            if (swar) {
                ok0 = expand_child_swar<W, MT>(C, nd, c, prune, ch0, leaf0);
                ok1 = expand_child_swar<W, MT>(C, nd, c + 1, prune, ch1, leaf1);
            } else {
                ok0 = expand_child<W, MT>(C, nd, c, t, tmask, prune, ch0, leaf0);
                ok1 = expand_child<W, MT>(C, nd, c + 1, t, tmask, prune, ch1, leaf1);
            }
        }
        // leaves -> candidate buffer; internal children -> stack
        const unsigned lb0 = __ballot_sync(0xffffffffu, ok0 && leaf0);
        const unsigned lb1 = __ballot_sync(0xffffffffu, ok1 && leaf1);
        const unsigned ib0 = __ballot_sync(0xffffffffu, ok0 && !leaf0);
        const unsigned ib1 = __ballot_sync(0xffffffffu, ok1 && !leaf1);
        const unsigned lt = lanemask_lt();
        if (ok0 && leaf0) C.cand()[ncand + __popc(lb0 & lt)] = ch0.c;
        if (ok1 && leaf1) C.cand()[ncand + __popc(lb0) + __popc(lb1 & lt)] = ch1.c;
        const int nl = __popc(lb0) + __popc(lb1);
        if (ok0 && !leaf0) ns[(bot + base + __popc(ib0 & lt)) & (NS - 1)] = ch0;
        if (ok1 && !leaf1) ns[(bot + base + __popc(ib0) + __popc(ib1 & lt)) & (NS - 1)] = ch1;
        ncand += nl;
        leaves += nl;
        nn = base + __popc(ib0) + __popc(ib1);
        __syncwarp();
        if (ncand > cand_cap - 64) {
            verify_all<W, MT>(C, L, entries, ncand);
            ncand = 0;
        }
    }
    if (ncand > 0) verify_all<W, MT>(C, L, entries, ncand);
done:
    C.add(W_TUPLES, ndon > 0 ? 0 : 1);
    C.add(W_LEAVES, leaves);
    C.add(W_NODES, nodes);
    C.add(W_CLKP, static_cast<unsigned long long>(clock64() - c0));
}

// ---------------------------------------------------------------- DFS driver
// Depth-first over levels kmin..t-1 (recurse, src/solver.cpp:406-419), the
// branch range of level kmin given by the task.
template <int W, int MT>
__device__ void dfs(WarpCtx<W, MT>& C, int kmin, int it0, int it1) {
    const SearchParams& P = *C.P;
    WarpFixed& S = *C.S();
    const int t = P.t;
    if (C.lane == 0) {
        S.iter[kmin] = it0;
        S.iter_end[kmin] = it1;
    }
    __syncwarp();
    // (the stack consensus bound is applied by the push filters to every
    // remaining row, so each branching-row entry already satisfies it)
    int k = kmin;
    while (k >= kmin) {
        const LevelMeta& L = S.lev[k];
        const int it = S.iter[k];
        const int end = S.iter_end[k];
        if (it >= end) {
            --k;
            continue;
        }
        const uint32_t uu = level_entries<W, MT>(C, k)[L.start[L.branch] + it];
        __syncwarp();
        if (C.lane == 0) {
            S.iter[k] = it + 1;
            S.stack_id[k] = uu;
        }
        __syncwarp();
        maybe_donate_dfs<W, MT>(C, kmin, k);
        const bool ok = (k + 1 == t && P.lazy) ? lazy_push<W, MT>(C, k) : filter_push<W, MT>(C, k);
        if (!ok) continue;
        if (k + 1 == t) {
            enumerate_verify<W, MT>(C, t, 0);
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

// Load the anchor's level-1 row table and set stack[0].
template <int W, int MT>
__device__ void begin_anchor(WarpCtx<W, MT>& C, int ai) {
    const SearchParams& P = *C.P;
    WarpFixed& S = *C.S();
    C.anchor = ai;
    C.l1 = P.l1_entries + static_cast<size_t>(ai) * P.K;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(P.l1_meta + ai);
    uint32_t* dstm = reinterpret_cast<uint32_t*>(&S.lev[1]);
    for (int x = C.lane; x < static_cast<int>(sizeof(LevelMeta) / 4); x += 32) dstm[x] = src[x];
    if (C.lane == 0) {
        const uint32_t a = static_cast<uint32_t>(P.anchor_off[ai]);
        S.stack_id[0] = a;
        if constexpr (MT >= 4) cache_member<W>(S, 0, C.lmer(a & ID_MASK));
    }
    __syncwarp();
}

}  // namespace

// NW is the launch bound (warps per block): 16 warps x 128 registers, or for
// the short-task l <= 32, t <= 3 searches 12 warps x 168 registers (no spills
// in the verification pass; measured faster on (13,4) and (17,6), slower on
// (21,8)).
template <int W, int MT, int NW>
__global__ void __launch_bounds__(32 * NW, 1) search_kernel(const __grid_constant__ SearchParams P) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    // strided copy of the l-mer table into shared memory (a TMA bulk copy,
    // tma_stage, measured 1-4 % slower here: it perturbs the register
    // allocation of the whole persistent kernel; the scanner uses it)
    Lmer<W>* T = reinterpret_cast<Lmer<W>*>(dyn_smem);
    const Lmer<W>* gT = static_cast<const Lmer<W>*>(P.table);
    WarpCtx<W, MT> C;
    uint32_t table_rows = 0;
    if constexpr (kGlobalTable<W>) {
        C.gt = gT;  // read in place (L2-resident, through L1)
    } else {
        C.gt = nullptr;
        for (int i = threadIdx.x; i < P.K; i += blockDim.x) T[i] = gT[i];
        table_rows = static_cast<uint32_t>(P.K);
        __syncthreads();
    }
    const uint32_t table_bytes = (table_rows * static_cast<uint32_t>(sizeof(Lmer<W>)) + 15u) / 16u * 16u;
    const uint32_t wbase = table_bytes + static_cast<uint32_t>(P.plan.bytes) * warp;

    C.P = &P;
    C.off_S = wbase;
    C.off_thr = wbase + P.plan.off_thr;
    C.off_cand = wbase + P.plan.off_cand;
    C.off_nodes = wbase + P.plan.off_nodes;
    const size_t gw = static_cast<size_t>(blockIdx.x) * nwarps + warp;
    uint32_t* scratch = P.scratch + gw * P.scratch_words;
    C.lvl_glob = scratch;
    C.node_glob = reinterpret_cast<Node<W>*>(scratch + static_cast<size_t>(P.t > 1 ? P.t - 1 : 0) * P.level_cap);
    C.thr_glob = reinterpret_cast<uint8_t*>(C.node_glob + P.node_cap);
    C.lane = lane;
    C.pushes_since_check = 0;
    if (lane < W_N) C.S()->ctr[lane] = 0;
    if (lane == 0) {
        C.S()->lazy_level = 0;
        C.S()->lazy_mask = 0u;
    }
    __syncwarp();
    WarpFixed& S = *C.S();
    const int t = P.t;
    const unsigned long long nstatic = P.nexplicit > 0 ? static_cast<unsigned long long>(P.nexplicit)
                                                     : static_cast<unsigned long long>(P.task_base[P.nanchors]);
    QueueState* qs = P.qs;
    const unsigned long long qcap = static_cast<unsigned long long>(P.qcap);
    if (lane == 0) {
        S.wait.waiting = 0;
        S.wait.chunk_next = S.wait.chunk_end = 0;
    }

    for (;;) {
        // ---- claim a task (lane 0), protocol in DESIGN.md §4
        unsigned long long idx = 0;
        int kind = lane == 0 ? claim_task(P, nstatic, S.wait, idx) : -1;
        kind = __shfl_sync(0xffffffffu, kind, 0);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (kind == 2) break;
        if (kind < 0) continue;
        if (P.jitter_ns && lane == 0) jitter_sleep(P, idx + 1 + (static_cast<unsigned long long>(kind) << 40) +
                                                         (static_cast<unsigned long long>(gw) << 44));
        const long long task_t0 = clock64();
        if ((P.timeline || P.log_cycles) && lane == 0) {
            // diagnostics only; kept in shared memory, not in registers
            unsigned long long ns0;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns0));
            S.diag[0] = S.ctr[W_TUPLES];
            S.diag[1] = S.ctr[W_LEAVES];
            S.diag[2] = S.ctr[W_NODES];
            S.diag[3] = S.ctr[W_VCMP];
            S.diag[4] = ns0;
        }
        C.add(W_TASKS, 1);
        if (kind == 0 && P.nexplicit > 0) {
            // explicit (S1 l-mer, depth-1 branch) task: locate u in the
            // anchor's branching row (t >= 2)
            begin_anchor<W, MT>(C, P.task_ai[idx]);
            const uint32_t u = P.task_u[idx];
            const LevelMeta& L1 = S.lev[1];
            int j = -1;
            if (L1.viable) {
                const int st = L1.start[L1.branch], cnt = L1.cnt[L1.branch];
                for (int b0 = 0; b0 < cnt && j < 0; b0 += 32) {
                    const bool hit = b0 + lane < cnt && (C.l1[st + b0 + lane] & ID_MASK) == u;
                    const unsigned bal = __ballot_sync(0xffffffffu, hit);
                    if (bal) j = b0 + __ffs(bal) - 1;
                }
            }
            if (j >= 0) dfs<W, MT>(C, 1, j, j + 1);
        } else if (kind == 0) {
            if (P.task_order) idx = P.task_order[idx];
            // anchor: last a with task_base[a] <= idx
            int lo = 0, hi = P.nanchors - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (static_cast<unsigned long long>(P.task_base[mid]) <= idx) lo = mid;
                else hi = mid - 1;
            }
            begin_anchor<W, MT>(C, lo);
            const int j = static_cast<int>(idx - static_cast<unsigned long long>(P.task_base[lo]));
            if (t == 1) enumerate_verify<W, MT>(C, 1, 0);
            else dfs<W, MT>(C, 1, j, j + 1);
        } else {
            const uint8_t* slot = P.qslots + (idx % static_cast<unsigned long long>(P.qcap)) * P.qslot_bytes;
            const uint32_t* hs = reinterpret_cast<const uint32_t*>(slot);
            uint32_t* hd = reinterpret_cast<uint32_t*>(&S.task);
            for (int x = lane; x < static_cast<int>(sizeof(TaskHeader) / 4); x += 32) hd[x] = __ldcg(hs + x);
            __syncwarp();
            // copy donated nodes out of the slot right away (the ring reuses it)
            const int ndon = S.task.kind == 1 ? S.task.a0 : 0;
            {
                const uint32_t* src = reinterpret_cast<const uint32_t*>(slot + sizeof(TaskHeader));
                constexpr int NW = sizeof(Node<W>) / 4;
                for (int x = lane; x < ndon; x += 32) {
                    Node<W> nd;
                    uint32_t* w = reinterpret_cast<uint32_t*>(&nd);
#pragma unroll
                    for (int q = 0; q < NW; ++q) w[q] = __ldcg(src + x * NW + q);
                    C.node_smem()[x] = nd;
                }
            }
            __syncwarp();
            // install the handed-off level (row table + entries) into this
            // warp's own level buffer
            const int hl = static_cast<int>(S.task.hlevel);
            if (hl >= 2) {
                const uint32_t* lm = reinterpret_cast<const uint32_t*>(slot + P.qslot_lvl_off);
                constexpr int MW = static_cast<int>(sizeof(LevelMeta) / 4);
                uint32_t* md = reinterpret_cast<uint32_t*>(&S.lev[hl]);
                for (int x = lane; x < MW; x += 32) md[x] = __ldcg(lm + x);
                __syncwarp();
                const int tot = S.lev[hl].total;
                uint32_t* ed = level_entries<W, MT>(C, hl);
                const uint32_t* es = lm + MW;
                for (int x = lane; x < tot; x += 32) ed[x] = __ldcg(es + x);
                __syncwarp();
            }
            if (lane == 0) {
                __threadfence();
                atomicExch(&P.qstate[idx % qcap], 2u * static_cast<unsigned int>(idx / qcap) + 2u);
            }
            const int tk = S.task.k;
            long long tdiag[3] = {0, 0, 0};
            if (P.log_cycles) tdiag[0] = clock64() - task_t0;
            begin_anchor<W, MT>(C, S.task.anchor);
            if (lane < MAXT && lane >= 1 && lane < tk) {
                S.stack_id[lane] = S.task.stack[lane];
                if constexpr (MT >= 4) cache_member<W>(S, lane, C.lmer(S.task.stack[lane] & ID_MASK));
            }
            __syncwarp();
            if (P.log_cycles) tdiag[1] = clock64() - task_t0;
            // replay the prefix pushes to rebuild levels 2..tk (from the
            // handed-off level on when there is one)
            bool ok = true;
            for (int i = hl >= 2 ? hl : 1; i < tk && ok; ++i) {
                ok = (i + 1 == t && P.lazy) ? lazy_push<W, MT>(C, i) : filter_push<W, MT>(C, i);
                if (P.log_cycles && i == 1) tdiag[2] = clock64() - task_t0;
                C.add(W_REPLAYS, 1);
                C.add(W_PUSH, ~0ull);  // replays are not new tree nodes
                if (ok) C.add(W_VIABLE, ~0ull);
            }
            if (P.log_cycles && lane == 0) {
                S.diag[3] = static_cast<unsigned long long>(clock64() - task_t0);
                S.diag[0] = S.ctr[W_TUPLES] - static_cast<unsigned long long>(tdiag[0]);  // decoded below
                S.diag[1] = S.ctr[W_LEAVES] - static_cast<unsigned long long>(tdiag[1]);
                S.diag[2] = S.ctr[W_NODES] - static_cast<unsigned long long>(tdiag[2]);
            }
            if (!ok) {
                if (lane == 0) raise_error<W, MT>(C, 4);
            } else if (S.task.kind == 0) {
                dfs<W, MT>(C, tk, S.task.a0, S.task.a1);
            } else {
                enumerate_verify<W, MT>(C, tk, ndon);
            }
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicSub(&qs->busy, 1u);
            const long long dt = clock64() - task_t0;
            if (P.timeline) {
                unsigned long long ns1;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns1));
                const unsigned long long slot = atomicAdd(P.counters + C_TLN, 1ull);
                if (static_cast<long long>(slot) < P.timeline_cap) {
                    const unsigned long long kd = kind == 0 ? 0ull : 1ull + S.task.kind;
                    P.timeline[2 * slot] = S.diag[4];
                    P.timeline[2 * slot + 1] = ns1 | (kd << 62);
                }
            }
            if ((P.log_cycles > 0 && dt > P.log_cycles) || (P.log_cycles < 0 && kind != 0 && dt > -P.log_cycles)) {
                const unsigned long long slot = atomicAdd(P.counters + C_LOGN, 1ull);
                if (slot < 32) {
                    unsigned long long* r = P.counters + C_LOG0 + 8 * slot;
                    r[0] = kind == 0 ? 0ull : 1ull + S.task.kind;
                    r[1] = static_cast<unsigned long long>(C.anchor);
                    r[2] = idx;
                    r[3] = static_cast<unsigned long long>(dt);
                    r[4] = S.ctr[W_TUPLES] - S.diag[0];
                    r[5] = S.ctr[W_LEAVES] - S.diag[1];
                    r[6] = S.ctr[W_NODES] - S.diag[2];
                    r[7] = kind == 0 ? 0ull : S.diag[3];  // cycles before the task's own search (claim + replays)
                }
            }
            const int hb = kind == 0 ? C_HIST0 : (S.task.kind == 0 ? C_HIST_DON0 : C_HIST_DON1);
            atomicAdd(P.counters + hb + min(39, 63 - __clzll(dt > 0 ? dt : 1)), 1ull);
        }
    }
    __syncwarp();
    if (lane == 0) {
        const int map[W_N] = {C_PUSHES, C_VIABLE, C_SLOTS,    C_TUPLES,   C_LEAVES,     C_EMITTED,
                              C_VCMP,   C_NODES,  C_PAIR_REJ, C_TRI_REJ,  C_TASKS,      C_DONATED,
                              C_REPLAYS, C_CLK_FILTER, C_CLK_PATTERN, C_CONS_REJ, C_ROUNDS};
#pragma unroll
        for (int i = 0; i < W_N; ++i) atomicAdd(P.counters + map[i], S.ctr[i]);
    }
}

// ---------------------------------------------------------------- host side

// which (W, MT) builds also exist with the 12-warp launch bound
template <int W, int MT>
constexpr bool has_deep() {
    return W == 1 && MT <= 3;
}

int search_default_warps(int W, int t) { return W == 1 && t <= 3 ? 12 : 16; }


template <int W>
WarpPlan make_plan_t(int l, int t) {
    WarpPlan p{};
    const int tt = t < 1 ? 1 : t;
    p.npair = tt * (tt - 1) / 2;
    p.ntri = tt * (tt - 1) * (tt - 2) / 6;
    int off = warp_fixed_bytes(tt < 2 ? 2 : tt);  // t = 1 runs the two-member build
    if ((tt < 2 ? 2 : tt) >= PMS8G_QUEUE_MT) off += (static_cast<int>(sizeof(PushQueue)) + 15) / 16 * 16;
    p.off_thr = off;
    const int generic_thr = (GEN_TBL_BYTES + (l + 1) * (p.npair + p.ntri) + 15) / 16 * 16;
    const int swar_thr = 16 * ((l + 3) & ~3) + 16 * (l + 1);
    p.thr_global_bytes = 0;
    if (tt >= 5) p.thr_global_bytes = generic_thr;  // (the SWAR tables serve t <= 4 only)
    else off += generic_thr > swar_thr ? generic_thr : swar_thr;
    // t >= 5: enumeration is rare (few tuples survive that deep); a small
    // per-warp footprint leaves more of the SM's 256 KB to the L1 that serves
    // the two-word l-mer table ((50,21): 195 -> 154 KB per CTA, -5%)
    p.cand_cap = tt >= 5 ? 64 : 32 * MAXCH;
    p.off_cand = off;
    off += p.cand_cap * static_cast<int>(sizeof(Lmer<W>));
    off = (off + 15) / 16 * 16;
    p.node_smem = NodeSmem<W>::N;
    p.off_nodes = off;
    off += p.node_smem * static_cast<int>(sizeof(Node<W>));
    p.bytes = (off + 15) / 16 * 16;
    return p;
}

WarpPlan make_plan(int W, int l, int t) { return W == 1 ? make_plan_t<1>(l, t) : make_plan_t<2>(l, t); }

size_t node_bytes(int W) { return W == 1 ? sizeof(Node<1>) : sizeof(Node<2>); }

size_t search_smem(int W, int K, int warps, const WarpPlan& plan) {
    // two-word builds read the table from global memory
    const size_t rows = W == 2 ? 0 : static_cast<size_t>(K);
    return (rows * lmer_bytes(W) + 15) / 16 * 16 + static_cast<size_t>(plan.bytes) * warps;
}

// slot = header | NDON nodes | (don_cap > 0) LevelMeta + don_cap entries
size_t task_slot_level_offset(int W) { return (sizeof(TaskHeader) + NDON * node_bytes(W) + 15) / 16 * 16; }
size_t task_slot_bytes(int W, int don_cap) {
    size_t b = task_slot_level_offset(W);
    if (don_cap > 0) b += sizeof(LevelMeta) + sizeof(uint32_t) * static_cast<size_t>(don_cap);
    return (b + 127) / 128 * 128;
}

template <int W, int MT>
cudaError_t set_smem_t(size_t bytes) {
    cudaError_t e = cudaFuncSetAttribute(search_kernel<W, MT, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bytes));
    if constexpr (has_deep<W, MT>()) {
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(search_kernel<W, MT, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(bytes));
    }
    return e;
}

// The kernel is specialised on the switch depth (tuple size) so that every
// per-member loop is unrolled over registers; t = 1 runs the MT = 2 build.
cudaError_t set_search_smem(int W, int t, size_t bytes) {
    const int mt = t < 2 ? 2 : t;
    // the attribute only ever grows (per build and device), so contexts with
    // smaller plans never lower it under another context's launch
    static std::mutex mu;
    static size_t granted[2][MAXT + 1][64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    size_t& cur = granted[W - 1][mt][dev & 63];
    if (bytes <= cur) return cudaSuccess;
#define PMS8G_CASE(WW, M)                                 \
    if (W == WW && mt == M) {                             \
        const cudaError_t e = set_smem_t<WW, M>(bytes);   \
        if (e == cudaSuccess) cur = bytes;                \
        return e;                                         \
    }
    PMS8G_CASE(1, 2) PMS8G_CASE(1, 3) PMS8G_CASE(1, 4) PMS8G_CASE(1, 5) PMS8G_CASE(1, 6) PMS8G_CASE(1, 7)
    PMS8G_CASE(2, 2) PMS8G_CASE(2, 3) PMS8G_CASE(2, 4) PMS8G_CASE(2, 5) PMS8G_CASE(2, 6) PMS8G_CASE(2, 7)
#undef PMS8G_CASE
    return cudaErrorInvalidValue;
}

cudaError_t launch_search(int W, const SearchParams& P, int blocks, int warps, size_t smem, cudaStream_t s) {
    const int mt = P.t < 2 ? 2 : P.t;
#define PMS8G_CASE(WW, M)                                                 \
    if (W == WW && mt == M) {                                             \
        if constexpr (has_deep<WW, M>()) {                                \
            if (warps <= 12) {                                            \
                search_kernel<WW, M, 12><<<blocks, warps * 32, smem, s>>>(P); \
                return cudaGetLastError();                                \
            }                                                             \
        }                                                                 \
        search_kernel<WW, M, 16><<<blocks, warps * 32, smem, s>>>(P);     \
        return cudaGetLastError();                                        \
    }
    PMS8G_CASE(1, 2) PMS8G_CASE(1, 3) PMS8G_CASE(1, 4) PMS8G_CASE(1, 5) PMS8G_CASE(1, 6) PMS8G_CASE(1, 7)
    PMS8G_CASE(2, 2) PMS8G_CASE(2, 3) PMS8G_CASE(2, 4) PMS8G_CASE(2, 5) PMS8G_CASE(2, 6) PMS8G_CASE(2, 7)
#undef PMS8G_CASE
    return cudaErrorInvalidValue;
}

}  // namespace pms8g
