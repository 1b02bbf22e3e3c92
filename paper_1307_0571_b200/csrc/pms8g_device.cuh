// pms8g_device.cuh — device-side data layout shared by the kernels and the host
// launcher. See DESIGN.md §3 for the HBM/SMEM layout.
#pragma once
#include <cstddef>
#include <cstdint>

namespace pms8g {

constexpr int MAXT = 7;   // deepest switch depth (stack size at enumeration)
constexpr int MAXN = 32;  // rows (sequences) handled by one warp's row tables
constexpr int NPAIR = MAXT * (MAXT - 1) / 2;
constexpr int NTRI = MAXT * (MAXT - 1) * (MAXT - 2) / 6;
constexpr int CANDCAP = 64;
constexpr uint32_t ID_MASK = 0xFFFFFFu;  // entry = row << 24 | l-mer id

// An l-mer as two bit planes: symbol code c at position p sets bit p of
// h (c >> 1) and of o (c & 1). W 32-bit words per plane (l <= 32W).
template <int W>
struct Lmer {
    uint32_t h[W];
    uint32_t o[W];
};

// Row table of one level: rows in physical storage order.
struct LevelMeta {
    uint32_t start[MAXN];
    uint32_t cnt[MAXN];
    uint8_t order[MAXN];  // row id at physical position j
    int32_t nrows;
    int32_t total;
    int32_t branch;  // physical position of the branching row
    int32_t viable;
};

// Global counters (index into SearchParams::counters).
enum Ctr {
    C_PUSHES = 0,
    C_VIABLE,
    C_SLOTS,
    C_TUPLES,
    C_LEAVES,
    C_EMITTED,
    C_VCMP,
    C_NODES,
    C_CLK_FILTER,
    C_CLK_PATTERN,
    C_PAIR_REJ,   // slots rejected by the pair rule
    C_TRI_REJ,    // slots rejected by the Theorem-1 triple rule
    C_TASKS,      // tasks processed
    C_DONATED,    // dynamic tasks donated
    C_REPLAYS,    // filter pushes replayed by receivers of donated tasks
    C_HIST0,      // task duration histogram: C_HIST0 + floor(log2(cycles)), 40 buckets
    C_IDLE = C_HIST0 + 40,  // warp cycles spent without a task (claim loop, incl. the final wait)
    C_HIST_DON0,            // the same histogram for donated branch ranges (kind 0), 40 buckets
    C_HIST_DON1 = C_HIST_DON0 + 40,  // ... and for donated node batches (kind 1)
    C_LOGN = C_HIST_DON1 + 40,       // diagnostics: number of long tasks logged
    C_LOG0,                          // 32 records x 8 words: kind, anchor, idx, cycles, tuples, leaves, nodes, vcmp
    C_TLN = C_LOG0 + 256,            // diagnostics: timeline records written
    C_STATIC,                        // static tasks claimed by this device
    C_CONS_REJ,                      // slots rejected by the stack consensus row rule
    C_ROUNDS,                        // enumeration rounds (a round pops up to 16 nodes)
    C_LVL0,                          // diagnostics (PMS8G_LEVELSTATS builds): per push level k, 6 words:
                                     // pushes, stopped early, slots, survivors of the cheap rules, kept, blocks with a cheap survivor
    C_NCTR = C_LVL0 + 48
};

constexpr int NDON = 32;  // enumeration nodes per donated task

// Global work-queue state (zeroed per run). Static tasks are the (S1 l-mer,
// depth-1 branch) pairs indexed through task_base; dynamic tasks are
// donated by busy warps while other warps wait.
struct QueueState {
    unsigned long long static_next;  // next static task
    unsigned long long head;         // next dynamic slot to consume
    unsigned long long alloc;        // dynamic slots reserved by producers
    unsigned long long heartbeat;    // bumped by busy warps while others wait (watchdog)
    unsigned int busy;               // warps holding a task
    unsigned int waiting;            // warps idle, waiting for work
    unsigned long long pad[4];
};

// Dynamic task slot: header, NDON nodes (kind 1), then the donor's row table
// and entries of one level (hand-off, see below).
struct TaskHeader {
    int32_t anchor;  // anchor index
    int16_t kind;    // 0: branch range [a0, a1) at level k; 1: a0 enumeration nodes of the k-tuple
    int16_t k;
    int32_t a0, a1;
    uint32_t stack[MAXT];
    // Level hand-off: the donor copies level `hlevel` (k for kind 0, k - 1
    // for kind 1) into the slot, so the receiver installs it instead of
    // replaying the prefix pushes 1..hlevel-1 (a replayed depth-1 push of
    // (50,21) filters ~9,500 entries; installing copies <= 8,000 words).
    // hlevel = 0: nothing handed off (level 1 is the shared row table, or the
    // level is larger than SearchParams::don_cap) - the receiver replays.
    uint32_t hlevel;
    uint32_t pad;
};

// Per-warp shared-memory plan (byte offsets inside the warp's region),
// computed on the host from (W, l, t).
struct WarpPlan {
    int bytes;
    int off_thr;    // uint8 [(l+1) * (npair(t) + ntri(t))]
    int off_cand;   // Lmer<W> [cand_cap]
    int off_nodes;  // Node<W> [node_smem]
    int cand_cap;
    int node_smem;
    int npair, ntri;
    int thr_global_bytes;  // > 0: the enumeration tables live in the warp's global scratch (t >= 5)
};

struct SearchParams {
    int n, m, l, d, w, K, t, prune, sort_rows;
    const void* table;            // Lmer<W>[K]
    const uint32_t* l1_entries;   // [nanchors][K]
    const LevelMeta* l1_meta;     // [nanchors]
    const int32_t* anchor_off;    // [nanchors]
    const long long* task_base;   // [nanchors + 1]
    int nanchors;
    const int32_t* task_ai;       // explicit branch tasks: anchor index ...
    const uint32_t* task_u;       // ... and depth-1 l-mer id (nexplicit > 0)
    long long nexplicit;
    QueueState* qs;
    uint8_t* qslots;              // [qcap][qslot_bytes]
    unsigned int* qstate;         // [qcap] slot round state (2r free, 2r+1 published)
    int qcap, qslot_bytes;
    int donate;                   // 1: donate work to idle warps
    int don_pushes;               // DFS pushes between starvation checks
    long long log_cycles;         // diagnostics: log tasks longer than this (0: off)
    unsigned long long* timeline; // diagnostics: per-task {start ns, end ns | kind << 62} records (or null)
    long long timeline_cap;
    const uint32_t* task_order;   // static task permutation (heaviest first), or null
    int don_rounds_mask;          // enumeration rounds between starvation checks - 1 (power of two - 1)
    int don_burst;                // node batches donated per check at most
    int don_gen_mask;             // generic enumeration loop: rounds between starvation checks - 1 (power of two - 1)
    int lazy;                     // 1: rows of the final level are filtered on demand
    int reorder;   // 1: agreement-first enumeration order (0: natural, exact_tree)
    uint32_t* scratch;            // per-warp level storage + node stack
    size_t scratch_words;         // uint32 words per warp
    int level_cap;                // entries per level buffer
    int node_cap;                 // nodes per warp stack (global part)
    WarpPlan plan;
    unsigned long long* keys;     // 2 x u64 per motif key {lo, hi}
    unsigned long long* key_count;
    long long key_cap;
    unsigned long long* counters;
    int* error_flag;
    // cross-GPU static queue (pms8g_queue): when set, static
    // tasks are claimed from this counter in another (or this) device's HBM,
    // shared by every rank over NVLink: value = epoch << 40 | next task
    unsigned long long* gqueue;
    unsigned long long gepoch;
    // test hook: sleep a seeded pseudo-random 0..jitter_ns ns before each task
    unsigned long long jitter_ns;
    unsigned long long jitter_seed;
    int cons_rows;  // 1: push filters apply the stack consensus bound to every remaining row
    int don_cap;       // level entries a dynamic task slot can carry (0: no hand-off)
    int qslot_lvl_off; // byte offset of the handed-off LevelMeta + entries inside a slot
    int claim_chunk;                // shared queue: static tasks per CAS far from the tail
    long long chunk_until;          // ... while more than this many remain
};

constexpr int GQ_SHIFT = 40;
constexpr unsigned long long GQ_MASK = (1ull << GQ_SHIFT) - 1ull;

}  // namespace pms8g
