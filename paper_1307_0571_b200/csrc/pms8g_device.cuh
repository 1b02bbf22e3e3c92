// pms8g_device.cuh — device-side data layout shared by the kernels and the host
// launcher. See DESIGN.md §3 for the HBM/SMEM layout.
#pragma once
#include <cstddef>
#include <cstdint>

namespace pms8g {

constexpr int MAXT = 6;   // deepest switch depth (stack size at enumeration)
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
    uint16_t start[MAXN];
    uint16_t cnt[MAXN];
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
    C_NCTR
};

struct SearchParams {
    int n, m, l, d, w, K, t, prune, sort_rows;
    const void* table;            // Lmer<W>[K]
    const uint32_t* l1_entries;   // [nanchors][K]
    const LevelMeta* l1_meta;     // [nanchors]
    const int32_t* anchor_off;    // [nanchors]
    const long long* task_base;   // [nanchors + 1]
    int nanchors;
    unsigned long long* task_counter;
    uint32_t* scratch;            // per-warp level storage + node stack
    size_t scratch_words;         // uint32 words per warp
    int level_cap;                // entries per level buffer
    int node_cap;                 // nodes per warp stack
    unsigned long long* keys;     // 2 x u64 per motif key {lo, hi}
    unsigned long long* key_count;
    long long key_cap;
    unsigned long long* counters;
    int* error_flag;
};

}  // namespace pms8g
