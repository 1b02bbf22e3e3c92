// pms8g_sigma.h — the search for alphabets of 5..32 symbols (pms8g_sigma.cu):
// parameters and host launchers. Shares the LevelMeta row tables, the task
// scan and the key sort of the DNA path (pms8g_device.cuh, pms8g_capi.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "pms8g_device.cuh"

namespace pms8g {

// per-warp counters of the sigma kernel (mapped onto the Ctr slots)
enum { W_SIGMA_PUSH, W_SIGMA_VIABLE, W_SIGMA_SLOTS, W_SIGMA_TUPLES, W_SIGMA_LEAVES, W_SIGMA_EMIT, W_SIGMA_VCMP,
       W_SIGMA_NODES, W_SIGMA_N };

struct SigmaParams {
    int n, m, l, d, w, K, t, sigma, prune;
    const void* table;            // LmerS<B>[K]
    const uint32_t* l1_entries;   // [nanchors][K]
    const LevelMeta* l1_meta;     // [nanchors]
    const int32_t* anchor_off;    // [nanchors]
    const long long* task_base;   // [nanchors + 1]
    int nanchors;
    unsigned long long* next_task;  // static task counter (zeroed per run)
    uint32_t* scratch;            // per warp: levels 2..t, then the node stack
    size_t scratch_words;
    int level_cap, node_cap;
    unsigned long long* keys;
    unsigned long long* key_count;
    long long key_cap;
    unsigned long long* counters;
    int* error_flag;
};

// bit planes per symbol for a sigma-symbol alphabet (ceil(log2 sigma), >= 2)
inline int sigma_planes(int sigma) {
    int b = 1;
    while ((1 << b) < sigma) ++b;
    return b < 2 ? 2 : b;
}

size_t sigma_lmer_bytes(int B);
size_t sigma_node_bytes();
size_t sigma_warp_smem();
cudaError_t launch_encode_sigma(int B, const uint8_t* codes, int n, int m, int l, int w, int sigma, void* table,
                                int* err, cudaStream_t s);
cudaError_t launch_rowbuild_sigma(int B, const void* table, int n, int w, int d, int K, const int32_t* anchor_off,
                                  int nanchors, uint32_t* l1_entries, LevelMeta* l1_meta,
                                  unsigned long long* counters, cudaStream_t s);
cudaError_t launch_search_sigma(int B, const SigmaParams& P, int blocks, int warps, cudaStream_t s);
cudaError_t launch_reverify_sigma(int B, const void* table, int n, int w, int l, int d,
                                  const unsigned long long* keys, long long count, int* fail, cudaStream_t s);

}  // namespace pms8g
