// pms8g_launch.h — host-side launchers of the kernels in pms8g_kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "pms8g_device.cuh"

namespace pms8g {

size_t lmer_bytes(int W);
size_t node_bytes(int W);
WarpPlan make_plan(int W, int l, int t);
size_t search_smem(int W, int K, int warps, const WarpPlan& plan);
size_t task_slot_bytes(int W, int don_cap);
size_t task_slot_level_offset(int W);

cudaError_t launch_encode(int W, const uint8_t* codes, int n, int m, int l, int w, void* table, int* err,
                          cudaStream_t s);
cudaError_t launch_rowbuild(int W, const void* table, int n, int w, int d, int K, int sort_rows,
                            const int32_t* anchor_off, int nanchors, uint32_t* l1_entries, LevelMeta* l1_meta,
                            unsigned long long* counters, cudaStream_t s);
cudaError_t launch_taskscan(const LevelMeta* l1_meta, int nanchors, int t, long long* task_base, cudaStream_t s);
int search_default_warps(int W, int t);  // launch shape: 12 or 16 warps per block
cudaError_t launch_taskorder(int W, const void* table, const uint32_t* l1_entries, const LevelMeta* l1_meta,
                             const int32_t* anchor_off, const long long* task_base, int nanchors, int K,
                             long long cap, uint32_t* keys, uint32_t* vals, cudaStream_t s);
cudaError_t set_search_smem(int W, int t, size_t bytes);
cudaError_t launch_search(int W, const SearchParams& P, int blocks, int warps, size_t smem, cudaStream_t s);
cudaError_t launch_reverify(int W, const void* table, int n, int w, int l, int d, const unsigned long long* keys,
                            long long count, int* fail, cudaStream_t s);
cudaError_t launch_witness(int W, const void* table, int n, int w, int l, int d, int sigma, const uint8_t* motifs,
                           long long nmotifs, int32_t* witness, uint8_t* pass, cudaStream_t s);
cudaError_t launch_sweep(int W, const void* table, int n, int w, int l, int d, int sigma, unsigned long long total,
                         unsigned long long* keys, unsigned long long* count, long long cap, int sms,
                         cudaStream_t s);
cudaError_t launch_intpeak(int which, int blocks, int threads, int iters, uint32_t* sink, cudaStream_t s);

}  // namespace pms8g
