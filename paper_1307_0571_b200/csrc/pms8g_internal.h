// pms8g_internal.h — host-side internals shared by the C ABI translation units
// (pms8g_capi.cu, pms8g_multi.cu). Not part of the public boundary.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <functional>

#include "../../include/pms8g.h"

// Cross-GPU static task queue (pms8g_queue_*): one 64-bit claim counter.
struct pms8g_queue {
    void* dptr = nullptr;          // the shared counter, mapped on this rank's device
    int device = 0;
    int owner = 0;                 // 1: cudaFree, 0: IPC-opened (cudaIpcCloseMemHandle), 2: borrowed
    unsigned long long epoch = 0;  // runs issued through this queue by this rank
};

namespace pms8g {

inline int fail(char* err, size_t errlen, int code, const char* fmt, ...) {
    if (err && errlen) {
        va_list ap;
        va_start(ap, fmt);
        std::vsnprintf(err, errlen, fmt, ap);
        va_end(ap);
    }
    return code;
}

// Grow-only device scratch for sorting + deduplicating 128-bit motif keys.
struct MergeScratch {
    int device = -1;
    void* sorted = nullptr;   // K128[cap]
    long long* count = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    long long cap = 0;
    long long* h_count = nullptr;  // pinned
};
// Sort + unique `count` keys at dev_in into dev_out on `stream` (device of the
// scratch); returns the unique count through *out_count.
int merge_keys_with(MergeScratch& m, const void* dev_in, long long count, void* dev_out, long long* out_count,
                    cudaStream_t stream, char* err, size_t errlen);
void merge_scratch_free(MergeScratch& m);

// n > 32 sequences: search the first 32 (solve_head), keep the motifs the GPU
// scanner confirms in all n (pms8g_capi.cu).
int solve_many_sequences(const uint8_t* codes, int n, int m, int l, int d, const char* alphabet,
                         const pms8g_options& opt, pms8g_result* out, char* err, size_t errlen,
                         const std::function<int(const pms8g_options&, pms8g_result*)>& solve_head);

}  // namespace pms8g

#define PMS8G_CU(call)                                                                                         \
    do {                                                                                                       \
        cudaError_t e__ = (call);                                                                              \
        if (e__ != cudaSuccess)                                                                                \
            return ::pms8g::fail(err, errlen, PMS8G_ERR_CUDA, "CUDA error %s at %s:%d (%s)",                  \
                                 cudaGetErrorName(e__), __FILE__, __LINE__, cudaGetErrorString(e__));          \
    } while (0)
