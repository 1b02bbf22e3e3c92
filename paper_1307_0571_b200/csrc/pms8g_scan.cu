// pms8g_scan.cu — the brute-force scanner on sm_100a (the reference's
// `pms8 verify` subcommand and exhaustive solver).
//
//   K6 witness_kernel  one warp per motif: for every sequence the first window
//                      within Hamming distance d (naive_is_motif,
//                      src/oracle.cpp:16-37 — stops at the first sequence
//                      without a window, like the reference)
//   K7 sweep_kernel    one lane per word of Sigma^l (code order, position 0
//                      most significant): the word is a motif iff every
//                      sequence has a window within d (brute_force_solve,
//                      src/oracle.cpp:65-75). The l-mer table is staged in
//                      shared memory; every lane of a warp reads the same
//                      window (broadcast), the warp leaves a sequence once all
//                      its lanes have a hit and leaves the word block once no
//                      lane is alive.
//
// Independent of the PMS8 search tree: used as an exactness check of the
// search path (tests) and as the CLI's `verify`.
#include <cuda_runtime.h>

#include <cstdint>

#include "pms8g_common.cuh"
#include "pms8g_device.cuh"
#include "pms8g_launch.h"

namespace pms8g {

using namespace dev;

template <int W>
__global__ void witness_kernel(const Lmer<W>* __restrict__ table, int n, int w, int l, int d, int sigma,
                               const uint8_t* __restrict__ motifs, long long nmotifs, int32_t* __restrict__ witness,
                               uint8_t* __restrict__ pass) {
    const int lane = threadIdx.x & 31;
    const long long i = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= nmotifs) return;
    Lmer<W> c;
#pragma unroll
    for (int x = 0; x < W; ++x) c.h[x] = c.o[x] = 0;
    const uint8_t* mc = motifs + i * l;
    for (int p = 0; p < l; ++p) set_code<W>(c, p, mc[p] & 3);
    int32_t* wit = witness + i * n;
    bool ok = true;
    for (int r = 0; r < n; ++r) {
        int found = -1;
        if (ok) {
            for (int base = 0; base < w; base += 32) {
                const int o = base + lane;
                const unsigned b = __ballot_sync(0xffffffffu, o < w && dist<W>(c, table[r * w + o]) <= d);
                if (b) {
                    found = base + __ffs(b) - 1;
                    break;
                }
            }
            ok = found >= 0;
        }
        if (lane == 0) wit[r] = found;
    }
    if (lane == 0) pass[i] = ok ? 1 : 0;
}

// Word x of Sigma^l -> bit planes and its 128-bit MSB-first key (the search
// path's key layout, include/pms8g.h: 2 bits per symbol, position 0 highest).
template <int W>
__device__ __forceinline__ void word_of(unsigned long long x, int l, int sigma, Lmer<W>& c, unsigned long long& klo,
                                        unsigned long long& khi) {
#pragma unroll
    for (int q = 0; q < W; ++q) c.h[q] = c.o[q] = 0;
    klo = khi = 0;
    for (int p = l - 1; p >= 0; --p) {
        int code;
        if (sigma == 4) {
            code = static_cast<int>(x & 3ull);
            x >>= 2;
        } else {
            code = static_cast<int>(x % static_cast<unsigned>(sigma));
            x /= static_cast<unsigned>(sigma);
        }
        set_code<W>(c, p, code);
        const int sh = 2 * (l - 1 - p);
        if (sh >= 64) khi |= static_cast<unsigned long long>(code) << (sh - 64);
        else klo |= static_cast<unsigned long long>(code) << sh;
    }
}

template <int W>
__global__ void __launch_bounds__(512) sweep_kernel(const Lmer<W>* __restrict__ gtable, int n, int w, int l, int d,
                                                    int sigma, unsigned long long total, int stage,
                                                    unsigned long long* __restrict__ keys,
                                                    unsigned long long* __restrict__ count, long long cap) {
    extern __shared__ __align__(16) uint8_t sweep_smem[];
    const int K = n * w;
    const Lmer<W>* table = gtable;
    if (stage) {
        // TMA bulk copy of the whole table into shared memory
        __shared__ unsigned long long bar;
        tma_stage(sweep_smem, gtable, (static_cast<uint32_t>(K) * sizeof(Lmer<W>) + 15u) / 16u * 16u, &bar);
        table = reinterpret_cast<const Lmer<W>*>(sweep_smem);
    }
    const int lane = threadIdx.x & 31;
    const unsigned long long warps = static_cast<unsigned long long>(gridDim.x) * (blockDim.x >> 5);
    for (unsigned long long wb = (static_cast<unsigned long long>(blockIdx.x) * (blockDim.x >> 5) +
                                  (threadIdx.x >> 5)) * 32ull;
         wb < total; wb += warps * 32ull) {
        const unsigned long long x = wb + lane;
        bool alive = x < total;
        Lmer<W> c;
        unsigned long long klo, khi;
        word_of<W>(alive ? x : 0ull, l, sigma, c, klo, khi);
        for (int r = 0; r < n; ++r) {
            const Lmer<W>* T = table + r * w;
            bool hit = !alive;
            int j = 0;
            // 8 windows per step; every lane reads the same window
            for (; j + 8 <= w; j += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) hit |= dist<W>(c, T[j + u]) <= d;
                if (__all_sync(0xffffffffu, hit)) break;
            }
            if (j + 8 > w)
                for (; j < w; ++j) hit |= dist<W>(c, T[j]) <= d;
            alive = alive && hit;
            if (!__any_sync(0xffffffffu, alive)) break;
        }
        if (alive) {
            const unsigned long long pos = atomicAdd(count, 1ull);
            if (static_cast<long long>(pos) < cap) {
                keys[2 * pos] = klo;
                keys[2 * pos + 1] = khi;
            }
        }
    }
}

cudaError_t launch_witness(int W, const void* table, int n, int w, int l, int d, int sigma, const uint8_t* motifs,
                           long long nmotifs, int32_t* witness, uint8_t* pass, cudaStream_t s) {
    if (nmotifs <= 0) return cudaSuccess;
    const int wpb = 8;
    const unsigned blocks = static_cast<unsigned>((nmotifs + wpb - 1) / wpb);
    if (W == 1)
        witness_kernel<1><<<blocks, 32 * wpb, 0, s>>>(static_cast<const Lmer<1>*>(table), n, w, l, d, sigma, motifs,
                                                      nmotifs, witness, pass);
    else
        witness_kernel<2><<<blocks, 32 * wpb, 0, s>>>(static_cast<const Lmer<2>*>(table), n, w, l, d, sigma, motifs,
                                                      nmotifs, witness, pass);
    return cudaGetLastError();
}

cudaError_t launch_sweep(int W, const void* table, int n, int w, int l, int d, int sigma, unsigned long long total,
                         unsigned long long* keys, unsigned long long* count, long long cap, int sms,
                         cudaStream_t s) {
    if (total == 0) return cudaSuccess;
    const size_t tbytes = (static_cast<size_t>(n) * w * lmer_bytes(W) + 15) / 16 * 16;
    int stage = tbytes <= 200 * 1024;
    const size_t smem = stage ? tbytes : 0;
    const int threads = 512;
    // persistent: as many resident blocks per SM as the staged table allows
    // (94 KB for K = 11,760 -> 2 x 16 warps), grid-stride over the words
    int per_sm = stage ? static_cast<int>((220 * 1024) / (smem + 1024)) : 4;
    per_sm = per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm);
    const unsigned long long need = (total + threads - 1) / threads;
    const unsigned long long grid = static_cast<unsigned long long>(sms) * per_sm;
    const unsigned blocks = static_cast<unsigned>(need < grid ? need : grid);
    cudaError_t e;
    if (W == 1) {
        if ((e = cudaFuncSetAttribute(sweep_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem))) != cudaSuccess)
            return e;
        sweep_kernel<1><<<blocks, threads, smem, s>>>(static_cast<const Lmer<1>*>(table), n, w, l, d, sigma, total,
                                                      stage, keys, count, cap);
    } else {
        if ((e = cudaFuncSetAttribute(sweep_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem))) != cudaSuccess)
            return e;
        sweep_kernel<2><<<blocks, threads, smem, s>>>(static_cast<const Lmer<2>*>(table), n, w, l, d, sigma, total,
                                                      stage, keys, count, cap);
    }
    return cudaGetLastError();
}

}  // namespace pms8g
