// pms8g_common.cuh — device helpers shared by the sm_100a kernels: bit-plane
// l-mers, Hamming distance by XOR/OR/POPC, key packing.
#pragma once
#include <cstdint>

#include "pms8g_device.cuh"

namespace pms8g {
namespace dev {

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// One-dimensional TMA bulk copy global -> shared (cp.async.bulk, completion
// counted on an mbarrier): used to stage the l-mer table into each CTA's
// shared memory with one instruction instead of a strided register copy.
// Call from every thread of the block; `bytes` must be a multiple of 16 and
// both addresses 16-byte aligned (the table is allocated rounded up).
__device__ __forceinline__ void tma_stage(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                          unsigned long long* mbar) {
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        // chunks of <= 64 KB (the copy size operand); all complete on one barrier
        for (uint32_t off = 0; off < bytes; off += 65536u) {
            const uint32_t n = bytes - off < 65536u ? bytes - off : 65536u;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    dst + off),
                "l"(static_cast<const char*>(gmem_src) + off), "r"(n), "r"(bar)
                : "memory");
        }
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar)
            : "memory");
    }
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
        if (W == 1) {
            if (lo <= 0) s += __popc(m.w[i]);
            else if (lo < 32) s += __popc(m.w[i] >> lo);
        } else {
            // branch-free for two-word l-mers (lanes hold different p and
            // straddle the word boundary): the clamped funnel shift gives 0
            // once the shift reaches 32
            s += __popc(__funnelshift_rc(m.w[i], 0u, static_cast<unsigned>(max(lo, 0))));
        }
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

}  // namespace dev
}  // namespace pms8g
