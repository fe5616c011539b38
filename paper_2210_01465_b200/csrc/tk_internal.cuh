// tk_internal.cuh -- device-side building blocks shared by the FFG, PageRank
// and C_p kernels (sm_100a).  See DESIGN.md for the data layout in HBM.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "tk_landscape.h"

namespace tk {

constexpr double kFailFitness = 1.0e10;  // include/tunekit/cache.hpp:15
constexpr int kMaxDims = TK_MAX_DIMS;
constexpr int kMaxSlots = 64;            // neighbour slots per node (u64 masks)
constexpr int kPackedSlots = 27;         // in-mask | outdeg << 27 fits one u32

// PageRank / mask layout modes
enum Mode : int {
    MODE_ADJ_PACKED = 0,  // Adjacent, 2D <= 27: u32 word = ordered in-mask | outdeg<<27
    MODE_ADJ_ORDERED = 1, // Adjacent, 2D <= 64: u32/u64 ordered in-mask + u8 outdeg
    MODE_HAM = 2,         // Hamming, S <= 64: u32/u64 canonical in-mask + u8 outdeg
    MODE_CSR = 3          // arbitrary in-CSR (tk_pagerank_csr)
};

// Search-space shape as the kernels see it.  Dimensions with a single value
// are dropped: they add no neighbours and do not change any stride.
struct DevShape {
    uint32_t n;        // nodes = prod(radix) (< 2^32)
    int dims;          // effective dims (radix >= 2), dim 0 most significant
    int kind;          // TK_HAMMING / TK_ADJACENT
    int slots;         // S: mask bits per node (Adjacent 2*dims, Hamming sum(m-1))
    uint32_t radix[kMaxDims];
    uint32_t stride[kMaxDims];
    unsigned long long magic[kMaxDims];  // ceil(2^64 / stride); 0 when stride == 1
    int base[kMaxDims];                  // Hamming: first canonical slot of dim i
    uint32_t nbo[2 * kMaxDims];          // Adjacent ordered-slot offsets (u32 wrap)
};

// a / d for 32-bit a via one 64x64 high multiply (Lemire et al. 2019):
// exact for every 32-bit a and d >= 2 with M = ceil(2^64 / d).
__device__ __forceinline__ uint32_t fdiv(uint32_t a, unsigned long long M) {
    return M ? static_cast<uint32_t>(__umul64hi(M, static_cast<unsigned long long>(a))) : a;
}

// ------------------------------------------------------- block primitives --

template <int THREADS, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T& total, T* s_warp) {
    constexpr int W = THREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T w = lane < W ? s_warp[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < W) s_warp[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    total = s_warp[W - 1];
    const T warp_excl = warp ? s_warp[warp - 1] : T(0);
    __syncthreads();  // s_warp may be reused right after
    return warp_excl + x - v;
}

// Deterministic block sum of doubles: fixed shuffle tree, then fixed order
// over warps.  Result valid in every thread.
template <int THREADS>
__device__ __forceinline__ double block_sum(double v, double* s_red) {
    constexpr int W = THREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < W; ++w) t = __dadd_rn(t, s_red[w]);
    __syncthreads();
    return t;
}

// ------------------------------------------------ decoupled look-back scan --
// Status word per tile: bits 63..62 flag (0 none, 1 aggregate, 2 inclusive
// prefix), bits 61..0 value.  Tiles are taken in ticket order, so every tile
// a block waits on belongs to a block that is already running.

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Called by ONE thread.  Returns the exclusive prefix of `tile`.
__device__ __forceinline__ unsigned long long lookback(unsigned long long* status,
                                                      uint32_t tile,
                                                      unsigned long long aggregate) {
    if (tile == 0) {
        st_relaxed(status, kFlagInc | aggregate);
        return 0;
    }
    st_relaxed(status + tile, kFlagAgg | aggregate);
    unsigned long long excl = 0;
    int64_t t = static_cast<int64_t>(tile) - 1;
    while (true) {
        const unsigned long long w = ld_relaxed(status + t);
        const unsigned long long f = w & ~kValMask;
        if (f == 0) continue;
        excl += w & kValMask;
        if (f == kFlagInc) break;
        --t;
    }
    st_relaxed(status + tile, kFlagInc | (excl + aggregate));
    return excl;
}

}  // namespace tk
