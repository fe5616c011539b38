// tk_descent.cu -- the GPU random-walk validator:
// batched randomized first-improvement descents, the reference's
// climb_random_first (/root/reference/proj/src/hillclimb.cpp:48-87), one
// walker per thread.
//
// SPEC.md:430 / acceptance 4 restate the paper's s7.2 claim as a property: the
// arrival frequency of such descents at each local minimum tracks PageRank
// restricted to the minima.  On the host that check is limited to spaces of a
// few thousand points; here every walker is one thread, so 1e6-1e8 descents
// over spaces of 1e6-1e7 points take milliseconds.
//
// Semantics (identical to oracle.c or_descents, bit for bit):
//   - slot universe of build_slots (hillclimb.cpp:26-38): dimensions
//     ascending; Adjacent {-1, +1} when m > 1, Hamming the m - 1 alternatives
//     a, resolved to index a < x ? a : a + 1 (resolve_slot :41-46);
//   - the scan walks a random permutation of the slots cyclically and moves
//     to the first strictly better neighbour (fp64 <, ties never improve);
//     with restart_scan a fresh permutation starts after every move; a full
//     cycle without improvement ends the descent (:60-85);
//   - draws: walker w owns the splitmix64 stream s = mix(seed ^ mix(w));
//     uniform(k) = mulhi64(next(), k); the start rank is the first draw and a
//     permutation is Fisher-Yates from the identity, i = S-1 .. 1.
//
// The walk is a dependent chain of random 8-byte fitness gathers per walker
// (latency-bound, not a streaming kernel); it is a validator beside the hot
// path, not part of it.
#include <cuda_runtime.h>

#include <cstdint>

#include "tk_kernels.cuh"

namespace tk {
namespace {

__device__ __forceinline__ unsigned long long sm_mix(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long sm_next(unsigned long long& s) {
    s += 0x9E3779B97F4A7C15ull;
    return sm_mix(s);
}
__device__ __forceinline__ unsigned long long uniform(unsigned long long& s, unsigned long long k) {
    return __umul64hi(sm_next(s), k);
}

__device__ __forceinline__ void shuffle_slots(uint8_t* order, int S, unsigned long long& st) {
    for (int i = 0; i < S; ++i) order[i] = static_cast<uint8_t>(i);
    for (int i = S - 1; i > 0; --i) {
        const int j = static_cast<int>(uniform(st, static_cast<unsigned long long>(i) + 1));
        const uint8_t t = order[i];
        order[i] = order[j];
        order[j] = t;
    }
}

__global__ void __launch_bounds__(256) descent_kernel(const __grid_constant__ DescentArgs a) {
    __shared__ uint8_t s_dim[kMaxDescentSlots];
    __shared__ int16_t s_alt[kMaxDescentSlots];
    __shared__ uint32_t s_radix[kMaxDims];
    __shared__ unsigned long long s_stride[kMaxDims];
    for (int i = threadIdx.x; i < a.slots; i += blockDim.x) {
        s_dim[i] = a.slot_dim[i];
        s_alt[i] = a.slot_alt[i];
    }
    for (int i = threadIdx.x; i < a.dims; i += blockDim.x) {
        s_radix[i] = a.radix[i];
        s_stride[i] = a.stride[i];
    }
    __syncthreads();
    const int S = a.slots;
    unsigned long long evals = 0;
    uint8_t order[kMaxDescentSlots];
    int x[kMaxDims];
    for (unsigned long long w = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
         w < a.walkers; w += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
        unsigned long long st = sm_mix(a.seed ^ sm_mix(w));
        unsigned long long rank = uniform(st, a.n);
        double f = a.fit[rank];
        if (S) {
            unsigned long long rem = rank;
            for (int i = 0; i < a.dims; ++i) {
                x[i] = static_cast<int>(rem / s_stride[i]);
                rem -= static_cast<unsigned long long>(x[i]) * s_stride[i];
            }
            shuffle_slots(order, S, st);
            int pos = 0, since = 0;
            while (since < S) {
                const int sl = order[pos];
                pos = pos + 1 == S ? 0 : pos + 1;
                const int d = s_dim[sl];
                const int m = static_cast<int>(s_radix[d]);
                const int cur = x[d];
                const int alt = s_alt[sl];
                const int j = a.kind == TK_HAMMING ? (alt < cur ? alt : alt + 1) : cur + alt;
                if (j < 0 || j >= m) {
                    ++since;
                    continue;
                }
                const unsigned long long nb =
                    rank + static_cast<unsigned long long>(static_cast<long long>(j - cur) *
                                                           static_cast<long long>(s_stride[d]));
                const double fn = __ldg(a.fit + nb);
                ++evals;
                if (fn < f) {
                    x[d] = j;
                    rank = nb;
                    f = fn;
                    since = 0;
                    if (a.restart_scan) {
                        shuffle_slots(order, S, st);
                        pos = 0;
                    }
                } else {
                    ++since;
                }
            }
        }
        atomicAdd(a.counts + rank, 1u);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
    if ((threadIdx.x & 31) == 0 && evals) atomicAdd(a.evaluations, evals);
}

__global__ void __launch_bounds__(256) gather_counts_kernel(const uint32_t* __restrict__ idx,
                                                            uint64_t m,
                                                            const uint32_t* __restrict__ counts,
                                                            unsigned long long* __restrict__ out) {
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < m;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[k] = counts[idx[k]];
}

}  // namespace

cudaError_t launch_descents(const DescentArgs& a, int num_sms, cudaStream_t stream) {
    const unsigned long long want = (a.walkers + 255) / 256;
    const unsigned long long cap = static_cast<unsigned long long>(num_sms) * 8;
    const unsigned int grid = static_cast<unsigned int>(want < cap ? (want ? want : 1) : cap);
    descent_kernel<<<grid, 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_gather_counts(const uint32_t* idx, uint64_t m, const uint32_t* counts,
                                 unsigned long long* out, cudaStream_t stream) {
    if (!m) return cudaSuccess;
    const uint64_t want = (m + 255) / 256;
    gather_counts_kernel<<<static_cast<unsigned int>(want < 148 * 16 ? want : 148 * 16), 256, 0,
                           stream>>>(idx, m, counts, out);
    return cudaGetLastError();
}

}  // namespace tk
