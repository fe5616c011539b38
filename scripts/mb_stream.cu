// mb_stream.cu -- streaming-read microbenchmarks on B200 (sm_100a): how many
// bytes per SM must be in flight, and in what shape, to reach HBM and L2
// bandwidth with 1-D bulk copies (cp.async.bulk) versus plain LDG.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_stream scripts/mb_stream.cu
//   ./mb_stream            # prints one line per configuration
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                            \
        }                                                                            \
    } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(sa(b)), "r"(ph)
            : "memory");
    }
}
// wait flavours: 0 try_wait (may suspend), 1 test_wait spin, 2 try_wait with a short suspend hint
template <int W>
__device__ __forceinline__ void mbar_wait_t(uint64_t* b, uint32_t ph) {
    if (W == 0) { mbar_wait(b, ph); return; }
    uint32_t done = 0;
    while (!done) {
        if (W == 1)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(sa(b)), "r"(ph)
                : "memory");
        else
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(sa(b)), "r"(ph), "r"(20)
                : "memory");
    }
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                     uint64_t pol, bool hint) {
    if (hint)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
            "[%0], [%1], %2, [%3], %4;" ::"r"(sa(dst)),
            "l"(src), "r"(bytes), "r"(sa(bar)), "l"(pol)
            : "memory");
    else
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(sa(dst)),
            "l"(src), "r"(bytes), "r"(sa(bar))
            : "memory");
}

// One producer warp (lane i issues copy i of the stage), one consumer warp.
// Reads `passes` times over [0, nbytes) in stage_bytes tiles.
template <int W>
__global__ void tma_stream(const uint8_t* __restrict__ src, size_t nbytes, int stage_bytes, int S,
                           int ncopy, int passes, int evict_first, unsigned long long* sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[32], empty[32];
    const int t = threadIdx.x, lane = t & 31;
    if (t == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    uint64_t pol = 0;
    if (evict_first)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const size_t ntiles = nbytes / stage_bytes;
    const size_t total = ntiles * passes;
    const uint32_t cb = stage_bytes / ncopy;
    if (t < 32) {
        uint32_t k = 0;
        for (size_t j = blockIdx.x; j < total; j += gridDim.x, ++k) {
            const int st = k % S;
            if (k >= (uint32_t)S) mbar_wait_t<W>(&empty[st], ((k / S) - 1) & 1u);
            const size_t tile = j % ntiles;
            if (lane == 0) mbar_expect_tx(&full[st], stage_bytes);
            __syncwarp();
            for (int c = lane; c < ncopy; c += 32)
                bulk(smem + (size_t)st * stage_bytes + c * cb, src + tile * stage_bytes + (size_t)c * cb,
                     cb, &full[st], pol, evict_first);
        }
    } else {
        uint32_t k = 0;
        unsigned long long acc = 0;
        for (size_t j = blockIdx.x; j < total; j += gridDim.x, ++k) {
            const int st = k % S;
            mbar_wait_t<W>(&full[st], (k / S) & 1u);
            acc += smem[(size_t)st * stage_bytes + lane * 4];
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        if (acc == 0x12345) *sink = acc;
    }
}


// P independent pipelines per CTA (producer warp 2p, consumer warp 2p+1)
__global__ void tma_pipes(const uint8_t* __restrict__ src, size_t nbytes, int stage_bytes, int S,
                          int ncopy, int P, int lane0_only, unsigned long long* sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[64], empty[64];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5, p = w >> 1;
    if (t == 0) {
        for (int i = 0; i < S * P; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const size_t ntiles = nbytes / stage_bytes;
    const uint32_t cb = stage_bytes / ncopy;
    uint8_t* base = smem + (size_t)p * S * stage_bytes;
    uint64_t* fb = full + p * S;
    uint64_t* eb = empty + p * S;
    const size_t step = (size_t)gridDim.x * P;
    if (!(w & 1)) {
        uint32_t k = 0;
        for (size_t j = (size_t)blockIdx.x * P + p; j < ntiles; j += step, ++k) {
            const int st = k % S;
            if (k >= (uint32_t)S) mbar_wait(&eb[st], ((k / S) - 1) & 1u);
            if (lane == 0) mbar_expect_tx(&fb[st], stage_bytes);
            __syncwarp();
            if (lane0_only) {
                if (lane == 0)
                    for (int c = 0; c < ncopy; ++c)
                        bulk(base + (size_t)st * stage_bytes + c * cb, src + j * stage_bytes + (size_t)c * cb,
                             cb, &fb[st], 0, false);
            } else {
                for (int c = lane; c < ncopy; c += 32)
                    bulk(base + (size_t)st * stage_bytes + c * cb, src + j * stage_bytes + (size_t)c * cb,
                         cb, &fb[st], 0, false);
            }
        }
    } else {
        uint32_t k = 0;
        unsigned long long acc = 0;
        for (size_t j = (size_t)blockIdx.x * P + p; j < ntiles; j += step, ++k) {
            const int st = k % S;
            mbar_wait(&fb[st], (k / S) & 1u);
            acc += base[(size_t)st * stage_bytes + lane * 4];
            __syncwarp();
            if (lane == 0) mbar_arrive(&eb[st]);
        }
        if (acc == 0x12345) *sink = acc;
    }
}


// P producer warps (stage k issued by warp k % P), C consumer warps, one pipeline
__global__ void tma_mp(const uint8_t* __restrict__ src, size_t nbytes, int stage_bytes, int S,
                       int ncopy, int P, int C, unsigned long long* sink, int passes = 1) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[32], empty[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], C);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const size_t nt1 = nbytes / stage_bytes;
    const size_t ntiles = nt1 * passes;
    const uint32_t cb = stage_bytes / ncopy;
    if (w < P) {
        uint32_t k = w;
        size_t jm = blockIdx.x + (size_t)w * gridDim.x;
        for (size_t j = jm; j < ntiles; j += (size_t)gridDim.x * P, k += P) {
            const int st = k % S;
            if (k >= (uint32_t)S) mbar_wait(&empty[st], ((k / S) - 1) & 1u);
            while (jm >= nt1) jm -= nt1;
            if (lane == 0) mbar_expect_tx(&full[st], (stage_bytes / ncopy) * ncopy);
            __syncwarp();
            for (int c = lane; c < ncopy; c += 32)
                bulk(smem + (size_t)st * stage_bytes + c * cb, src + jm * stage_bytes + (size_t)c * cb, cb,
                     &full[st], 0, false);
            jm += (size_t)gridDim.x * P;
        }
    } else {
        uint32_t k = 0;
        unsigned long long acc = 0;
        for (size_t j = blockIdx.x; j < ntiles; j += gridDim.x, ++k) {
            const int st = k % S;
            mbar_wait(&full[st], (k / S) & 1u);
            acc += smem[(size_t)st * stage_bytes + lane * 4];
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        if (acc == 0x12345) *sink = acc;
    }
}

// Plain coalesced LDG.128: each thread U independent 16-byte loads per step.
template <int U>
__global__ void ldg_stream(const double2* __restrict__ src, size_t n2, int passes, double* sink) {
    double a = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride * U) {
            double2 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const size_t k = i + u * stride;
                v[u] = k < n2 ? __ldg(src + k) : make_double2(0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) a += v[u].x + v[u].y;
        }
    if (a == 1.2345) *sink = a;
}

// copy (read + write) with LDG/STG.128, U-deep
template <int U>
__global__ void copy_stream(const double2* __restrict__ src, double2* __restrict__ dst, size_t n2) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride * U) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t k = i + u * stride;
            if (k < n2) v[u] = __ldg(src + k);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t k = i + u * stride;
            if (k < n2) dst[k] = v[u];
        }
    }
}

int main(int argc, char** argv) {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t big = 4ull << 30;  // 4 GiB >> L2
    const size_t l2 = 32ull << 20;  // 32 MiB, L2-resident
    uint8_t* buf;
    CK(cudaMalloc(&buf, big + (1 << 20)));
    CK(cudaMemset(buf, 1, big));
    uint8_t* dst;
    CK(cudaMalloc(&dst, big / 2));
    unsigned long long* sink;
    CK(cudaMalloc(&sink, 64));
    CK(cudaFuncSetAttribute(tma_stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(tma_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(tma_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto tma = [&](const char* what, size_t nbytes, int passes, int stage_bytes, int S, int ncopy,
                   int cps, int ef, int W = 0) {
        auto kern = W == 0 ? tma_stream<0> : W == 1 ? tma_stream<1> : tma_stream<2>;
        const size_t smem = (size_t)stage_bytes * S;
        if (smem * cps > 227 * 1024) return;
        const int g = sms * cps;
        kern<<<g, 64, smem>>>(buf, nbytes, stage_bytes, S, ncopy, 1, ef, sink);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e0));
        kern<<<g, 64, smem>>>(buf, nbytes, stage_bytes, S, ncopy, passes, ef, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double bytes = (double)(nbytes / stage_bytes) * stage_bytes * passes;
        std::printf("W=%d tma %-4s stage=%6d S=%2d copies=%2d (%5d B) cta/sm=%d inflight/sm=%4zu KB ef=%d : %8.1f GB/s\n",
                    W, what, stage_bytes, S, ncopy, stage_bytes / ncopy, cps, smem * cps / 1024, ef,
                    bytes / ms / 1e6);
    };
    const int mode = argc > 1 ? std::atoi(argv[1]) : 0;
    if (mode == 4) {
        CK(cudaFuncSetAttribute(tma_mp, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
        for (size_t buf_mb : {32, 96, 4096})
            for (int S : {3, 4})
                for (int nc : {2, 4, 7, 14, 28}) {
                    const int stage = 57344 / (nc * 16) * 16 * nc;
                    const int P = 2, C = 16;
                    const size_t nb = buf_mb << 20;
                    const int passes = (int)((4096ull << 20) / nb);
                    const size_t smem = (size_t)stage * S;
                    tma_mp<<<sms, 32 * (P + C), smem>>>(buf, nb, stage, S, nc, P, C, sink, 1);
                    CK(cudaGetLastError());
                    CK(cudaEventRecord(e0));
                    tma_mp<<<sms, 32 * (P + C), smem>>>(buf, nb, stage, S, nc, P, C, sink, passes);
                    CK(cudaEventRecord(e1));
                    CK(cudaEventSynchronize(e1));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, e0, e1));
                    const double bytes = (double)(nb / stage) * stage * passes;
                    std::printf("mp4 buf=%5zuMB S=%d stage=%6d copies=%2d (%5d B) : %8.1f GB/s  %.1f B/clk/SM\n",
                                buf_mb, S, stage, nc, stage / nc, bytes / ms / 1e6,
                                bytes / ms / 1e6 / sms / 1.92);
                }
        return 0;
    }
    if (mode == 3) {
        CK(cudaFuncSetAttribute(tma_mp, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        for (int C : {1, 16})
            for (int P : {1, 2, 3, 4, 6})
                for (int stage : {16384, 32768, 65536})
                    for (int nc : {4, 16}) {
                        int S = (200 * 1024) / stage;
                        if (S > 12) S = 12;
                        if (S < P) continue;
                        const size_t smem = (size_t)stage * S;
                        tma_mp<<<sms, 32 * (P + C), smem>>>(buf, big, stage, S, nc, P, C, sink);
                        CK(cudaGetLastError());
                        CK(cudaEventRecord(e0));
                        tma_mp<<<sms, 32 * (P + C), smem>>>(buf, big, stage, S, nc, P, C, sink);
                        CK(cudaEventRecord(e1));
                        CK(cudaEventSynchronize(e1));
                        float ms;
                        CK(cudaEventElapsedTime(&ms, e0, e1));
                        std::printf("mp C=%2d P=%d S=%2d stage=%6d copies=%2d : %8.1f GB/s\n", C, P, S, stage,
                                    nc, (double)(big / stage) * stage / ms / 1e6);
                    }
        return 0;
    }
    if (mode == 2) {
        CK(cudaFuncSetAttribute(tma_pipes, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        for (int l0 : {0, 1})
            for (int P : {1, 2, 4, 8})
                for (int stage : {8192, 16384})
                    for (int nc : {1, 4, 16}) {
                        const int S = 3;
                        const size_t smem = (size_t)stage * S * P;
                        if (smem > 220 * 1024) continue;
                        for (int which = 0; which < 2; ++which) {
                            const size_t nb = which ? l2 : big;
                            const int reps = which ? 64 : 1;
                            tma_pipes<<<sms, 64 * P, smem>>>(buf, nb, stage, S, nc, P, l0, sink);
                            CK(cudaGetLastError());
                            CK(cudaEventRecord(e0));
                            for (int r = 0; r < reps; ++r)
                                tma_pipes<<<sms, 64 * P, smem>>>(buf, nb, stage, S, nc, P, l0, sink);
                            CK(cudaEventRecord(e1));
                            CK(cudaEventSynchronize(e1));
                            float ms;
                            CK(cudaEventElapsedTime(&ms, e0, e1));
                            std::printf("pipes %s P=%d lane0=%d stage=%6d copies=%2d : %8.1f GB/s\n",
                                        which ? "l2 " : "hbm", P, l0, stage, nc,
                                        (double)(nb / stage) * stage * reps / ms / 1e6);
                        }
                    }
        return 0;
    }
    if (mode == 1) {
        for (int W : {0, 1, 2})
            for (int stage : {8192, 16384, 65536})
                for (int S : {3, 6})
                    for (int nc : {1, 4, 16}) {
                        tma("hbm", big, 1, stage, S, nc, 1, 0, W);
                        tma("l2", l2, 64, stage, S, nc, 1, 0, W);
                    }
        return 0;
    }
    // LDG
    auto ldg = [&](int U, int bpsm, int threads) {
        const size_t n2 = big / 16;
        const int g = sms * bpsm;
        auto k = U == 1 ? ldg_stream<1> : U == 2 ? ldg_stream<2> : U == 4 ? ldg_stream<4> : ldg_stream<8>;
        k<<<g, threads>>>(reinterpret_cast<double2*>(buf), n2, 1, reinterpret_cast<double*>(sink));
        CK(cudaEventRecord(e0));
        k<<<g, threads>>>(reinterpret_cast<double2*>(buf), n2, 1, reinterpret_cast<double*>(sink));
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        std::printf("ldg U=%d blocks/sm=%d threads=%d : %8.1f GB/s\n", U, bpsm, threads,
                    big / ms / 1e6);
    };
    for (int U : {1, 2, 4, 8})
        for (int b : {2, 4, 8}) ldg(U, b, 256);
    auto cp = [&](int U, int bpsm) {
        const size_t n2 = big / 2 / 16;
        const int g = sms * bpsm;
        auto k = U == 1 ? copy_stream<1> : U == 2 ? copy_stream<2> : copy_stream<4>;
        k<<<g, 256>>>(reinterpret_cast<double2*>(buf), reinterpret_cast<double2*>(dst), n2);
        CK(cudaEventRecord(e0));
        k<<<g, 256>>>(reinterpret_cast<double2*>(buf), reinterpret_cast<double2*>(dst), n2);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        std::printf("copy U=%d blocks/sm=%d : %8.1f GB/s (read+write)\n", U, bpsm, big / ms / 1e6);
    };
    for (int U : {1, 2, 4})
        for (int b : {4, 8}) cp(U, b);
    return 0;
}
