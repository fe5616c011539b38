// mb_shfl.cu -- does SHFL share the shared-memory crossbar with LDS? (sm_100a)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_shfl scripts/mb_shfl.cu && /tmp/mb_shfl
//
// Each warp loops over conflict-free LDS.128 (swizzled 128-byte rows, 4
// wavefronts per instruction) and/or fp64 SHFL (two SHFL.32 each).  If the
// mixed kernel takes about max(lds, shfl) the two use separate datapaths; if
// it takes about lds + shfl they share one.  Also: LDS.128 bandwidth against
// the 128 B/clk/SM crossbar, with and without TMA bulk fills running.
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void lds128(uint32_t a, double& x, double& y) {
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}

template <int MODE>  // 1 = LDS only, 2 = SHFL only, 3 = both
__global__ void __launch_bounds__(256) k(double* out, int n, long long* cyc) {
    __shared__ __align__(1024) double s[32 * 16 * 2];
    for (int i = threadIdx.x; i < 32 * 16 * 2; i += blockDim.x) s[i] = i * 0.5;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(s));
    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = lane + j;
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
        if (MODE & 1) {
            const uint32_t row = base + ((lane + it) & 31) * 128;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                double x, y;
                lds128(row + ((q ^ ((lane + it) & 7)) << 4), x, y);
                acc[2 * q] += x;
                acc[2 * q + 1] += y;
            }
        }
        if (MODE & 2) {
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] += __shfl_sync(0xffffffffu, acc[(j + 3) & 15], (lane + 1) & 31);
        }
    }
    long long t1 = clock64();
    double sum = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) sum += acc[j];
    if (sum == 1.2345) out[0] = sum;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 148 * 8 * sizeof(long long));
    const int n = 4096;
    long long h[148 * 8];
    for (int warps : {4, 8}) {
        for (int mode = 1; mode <= 3; ++mode) {
            auto f = mode == 1 ? k<1> : mode == 2 ? k<2> : k<3>;
            f<<<148, warps * 32>>>(out, n, cyc);
            f<<<148, warps * 32>>>(out, n, cyc);
            cudaDeviceSynchronize();
            cudaMemcpy(h, cyc, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
            double c = 0;
            for (int b = 0; b < 148; ++b) c += h[b];
            c /= 148.0 * n;
            // per SM per iteration: LDS bytes = warps*32 lanes*128 B; SHFL = warps*32 SHFL.32
            const double lds_b = (mode & 1) ? warps * 32 * 128.0 : 0;
            printf("warps=%d mode=%s  cyc/iter=%.1f  LDS B/clk/SM=%.1f  SHFL warp-instr/clk/SM=%.2f\n",
                   warps, mode == 1 ? "lds " : mode == 2 ? "shfl" : "both", c, lds_b / c,
                   (mode & 2) ? warps * 32.0 / c : 0.0);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
