// mb_lat.cu -- FP64 / shared-memory latency and throughput probes (sm_100a).
#include <cstdio>
#include <cstdint>
__global__ void dadd_chain(double* out, int n, double x) {
    double a = x, b = x * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a = __dadd_rn(a, b);
        a = __dadd_rn(a, b);
        a = __dadd_rn(a, b);
        a = __dadd_rn(a, b);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / (4.0 * n);
    if (a == 1.2345) out[1] = a;
}
__global__ void dfma_chain(double* out, int n, double x) {
    double a = x, b = x * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a = __fma_rn(a, b, b);
        a = __fma_rn(a, b, b);
        a = __fma_rn(a, b, b);
        a = __fma_rn(a, b, b);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / (4.0 * n);
    if (a == 1.2345) out[1] = a;
}
__global__ void ddiv_chain(double* out, int n, double x) {
    double a = x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = __ddiv_rn(a, 3.0) + 1.0;
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / n;
    if (a == 1.2345) out[1] = a;
}
__global__ void lds_chain(double* out, int n) {
    __shared__ uint32_t s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
    __syncthreads();
    uint32_t p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) p = s[p];
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / n;
    if (p == 12345) out[1] = p;
}
// throughput: W warps per SM, each 8 independent DADD chains
__global__ void dadd_tput(double* out, int n, double x) {
    double a[8];
    for (int k = 0; k < 8; ++k) a[k] = x + k;
    const double b = x * 0.5;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __dadd_rn(a[k], b);
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 1.2345) out[1] = s;
}
int main() {
    double* d;
    cudaMalloc(&d, 64);
    double h;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    dadd_chain<<<1, 32>>>(d, 4096, 1.0);
    dadd_chain<<<1, 32>>>(d, 4096, 1.0);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.1f cycles\n", h);
    dfma_chain<<<1, 32>>>(d, 4096, 0.5);
    dfma_chain<<<1, 32>>>(d, 4096, 0.5);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.1f cycles\n", h);
    ddiv_chain<<<1, 32>>>(d, 4096, 0.5);
    ddiv_chain<<<1, 32>>>(d, 4096, 0.5);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("ddiv_rn + DADD dependent latency: %.1f cycles\n", h);
    lds_chain<<<1, 32>>>(d, 4096);
    lds_chain<<<1, 32>>>(d, 4096);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("LDS.32 dependent latency: %.1f cycles\n", h);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w : {1, 2, 4, 8, 16, 32}) {
        const int n = 1 << 14;
        dadd_tput<<<sms, 32 * w>>>(d, n, 1.0);
        cudaEventRecord(e0);
        dadd_tput<<<sms, 32 * w>>>(d, n, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)sms * 32 * w * 8 * n;
        printf("DADD throughput warps/SM=%2d: %.1f G thread-DADD/s = %.2f warp-DADD/clk/SM @1.92GHz\n", w,
               ops / ms / 1e6, ops / 32 / sms / (ms * 1e-3 * 1.92e9));
    }
    return 0;
}
