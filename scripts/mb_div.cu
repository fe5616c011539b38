// mb_div.cu -- exhaustive-ish check that div_small (reciprocal + Markstein
// correction) equals __ddiv_rn for d = 1..27 on random x in (2^-40, 1].
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double div_small(double x, double d, double y) {
    const double q0 = __dmul_rn(x, y);
    const double r = __fma_rn(-q0, d, x);
    return __fma_rn(r, y, q0);
}
__global__ void check(unsigned long long seed, unsigned long long n, unsigned long long* bad) {
    unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    unsigned long long cnt = 0;
    for (; i < n; i += stride) {
        unsigned long long z = (i + seed) * 0x9E3779B97F4A7C15ull;
        z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27;
        // random mantissa, exponent in [-40, 0]
        const int e = (int)(z >> 58) % 41;
        const double x = ldexp(1.0 + (double)(z & ((1ull << 52) - 1)) * 0x1p-52, -e);
        for (int d = 1; d <= 27; ++d) {
            const double dd = d;
            const double y = __drcp_rn(dd);
            if (div_small(x, dd, y) != __ddiv_rn(x, dd)) ++cnt;
        }
    }
    if (cnt) atomicAdd(bad, cnt);
}
int main() {
    unsigned long long* b;
    cudaMalloc(&b, 8);
    cudaMemset(b, 0, 8);
    const unsigned long long n = 1ull << 32;
    check<<<148 * 8, 256>>>(12345, n, b);
    unsigned long long h = 0;
    cudaMemcpy(&h, b, 8, cudaMemcpyDeviceToHost);
    printf("div_small mismatches over %llu x * 27 divisors: %llu\n", n, h);
    return h != 0;
}
