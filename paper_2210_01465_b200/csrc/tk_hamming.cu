// tk_hamming.cu -- tiled PageRank for the Hamming neighbourhood (sm_100a).
//
// Hamming neighbours of rank v are v + (j - x_i) * s_i for every dimension i
// and every value j != x_i (space.cpp:167-181): whole lines of the grid, up to
// sum(m_i - 1) = 50 per node on C5.  Staging them is out of reach (the far
// lines of one 512-rank tile are ~36 ranges, ~150 KB), so this kernel gathers
// with coalesced loads -- consecutive lanes hold consecutive ranks, so every
// line load of a warp is one 256-byte run.  Measured on C5 (B200): ~11.7 ms
// per iteration against 14.7 for the per-lane kernel (tk_kernels.cu MODE_HAM)
// it replaces; both are bound by gather latency (DRAM at ~20 % of peak even
// though the lines of the slowest dimensions miss L2, ~190 B per rank and
// iteration).  Unrolling the per-value loops by two beats one, four and
// eight (445 / 570 / 544 / 854 ms on C5); re-ordering the tile sweep did not
// help (profiles/r01_ab_log.md).
//
// Tiles are 512 consecutive ranks aligned to 512.  For the shapes this kernel
// takes (StagePlan-style digit classes, see tk_kernels.cuh) each digit is
// either fixed per thread (period divides the tile), fixed per tile (the tile
// divides the stride: computed once per tile from v0 with one fast division
// per dimension), or one fast division of (v0 mod P_i) + t per rank -- no
// per-rank mixed-radix decode.
//
// The iteration is the contribution-only one of the Adjacent kernel
// (tk_staged.cu pr_tile_c): only c' is stored in the loop, the
// residual takes r = c * outdeg from the node's own contribution, and a
// closing sweep re-computes r' of the last iteration into a.r0.  The in-edge
// sum runs in ascending source rank (lower neighbours: dims ascending, values
// ascending; then upper: dims descending, values ascending), so each node's
// r' is bit-identical to the oracle's (oracle/oracle.c pagerank order).
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "tk_kernels.cuh"

namespace cg = cooperative_groups;

namespace tk {

namespace {

constexpr int kHT = 512;  // ranks per tile = threads per CTA
#ifndef TK_HAM_UNROLL
#define TK_HAM_UNROLL 2
#endif
constexpr int kHamUnroll = TK_HAM_UNROLL;  // values per dimension whose loads issue together
#ifndef TK_HAM_MINB
#define TK_HAM_MINB 2
#endif
constexpr int kMaxHamDeg = 64;

struct HamTilePlan {
    uint32_t inv;   // dims whose period divides the tile
    uint32_t uni;   // dims whose stride the tile divides (digit fixed per tile)
    uint32_t tile;  // other dims whose period the tile divides
};

__device__ __forceinline__ double div_small_h(double x, double d, double y) {
    const double q0 = __dmul_rn(x, y);
    const double r = __fma_rn(-q0, d, x);
    return __fma_rn(r, y, q0);
}

// the digits of rank v0 + t (see the file comment); q_prev carries v0 / s_{i-1}
template <int DIMS>
__device__ __forceinline__ void tile_digits(const DevShape& s, const HamTilePlan& hp, uint32_t v0,
                                            int t, const uint32_t (&xinv)[DIMS],
                                            uint32_t (&x)[DIMS]) {
    uint32_t q_prev = 0;  // v0 / s_{i-1} along the leading (tile-uniform) dims
#pragma unroll
    for (int i = 0; i < DIMS; ++i) {
        if ((hp.inv >> i) & 1u) {
            x[i] = xinv[i];
        } else if ((hp.uni >> i) & 1u) {  // a prefix of the dims: strides fall
            const uint32_t q = fdiv(v0, s.magic[i]);
            x[i] = q - q_prev * s.radix[i];
            q_prev = q;
        } else {  // tile class: (v0 mod P_i) + t with P_i = s_{i-1}
            const uint32_t r = i ? v0 - fdiv(v0, s.magic[i - 1]) * s.stride[i - 1] : v0;
            x[i] = fdiv(r + static_cast<uint32_t>(t), s.magic[i]);
        }
    }
}

// sum over the in-neighbours of v in ascending source rank: lower neighbours
// (dims ascending, values ascending; bit base_i + j), then upper (dims
// descending, values ascending; bit base_i + j - 1).  Tight per-value loops,
// unrolled by four so the loads of a group issue before its adds.
template <int DIMS>
__device__ __forceinline__ double ham_in_sum(const DevShape& s, const double* c, uint32_t v,
                                             const uint32_t (&x)[DIMS], unsigned long long mask) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < DIMS; ++i) {
        const uint32_t st = s.stride[i], xi = x[i];
        const double* row = c + (v - xi * st);
        const unsigned long long mi = mask >> s.base[i];
#pragma unroll kHamUnroll
        for (uint32_t j = 0; j < xi; ++j)
            if ((mi >> j) & 1ull) acc = __dadd_rn(acc, __ldca(row + j * st));
    }
#pragma unroll
    for (int ii = 0; ii < DIMS; ++ii) {
        const int i = DIMS - 1 - ii;
        const uint32_t st = s.stride[i], xi = x[i], m = s.radix[i];
        const double* row = c + (v - xi * st);
        const unsigned long long mi = mask >> (s.base[i] + xi);  // value j at bit j - xi - 1
#pragma unroll kHamUnroll
        for (uint32_t j = xi + 1; j < m; ++j)
            if ((mi >> (j - xi - 1)) & 1ull) acc = __dadd_rn(acc, __ldca(row + j * st));
    }
    return acc;
}

__device__ __forceinline__ double reduce_parts_h(const double* part, int nblocks, int k,
                                                 double* s_red) {
    double acc = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += kHT) acc = __dadd_rn(acc, part[b * 3 + k]);
    return block_sum<kHT>(acc, s_red);
}

template <int DIMS, typename MW>
__global__ void __launch_bounds__(kHT, TK_HAM_MINB)
    pagerank_ham_tiled_kernel(const DevShape s, const HamTilePlan hp, const PrArgs a) {
    __shared__ double s_red[kHT / 32];
    __shared__ double s_rcp[kMaxHamDeg + 1];
    cg::grid_group grid = cg::this_grid();
    const int t = threadIdx.x;
    const uint32_t G = gridDim.x;
    const uint32_t ntiles = (a.n + kHT - 1) / kHT;
    const MW* __restrict__ inm = static_cast<const MW*>(a.inm);
    if (t <= kMaxHamDeg) s_rcp[t] = t ? __drcp_rn(t) : 0.0;
    uint32_t xinv[DIMS];
#pragma unroll
    for (int i = 0; i < DIMS; ++i) {
        const uint32_t P = s.stride[i] * s.radix[i];
        xinv[i] = ((hp.inv >> i) & 1u) ? (static_cast<uint32_t>(t) % P) / s.stride[i] : 0u;
    }

    // r_0 = 1/N: c_0 = r_0 / outdeg (r_0 for sinks), D_0 = sum over sinks
    double dang = 0.0;
    const uint64_t gsize = static_cast<uint64_t>(G) * kHT;
    for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * kHT + t; v < a.n; v += gsize) {
        const uint32_t deg = __ldg(a.odeg + v);
        if (deg) {
            a.c0[v] = __ddiv_rn(a.inv_n, static_cast<double>(deg));
        } else {
            a.c0[v] = a.inv_n;
            dang = __dadd_rn(dang, a.inv_n);
        }
    }
    dang = block_sum<kHT>(dang, s_red);
    if (t == 0) a.part[blockIdx.x * 3 + 1] = dang;
    grid.sync();
    double D = reduce_parts_h(a.part, G, 1, s_red);

    // c is re-written every iteration by other CTAs: coherent loads (ld.ca,
    // L1 invalidated by the grid barrier's fence), never the .nc path
    auto sweep = [&](const double* cc, double dn, double* out, bool final_pass,
                     double& lres, double& ldang, double& lsum) {
        for (uint32_t tile = blockIdx.x; tile < ntiles; tile += G) {
            const uint32_t v0 = tile * kHT;
            const uint32_t v = v0 + t;
            if (v >= a.n) continue;
            uint32_t x[DIMS];
            tile_digits<DIMS>(s, hp, v0, t, xinv, x);
            const unsigned long long mask = static_cast<unsigned long long>(__ldcs(inm + v));
            const uint32_t deg = __ldcs(a.odeg + v);
            const double acc = ham_in_sum<DIMS>(s, cc, v, x, mask);
            const double xr = __dadd_rn(a.teleport, __dmul_rn(a.damping, __dadd_rn(acc, dn)));
            if (final_pass) {
                out[v] = xr;
                continue;
            }
            const double cold = __ldca(cc + v);
            double q, d;
            if (deg) {
                const double dd = static_cast<double>(deg);
                q = div_small_h(xr, dd, s_rcp[deg]);
                d = fabs(__fma_rn(cold, dd, -xr));
            } else {
                q = xr;
                d = fabs(__dsub_rn(xr, cold));
                ldang = __dadd_rn(ldang, xr);
            }
            lres = __dadd_rn(lres, d);
            lsum = __dadd_rn(lsum, xr);
            __stcs(out + v, q);
        }
    };

    int cur = 0;
    long long it = 0;
    double res = 0.0, sum = 0.0, dn_last = 0.0;
    int status = 1;
    while (it < a.max_iter) {
        const double dn = __ddiv_rn(D, a.nd);
        const double* cc = cur ? a.c1 : a.c0;
        double* cn = cur ? a.c0 : a.c1;
        double lres = 0.0, ldang = 0.0, lsum = 0.0;
        sweep(cc, dn, cn, false, lres, ldang, lsum);
        lres = block_sum<kHT>(lres, s_red);
        ldang = block_sum<kHT>(ldang, s_red);
        lsum = block_sum<kHT>(lsum, s_red);
        double* part = a.part + static_cast<size_t>((it + 1) & 1) * G * 3;
        if (t == 0) {
            part[blockIdx.x * 3 + 0] = lres;
            part[blockIdx.x * 3 + 1] = ldang;
            part[blockIdx.x * 3 + 2] = lsum;
        }
        grid.sync();
        res = reduce_parts_h(part, G, 0, s_red);
        D = reduce_parts_h(part, G, 1, s_red);
        sum = reduce_parts_h(part, G, 2, s_red);
        dn_last = dn;
        ++it;
        cur ^= 1;
        if (res < a.tol) {
            status = 0;
            break;
        }
    }
    {
        double l0 = 0.0, l1 = 0.0, l2 = 0.0;
        sweep(cur ? a.c0 : a.c1, dn_last, a.r0, true, l0, l1, l2);
    }
    if (blockIdx.x == 0 && t == 0) {
        *a.out_iter = it;
        *a.out_res = res;
        *a.out_sum = sum;
        *a.out_parity = 0;
        *a.out_status = status;
    }
}

template <typename MW>
void* ham_kernel(int dims) {
    switch (dims) {
#define TK_HAM_CASE(D) \
    case D: return reinterpret_cast<void*>(pagerank_ham_tiled_kernel<D, MW>);
        TK_HAM_CASE(1) TK_HAM_CASE(2) TK_HAM_CASE(3) TK_HAM_CASE(4) TK_HAM_CASE(5)
        TK_HAM_CASE(6) TK_HAM_CASE(7) TK_HAM_CASE(8) TK_HAM_CASE(9) TK_HAM_CASE(10)
        TK_HAM_CASE(11) TK_HAM_CASE(12) TK_HAM_CASE(13) TK_HAM_CASE(14) TK_HAM_CASE(15)
        TK_HAM_CASE(16)
#undef TK_HAM_CASE
        default: return nullptr;
    }
}

}  // namespace

bool ham_tiled_supported(const DevShape& s) {
    if (s.kind != TK_HAMMING || s.dims < 1 || s.dims > 16 || s.slots > kMaxHamDeg) return false;
    for (int i = 0; i < s.dims; ++i) {
        const unsigned long long P = static_cast<unsigned long long>(s.stride[i]) * s.radix[i];
        const bool inv = P <= kHT && kHT % P == 0;
        const bool tiled = P % kHT == 0;
        if (!inv && !tiled) return false;
    }
    return true;
}

cudaError_t launch_pagerank_ham_tiled(const DevShape& s, bool wide, const PrArgs& a, int num_sms,
                                      int* grid_out, cudaStream_t stream) {
    if (!ham_tiled_supported(s)) return cudaErrorNotSupported;
    HamTilePlan hp{0u, 0u, 0u};
    for (int i = 0; i < s.dims; ++i) {
        const unsigned long long P = static_cast<unsigned long long>(s.stride[i]) * s.radix[i];
        if (P <= kHT && kHT % P == 0) hp.inv |= 1u << i;
        else if (s.stride[i] % kHT == 0) hp.uni |= 1u << i;
        else hp.tile |= 1u << i;
    }
    void* k = wide ? ham_kernel<unsigned long long>(s.dims) : ham_kernel<uint32_t>(s.dims);
    if (!k) return cudaErrorInvalidValue;
    int bps = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, kHT, 0);
    if (e != cudaSuccess) return e;
    if (bps < 1) return cudaErrorInvalidConfiguration;
    const uint64_t ntiles = (static_cast<uint64_t>(a.n) + kHT - 1) / kHT;
    uint64_t g = static_cast<uint64_t>(bps) * num_sms;
    if (g > ntiles) g = ntiles;
    if (g < 1) g = 1;
    *grid_out = static_cast<int>(g);
    if (std::getenv("TK_DEBUG"))
        std::fprintf(stderr, "[tk] pagerank_ham_tiled inv=%x uni=%x tile=%x bps=%d grid=%llu\n",
                     hp.inv, hp.uni, hp.tile, bps, static_cast<unsigned long long>(g));
    DevShape sc = s;
    PrArgs ac = a;
    void* args[] = {&sc, &hp, &ac};
    return cudaLaunchCooperativeKernel(k, dim3(static_cast<unsigned>(g)), dim3(kHT), args, 0,
                                       stream);
}

}  // namespace tk
