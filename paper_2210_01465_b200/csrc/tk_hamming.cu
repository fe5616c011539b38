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
#include "tk_pipe.cuh"

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

// ================================================== staged Hamming kernel --
//
// The tiled kernel above gathers every line value with a warp load and keeps
// only two loads in flight per thread: it is bound by memory-level parallelism
// (DRAM at ~20 %) and re-reads the lines of the slowest dimensions from DRAM
// (~190 B per rank and iteration on C5).
//
// This kernel streams the lines through shared memory instead.  The dims split
// into OUTER dims 0..k-1, whose strides are multiples of the tile (their digit
// is fixed over a tile), and INNER dims k..D-1, whose lines stay inside the
// aligned block of B = s_{k-1} ranks that holds the tile.  For a tile at v0:
//   - every outer neighbour line (i, j) is one whole range c[v0 + (j - x_i) s_i,
//     + T).  A tile's R = sum_{i<k} (m_i - 1) ranges, in the order the in-edge
//     sum consumes them, are cut into chunks of at most C ranges; a chunk is
//     one ring stage with one full / empty mbarrier pair, filled by one
//     producer warp with one 1-D bulk copy (TMA) per lane;
//   - the inner lines come from a copy of the block (double-buffered).
// Per-range barriers cost ~650 cycles per range in handshakes (measured: a
// variant without any copies ran as slow), so the handshake is per chunk.
// The in-edge sum keeps the oracle's order (ascending source rank): lower
// ranges dims 0..k-1, inner lower / upper from the block, upper ranges dims
// k-1..0 -- so r' stays bit-identical.
constexpr int kHsT = 512;                      // ranks per tile = consumer threads
constexpr int kHsConsumerWarps = kHsT / 32;
constexpr int kHsProdWarps = 2;
constexpr int kHsThreads = kHsT + 32 * kHsProdWarps;
constexpr int kHsMaxStages = 8;
constexpr int kHsMaxChunk = 16;                // ranges per stage (one lane each)
constexpr int kHsMaxNear = 4096;               // block values (32 KB per buffer)

struct HamStagePlan {
    int k;                                  // outer dims
    uint32_t B;                             // block = s_{k-1} ranks
    uint32_t tpb;                           // tiles per block = B / T
    int R;                                  // outer ranges per tile
    int C;                                  // ranges per stage (chunk)
    int stages;                             // ring stages
    int order;                              // tile sweep order (ham_tile_of)
    unsigned long long tpb_magic;           // fdiv by tpb (0 when tpb == 1)
    unsigned long long rmagic[kMaxDims];    // fdiv by radix[i]
};

struct HamPipe {
    uint64_t full[kHsMaxStages];
    uint64_t empty[kHsMaxStages];
    uint64_t nfull[2];
    uint64_t nempty[2];
};

// sweep position g -> tile origin v0 and the outer digits.  hp.order 0: rank
// order (tile g); 1: block offset fastest, then x_0 .. x_{k-1}
template <int DIMS>
__device__ __forceinline__ uint32_t ham_tile_of(const DevShape& s, const HamStagePlan& hp,
                                                uint32_t g, uint32_t (&x)[DIMS],
                                                uint32_t& w) {
    const uint32_t r0 = fdiv(g, hp.tpb_magic);
    w = g - r0 * hp.tpb;
    if (hp.order == 0) {
        const uint32_t v0 = g * kHsT;
#pragma unroll
        for (int i = 0; i < DIMS; ++i)
            if (i < hp.k) {
                const uint32_t q = fdiv(v0, s.magic[i]);
                x[i] = q - fdiv(q, hp.rmagic[i]) * s.radix[i];
            }
        return v0;
    }
    uint32_t r = r0, v0 = w * kHsT;
#pragma unroll
    for (int i = 0; i < DIMS; ++i) {
        if (i < hp.k) {
            const uint32_t q = fdiv(r, hp.rmagic[i]);
            x[i] = r - q * s.radix[i];
            r = q;
            v0 += x[i] * s.stride[i];
        }
    }
    return v0;
}

// range r of a tile's consumption sequence -> signed line offset (j - x_i) s_i
template <int DIMS>
__device__ __forceinline__ long long ham_range_offset(const DevShape& s, const HamStagePlan& hp,
                                                      const uint32_t (&x)[DIMS], int r) {
    long long off = 0;
    bool found = false;
#pragma unroll
    for (int i = 0; i < DIMS; ++i)
        if (i < hp.k && !found) {
            if (r < static_cast<int>(x[i])) {
                off = static_cast<long long>(r - static_cast<int>(x[i])) * s.stride[i];
                found = true;
            } else {
                r -= static_cast<int>(x[i]);
            }
        }
#pragma unroll
    for (int ii = 0; ii < DIMS; ++ii) {
        const int i = DIMS - 1 - ii;
        if (i < hp.k && !found) {
            const int up = static_cast<int>(s.radix[i] - 1 - x[i]);
            if (r < up) {
                off = static_cast<long long>(r + 1) * s.stride[i];
                found = true;
            } else {
                r -= up;
            }
        }
    }
    return off;
}

template <int DIMS, typename MW>
__global__ void __launch_bounds__(kHsThreads, 1)
    pagerank_ham_staged_kernel(const __grid_constant__ DevShape s,
                               const __grid_constant__ HamStagePlan hp, const PrArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ HamPipe pp;
    __shared__ double s_red[kHsThreads / 32];
    __shared__ double s_rcp[kMaxHamDeg + 1];
    cg::grid_group grid = cg::this_grid();
    const int t = threadIdx.x;
    const uint32_t G = gridDim.x;
    const uint32_t ntiles = a.n / kHsT;  // outer dims exist: T divides N
    const int S = hp.stages, C = hp.C;
    const int nchunks = (hp.R + C - 1) / C;  // stages per tile
    const MW* __restrict__ inm = static_cast<const MW*>(a.inm);
    double* ring = reinterpret_cast<double*>(smem);
    const size_t stage_elems = static_cast<size_t>(C) * kHsT;
    double* nearb = ring + static_cast<size_t>(S) * stage_elems;
    if (t <= kMaxHamDeg) s_rcp[t] = t ? __drcp_rn(t) : 0.0;
    if (t == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&pp.full[i], 1);
            mbar_init(&pp.empty[i], kHsConsumerWarps);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&pp.nfull[i], 1);
            mbar_init(&pp.nempty[i], kHsConsumerWarps);
        }
        fence_async_smem();
    }

    // r_0 = 1/N: c_0 = r_0 / outdeg (r_0 for sinks), D_0 = sum over sinks
    double dang = 0.0;
    const uint64_t gsize = static_cast<uint64_t>(G) * kHsThreads;
    for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * kHsThreads + t; v < a.n; v += gsize) {
        const uint32_t deg = __ldg(a.odeg + v);
        if (deg) {
            a.c0[v] = __ddiv_rn(a.inv_n, static_cast<double>(deg));
        } else {
            a.c0[v] = a.inv_n;
            dang = __dadd_rn(dang, a.inv_n);
        }
    }
    dang = block_sum<kHsThreads>(dang, s_red);
    if (t == 0) a.part[blockIdx.x * 3 + 1] = dang;
    fence_async_all();
    grid.sync();
    double D;
    {
        double acc = 0.0;
        for (uint32_t b = t; b < G; b += kHsThreads) acc = __dadd_rn(acc, a.part[b * 3 + 1]);
        D = block_sum<kHsThreads>(acc, s_red);
    }

    // ring position (continues across sweeps on both sides)
    int st = 0;
    uint32_t sph = 0;     // phase of stage st
    uint32_t uses = 0;    // stage uses so far
    uint32_t ntile = 0;   // tiles so far (block buffer ntile & 1, phase (ntile >> 1) & 1)
    auto advance = [&]() {
        ++uses;
        if (++st == S) {
            st = 0;
            sph ^= 1u;
        }
    };

    auto sweep = [&](const double* cc, double dn, double* out, bool final_pass, double& lres,
                     double& ldang, double& lsum) {
        if (t >= kHsT) {  // ------------------------------------------ producers
            const int pw = (t - kHsT) >> 5, lane = t & 31;
            for (uint32_t g = blockIdx.x; g < ntiles; g += G, ++ntile) {
                uint32_t x[DIMS], w;
                const uint32_t v0 = ham_tile_of<DIMS>(s, hp, g, x, w);
                if (pw == 0 && lane == 0) {
                    const int nb = ntile & 1;
                    if (ntile >= 2) mbar_wait(&pp.nempty[nb], ((ntile >> 1) & 1u) ^ 1u);
                    mbar_expect_tx(&pp.nfull[nb], hp.B * 8);
                    bulk_g2s(nearb + static_cast<size_t>(nb) * hp.B, cc + (v0 - w * kHsT),
                             hp.B * 8, &pp.nfull[nb]);
                }
                // chunk q of the stream is filled by producer warp q % P, one
                // range per lane
                for (int ch = 0; ch < nchunks; ++ch) {
                    if (static_cast<int>(uses % kHsProdWarps) == pw) {
                        const int r0 = ch * C;
                        const int cnt = min(C, hp.R - r0);
                        if (lane == 0) {
                            if (uses >= static_cast<uint32_t>(S)) mbar_wait(&pp.empty[st], sph ^ 1u);
#ifndef TK_HX_NOCOPY
                            mbar_expect_tx(&pp.full[st], static_cast<uint32_t>(cnt) * kHsT * 8);
#else
                            mbar_arrive(&pp.full[st]);  // timing experiment: no data movement
#endif
                        }
                        __syncwarp();
#ifndef TK_HX_NOCOPY
                        if (lane < cnt) {
                            const long long off = ham_range_offset<DIMS>(s, hp, x, r0 + lane);
                            bulk_g2s(ring + st * stage_elems + static_cast<size_t>(lane) * kHsT,
                                     cc + (static_cast<long long>(v0) + off), kHsT * 8, &pp.full[st]);
                        }
#endif
                    }
                    advance();
                }
            }
            return;
        }
        // ------------------------------------------------------- consumers
        const int lane = t & 31;
        // in-masks and out-degrees are streamed kAhead tiles ahead of use
        // (their DRAM latency would otherwise stall every warp of the CTA at
        // the start of each tile: the warps move in lockstep through the ring)
        constexpr int kAhead = 2;
        auto rank_of = [&](uint32_t gg) -> uint32_t {
            uint32_t xx[DIMS], ww;
            return ham_tile_of<DIMS>(s, hp, gg, xx, ww) + t;
        };
        unsigned long long mq[kAhead];
        uint32_t dq[kAhead];
#pragma unroll
        for (int i = 0; i < kAhead; ++i) {
            const uint32_t gg = blockIdx.x + i * G;
            const uint32_t vv = gg < ntiles ? rank_of(gg) : 0u;
            mq[i] = gg < ntiles ? static_cast<unsigned long long>(__ldcs(inm + vv)) : 0ull;
            dq[i] = gg < ntiles ? __ldcs(a.odeg + vv) : 0u;
        }
        for (uint32_t g = blockIdx.x; g < ntiles; g += G, ++ntile) {
            uint32_t x[DIMS], w;
            const uint32_t v0 = ham_tile_of<DIMS>(s, hp, g, x, w);
            const uint32_t v = v0 + t;
            const uint32_t o = w * kHsT + t;  // offset in the block
#pragma unroll
            for (int i = 0; i < DIMS; ++i)
                if (i >= hp.k) {
                    const uint32_t q = fdiv(o, s.magic[i]);
                    x[i] = q - fdiv(q, hp.rmagic[i]) * s.radix[i];
                }
            const unsigned long long mask = mq[0];
            const uint32_t deg = dq[0];
#pragma unroll
            for (int i = 0; i + 1 < kAhead; ++i) {
                mq[i] = mq[i + 1];
                dq[i] = dq[i + 1];
            }
            {
                const uint32_t gg = g + kAhead * G;
                const uint32_t vv = gg < ntiles ? rank_of(gg) : 0u;
                mq[kAhead - 1] = gg < ntiles ? static_cast<unsigned long long>(__ldcs(inm + vv)) : 0ull;
                dq[kAhead - 1] = gg < ntiles ? __ldcs(a.odeg + vv) : 0u;
            }
            // the tile's outer in-bits in consumption order: lower segments
            // dims 0..k-1 (bits base_i + [0, x_i)), then upper segments dims
            // k-1..0 (bits base_i + [x_i, m_i - 1)); L = lower ranges
            unsigned long long seq = 0;
            int L = 0, pos = 0;
#pragma unroll
            for (int i = 0; i < DIMS; ++i)
                if (i < hp.k) {
                    const int n = static_cast<int>(x[i]);
                    if (n) seq |= ((mask >> s.base[i]) & (~0ull >> (64 - n))) << pos;
                    pos += n;
                }
            L = pos;
#pragma unroll
            for (int ii = 0; ii < DIMS; ++ii) {
                const int i = DIMS - 1 - ii;
                if (i < hp.k) {
                    const int n = static_cast<int>(s.radix[i] - 1 - x[i]);
                    if (n) seq |= ((mask >> (s.base[i] + x[i])) & (~0ull >> (64 - n))) << pos;
                    pos += n;
                }
            }
            double acc = 0.0;
            int rin = C;  // position in the open stage (C: none open)
            const double* stg = ring;
            // ranges [rb, re) of the sequence, stage by stage
            auto outer = [&](int rb, int re) {
                int r = rb;
                while (r < re) {
                    if (rin == C) {
                        mbar_wait(&pp.full[st], sph);
                        stg = ring + st * stage_elems + t;
                        rin = 0;
                    }
                    const int n = min(C - rin, re - r);
                    const double* p0 = stg + static_cast<size_t>(rin) * kHsT;
                    // this call's n in-bits as a 32-bit word: immediate bit tests
                    const uint32_t sb = static_cast<uint32_t>(seq >> r) &
                                        (n >= 32 ? ~0u : ((1u << n) - 1u));
#pragma unroll
                    for (int q = 0; q < kHsMaxChunk; ++q) {
                        if (q < n) {
                            const double val = p0[static_cast<size_t>(q) * kHsT];
                            if (sb & (1u << q)) acc = __dadd_rn(acc, val);
                        }
                    }
                    rin += n;
                    r += n;
                    if (rin == C) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&pp.empty[st]);
                        advance();
                    }
                }
            };
            outer(0, L);  // lower neighbours of the outer dims
            // inner dims from the block copy: warp-uniform trip counts (m_i - 1),
            // the lane's own digit only in the predicate
            const int nb = ntile & 1;
            mbar_wait(&pp.nfull[nb], (ntile >> 1) & 1u);
            const double* blk = nearb + static_cast<size_t>(nb) * hp.B + o;
#pragma unroll
            for (int i = 0; i < DIMS; ++i) {
                if (i < hp.k) continue;
                const uint32_t sti = s.stride[i], xi = x[i], m1 = s.radix[i] - 1;
                const double* row = blk - static_cast<int>(xi * sti);
                const uint32_t mi = static_cast<uint32_t>(mask >> s.base[i]);
                if (m1 <= 8) {  // the usual radices: bit tests with immediates
#pragma unroll
                    for (uint32_t j = 0; j < 8; ++j)
                        if (j < m1 && j < xi && (mi & (1u << j))) acc = __dadd_rn(acc, row[j * sti]);
                } else {
                    for (uint32_t j = 0; j < m1; ++j)
                        if (j < xi && ((mask >> (s.base[i] + j)) & 1ull))
                            acc = __dadd_rn(acc, row[j * sti]);
                }
            }
            const double cold = final_pass ? 0.0 : blk[0];
#pragma unroll
            for (int ii = 0; ii < DIMS; ++ii) {
                const int i = DIMS - 1 - ii;
                if (i < hp.k) continue;
                const uint32_t sti = s.stride[i], xi = x[i], m = s.radix[i];
                const double* row = blk - static_cast<int>(xi * sti);
                const uint32_t mi = static_cast<uint32_t>(mask >> s.base[i]);  // value j > x_i: bit j - 1
                if (m <= 9) {
#pragma unroll
                    for (uint32_t j = 1; j < 9; ++j)
                        if (j < m && j > xi && (mi & (1u << (j - 1)))) acc = __dadd_rn(acc, row[j * sti]);
                } else {
                    for (uint32_t j = 1; j < m; ++j)
                        if (j > xi && ((mask >> (s.base[i] + j - 1)) & 1ull))
                            acc = __dadd_rn(acc, row[j * sti]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&pp.nempty[nb]);
            outer(L, hp.R);  // upper neighbours of the outer dims
            if (rin != C) {  // the tile's last, partial stage
                __syncwarp();
                if (lane == 0) mbar_arrive(&pp.empty[st]);
                advance();
            }
            const double xr = __dadd_rn(a.teleport, __dmul_rn(a.damping, __dadd_rn(acc, dn)));
            if (final_pass) {
                out[v] = xr;
                continue;
            }
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
        fence_async_all();  // this sweep's stores before the next sweep's bulk reads
        lres = block_sum<kHsThreads>(lres, s_red);
        ldang = block_sum<kHsThreads>(ldang, s_red);
        lsum = block_sum<kHsThreads>(lsum, s_red);
        double* part = a.part + static_cast<size_t>((it + 1) & 1) * G * 3;
        if (t == 0) {
            part[blockIdx.x * 3 + 0] = lres;
            part[blockIdx.x * 3 + 1] = ldang;
            part[blockIdx.x * 3 + 2] = lsum;
        }
        grid.sync();
        double r3[3] = {0.0, 0.0, 0.0};
        for (uint32_t b = t; b < G; b += kHsThreads)
            for (int k3 = 0; k3 < 3; ++k3) r3[k3] = __dadd_rn(r3[k3], part[b * 3 + k3]);
        res = block_sum<kHsThreads>(r3[0], s_red);
        D = block_sum<kHsThreads>(r3[1], s_red);
        sum = block_sum<kHsThreads>(r3[2], s_red);
        dn_last = dn;
        ++it;
        cur ^= 1;
#ifdef TK_X_ITERS
        if (it >= TK_X_ITERS) {
#else
        if (res < a.tol) {
#endif
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
void* ham_staged_kernel(int dims) {
    switch (dims) {
#define TK_HAM_CASE(D) \
    case D: return reinterpret_cast<void*>(pagerank_ham_staged_kernel<D, MW>);
        TK_HAM_CASE(2) TK_HAM_CASE(3) TK_HAM_CASE(4) TK_HAM_CASE(5) TK_HAM_CASE(6)
        TK_HAM_CASE(7) TK_HAM_CASE(8) TK_HAM_CASE(9) TK_HAM_CASE(10) TK_HAM_CASE(11)
        TK_HAM_CASE(12) TK_HAM_CASE(13) TK_HAM_CASE(14) TK_HAM_CASE(15) TK_HAM_CASE(16)
#undef TK_HAM_CASE
        default: return nullptr;
    }
}

unsigned long long magic_of(uint32_t d) {
    return d <= 1 ? 0ull : (~0ull) / d + 1ull;  // ceil(2^64 / d) for d >= 2
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

// Shapes the staged kernel takes: k >= 1 outer dims (strides multiples of the
// tile), a block B = s_{k-1} of at most kHsMaxNear ranks, at least one inner
// dim, and slots <= 64 (u64 in-mask).
bool ham_staged_plan(const DevShape& s, int smem_budget, HamStagePlanOut* out) {
    if (s.kind != TK_HAMMING || s.dims < 2 || s.dims > 16 || s.slots > kMaxHamDeg) return false;
    // opt-in (TK_HAM_STAGED=1): correct, but slower than the tiled kernel on C5
    // (454-468 vs 427-449 ms; profiles/r01_ab_log.md, round 2)
    if (!std::getenv("TK_HAM_STAGED")) return false;
    int k = 0;
    while (k < s.dims && s.stride[k] >= static_cast<uint32_t>(kHsT)) ++k;
    if (k == 0 || k == s.dims) return false;
    for (int i = 0; i < k; ++i)
        if (s.stride[i] % kHsT) return false;
    const uint32_t B = s.stride[k - 1];
    if (B > static_cast<uint32_t>(kHsMaxNear)) return false;
    int R = 0;
    for (int i = 0; i < k; ++i) R += static_cast<int>(s.radix[i]) - 1;
    const long long ring_bytes = smem_budget - 2ll * B * 8 - 256;
    // chunk: the fewest stages per tile that still leave >= 3 stages in the ring
    int C = 0, S = 0;
    for (int per = 1; per <= R; ++per) {
        const int c = (R + per - 1) / per;
        if (c > kHsMaxChunk) continue;
        const int st = static_cast<int>(ring_bytes / (static_cast<long long>(c) * kHsT * 8));
        if (st >= 3) {
            C = c;
            S = st > kHsMaxStages ? kHsMaxStages : st;
            break;
        }
    }
    if (!C) return false;
    out->k = k;
    out->B = B;
    out->R = R;
    out->C = C;
    out->stages = S;
    return true;
}

cudaError_t launch_pagerank_ham_staged(const DevShape& s, bool wide, const HamStagePlanOut& po,
                                       const PrArgs& a, int num_sms, int* grid_out,
                                       cudaStream_t stream) {
    HamStagePlan hp{};
    hp.k = po.k;
    hp.B = po.B;
    hp.tpb = po.B / kHsT;
    hp.R = po.R;
    hp.C = po.C;
    hp.stages = po.stages;
    hp.tpb_magic = magic_of(hp.tpb);
    {
        const char* e = std::getenv("TK_HAM_ORDER");  // A/B: 0 rank order, 1 digit order
        hp.order = e ? std::atoi(e) : 0;
    }
    for (int i = 0; i < s.dims; ++i) hp.rmagic[i] = magic_of(s.radix[i]);
    void* k = wide ? ham_staged_kernel<unsigned long long>(s.dims) : ham_staged_kernel<uint32_t>(s.dims);
    if (!k) return cudaErrorInvalidValue;
    const int smem = po.stages * po.C * kHsT * 8 + 2 * static_cast<int>(po.B) * 8;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int bps = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, kHsThreads, smem);
    if (e != cudaSuccess) return e;
    if (bps < 1) return cudaErrorInvalidConfiguration;
    const uint64_t ntiles = static_cast<uint64_t>(a.n) / kHsT;
    uint64_t g = static_cast<uint64_t>(num_sms);
    if (g > ntiles) g = ntiles;
    *grid_out = static_cast<int>(g);
    if (std::getenv("TK_DEBUG"))
        std::fprintf(stderr, "[tk] pagerank_ham_staged k=%d B=%u R=%d C=%d stages=%d grid=%llu smem=%d\n",
                     hp.k, hp.B, hp.R, hp.C, hp.stages, static_cast<unsigned long long>(g), smem);
    DevShape sc = s;
    PrArgs ac = a;
    void* args[] = {&sc, &hp, &ac};
    return cudaLaunchCooperativeKernel(k, dim3(static_cast<unsigned>(g)), dim3(kHsThreads), args,
                                       static_cast<size_t>(smem), stream);
}

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
