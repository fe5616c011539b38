// tk_ring.cu -- Adjacent PageRank with a per-CTA shared-memory ring of c
// (sm_100a).  The same iteration as pagerank_staged_kernel (tk_staged.cu:
// contribution-only sweeps, ordered in-edge sums, bit-identical r'), with a
// different way of getting the neighbour values into shared memory.
//
// Where the staged kernel's time goes (profiles/r01_ab_log.md
// round 2): a 512-rank tile needs 14 values per rank copied L2 -> shared
// memory (a near window of 2 per rank, 12 far ranges) and 25 shared loads per
// rank; the copies alone run in 24 ms, the consumers alone in 21 ms, together
// 33 ms -- both sides share the SM's shared-memory datapath.
//
// Here each CTA sweeps CHUNKS of consecutive tiles and keeps the last W = 8
// tiles of c in a shared-memory ring: tile k lives in slot k mod W, and the
// first / last A slots are mirrored past the ends, so the window [k - A, k + A]
// a consumer reads is linear and every neighbour source is one uniform pointer
// per tile.  Dims with stride <= A tiles (C5, A = 2: dims 5-11) read the ring;
// per tile the producers copy one new ring tile (plus its mirror for 2A of the W
// slots) and the far ranges of the other dims (C5: dims 0-4, 10 ranges): 11.5
// values per rank instead of 14.  W >= 2A + S (S stages) keeps every slot a
// consumer may still read out of the producers' way; at a chunk boundary the
// producer drains the pipeline before the warm-up.  Chunks are dealt
// round-robin to the CTAs.
//
// Measured (C5, profiles/r01_ab_log.md round 2): 57-58 ms against 33 ms for the
// staged kernel.  The consumers wait on the stage barriers (30 % of the stall
// samples): the chunked sweep turns the grid's far-range reads from a few
// contiguous fronts into ~1,500 scattered 4 KB streams (L2 hit 50 vs 61 %,
// DRAM read 106 vs 89 GB per launch).  Opt-in: TK_PR_RING=1.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "tk_kernels.cuh"
#include "tk_pipe.cuh"

namespace cg = cooperative_groups;

namespace tk {

namespace {

constexpr int kRT = 512;                          // ranks per tile = consumer threads
constexpr int kRConsumerWarps = kRT / 32;
constexpr int kRProdWarps = 4;
constexpr int kRThreads = kRT + 32 * kRProdWarps;
constexpr int kRW = 8;                            // ring slots (tile k -> slot k mod W)
constexpr int kRMaxStages = 4;
constexpr int kRMaxFar = 2 * kMaxDims;
constexpr int kRPwAhead = 2;
constexpr uint32_t kRPackMask = (1u << kPackedSlots) - 1;

struct RingPlan {
    int A;                         // ring reach (tiles each side)
    int stages;                    // pipeline stages (far ranges)
    int chunk;                     // tiles per chunk
    int nfar;                      // far ranges per tile
    unsigned int ring_dims;        // bit i: dim i reads the ring
    unsigned int far_ef;           // far range f loaded evict-first
    long long far_off[kRMaxFar];   // element offset of far range f from v0
    int lo_far[kMaxDims];          // far range holding the lower neighbour of dim i
    int hi_far[kMaxDims];          // ... the upper neighbour
    int stage_elems;               // nfar * T
};

struct RingPipe {
    uint64_t full[kRMaxStages];
    uint64_t empty[kRMaxStages];
};

__device__ __forceinline__ double div_small_r(double x, double d, double y) {
    const double q0 = __dmul_rn(x, y);
    const double r = __fma_rn(-q0, d, x);
    return __fma_rn(r, y, q0);
}

// m-th tile of CTA b: chunk b + (m / chunk) * G, tile (m mod chunk) of it
__device__ __forceinline__ uint32_t ring_tile(uint32_t m, uint32_t b, uint32_t G, uint32_t chunk) {
    const uint32_t c = m / chunk;
    return (b + c * G) * chunk + (m - c * chunk);
}

template <int DIMS>
__global__ void __launch_bounds__(kRThreads, 1)
    pagerank_ring_kernel(const __grid_constant__ DevShape s, const __grid_constant__ RingPlan p,
                         const PrArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ RingPipe pp;
    __shared__ double s_red[kRThreads / 32];
    __shared__ double s_rcp[kPackedSlots + 1];
    cg::grid_group grid = cg::this_grid();
    const int t = threadIdx.x;
    const uint32_t G = gridDim.x;
    const uint32_t ntiles = (a.n + kRT - 1) / kRT;
    const uint32_t chunk = static_cast<uint32_t>(p.chunk);
    const uint32_t nchunks = (ntiles + chunk - 1) / chunk;
    // tiles of this CTA per sweep (chunks b, b + G, ...; the last chunk may be short)
    uint32_t mine = 0;
    for (uint32_t c = blockIdx.x; c < nchunks; c += G)
        mine += min(chunk, ntiles - c * chunk);
    const int S = p.stages;
    double* ring = reinterpret_cast<double*>(smem);
    double* stages = ring + static_cast<size_t>(kRW + 2 * p.A) * kRT;
    if (t <= kPackedSlots) s_rcp[t] = t ? __drcp_rn(t) : 0.0;
    if (t == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&pp.full[i], kRProdWarps);
            mbar_init(&pp.empty[i], kRConsumerWarps);
        }
        fence_async_smem();
    }

    // r_0 = 1/N: c_0 = r_0 / outdeg (r_0 for sinks), D_0 = sum over sinks
    double dang = 0.0;
    const uint64_t gsize = static_cast<uint64_t>(G) * kRThreads;
    for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * kRThreads + t; v < a.n; v += gsize) {
        const uint32_t deg = __ldg(a.pw + v) >> kPackedSlots;
        if (deg) {
            a.c0[v] = __ddiv_rn(a.inv_n, static_cast<double>(deg));
        } else {
            a.c0[v] = a.inv_n;
            dang = __dadd_rn(dang, a.inv_n);
        }
    }
    dang = block_sum<kRThreads>(dang, s_red);
    if (t == 0) a.part[blockIdx.x * 3 + 1] = dang;
    fence_async_all();
    grid.sync();
    double D;
    {
        double acc = 0.0;
        for (uint32_t b = t; b < G; b += kRThreads) acc = __dadd_rn(acc, a.part[b * 3 + 1]);
        D = block_sum<kRThreads>(acc, s_red);
    }

    uint32_t kk = 0;  // stage uses so far (both sides, across sweeps)
    auto sweep = [&](const double* cc, double dn, double* out, bool final_pass, double& lres,
                     double& ldang, double& lsum) {
        if (t >= kRT) {  // ---------------------------------------- producers
            const int pw = (t - kRT) >> 5, lane = t & 31;
            const uint64_t pol = evict_first_policy();
            for (uint32_t m = 0; m < mine; ++m, ++kk) {
                const uint32_t k = ring_tile(m, blockIdx.x, G, chunk);
                const int st = static_cast<int>(kk % S);
                const uint32_t ph = (kk / S) & 1u;
                if (kk >= static_cast<uint32_t>(S)) mbar_wait(&pp.empty[st], ph ^ 1u);
                const bool first = m % chunk == 0;
                if (first && m > 0 && S > 1) {
                    // chunk boundary: the warm-up below rewrites ring tiles the
                    // previous chunk's last tiles may still read -- drain
                    const uint32_t pk = kk - 1;
                    mbar_wait(&pp.empty[pk % S], (pk / S) & 1u);
                }
                // copies of this tile: far ranges f < nfar into the stage, then
                // ring tiles -- the leading edge k + A and, at a chunk start, the
                // warm-up k - A .. k + A - 1 -- each into its slot's main position
                // and, for the first / last A slots, its mirror position (so that
                // every window [k - A, k + A] is linear in shared memory).
                // Copy q goes to lane q / P of warp q % P.
                const int nring = first ? 2 * p.A + 1 : 1;
                const int ncopy = p.nfar + 2 * nring;
                auto copy_of = [&](int q, const double*& src, double*& dst, bool& ef) -> uint32_t {
                    ef = false;
                    if (q < p.nfar) {
                        const long long lo = static_cast<long long>(k) * kRT + p.far_off[q];
                        const long long aa = lo < 0 ? 0 : lo;
                        const long long bb = lo + kRT > static_cast<long long>(a.n) ? a.n : lo + kRT;
                        if (bb <= aa) return 0u;
                        src = cc + aa;
                        dst = stages + static_cast<size_t>(st) * p.stage_elems +
                              static_cast<size_t>(q) * kRT + (aa - lo);
                        ef = (p.far_ef >> q) & 1u;
                        return static_cast<uint32_t>((bb - aa + 1) & ~1ll) * 8;
                    }
                    const int rq = q - p.nfar, ri = rq >> 1, mirror = rq & 1;
                    const long long rt = ri == 0 ? static_cast<long long>(k) + p.A
                                                 : static_cast<long long>(k) - p.A + (ri - 1);
                    if (rt < 0 || rt >= static_cast<long long>(ntiles)) return 0u;
                    const int slot = static_cast<int>(rt % kRW);
                    int pos = slot + p.A;
                    if (mirror) {
                        if (slot < p.A) pos = slot + p.A + kRW;
                        else if (slot >= kRW - p.A) pos = slot + p.A - kRW;
                        else return 0u;
                    }
                    const long long v0 = rt * kRT;
                    const long long cnt = v0 + kRT > static_cast<long long>(a.n) ? a.n - v0 : kRT;
                    src = cc + v0;
                    dst = ring + static_cast<size_t>(pos) * kRT;
                    return static_cast<uint32_t>((cnt + 1) & ~1ll) * 8;
                };
                // copy q goes to lane q / P of warp q % P; each warp announces its
                // bytes (arrive.expect_tx) before issuing its copies
                uint32_t bytes_w = 0;
                for (int q = lane * kRProdWarps + pw; q < ncopy; q += 32 * kRProdWarps) {
                    const double* src;
                    double* dst;
                    bool ef;
                    bytes_w += copy_of(q, src, dst, ef);
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) bytes_w += __shfl_xor_sync(0xffffffffu, bytes_w, o);
                if (lane == 0) {
                    fence_async_smem();
                    mbar_expect_tx(&pp.full[st], bytes_w);
                }
                __syncwarp();
                for (int q = lane * kRProdWarps + pw; q < ncopy; q += 32 * kRProdWarps) {
                    const double* src = nullptr;
                    double* dst = nullptr;
                    bool ef = false;
                    const uint32_t bytes = copy_of(q, src, dst, ef);
                    if (!bytes) continue;
                    if (ef)
                        bulk_g2s_ef(dst, src, bytes, &pp.full[st], pol);
                    else
                        bulk_g2s(dst, src, bytes, &pp.full[st]);
                }
            }
            return;
        }
        // --------------------------------------------------------- consumers
        const int lane = t & 31;
        auto pw_of = [&](uint32_t m) -> uint32_t {
            if (m >= mine) return 0u;
            const uint32_t v = ring_tile(m, blockIdx.x, G, chunk) * kRT + t;
            return v < a.n ? __ldcs(a.pw + v) : 0u;
        };
        uint32_t wq[kRPwAhead];
#pragma unroll
        for (int i = 0; i < kRPwAhead; ++i) wq[i] = pw_of(i);
        uint32_t k = blockIdx.x * chunk, inch = 0;  // current tile, position in its chunk
        // the prefetch tile (m + kRPwAhead), advanced the same way
        uint32_t kp = ring_tile(kRPwAhead, blockIdx.x, G, chunk), inchp = kRPwAhead % chunk;
        for (uint32_t m = 0; m < mine; ++m, ++kk) {
            const int st = static_cast<int>(kk % S);
            const uint32_t ph = (kk / S) & 1u;
            const uint32_t w = wq[0];
#pragma unroll
            for (int i = 0; i + 1 < kRPwAhead; ++i) wq[i] = wq[i + 1];
            {
                const uint32_t vp = kp * kRT + t;
                wq[kRPwAhead - 1] = m + kRPwAhead < mine && vp < a.n ? __ldcs(a.pw + vp) : 0u;
                if (++inchp == chunk) {
                    inchp = 0;
                    kp += (G - 1) * chunk + 1;
                } else {
                    ++kp;
                }
            }
            mbar_wait(&pp.full[st], ph);
            const uint32_t mask = w & kRPackMask;
            // tile k's window [k - A, k + A] starts at ring position k mod W;
            // every neighbour source is a uniform pointer per tile (ring or stage)
            const double* nb = ring + static_cast<size_t>(k % kRW + p.A) * kRT;
            const double* fb = stages + static_cast<size_t>(st) * p.stage_elems;
            double acc = 0.0;
            // in-neighbours in ascending rank: v-s_0 < ... < v-s_{D-1} < v+s_{D-1} < ... < v+s_0
            const double* src[2 * DIMS];
#pragma unroll
            for (int i = 0; i < DIMS; ++i) {
                const bool rg = (p.ring_dims >> i) & 1u;
                src[i] = rg ? nb - s.stride[i] : fb + static_cast<size_t>(p.lo_far[i]) * kRT;
                src[2 * DIMS - 1 - i] = rg ? nb + s.stride[i] : fb + static_cast<size_t>(p.hi_far[i]) * kRT;
            }
#pragma unroll
            for (int j = 0; j < 2 * DIMS; ++j)
                if ((mask >> j) & 1u) acc = __dadd_rn(acc, src[j][t]);
            const double cold = final_pass ? 0.0 : nb[t];
            __syncwarp();
            if (lane == 0) mbar_arrive(&pp.empty[st]);  // this warp is done with the stage
            const uint32_t v = k * kRT + t;
            // next tile of this CTA: the next one in the chunk, or the next chunk
            if (++inch == chunk) {
                inch = 0;
                k += (G - 1) * chunk + 1;
            } else {
                ++k;
            }
            if (v >= a.n) continue;
            const uint32_t deg = w >> kPackedSlots;
            const double x = __dadd_rn(a.teleport, __dmul_rn(a.damping, __dadd_rn(acc, dn)));
            if (final_pass) {
                out[v] = x;
                continue;
            }
            double q, d;
            if (deg) {
                const double dd = static_cast<double>(deg);
                q = div_small_r(x, dd, s_rcp[deg]);
                d = fabs(__fma_rn(cold, dd, -x));
            } else {
                q = x;
                d = fabs(__dsub_rn(x, cold));
                ldang = __dadd_rn(ldang, x);
            }
            lres = __dadd_rn(lres, d);
            lsum = __dadd_rn(lsum, x);
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
        fence_async_all();  // this sweep's c' stores before the next sweep's bulk reads
        lres = block_sum<kRThreads>(lres, s_red);
        ldang = block_sum<kRThreads>(ldang, s_red);
        lsum = block_sum<kRThreads>(lsum, s_red);
        double* part = a.part + static_cast<size_t>((it + 1) & 1) * G * 3;
        if (t == 0) {
            part[blockIdx.x * 3 + 0] = lres;
            part[blockIdx.x * 3 + 1] = ldang;
            part[blockIdx.x * 3 + 2] = lsum;
        }
        grid.sync();
        double r3[3] = {0.0, 0.0, 0.0};
        for (uint32_t b = t; b < G; b += kRThreads)
            for (int k3 = 0; k3 < 3; ++k3) r3[k3] = __dadd_rn(r3[k3], part[b * 3 + k3]);
        res = block_sum<kRThreads>(r3[0], s_red);
        D = block_sum<kRThreads>(r3[1], s_red);
        sum = block_sum<kRThreads>(r3[2], s_red);
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
    // r' of the last iteration, from the contributions it read (buffer cur ^ 1)
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

void* ring_kernel(int dims) {
    switch (dims) {
#define TK_RING_CASE(D) \
    case D: return reinterpret_cast<void*>(pagerank_ring_kernel<D>);
        TK_RING_CASE(1) TK_RING_CASE(2) TK_RING_CASE(3) TK_RING_CASE(4) TK_RING_CASE(5)
        TK_RING_CASE(6) TK_RING_CASE(7) TK_RING_CASE(8) TK_RING_CASE(9) TK_RING_CASE(10)
        TK_RING_CASE(11) TK_RING_CASE(12) TK_RING_CASE(13)
#undef TK_RING_CASE
        default: return nullptr;
    }
}

bool make_ring_plan(const DevShape& s, int smem_budget, int num_sms, RingPlan* out) {
    if (s.kind != TK_ADJACENT || s.dims < 1 || 2 * s.dims > kPackedSlots) return false;
    const uint64_t ntiles = (static_cast<uint64_t>(s.n) + kRT - 1) / kRT;
    RingPlan p{};
    p.chunk = 64;
    if (const char* e = std::getenv("TK_RING_CHUNK")) p.chunk = std::atoi(e);
    if (p.chunk < 1) return false;
    // every CTA sweeps at least one whole chunk
    if (ntiles < static_cast<uint64_t>(num_sms) * p.chunk) return false;
    // reach A: W >= 2A + S keeps every slot a consumer may still read out of the
    // producers' way; the ring region holds W slots plus A mirror slots each side
    int best = -1;
    for (int S = kRMaxStages; S >= 2 && best < 0; --S) {
        for (int A = (kRW - S) / 2; A >= 1; --A) {
            int nfar = 0;
            bool even = true;
            for (int i = 0; i < s.dims; ++i)
                if (static_cast<long long>(s.stride[i]) > static_cast<long long>(A) * kRT) {
                    nfar += 2;
                    even = even && (s.stride[i] % 2 == 0);
                }
            if (!even) continue;  // far ranges must start 16-byte aligned
            const long long need = static_cast<long long>(kRW + 2 * A) * kRT * 8 +
                                   static_cast<long long>(S) * nfar * kRT * 8;
            if (need > smem_budget) continue;
            p.A = A;
            p.stages = S;
            p.nfar = nfar;
            best = A;
            break;
        }
    }
    if (best < 0) return false;
    int f = 0;
    p.ring_dims = 0;
    for (int i = 0; i < s.dims; ++i) {
        if (static_cast<long long>(s.stride[i]) <= static_cast<long long>(p.A) * kRT) {
            p.ring_dims |= 1u << i;
            p.lo_far[i] = p.hi_far[i] = 0;
        } else {
            p.far_off[f] = -static_cast<long long>(s.stride[i]);
            p.lo_far[i] = f++;
            p.far_off[f] = static_cast<long long>(s.stride[i]);
            p.hi_far[i] = f++;
        }
    }
    p.stage_elems = p.nfar * kRT;
    // far ranges whose reuse distance outlives L2 (as StagePlan::far_ef)
    p.far_ef = 0;
    {
        const char* e = std::getenv("TK_EF_RANKS");
        const long long lim = e ? std::atoll(e) : (64ll << 20) / 24;
        for (int q = 0; q < p.nfar; ++q) {
            const long long d = p.far_off[q] < 0 ? -p.far_off[q] : p.far_off[q];
            if (d > lim) p.far_ef |= 1u << q;
        }
    }
    if (p.nfar + 2 * (2 * p.A + 1) > 32 * kRProdWarps) return false;
    *out = p;
    return true;
}

}  // namespace

bool ring_plan_available(const DevShape& s, int smem_budget, int num_sms) {
    // opt-in (TK_PR_RING=1): correct, but slower than the staged kernel on C5
    // (63 vs 33 ms: ~2x the instructions for the ring addressing at the same
    // issue rate; profiles/r01_ab_log.md, round 2)
    if (!std::getenv("TK_PR_RING") || std::getenv("TK_PR_STAGED")) return false;
    RingPlan p{};
    return make_ring_plan(s, smem_budget, num_sms, &p);
}

cudaError_t launch_pagerank_ring(const DevShape& s, const PrArgs& a, int smem_budget, int num_sms,
                                 int* grid_out, cudaStream_t stream) {
    RingPlan p{};
    if (!make_ring_plan(s, smem_budget, num_sms, &p)) return cudaErrorNotSupported;
    void* k = ring_kernel(s.dims);
    if (!k) return cudaErrorInvalidValue;
    const size_t smem = static_cast<size_t>(kRW + 2 * p.A) * kRT * 8 +
                        static_cast<size_t>(p.stages) * p.nfar * kRT * 8;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int bps = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, kRThreads, smem);
    if (e != cudaSuccess) return e;
    if (bps < 1) return cudaErrorInvalidConfiguration;
    const uint64_t ntiles = (static_cast<uint64_t>(a.n) + kRT - 1) / kRT;
    const uint64_t nchunks = (ntiles + p.chunk - 1) / p.chunk;
    uint64_t g = static_cast<uint64_t>(num_sms);
    if (g > nchunks) g = nchunks;
    *grid_out = static_cast<int>(g);
    if (std::getenv("TK_DEBUG"))
        std::fprintf(stderr, "[tk] pagerank_ring A=%d stages=%d nfar=%d chunk=%d ring_dims=%x smem=%zu grid=%llu\n",
                     p.A, p.stages, p.nfar, p.chunk, p.ring_dims, smem,
                     static_cast<unsigned long long>(g));
    DevShape sc = s;
    PrArgs ac = a;
    void* args[] = {&sc, &p, &ac};
    return cudaLaunchCooperativeKernel(k, dim3(static_cast<unsigned>(g)), dim3(kRThreads), args,
                                       smem, stream);
}

}  // namespace tk
