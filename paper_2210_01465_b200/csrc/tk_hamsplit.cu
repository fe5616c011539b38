// tk_hamsplit.cu -- Hamming PageRank by dimension groups (sm_100a).
//
// The tiled kernel (tk_hamming.cu) gathers all ~50 Hamming neighbour values
// of a rank in one pass; the lines of the slowest dimensions miss L2, so it
// moves ~190 B per rank and iteration at DRAM latency (C5: ~12 ms per
// iteration).  This kernel family splits the in-edge sum by dimension groups
// instead, keeping the oracle's summation order bit for bit.
//
// The dims are cut into contiguous groups g_0 (outermost) .. g_{G-1}.  A
// WINDOW of group g = [a, b) is the set of ranks that agree on every digit
// outside g and whose inner offset lies in one run of W consecutive values:
// it holds every g-line through its ranks, so the g-part of each rank's
// in-edge sum only needs the window (staged in shared memory, ~32 KB).
//
// The oracle sums the in-edges of v in ascending source rank (oracle.c
// or_pagerank): lower neighbours dims 0..D-1, then upper neighbours dims
// D-1..0, values ascending inside a dim.  Split by groups this chain is
//   lo(g_0) lo(g_1) .. lo(g_{G-1}) hi(g_{G-1}) .. hi(g_1) hi(g_0)
// and the partial sum travels between passes through HBM (acc[], 8 B):
//   LO(g_1) .. LO(g_{G-2}), LOHI(g_{G-1}), HI(g_{G-2}) .. HI(g_1), OUTER(g_0)
// where OUTER finishes iteration t (hi(g_0), r' = (1-d)/N + d (sum + D/N),
// c' = r'/outdeg, residual / sink-mass / sum partials) and, on the window it
// already holds, starts iteration t+1 (lo(g_0) of c').  Each pass streams its
// c, acc and in-mask words once: ~32-41 B per rank and pass, all coalesced.
//
// Inside a window a thread owns one line along the group's first dim (its
// values stay in registers, so that dim costs no shared loads); the other
// dims of the group read shared memory.  Every neighbour loop is unrolled
// over the value j (radix <= 8) with the in-mask bit and j <> x_i as
// predicates, so the order of the fp64 adds is the oracle's.
//
// Passes are plain launches (4 per iteration on C5) driven from the host in
// chunks of iterations; the OUTER pass's last CTA reduces the partials in a
// fixed order, advances the iteration counter and raises `done` on
// convergence, after which the queued passes exit at once.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "tk_kernels.cuh"

namespace tk {

namespace {

constexpr int kSpRmax = 32;       // radix bound (a dim's in-mask field fits a u32)
constexpr int kSpMaxGD = 8;       // dims per group
constexpr int kSpMaxThreads = 512;
constexpr int kSpMaxWinBytes = 32 * 1024;
constexpr int kSpNS = kSpMaxWinBytes / 8 / kSpMaxThreads;  // window slots per thread
constexpr int kSpMaxDeg = 64;
constexpr int kSpChunk = 4;       // iterations enqueued per host round trip
constexpr int kSpMaxPartCtas = 4096;
constexpr uint32_t kSpMinW = 8;   // outer windows: >= 64-byte runs per line value

#ifndef TK_SP_MINB
#define TK_SP_MINB 2  // CTAs per SM the register budget is sized for
#endif

enum SpMode : int { SP_LO = 0, SP_HI = 1, SP_LOHI = 2, SP_OUTER = 3, SP_INIT = 4, SP_FINAL = 5 };

struct SpGroup {
    int a, gd;            // dims [a, a + gd)
    uint32_t C;           // combos of the group's digits
    uint32_t I;           // inner size (stride of the group's last dim)
    uint32_t W;           // window width (consecutive inner offsets), a power of two
    int wshift;           // log2 W
    uint32_t nwin;        // N / (C * W)
    uint32_t ipw;         // I / W
    int base0;            // first in-mask slot of dim a
    int threads;          // CTA size
    uint32_t m[kSpMaxGD];
    int off[kSpMaxGD];                   // dim a + k's first slot, relative to base0
    int dkB[kSpMaxGD];                   // shared-memory bytes between values of dim a + k
    unsigned long long cmagic[kSpMaxGD];  // fdiv by the combo stride of dim a + k
};

struct SpState {
    long long it;
    double D;        // sink mass of the current iterate
    double dn_last;  // D / N used by the last OUTER pass
    double res, sum;
    int done, status;
    unsigned int count;
};

struct SpArgs {
    uint32_t n;
    double inv_n, nd, teleport, damping, tol;
    long long max_iter;
    const void* inm;
    const uint8_t* odeg;
    double* c0;
    double* c1;
    double* acc0;
    double* acc1;
    double* out_r;
    double* part;  // [grid][3]
    SpState* st;
    long long* out_iter;
    double* out_res;
    double* out_sum;
    int* out_parity;
    int* out_status;
};

__device__ __forceinline__ double sp_div_small(double x, double d, double y) {
    const double q0 = __dmul_rn(x, y);
    const double r = __fma_rn(-q0, d, x);
    return __fma_rn(r, y, q0);
}

// deterministic block sum for any blockDim (multiple of 32)
__device__ __forceinline__ double sp_block_sum(double v, double* s_red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t = __dadd_rn(t, s_red[w]);
    __syncthreads();
    return t;
}

// the group's in-mask bits, bit 0 = first slot of dim a (plan: span <= 32)
template <typename MW>
__device__ __forceinline__ uint32_t sp_mask(const void* inm, uint32_t v, int base0) {
    return static_cast<uint32_t>(
        static_cast<unsigned long long>(__ldcs(static_cast<const MW*>(inm) + v)) >> base0);
}

__device__ __forceinline__ void sp_cp8(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

__device__ __forceinline__ void sp_cp_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// A rank of the window: slot q = c * W + w (c = combo of the group's digits).
struct SpRank {
    uint32_t x[kSpMaxGD];  // the group's digits
};

template <int GD>
__device__ __forceinline__ void sp_digits(const SpGroup& g, uint32_t c, SpRank& r) {
    uint32_t qprev = 0;
#pragma unroll
    for (int k = 0; k < GD; ++k) {  // q_k = c / cst_k; x_k = q_k - q_{k-1} m_k
        const uint32_t qk = fdiv(c, g.cmagic[k]);
        r.x[k] = qk - qprev * g.m[k];
        qprev = qk;
    }
}

__device__ __forceinline__ double sp_lds(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

// acc += the values at row + j * dkB for the set bits j of the field, lowest
// first; fr is the bit-reversed field, so its highest set bit (bfind: position
// p) is j = 31 - p, at address row + 31 dkB - p dkB
__device__ __forceinline__ double sp_walk(double acc, uint32_t fr, uint32_t row, uint32_t dkB) {
    const uint32_t top = row + 31u * dkB;
    while (fr) {
        uint32_t pos;
        asm("bfind.u32 %0, %1;" : "=r"(pos) : "r"(fr));
        fr ^= 1u << pos;
        acc = __dadd_rn(acc, sp_lds(top - pos * dkB));
    }
    return acc;
}

// lower in-neighbours of the group's dims, ascending dims and values: the set
// bits of the dim's lower field (value j at bit j), lowest first (leading-zero
// count of the bit-reversed field).  qB: shared address of the rank's slot.
template <int GD>
__device__ __forceinline__ double sp_lo(double acc, uint32_t qB, uint32_t mk, const SpGroup& g,
                                        const SpRank& r) {
#pragma unroll
    for (int k = 0; k < GD; ++k) {
        const uint32_t xk = r.x[k];
        const uint32_t dkB = static_cast<uint32_t>(g.dkB[k]);
        const uint32_t fr = __brev((mk >> g.off[k]) & ((1u << xk) - 1u));
        acc = sp_walk(acc, fr, qB - xk * dkB, dkB);
    }
    return acc;
}

// upper in-neighbours, descending dims, ascending values (value j > x_k at
// bit j - 1 of the dim's field)
template <int GD>
__device__ __forceinline__ double sp_hi(double acc, uint32_t qB, uint32_t mk, const SpGroup& g,
                                        const SpRank& r) {
#pragma unroll
    for (int kk = 0; kk < GD; ++kk) {
        const int k = GD - 1 - kk;
        const uint32_t xk = r.x[k];
        const uint32_t dkB = static_cast<uint32_t>(g.dkB[k]);
        const uint32_t fr = __brev((mk >> (g.off[k] + xk)) & ((1u << (g.m[k] - 1u - xk)) - 1u));
        acc = sp_walk(acc, fr, qB + dkB, dkB);  // value x_k + 1 at bit 0
    }
    return acc;
}

template <int GD, int MODE, typename MW>
__global__ void __launch_bounds__(kSpMaxThreads, TK_SP_MINB)
    ham_split_kernel(const SpGroup g, const SpArgs a) {
    extern __shared__ double sp_smem[];
    __shared__ double s_red[kSpMaxThreads / 32];
    __shared__ double s_rcp[kSpMaxDeg + 1];
    __shared__ int s_last;
    SpState* st = a.st;
    if (MODE != SP_INIT && MODE != SP_FINAL && st->done) return;  // converged: queued passes exit
    const int tid = threadIdx.x;
    constexpr int T = kSpMaxThreads;  // every pass runs 512-thread CTAs
    if (MODE == SP_OUTER || MODE == SP_INIT)
        if (tid <= kSpMaxDeg) s_rcp[tid] = tid ? __drcp_rn(tid) : 0.0;
    const long long it = st->it;
    // iteration t works on c[t & 1], acc[t & 1]; OUTER writes c / acc [(t+1) & 1].
    // FINAL re-derives r' of the last OUTER pass (iteration it - 1).
    const int par = MODE == SP_FINAL ? static_cast<int>((it - 1) & 1) : static_cast<int>(it & 1);
    const double* cc = par ? a.c1 : a.c0;
    double* cn = (MODE == SP_INIT) ? a.c0 : (par ? a.c0 : a.c1);
    double* accb = par ? a.acc1 : a.acc0;
    double* accn = (MODE == SP_INIT) ? a.acc0 : (par ? a.acc0 : a.acc1);
    const double dn = MODE == SP_FINAL ? st->dn_last : __ddiv_rn(st->D, a.nd);

    const int nq = static_cast<int>(g.C * g.W);  // ranks per window
    double* cs = sp_smem;                         // c of the window (slot q)
    double* cs2 = sp_smem + nq;                   // OUTER: c' of the window
    const uint32_t csB = static_cast<uint32_t>(__cvta_generic_to_shared(cs));
    const uint32_t cs2B = static_cast<uint32_t>(__cvta_generic_to_shared(cs2));
    const int wsh = g.wshift;                     // W = 1 << wsh
    const uint32_t wmask = g.W - 1;

    double lres = 0.0, ldang = 0.0, lsum = 0.0;
    for (uint32_t widx = blockIdx.x; widx < g.nwin; widx += gridDim.x) {
        const uint32_t o = widx / g.ipw, ib = widx - o * g.ipw;
        const uint32_t vbase = o * g.C * g.I + ib * g.W;
        // slot q = tid + si * T: W divides T, so the rank advances by a fixed
        // stride per si and the inner offset is the thread's own
        const uint32_t v_t = vbase + (static_cast<uint32_t>(tid) >> wsh) * g.I +
                             (static_cast<uint32_t>(tid) & wmask);
        const uint32_t v_step = (static_cast<uint32_t>(T) >> wsh) * g.I;
        auto rank_of = [&](int si) -> uint32_t {  // recomputed at each use (no hoisted addresses)
            uint32_t st = v_step;
            asm volatile("" : "+r"(st));
            return v_t + static_cast<uint32_t>(si) * st;
        };
        // every global load of the window at once: c straight into shared memory
        // (cp.async), the partial sums, in-mask fields and out-degrees into registers
        double accv[kSpNS];
        uint32_t mkv[kSpNS], degw[(kSpNS + 3) / 4];  // out-degrees packed 4 per word
#pragma unroll
        for (int k4 = 0; k4 < (kSpNS + 3) / 4; ++k4) degw[k4] = 0u;
#pragma unroll
        for (int si = 0; si < kSpNS; ++si) {
            const int q = tid + si * T;
            accv[si] = 0.0;
            mkv[si] = 0u;
            if (q < nq) {
                const uint32_t v = rank_of(si);
                if (MODE != SP_INIT) sp_cp8(cs + q, cc + v);
                mkv[si] = sp_mask<MW>(a.inm, v, g.base0);
                if (MODE != SP_INIT) accv[si] = __ldcs(accb + v);
                if (MODE == SP_OUTER || MODE == SP_INIT)
                    degw[si >> 2] |= static_cast<uint32_t>(__ldcs(a.odeg + v)) << (8 * (si & 3));
            }
        }
        if (MODE == SP_INIT) {  // c_0 = 1/N / outdeg, 1/N for sinks
#pragma unroll
            for (int si = 0; si < kSpNS; ++si) {
                const int q = tid + si * T;
                if (q >= nq) continue;
                double cv;
                const uint32_t deg = (degw[si >> 2] >> (8 * (si & 3))) & 0xffu;
                if (deg) {
                    cv = __ddiv_rn(a.inv_n, static_cast<double>(deg));
                } else {
                    cv = a.inv_n;
                    ldang = __dadd_rn(ldang, a.inv_n);
                }
                __stcg(cn + rank_of(si), cv);
                cs[q] = cv;
            }
        } else {
            sp_cp_wait();
        }
        __syncthreads();
        if (MODE != SP_INIT) {
#pragma unroll
            for (int si = 0; si < kSpNS; ++si) {
                const int q = tid + si * T;
                if (q >= nq) continue;
                SpRank r;
                sp_digits<GD>(g, static_cast<uint32_t>(q) >> wsh, r);
                const uint32_t mk = mkv[si];
                double acc = accv[si];
                const uint32_t qB = csB + static_cast<uint32_t>(q) * 8u;
                if (MODE == SP_LO || MODE == SP_LOHI) acc = sp_lo<GD>(acc, qB, mk, g, r);
                if (MODE != SP_LO) acc = sp_hi<GD>(acc, qB, mk, g, r);
                const uint32_t v = rank_of(si);
                if (MODE == SP_LO || MODE == SP_HI || MODE == SP_LOHI) {
                    __stcs(accb + v, acc);
                    continue;
                }
                const double xr = __dadd_rn(a.teleport, __dmul_rn(a.damping, __dadd_rn(acc, dn)));
                if (MODE == SP_FINAL) {
                    __stcs(a.out_r + v, xr);
                    continue;
                }
                // OUTER: r' and c' of rank v
                const double cold = cs[q];
                const uint32_t deg = (degw[si >> 2] >> (8 * (si & 3))) & 0xffu;
                double qv, d;
                if (deg) {
                    const double dd = static_cast<double>(deg);
                    qv = sp_div_small(xr, dd, s_rcp[deg]);
                    d = fabs(__fma_rn(cold, dd, -xr));
                } else {
                    qv = xr;
                    d = fabs(__dsub_rn(xr, cold));
                    ldang = __dadd_rn(ldang, xr);
                }
                lres = __dadd_rn(lres, d);
                lsum = __dadd_rn(lsum, xr);
                cs2[q] = qv;
                __stcg(cn + v, qv);
            }
        }
        if (MODE == SP_OUTER || MODE == SP_INIT) {  // lo(g_0) of the next iterate
            const uint32_t cnewB = MODE == SP_OUTER ? cs2B : csB;
            if (MODE == SP_OUTER) __syncthreads();
#pragma unroll
            for (int si = 0; si < kSpNS; ++si) {
                const int q = tid + si * T;
                if (q >= nq) continue;
                SpRank r;
                sp_digits<GD>(g, static_cast<uint32_t>(q) >> wsh, r);
                __stcs(accn + rank_of(si),
                       sp_lo<GD>(0.0, cnewB + static_cast<uint32_t>(q) * 8u, mkv[si], g, r));
            }
        }
        __syncthreads();  // the window's slots are refilled next round
    }

    if (MODE == SP_OUTER || MODE == SP_INIT) {
        lres = sp_block_sum(lres, s_red);
        ldang = sp_block_sum(ldang, s_red);
        lsum = sp_block_sum(lsum, s_red);
        if (tid == 0) {
            a.part[blockIdx.x * 3 + 0] = lres;
            a.part[blockIdx.x * 3 + 1] = ldang;
            a.part[blockIdx.x * 3 + 2] = lsum;
            __threadfence();
            s_last = atomicAdd(&st->count, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            double r3[3] = {0.0, 0.0, 0.0};
            for (uint32_t b = tid; b < gridDim.x; b += blockDim.x)
                for (int k3 = 0; k3 < 3; ++k3)
                    r3[k3] = __dadd_rn(r3[k3], __ldcg(a.part + b * 3 + k3));
            const double res = sp_block_sum(r3[0], s_red);
            const double D = sp_block_sum(r3[1], s_red);
            const double sum = sp_block_sum(r3[2], s_red);
            if (tid == 0) {
                st->count = 0;
                st->D = D;
                if (MODE == SP_INIT) {
                    st->it = 0;
                    st->done = 0;
                    st->status = 1;
                } else {
                    st->res = res;
                    st->sum = sum;
                    st->dn_last = dn;
                    st->it = it + 1;
                    if (res < a.tol) {
                        st->done = 1;
                        st->status = 0;
                    } else if (it + 1 >= a.max_iter) {
                        st->done = 1;
                        st->status = 1;
                    }
                }
            }
        }
    }
    if (MODE == SP_FINAL && blockIdx.x == 0 && tid == 0) {
        *a.out_iter = st->it;
        *a.out_res = st->res;
        *a.out_sum = st->sum;
        *a.out_parity = 0;
        *a.out_status = st->status;
    }
}

template <int MODE, typename MW>
void* sp_kernel(int gd) {
    switch (gd) {
#define SP_CASE(G) \
    case G: return reinterpret_cast<void*>(ham_split_kernel<G, MODE, MW>);
        SP_CASE(1) SP_CASE(2) SP_CASE(3) SP_CASE(4) SP_CASE(5) SP_CASE(6) SP_CASE(7) SP_CASE(8)
#undef SP_CASE
        default: return nullptr;
    }
}

void* sp_select(int mode, int gd, bool wide) {
    switch (mode) {
#define SP_M(M)                                                                       \
    case M:                                                                           \
        return wide ? sp_kernel<M, unsigned long long>(gd) : sp_kernel<M, uint32_t>(gd);
        SP_M(SP_LO) SP_M(SP_HI) SP_M(SP_LOHI) SP_M(SP_OUTER) SP_M(SP_INIT) SP_M(SP_FINAL)
#undef SP_M
        default: return nullptr;
    }
}

unsigned long long sp_magic(uint32_t d) {
    return d <= 1 ? 0ull : (~0ull) / d + 1ull;  // ceil(2^64 / d) for d >= 2
}

// a group [a, b) with window width W; false when it does not fit
bool sp_make_group(const DevShape& s, int a, int b, uint32_t W, SpGroup* g) {
    if (b - a < 1 || b - a > kSpMaxGD) return false;
    uint64_t C = 1;
    for (int i = a; i < b; ++i) C *= s.radix[i];
    const uint32_t I = s.stride[b - 1];
    if (I % W) return false;
    if (C * W * 8 > static_cast<uint64_t>(kSpMaxWinBytes)) return false;
    // the group's in-mask slots must fit one u32 (bits base[a] .. base[b-1] + m - 2)
    if (s.base[b - 1] + static_cast<int>(s.radix[b - 1]) - 1 - s.base[a] > 32) return false;
    SpGroup t{};
    t.a = a;
    t.gd = b - a;
    t.C = static_cast<uint32_t>(C);
    t.I = I;
    t.W = W;
    t.wshift = 0;
    while ((1u << t.wshift) < W) ++t.wshift;
    t.nwin = static_cast<uint32_t>(static_cast<uint64_t>(s.n) / (C * W));
    t.ipw = I / W;
    t.base0 = s.base[a];
    if (kSpMaxThreads % W) return false;
    t.threads = kSpMaxThreads;
    for (int k = 0; k < t.gd; ++k) {
        const uint32_t cst = s.stride[a + k] / I;
        t.m[k] = s.radix[a + k];
        t.off[k] = s.base[a + k] - s.base[a];
        t.dkB[k] = static_cast<int>(cst * W * 8);
        t.cmagic[k] = sp_magic(cst);
    }
    *g = t;
    return true;
}

struct SpPlan {
    int G = 0;
    SpGroup grp[kMaxDims];
};

// groups from the innermost dim outwards, each as wide as a window allows;
// window width W = 1 when the group reaches the last dim, else 16 or 8
// (line-value runs of at least 64 bytes, whole sectors)
bool sp_plan(const DevShape& s, SpPlan* plan) {
    if (s.kind != TK_HAMMING || s.dims < 1 || s.dims > kMaxDims || s.slots > kMaxSlots)
        return false;
    for (int i = 0; i < s.dims; ++i)
        if (s.radix[i] < 2 || s.radix[i] > static_cast<uint32_t>(kSpRmax)) return false;
    SpGroup tmp[kMaxDims];
    int G = 0, b = s.dims;
    while (b > 0) {
        int best_a = -1;
        SpGroup best{};
        for (int a = b - 1; a >= 0; --a) {
            SpGroup g{};
            bool ok = false;
            const uint32_t wmin = (b == s.dims) ? 1u : kSpMinW;
            for (uint32_t W = (b == s.dims) ? 1u : 16u; W >= wmin; W >>= 1)
                if (sp_make_group(s, a, b, W, &g)) {
                    ok = true;
                    break;
                }
            if (!ok) break;
            best_a = a;
            best = g;
        }
        if (best_a < 0) return false;
        tmp[G++] = best;
        b = best_a;
    }
    plan->G = G;
    for (int k = 0; k < G; ++k) plan->grp[k] = tmp[G - 1 - k];  // outermost first
    return true;
}

int sp_smem_bytes(int mode, const SpGroup& g) {
    const int win = static_cast<int>(g.C * g.W * 8);
    return mode == SP_OUTER ? 2 * win : win;
}

cudaError_t sp_launch(int mode, const SpGroup& g, bool wide, const SpArgs& a, int num_sms,
                      int* grid_out, cudaStream_t stream) {
    void* k = sp_select(mode, g.gd, wide);
    if (!k) return cudaErrorInvalidValue;
    const int smem = sp_smem_bytes(mode, g);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int bps = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, g.threads, smem);
    if (e != cudaSuccess) return e;
    if (bps < 1) return cudaErrorInvalidConfiguration;
    uint64_t grid = static_cast<uint64_t>(bps) * num_sms;
    if (grid > g.nwin) grid = g.nwin;
    if (grid > static_cast<uint64_t>(kSpMaxPartCtas)) grid = kSpMaxPartCtas;
    if (grid < 1) grid = 1;
    if (grid_out) *grid_out = static_cast<int>(grid);
    SpGroup gc = g;
    SpArgs ac = a;
    void* args[] = {&gc, &ac};
    return cudaLaunchKernel(k, dim3(static_cast<unsigned>(grid)), dim3(g.threads), args,
                            static_cast<size_t>(smem), stream);
}

}  // namespace

bool ham_split_available(const DevShape& s) {
    SpPlan p;
    return sp_plan(s, &p) && p.G >= 1;
}

size_t ham_split_workspace_bytes(const DevShape& s) {
    (void)s;
    return static_cast<size_t>(kSpMaxPartCtas) * 3 * 8 + 256;
}

cudaError_t launch_pagerank_ham_split(const DevShape& s, bool wide, const PrArgs& pa,
                                      double* acc1, void* ws, int num_sms, int* grid_out,
                                      cudaStream_t stream) {
    SpPlan plan;
    if (!sp_plan(s, &plan)) return cudaErrorNotSupported;
    SpArgs a{};
    a.n = pa.n;
    a.inv_n = pa.inv_n;
    a.nd = pa.nd;
    a.teleport = pa.teleport;
    a.damping = pa.damping;
    a.tol = pa.tol;
    a.max_iter = pa.max_iter;
    a.inm = pa.inm;
    a.odeg = pa.odeg;
    a.c0 = pa.c0;
    a.c1 = pa.c1;
    a.acc0 = pa.r1;
    a.acc1 = acc1;
    a.out_r = pa.r0;
    a.st = static_cast<SpState*>(ws);
    a.part = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
    a.out_iter = pa.out_iter;
    a.out_res = pa.out_res;
    a.out_sum = pa.out_sum;
    a.out_parity = pa.out_parity;
    a.out_status = pa.out_status;
    const SpGroup& g0 = plan.grp[0];
    cudaError_t e = cudaMemsetAsync(ws, 0, 256, stream);
    if (e != cudaSuccess) return e;
    if (std::getenv("TK_DEBUG")) {
        for (int k = 0; k < plan.G; ++k) {
            const SpGroup& g = plan.grp[k];
            std::fprintf(stderr, "[tk] ham_split group %d: dims [%d,%d) C=%u I=%u W=%u threads=%d nwin=%u\n",
                         k, g.a, g.a + g.gd, g.C, g.I, g.W, g.threads, g.nwin);
        }
    }
    int grid = 0;
    if ((e = sp_launch(SP_INIT, g0, wide, a, num_sms, &grid, stream)) != cudaSuccess) return e;
    if (grid_out) *grid_out = grid;
    // one iteration: LO(g_1..g_{G-2}), LOHI(g_{G-1}), HI(g_{G-2}..g_1), OUTER(g_0)
    auto iteration = [&]() -> cudaError_t {
        cudaError_t ee;
        const int G = plan.G;
        for (int k = 1; k + 1 < G; ++k)
            if ((ee = sp_launch(SP_LO, plan.grp[k], wide, a, num_sms, nullptr, stream)) != cudaSuccess)
                return ee;
        if (G >= 2)
            if ((ee = sp_launch(SP_LOHI, plan.grp[G - 1], wide, a, num_sms, nullptr, stream)) !=
                cudaSuccess)
                return ee;
        for (int k = G - 2; k >= 1; --k)
            if ((ee = sp_launch(SP_HI, plan.grp[k], wide, a, num_sms, nullptr, stream)) != cudaSuccess)
                return ee;
        return sp_launch(SP_OUTER, g0, wide, a, num_sms, nullptr, stream);
    };
    // chunks of iterations, one chunk queued ahead of the convergence check
    SpState* host = nullptr;
    if ((e = cudaMallocHost(&host, 2 * sizeof(SpState))) != cudaSuccess) return e;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    for (int i = 0; i < 2 && e == cudaSuccess; ++i)
        e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    long long queued = 0;
    auto enqueue_chunk = [&](int slot) -> cudaError_t {
        cudaError_t ee = cudaSuccess;
        for (int i = 0; i < kSpChunk && queued < pa.max_iter && ee == cudaSuccess; ++i, ++queued)
            ee = iteration();
        if (ee != cudaSuccess) return ee;
        if ((ee = cudaMemcpyAsync(host + slot, a.st, sizeof(SpState), cudaMemcpyDeviceToHost,
                                  stream)) != cudaSuccess)
            return ee;
        return cudaEventRecord(ev[slot], stream);
    };
    if (e == cudaSuccess) e = enqueue_chunk(0);
    int slot = 0;
    bool more = queued < pa.max_iter;
    if (e == cudaSuccess && more) e = enqueue_chunk(1);
    while (e == cudaSuccess) {
        e = cudaEventSynchronize(ev[slot]);
        if (e != cudaSuccess) break;
        if (host[slot].done || queued >= pa.max_iter) break;
        e = enqueue_chunk(slot);
        slot ^= 1;
    }
    if (e == cudaSuccess) e = sp_launch(SP_FINAL, g0, wide, a, num_sms, nullptr, stream);
    for (int i = 0; i < 2; ++i)
        if (ev[i]) cudaEventDestroy(ev[i]);
    cudaStreamSynchronize(stream);
    cudaFreeHost(host);
    return e;
}

}  // namespace tk
