// tk_batch.cu -- a batch of small search spaces analysed by one launch
// (sm_100a): one CTA per space runs the whole analyze_landscape pipeline
// (landscape.hpp:77-79) -- FFG masks, f_opt, the ascending minima, the fp64
// PageRank power iteration, the C_p curve and the report rows -- with only
// block-level barriers between its phases.
//
// The per-space path (tk_analyze) launches ~10 kernels and synchronises with
// the host several times per space; for the 10^3-10^5-configuration spaces of
// real tuning problems (C4: 864..82,944 configurations) that latency, not the
// GPU, sets the pace.  Here a batch of spaces costs one upload, one launch and
// one read-back; the CTAs of different spaces run concurrently on the SMs.
//
// Semantics are those of the per-space path: edges
// u -> v for f(v) < f(u) (fp64, strict), minima = ok sinks in ascending rank,
// r_0 = 1/N, dangling mass over all sinks, the in-edge sum of each node in
// ascending source rank (so each r'[v] is bit-identical to the oracle's given
// the same dangling term), stop at the first iteration with L1 change < tol,
// C_p bands p = 0: f <= f_opt, p > 0: f < (1 + p) f_opt.  The global sums
// (dangling mass, residual, sum of r, C_p numerators) are block reductions in
// a fixed order: deterministic, equal to the oracle's up to summation order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "tk_kernels.cuh"

namespace tk {

namespace {

constexpr int kBT = 1024;  // threads per space

struct BatchDesc {
    const double* fit;
    const uint8_t* ok;
    uint32_t n;
    int dims;
    uint32_t radix[kMaxDims];
    uint32_t stride[kMaxDims];
    unsigned long long* inm;  // in-neighbour bits in ascending source order
    uint8_t* deg;
    uint8_t* flags;           // bit0 sink, bit1 ok sink, bit2 strict minimum, bit3 ok
    double* r0;
    double* r1;
    double* c;
    uint32_t* minima;
    uint32_t* inoff;          // in-CSR: N + 1 offsets, sources in ascending rank
    uint32_t* src;
    unsigned int* bar;        // group barrier {count, generation} (zeroed by the host)
    double* part;             // group partials: [kGroupMax][kPartW]
    // outputs
    BatchOut* out;
    double* rows;                   // report rows, 4 doubles each (rank bits, f, f_opt / f, r),
    unsigned long long* row_cursor; // packed for all spaces: one read-back (null: no rows)
};

// The neighbours of v in ascending rank (space.cpp:167-187 lists them per
// dimension; sorted by rank they are: lower ones dims ascending, values
// ascending, then upper ones dims descending, values ascending).  Adjacent
// keeps j = x - 1 and j = x + 1 only.  f(k, u) is called for the k-th one.
template <typename F>
__device__ __forceinline__ void walk_neighbours(const BatchDesc& d, int kind, uint32_t v,
                                                const uint32_t* x, F&& f) {
    int k = 0;
    for (int i = 0; i < d.dims; ++i) {
        const uint32_t xi = x[i], st = d.stride[i];
        const uint32_t j0 = kind == TK_ADJACENT ? (xi > 0 ? xi - 1 : xi) : 0;
        for (uint32_t j = j0; j < xi; ++j) f(k++, v - (xi - j) * st);
    }
    for (int i = d.dims - 1; i >= 0; --i) {
        const uint32_t xi = x[i], st = d.stride[i], m = d.radix[i];
        const uint32_t j1 = kind == TK_ADJACENT ? (xi + 2 < m ? xi + 2 : m) : m;
        for (uint32_t j = xi + 1; j < j1; ++j) f(k++, v + (j - xi) * st);
    }
}

__device__ __forceinline__ void digits_of(const BatchDesc& d, uint32_t v, uint32_t* x) {
    for (int i = 0; i < d.dims; ++i) x[i] = (v / d.stride[i]) % d.radix[i];
}

__global__ void __launch_bounds__(kBT) batch_analyze_kernel(const BatchDesc* __restrict__ descs,
                                                             uint32_t n_items, BatchParams P) {
    __shared__ double s_red[kBT / 32];
    __shared__ unsigned long long s_scan[kBT / 32];
    __shared__ double s_bf[kBT / 32];
    __shared__ unsigned long long s_br[kBT / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const BatchDesc& d = descs[item];
        BatchOut* o = d.out;
        const uint32_t n = d.n;
        uint32_t x[kMaxDims];
        // ---- FFG masks, flags, counts and f_opt (landscape.hpp:26-45, cache.cpp:55-72)
        unsigned long long e_loc = 0, ok_loc = 0, strict_loc = 0;
        double best_f = 0.0;
        unsigned long long best_r = ~0ull;
        for (uint32_t v = t; v < n; v += kBT) {
            digits_of(d, v, x);
            const double fv = d.fit[v];
            const bool okv = d.ok[v] != 0;
            unsigned long long inm = 0;
            uint32_t deg = 0;
            bool allgt = true;
            walk_neighbours(d, P.kind, v, x, [&](int k, uint32_t u) {
                const double fu = d.fit[u];
                if (fu < fv) ++deg;
                if (fu > fv)
                    inm |= 1ull << k;
                else
                    allgt = false;
            });
            d.inm[v] = inm;
            d.deg[v] = static_cast<uint8_t>(deg);
            const bool sink = deg == 0, okmin = sink && okv, strict = okv && allgt;
            d.flags[v] = static_cast<uint8_t>((sink ? 1 : 0) | (okmin ? 2 : 0) | (strict ? 4 : 0) |
                                              (okv ? 8 : 0));
            e_loc += deg;
            ok_loc += okv;
            strict_loc += strict;
            if (okv && (best_r == ~0ull || fv < best_f)) {  // ranks rise: lowest rank on ties
                best_f = fv;
                best_r = v;
            }
        }
        // block argmin of (f, rank) and the counts
#pragma unroll
        for (int s = 16; s; s >>= 1) {
            const double of = __shfl_xor_sync(0xffffffffu, best_f, s);
            const unsigned long long orr = __shfl_xor_sync(0xffffffffu, best_r, s);
            if (orr != ~0ull && (best_r == ~0ull || of < best_f || (of == best_f && orr < best_r))) {
                best_f = of;
                best_r = orr;
            }
        }
        if (lane == 0) {
            s_bf[warp] = best_f;
            s_br[warp] = best_r;
        }
        unsigned long long tot;
        block_exclusive_scan<kBT, unsigned long long>(e_loc, tot, s_scan);
        const unsigned long long n_edges = tot;
        block_exclusive_scan<kBT, unsigned long long>(ok_loc, tot, s_scan);
        const unsigned long long n_ok = tot;
        block_exclusive_scan<kBT, unsigned long long>(strict_loc, tot, s_scan);
        (void)n_ok;
        best_f = 0.0;
        best_r = ~0ull;
        for (int w = 0; w < kBT / 32; ++w) {
            const double of = s_bf[w];
            const unsigned long long orr = s_br[w];
            if (orr != ~0ull && (best_r == ~0ull || of < best_f || (of == best_f && orr < best_r))) {
                best_f = of;
                best_r = orr;
            }
        }
        __syncthreads();
        if (t == 0) {
            o->n_edges = n_edges;
            o->n_nodes = n;
            o->f_opt = best_f;
            o->opt_rank = best_r;
            o->iterations = 0;
            o->residual = 0.0;
            o->n_minima = 0;
        }
        if (best_r == ~0ull) {  // NoFeasiblePoint (errors.hpp:32-35)
            if (t == 0) o->status = TK_ENOFEAS;
            continue;
        }
        const double f_opt = best_f;
        // ---- minima: ok sinks in ascending rank
        unsigned long long mbase = 0;
        for (uint32_t v0 = 0; v0 < n; v0 += kBT) {
            const uint32_t v = v0 + t;
            const unsigned long long fm = (v < n && (d.flags[v] & 2)) ? 1ull : 0ull;
            const unsigned long long pos = block_exclusive_scan<kBT, unsigned long long>(fm, tot, s_scan);
            if (fm) d.minima[mbase + pos] = v;
            mbase += tot;
        }
        const uint64_t m = mbase;
        // ---- in-CSR of the in-edges, sources in ascending rank (the order of
        // the in-edge sums), so the power iteration needs no digit decoding
        unsigned long long ebase = 0;
        for (uint32_t v0 = 0; v0 < n; v0 += kBT) {
            const uint32_t v = v0 + t;
            const unsigned long long c = v < n ? __popcll(d.inm[v]) : 0ull;
            const unsigned long long pos = block_exclusive_scan<kBT, unsigned long long>(c, tot, s_scan);
            if (v < n) d.inoff[v] = static_cast<uint32_t>(ebase + pos);
            ebase += tot;
        }
        if (t == 0) d.inoff[n] = static_cast<uint32_t>(ebase);
        for (uint32_t v = t; v < n; v += kBT) {
            digits_of(d, v, x);
            const unsigned long long inm = d.inm[v];
            uint32_t* out = d.src + d.inoff[v];
            walk_neighbours(d, P.kind, v, x, [&](int k, uint32_t u) {
                if ((inm >> k) & 1ull) *out++ = u;
            });
        }
        __syncthreads();
        // ---- PageRank (landscape.hpp:47-52)
        const double nd = static_cast<double>(n);
        const double inv_n = __ddiv_rn(1.0, nd);
        const double teleport = __ddiv_rn(__dsub_rn(1.0, P.damping), nd);
        double dl = 0.0;
        for (uint32_t v = t; v < n; v += kBT) {
            d.r0[v] = inv_n;
            const uint32_t dg = d.deg[v];
            d.c[v] = dg ? __ddiv_rn(inv_n, static_cast<double>(dg)) : inv_n;
            if (!dg) dl = __dadd_rn(dl, inv_n);
        }
        double D = block_sum<kBT>(dl, s_red);
        double* r = d.r0;
        double* rn = d.r1;
        long long it = 0;
        double res = 0.0, sum = 0.0;
        int status = TK_ENOCONV;
        while (it < P.max_iter) {
            const double dn = __ddiv_rn(D, nd);
            double lres = 0.0, ldang = 0.0, lsum = 0.0;
            for (uint32_t v = t; v < n; v += kBT) {
                double acc = 0.0;
                uint32_t e = d.inoff[v];
                const uint32_t e1 = d.inoff[v + 1];
                // four in-edges at a time: the gathers issue together, the adds
                // stay in ascending source order
                for (; e + 4 <= e1; e += 4) {
                    const uint4 s4 = make_uint4(d.src[e], d.src[e + 1], d.src[e + 2], d.src[e + 3]);
                    const double c0 = __ldcg(d.c + s4.x), c1 = __ldcg(d.c + s4.y);
                    const double c2 = __ldcg(d.c + s4.z), c3 = __ldcg(d.c + s4.w);
                    acc = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(acc, c0), c1), c2), c3);
                }
                for (; e < e1; ++e) acc = __dadd_rn(acc, __ldcg(d.c + d.src[e]));
                const double xr = __dadd_rn(teleport, __dmul_rn(P.damping, __dadd_rn(acc, dn)));
                rn[v] = xr;
                lres = __dadd_rn(lres, fabs(__dsub_rn(xr, r[v])));
                if (!d.deg[v]) ldang = __dadd_rn(ldang, xr);
                lsum = __dadd_rn(lsum, xr);
            }
            res = block_sum<kBT>(lres, s_red);  // (its barriers order the rn stores too)
            D = block_sum<kBT>(ldang, s_red);
            sum = block_sum<kBT>(lsum, s_red);
            for (uint32_t v = t; v < n; v += kBT) {
                const uint32_t dg = d.deg[v];
                const double xr = rn[v];
                __stcg(d.c + v, dg ? __ddiv_rn(xr, static_cast<double>(dg)) : xr);
            }
            __syncthreads();
            double* tmp = r;
            r = rn;
            rn = tmp;
            ++it;
            if (res < P.tol) {
                status = TK_OK;
                break;
            }
        }
        if (t == 0) {
            o->iterations = it;
            o->residual = res;
            o->pagerank_sum = sum;
            o->n_minima = m;
        }
        if (status != TK_OK) {
            if (t == 0) o->status = status;
            continue;
        }
        // ---- C_p curve (landscape.hpp:54-58) and the report rows (MinimumInfo)
        if (m == 0) {
            if (t == 0) o->status = TK_EDEGEN;
            continue;
        }
        double den_l = 0.0;
        for (uint64_t i = t; i < m; i += kBT) den_l = __dadd_rn(den_l, r[d.minima[i]]);
        const double den = block_sum<kBT>(den_l, s_red);
        for (int p = 0; p < P.n_p; ++p) {
            double num_l = 0.0;
            for (uint64_t i = t; i < m; i += kBT) {
                const uint32_t u = d.minima[i];
                const double f = d.fit[u];
                if (P.zero[p] ? (f <= f_opt) : (f < __dmul_rn(P.onep[p], f_opt)))
                    num_l = __dadd_rn(num_l, r[u]);
            }
            const double num = block_sum<kBT>(num_l, s_red);
            if (t == 0) o->c_p[p] = __ddiv_rn(num, den);
        }
        if (d.rows) {
            __shared__ unsigned long long s_rb;
            if (t == 0) s_rb = atomicAdd(d.row_cursor, static_cast<unsigned long long>(m));
            __syncthreads();
            const unsigned long long rb = s_rb;
            if (t == 0) o->row_base = rb;
            for (uint64_t i = t; i < m; i += kBT) {
                const uint32_t u = d.minima[i];
                double* row = d.rows + (rb + i) * 4;
                row[0] = __longlong_as_double(static_cast<long long>(u));
                row[1] = d.fit[u];
                row[2] = __ddiv_rn(f_opt, d.fit[u]);
                row[3] = r[u];
            }
        }
        if (t == 0) o->status = den > 0.0 ? TK_OK : TK_EDEGEN;
        __syncthreads();
    }
}


// ---------------------------------------------------------------------------
// Groups of CTAs per space.  One CTA per space leaves the largest spaces of a
// batch (C4: 82,944 configurations) on one SM each, and they set the batch's
// length.  A job is (space, member r of g): the g CTAs of a space split its
// ranks into contiguous slices and meet at a group barrier (a counter and a
// generation word in global memory) between phases; their partial sums are
// combined in member order, so the result is deterministic.  The launch is
// cooperative (every CTA resident) and the host deals the jobs into waves
// of at most one job per CTA, a space's members in one wave -- a CTA only
// ever waits for members of its current job, which are in the same or an
// earlier wave of their own CTAs, so the barriers cannot deadlock.
constexpr int kGroupMax = 16;
constexpr int kPartW = 24;  // doubles per member partial (C_p needs n_p + 1 <= 17 + slack)

__device__ __forceinline__ void group_sync(unsigned int* bar, int g) {
    __syncthreads();
    if (g > 1 && threadIdx.x == 0) {
        __threadfence();
        volatile unsigned int* vb = bar;
        const unsigned int gen = vb[1];
        if (atomicAdd(bar, 1u) == static_cast<unsigned int>(g - 1)) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (vb[1] == gen) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

struct BatchJob {
    int item;    // -1: idle in this wave
    int member;
    int g;
};

__global__ void __launch_bounds__(kBT) batch_group_kernel(const BatchDesc* __restrict__ descs,
                                                          const BatchJob* __restrict__ jobs,
                                                          int waves, BatchParams P) {
    __shared__ double s_red[kBT / 32];
    __shared__ unsigned long long s_scan[kBT / 32];
    __shared__ double s_bf[kBT / 32];
    __shared__ unsigned long long s_br[kBT / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    for (int w = 0; w < waves; ++w) {
        const BatchJob job = jobs[static_cast<size_t>(w) * gridDim.x + blockIdx.x];
        if (job.item < 0) continue;
        const BatchDesc& d = descs[job.item];
        const int g = job.g, me = job.member;
        BatchOut* o = d.out;
        const uint32_t n = d.n;
        const uint32_t chunk = (n + g - 1) / g;
        const uint32_t lo = min(n, static_cast<uint32_t>(me) * chunk), hi = min(n, lo + chunk);
        double* mypart = d.part + static_cast<size_t>(me) * kPartW;
        uint32_t x[kMaxDims];
        // ---- FFG masks, flags, counts and f_opt over this member's slice
        unsigned long long e_loc = 0, m_loc = 0, in_loc = 0;
        double best_f = 0.0;
        unsigned long long best_r = ~0ull;
        for (uint32_t v = lo + t; v < hi; v += kBT) {
            digits_of(d, v, x);
            const double fv = d.fit[v];
            const bool okv = d.ok[v] != 0;
            unsigned long long inm = 0;
            uint32_t deg = 0;
            bool allgt = true;
            walk_neighbours(d, P.kind, v, x, [&](int k, uint32_t u) {
                const double fu = d.fit[u];
                if (fu < fv) ++deg;
                if (fu > fv)
                    inm |= 1ull << k;
                else
                    allgt = false;
            });
            d.inm[v] = inm;
            d.deg[v] = static_cast<uint8_t>(deg);
            const bool sink = deg == 0, okmin = sink && okv, strict = okv && allgt;
            d.flags[v] = static_cast<uint8_t>((sink ? 1 : 0) | (okmin ? 2 : 0) | (strict ? 4 : 0) |
                                              (okv ? 8 : 0));
            e_loc += deg;
            m_loc += okmin;
            in_loc += __popcll(inm);
            if (okv && (best_r == ~0ull || fv < best_f)) {
                best_f = fv;
                best_r = v;
            }
        }
#pragma unroll
        for (int sh = 16; sh; sh >>= 1) {
            const double of = __shfl_xor_sync(0xffffffffu, best_f, sh);
            const unsigned long long orr = __shfl_xor_sync(0xffffffffu, best_r, sh);
            if (orr != ~0ull && (best_r == ~0ull || of < best_f || (of == best_f && orr < best_r))) {
                best_f = of;
                best_r = orr;
            }
        }
        if (lane == 0) {
            s_bf[warp] = best_f;
            s_br[warp] = best_r;
        }
        unsigned long long tot;
        block_exclusive_scan<kBT, unsigned long long>(e_loc, tot, s_scan);
        const unsigned long long e_cta = tot;
        block_exclusive_scan<kBT, unsigned long long>(m_loc, tot, s_scan);
        const unsigned long long m_cta = tot;
        block_exclusive_scan<kBT, unsigned long long>(in_loc, tot, s_scan);
        const unsigned long long in_cta = tot;
        if (t == 0) {
            double bf = 0.0;
            unsigned long long br = ~0ull;
            for (int q = 0; q < kBT / 32; ++q) {
                const double of = s_bf[q];
                const unsigned long long orr = s_br[q];
                if (orr != ~0ull && (br == ~0ull || of < bf || (of == bf && orr < br))) {
                    bf = of;
                    br = orr;
                }
            }
            mypart[0] = __longlong_as_double(static_cast<long long>(e_cta));
            mypart[1] = __longlong_as_double(static_cast<long long>(m_cta));
            mypart[2] = __longlong_as_double(static_cast<long long>(in_cta));
            mypart[3] = bf;
            mypart[4] = __longlong_as_double(static_cast<long long>(br));
        }
        group_sync(d.bar, g);
        // combine the members' partials in member order (slices ascend)
        unsigned long long n_edges = 0, mbase = 0, ebase = 0, m_all = 0, e_in_all = 0;
        double f_opt = 0.0;
        unsigned long long opt_r = ~0ull;
        for (int q = 0; q < g; ++q) {
            const double* pq = d.part + static_cast<size_t>(q) * kPartW;
            const unsigned long long eq = static_cast<unsigned long long>(__double_as_longlong(__ldcg(pq + 0)));
            const unsigned long long mq = static_cast<unsigned long long>(__double_as_longlong(__ldcg(pq + 1)));
            const unsigned long long iq = static_cast<unsigned long long>(__double_as_longlong(__ldcg(pq + 2)));
            const double bf = __ldcg(pq + 3);
            const unsigned long long br = static_cast<unsigned long long>(__double_as_longlong(__ldcg(pq + 4)));
            if (q < me) {
                mbase += mq;
                ebase += iq;
            }
            n_edges += eq;
            m_all += mq;
            e_in_all += iq;
            if (br != ~0ull && (opt_r == ~0ull || bf < f_opt)) {
                f_opt = bf;
                opt_r = br;
            }
        }
        group_sync(d.bar, g);  // partials read: they are reused below
        if (me == 0 && t == 0) {
            o->n_edges = n_edges;
            o->n_nodes = n;
            o->f_opt = f_opt;
            o->opt_rank = opt_r;
            o->iterations = 0;
            o->residual = 0.0;
            o->n_minima = m_all;
        }
        if (opt_r == ~0ull) {  // NoFeasiblePoint (errors.hpp:32-35)
            if (me == 0 && t == 0) o->status = TK_ENOFEAS;
            continue;
        }
        // report-row base in the packed region (read by every member after the
        // group barriers below)
        if (me == 0 && t == 0 && d.rows)
            o->row_base = atomicAdd(d.row_cursor, static_cast<unsigned long long>(m_all));
        // ---- this slice's minima and in-CSR rows at their group offsets
        for (uint32_t v0 = lo; v0 < hi; v0 += kBT) {
            const uint32_t v = v0 + t;
            const unsigned long long fm = (v < hi && (d.flags[v] & 2)) ? 1ull : 0ull;
            const unsigned long long pos = block_exclusive_scan<kBT, unsigned long long>(fm, tot, s_scan);
            if (fm) d.minima[mbase + pos] = v;
            mbase += tot;
            const unsigned long long c = v < hi ? __popcll(d.inm[v]) : 0ull;
            const unsigned long long cpos = block_exclusive_scan<kBT, unsigned long long>(c, tot, s_scan);
            if (v < hi) d.inoff[v] = static_cast<uint32_t>(ebase + cpos);
            ebase += tot;
        }
        if (me == g - 1 && t == 0) d.inoff[n] = static_cast<uint32_t>(e_in_all);
        __syncthreads();
        for (uint32_t v = lo + t; v < hi; v += kBT) {
            digits_of(d, v, x);
            const unsigned long long inm = d.inm[v];
            uint32_t* out = d.src + d.inoff[v];
            walk_neighbours(d, P.kind, v, x, [&](int k, uint32_t u) {
                if ((inm >> k) & 1ull) *out++ = u;
            });
        }
        // ---- PageRank (landscape.hpp:47-52)
        const double nd = static_cast<double>(n);
        const double inv_n = __ddiv_rn(1.0, nd);
        const double teleport = __ddiv_rn(__dsub_rn(1.0, P.damping), nd);
        double dl = 0.0;
        for (uint32_t v = lo + t; v < hi; v += kBT) {
            d.r0[v] = inv_n;
            const uint32_t dg = d.deg[v];
            __stcg(d.c + v, dg ? __ddiv_rn(inv_n, static_cast<double>(dg)) : inv_n);
            if (!dg) dl = __dadd_rn(dl, inv_n);
        }
        dl = block_sum<kBT>(dl, s_red);
        if (t == 0) mypart[0] = dl;
        group_sync(d.bar, g);
        double D = 0.0;
        for (int q = 0; q < g; ++q) D = __dadd_rn(D, __ldcg(d.part + static_cast<size_t>(q) * kPartW));
        group_sync(d.bar, g);
        double* r = d.r0;
        double* rn = d.r1;
        long long it = 0;
        double res = 0.0, sum = 0.0;
        int status = TK_ENOCONV;
        while (it < P.max_iter) {
            const double dn = __ddiv_rn(D, nd);
            double lres = 0.0, ldang = 0.0, lsum = 0.0;
            for (uint32_t v = lo + t; v < hi; v += kBT) {
                double acc = 0.0;
                uint32_t e = d.inoff[v];
                const uint32_t e1 = d.inoff[v + 1];
                for (; e + 4 <= e1; e += 4) {
                    const uint4 s4 = make_uint4(d.src[e], d.src[e + 1], d.src[e + 2], d.src[e + 3]);
                    const double c0 = __ldcg(d.c + s4.x), c1 = __ldcg(d.c + s4.y);
                    const double c2 = __ldcg(d.c + s4.z), c3 = __ldcg(d.c + s4.w);
                    acc = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(acc, c0), c1), c2), c3);
                }
                for (; e < e1; ++e) acc = __dadd_rn(acc, __ldcg(d.c + d.src[e]));
                const double xr = __dadd_rn(teleport, __dmul_rn(P.damping, __dadd_rn(acc, dn)));
                rn[v] = xr;
                lres = __dadd_rn(lres, fabs(__dsub_rn(xr, r[v])));
                if (!d.deg[v]) ldang = __dadd_rn(ldang, xr);
                lsum = __dadd_rn(lsum, xr);
            }
            lres = block_sum<kBT>(lres, s_red);
            ldang = block_sum<kBT>(ldang, s_red);
            lsum = block_sum<kBT>(lsum, s_red);
            if (t == 0) {
                mypart[0] = lres;
                mypart[1] = ldang;
                mypart[2] = lsum;
            }
            group_sync(d.bar, g);  // every member's pull done: the c update may start
            res = 0.0;
            D = 0.0;
            sum = 0.0;
            for (int q = 0; q < g; ++q) {
                const double* pq = d.part + static_cast<size_t>(q) * kPartW;
                res = __dadd_rn(res, __ldcg(pq + 0));
                D = __dadd_rn(D, __ldcg(pq + 1));
                sum = __dadd_rn(sum, __ldcg(pq + 2));
            }
            for (uint32_t v = lo + t; v < hi; v += kBT) {
                const uint32_t dg = d.deg[v];
                const double xr = rn[v];
                __stcg(d.c + v, dg ? __ddiv_rn(xr, static_cast<double>(dg)) : xr);
            }
            group_sync(d.bar, g);  // c complete and the partials read before reuse
            double* tmp = r;
            r = rn;
            rn = tmp;
            ++it;
            if (res < P.tol) {
                status = TK_OK;
                break;
            }
        }
        if (me == 0 && t == 0) {
            o->iterations = it;
            o->residual = res;
            o->pagerank_sum = sum;
        }
        if (status != TK_OK) {
            if (me == 0 && t == 0) o->status = status;
            continue;
        }
        // ---- C_p curve (landscape.hpp:54-58) and the report rows (MinimumInfo)
        const uint64_t m = m_all;
        if (m == 0) {
            if (me == 0 && t == 0) o->status = TK_EDEGEN;
            continue;
        }
        const uint64_t mch = (m + g - 1) / g;
        const uint64_t mlo0 = static_cast<uint64_t>(me) * mch;
        const uint64_t mlo = mlo0 < m ? mlo0 : m;
        const uint64_t mhi = mlo + mch < m ? mlo + mch : m;
        double den_l = 0.0;
        for (uint64_t i = mlo + t; i < mhi; i += kBT) den_l = __dadd_rn(den_l, __ldcg(r + d.minima[i]));
        den_l = block_sum<kBT>(den_l, s_red);
        if (t == 0) mypart[P.n_p] = den_l;
        for (int p = 0; p < P.n_p; ++p) {
            double num_l = 0.0;
            for (uint64_t i = mlo + t; i < mhi; i += kBT) {
                const uint32_t u = d.minima[i];
                const double f = d.fit[u];
                if (P.zero[p] ? (f <= f_opt) : (f < __dmul_rn(P.onep[p], f_opt)))
                    num_l = __dadd_rn(num_l, __ldcg(r + u));
            }
            num_l = block_sum<kBT>(num_l, s_red);
            if (t == 0) mypart[p] = num_l;
        }
        if (d.rows) {
            const unsigned long long rb =
                *reinterpret_cast<volatile unsigned long long*>(&o->row_base);
            for (uint64_t i = mlo + t; i < mhi; i += kBT) {
                const uint32_t u = d.minima[i];
                double* row = d.rows + (rb + i) * 4;
                row[0] = __longlong_as_double(static_cast<long long>(u));
                row[1] = d.fit[u];
                row[2] = __ddiv_rn(f_opt, d.fit[u]);
                row[3] = __ldcg(r + u);
            }
        }
        group_sync(d.bar, g);
        if (me == 0 && t < P.n_p + 1) {
            double acc = 0.0;
            for (int q = 0; q < g; ++q) acc = __dadd_rn(acc, __ldcg(d.part + static_cast<size_t>(q) * kPartW + t));
            s_red[t] = acc;
        }
        __syncthreads();
        if (me == 0 && t == 0) {
            const double den = s_red[P.n_p];
            for (int p = 0; p < P.n_p; ++p) o->c_p[p] = __ddiv_rn(s_red[p], den);
            o->status = den > 0.0 ? TK_OK : TK_EDEGEN;
        }
        group_sync(d.bar, g);  // partials read before the next job of these CTAs reuses them
    }
}

}  // namespace

bool batch_item_supported(uint32_t dims, const uint32_t* radix, int kind, uint64_t* n_out) {
    uint64_t n = 1;
    int slots = 0, d = 0;
    for (uint32_t i = 0; i < dims; ++i) {
        if (radix[i] < 1) return false;
        n *= radix[i];
        if (radix[i] >= 2) {
            ++d;
            slots += kind == TK_ADJACENT ? 2 : static_cast<int>(radix[i]) - 1;
        }
    }
    if (n_out) *n_out = n;
    return n >= 1 && n <= kBatchMaxNodes && d <= kMaxDims && slots <= 64;
}

cudaError_t launch_batch_analyze(const void* descs_dev, uint32_t n_items, const BatchParams& P,
                                 int num_sms, cudaStream_t stream) {
    const uint32_t grid = std::min<uint32_t>(n_items, static_cast<uint32_t>(num_sms) * 4);
    batch_analyze_kernel<<<grid ? grid : 1, kBT, 0, stream>>>(
        static_cast<const BatchDesc*>(descs_dev), n_items, P);
    return cudaGetLastError();
}

size_t batch_desc_bytes() { return sizeof(BatchDesc); }

int batch_group_max() { return kGroupMax; }
size_t batch_group_state_bytes() { return 64 + 8ull * kGroupMax * kPartW; }
int batch_group_max_np() { return kPartW - 1; }
size_t batch_job_bytes() { return sizeof(BatchJob); }

// jobs: waves x grid entries (item, member, g); grid must be resident (cooperative)
cudaError_t launch_batch_group(const void* descs_dev, const void* jobs_dev, int waves, int grid,
                               const BatchParams& P, cudaStream_t stream) {
    const BatchDesc* dd = static_cast<const BatchDesc*>(descs_dev);
    const BatchJob* jj = static_cast<const BatchJob*>(jobs_dev);
    BatchParams pc = P;
    void* args[] = {&dd, &jj, &waves, &pc};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(batch_group_kernel), dim3(grid),
                                       dim3(kBT), args, 0, stream);
}

int batch_group_resident(int num_sms) {
    int bps = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, batch_group_kernel, kBT, 0) !=
        cudaSuccess)
        return 0;
    return bps * num_sms;
}

void batch_set_job(void* jobs_host, size_t idx, int item, int member, int g) {
    static_cast<BatchJob*>(jobs_host)[idx] = BatchJob{item, member, g};
}

// Host-side description of one space in the device workspace.
void batch_fill_desc(void* desc_host, const double* fit, const uint8_t* ok, uint32_t n,
                     uint32_t slots, uint32_t dims_in, const uint32_t* radix_in, uint8_t* ws,
                     unsigned int* bar, double* part, BatchOut* out, double* rows,
                     unsigned long long* row_cursor) {
    BatchDesc d{};
    d.fit = fit;
    d.ok = ok;
    d.n = n;
    // dims with a single value carry no neighbours (DevShape convention)
    uint32_t st = 1;
    std::vector<uint32_t> r, s;
    for (int i = static_cast<int>(dims_in) - 1; i >= 0; --i) {
        if (radix_in[i] >= 2) {
            r.push_back(radix_in[i]);
            s.push_back(st);
        }
        st *= radix_in[i];
    }
    d.dims = static_cast<int>(r.size());
    for (int i = 0; i < d.dims; ++i) {  // reverse: dim 0 most significant
        d.radix[i] = r[d.dims - 1 - i];
        d.stride[i] = s[d.dims - 1 - i];
    }
    auto carve = [&](size_t bytes) {
        uint8_t* p = ws;
        ws += (bytes + 255) & ~static_cast<size_t>(255);
        return p;
    };
    d.inm = reinterpret_cast<unsigned long long*>(carve(8ull * n));
    d.r0 = reinterpret_cast<double*>(carve(8ull * n));
    d.r1 = reinterpret_cast<double*>(carve(8ull * n));
    d.c = reinterpret_cast<double*>(carve(8ull * n));
    d.minima = reinterpret_cast<uint32_t*>(carve(4ull * n));
    d.inoff = reinterpret_cast<uint32_t*>(carve(4ull * (n + 1)));
    d.src = reinterpret_cast<uint32_t*>(carve(4ull * n * slots));
    d.deg = carve(n);
    d.flags = carve(n);
    d.bar = bar;
    d.part = part;
    d.out = out;
    d.rows = rows;
    d.row_cursor = row_cursor;
    std::memcpy(desc_host, &d, sizeof(d));
}

size_t batch_workspace_bytes(uint32_t n, uint32_t slots) {
    auto a = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
    return 4 * a(8ull * n) + a(4ull * n) + a(4ull * (n + 1)) + a(4ull * n * slots) + 2 * a(n);
}

uint32_t batch_slots(uint32_t dims, const uint32_t* radix, int kind) {
    uint32_t s = 0;
    for (uint32_t i = 0; i < dims; ++i)
        if (radix[i] >= 2) s += kind == TK_ADJACENT ? 2 : radix[i] - 1;
    return s;
}

}  // namespace tk
