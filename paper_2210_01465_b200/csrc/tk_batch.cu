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
    // outputs
    BatchOut* out;
    unsigned long long* rep_rank;
    double* rep_fit;
    double* rep_frac;
    double* rep_pr;
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
        if (d.rep_rank) {
            for (uint64_t i = t; i < m; i += kBT) {
                const uint32_t u = d.minima[i];
                d.rep_rank[i] = u;
                d.rep_fit[i] = d.fit[u];
                d.rep_frac[i] = __ddiv_rn(f_opt, d.fit[u]);
                d.rep_pr[i] = r[u];
            }
        }
        if (t == 0) o->status = den > 0.0 ? TK_OK : TK_EDEGEN;
        __syncthreads();
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

// Host-side description of one space in the device workspace.
void batch_fill_desc(void* desc_host, const double* fit, const uint8_t* ok, uint32_t n,
                     uint32_t slots, uint32_t dims_in, const uint32_t* radix_in, uint8_t* ws,
                     BatchOut* out,
                     unsigned long long* rep_rank, double* rep_fit, double* rep_frac,
                     double* rep_pr) {
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
    d.out = out;
    d.rep_rank = rep_rank;
    d.rep_fit = rep_fit;
    d.rep_frac = rep_frac;
    d.rep_pr = rep_pr;
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
