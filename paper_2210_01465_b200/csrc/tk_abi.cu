// tk_abi.cu -- the extern "C" boundary declared in include/tk_landscape.h.
//
// Host orchestration only: argument checks with the reference's error
// classes (errors.hpp:10-44 mapped onto tk_status), device buffer ownership,
// stream ordering, and the few D2H reads the API returns.  All computation is
// in tk_kernels.cu; there is no host fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "tk_kernels.cuh"

namespace {

thread_local std::string g_err;

int fail(int st, const std::string& msg) {
    g_err = msg;
    return st;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(e == cudaErrorMemoryAllocation ? TK_ENOMEM : TK_ECUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

#define TKC(expr)                                              \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr);    \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

cudaError_t ensure(DevBuf& b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.p && b.cap >= bytes) return cudaSuccess;
    b.release();
    cudaError_t e = cudaMalloc(&b.p, bytes);
    if (e == cudaSuccess) b.cap = bytes;
    else b.p = nullptr;
    return e;
}

constexpr uint64_t kMaxNodes = 0xFFF00000ull;  // u32 ids with grid-stride headroom
// per-rank arrays are padded so tile-granular bulk copies may round the last
// tile up to 16 elements (tk_staged.cu)
constexpr uint64_t kPad = 16;

// TK_KERNELS=v1 selects the per-lane-gather kernels instead of the TMA-staged
// ones (A/B comparisons and parity tests of both paths).
bool staged_enabled() {
    const char* e = std::getenv("TK_KERNELS");
    return !(e && std::string(e) == "v1");
}

struct PrOut {
    long long iter;
    double res;
    double sum;
    int parity;
    int status;
};

struct Small {  // device-side scalars read back by the host
    unsigned long long totals[4];
    double f_opt;
    unsigned long long rank;
    int has;
    int err;
    int degenerate;
    int pad;
    PrOut pr;
    double totals_f[3];  // shard PageRank partials (residual, dangling, sum)
};

}  // namespace

struct tk_land {
    int device = 0;
    int num_sms = 148;
    int smem_optin = 0;  // max dynamic shared memory per block
    int smem_per_sm = 0;
    cudaStream_t stream = nullptr;
    std::vector<uint32_t> radix_in;
    std::vector<unsigned long long> strides_in;
    uint64_t n = 0;

    DevBuf fit, ok;
    bool loaded = false;
    bool fit_clean = false;  // every fitness finite and none -0 (FFG count fast compares)
    DevBuf hkeys, hvals, staging_keys, staging_vals, staging_cfg, claimed;
    uint64_t hcap = 0;  // 0 = no valid-set hash table for the loaded table yet

    bool built = false, emitted = false;
    int kind = TK_ADJACENT, mode = 0;
    bool wide = false;
    tk::DevShape shape{};
    DevBuf pw, inm, odeg, flags, offsets, targets, minima, e_status, m_status, counter;
    DevBuf om, tile_cnt, tile_base;  // staged two-pass build
    uint64_t n_edges = 0, n_minima = 0, n_strict = 0, n_ok = 0;

    DevBuf r0, r1, c0, c1, part;
    bool pr_done = false;
    int pr_parity = 0;
    long long iterations = 0;
    double residual = 0.0, pr_sum = 0.0;

    DevBuf small, opt_part, cp_part, cp_out, tmp;
    Small* hsmall = nullptr;  // pinned mirror
    cudaEvent_t ev[6] = {};
    float ms_build = 0.f, ms_pr = 0.f;  // kernel-only device time of the last launch
    bool staged = false;                // last build used the TMA-staged kernel
    int pr_staged = 0;  // last PageRank kernel: 0 per-lane, 1 staged, 2 row-tiled,
                        // 3 Hamming staged, 4 Hamming tiled
    int pr_grid = 0;
    bool opt_ready = false;  // small->f_opt/rank/has hold f_opt of the loaded table

    // key-range sharding (tk_land_set_shard)
    bool sharded = false;
    int shard_rank = 0, shard_n = 1;
    uint64_t shard_lo = 0, shard_hi = 0, shard_chunk = 0;
    void* peer_c0[tk::kMaxShards] = {};
    void* peer_c1[tk::kMaxShards] = {};
    std::vector<void*> ipc_opened;
    int shard_cur = 0;          // parity holding the current iterate
    bool shard_pr = false;      // tk_shard_pagerank_init done
    bool shard_r_fresh = false; // r0 holds the rank vector of the current iterate
};

namespace {

cudaError_t set_dev(const tk_land* l) { return cudaSetDevice(l->device); }

// Shared memory the staged pipeline may use per block: TK_CTAS_PER_SM blocks
// share an SM (1 by default; the 256-rank-tile build variant uses 2).
#ifndef TK_CTAS_PER_SM
#define TK_CTAS_PER_SM 1
#endif
int stage_budget(const tk_land* l) {
    // per CTA: 1 KB driver reservation + static shared memory + margin
    const int per = l->smem_per_sm / TK_CTAS_PER_SM - 3072;
    return std::min(l->smem_optin - 2048, per);
}

int check_land(const tk_land* l) {
    if (!l) return fail(TK_EINVAL, "null tk_land handle");
    return TK_OK;
}

tk::DevShape make_shape(const tk_land* l, int kind) {
    tk::DevShape s{};
    s.n = static_cast<uint32_t>(l->n);
    s.kind = kind;
    int d = 0;
    for (size_t i = 0; i < l->radix_in.size(); ++i) {
        if (l->radix_in[i] < 2) continue;  // single-value dims add no neighbours
        s.radix[d] = l->radix_in[i];
        s.stride[d] = static_cast<uint32_t>(l->strides_in[i]);
        ++d;
    }
    s.dims = d;
    int slots = 0;
    for (int i = 0; i < d; ++i) {
        s.magic[i] = s.stride[i] == 1 ? 0ull : (~0ull / s.stride[i] + 1ull);
        s.base[i] = slots;
        slots += kind == TK_HAMMING ? static_cast<int>(s.radix[i]) - 1 : 2;
    }
    s.slots = slots;
    if (kind == TK_ADJACENT) {
        // ordered in-slots: v - s_0 < v - s_1 < ... < v - s_{D-1} < v + s_{D-1} < ... < v + s_0
        for (int j = 0; j < d; ++j) s.nbo[j] = 0u - s.stride[j];
        for (int j = d; j < 2 * d; ++j) s.nbo[j] = s.stride[2 * d - 1 - j];
    }
    return s;
}

// Undirected neighbour pairs: the edge count when fitness is tie-free and
// no two failed nodes meet; an upper bound on E always.
uint64_t max_edges(const tk::DevShape& s) {
    uint64_t e = 0;
    for (int i = 0; i < s.dims; ++i) {
        const uint64_t m = s.radix[i];
        if (s.kind == TK_HAMMING) e += static_cast<uint64_t>(s.n) / m * (m * (m - 1) / 2);
        else e += static_cast<uint64_t>(s.n) / m * (m - 1);
    }
    return e;
}

int do_build(tk_land* l, int kind, uint64_t node_limit, int emit) {
    if (!l->loaded) return fail(TK_ESTATE, "build_ffg: no fitness table loaded");
    if (kind != TK_HAMMING && kind != TK_ADJACENT)
        return fail(TK_EINVAL, "build_ffg: unknown neighbourhood kind");
    if (l->n > node_limit) {
        char buf[256];
        std::snprintf(buf, sizeof buf,
                      "search space has %llu configurations, above the FFG node limit of %llu; "
                      "sample the space or raise node_limit",
                      static_cast<unsigned long long>(l->n),
                      static_cast<unsigned long long>(node_limit));
        return fail(TK_ELIMIT, buf);
    }
    tk::DevShape s = make_shape(l, kind);
    if (s.slots > tk::kMaxSlots)
        return fail(TK_EINVAL, "neighbourhood has " + std::to_string(s.slots) +
                                   " slots per node; at most 64 are supported");
    int mode;
    bool wide = s.slots > 32;
    if (kind == TK_ADJACENT) mode = s.slots <= tk::kPackedSlots ? tk::MODE_ADJ_PACKED : tk::MODE_ADJ_ORDERED;
    else mode = tk::MODE_HAM;

    const uint64_t n = l->n;
    const uint32_t ntiles = static_cast<uint32_t>((n + tk::kBuildThreads - 1) / tk::kBuildThreads);
    TKC(set_dev(l));
    if (mode == tk::MODE_ADJ_PACKED) {
        TKC(ensure(l->pw, (n + kPad) * 4));
    } else {
        TKC(ensure(l->inm, n * (wide ? 8 : 4)));
        TKC(ensure(l->odeg, n));
    }
    TKC(ensure(l->flags, n));
    TKC(ensure(l->minima, n * 4));
    TKC(ensure(l->e_status, static_cast<size_t>(ntiles) * 8));
    TKC(ensure(l->m_status, static_cast<size_t>(ntiles) * 8));
    TKC(ensure(l->counter, 16));
    if (emit) {
        TKC(ensure(l->offsets, (n + 1) * 8));
        TKC(ensure(l->targets, std::max<uint64_t>(1, max_edges(s)) * 4));
    }
    Small* ds = l->small.as<Small>();
    TKC(cudaMemsetAsync(l->e_status.p, 0, static_cast<size_t>(ntiles) * 8, l->stream));
    TKC(cudaMemsetAsync(l->m_status.p, 0, static_cast<size_t>(ntiles) * 8, l->stream));
    TKC(cudaMemsetAsync(l->counter.p, 0, 16, l->stream));
    TKC(cudaMemsetAsync(ds->totals, 0, sizeof(ds->totals), l->stream));

    tk::BuildArgs a{};
    a.fit = l->fit.as<double>();
    a.ok = l->ok.as<uint8_t>();
    a.inm = l->inm.p;
    a.odeg = l->odeg.as<uint8_t>();
    a.pw = l->pw.as<uint32_t>();
    a.flags = l->flags.as<uint8_t>();
    a.offsets = emit ? l->offsets.as<unsigned long long>() : nullptr;
    a.targets = emit ? l->targets.as<uint32_t>() : nullptr;
    a.minima = l->minima.as<uint32_t>();
    a.e_status = l->e_status.as<unsigned long long>();
    a.m_status = l->m_status.as<unsigned long long>();
    a.tile_counter = l->counter.as<unsigned int>();
    a.totals = ds->totals;
    a.ntiles = ntiles;
    TKC(cudaEventRecord(l->ev[0], l->stream));
    tk::StagePlan plan{};
    // one-pass build (count + warp-slot look-back + CSR emission), opt-in with
    // TK_FFG_FUSED=1: correct, but the look-back over the warp slots of the
    // tiles in flight (~2,400 slots) serialises it: 15 ms vs 3.4 ms for the
    // count / scan / fill kernels on C5 (profiles/r01_ab_log.md, round 2)
    const bool fused = emit && !l->sharded && mode == tk::MODE_ADJ_PACKED && staged_enabled() &&
                       std::getenv("TK_FFG_FUSED") &&
                       tk::make_stage_plan(s, false,
                                           stage_budget(l) - static_cast<int>(tk::fused_seg_bytes()),
                                           &plan);
    if (fused) {
        plan.fast = l->fit_clean && !std::getenv("TK_FFG_SLOW") ? 1 : 0;
        const uint32_t nt = static_cast<uint32_t>((n + plan.T - 1) / plan.T);
        a.ntiles = nt;
        a.tile_lo = 0;
        const size_t ns = static_cast<size_t>(nt) * (plan.T / 32);
        TKC(ensure(l->tile_base, (ns + 1) * 16));
        a.e_status = l->tile_base.as<unsigned long long>();
        a.m_status = a.e_status + (ns + 1);
        TKC(ensure(l->opt_part, static_cast<size_t>(l->num_sms) * 4 * 16));
        a.opt_part_f = l->opt_part.as<double>();
        a.opt_part_r = reinterpret_cast<unsigned long long*>(a.opt_part_f + l->num_sms * 4);
        a.f_opt = &ds->f_opt;
        a.opt_rank = &ds->rank;
        a.opt_has = &ds->has;
        l->opt_ready = true;
        TKC(tk::launch_ffg_build_fused(s, plan, a, l->num_sms, l->stream));
        l->staged = true;
    } else if (mode == tk::MODE_ADJ_PACKED && staged_enabled() &&
        tk::make_stage_plan(s, false, stage_budget(l), &plan)) {
        plan.fast = l->fit_clean && !std::getenv("TK_FFG_SLOW") ? 1 : 0;
        // T-rank tiles over the whole space, or over this handle's shard
        const uint64_t lo = l->sharded ? l->shard_lo : 0, hi = l->sharded ? l->shard_hi : n;
        const uint32_t nt = static_cast<uint32_t>((hi - lo + plan.T - 1) / plan.T);
        a.ntiles = nt;
        a.tile_lo = static_cast<uint32_t>(lo / plan.T);
        if (l->sharded) {
            a.offsets = nullptr;
            a.targets = nullptr;
            emit = 0;
        }
        TKC(ensure(l->om, (n + kPad) * 4));
        // per-warp-slot (32 ranks) counts and their exclusive scans
        const size_t ns = static_cast<size_t>(nt) * (plan.T / 32);
        TKC(ensure(l->tile_cnt, ns * 8 + 16));
        TKC(ensure(l->tile_base, (ns + 1) * 16));
        a.om = l->om.as<uint32_t>();
        a.tile_e = l->tile_cnt.as<uint32_t>();
        a.tile_m = a.tile_e + ns;
        a.ebase = l->tile_base.as<unsigned long long>();
        a.mbase = a.ebase + (ns + 1);
        TKC(ensure(l->opt_part, static_cast<size_t>(l->num_sms) * 4 * 16));
        a.opt_part_f = l->opt_part.as<double>();
        a.opt_part_r = reinterpret_cast<unsigned long long*>(a.opt_part_f + l->num_sms * 4);
        a.f_opt = &ds->f_opt;
        a.opt_rank = &ds->rank;
        a.opt_has = &ds->has;
        l->opt_ready = true;
        TKC(tk::launch_ffg_build_staged(s, plan, emit != 0, a, l->num_sms, l->stream));
        TKC(cudaMemcpyAsync(ds->totals + 0, a.ebase + ns, 8, cudaMemcpyDeviceToDevice, l->stream));
        TKC(cudaMemcpyAsync(ds->totals + 1, a.mbase + ns, 8, cudaMemcpyDeviceToDevice, l->stream));
        l->staged = true;
    } else {
        if (l->sharded)
            return fail(TK_EINVAL, "sharded builds need an Adjacent space with 2*dims <= 27 "
                                   "(the TMA-staged path)");
        TKC(tk::launch_ffg_build(s, mode, wide, emit != 0, a, l->num_sms, l->stream));
        l->staged = false;
    }
    TKC(cudaEventRecord(l->ev[1], l->stream));
    TKC(cudaMemcpyAsync(l->hsmall->totals, ds->totals, sizeof(ds->totals),
                        cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    l->n_edges = l->hsmall->totals[0];
    l->n_minima = l->hsmall->totals[1];
    l->n_strict = l->hsmall->totals[2];
    l->n_ok = l->hsmall->totals[3];
    TKC(cudaEventElapsedTime(&l->ms_build, l->ev[0], l->ev[1]));
    l->shape = s;
    l->kind = kind;
    l->mode = mode;
    l->wide = wide;
    l->built = true;
    l->emitted = emit != 0;
    l->pr_done = false;
    l->shard_pr = false;
    return TK_OK;
}

int do_optimum(tk_land* l, double* f_opt, uint64_t* rank) {
    if (!l->loaded) return fail(TK_ESTATE, "optimum: no fitness table loaded");
    TKC(set_dev(l));
    Small* ds = l->small.as<Small>();
    if (!l->opt_ready) {  // the staged FFG count pass already reduced it otherwise
        TKC(ensure(l->opt_part, 148 * 4 * 16));
        TKC(tk::launch_optimum(l->fit.as<double>(), l->ok.as<uint8_t>(),
                               static_cast<uint32_t>(l->n), l->opt_part.as<double>(),
                               reinterpret_cast<unsigned long long*>(l->opt_part.as<double>() + 148 * 4),
                               &ds->f_opt, &ds->rank, &ds->has, l->stream));
        l->opt_ready = true;
    }
    TKC(cudaMemcpyAsync(&l->hsmall->f_opt, &ds->f_opt, 8 + 8 + 4, cudaMemcpyDeviceToHost,
                        l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    if (!l->hsmall->has) return fail(TK_ENOFEAS, "search space has no ok entry");
    if (f_opt) *f_opt = l->hsmall->f_opt;
    if (rank) *rank = l->hsmall->rank;
    return TK_OK;
}

int check_pr_args(double d, double tol, int64_t max_iter) {
    if (!(d >= 0.0 && d <= 1.0)) return fail(TK_EINVAL, "pagerank: damping must lie in [0, 1]");
    if (!(tol > 0.0)) return fail(TK_EINVAL, "pagerank: tol must be positive");
    if (max_iter < 1) return fail(TK_EINVAL, "pagerank: max_iter must be >= 1");
    return TK_OK;
}

int nonconv(long long it, double res) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "PageRank did not converge: iterations=%lld residual=%.6e", it,
                  res);
    return fail(TK_ENOCONV, buf);
}

// Runs the persistent PageRank kernel over buffers already described by `a`.
// Cooperative (grid-synchronising) PageRank launches from different streams
// (tk.BatchAnalyzer drives several handles at once) may run concurrently only
// while their SM footprints sum to at most the device's SM count: two
// persistent cooperative grids that each hold part of the SMs the other needs
// would spin in grid.sync forever.  Per device, the in-flight cooperative
// launches are tracked as (completion event, SMs); a launch that does not fit
// makes its stream wait for the oldest ones first.  Non-cooperative kernels
// always finish, so they cannot close such a cycle.
struct CoopGate {
    std::mutex mu;
    struct Flight {
        cudaEvent_t ev;
        int sms;
    };
    std::vector<Flight> inflight[64];
    std::vector<cudaEvent_t> spare;
};
CoopGate& coop_gate() {
    static CoopGate g;
    return g;
}
template <class F>
cudaError_t gated_coop_launch(int device, int num_sms, int footprint_sms, cudaStream_t stream,
                              F&& launch) {
    CoopGate& g = coop_gate();
    std::lock_guard<std::mutex> lk(g.mu);
    auto& fl = g.inflight[device & 63];
    int used = 0;
    for (size_t i = 0; i < fl.size();) {  // drop completed launches
        if (cudaEventQuery(fl[i].ev) == cudaSuccess) {
            g.spare.push_back(fl[i].ev);
            fl.erase(fl.begin() + static_cast<long>(i));
        } else {
            used += fl[i].sms;
            ++i;
        }
    }
    (void)cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error here
    const int need = std::min(footprint_sms, num_sms);
    while (!fl.empty() && used + need > num_sms) {  // wait for the oldest
        cudaError_t e = cudaStreamWaitEvent(stream, fl.front().ev, 0);
        if (e != cudaSuccess) return e;
        used -= fl.front().sms;
        g.spare.push_back(fl.front().ev);
        fl.erase(fl.begin());
    }
    cudaError_t e = launch();
    if (e != cudaSuccess) return e;
    cudaEvent_t ev;
    if (!g.spare.empty()) {
        ev = g.spare.back();
        g.spare.pop_back();
    } else if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) {
        return e;
    }
    e = cudaEventRecord(ev, stream);
    if (e != cudaSuccess) return e;
    fl.push_back({ev, need});
    return cudaSuccess;
}

int run_pagerank(int device, int num_sms, const tk::DevShape& s, int mode, bool wide,
                 tk::PrArgs a, DevBuf& part, Small* ds, Small* hs, cudaStream_t stream,
                 double d, double tol, int64_t max_iter, cudaEvent_t e0 = nullptr,
                 cudaEvent_t e1 = nullptr, float* ms = nullptr, int* grid = nullptr,
                 const tk::StagePlan* plan = nullptr, const tk::RowPlan* rplan = nullptr,
                 int smem_budget = 0, int* kernel_used = nullptr, bool ring = false) {
    const int maxg = (plan || rplan) ? num_sms * 4 : tk::pagerank_max_grid(mode, wide, num_sms);
    if (maxg <= 0) return fail(TK_ECUDA, "pagerank: kernel cannot be made resident");
    // Hamming by dimension groups (tk_hamsplit.cu; TK_HAM_SPLIT=0: the tiled / staged kernels)
    const char* hs_env = std::getenv("TK_HAM_SPLIT");
    const bool ham_split = !plan && !rplan && !ring && mode == tk::MODE_HAM && staged_enabled() &&
                           !(hs_env && hs_env[0] == '0') && tk::ham_split_available(s);
    TKC(ensure(part, std::max(static_cast<size_t>(maxg) * 2 * 3 * 8,
                              ham_split ? tk::ham_split_workspace_bytes(s) : size_t{0})));
    const double nd = static_cast<double>(a.n);
    a.inv_n = 1.0 / nd;
    a.nd = nd;
    a.teleport = (1.0 - d) / nd;
    a.damping = d;
    a.tol = tol;
    a.max_iter = max_iter;
    a.part = part.as<double>();
    a.out_iter = &ds->pr.iter;
    a.out_res = &ds->pr.res;
    a.out_sum = &ds->pr.sum;
    a.out_parity = &ds->pr.parity;
    a.out_status = &ds->pr.status;
    int g = 0;
    if (e0) TKC(cudaEventRecord(e0, stream));
    // SM footprint: the staged kernel runs one CTA per SM on min(SMs, tiles)
    // SMs; the per-lane kernel is sized to the whole device
    const int footprint = rplan ? static_cast<int>(std::min<uint64_t>(num_sms, rplan->ncols))
                          : plan ? static_cast<int>(std::min<uint64_t>(
                                     num_sms, (static_cast<uint64_t>(a.n) + plan->T - 1) / plan->T))
                               : num_sms;
    tk::HamStagePlanOut hplan{};
    const bool ham_staged = !ham_split && !plan && !rplan && mode == tk::MODE_HAM && staged_enabled() &&
                            smem_budget > 0 && tk::ham_staged_plan(s, smem_budget, &hplan);
    const bool ham_tiled = !ham_split && !plan && !ham_staged && mode == tk::MODE_HAM && staged_enabled() &&
                           tk::ham_tiled_supported(s);
    TKC(gated_coop_launch(device, num_sms, (ham_tiled || ham_staged || ham_split || ring) ? num_sms : footprint, stream, [&] {
        if (ring) return tk::launch_pagerank_ring(s, a, smem_budget, num_sms, &g, stream);
        if (ham_split)
            return tk::launch_pagerank_ham_split(s, wide, a, a.r0, part.p, num_sms, &g, stream);
        if (rplan) return tk::launch_pagerank_rows(s, *rplan, a, num_sms, &g, stream);
        if (plan) return tk::launch_pagerank_staged(s, *plan, a, num_sms, &g, stream);
        if (ham_staged)
            return tk::launch_pagerank_ham_staged(s, wide, hplan, a, num_sms, &g, stream);
        if (ham_tiled) return tk::launch_pagerank_ham_tiled(s, wide, a, num_sms, &g, stream);
        return tk::launch_pagerank(s, mode, wide, a, num_sms, &g, stream);
    }));
    if (e1) TKC(cudaEventRecord(e1, stream));
    // 0 per-lane, 1 staged (Adjacent), 2 row-tiled, 3 Hamming staged, 4 Hamming tiled, 5 ring,
    // 6 Hamming by dimension groups
    if (kernel_used)
        *kernel_used = ring ? 5 : rplan ? 2 : plan ? 1 : ham_split ? 6 : ham_staged ? 3 : ham_tiled ? 4 : 0;
    TKC(cudaMemcpyAsync(&hs->pr, &ds->pr, sizeof(PrOut), cudaMemcpyDeviceToHost, stream));
    TKC(cudaStreamSynchronize(stream));
    if (e0 && e1 && ms) TKC(cudaEventElapsedTime(ms, e0, e1));
    if (grid) *grid = g;
    return TK_OK;
}

int do_pagerank(tk_land* l, double d, double tol, int64_t max_iter) {
    if (!l->built) return fail(TK_ESTATE, "pagerank: build the FFG first");
    int st = check_pr_args(d, tol, max_iter);
    if (st) return st;
    TKC(set_dev(l));
    const uint64_t n = l->n;
    TKC(ensure(l->r0, (n + kPad) * 8));
    TKC(ensure(l->r1, (n + kPad) * 8));
    TKC(ensure(l->c0, (n + kPad) * 8));
    TKC(ensure(l->c1, (n + kPad) * 8));
    tk::PrArgs a{};
    a.n = static_cast<uint32_t>(n);
    a.pw = l->pw.as<uint32_t>();
    a.inm = l->inm.p;
    a.odeg = l->odeg.as<uint8_t>();
    a.r0 = l->r0.as<double>();
    a.r1 = l->r1.as<double>();
    a.c0 = l->c0.as<double>();
    a.c1 = l->c1.as<double>();
    tk::StagePlan plan{};
    tk::RowPlan rplan{};
    const bool have_rows = l->mode == tk::MODE_ADJ_PACKED && staged_enabled() &&
                           tk::make_row_plan(l->shape, l->num_sms, &rplan);
    const bool have_ring = !have_rows && l->mode == tk::MODE_ADJ_PACKED && staged_enabled() &&
                           tk::ring_plan_available(l->shape, stage_budget(l), l->num_sms);
    const bool have_plan = !have_rows && !have_ring && l->mode == tk::MODE_ADJ_PACKED &&
                           staged_enabled() &&
                           tk::make_stage_plan(l->shape, true, stage_budget(l), &plan, false);
    l->pr_staged = have_rows ? 2 : have_plan ? 1 : 0;
    l->pr_done = false;
    st = run_pagerank(l->device, l->num_sms, l->shape, l->mode, l->wide, a, l->part,
                      l->small.as<Small>(), l->hsmall, l->stream, d, tol, max_iter, l->ev[2],
                      l->ev[3], &l->ms_pr, &l->pr_grid, have_plan ? &plan : nullptr,
                      have_rows ? &rplan : nullptr, stage_budget(l), &l->pr_staged, have_ring);
    if (st) return st;
    const PrOut& o = l->hsmall->pr;
    l->iterations = o.iter;
    l->residual = o.res;
    l->pr_sum = o.sum;
    l->pr_parity = o.parity;
    if (o.status != 0) return nonconv(o.iter, o.res);
    l->pr_done = true;
    return TK_OK;
}

// Sharded PageRank stores contributions only; the shard's rank vector is
// rebuilt into r0 (shard_materialize_kernel) the first time a reader needs it
// after a step.  Enqueued on the handle's stream ahead of the reader.
cudaError_t shard_refresh_r(tk_land* l) {
    if (!l->sharded || !l->shard_pr || l->shard_r_fresh) return cudaSuccess;
    const double* c = l->shard_cur ? l->c1.as<double>() : l->c0.as<double>();
    cudaError_t e = tk::launch_shard_materialize(l->shard_lo, l->shard_hi, l->pw.as<uint32_t>(), c,
                                                 l->r0.as<double>(), l->num_sms, l->stream);
    if (e == cudaSuccess) l->shard_r_fresh = true;
    return e;
}

// (sharded handles: call shard_refresh_r first)
const double* pr_result(const tk_land* l) {
    if (l->sharded && l->shard_pr) return l->r0.as<double>();
    return l->pr_parity ? l->r1.as<double>() : l->r0.as<double>();
}

int do_centrality(tk_land* l, double f_opt, const double* p, int n_p, double* c_p) {
    if (!l->pr_done) return fail(TK_ESTATE, "centrality: run pagerank first");
    if (n_p < 1 || n_p > TK_MAX_CP) return fail(TK_EINVAL, "centrality: 1..101 values of p");
    if (l->n_minima == 0) return fail(TK_EDEGEN, "proportion_of_centrality: no local minima");
    TKC(set_dev(l));
    TKC(ensure(l->cp_part, static_cast<size_t>(TK_MAX_CP + 1) * tk::kCpBlocks * 8));
    TKC(ensure(l->cp_out, TK_MAX_CP * 8));
    Small* ds = l->small.as<Small>();
    TKC(shard_refresh_r(l));
    TKC(tk::launch_centrality(l->minima.as<uint32_t>(), l->n_minima, l->fit.as<double>(),
                              pr_result(l), p, n_p, f_opt, l->cp_part.as<double>(),
                              l->cp_out.as<double>(), &ds->degenerate, l->stream));
    TKC(cudaMemcpyAsync(c_p, l->cp_out.p, static_cast<size_t>(n_p) * 8, cudaMemcpyDeviceToHost,
                        l->stream));
    TKC(cudaMemcpyAsync(&l->hsmall->degenerate, &ds->degenerate, 4, cudaMemcpyDeviceToHost,
                        l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    if (l->hsmall->degenerate)
        return fail(TK_EDEGEN, "proportion_of_centrality: minima hold zero PageRank mass");
    return TK_OK;
}

cudaMemcpyKind h2x(int mem) {
    return mem == TK_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
}

// Valid (key, fitness) pairs -> the dense rank-indexed table (perfect hash:
// keys are ranks < N).  Absent keys are failed points (SPEC.md:82,
// cache_io.cpp:79-112).
int do_load_sparse_keys(tk_land* l, const unsigned long long* dkeys, const double* dvals,
                        uint64_t nv) {
    TKC(ensure(l->fit, (l->n + kPad) * 8));
    TKC(ensure(l->ok, l->n + kPad));
    TKC(ensure(l->claimed, ((l->n + 31) / 32) * 4));
    l->hcap = 0;
    Small* ds = l->small.as<Small>();
    TKC(cudaMemsetAsync(&ds->err, 0, 4, l->stream));
    // TK_INGEST_PARTITION=1: pairs partitioned by table slice first, so the
    // scatter stays in L2 (scatter 8.5 -> 3.3 ms on C5, but the partition pass
    // costs 4.4 ms: 8.2 vs 8.7 ms in total; profiles/hash/r02_partition.md)
    void* scratch = nullptr;
    if (std::getenv("TK_INGEST_PARTITION") && nv) {
        TKC(ensure(l->tmp, tk::load_valid_scratch_bytes(nv, static_cast<uint32_t>(l->n))));
        scratch = l->tmp.p;
    }
    TKC(tk::launch_load_valid(dkeys, dvals, nv, static_cast<uint32_t>(l->n), l->fit.as<double>(),
                              l->ok.as<uint8_t>(), l->claimed.as<unsigned int>(), &ds->err,
                              l->stream, scratch));
    TKC(cudaMemcpyAsync(&l->hsmall->err, &ds->err, 4, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    l->built = l->pr_done = false;
    l->loaded = false;
    l->opt_ready = false;
    const int err = l->hsmall->err;
    if (err & 1) return fail(TK_EINVAL, "load: configuration key outside the search space");
    if (err & 4)
        return fail(TK_EINVAL, "load: an ok mean >= kFailFitness (1e10) would order above failed "
                               "points (cache.hpp:15)");
    if (err & 2) return fail(TK_EINVAL, "load: duplicate configuration key");
    l->loaded = true;
    l->fit_clean = !(err & 16);
    return TK_OK;
}

// Build the open-addressing table of the loaded table's ok ranks (lazily, on
// the first tk_land_lookup after a load).
int ensure_hash(tk_land* l) {
    if (l->hcap) return TK_OK;
    Small* ds = l->small.as<Small>();
    TKC(tk::launch_count_ok(l->ok.as<uint8_t>(), static_cast<uint32_t>(l->n), &ds->totals[0],
                            l->stream));
    TKC(cudaMemcpyAsync(&l->hsmall->totals[0], &ds->totals[0], 8, cudaMemcpyDeviceToHost,
                        l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    const uint64_t nv = l->hsmall->totals[0];
    uint64_t cap = 64;
    while (cap < 2 * nv) cap <<= 1;
    TKC(ensure(l->hkeys, cap * 8));
    TKC(ensure(l->hvals, cap * 8));
    TKC(cudaMemsetAsync(&ds->err, 0, 4, l->stream));
    TKC(tk::launch_hash_build(l->fit.as<double>(), l->ok.as<uint8_t>(), static_cast<uint32_t>(l->n),
                              l->hkeys.as<unsigned long long>(), l->hvals.as<double>(), cap,
                              &ds->err, l->stream));
    TKC(cudaMemcpyAsync(&l->hsmall->err, &ds->err, 4, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    if (l->hsmall->err) return fail(TK_ECUDA, "valid-set hash table: probe bound exceeded");
    l->hcap = cap;
    return TK_OK;
}

}  // namespace

// ================================================================ the ABI ==

#define TK_GUARD_BEGIN try {
#define TK_GUARD_END                                                   \
    }                                                                  \
    catch (const std::bad_alloc&) {                                    \
        return fail(TK_ENOMEM, "host allocation failed");              \
    }                                                                  \
    catch (const std::exception& e) {                                  \
        return fail(TK_EINVAL, e.what());                              \
    }

extern "C" {

int tk_abi_version(void) { return TK_ABI_VERSION; }

const char* tk_last_error(void) { return g_err.c_str(); }

const char* tk_status_name(int st) {
    switch (st) {
        case TK_OK: return "TK_OK";
        case TK_EINVAL: return "TK_EINVAL";
        case TK_ELIMIT: return "TK_ELIMIT";
        case TK_ENOFEAS: return "TK_ENOFEAS";
        case TK_ENOCONV: return "TK_ENOCONV";
        case TK_EDEGEN: return "TK_EDEGEN";
        case TK_ENOMEM: return "TK_ENOMEM";
        case TK_ECUDA: return "TK_ECUDA";
        case TK_ENCCL: return "TK_ENCCL";
        case TK_ESTATE: return "TK_ESTATE";
        default: return "TK_UNKNOWN";
    }
}

int tk_device_count(int* count) {
    TKC(cudaGetDeviceCount(count));
    return TK_OK;
}

int tk_land_create(int device, uint32_t dims, const uint32_t* radix, tk_land** out) {
    TK_GUARD_BEGIN
    if (!out) return fail(TK_EINVAL, "tk_land_create: null out pointer");
    *out = nullptr;
    if (dims == 0 || dims > TK_MAX_DIMS || !radix)
        return fail(TK_EINVAL, "a space needs 1..32 parameters");
    uint64_t n = 1;
    for (uint32_t i = 0; i < dims; ++i) {
        if (radix[i] == 0) return fail(TK_EINVAL, "parameter with an empty value list");
        n *= radix[i];
        if (n > kMaxNodes)
            return fail(TK_ELIMIT, "search space exceeds the u32 node-id range of the FFG");
    }
    int ndev = 0;
    TKC(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(TK_EINVAL, "no such CUDA device");
    TKC(cudaSetDevice(device));
    tk_land* l = new tk_land();
    l->device = device;
    l->radix_in.assign(radix, radix + dims);
    l->strides_in.assign(dims, 1);
    for (int i = static_cast<int>(dims) - 2; i >= 0; --i)
        l->strides_in[i] = l->strides_in[i + 1] * radix[i + 1];
    l->n = n;
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e == cudaSuccess) {
        l->num_sms = prop.multiProcessorCount;
        l->smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
        l->smem_per_sm = static_cast<int>(prop.sharedMemPerMultiprocessor);
        if (!prop.cooperativeLaunch) e = cudaErrorNotSupported;
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = ensure(l->small, sizeof(Small));
    if (e == cudaSuccess) e = cudaMallocHost(&l->hsmall, sizeof(Small));
    for (int i = 0; i < 6 && e == cudaSuccess; ++i) e = cudaEventCreate(&l->ev[i]);
    if (e != cudaSuccess) {
        tk_land_destroy(l);
        return cuda_fail(e, "tk_land_create");
    }
    *out = l;
    return TK_OK;
    TK_GUARD_END
}

int tk_land_reshape(tk_land* l, uint32_t dims, const uint32_t* radix) {
    if (int st = check_land(l)) return st;
    if (dims == 0 || dims > TK_MAX_DIMS || !radix)
        return fail(TK_EINVAL, "a space needs 1..32 parameters");
    uint64_t n = 1;
    for (uint32_t i = 0; i < dims; ++i) {
        if (radix[i] == 0) return fail(TK_EINVAL, "parameter with an empty value list");
        n *= radix[i];
        if (n > kMaxNodes)
            return fail(TK_ELIMIT, "search space exceeds the u32 node-id range of the FFG");
    }
    if (l->sharded) return fail(TK_ESTATE, "reshape of a sharded handle");
    l->radix_in.assign(radix, radix + dims);
    l->strides_in.assign(dims, 1);
    for (int i = static_cast<int>(dims) - 2; i >= 0; --i)
        l->strides_in[i] = l->strides_in[i + 1] * radix[i + 1];
    l->n = n;
    l->loaded = l->built = l->emitted = l->pr_done = l->opt_ready = false;
    l->hcap = 0;
    return TK_OK;
}

int tk_land_destroy(tk_land* l) {
    if (!l) return TK_OK;
    cudaSetDevice(l->device);
    if (l->stream) cudaStreamSynchronize(l->stream);
    for (void* p : l->ipc_opened) cudaIpcCloseMemHandle(p);
    DevBuf* bufs[] = {&l->fit, &l->ok, &l->claimed, &l->hkeys, &l->hvals, &l->staging_keys, &l->staging_vals,
                      &l->staging_cfg, &l->pw, &l->inm, &l->odeg, &l->flags, &l->offsets,
                      &l->targets, &l->minima, &l->e_status, &l->m_status, &l->counter,
                      &l->om, &l->tile_cnt, &l->tile_base,
                      &l->r0, &l->r1, &l->c0, &l->c1, &l->part, &l->small, &l->opt_part,
                      &l->cp_part, &l->cp_out, &l->tmp};
    for (DevBuf* b : bufs) b->release();
    if (l->hsmall) cudaFreeHost(l->hsmall);
    for (auto& ev : l->ev)
        if (ev) cudaEventDestroy(ev);
    if (l->stream) cudaStreamDestroy(l->stream);
    delete l;
    return TK_OK;
}

int tk_land_info(const tk_land* l, uint64_t* n_nodes, int* device) {
    if (int st = check_land(l)) return st;
    if (n_nodes) *n_nodes = l->n;
    if (device) *device = l->device;
    return TK_OK;
}

void* tk_land_stream(tk_land* l) { return l ? static_cast<void*>(l->stream) : nullptr; }

int tk_land_kernel_info(const tk_land* l, int* staged_build, int* staged_pagerank,
                        int* pagerank_grid, float* ms_build, float* ms_pagerank) {
    if (int st = check_land(l)) return st;
    if (staged_build) *staged_build = l->staged ? 1 : 0;
    if (staged_pagerank) *staged_pagerank = l->pr_staged;
    if (pagerank_grid) *pagerank_grid = l->pr_grid;
    if (ms_build) *ms_build = l->ms_build;
    if (ms_pagerank) *ms_pagerank = l->ms_pr;
    return TK_OK;
}

int tk_land_load_dense(tk_land* l, const double* fitness, const uint8_t* ok, int mem) {
    if (int st = check_land(l)) return st;
    if (!fitness || !ok) return fail(TK_EINVAL, "load_dense: null buffer");
    TKC(set_dev(l));
    TKC(ensure(l->fit, (l->n + kPad) * 8));
    TKC(ensure(l->ok, l->n + kPad));
    TKC(cudaMemcpyAsync(l->fit.p, fitness, l->n * 8, h2x(mem), l->stream));
    TKC(cudaMemcpyAsync(l->ok.p, ok, l->n, h2x(mem), l->stream));
    Small* ds = l->small.as<Small>();
    TKC(cudaMemsetAsync(&ds->err, 0, 4, l->stream));
    TKC(tk::launch_normalize_dense(static_cast<uint32_t>(l->n), l->fit.as<double>(),
                                   l->ok.as<uint8_t>(), &ds->err, l->stream));
    TKC(cudaMemcpyAsync(&l->hsmall->err, &ds->err, 4, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    l->hcap = 0;
    l->opt_ready = false;
    l->built = l->pr_done = false;
    l->loaded = !(l->hsmall->err & 4);
    l->fit_clean = !(l->hsmall->err & 16);
    if (!l->loaded)
        return fail(TK_EINVAL, "load_dense: an ok mean >= kFailFitness (1e10) would order above "
                               "failed points (cache.hpp:15)");
    return TK_OK;
}

int tk_land_load_sparse(tk_land* l, const uint64_t* keys, const double* fitness,
                        uint64_t n_valid, int mem) {
    if (int st = check_land(l)) return st;
    if ((!keys || !fitness) && n_valid) return fail(TK_EINVAL, "load_sparse: null buffer");
    TKC(set_dev(l));
    const unsigned long long* dk = reinterpret_cast<const unsigned long long*>(keys);
    const double* dv = fitness;
    if (mem != TK_MEM_DEVICE) {
        TKC(ensure(l->staging_keys, n_valid * 8));
        TKC(ensure(l->staging_vals, n_valid * 8));
        if (n_valid) {
            TKC(cudaMemcpyAsync(l->staging_keys.p, keys, n_valid * 8, cudaMemcpyHostToDevice,
                                l->stream));
            TKC(cudaMemcpyAsync(l->staging_vals.p, fitness, n_valid * 8, cudaMemcpyHostToDevice,
                                l->stream));
        }
        dk = l->staging_keys.as<unsigned long long>();
        dv = l->staging_vals.as<double>();
    }
    return do_load_sparse_keys(l, dk, dv, n_valid);
}

int tk_land_load_configs(tk_land* l, const int32_t* configs, const double* fitness,
                         uint64_t n_valid, int mem) {
    if (int st = check_land(l)) return st;
    if ((!configs || !fitness) && n_valid) return fail(TK_EINVAL, "load_configs: null buffer");
    TKC(set_dev(l));
    const size_t dims = l->radix_in.size();
    const int32_t* dc = configs;
    const double* dv = fitness;
    if (mem != TK_MEM_DEVICE) {
        TKC(ensure(l->staging_cfg, n_valid * dims * 4));
        TKC(ensure(l->staging_vals, n_valid * 8));
        if (n_valid) {
            TKC(cudaMemcpyAsync(l->staging_cfg.p, configs, n_valid * dims * 4,
                                cudaMemcpyHostToDevice, l->stream));
            TKC(cudaMemcpyAsync(l->staging_vals.p, fitness, n_valid * 8, cudaMemcpyHostToDevice,
                                l->stream));
        }
        dc = l->staging_cfg.as<int32_t>();
        dv = l->staging_vals.as<double>();
    }
    TKC(ensure(l->staging_keys, n_valid * 8));
    Small* ds = l->small.as<Small>();
    TKC(cudaMemsetAsync(&ds->err, 0, 4, l->stream));
    TKC(tk::launch_encode_configs(dc, n_valid, static_cast<int>(dims), l->radix_in.data(),
                                  l->strides_in.data(), l->staging_keys.as<unsigned long long>(),
                                  &ds->err, l->stream));
    TKC(cudaMemcpyAsync(&l->hsmall->err, &ds->err, 4, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    if (l->hsmall->err)
        return fail(TK_EINVAL, "load_configs: configuration index outside its value list");
    return do_load_sparse_keys(l, l->staging_keys.as<unsigned long long>(), dv, n_valid);
}

int tk_land_generate(tk_land* l, int gen, double fail_fraction, uint64_t seed) {
    if (int st = check_land(l)) return st;
    if (gen != TK_GEN_IID && gen != TK_GEN_HEAVY) return fail(TK_EINVAL, "unknown generator");
    if (!(fail_fraction >= 0.0 && fail_fraction < 1.0))
        return fail(TK_EINVAL, "fail_fraction must be in [0, 1)");
    TKC(set_dev(l));
    TKC(ensure(l->fit, (l->n + kPad) * 8));
    TKC(ensure(l->ok, l->n + kPad));
    TKC(tk::launch_generate(gen, static_cast<uint32_t>(l->n), fail_fraction, seed,
                            l->fit.as<double>(), l->ok.as<uint8_t>(), l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    l->hcap = 0;
    l->loaded = true;
    l->fit_clean = true;  // 1 + u or 1 / (1 - u), u in [0, 1), and kFailFitness: finite, > 0
    l->opt_ready = false;
    l->built = l->pr_done = false;
    return TK_OK;
}

int tk_land_copy_fitness(tk_land* l, double* fitness, uint8_t* ok) {
    if (int st = check_land(l)) return st;
    if (!l->loaded) return fail(TK_ESTATE, "copy_fitness: nothing loaded");
    TKC(set_dev(l));
    if (fitness)
        TKC(cudaMemcpyAsync(fitness, l->fit.p, l->n * 8, cudaMemcpyDeviceToHost, l->stream));
    if (ok) TKC(cudaMemcpyAsync(ok, l->ok.p, l->n, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    return TK_OK;
}

int tk_land_lookup(tk_land* l, const uint64_t* keys, uint64_t n, double* fitness,
                   uint8_t* found) {
    if (int st = check_land(l)) return st;
    if (!l->loaded) return fail(TK_ESTATE, "lookup: nothing loaded");
    if (n && !keys) return fail(TK_EINVAL, "lookup: null keys");
    TKC(set_dev(l));
    if (int st = ensure_hash(l)) return st;
    if (n == 0) return TK_OK;
    TKC(ensure(l->tmp, n * 17 + 16));
    unsigned long long* dq = l->tmp.as<unsigned long long>();
    double* dout = reinterpret_cast<double*>(dq + n);
    uint8_t* dfound = reinterpret_cast<uint8_t*>(dout + n);
    Small* ds = l->small.as<Small>();
    TKC(cudaMemsetAsync(&ds->err, 0, 4, l->stream));
    TKC(cudaMemcpyAsync(dq, keys, n * 8, cudaMemcpyHostToDevice, l->stream));
    TKC(tk::launch_hash_lookup(l->hkeys.as<unsigned long long>(), l->hvals.as<double>(), l->hcap,
                               dq, n, dout, dfound, &ds->err, l->stream));
    if (fitness) TKC(cudaMemcpyAsync(fitness, dout, n * 8, cudaMemcpyDeviceToHost, l->stream));
    if (found) TKC(cudaMemcpyAsync(found, dfound, n, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaMemcpyAsync(&l->hsmall->err, &ds->err, 4, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    if (l->hsmall->err) return fail(TK_ECUDA, "valid-set hash table: probe bound exceeded");
    return TK_OK;
}

// Whole-space entry points refuse a sharded handle: its FFG rows, flags and
// PageRank cover only its own key range (tk_shard_* are the per-shard calls).
static int check_unsharded(const tk_land* l, const char* what) {
    if (l->sharded)
        return fail(TK_ESTATE, std::string(what) + ": sharded handle (use the tk_shard_* calls)");
    return TK_OK;
}

int tk_optimum(tk_land* l, double* f_opt, uint64_t* rank) {
    if (int st = check_land(l)) return st;
    if (int st = check_unsharded(l, "optimum")) return st;
    return do_optimum(l, f_opt, rank);
}

int tk_ffg_build(tk_land* l, int kind, uint64_t node_limit, int emit_csr, uint64_t* n_edges,
                 uint64_t* n_minima) {
    if (int st = check_land(l)) return st;
    TK_GUARD_BEGIN
    int st = do_build(l, kind, node_limit, emit_csr);
    if (st) return st;
    if (n_edges) *n_edges = l->n_edges;
    if (n_minima) *n_minima = l->n_minima;
    return TK_OK;
    TK_GUARD_END
}

int tk_ffg_copy_out(tk_land* l, uint64_t* offsets, uint32_t* targets, uint8_t* is_sink,
                    uint32_t* minima) {
    if (int st = check_land(l)) return st;
    if (!l->built) return fail(TK_ESTATE, "copy_out: build the FFG first");
    if (offsets || targets || is_sink)
        if (int st = check_unsharded(l, "ffg_copy_out")) return st;
    TKC(set_dev(l));
    if ((offsets || targets) && !l->emitted) {
        const bool pr = l->pr_done;
        int st = do_build(l, l->kind, ~0ull, 1);  // re-emit the CSR rows (same graph)
        if (st) return st;
        l->pr_done = pr;
    }
    if (offsets)
        TKC(cudaMemcpyAsync(offsets, l->offsets.p, (l->n + 1) * 8, cudaMemcpyDeviceToHost,
                            l->stream));
    if (targets && l->n_edges)
        TKC(cudaMemcpyAsync(targets, l->targets.p, l->n_edges * 4, cudaMemcpyDeviceToHost,
                            l->stream));
    if (minima && l->n_minima)
        TKC(cudaMemcpyAsync(minima, l->minima.p, l->n_minima * 4, cudaMemcpyDeviceToHost,
                            l->stream));
    if (is_sink) {
        TKC(ensure(l->tmp, l->n));
        TKC(tk::launch_flags_to_sink(l->flags.as<uint8_t>(), static_cast<uint32_t>(l->n),
                                     l->tmp.as<uint8_t>(), l->stream));
        TKC(cudaMemcpyAsync(is_sink, l->tmp.p, l->n, cudaMemcpyDeviceToHost, l->stream));
    }
    TKC(cudaStreamSynchronize(l->stream));
    return TK_OK;
}

int tk_census(tk_land* l, uint64_t* fail_points, uint64_t* local_minima, uint64_t* interior,
              uint64_t* minima_ranks) {
    if (int st = check_land(l)) return st;
    if (int st = check_unsharded(l, "census")) return st;
    if (!l->built) return fail(TK_ESTATE, "census: build the FFG first");
    TKC(set_dev(l));
    // strict minima (flag bit2) compacted in ascending rank with a look-back scan
    const uint32_t ntiles = static_cast<uint32_t>((l->n + 255) / 256);
    if (minima_ranks && l->n_strict) {
        TKC(ensure(l->tmp, l->n_strict * 8));
        TKC(cudaMemsetAsync(l->e_status.p, 0, static_cast<size_t>(ntiles) * 8, l->stream));
        TKC(cudaMemsetAsync(l->counter.p, 0, 16, l->stream));
        TKC(tk::launch_compact_flags(l->flags.as<uint8_t>(), 4, static_cast<uint32_t>(l->n),
                                     l->tmp.as<unsigned long long>(),
                                     l->e_status.as<unsigned long long>(),
                                     l->counter.as<unsigned int>(), ntiles, l->num_sms,
                                     l->stream));
        TKC(cudaMemcpyAsync(minima_ranks, l->tmp.p, l->n_strict * 8, cudaMemcpyDeviceToHost,
                            l->stream));
        TKC(cudaStreamSynchronize(l->stream));
    }
    if (fail_points) *fail_points = l->n - l->n_ok;
    if (local_minima) *local_minima = l->n_strict;
    if (interior) *interior = l->n_ok - l->n_strict;
    return TK_OK;
}

int tk_pagerank(tk_land* l, double damping, double tol, int64_t max_iter, int64_t* iterations,
                double* residual, double* sum) {
    if (int st = check_land(l)) return st;
    if (int st = check_unsharded(l, "pagerank")) return st;
    int st = do_pagerank(l, damping, tol, max_iter);
    if (iterations) *iterations = l->iterations;
    if (residual) *residual = l->residual;
    if (sum) *sum = l->pr_sum;
    return st;
}

int tk_pagerank_copy_out(tk_land* l, double* r) {
    if (int st = check_land(l)) return st;
    if (!l->pr_done) return fail(TK_ESTATE, "pagerank_copy_out: no converged PageRank");
    TKC(set_dev(l));
    TKC(shard_refresh_r(l));
    TKC(cudaMemcpyAsync(r, pr_result(l), l->n * 8, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    return TK_OK;
}

int tk_centrality(tk_land* l, double f_opt, const double* p, int n_p, double* c_p) {
    if (int st = check_land(l)) return st;
    if (int st = check_unsharded(l, "centrality")) return st;
    if (!p || !c_p) return fail(TK_EINVAL, "centrality: null buffer");
    return do_centrality(l, f_opt, p, n_p, c_p);
}

int tk_report_copy_out(tk_land* l, double f_opt, uint64_t* ranks, double* fitness,
                       double* fraction, double* pagerank) {
    if (int st = check_land(l)) return st;
    if (!l->pr_done && !(l->sharded && l->shard_pr))
        return fail(TK_ESTATE, "report: run pagerank first");
    const uint64_t m = l->n_minima;
    if (!m) return TK_OK;
    TKC(set_dev(l));
    TKC(ensure(l->tmp, m * 32));
    unsigned long long* dr = l->tmp.as<unsigned long long>();
    double* df = reinterpret_cast<double*>(dr + m);
    double* dfr = df + m;
    double* dp = dfr + m;
    TKC(shard_refresh_r(l));
    TKC(tk::launch_report(l->minima.as<uint32_t>(), m, l->fit.as<double>(), pr_result(l), f_opt,
                          dr, df, dfr, dp, l->stream));
    if (ranks) TKC(cudaMemcpyAsync(ranks, dr, m * 8, cudaMemcpyDeviceToHost, l->stream));
    if (fitness) TKC(cudaMemcpyAsync(fitness, df, m * 8, cudaMemcpyDeviceToHost, l->stream));
    if (fraction) TKC(cudaMemcpyAsync(fraction, dfr, m * 8, cudaMemcpyDeviceToHost, l->stream));
    if (pagerank) TKC(cudaMemcpyAsync(pagerank, dp, m * 8, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    return TK_OK;
}

int tk_analyze(tk_land* l, int kind, double damping, double tol, int64_t max_iter,
               uint64_t node_limit, int p_max_percent, int emit_csr, tk_report_summary* out) {
    if (int st = check_land(l)) return st;
    if (int st = check_unsharded(l, "analyze")) return st;
    if (!out) return fail(TK_EINVAL, "analyze: null summary");
    if (p_max_percent < 0 || p_max_percent >= TK_MAX_CP)
        return fail(TK_EINVAL, "analyze: p_max_percent must be in [0, 100]");
    int st = check_pr_args(damping, tol, max_iter);
    if (st) return st;
    TK_GUARD_BEGIN
    std::memset(out, 0, sizeof(*out));
    TKC(set_dev(l));
    st = do_build(l, kind, node_limit, emit_csr);
    if (st) return st;
    double f_opt = 0.0;
    uint64_t orank = 0;
    st = do_optimum(l, &f_opt, &orank);
    if (st) return st;
    st = do_pagerank(l, damping, tol, max_iter);
    out->iterations = l->iterations;
    out->residual = l->residual;
    if (st) return st;
    TKC(cudaEventRecord(l->ev[4], l->stream));
    double ps[TK_MAX_CP];
    const int np = p_max_percent + 1;
    for (int k = 0; k < np; ++k) ps[k] = k / 100.0;
    st = do_centrality(l, f_opt, ps, np, out->c_p);
    if (st) return st;
    TKC(cudaEventRecord(l->ev[5], l->stream));
    TKC(cudaEventSynchronize(l->ev[5]));
    out->n_nodes = l->n;
    out->n_edges = l->n_edges;
    out->n_minima = l->n_minima;
    out->f_opt = f_opt;
    out->opt_rank = orank;
    out->pagerank_sum = l->pr_sum;
    out->n_cp = np;
    out->ms_load = 0.f;
    out->ms_ffg = l->ms_build;
    out->ms_pagerank = l->ms_pr;
    TKC(cudaEventElapsedTime(&out->ms_centrality, l->ev[4], l->ev[5]));
    return TK_OK;
    TK_GUARD_END
}

// ---------------------------------------------- batches of small spaces --

namespace {
// per-device batch context: one stream, a device workspace and a pinned
// read-back buffer, reused across calls (guarded: one batch at a time per device)
struct BatchCtx {
    std::mutex mu;
    bool init = false;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    DevBuf ws, jobs;
    void* host_out = nullptr;
    size_t host_out_cap = 0;
    void* host_rows = nullptr;
    size_t host_rows_cap = 0;
};
BatchCtx& batch_ctx(int device) {
    static BatchCtx ctx[64];
    return ctx[device & 63];
}
}  // namespace

int tk_batch_analyze(int device, tk_batch_item* items, uint32_t n_items, int kind, double damping,
                     double tol, int64_t max_iter, int p_max_percent, int mem) {
    if (!items && n_items) return fail(TK_EINVAL, "batch_analyze: null items");
    if (kind != TK_ADJACENT && kind != TK_HAMMING) return fail(TK_EINVAL, "batch_analyze: kind");
    if (p_max_percent < 0 || p_max_percent >= TK_MAX_CP)
        return fail(TK_EINVAL, "batch_analyze: p_max_percent must be in [0, 100]");
    if (int st = check_pr_args(damping, tol, max_iter)) return st;
    if (n_items == 0) return TK_OK;
    TK_GUARD_BEGIN
    BatchCtx& C = batch_ctx(device);
    std::lock_guard<std::mutex> lk(C.mu);
    TKC(cudaSetDevice(device));
    if (!C.init) {
        TKC(cudaStreamCreateWithFlags(&C.stream, cudaStreamNonBlocking));
        TKC(cudaDeviceGetAttribute(&C.num_sms, cudaDevAttrMultiProcessorCount, device));
        C.init = true;
    }
    // workspace layout: [descs][outs][per item: fitness, ok, scratch, report rows]
    const size_t dsz = tk::batch_desc_bytes();
    auto a256 = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
    std::vector<uint64_t> ns(n_items, 0);
    std::vector<size_t> off(n_items, 0);
    const size_t gsb = tk::batch_group_state_bytes();
    uint64_t rows_cap = 0;  // report rows of all spaces, packed (<= sum of N)
    size_t total = a256(dsz * n_items) + a256(sizeof(tk::BatchOut) * n_items) +
                   a256(gsb * n_items);
    for (uint32_t i = 0; i < n_items; ++i) {
        items[i].status = TK_OK;
        std::memset(&items[i].summary, 0, sizeof(items[i].summary));
        if (items[i].dims < 1 || items[i].dims > TK_MAX_DIMS ||
            !tk::batch_item_supported(items[i].dims, items[i].radix, kind, &ns[i]) ||
            !items[i].fitness || !items[i].ok) {
            items[i].status = TK_EINVAL;
            ns[i] = 0;
            continue;
        }
        off[i] = total;
        total += a256(8 * ns[i]) + a256(ns[i]) +
                 tk::batch_workspace_bytes(static_cast<uint32_t>(ns[i]),
                                           tk::batch_slots(items[i].dims, items[i].radix, kind));
        rows_cap += ns[i];
    }
    const size_t rows_at = total;
    total += 256 + a256(32 * rows_cap);  // row cursor, then the rows
    TKC(ensure(C.ws, total));
    uint8_t* base = C.ws.as<uint8_t>();
    unsigned long long* row_cursor = reinterpret_cast<unsigned long long*>(base + rows_at);
    double* rows_dev = reinterpret_cast<double*>(base + rows_at + 256);
    tk::BatchOut* dout = reinterpret_cast<tk::BatchOut*>(base + a256(dsz * n_items));
    uint8_t* gstate = base + a256(dsz * n_items) + a256(sizeof(tk::BatchOut) * n_items);
    std::vector<uint8_t> descs(dsz * n_items, 0);
    std::vector<uint32_t> live;
    for (uint32_t i = 0; i < n_items; ++i) {
        if (!ns[i]) continue;
        uint8_t* p = base + off[i];
        const uint64_t n = ns[i];
        double* fit = reinterpret_cast<double*>(p);
        uint8_t* ok = p + a256(8 * n);
        uint8_t* scr = ok + a256(n);
        const uint32_t slots = tk::batch_slots(items[i].dims, items[i].radix, kind);
        if (mem == TK_MEM_DEVICE) {
            fit = const_cast<double*>(items[i].fitness);
            ok = const_cast<uint8_t*>(items[i].ok);
        } else {
            TKC(cudaMemcpyAsync(fit, items[i].fitness, 8 * n, cudaMemcpyHostToDevice, C.stream));
            TKC(cudaMemcpyAsync(ok, items[i].ok, n, cudaMemcpyHostToDevice, C.stream));
        }
        const bool want_rows = items[i].minima_ranks || items[i].minima_fitness ||
                               items[i].minima_fraction || items[i].minima_pagerank;
        tk::batch_fill_desc(descs.data() + dsz * live.size(), fit, ok, static_cast<uint32_t>(n),
                            slots, items[i].dims, items[i].radix, scr,
                            reinterpret_cast<unsigned int*>(gstate + gsb * live.size()),
                            reinterpret_cast<double*>(gstate + gsb * live.size() + 64),
                            dout + live.size(), want_rows ? rows_dev : nullptr, row_cursor);
        live.push_back(i);
    }
    if (live.empty()) return TK_OK;
    const uint32_t nl = static_cast<uint32_t>(live.size());
    TKC(cudaMemcpyAsync(base, descs.data(), dsz * nl, cudaMemcpyHostToDevice, C.stream));
    TKC(cudaMemsetAsync(row_cursor, 0, 8, C.stream));
    tk::BatchParams P{};
    P.kind = kind;
    P.damping = damping;
    P.tol = tol;
    P.max_iter = max_iter;
    P.n_p = p_max_percent + 1;
    for (int k = 0; k < P.n_p; ++k) {
        const double pk = k / 100.0;
        P.onep[k] = 1.0 + pk;  // the band of launch_centrality: f < (1 + p) * f_opt
        P.zero[k] = pk == 0.0;
    }
    const int R = tk::batch_group_resident(C.num_sms);
    const bool grouped = R > 0 && P.n_p <= tk::batch_group_max_np() && !std::getenv("TK_BATCH_NOGROUP");
    if (grouped) {
        // spaces largest first; a space of n ranks gets ceil(n / 8192) CTAs (at
        // most batch_group_max); jobs dealt into waves of R CTAs, a space's
        // members in one wave
        std::vector<uint32_t> order(nl);
        for (uint32_t j = 0; j < nl; ++j) order[j] = j;
        std::stable_sort(order.begin(), order.end(),
                         [&](uint32_t a, uint32_t b) { return ns[live[a]] > ns[live[b]]; });
        std::vector<int> gsz(nl);
        for (uint32_t j = 0; j < nl; ++j) {
            const uint64_t g = (ns[live[j]] + 8191) / 8192;
            gsz[j] = static_cast<int>(std::min<uint64_t>(std::max<uint64_t>(g, 1),
                                                         std::min(tk::batch_group_max(), R)));
        }
        std::vector<std::vector<std::pair<int, int>>> waves;  // per wave: (item, g) placed
        std::vector<int> fill;
        for (uint32_t oi : order) {
            const int g = gsz[oi];
            size_t w = 0;
            while (w < waves.size() && fill[w] + g > R) ++w;
            if (w == waves.size()) {
                waves.emplace_back();
                fill.push_back(0);
            }
            waves[w].push_back({static_cast<int>(oi), g});
            fill[w] += g;
        }
        const int nw = static_cast<int>(waves.size());
        std::vector<uint8_t> jobs(tk::batch_job_bytes() * static_cast<size_t>(nw) * R);
        for (int w = 0; w < nw; ++w) {
            int cta = 0;
            for (const auto& ig : waves[w])
                for (int r = 0; r < ig.second; ++r)
                    tk::batch_set_job(jobs.data(), static_cast<size_t>(w) * R + cta++, ig.first, r,
                                      ig.second);
            for (; cta < R; ++cta) tk::batch_set_job(jobs.data(), static_cast<size_t>(w) * R + cta, -1, 0, 1);
        }
        TKC(ensure(C.jobs, jobs.size()));
        TKC(cudaMemcpyAsync(C.jobs.p, jobs.data(), jobs.size(), cudaMemcpyHostToDevice, C.stream));
        TKC(cudaMemsetAsync(gstate, 0, gsb * nl, C.stream));  // group barriers start at {0, 0}
        TKC(tk::launch_batch_group(base, C.jobs.p, nw, R, P, C.stream));
    } else {
        TKC(tk::launch_batch_analyze(base, nl, P, C.num_sms, C.stream));
    }
    const size_t ob = sizeof(tk::BatchOut) * nl;
    if (C.host_out_cap < ob) {
        if (C.host_out) cudaFreeHost(C.host_out);
        C.host_out = nullptr;
        C.host_out_cap = 0;
        TKC(cudaMallocHost(&C.host_out, ob));
        C.host_out_cap = ob;
    }
    TKC(cudaMemcpyAsync(C.host_out, dout, ob, cudaMemcpyDeviceToHost, C.stream));
    unsigned long long n_rows = 0;
    TKC(cudaMemcpyAsync(&n_rows, row_cursor, 8, cudaMemcpyDeviceToHost, C.stream));
    TKC(cudaStreamSynchronize(C.stream));
    // the packed report rows: one read-back into pinned staging
    const size_t rb = static_cast<size_t>(n_rows) * 32;
    if (C.host_rows_cap < rb) {
        if (C.host_rows) cudaFreeHost(C.host_rows);
        C.host_rows = nullptr;
        C.host_rows_cap = 0;
        TKC(cudaMallocHost(&C.host_rows, rb));
        C.host_rows_cap = rb;
    }
    if (rb) TKC(cudaMemcpyAsync(C.host_rows, rows_dev, rb, cudaMemcpyDeviceToHost, C.stream));
    TKC(cudaStreamSynchronize(C.stream));
    const tk::BatchOut* ho = static_cast<const tk::BatchOut*>(C.host_out);
    const double* hrows = static_cast<const double*>(C.host_rows);
    for (uint32_t j = 0; j < nl; ++j) {
        tk_batch_item& it = items[live[j]];
        const tk::BatchOut& o = ho[j];
        tk_report_summary& s = it.summary;
        s.n_nodes = o.n_nodes;
        s.n_edges = o.n_edges;
        s.n_minima = o.n_minima;
        s.f_opt = o.f_opt;
        s.opt_rank = o.opt_rank;
        s.iterations = o.iterations;
        s.residual = o.residual;
        s.pagerank_sum = o.pagerank_sum;
        s.n_cp = P.n_p;
        for (int k = 0; k < P.n_p; ++k) s.c_p[k] = o.c_p[k];
        it.status = o.status;
        const uint64_t m = std::min<uint64_t>(o.n_minima, it.minima_capacity);
        if (o.status != TK_OK || !m) continue;
        const double* row = hrows + o.row_base * 4;
        for (uint64_t i = 0; i < m; ++i, row += 4) {
            if (it.minima_ranks) std::memcpy(it.minima_ranks + i, row, 8);
            if (it.minima_fitness) it.minima_fitness[i] = row[1];
            if (it.minima_fraction) it.minima_fraction[i] = row[2];
            if (it.minima_pagerank) it.minima_pagerank[i] = row[3];
        }
    }
    TKC(cudaStreamSynchronize(C.stream));
    return TK_OK;
    TK_GUARD_END
}

// ------------------------------------------------ random-walk validator --

int tk_descents(tk_land* l, uint64_t walkers, uint64_t seed, int restart_scan,
                uint64_t* arrivals, uint64_t* fail_arrivals, uint64_t* evaluations) {
    if (int st = check_land(l)) return st;
    if (int st = check_unsharded(l, "descents")) return st;
    if (!l->built) return fail(TK_ESTATE, "descents: build the FFG first (neighbourhood, minima)");
    TK_GUARD_BEGIN
    TKC(set_dev(l));
    tk::DescentArgs a{};
    a.fit = l->fit.as<double>();
    a.n = l->n;
    a.dims = static_cast<int>(l->radix_in.size());
    a.kind = l->kind;
    a.restart_scan = restart_scan ? 1 : 0;
    a.walkers = walkers;
    a.seed = seed;
    int S = 0;
    for (int i = 0; i < a.dims; ++i) {  // build_slots (hillclimb.cpp:26-38)
        a.radix[i] = l->radix_in[i];
        a.stride[i] = l->strides_in[i];
        const int m = static_cast<int>(l->radix_in[i]);
        if (l->kind == TK_HAMMING) {
            for (int alt = 0; alt + 1 < m; ++alt) {
                if (S == tk::kMaxDescentSlots) return fail(TK_EINVAL, "descents: more than 256 slots");
                a.slot_dim[S] = static_cast<uint8_t>(i);
                a.slot_alt[S++] = static_cast<int16_t>(alt);
            }
        } else if (m > 1) {
            if (S + 2 > tk::kMaxDescentSlots) return fail(TK_EINVAL, "descents: more than 256 slots");
            a.slot_dim[S] = static_cast<uint8_t>(i);
            a.slot_alt[S++] = -1;
            a.slot_dim[S] = static_cast<uint8_t>(i);
            a.slot_alt[S++] = 1;
        }
    }
    a.slots = S;
    const uint64_t m = l->n_minima;
    TKC(ensure(l->tmp, l->n * 4 + 16 + m * 8));
    a.counts = l->tmp.as<uint32_t>();
    a.evaluations = reinterpret_cast<unsigned long long*>(l->tmp.as<uint8_t>() + ((l->n * 4 + 7) & ~7ull));
    unsigned long long* dout = a.evaluations + 1;
    TKC(cudaMemsetAsync(l->tmp.p, 0, ((l->n * 4 + 7) & ~7ull) + 8, l->stream));
    if (walkers) TKC(tk::launch_descents(a, l->num_sms, l->stream));
    TKC(tk::launch_gather_counts(l->minima.as<uint32_t>(), m, a.counts, dout, l->stream));
    std::vector<unsigned long long> h(m);
    unsigned long long ev = 0;
    if (m) TKC(cudaMemcpyAsync(h.data(), dout, m * 8, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaMemcpyAsync(&ev, a.evaluations, 8, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    uint64_t at_minima = 0;
    for (uint64_t k = 0; k < m; ++k) at_minima += h[k];
    if (arrivals && m) std::memcpy(arrivals, h.data(), m * 8);
    if (fail_arrivals) *fail_arrivals = walkers - at_minima;
    if (evaluations) *evaluations = ev;
    return TK_OK;
    TK_GUARD_END
}

// ------------------------------------------------ key-range sharding ABI --

int tk_land_set_shard(tk_land* l, int rank, int nranks, uint64_t* lo, uint64_t* hi) {
    if (int st = check_land(l)) return st;
    if (nranks < 1 || nranks > tk::kMaxShards || rank < 0 || rank >= nranks)
        return fail(TK_EINVAL, "set_shard: need 0 <= rank < nranks <= 8");
    uint64_t chunk = (l->n + nranks - 1) / nranks;
    chunk = (chunk + 511) / 512 * 512;
    l->shard_rank = rank;
    l->shard_n = nranks;
    l->shard_chunk = chunk;
    l->shard_lo = std::min<uint64_t>(l->n, static_cast<uint64_t>(rank) * chunk);
    l->shard_hi = std::min<uint64_t>(l->n, l->shard_lo + chunk);
    l->sharded = true;
    l->built = l->pr_done = l->shard_pr = false;
    TKC(set_dev(l));
    TKC(ensure(l->c0, (l->n + kPad) * 8));  // replicas exist before peers map them
    TKC(ensure(l->c1, (l->n + kPad) * 8));
    for (int g = 0; g < tk::kMaxShards; ++g) l->peer_c0[g] = l->peer_c1[g] = nullptr;
    l->peer_c0[rank] = l->c0.p;
    l->peer_c1[rank] = l->c1.p;
    if (lo) *lo = l->shard_lo;
    if (hi) *hi = l->shard_hi;
    return TK_OK;
}

int tk_land_replica_ptrs(tk_land* l, void** c0, void** c1) {
    if (int st = check_land(l)) return st;
    if (!l->sharded) return fail(TK_ESTATE, "replica_ptrs: call tk_land_set_shard first");
    if (c0) *c0 = l->c0.p;
    if (c1) *c1 = l->c1.p;
    return TK_OK;
}

int tk_land_set_peer_ptrs(tk_land* l, void* const* c0, void* const* c1) {
    if (int st = check_land(l)) return st;
    if (!l->sharded) return fail(TK_ESTATE, "set_peer_ptrs: call tk_land_set_shard first");
    for (int g = 0; g < l->shard_n; ++g) {
        if (g == l->shard_rank) continue;
        if (!c0[g] || !c1[g]) return fail(TK_EINVAL, "set_peer_ptrs: null replica pointer");
        l->peer_c0[g] = c0[g];
        l->peer_c1[g] = c1[g];
    }
    return TK_OK;
}

int tk_land_ipc_handles(tk_land* l, void* handles128) {
    if (int st = check_land(l)) return st;
    if (!l->sharded) return fail(TK_ESTATE, "ipc_handles: call tk_land_set_shard first");
    TKC(set_dev(l));
    cudaIpcMemHandle_t h[2];
    TKC(cudaIpcGetMemHandle(&h[0], l->c0.p));
    TKC(cudaIpcGetMemHandle(&h[1], l->c1.p));
    std::memcpy(handles128, h, sizeof h);
    return TK_OK;
}

int tk_land_open_peers(tk_land* l, const void* handles) {
    if (int st = check_land(l)) return st;
    if (!l->sharded) return fail(TK_ESTATE, "open_peers: call tk_land_set_shard first");
    TKC(set_dev(l));
    const auto* h = static_cast<const cudaIpcMemHandle_t*>(handles);
    for (int g = 0; g < l->shard_n; ++g) {
        if (g == l->shard_rank) continue;
        void* p0 = nullptr;
        void* p1 = nullptr;
        TKC(cudaIpcOpenMemHandle(&p0, h[2 * g], cudaIpcMemLazyEnablePeerAccess));
        l->ipc_opened.push_back(p0);
        TKC(cudaIpcOpenMemHandle(&p1, h[2 * g + 1], cudaIpcMemLazyEnablePeerAccess));
        l->ipc_opened.push_back(p1);
        l->peer_c0[g] = p0;
        l->peer_c1[g] = p1;
    }
    return TK_OK;
}

namespace {
int shard_ready(tk_land* l) {
    if (!l->sharded) return fail(TK_ESTATE, "shard call on an unsharded handle");
    if (!l->built || !l->staged) return fail(TK_ESTATE, "shard call before tk_ffg_build");
    for (int g = 0; g < l->shard_n; ++g)
        if (!l->peer_c0[g] || !l->peer_c1[g])
            return fail(TK_ESTATE, "shard peers not connected (tk_land_set_peer_ptrs / open_peers)");
    return TK_OK;
}

tk::ShardInfo shard_info(const tk_land* l) {
    tk::ShardInfo sh{};
    sh.nranks = l->shard_n;
    sh.self = l->shard_rank;
    sh.lo = static_cast<uint32_t>(l->shard_lo);
    sh.hi = static_cast<uint32_t>(l->shard_hi);
    sh.chunk_magic = l->shard_chunk == 1 ? 0ull : (~0ull / l->shard_chunk + 1ull);
    for (int g = 0; g < l->shard_n; ++g) {
        sh.peer_c[0][g] = static_cast<double*>(l->peer_c0[g]);
        sh.peer_c[1][g] = static_cast<double*>(l->peer_c1[g]);
    }
    // TK_SHARD_PUSH=edges: push c' only along out-edges (half the NVLink
    // volume, out-mask load + partial-sector stores); default: along every
    // crossing direction (Exchange volume)
    const char* e = std::getenv("TK_SHARD_PUSH");
    sh.edges_om = (e && std::strcmp(e, "edges") == 0) ? l->om.as<uint32_t>() : nullptr;
    return sh;
}

tk::PrArgs shard_pr_args(tk_land* l, double d) {
    tk::PrArgs a{};
    a.n = static_cast<uint32_t>(l->n);
    const double nd = static_cast<double>(l->n);
    a.inv_n = 1.0 / nd;
    a.nd = nd;
    a.teleport = (1.0 - d) / nd;
    a.damping = d;
    a.pw = l->pw.as<uint32_t>();
    a.r0 = l->r0.as<double>();
    a.r1 = l->r1.as<double>();
    a.c0 = l->c0.as<double>();
    a.c1 = l->c1.as<double>();
    return a;
}
}  // namespace

int tk_shard_optimum(tk_land* l, double* f, uint64_t* rank, int* has) {
    if (int st = check_land(l)) return st;
    if (int st = shard_ready(l)) return st;
    TKC(set_dev(l));
    Small* ds = l->small.as<Small>();
    TKC(cudaMemcpyAsync(&l->hsmall->f_opt, &ds->f_opt, 8 + 8 + 4, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    if (f) *f = l->hsmall->f_opt;
    if (rank) *rank = l->hsmall->rank;
    if (has) *has = l->hsmall->has;
    return TK_OK;
}

int tk_shard_pagerank_init(tk_land* l, double damping, double* dangling) {
    if (int st = check_land(l)) return st;
    if (int st = shard_ready(l)) return st;
    if (int st = check_pr_args(damping, 1.0, 1)) return st;
    TKC(set_dev(l));
    TKC(ensure(l->r0, (l->n + kPad) * 8));
    TKC(ensure(l->part, static_cast<size_t>(l->num_sms) * 4 * 3 * 8));
    Small* ds = l->small.as<Small>();
    tk::PrArgs a = shard_pr_args(l, damping);
    TKC(tk::launch_pagerank_shard_init(l->shape, shard_info(l), a, l->om.as<uint32_t>(),
                                       l->part.as<double>(), ds->totals_f, l->num_sms, l->stream));
    TKC(cudaMemcpyAsync(l->hsmall->totals_f, ds->totals_f, 24, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    if (dangling) *dangling = l->hsmall->totals_f[1];
    l->shard_cur = 0;
    l->shard_pr = true;
    l->shard_r_fresh = false;
    l->iterations = 0;
    return TK_OK;
}

int tk_shard_pagerank_step(tk_land* l, double dangling_total, double damping, double* residual,
                           double* dangling, double* sum) {
    if (int st = check_land(l)) return st;
    if (int st = shard_ready(l)) return st;
    if (!l->shard_pr) return fail(TK_ESTATE, "shard step before tk_shard_pagerank_init");
    TKC(set_dev(l));
    tk::StagePlan plan{};
    if (!tk::make_stage_plan(l->shape, true, stage_budget(l), &plan, false))
        return fail(TK_EINVAL, "shard step: no staging plan for this shape");
    Small* ds = l->small.as<Small>();
    tk::PrArgs a = shard_pr_args(l, damping);
    const double dn = dangling_total / static_cast<double>(l->n);
    TKC(tk::launch_pagerank_shard_step(l->shape, plan, shard_info(l), a,
                                       l->shard_cur, dn, l->part.as<double>(), ds->totals_f,
                                       l->num_sms, l->stream));
    TKC(cudaMemcpyAsync(l->hsmall->totals_f, ds->totals_f, 24, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    l->shard_cur ^= 1;
    l->shard_r_fresh = false;
    ++l->iterations;
    if (residual) *residual = l->hsmall->totals_f[0];
    if (dangling) *dangling = l->hsmall->totals_f[1];
    if (sum) *sum = l->hsmall->totals_f[2];
    return TK_OK;
}

// Device-side iteration control: the same init / step as
// above, enqueued on the handle's stream without any host synchronisation.
// Partials land in caller device memory (three doubles), so a collective can
// all-reduce them in place on that stream and the next step reads the reduced
// dangling mass from there; the host reads back only what its stop test needs.
int tk_shard_pagerank_init_dev(tk_land* l, double damping, double* d_partials) {
    if (int st = check_land(l)) return st;
    if (int st = shard_ready(l)) return st;
    if (int st = check_pr_args(damping, 1.0, 1)) return st;
    if (!d_partials) return fail(TK_EINVAL, "shard init: null partials buffer");
    TKC(set_dev(l));
    TKC(ensure(l->r0, (l->n + kPad) * 8));
    TKC(ensure(l->part, static_cast<size_t>(l->num_sms) * 4 * 3 * 8));
    TKC(cudaMemsetAsync(l->part.p, 0, static_cast<size_t>(l->num_sms) * 4 * 3 * 8, l->stream));
    tk::PrArgs a = shard_pr_args(l, damping);
    TKC(tk::launch_pagerank_shard_init(l->shape, shard_info(l), a, l->om.as<uint32_t>(),
                                       l->part.as<double>(), d_partials, l->num_sms, l->stream));
    l->shard_cur = 0;
    l->shard_pr = true;
    l->shard_r_fresh = false;
    l->iterations = 0;
    return TK_OK;
}

int tk_shard_pagerank_step_dev(tk_land* l, const double* d_totals, double damping,
                               double* d_partials) {
    if (int st = check_land(l)) return st;
    if (int st = shard_ready(l)) return st;
    if (!l->shard_pr) return fail(TK_ESTATE, "shard step before tk_shard_pagerank_init");
    if (!d_totals || !d_partials) return fail(TK_EINVAL, "shard step: null device buffer");
    TKC(set_dev(l));
    tk::StagePlan plan{};
    if (!tk::make_stage_plan(l->shape, true, stage_budget(l), &plan, false))
        return fail(TK_EINVAL, "shard step: no staging plan for this shape");
    tk::PrArgs a = shard_pr_args(l, damping);
    TKC(tk::launch_pagerank_shard_step(l->shape, plan, shard_info(l), a,
                                       l->shard_cur, 0.0, l->part.as<double>(), d_partials,
                                       l->num_sms, l->stream, d_totals));
    l->shard_cur ^= 1;
    l->shard_r_fresh = false;
    ++l->iterations;
    return TK_OK;
}

// Drop the last tk_shard_pagerank_step_dev (a speculative step issued before
// the previous step's stop test was read): its r' went to the other parity
// buffer, so the previous iterate is intact; only the bookkeeping rewinds.
int tk_shard_pagerank_rewind(tk_land* l) {
    if (int st = check_land(l)) return st;
    if (!l->shard_pr || l->iterations < 1) return fail(TK_ESTATE, "shard rewind: no step to drop");
    l->shard_cur ^= 1;
    l->shard_r_fresh = false;
    --l->iterations;
    return TK_OK;
}

int tk_shard_centrality(tk_land* l, double f_opt, const double* p, int n_p, double* nums,
                        double* den) {
    if (int st = check_land(l)) return st;
    if (int st = shard_ready(l)) return st;
    if (!l->shard_pr) return fail(TK_ESTATE, "shard centrality before PageRank");
    if (n_p < 1 || n_p > TK_MAX_CP) return fail(TK_EINVAL, "centrality: 1..101 values of p");
    TKC(set_dev(l));
    if (l->n_minima == 0) {
        for (int k = 0; k < n_p; ++k) nums[k] = 0.0;
        *den = 0.0;
        return TK_OK;
    }
    TKC(ensure(l->cp_part, static_cast<size_t>(TK_MAX_CP + 1) * tk::kCpBlocks * 8));
    TKC(ensure(l->cp_out, (TK_MAX_CP + 1) * 8));
    Small* ds = l->small.as<Small>();
    TKC(shard_refresh_r(l));
    const double* r = pr_result(l);
    TKC(tk::launch_centrality(l->minima.as<uint32_t>(), l->n_minima, l->fit.as<double>(), r, p, n_p,
                              f_opt, l->cp_part.as<double>(), l->cp_out.as<double>(),
                              &ds->degenerate, l->stream, true));
    TKC(cudaMemcpyAsync(nums, l->cp_out.p, static_cast<size_t>(n_p) * 8, cudaMemcpyDeviceToHost,
                        l->stream));
    TKC(cudaMemcpyAsync(den, l->cp_out.as<double>() + n_p, 8, cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    return TK_OK;
}

int tk_shard_pagerank_copy_out(tk_land* l, double* r_slice) {
    if (int st = check_land(l)) return st;
    if (!l->sharded || !l->shard_pr) return fail(TK_ESTATE, "no sharded PageRank state");
    TKC(set_dev(l));
    TKC(shard_refresh_r(l));
    const double* r = pr_result(l);
    TKC(cudaMemcpyAsync(r_slice, r + l->shard_lo, (l->shard_hi - l->shard_lo) * 8,
                        cudaMemcpyDeviceToHost, l->stream));
    TKC(cudaStreamSynchronize(l->stream));
    return TK_OK;
}

int tk_pagerank_csr(int device, uint64_t n, const uint64_t* offsets, const uint32_t* targets,
                    double damping, double tol, int64_t max_iter, double* r_out,
                    int64_t* iterations, double* residual) {
    if (n == 0) return fail(TK_EINVAL, "pagerank: empty graph");
    if (n > kMaxNodes) return fail(TK_ELIMIT, "pagerank: graph exceeds u32 node ids");
    if (!offsets || !r_out) return fail(TK_EINVAL, "pagerank: null buffer");
    int st = check_pr_args(damping, tol, max_iter);
    if (st) return st;
    const uint64_t e = offsets[n];
    if (e && !targets) return fail(TK_EINVAL, "pagerank: null targets");
    for (uint64_t i = 0; i < n; ++i)
        if (offsets[i] > offsets[i + 1]) return fail(TK_EINVAL, "pagerank: offsets not monotone");
    TK_GUARD_BEGIN
    int ndev = 0;
    TKC(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(TK_EINVAL, "no such CUDA device");
    TKC(cudaSetDevice(device));
    cudaDeviceProp prop;
    TKC(cudaGetDeviceProperties(&prop, device));
    cudaStream_t stream;
    TKC(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    DevBuf off, tg, odeg, indeg, in_off, src, status, counter, r0, r1, c0, c1, part, small;
    Small* hs = nullptr;
    auto cleanup = [&]() {
        cudaStreamSynchronize(stream);
        for (DevBuf* b : {&off, &tg, &odeg, &indeg, &in_off, &src, &status, &counter, &r0, &r1,
                          &c0, &c1, &part, &small})
            b->release();
        if (hs) cudaFreeHost(hs);
        cudaStreamDestroy(stream);
    };
    auto run = [&]() -> int {
        const uint32_t nn = static_cast<uint32_t>(n);
        const uint32_t ntiles = static_cast<uint32_t>((n + 255) / 256);
        TKC(ensure(off, (n + 1) * 8));
        TKC(ensure(tg, std::max<uint64_t>(e, 1) * 4));
        TKC(ensure(odeg, n * 4));
        TKC(ensure(indeg, n * 4));
        TKC(ensure(in_off, (n + 1) * 8));
        TKC(ensure(src, std::max<uint64_t>(e, 1) * 4));
        TKC(ensure(status, static_cast<size_t>(ntiles) * 8));
        TKC(ensure(counter, 16));
        TKC(ensure(r0, n * 8));
        TKC(ensure(r1, n * 8));
        TKC(ensure(c0, n * 8));
        TKC(ensure(c1, n * 8));
        TKC(ensure(small, sizeof(Small)));
        TKC(cudaMallocHost(&hs, sizeof(Small)));
        TKC(cudaMemcpyAsync(off.p, offsets, (n + 1) * 8, cudaMemcpyHostToDevice, stream));
        if (e) TKC(cudaMemcpyAsync(tg.p, targets, e * 4, cudaMemcpyHostToDevice, stream));
        TKC(cudaMemsetAsync(indeg.p, 0, n * 4, stream));
        TKC(cudaMemsetAsync(status.p, 0, static_cast<size_t>(ntiles) * 8, stream));
        TKC(cudaMemsetAsync(counter.p, 0, 16, stream));
        Small* ds = small.as<Small>();
        TKC(cudaMemsetAsync(&ds->err, 0, 4, stream));
        // target range check happens on the host: cheap, and keeps the kernel simple
        for (uint64_t i = 0; i < e; ++i)
            if (targets[i] >= n) return fail(TK_EINVAL, "pagerank: edge target out of range");
        TKC(tk::launch_csr_prepare(nn, off.as<unsigned long long>(), tg.as<uint32_t>(), e,
                                   odeg.as<uint32_t>(), indeg.as<uint32_t>(), stream));
        TKC(tk::launch_exclusive_scan_u32(indeg.as<uint32_t>(), nn, in_off.as<unsigned long long>(),
                                          status.as<unsigned long long>(),
                                          counter.as<unsigned int>(), ntiles,
                                          prop.multiProcessorCount, stream));
        TKC(cudaMemsetAsync(indeg.p, 0, n * 4, stream));  // reuse as scatter cursor
        TKC(tk::launch_csr_scatter(nn, off.as<unsigned long long>(), tg.as<uint32_t>(),
                                   in_off.as<unsigned long long>(), indeg.as<uint32_t>(),
                                   src.as<uint32_t>(), stream));
        TKC(tk::launch_csr_sort_rows(nn, in_off.as<unsigned long long>(), src.as<uint32_t>(),
                                     stream));
        tk::DevShape s{};
        s.n = nn;
        tk::PrArgs a{};
        a.n = nn;
        a.in_off = in_off.as<unsigned long long>();
        a.src = src.as<uint32_t>();
        a.odeg32 = odeg.as<uint32_t>();
        a.r0 = r0.as<double>();
        a.r1 = r1.as<double>();
        a.c0 = c0.as<double>();
        a.c1 = c1.as<double>();
        int rs = run_pagerank(device, prop.multiProcessorCount, s, tk::MODE_CSR, false, a, part,
                              ds, hs, stream, damping, tol, max_iter);
        if (rs) return rs;
        if (iterations) *iterations = hs->pr.iter;
        if (residual) *residual = hs->pr.res;
        if (hs->pr.status != 0) return nonconv(hs->pr.iter, hs->pr.res);
        TKC(cudaMemcpyAsync(r_out, hs->pr.parity ? r1.p : r0.p, n * 8, cudaMemcpyDeviceToHost,
                            stream));
        TKC(cudaStreamSynchronize(stream));
        return TK_OK;
    };
    st = run();
    cleanup();
    return st;
    TK_GUARD_END
}

int tk_proportion_of_centrality(int device, uint64_t n_minima, const double* min_fitness,
                                const double* min_pagerank, double f_opt, double p,
                                double* out) {
    if (!out) return fail(TK_EINVAL, "proportion_of_centrality: null out");
    if (n_minima == 0) return fail(TK_EDEGEN, "proportion_of_centrality: no local minima");
    if (!min_fitness || !min_pagerank) return fail(TK_EINVAL, "proportion_of_centrality: null buffer");
    TKC(cudaSetDevice(device));
    cudaStream_t stream;
    TKC(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    DevBuf f, r, part, cp, small;
    int deg = 0;
    auto run = [&]() -> int {
        TKC(ensure(f, n_minima * 8));
        TKC(ensure(r, n_minima * 8));
        TKC(ensure(part, 2 * tk::kCpBlocks * 8));
        TKC(ensure(cp, 8));
        TKC(ensure(small, sizeof(Small)));
        TKC(cudaMemcpyAsync(f.p, min_fitness, n_minima * 8, cudaMemcpyHostToDevice, stream));
        TKC(cudaMemcpyAsync(r.p, min_pagerank, n_minima * 8, cudaMemcpyHostToDevice, stream));
        Small* ds = small.as<Small>();
        TKC(tk::launch_centrality(nullptr, n_minima, f.as<double>(), r.as<double>(), &p, 1, f_opt,
                                  part.as<double>(), cp.as<double>(), &ds->degenerate, stream));
        TKC(cudaMemcpyAsync(out, cp.p, 8, cudaMemcpyDeviceToHost, stream));
        TKC(cudaMemcpyAsync(&deg, &ds->degenerate, 4, cudaMemcpyDeviceToHost, stream));
        TKC(cudaStreamSynchronize(stream));
        if (deg) return fail(TK_EDEGEN, "proportion_of_centrality: minima hold zero PageRank mass");
        return TK_OK;
    };
    int st = run();
    cudaStreamSynchronize(stream);
    for (DevBuf* b : {&f, &r, &part, &cp, &small}) b->release();
    cudaStreamDestroy(stream);
    return st;
}

}  // extern "C"
