// landscape.cpp -- the drop-in implementation of tunekit/landscape.hpp
// (/root/reference/proj/include/tunekit/landscape.hpp:12-102 declares these
// and ships no definition).  Every FFG / PageRank / C_p computation runs on
// the GPU through the C-ABI of tk_landscape.h; this file only marshals the
// cache, maps status codes onto the reference's exceptions and shapes the
// results into the reference's structs.
//
// It is compiled against the reference's own proj/include/tunekit/ headers and
// linked with the reference's own host classes (value/space/cache/generators/
// cache_io .cpp, built where they lie -- cpp/Makefile): this repo ships only
// the landscape implementation, not copies of the reference's sources.
#include "tunekit/landscape.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <string>

#include "tk_landscape.h"
#include "tunekit/errors.hpp"
#include "tunekit_b200/extensions.hpp"

namespace tunekit {

namespace {

int device_index() {
    const char* e = std::getenv("TK_DEVICE");
    return e ? std::atoi(e) : 0;
}

[[noreturn]] void rethrow(int st, long iterations = 0, double residual = 0.0) {
    const std::string msg = tk_last_error();
    switch (st) {
        case TK_EINVAL:
        case TK_ELIMIT: throw InvalidArgument(msg);
        case TK_ENOFEAS: throw NoFeasiblePoint(msg);
        case TK_ENOCONV: throw NonConvergence(msg, iterations, residual);
        default: throw Error(std::string(tk_status_name(st)) + ": " + msg);
    }
}

void check(int st) {
    if (st != TK_OK) rethrow(st);
}

int kind_code(NeighbourhoodKind k) { return k == NeighbourhoodKind::Adjacent ? TK_ADJACENT : TK_HAMMING; }

struct LandDeleter {
    void operator()(tk_land* l) const { tk_land_destroy(l); }
};
using Land = std::unique_ptr<tk_land, LandDeleter>;

std::string limit_message(std::uint64_t n, std::uint64_t limit) {
    return "search space has " + std::to_string(n) +
           " configurations, above the FFG node limit of " + std::to_string(limit) +
           "; sample the space or raise node_limit";
}

// landscape analysis needs a complete cache.  Uploads the
// rank-indexed mean/ok tables (cache.hpp:42-48) to a fresh device handle.
Land upload(const SearchSpaceCache& cache) {
    if (!cache.complete())
        throw Error("landscape analysis needs a complete cache (" +
                    std::to_string(cache.present_count()) + " of " +
                    std::to_string(cache.size()) + " configurations present)");
    const ParameterSpace& s = cache.space();
    std::vector<std::uint32_t> radix(s.dims());
    for (std::size_t i = 0; i < s.dims(); ++i) radix[i] = static_cast<std::uint32_t>(s.list_size(i));
    tk_land* raw = nullptr;
    check(tk_land_create(device_index(), static_cast<std::uint32_t>(radix.size()), radix.data(), &raw));
    Land land(raw);
    const std::uint64_t n = cache.size();
    std::vector<double> fit(n);
    std::vector<std::uint8_t> ok(n);
    for (std::uint64_t r = 0; r < n; ++r) {
        fit[r] = cache.mean(r);
        ok[r] = cache.ok(r) ? 1 : 0;
    }
    check(tk_land_load_dense(land.get(), fit.data(), ok.data(), TK_MEM_HOST));
    return land;
}

std::vector<double> fitness_of(const SearchSpaceCache& cache) {
    std::vector<double> f(cache.size());
    for (std::uint64_t r = 0; r < cache.size(); ++r) f[r] = cache.mean(r);
    return f;
}

}  // namespace

// landscape.hpp:24 -- strict census
PointCensus classify_points(const SearchSpaceCache& cache, NeighbourhoodKind kind) {
    Land land = upload(cache);
    check(tk_ffg_build(land.get(), kind_code(kind), std::numeric_limits<std::uint64_t>::max(), 0,
                       nullptr, nullptr));
    PointCensus c;
    c.kind = kind;
    c.total = cache.size();
    check(tk_census(land.get(), &c.fail_points, &c.local_minima, &c.interior, nullptr));
    c.minima_ranks.resize(c.local_minima);
    if (c.local_minima)
        check(tk_census(land.get(), &c.fail_points, &c.local_minima, &c.interior,
                        c.minima_ranks.data()));
    return c;
}

// landscape.hpp:44-45
FitnessFlowGraph build_ffg(const SearchSpaceCache& cache, NeighbourhoodKind kind,
                           std::uint64_t node_limit) {
    if (cache.size() > node_limit) throw InvalidArgument(limit_message(cache.size(), node_limit));
    Land land = upload(cache);
    std::uint64_t e = 0, m = 0;
    check(tk_ffg_build(land.get(), kind_code(kind), node_limit, 1, &e, &m));
    FitnessFlowGraph g;
    g.kind = kind;
    g.node_count = static_cast<std::uint32_t>(cache.size());
    g.offsets.resize(cache.size() + 1);
    g.targets.resize(e);
    g.is_sink.resize(cache.size());
    g.minima.resize(m);
    check(tk_ffg_copy_out(land.get(), g.offsets.data(), g.targets.data(), g.is_sink.data(),
                          g.minima.data()));
    g.fitness = fitness_of(cache);
    return g;
}

// landscape.hpp:51-52 -- any out-CSR; transposed and iterated on the GPU
std::vector<double> pagerank(const FitnessFlowGraph& g, double damping, double tol, int max_iter) {
    const std::uint64_t n = g.node_count;
    if (n == 0 || g.offsets.size() != n + 1)
        throw InvalidArgument("pagerank: graph needs node_count + 1 offsets and at least one node");
    std::vector<double> r(n);
    std::int64_t it = 0;
    double res = 0.0;
    const int st = tk_pagerank_csr(device_index(), n, g.offsets.data(),
                                   g.targets.empty() ? nullptr : g.targets.data(), damping, tol,
                                   max_iter, r.data(), &it, &res);
    if (st != TK_OK) rethrow(st, static_cast<long>(it), res);
    return r;
}

// landscape.hpp:56-58 (SURVEY.md A8 threshold rule)
double proportion_of_centrality(const FitnessFlowGraph& g, const std::vector<double>& pr,
                                double f_opt, double p) {
    if (pr.size() != g.node_count) throw InvalidArgument("pagerank vector size != node_count");
    if (g.fitness.size() != g.node_count) throw InvalidArgument("graph carries no fitness table");
    std::vector<double> mf(g.minima.size()), mp(g.minima.size());
    for (std::size_t i = 0; i < g.minima.size(); ++i) {
        mf[i] = g.fitness[g.minima[i]];
        mp[i] = pr[g.minima[i]];
    }
    double out = 0.0;
    check(tk_proportion_of_centrality(device_index(), mf.size(), mf.data(), mp.data(), f_opt, p, &out));
    return out;
}

// landscape.hpp:77-79, with the node limit of build_ffg's default
// (SURVEY.md A9); analyze_landscape_limited lifts it.
CentralityReport analyze_landscape_limited(const SearchSpaceCache& cache, NeighbourhoodKind kind,
                                           double damping, int p_max_percent,
                                           std::uint64_t node_limit) {
    if (cache.size() > node_limit) throw InvalidArgument(limit_message(cache.size(), node_limit));
    Land land = upload(cache);
    tk_report_summary s{};
    const int st = tk_analyze(land.get(), kind_code(kind), damping, 1e-10, 100000, node_limit,
                              p_max_percent, 0, &s);
    if (st != TK_OK) rethrow(st, static_cast<long>(s.iterations), s.residual);
    CentralityReport rep;
    rep.kind = kind;
    rep.damping = damping;
    rep.f_opt = s.f_opt;
    rep.pagerank_iterations = static_cast<int>(s.iterations);
    rep.pagerank_sum = s.pagerank_sum;
    for (int k = 0; k < s.n_cp; ++k) rep.c_p_curve.emplace_back(k, s.c_p[k]);
    const std::uint64_t m = s.n_minima;
    std::vector<std::uint64_t> ranks(m);
    std::vector<double> fit(m), frac(m), prv(m);
    if (m)
        check(tk_report_copy_out(land.get(), s.f_opt, ranks.data(), fit.data(), frac.data(),
                                 prv.data()));
    rep.minima.reserve(m);
    for (std::uint64_t i = 0; i < m; ++i) rep.minima.push_back({ranks[i], fit[i], frac[i], prv[i]});
    return rep;
}

CentralityReport analyze_landscape(const SearchSpaceCache& cache, NeighbourhoodKind kind,
                                   double damping, int p_max_percent) {
    return analyze_landscape_limited(cache, kind, damping, p_max_percent, 1'000'000);
}

// landscape.hpp:87-94: f_opt / f over the FFG minima
MinimaFractionReport minima_fraction_report(const SearchSpaceCache& cache, NeighbourhoodKind kind) {
    Land land = upload(cache);
    std::uint64_t e = 0, m = 0;
    check(tk_ffg_build(land.get(), kind_code(kind), std::numeric_limits<std::uint64_t>::max(), 0,
                       &e, &m));
    double f_opt = 0.0;
    std::uint64_t orank = 0;
    check(tk_optimum(land.get(), &f_opt, &orank));
    std::vector<std::uint32_t> mins(m);
    if (m) check(tk_ffg_copy_out(land.get(), nullptr, nullptr, nullptr, mins.data()));
    MinimaFractionReport rep;
    rep.fractions.reserve(m);
    for (std::uint32_t r : mins) rep.fractions.push_back(f_opt / cache.mean(r));
    std::sort(rep.fractions.begin(), rep.fractions.end());
    if (!rep.fractions.empty()) {
        const std::size_t k = rep.fractions.size();
        rep.median = k % 2 ? rep.fractions[k / 2]
                           : 0.5 * (rep.fractions[k / 2 - 1] + rep.fractions[k / 2]);
        double sum = 0.0;
        for (double f : rep.fractions) sum += f;
        rep.mean = sum / static_cast<double>(k);
    }
    return rep;
}

}  // namespace tunekit

namespace tunekit {

// SURVEY.md s8(f) row 3 over tk_descents (include/tk_landscape.h)
DescentReport random_descents(const SearchSpaceCache& cache, NeighbourhoodKind kind,
                              std::uint64_t walkers, std::uint64_t seed, bool restart_scan) {
    Land land = upload(cache);
    std::uint64_t e = 0, m = 0;
    check(tk_ffg_build(land.get(), kind_code(kind), std::numeric_limits<std::uint64_t>::max(), 0,
                       &e, &m));
    DescentReport rep;
    std::vector<std::uint32_t> mins(m);
    if (m) check(tk_ffg_copy_out(land.get(), nullptr, nullptr, nullptr, mins.data()));
    rep.minima.assign(mins.begin(), mins.end());
    rep.arrivals.resize(m);
    check(tk_descents(land.get(), walkers, seed, restart_scan ? 1 : 0,
                      m ? rep.arrivals.data() : nullptr, &rep.fail_arrivals, &rep.evaluations));
    return rep;
}

}  // namespace tunekit

namespace tunekit {

std::vector<CentralityReport> analyze_landscapes(const std::vector<const SearchSpaceCache*>& caches,
                                                 NeighbourhoodKind kind, double damping,
                                                 int p_max_percent) {
    const std::size_t n = caches.size();
    std::vector<CentralityReport> out(n);
    std::vector<tk_batch_item> items(n);
    std::vector<std::vector<double>> fit(n);
    std::vector<std::vector<std::uint8_t>> ok(n);
    std::vector<std::vector<std::uint64_t>> ranks(n);
    std::vector<std::vector<double>> fmin(n), frac(n), prv(n);
    std::vector<bool> batched(n, false);
    for (std::size_t k = 0; k < n; ++k) {
        const SearchSpaceCache& c = *caches[k];
        if (!c.complete())
            throw Error("landscape analysis needs a complete cache (" +
                        std::to_string(c.present_count()) + " of " + std::to_string(c.size()) +
                        " configurations present)");
        const ParameterSpace& s = c.space();
        tk_batch_item& it = items[k];
        std::memset(&it, 0, sizeof(it));
        std::uint64_t slots = 0;
        it.dims = static_cast<std::uint32_t>(s.dims());
        for (std::size_t i = 0; i < s.dims(); ++i) {
            it.radix[i] = static_cast<std::uint32_t>(s.list_size(i));
            if (it.radix[i] >= 2) slots += kind == NeighbourhoodKind::Adjacent ? 2 : it.radix[i] - 1;
        }
        if (c.size() > 1'000'000) throw InvalidArgument(limit_message(c.size(), 1'000'000));
        batched[k] = s.dims() <= TK_MAX_DIMS && c.size() <= (1ull << 20) && slots <= 64;
        if (!batched[k]) continue;
        fit[k].resize(c.size());
        ok[k].resize(c.size());
        for (std::uint64_t r = 0; r < c.size(); ++r) {
            fit[k][r] = c.mean(r);
            ok[k][r] = c.ok(r) ? 1 : 0;
        }
        // room for every possible minimum: the count is only known afterwards
        ranks[k].resize(c.size());
        fmin[k].resize(c.size());
        frac[k].resize(c.size());
        prv[k].resize(c.size());
        it.fitness = fit[k].data();
        it.ok = ok[k].data();
        it.minima_ranks = ranks[k].data();
        it.minima_fitness = fmin[k].data();
        it.minima_fraction = frac[k].data();
        it.minima_pagerank = prv[k].data();
        it.minima_capacity = c.size();
    }
    std::vector<tk_batch_item> live;
    std::vector<std::size_t> idx;
    for (std::size_t k = 0; k < n; ++k)
        if (batched[k]) {
            live.push_back(items[k]);
            idx.push_back(k);
        }
    if (!live.empty())
        check(tk_batch_analyze(device_index(), live.data(), static_cast<std::uint32_t>(live.size()),
                               kind_code(kind), damping, 1e-10, 100000, p_max_percent,
                               TK_MEM_HOST));
    for (std::size_t j = 0; j < live.size(); ++j) {
        const std::size_t k = idx[j];
        const tk_batch_item& it = live[j];
        const tk_report_summary& s = it.summary;
        if (it.status != TK_OK) {
            if (it.status == TK_ENOFEAS) throw NoFeasiblePoint("no feasible point in cache " + std::to_string(k));
            if (it.status == TK_ENOCONV)
                throw NonConvergence("pagerank did not converge", static_cast<long>(s.iterations), s.residual);
            throw Error("proportion_of_centrality: minima hold zero PageRank mass (cache " +
                        std::to_string(k) + ")");
        }
        CentralityReport& rep = out[k];
        rep.kind = kind;
        rep.damping = damping;
        rep.f_opt = s.f_opt;
        rep.pagerank_iterations = static_cast<int>(s.iterations);
        rep.pagerank_sum = s.pagerank_sum;
        for (int p = 0; p < s.n_cp; ++p) rep.c_p_curve.emplace_back(p, s.c_p[p]);
        rep.minima.reserve(s.n_minima);
        for (std::uint64_t i = 0; i < s.n_minima; ++i)
            rep.minima.push_back({ranks[k][i], fmin[k][i], frac[k][i], prv[k][i]});
    }
    for (std::size_t k = 0; k < n; ++k)
        if (!batched[k]) out[k] = analyze_landscape(*caches[k], kind, damping, p_max_percent);
    return out;
}

}  // namespace tunekit
