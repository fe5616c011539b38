// cache_records.cpp -- analyze_cache_file: cache JSON -> valid-set records ->
// GPU hash-table ingestion (tk_land_load_configs) -> tk_analyze.
// Record semantics follow cache_io.cpp (/root/reference/proj/src/cache_io.cpp:
// 33-75): a record is ok iff it has a numeric "times" array or a numeric
// "time"; everything else, and every configuration without a record, is a
// failed node (kFailFitness).  Absent configurations are how constraints
// appear in a cache, so a partial cache is the normal input here.
#include <fstream>
#include <memory>
#include <vector>

#include "tk_landscape.h"
#include "tunekit/errors.hpp"
#include "tunekit_b200/extensions.hpp"

namespace tunekit {

namespace {

[[noreturn]] void raise(int st, long it = 0, double res = 0.0) {
    const std::string msg = tk_last_error();
    if (st == TK_EINVAL || st == TK_ELIMIT) throw InvalidArgument(msg);
    if (st == TK_ENOFEAS) throw NoFeasiblePoint(msg);
    if (st == TK_ENOCONV) throw NonConvergence(msg, it, res);
    throw Error(std::string(tk_status_name(st)) + ": " + msg);
}

ParameterSpace parse_space(const Json& j) {
    if (j.contains("space")) return ParameterSpace::from_json(j.at("space"));
    if (!j.contains("tune_params")) throw ParseError("cache file needs 'space' or 'tune_params'");
    std::vector<std::string> order;
    if (j.contains("tune_params_keys")) {
        for (const Json& k : j.at("tune_params_keys")) order.push_back(k.get<std::string>());
    } else {
        for (auto it = j.at("tune_params").begin(); it != j.at("tune_params").end(); ++it)
            order.push_back(it.key());
    }
    std::vector<Parameter> ps;
    for (const std::string& n : order) {
        Parameter p;
        p.name = n;
        for (const Json& v : j.at("tune_params").at(n)) p.values.push_back(value_from_json(v));
        ps.push_back(std::move(p));
    }
    return ParameterSpace(std::move(ps));
}

bool record_mean(const Json& e, double* mean) {
    if (!e.is_object()) return false;
    if (e.contains("times") && e.at("times").is_array() && !e.at("times").empty()) {
        double sum = 0.0;
        std::size_t n = 0;
        bool numeric = true;
        for (const Json& x : e.at("times")) {
            if (!x.is_number()) {
                numeric = false;
                break;
            }
            sum += x.get<double>();  // left-to-right, as SearchSpaceCache::set_ok
            ++n;
        }
        if (numeric) {
            *mean = sum / static_cast<double>(n);
            return true;
        }
    }
    if (e.contains("time") && e.at("time").is_number()) {
        *mean = e.at("time").get<double>();
        return true;
    }
    return false;
}

}  // namespace

CentralityReport analyze_cache_file(const std::string& path, NeighbourhoodKind kind,
                                    double damping, int p_max_percent, std::uint64_t node_limit,
                                    ParameterSpace* space_out) {
    std::ifstream in(path);
    if (!in) throw ParseError("cannot open cache file: " + path);
    Json j;
    try {
        in >> j;
    } catch (const std::exception& e) {
        throw ParseError("invalid JSON in " + path + ": " + e.what());
    }
    if (!j.is_object() || !j.contains("cache")) throw ParseError("cache file needs a 'cache' object");
    const ParameterSpace space = parse_space(j);
    const std::size_t dims = space.dims();
    std::vector<std::int32_t> configs;
    std::vector<double> fitness;
    std::uint64_t records = 0;
    for (auto it = j.at("cache").begin(); it != j.at("cache").end(); ++it) {
        Configuration x;
        try {
            x = space.config_from_key(it.key());
        } catch (const Error& e) {
            throw ParseError("cache key '" + it.key() + "': " + e.what());
        }
        ++records;
        double mean = 0.0;
        if (!record_mean(it.value(), &mean)) continue;
        configs.insert(configs.end(), x.begin(), x.end());
        fitness.push_back(mean);
    }
    // A configuration without a record is infeasible: Kernel Tuner never writes
    // the configurations its restrictions exclude, and the reference models
    // constraints as fail fitness (cache.cpp:9-16 leaves an absent
    // rank at kFailFitness, not ok).  The valid set is exactly the ok records.
    (void)records;
    if (space_out) *space_out = space;
    std::vector<std::uint32_t> radix(dims);
    for (std::size_t i = 0; i < dims; ++i) radix[i] = static_cast<std::uint32_t>(space.list_size(i));
    const char* dev = std::getenv("TK_DEVICE");
    tk_land* raw = nullptr;
    int st = tk_land_create(dev ? std::atoi(dev) : 0, static_cast<std::uint32_t>(dims), radix.data(),
                            &raw);
    if (st) raise(st);
    std::unique_ptr<tk_land, int (*)(tk_land*)> land(raw, tk_land_destroy);
    st = tk_land_load_configs(land.get(), configs.data(), fitness.data(), fitness.size(), TK_MEM_HOST);
    if (st) raise(st);
    tk_report_summary s{};
    st = tk_analyze(land.get(), kind == NeighbourhoodKind::Adjacent ? TK_ADJACENT : TK_HAMMING,
                    damping, 1e-10, 100000, node_limit, p_max_percent, 0, &s);
    if (st) raise(st, static_cast<long>(s.iterations), s.residual);
    CentralityReport rep;
    rep.kind = kind;
    rep.damping = damping;
    rep.f_opt = s.f_opt;
    rep.pagerank_iterations = static_cast<int>(s.iterations);
    rep.pagerank_sum = s.pagerank_sum;
    for (int k = 0; k < s.n_cp; ++k) rep.c_p_curve.emplace_back(k, s.c_p[k]);
    std::vector<std::uint64_t> ranks(s.n_minima);
    std::vector<double> f(s.n_minima), frac(s.n_minima), pr(s.n_minima);
    if (s.n_minima) {
        st = tk_report_copy_out(land.get(), s.f_opt, ranks.data(), f.data(), frac.data(), pr.data());
        if (st) raise(st);
    }
    for (std::uint64_t i = 0; i < s.n_minima; ++i) rep.minima.push_back({ranks[i], f[i], frac[i], pr[i]});
    return rep;
}

}  // namespace tunekit
