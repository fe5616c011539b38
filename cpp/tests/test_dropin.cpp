// test_dropin -- drives the C++ drop-in (tunekit/landscape.hpp over the C-ABI)
// on a GPU the way a reference user would -- built against the reference's own
// headers and host classes (cpp/Makefile) -- and dumps every result for
// tests/test_cpp_dropin.py to compare with the CPU oracle:
//   test_dropin <outdir> <q> <profile> <seed> <m0> <m1> ...
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "tunekit/errors.hpp"
#include "tunekit/generators.hpp"
#include "tunekit/landscape.hpp"
#include "tunekit_b200/extensions.hpp"

using namespace tunekit;

template <typename T>
static void dump(const std::string& path, const std::vector<T>& v) {
    std::ofstream o(path, std::ios::binary);
    o.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

static int fails = 0;
#define EXPECT(cond)                                                        \
    do {                                                                    \
        if (!(cond)) {                                                      \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++fails;                                                        \
        }                                                                   \
    } while (0)

int main(int argc, char** argv) {
    if (argc < 6) return 2;
    const std::string dir = argv[1];
    const double q = std::atof(argv[2]);
    const SyntheticProfile prof = synthetic_profile(argv[3]);
    const std::uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    std::vector<Parameter> ps;
    for (int i = 5; i < argc; ++i) {
        Parameter p;
        p.name = "p" + std::to_string(i - 5);
        for (int v = 0; v < std::atoi(argv[i]); ++v) p.values.push_back(std::int64_t{v * 16});
        ps.push_back(std::move(p));
    }
    const ParameterSpace space(std::move(ps));
    const SearchSpaceCache cache = generate_synthetic_kernel_space(space, q, prof, seed);

    for (NeighbourhoodKind kind : {NeighbourhoodKind::Hamming, NeighbourhoodKind::Adjacent}) {
        const std::string k = to_string(kind);
        const FitnessFlowGraph g = build_ffg(cache, kind);
        dump(dir + "/ffg_" + k + "_offsets.bin", g.offsets);
        dump(dir + "/ffg_" + k + "_targets.bin", g.targets);
        dump(dir + "/ffg_" + k + "_is_sink.bin", g.is_sink);
        dump(dir + "/ffg_" + k + "_minima.bin", g.minima);
        const std::vector<double> pr = pagerank(g);
        dump(dir + "/pr_" + k + ".bin", pr);
        std::ofstream cp(dir + "/cp_" + k + ".txt");
        for (int pct = 0; pct <= 15; ++pct)
            cp << pct << ' ' << std::hexfloat
               << proportion_of_centrality(g, pr, cache.optimum(), pct / 100.0) << '\n';
        const CentralityReport rep = analyze_landscape(cache, kind);
        std::ofstream(dir + "/report_" + k + ".json") << centrality_report_to_json(rep, cache).dump(1);
        std::ofstream mcsv(dir + "/minima_" + k + ".csv");
        write_minima_csv(rep, cache, mcsv);
        std::ofstream ccsv(dir + "/cpcurve_" + k + ".csv");
        write_cp_curve_csv(rep, ccsv);
        const PointCensus c = classify_points(cache, kind);
        std::ofstream cen(dir + "/census_" + k + ".txt");
        cen << c.total << ' ' << c.fail_points << ' ' << c.local_minima << ' ' << c.interior << '\n';
        dump(dir + "/census_" + k + "_ranks.bin", c.minima_ranks);
        const MinimaFractionReport mf = minima_fraction_report(cache, kind);
        std::ofstream fr(dir + "/fraction_" + k + ".txt");
        fr << std::hexfloat << mf.median << ' ' << mf.mean << ' ' << mf.fractions.size() << '\n';
        dump(dir + "/fraction_" + k + ".bin", mf.fractions);
        const DescentReport dr = random_descents(cache, kind, 100000, 7);
        dump(dir + "/descents_" + k + "_arrivals.bin", dr.arrivals);
        {
            std::ofstream df(dir + "/descents_" + k + ".txt");
            df << dr.fail_arrivals << ' ' << dr.evaluations << '\n';
        }
        EXPECT(dr.minima.size() == g.minima.size());
        EXPECT(rep.minima.size() == g.minima.size());
        EXPECT(mf.fractions.size() == g.minima.size());
        if (kind == NeighbourhoodKind::Adjacent) {
            for (GraphFormat f : {GraphFormat::Dot, GraphFormat::GraphML, GraphFormat::EdgeCsv}) {
                std::ostringstream os;
                export_graph(g, cache, f, os);
                const char* ext = f == GraphFormat::Dot ? "dot" : f == GraphFormat::GraphML ? "graphml" : "csv";
                std::ofstream(dir + "/graph." + ext) << os.str();
            }
        }
    }

    // analyze_landscapes (extensions.hpp): the batched device path against the
    // per-space one, for three caches (two spaces)
    {
        std::vector<Parameter> ps2;
        for (int i = 0; i < 4; ++i) {
            Parameter p;
            p.name = "q" + std::to_string(i);
            for (int v = 0; v < 5 + i; ++v) p.values.push_back(std::int64_t{v});
            ps2.push_back(std::move(p));
        }
        const SearchSpaceCache other =
            generate_synthetic_kernel_space(ParameterSpace(std::move(ps2)), 0.2, prof, seed + 1);
        const std::vector<const SearchSpaceCache*> cs = {&cache, &other, &cache};
        for (NeighbourhoodKind kind : {NeighbourhoodKind::Hamming, NeighbourhoodKind::Adjacent}) {
            const std::vector<CentralityReport> reps = analyze_landscapes(cs, kind);
            EXPECT(reps.size() == 3);
            for (std::size_t k = 0; k < cs.size(); ++k) {
                const CentralityReport one = analyze_landscape(*cs[k], kind);
                const CentralityReport& b = reps[k];
                EXPECT(b.pagerank_iterations == one.pagerank_iterations);
                EXPECT(b.minima.size() == one.minima.size());
                EXPECT(b.f_opt == one.f_opt);
                for (std::size_t i = 0; i < b.minima.size() && i < one.minima.size(); ++i) {
                    EXPECT(b.minima[i].rank == one.minima[i].rank);
                    EXPECT(b.minima[i].fitness == one.minima[i].fitness);
                    EXPECT(b.minima[i].fraction_of_optimum == one.minima[i].fraction_of_optimum);
                    EXPECT(std::abs(b.minima[i].pagerank - one.minima[i].pagerank) <= 1e-12);
                }
                for (std::size_t p = 0; p < b.c_p_curve.size(); ++p)
                    EXPECT(std::abs(b.c_p_curve[p].second - one.c_p_curve[p].second) <= 1e-9);
            }
        }
    }

    // error behaviour (errors.hpp:10-44 classes)
    try {
        build_ffg(cache, NeighbourhoodKind::Adjacent, cache.size() - 1);
        EXPECT(false);
    } catch (const InvalidArgument&) {
    }
    try {
        analyze_landscape_limited(cache, NeighbourhoodKind::Adjacent, 0.85, 15, cache.size() - 1);
        EXPECT(false);
    } catch (const InvalidArgument&) {
    }
    try {
        pagerank(build_ffg(cache, NeighbourhoodKind::Adjacent), 0.85, 1e-10, 2);
        EXPECT(false);
    } catch (const NonConvergence& e) {
        EXPECT(e.iterations == 2 && e.residual > 0);
    }
    try {
        pagerank(build_ffg(cache, NeighbourhoodKind::Adjacent), 1.5);
        EXPECT(false);
    } catch (const InvalidArgument&) {
    }
    try {
        graph_format_from_string("svg");
        EXPECT(false);
    } catch (const InvalidArgument&) {
    }
    {
        SearchSpaceCache dead(ParameterSpace({Parameter{"a", {std::int64_t{1}, std::int64_t{2}}}}),
                              CacheMetadata{});
        dead.set_failed(0);
        dead.set_failed(1);
        dead.finalize(true);
        try {
            analyze_landscape(dead, NeighbourhoodKind::Adjacent);
            EXPECT(false);
        } catch (const NoFeasiblePoint&) {
        }
    }
    {
        SearchSpaceCache partial(space, CacheMetadata{});
        partial.set_ok_mean(0, 1.0);
        partial.finalize(false);
        try {
            build_ffg(partial, NeighbourhoodKind::Adjacent);
            EXPECT(false);
        } catch (const Error&) {
        }
    }
    std::printf(fails ? "FAILED %d\n" : "OK\n", fails);
    return fails ? 1 : 0;
}
