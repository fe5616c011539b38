// tk_analyze -- the `analyze` command of the reference's CLI (SPEC.md:550-555,
// not shipped by the reference) on the B200 path.
//
//   tk_analyze <cache.json> [--neighbourhood adjacent|hamming] [--damping D]
//              [--p-max P] [--node-limit N] [--device-ingest]
//              [--json FILE] [--minima-csv FILE] [--curve-csv FILE]
//
// Default: load_cache -> analyze_landscape (the reference's stack A, SURVEY.md
// s3).  --device-ingest: analyze_cache_file (valid-set records hashed on the
// GPU).  Exit codes follow errors.hpp:8-9: Error -> 1, InvalidArgument -> 2.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>

#include "tunekit/cache_io.hpp"
#include "tunekit/errors.hpp"
#include "tunekit/landscape.hpp"
#include "tunekit_b200/extensions.hpp"

using namespace tunekit;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: tk_analyze <cache.json> [options]\n");
        return 2;
    }
    std::string path = argv[1], json_out, minima_csv, curve_csv;
    NeighbourhoodKind kind = NeighbourhoodKind::Adjacent;
    double damping = 0.85;
    int p_max = 15;
    unsigned long long node_limit = 1'000'000;
    bool device_ingest = false;
    try {
        for (int i = 2; i < argc; ++i) {
            const std::string a = argv[i];
            auto next = [&]() -> std::string {
                if (i + 1 >= argc) throw InvalidArgument("missing value after " + a);
                return argv[++i];
            };
            if (a == "--neighbourhood") kind = neighbourhood_from_string(next());
            else if (a == "--damping") damping = std::stod(next());
            else if (a == "--p-max") p_max = std::stoi(next());
            else if (a == "--node-limit") node_limit = std::stoull(next());
            else if (a == "--device-ingest") device_ingest = true;
            else if (a == "--json") json_out = next();
            else if (a == "--minima-csv") minima_csv = next();
            else if (a == "--curve-csv") curve_csv = next();
            else throw InvalidArgument("unknown option " + a);
        }
        CentralityReport rep;
        SearchSpaceCache cache;
        if (device_ingest) {
            ParameterSpace space;
            rep = analyze_cache_file(path, kind, damping, p_max, node_limit, &space);
            cache = SearchSpaceCache(space, CacheMetadata{});
        } else {
            cache = load_cache(path);
            rep = analyze_landscape_limited(cache, kind, damping, p_max, node_limit);
        }
        const Json j = centrality_report_to_json(rep, cache);
        if (!json_out.empty()) std::ofstream(json_out) << j.dump(1) << '\n';
        if (!minima_csv.empty()) {
            std::ofstream o(minima_csv);
            write_minima_csv(rep, cache, o);
        }
        if (!curve_csv.empty()) {
            std::ofstream o(curve_csv);
            write_cp_curve_csv(rep, o);
        }
        std::printf("minima=%zu iterations=%d f_opt=%.17g C_0=%.9f C_%d=%.9f\n", rep.minima.size(),
                    rep.pagerank_iterations, rep.f_opt, rep.c_p_curve.front().second, p_max,
                    rep.c_p_curve.back().second);
        return 0;
    } catch (const InvalidArgument& e) {
        std::fprintf(stderr, "tk_analyze: %s\n", e.what());
        return 2;
    } catch (const Error& e) {
        std::fprintf(stderr, "tk_analyze: %s\n", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "tk_analyze: %s\n", e.what());
        return 2;
    }
}
