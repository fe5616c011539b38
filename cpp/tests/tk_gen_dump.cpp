// tk_gen_dump -- CPU-only probe of the drop-in host classes, used by
// tests/test_cpp_dropin.py to pin them against the golden fixtures of the
// reference's own build:
//   tk_gen_dump synthetic <q> <profile> <seed> <m0> <m1> ...   -> fitness f64[N], ok u8[N]
//   tk_gen_dump nk <n> <k> <seed>                                -> fitness f64[2^n]
//   tk_gen_dump neighbours <kind 0|1> <m0> <m1> ...              -> counts u32[N], ranks u64[]
//   tk_gen_dump optimum <q> <profile> <seed> <m0> ...            -> "f_opt_hex rank" (text)
// Binary output goes to stdout.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "tunekit/cache_io.hpp"
#include "tunekit/errors.hpp"
#include "tunekit/generators.hpp"

using namespace tunekit;

static ParameterSpace space_from(int argc, char** argv, int first) {
    std::vector<Parameter> ps;
    for (int i = first; i < argc; ++i) {
        Parameter p;
        p.name = "p" + std::to_string(i - first);
        const int m = std::atoi(argv[i]);
        for (int v = 0; v < m; ++v) p.values.push_back(std::int64_t{v});
        ps.push_back(std::move(p));
    }
    return ParameterSpace(std::move(ps));
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string mode = argv[1];
    try {
        if (mode == "synthetic" || mode == "optimum") {
            const double q = std::atof(argv[2]);
            const SyntheticProfile prof = synthetic_profile(argv[3]);
            const std::uint64_t seed = std::strtoull(argv[4], nullptr, 10);
            SearchSpaceCache c = generate_synthetic_kernel_space(space_from(argc, argv, 5), q, prof, seed);
            if (mode == "optimum") {
                std::printf("%a %llu\n", c.optimum(), static_cast<unsigned long long>(c.optimum_rank()));
                return 0;
            }
            std::vector<double> f(c.size());
            std::vector<std::uint8_t> ok(c.size());
            for (std::uint64_t r = 0; r < c.size(); ++r) {
                f[r] = c.mean(r);
                ok[r] = c.ok(r);
            }
            std::fwrite(f.data(), 8, f.size(), stdout);
            std::fwrite(ok.data(), 1, ok.size(), stdout);
            return 0;
        }
        if (mode == "loadcache") {  // tk_gen_dump loadcache <path> -> f64 fit, u8 ok, u8 present
            SearchSpaceCache c = load_cache(argv[2]);
            for (std::uint64_t r = 0; r < c.size(); ++r) {
                const double v = c.mean(r);
                std::fwrite(&v, 8, 1, stdout);
            }
            for (std::uint64_t r = 0; r < c.size(); ++r) {
                const std::uint8_t o = c.present(r) && c.ok(r);
                std::fwrite(&o, 1, 1, stdout);
            }
            for (std::uint64_t r = 0; r < c.size(); ++r) {
                const std::uint8_t p = c.present(r);
                std::fwrite(&p, 1, 1, stdout);
            }
            return 0;
        }
        if (mode == "savecache") {  // tk_gen_dump savecache <path> <q> <profile> <seed> <m0> ...
            SearchSpaceCache c = generate_synthetic_kernel_space(
                space_from(argc, argv, 6), std::atof(argv[3]), synthetic_profile(argv[4]),
                std::strtoull(argv[5], nullptr, 10));
            save_cache(c, argv[2]);
            return 0;
        }
        if (mode == "nk") {
            SearchSpaceCache c = generate_nk_landscape(std::atoi(argv[2]), std::atoi(argv[3]),
                                                       std::strtoull(argv[4], nullptr, 10));
            for (std::uint64_t r = 0; r < c.size(); ++r) {
                const double v = c.mean(r);
                std::fwrite(&v, 8, 1, stdout);
            }
            return 0;
        }
        if (mode == "neighbours") {
            const NeighbourhoodKind kind = std::atoi(argv[2]) ? NeighbourhoodKind::Adjacent
                                                              : NeighbourhoodKind::Hamming;
            ParameterSpace s = space_from(argc, argv, 3);
            std::vector<std::uint32_t> counts(s.size());
            std::vector<std::uint64_t> all, nb;
            for (std::uint64_t r = 0; r < s.size(); ++r) {
                s.neighbour_ranks(r, kind, nb);
                counts[r] = static_cast<std::uint32_t>(nb.size());
                all.insert(all.end(), nb.begin(), nb.end());
                // the Configuration-based path must agree with the rank path
                const auto cfgs = s.neighbours(s.config_at(r), kind);
                for (std::size_t i = 0; i < cfgs.size(); ++i)
                    if (s.rank_of(cfgs[i]) != nb[i]) return 3;
            }
            std::fwrite(counts.data(), 4, counts.size(), stdout);
            std::fwrite(all.data(), 8, all.size(), stdout);
            return 0;
        }
    } catch (const NoFeasiblePoint& e) {
        std::fprintf(stderr, "NoFeasiblePoint: %s\n", e.what());
        return 4;
    } catch (const Error& e) {
        std::fprintf(stderr, "Error: %s\n", e.what());
        return 1;
    }
    return 2;
}
