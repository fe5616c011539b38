// ref_shim.cpp -- extern "C" probes into the reference's OWN compiled code.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/ from
// the reference sources where they lie (/root/reference/proj/src/{value,space,
// cache,generators}.cpp), never copied.  Used to generate the golden fixtures
// in tests/golden/ that pin the oracle restatement (oracle.c):
//   * neighbour order        -> ParameterSpace::neighbour_ranks (space.cpp:167-187)
//   * rank arithmetic        -> ParameterSpace strides/config_at (space.cpp:48-88)
//   * synthetic inputs       -> generate_synthetic_kernel_space (generators.cpp:89-145)
//                               generate_nk_landscape (generators.cpp:25-79)
//   * f_opt                  -> SearchSpaceCache::finalize/optimum (cache.cpp:55-98)
//   * FFG edge lists         -> the intended build_ffg loop (SURVEY.md s3 stack A,
//                               HOT LOOP 1) driven entirely by the reference's
//                               neighbour_ranks and SearchSpaceCache::mean/ok.
// The reference ships no landscape.cpp, so the FFG loop body below (a strict
// comparison and a push_back) is the only non-reference code on that path.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "tunekit/cache.hpp"
#include "tunekit/cache_io.hpp"
#include "tunekit/errors.hpp"
#include "tunekit/generators.hpp"
#include "tunekit/space.hpp"

using namespace tunekit;

namespace {
ParameterSpace make_space(std::uint32_t dims, const std::uint32_t* radix) {
    std::vector<Parameter> ps(dims);
    for (std::uint32_t i = 0; i < dims; ++i) {
        ps[i].name = "p" + std::to_string(i);
        for (std::uint32_t v = 0; v < radix[i]; ++v)
            ps[i].values.push_back(static_cast<std::int64_t>(v));
    }
    return ParameterSpace(std::move(ps));
}
NeighbourhoodKind nk(int kind) {
    return kind == 0 ? NeighbourhoodKind::Hamming : NeighbourhoodKind::Adjacent;
}
SearchSpaceCache make_cache(std::uint32_t dims, const std::uint32_t* radix,
                            const double* fit, const std::uint8_t* ok) {
    SearchSpaceCache c(make_space(dims, radix), CacheMetadata{});
    for (std::uint64_t r = 0; r < c.size(); ++r) {
        if (ok[r]) c.set_ok_mean(r, fit[r]);
        else c.set_failed(r);
    }
    c.finalize(true);
    return c;
}
}  // namespace

extern "C" {

std::uint64_t ref_space_size(std::uint32_t dims, const std::uint32_t* radix,
                             std::uint64_t* strides) {
    ParameterSpace s = make_space(dims, radix);
    for (std::uint32_t i = 0; i < dims; ++i) strides[i] = s.stride(i);
    return s.size();
}

std::uint32_t ref_neighbour_ranks(std::uint32_t dims, const std::uint32_t* radix,
                                  std::uint64_t rank, int kind, std::uint64_t* out) {
    static thread_local std::vector<std::uint64_t> nb;
    ParameterSpace s = make_space(dims, radix);
    s.neighbour_ranks(rank, nk(kind), nb);
    std::memcpy(out, nb.data(), nb.size() * sizeof(std::uint64_t));
    return static_cast<std::uint32_t>(nb.size());
}

// All neighbour lists of a space, concatenated in rank order (fixture dump).
std::uint64_t ref_all_neighbours(std::uint32_t dims, const std::uint32_t* radix, int kind,
                                 std::uint64_t* out, std::uint32_t* counts) {
    ParameterSpace s = make_space(dims, radix);
    std::vector<std::uint64_t> nb;
    std::uint64_t k = 0;
    for (std::uint64_t r = 0; r < s.size(); ++r) {
        s.neighbour_ranks(r, nk(kind), nb);
        counts[r] = static_cast<std::uint32_t>(nb.size());
        for (auto v : nb) out[k++] = v;
    }
    return k;
}

int ref_generate_synthetic(std::uint32_t dims, const std::uint32_t* radix, double q,
                           const char* profile, std::uint64_t seed, double* fit,
                           std::uint8_t* ok, double* f_opt, std::uint64_t* opt_rank) {
    try {
        SearchSpaceCache c = generate_synthetic_kernel_space(
            make_space(dims, radix), q, synthetic_profile(profile), seed);
        for (std::uint64_t r = 0; r < c.size(); ++r) {
            fit[r] = c.mean(r);
            ok[r] = c.ok(r) ? 1 : 0;
        }
        *f_opt = c.optimum();
        *opt_rank = c.optimum_rank();
        return 0;
    } catch (const NoFeasiblePoint&) {
        return 3;
    } catch (const std::exception&) {
        return 1;
    }
}

int ref_generate_nk(int n, int k, std::uint64_t seed, double* fit) {
    try {
        SearchSpaceCache c = generate_nk_landscape(n, k, seed);
        for (std::uint64_t r = 0; r < c.size(); ++r) fit[r] = c.mean(r);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

int ref_optimum(std::uint32_t dims, const std::uint32_t* radix, const double* fit,
                const std::uint8_t* ok, double* f_opt, std::uint64_t* rank) {
    try {
        SearchSpaceCache c = make_cache(dims, radix, fit, ok);
        *f_opt = c.optimum();
        *rank = c.optimum_rank();
        return 0;
    } catch (const NoFeasiblePoint&) {
        return 3;
    }
}

// FFG through the reference's own neighbour_ranks + SearchSpaceCache::mean/ok.
// targets_cap bounds the edge buffer; returns 0 or 2 if it is too small.
int ref_ffg(std::uint32_t dims, const std::uint32_t* radix, const double* fit,
            const std::uint8_t* ok, int kind, std::uint64_t* offsets,
            std::uint32_t* targets, std::uint64_t targets_cap, std::uint8_t* is_sink,
            std::uint32_t* minima, std::uint64_t* n_edges, std::uint64_t* n_minima) {
    SearchSpaceCache c = make_cache(dims, radix, fit, ok);
    const ParameterSpace& s = c.space();
    std::vector<std::uint64_t> nb;
    std::uint64_t e = 0, m = 0;
    offsets[0] = 0;
    for (std::uint64_t u = 0; u < s.size(); ++u) {
        s.neighbour_ranks(u, nk(kind), nb);
        for (auto v : nb) {
            if (c.mean(v) < c.mean(u)) {
                if (e >= targets_cap) return 2;
                targets[e++] = static_cast<std::uint32_t>(v);
            }
        }
        offsets[u + 1] = e;
        is_sink[u] = offsets[u + 1] == offsets[u];
        if (is_sink[u] && c.ok(u)) minima[m++] = static_cast<std::uint32_t>(u);
    }
    *n_edges = e;
    *n_minima = m;
    return 0;
}

// load_cache (cache_io.cpp:114-124) -> size, means, ok, present flags.
// Call with fit == nullptr to query the size; returns -1 on a parse error.
long long ref_load_cache(const char* path, double* fit, std::uint8_t* ok, std::uint8_t* present) {
    try {
        SearchSpaceCache c = load_cache(path);
        if (fit) {
            for (std::uint64_t r = 0; r < c.size(); ++r) {
                fit[r] = c.mean(r);
                ok[r] = c.present(r) && c.ok(r);
                present[r] = c.present(r);
            }
        }
        return static_cast<long long>(c.size());
    } catch (const std::exception&) {
        return -1;
    }
}

// save_cache of generate_synthetic_kernel_space (cache_io.cpp:126-160)
int ref_save_synthetic(std::uint32_t dims, const std::uint32_t* radix, double q,
                       const char* profile, std::uint64_t seed, const char* path) {
    try {
        save_cache(generate_synthetic_kernel_space(make_space(dims, radix), q,
                                                   synthetic_profile(profile), seed),
                   path);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

}  // extern "C"
