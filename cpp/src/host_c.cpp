// host_c.cpp -- C-linkage access to the drop-in's host-side generators, so
// non-C++ callers (bench.py's C4 batch) can build reference-identical
// synthetic caches (the reference's own generators.cpp:89-145, linked from
// its sources -- cpp/Makefile).
#include <cstdint>
#include <string>
#include <vector>

#include "tunekit/errors.hpp"
#include "tunekit/generators.hpp"
#include "tunekit_b200/host_c.h"

using namespace tunekit;

extern "C" int tk_host_generate_synthetic(uint32_t dims, const uint32_t* radix, double fail_fraction,
                                          const char* profile, uint64_t seed, double* fitness,
                                          uint8_t* ok) {
    try {
        std::vector<Parameter> ps(dims);
        for (uint32_t i = 0; i < dims; ++i) {
            ps[i].name = "p" + std::to_string(i);
            for (uint32_t v = 0; v < radix[i]; ++v) ps[i].values.push_back(std::int64_t{v});
        }
        const SearchSpaceCache c = generate_synthetic_kernel_space(
            ParameterSpace(std::move(ps)), fail_fraction, synthetic_profile(profile), seed);
        for (std::uint64_t r = 0; r < c.size(); ++r) {
            fitness[r] = c.mean(r);
            ok[r] = c.ok(r) ? 1 : 0;
        }
        return 0;
    } catch (const InvalidArgument&) {
        return 1;
    } catch (const std::exception&) {
        return 2;
    }
}
