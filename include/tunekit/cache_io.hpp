// tunekit/cache_io.hpp -- cache files of the drop-in C++ surface
// (API of /root/reference/proj/include/tunekit/cache_io.hpp:9-22).
//
// Native schema: {"metadata": {"kernel", "device", "units"},
//                 "space": {"parameters": [...]},
//                 "cache": {"v1,...,vn": {"times": [..]|null, "time": x|null}}}
// Kernel Tuner files: "tune_params" (+ optional "tune_params_keys") as the
// space, "time" holding a mean or an error string (a failed configuration).
#pragma once

#include <string>

#include "tunekit/cache.hpp"

namespace tunekit {

SearchSpaceCache load_cache(const std::string& path);
SearchSpaceCache cache_from_json(const Json& j);
Json cache_to_json(const SearchSpaceCache& cache);
void save_cache(const SearchSpaceCache& cache, const std::string& path);

}  // namespace tunekit
