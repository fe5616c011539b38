// tunekit_b200/extensions.hpp -- additions beyond the reference's landscape.hpp.
#pragma once

#include <cstdint>
#include <vector>

#include "tunekit/landscape.hpp"

namespace tunekit {

// analyze_landscape with an explicit FFG node limit.  The reference's
// analyze_landscape (landscape.hpp:77-79) has no node_limit parameter while
// build_ffg defaults to 1e6 (landscape.hpp:44-45), so spaces above 1e6
// configurations need this overload.
CentralityReport analyze_landscape_limited(const SearchSpaceCache& cache, NeighbourhoodKind kind,
                                           double damping, int p_max_percent,
                                           std::uint64_t node_limit);

// analyze_landscape straight from a cache file (native or Kernel Tuner JSON,
// cache_io.hpp): only the ok records travel to the GPU, as configuration
// index vectors; the device encodes them to mixed-radix keys, builds an
// open-addressing hash table of the valid set and densifies it (absent keys
// become failed nodes).  No rank-indexed host table is built.  `space_out`
// receives the parsed space (for report keys).
CentralityReport analyze_cache_file(const std::string& path, NeighbourhoodKind kind,
                                    double damping, int p_max_percent, std::uint64_t node_limit,
                                    ParameterSpace* space_out = nullptr);

// analyze_landscape over many caches in one device call (tk_batch_analyze:
// one upload, one launch with a CTA group per space, one read-back) -- for
// the 10^3-10^5-configuration spaces of real tuning problems, where the
// per-space path is bound by launch and synchronisation latency.  Caches of
// more than 2^20 configurations (or > 64 neighbour slots) are analysed one by
// one.  Same results and exceptions as analyze_landscape per cache.
std::vector<CentralityReport> analyze_landscapes(const std::vector<const SearchSpaceCache*>& caches,
                                                 NeighbourhoodKind kind, double damping = 0.85,
                                                 int p_max_percent = 15);

// The GPU random-walk validator: `walkers` randomized
// first-improvement descents -- hillclimb.cpp:48-87 climb_random_first, with a
// fresh scan order after every move when restart_scan -- from uniform starts,
// all on the device (tk_descents).  Walker w draws from its own splitmix64
// stream (seed, w), so the result is deterministic.  arrivals[i] counts the
// descents that ended at minima[i] (the FFG minima, ascending); fail_arrivals
// those that ended on a failed sink.  SPEC.md:430: the arrival frequencies
// track PageRank over the minima.
struct DescentReport {
    std::vector<std::uint64_t> minima;
    std::vector<std::uint64_t> arrivals;
    std::uint64_t fail_arrivals = 0;
    std::uint64_t evaluations = 0;
};
DescentReport random_descents(const SearchSpaceCache& cache, NeighbourhoodKind kind,
                              std::uint64_t walkers, std::uint64_t seed, bool restart_scan = true);

}  // namespace tunekit
