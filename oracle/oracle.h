/*
 * oracle.h -- CPU restatement of the reference's FFG / PageRank / C_p path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker: tests/, the smoke()
 * entry point and bench.py's cpu_baseline / --impl reference leg may load it.
 * The product (paper_2210_01465_b200, libtk_landscape.so) never links or calls
 * it; there is no CPU fallback through this file.
 *
 * Reference interface restated: /root/reference/proj/include/tunekit/landscape.hpp
 * (declarations only -- the reference ships no implementation).
 * Semantics follow the pinned decisions of SURVEY.md Appendix A (A1..A10).
 *
 * Parity pinning: neighbour order, rank arithmetic, the synthetic generators and
 * the FFG edge lists are checked against the reference's own compiled code
 * (oracle/_ref, built from /root/reference/proj/src by oracle/Makefile) through
 * the golden fixtures in tests/golden/.  PageRank and C_p have no reference
 * implementation to pin against: they are checked against the SPEC.md known
 * answers and against networkx.pagerank (an independent implementation).
 */
#ifndef TK_ORACLE_H
#define TK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_HAMMING = 0, OR_ADJACENT = 1 };           /* space.hpp:17 order */
enum { OR_OK = 0, OR_EINVAL = 1, OR_ELIMIT = 2, OR_ENOFEAS = 3,
       OR_ENOCONV = 4, OR_EDEGEN = 5 };

/* space.cpp:48-53 strides (dim 0 most significant); returns N = prod(radix). */
uint64_t or_space_strides(uint32_t dims, const uint32_t* radix, uint64_t* strides);
/* space.cpp:189-197 */
uint32_t or_max_neighbours(uint32_t dims, const uint32_t* radix, int kind);
/* space.cpp:167-187: neighbour ranks in canonical order; returns the count. */
uint32_t or_neighbour_ranks(uint32_t dims, const uint32_t* radix, uint64_t rank,
                            int kind, uint64_t* out);

/* landscape.hpp:44-45 build_ffg, split in a counting and a filling pass.
 * fit/ok are the rank-indexed SearchSpaceCache::mean/ok (cache.hpp:42-48). */
int or_ffg_count(uint32_t dims, const uint32_t* radix, const double* fit,
                 const uint8_t* ok, int kind, uint64_t node_limit,
                 uint64_t* n_edges, uint64_t* n_minima, int nthreads);
int or_ffg_fill(uint32_t dims, const uint32_t* radix, const double* fit,
                const uint8_t* ok, int kind, uint64_t* offsets, uint32_t* targets,
                uint8_t* is_sink, uint32_t* minima, int nthreads);

/* landscape.hpp:47-52 pagerank over an out-CSR.  fixed_iters > 0 runs exactly
 * that many iterations with no stop test (CPU baseline sampling). */
int or_pagerank(uint64_t n, const uint64_t* offsets, const uint32_t* targets,
                double damping, double tol, int64_t max_iter, double* r_out,
                int64_t* iterations, double* residual, int nthreads,
                int64_t fixed_iters);

/* landscape.hpp:56-58 */
int or_proportion_of_centrality(uint64_t n_minima, const uint32_t* minima,
                                const double* fit, const double* pr, double f_opt,
                                double p, double* out);

/* cache.cpp:55-72 f_opt: min over ok entries, strict <, lowest rank on ties */
int or_optimum(uint64_t n, const double* fit, const uint8_t* ok, double* f_opt,
               uint64_t* rank);

/* landscape.hpp:12-24 classify_points: strict census.  minima_ranks may be
 * NULL (count only). */
int or_census(uint32_t dims, const uint32_t* radix, const double* fit,
              const uint8_t* ok, int kind, uint64_t* fail_points,
              uint64_t* local_minima, uint64_t* interior, uint64_t* minima_ranks);

/* Synthetic inputs.  hash_uniform is generators.cpp:20-23. */
double or_hash_uniform(uint64_t seed, uint64_t rank, uint64_t slot);
void or_gen_iid(uint64_t n, double q, uint64_t seed, double* fit, uint8_t* ok,
                int nthreads);
void or_gen_heavy(uint64_t n, double q, uint64_t seed, double* fit, uint8_t* ok,
                  int nthreads);
/* generators.cpp:89-145, mean-only: the same 32 jittered samples summed left
 * to right and divided by 32, without storing them. */
int or_gen_synthetic(uint32_t dims, const uint32_t* radix, double fail_fraction,
                     double ridge_strength, double noise, double jitter,
                     uint64_t seed, double* fit, uint8_t* ok, int nthreads);

/* hillclimb.cpp:48-87 climb_random_first, batched: `walkers` descents from
 * uniform starts, each with its own splitmix64 stream (seed, walker) -- the
 * same draws, in the same order, as the device validator (tk_descents), so the
 * per-rank arrival counts are bit-identical.  counts: N u32 (arrivals per
 * end rank); evaluations: fitness lookups made.  Slots as build_slots
 * (hillclimb.cpp:26-38); at most 256 slots. */
int or_descents(uint32_t dims, const uint32_t* radix, const double* fit, int kind,
                uint64_t walkers, uint64_t seed, int restart_scan, uint32_t* counts,
                uint64_t* evaluations, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
