/*
 * tk_landscape.h -- the C-ABI drop-in boundary for the FFG / PageRank / C_p path.
 *
 * Plain C: pointers, sizes, status codes.  No exceptions, no torch or C++ types
 * cross this boundary.  The C++ drop-in (cpp/src/landscape.cpp, the reference's
 * include/tunekit/landscape.hpp implemented on top of this ABI) rethrows the status codes as the reference's exception types.
 *
 * Every entry point names the reference interface it replaces.  Paths are
 * relative to /root/reference/proj (read-only reference; the declarations there
 * have no implementation anywhere -- SURVEY.md s0.1):
 *   landscape.hpp = include/tunekit/landscape.hpp
 *   cache.hpp     = include/tunekit/cache.hpp
 *   space.hpp     = include/tunekit/space.hpp
 *   errors.hpp    = include/tunekit/errors.hpp
 *
 * Threading: a tk_land handle is bound to one device and one CUDA stream and is
 * not thread-safe; use one host thread per handle.  All calls are synchronous
 * with respect to the host unless stated otherwise.
 */
#ifndef TK_LANDSCAPE_H
#define TK_LANDSCAPE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TK_ABI_VERSION 1
#define TK_MAX_DIMS 32
#define TK_MAX_CP 101

/* Status codes.  Mapping onto errors.hpp:10-44:
 *   TK_EINVAL, TK_ELIMIT -> InvalidArgument   TK_ENOFEAS -> NoFeasiblePoint
 *   TK_ENOCONV -> NonConvergence              everything else -> Error       */
enum tk_status {
    TK_OK = 0,
    TK_EINVAL = 1,  /* bad argument (errors.hpp:15-17) */
    TK_ELIMIT = 2,  /* N > node_limit (landscape.hpp:44-45) */
    TK_ENOFEAS = 3, /* no ok entry (cache.cpp:89-92) */
    TK_ENOCONV = 4, /* PageRank hit max_iter (errors.hpp:37-42) */
    TK_EDEGEN = 5,  /* zero minima centrality */
    TK_ENOMEM = 6,
    TK_ECUDA = 7,
    TK_ENCCL = 8,
    TK_ESTATE = 9   /* call out of order (e.g. pagerank before build) */
};

/* NeighbourhoodKind, same order as space.hpp:17 */
enum tk_kind { TK_HAMMING = 0, TK_ADJACENT = 1 };
/* where a buffer argument lives */
enum tk_mem { TK_MEM_HOST = 0, TK_MEM_DEVICE = 1 };
/* device-side synthetic generators (SURVEY.md s8d G_iid / G_heavy), bit-identical
 * to oracle/oracle.c or_gen_iid / or_gen_heavy */
enum tk_gen { TK_GEN_IID = 0, TK_GEN_HEAVY = 1 };

typedef struct tk_land tk_land; /* one search space resident on one device */

typedef struct tk_report_summary {
    uint64_t n_nodes, n_edges, n_minima;
    double f_opt;         /* cache.hpp:75 optimum() */
    uint64_t opt_rank;    /* cache.hpp:76 optimum_rank() */
    int64_t iterations;   /* landscape.hpp:73 pagerank_iterations */
    double residual;      /* final L1 change */
    double pagerank_sum;  /* landscape.hpp:74 */
    int32_t n_cp;         /* p_max_percent + 1 */
    double c_p[TK_MAX_CP];/* landscape.hpp:72 c_p_curve, pct = 0..p_max */
    float ms_load, ms_ffg, ms_pagerank, ms_centrality; /* device time per phase */
} tk_report_summary;

int tk_abi_version(void);
/* Thread-local message for the last non-OK status on this thread. */
const char* tk_last_error(void);
const char* tk_status_name(int status);
int tk_device_count(int* count);

/* ---------------------------------------------------------------- spaces -- */

/* ParameterSpace shape (space.hpp:26-53): radix[i] = list_size(i), dim 0 most
 * significant.  N = prod(radix) must be < 2^32 (u32 node ids, landscape.hpp:32). */
int tk_land_create(int device, uint32_t dims, const uint32_t* radix, tk_land** out);
int tk_land_destroy(tk_land* land);
/* Re-target a handle at another space shape, keeping its device buffers
 * (they only grow): many small landscapes back to back without cudaMalloc. */
int tk_land_reshape(tk_land* land, uint32_t dims, const uint32_t* radix);
int tk_land_info(const tk_land* land, uint64_t* n_nodes, int* device);
/* The cudaStream_t every kernel of this handle is launched on (for events). */
void* tk_land_stream(tk_land* land);
/* Which kernels the last build / PageRank used (build: 1 = TMA-staged Adjacent
 * path, 0 = per-lane gathers; PageRank: 2 = row-tiled Adjacent kernel, 1 =
 * TMA-staged, 0 = per-lane gathers), the PageRank grid size and the kernel-only device
 * times of the last build and PageRank launches (ms).  Any pointer may be NULL. */
int tk_land_kernel_info(const tk_land* land, int* staged_build, int* staged_pagerank,
                        int* pagerank_grid, float* ms_build, float* ms_pagerank);

/* SearchSpaceCache::mean/ok (cache.hpp:42-48): rank-indexed fitness and ok
 * flags.  The cache must be complete.  Failed entries are forced
 * to kFailFitness = 1e10 (cache.hpp:15, cache.cpp:49-53); an ok mean >= 1e10
 * -> TK_EINVAL. */
int tk_land_load_dense(tk_land* land, const double* fitness, const uint8_t* ok, int mem);
/* Valid set as (key = rank, fitness) pairs (cache_io.cpp:79-112: constrained
 * configurations are absent or failed entries).  Keys are ranks < N,
 * so the valid set is scattered straight into the rank-indexed table; every
 * absent key becomes a failed node (1e10).  Duplicate keys, keys >= N, or an
 * ok mean >= 1e10 (cache.hpp:15) -> TK_EINVAL. */
int tk_land_load_sparse(tk_land* land, const uint64_t* keys, const double* fitness,
                        uint64_t n_valid, int mem);
/* Same, with configurations as index vectors (row-major int32[n_valid][dims]),
 * encoded on the device with the mixed-radix rank of space.cpp:72-78. */
int tk_land_load_configs(tk_land* land, const int32_t* configs, const double* fitness,
                         uint64_t n_valid, int mem);
int tk_land_generate(tk_land* land, int gen, double fail_fraction, uint64_t seed);
int tk_land_copy_fitness(tk_land* land, double* fitness, uint8_t* ok);
/* Lookup of arbitrary keys in the valid set of the loaded table through a GPU
 * open-addressing hash table (built on the first lookup after a load):
 * fitness and found = 1 for an ok rank, 1e10 and found = 0 otherwise. */
int tk_land_lookup(tk_land* land, const uint64_t* keys, uint64_t n, double* fitness,
                   uint8_t* found);

/* cache.cpp:55-72,89-98: f_opt = min mean over ok entries, lowest rank on ties. */
int tk_optimum(tk_land* land, double* f_opt, uint64_t* rank);

/* --------------------------------------------------------------- the FFG -- */

/* build_ffg (landscape.hpp:44-45).  emit_csr = 0 keeps only the compact
 * per-node neighbour masks (enough for PageRank, C_p and census); 1 also
 * materialises the out-CSR for tk_ffg_copy_out. */
int tk_ffg_build(tk_land* land, int kind, uint64_t node_limit, int emit_csr,
                 uint64_t* n_edges, uint64_t* n_minima);
/* FitnessFlowGraph fields (landscape.hpp:30-37); caller-allocated host buffers
 * of N+1, n_edges, N, n_minima elements.  Any pointer may be NULL. */
int tk_ffg_copy_out(tk_land* land, uint64_t* offsets, uint32_t* targets,
                    uint8_t* is_sink, uint32_t* minima);
/* classify_points (landscape.hpp:12-24): strict census on the built FFG's kind.
 * minima_ranks (host, local_minima entries) may be NULL. */
int tk_census(tk_land* land, uint64_t* fail_points, uint64_t* local_minima,
              uint64_t* interior, uint64_t* minima_ranks);

/* ------------------------------------------------------------- PageRank -- */

/* pagerank (landscape.hpp:47-52) on the handle's FFG.  TK_ENOCONV leaves
 * iterations/residual set (NonConvergence fields, errors.hpp:37-42). */
int tk_pagerank(tk_land* land, double damping, double tol, int64_t max_iter,
                int64_t* iterations, double* residual, double* sum);
int tk_pagerank_copy_out(tk_land* land, double* rank_vector);
/* proportion_of_centrality (landscape.hpp:56-58) for n_p values of p at once. */
int tk_centrality(tk_land* land, double f_opt, const double* p, int n_p, double* c_p);
/* MinimumInfo rows (landscape.hpp:60-65) in ascending rank. */
int tk_report_copy_out(tk_land* land, double f_opt, uint64_t* ranks, double* fitness,
                       double* fraction_of_optimum, double* pagerank);

/* analyze_landscape (landscape.hpp:77-79) fused on the device: optimum, FFG,
 * PageRank, C_p for pct = 0..p_max_percent.  Only the summary leaves the GPU;
 * minima rows via tk_report_copy_out. */
int tk_analyze(tk_land* land, int kind, double damping, double tol, int64_t max_iter,
               uint64_t node_limit, int p_max_percent, int emit_csr,
               tk_report_summary* out);

/* ---------------------------------------- batches of small spaces (C4) -- */
/* analyze_landscape (landscape.hpp:77-79) for many small spaces in one call:
 * one upload, one launch (one CTA per space runs FFG, f_opt, minima, PageRank,
 * C_p and the report rows), one read-back.  For N <= 2^20 configurations and
 * <= 64 neighbour slots per space; other items get status TK_EINVAL.  fitness
 * / ok are host (TK_MEM_HOST) or device (TK_MEM_DEVICE) pointers per item;
 * the minima_* outputs are host pointers with room for minima_capacity rows
 * (NULL: no rows).  Per-item results in summary and status (TK_OK,
 * TK_ENOFEAS, TK_ENOCONV, TK_EDEGEN, TK_EINVAL); the call itself returns
 * TK_OK unless the arguments or the device fail.  The global sums are block
 * reductions, so per-node ranks can differ from tk_analyze's in the last bits
 * (its dangling mass is summed in another order); both are checked against
 * the oracle. */
typedef struct tk_batch_item {
    uint32_t dims;
    uint32_t radix[TK_MAX_DIMS];
    const double* fitness;
    const uint8_t* ok;
    uint64_t* minima_ranks;
    double* minima_fitness;
    double* minima_fraction;
    double* minima_pagerank;
    uint64_t minima_capacity;
    tk_report_summary summary;
    int32_t status;
} tk_batch_item;
int tk_batch_analyze(int device, tk_batch_item* items, uint32_t n_items, int kind, double damping,
                     double tol, int64_t max_iter, int p_max_percent, int mem);

/* ------------------------------- random-walk validator -- */
/* hillclimb.cpp:48-87 climb_random_first, batched on the device: `walkers`
 * randomized first-improvement descents from uniform starts over the loaded
 * table, in the neighbourhood of the last tk_ffg_build (the
 * paper's s7.2 random-walk claim).  Walker w draws from its own splitmix64
 * stream (seed, w); results are deterministic and bit-identical to the
 * oracle's restatement.  arrivals: n_minima u64, the descents that ended at
 * each FFG minimum (tk_ffg_copy_out order); fail_arrivals: those that ended on
 * a failed sink; evaluations: fitness lookups made.  Any output may be NULL.
 * At most 256 neighbour slots (build_slots).  TK_ESTATE before a build. */
int tk_descents(tk_land* land, uint64_t walkers, uint64_t seed, int restart_scan,
                uint64_t* arrivals, uint64_t* fail_arrivals, uint64_t* evaluations);

/* ------------------------------------- key-range sharding -- */
/* Multi-GPU analyze_landscape: one handle per GPU, every handle loads the full
 * fitness table, handle `rank` of `nranks` owns ranks [lo, hi) (lo = rank *
 * chunk, chunk = ceil(N/nranks) rounded up to 512).  Adjacent spaces with
 * 2*dims <= 27 only.  After tk_land_set_shard, tk_ffg_build builds the
 * shard's rows only (n_edges / n_minima are the shard's counts, no CSR).
 * The host sums the per-shard partials across ranks between calls (see
 * paper_2210_01465_b200/sharded.py); that reduction is the iteration barrier.
 * The whole-space calls (tk_optimum, tk_ffg_copy_out of offsets / targets /
 * is_sink, tk_census, tk_pagerank, tk_centrality, tk_analyze) return
 * TK_ESTATE on a sharded handle: its rows cover only [lo, hi). */
int tk_land_set_shard(tk_land* land, int rank, int nranks, uint64_t* lo, uint64_t* hi);
/* device pointers of this handle's two PageRank contribution replicas */
int tk_land_replica_ptrs(tk_land* land, void** c0, void** c1);
/* peers' replicas (nranks entries each, own entry ignored): same process */
int tk_land_set_peer_ptrs(tk_land* land, void* const* c0, void* const* c1);
/* the replicas as two cudaIpcMemHandle_t (128 bytes); tk_land_open_peers maps
 * the nranks*128 bytes of every rank's handles (own entry ignored) */
int tk_land_ipc_handles(tk_land* land, void* handles128);
int tk_land_open_peers(tk_land* land, const void* handles);
/* shard partials: (fitness, rank) minimum over the shard's ok ranks; has = 0 if none */
int tk_shard_optimum(tk_land* land, double* f, uint64_t* rank, int* has);
int tk_shard_pagerank_init(tk_land* land, double damping, double* dangling);
/* one iteration: dangling_total = summed dangling mass of the previous iterate */
int tk_shard_pagerank_step(tk_land* land, double dangling_total, double damping,
                           double* residual, double* dangling, double* sum);
/* nums[n_p] and den: the shard's C_p numerators / denominator */
/* Device-side iteration control: the same init / step, asynchronous on the
 * handle's stream (tk_land_stream).  d_partials (device, 3 doubles) receives
 * this shard's (L1 change, dangling mass, sum of r'); the step reads the
 * all-reduced totals of the previous step from d_totals (device) -- the caller
 * all-reduces d_partials in place on that stream (NCCL) between calls. */
int tk_shard_pagerank_init_dev(tk_land* land, double damping, double* d_partials);
int tk_shard_pagerank_step_dev(tk_land* land, const double* d_totals, double damping,
                               double* d_partials);
/* Undo the bookkeeping of the last step (after a speculative step past the
 * stop: that step wrote its contributions to the other parity buffer, the
 * previous iterate stays where it was).  The shard steps store contributions
 * only; readers of the rank vector (copy_out, centrality, report) rebuild it
 * from the current iterate's contributions on first use. */
int tk_shard_pagerank_rewind(tk_land* land);
int tk_shard_centrality(tk_land* land, double f_opt, const double* p, int n_p, double* nums,
                        double* den);
/* the shard's slice [lo, hi) of the current rank vector */
int tk_shard_pagerank_copy_out(tk_land* land, double* r_slice);

/* ---------------------------------------------- free-standing (host CSR) -- */

/* pagerank(const FitnessFlowGraph&) (landscape.hpp:51-52) for an arbitrary
 * host out-CSR: uploaded, transposed on the device, iterated.  r_out: n doubles. */
int tk_pagerank_csr(int device, uint64_t n, const uint64_t* offsets,
                    const uint32_t* targets, double damping, double tol,
                    int64_t max_iter, double* r_out, int64_t* iterations,
                    double* residual);
/* proportion_of_centrality(g, pr, f_opt, p) (landscape.hpp:56-58) over the
 * minima's fitness and PageRank values (host arrays, ascending rank order). */
int tk_proportion_of_centrality(int device, uint64_t n_minima, const double* min_fitness,
                                const double* min_pagerank, double f_opt, double p,
                                double* out);

#ifdef __cplusplus
}
#endif
#endif /* TK_LANDSCAPE_H */
