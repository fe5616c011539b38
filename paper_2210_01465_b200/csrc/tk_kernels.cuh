// tk_kernels.cuh -- host-side launch wrappers for the sm_100a kernels.
// Every wrapper enqueues on `stream` and returns a cudaError_t; none blocks.
#pragma once

#include <cuda.h>

#include "tk_internal.cuh"

namespace tk {

// ---- ingestion -------------------------------------------------------------
cudaError_t launch_generate(int gen, uint32_t n, double q, uint64_t seed, double* fit,
                            uint8_t* ok, cudaStream_t stream);
cudaError_t launch_encode_configs(const int32_t* configs, uint64_t n_valid, int dims_in,
                                  const uint32_t* radix_in_host,
                                  const unsigned long long* strides_in_host,
                                  unsigned long long* keys_out, int* err_flag,
                                  cudaStream_t stream);
// valid (key, fitness) pairs -> dense rank-indexed table; err bits 1 key >= N,
// 2 duplicate key, 4 mean >= kFailFitness.  claimed: ceil(n/32) u32 scratch.
// scratch (load_valid_scratch_bytes, or null for the direct scatter): the pairs
// are first partitioned by 2^17-rank slices so the scatter stays in L2
cudaError_t launch_load_valid(const unsigned long long* keys, const double* vals,
                              uint64_t n_valid, uint32_t n, double* fit, uint8_t* ok,
                              unsigned int* claimed, int* err_flag, cudaStream_t stream,
                              void* scratch);
size_t load_valid_scratch_bytes(uint64_t n_valid, uint32_t n);
// failed entries -> kFailFitness; err bit 4 if an ok mean >= kFailFitness
cudaError_t launch_normalize_dense(uint32_t n, double* fit, const uint8_t* ok, int* err_flag,
                                   cudaStream_t stream);
cudaError_t launch_count_ok(const uint8_t* ok, uint32_t n, unsigned long long* count,
                            cudaStream_t stream);
// open-addressing table of the ok ranks (cap a power of two >= 2 * ok count);
// err bit 8 if a probe loop hit its bound
cudaError_t launch_hash_build(const double* fit, const uint8_t* ok, uint32_t n,
                              unsigned long long* hkeys, double* hvals, uint64_t cap,
                              int* err_flag, cudaStream_t stream);
cudaError_t launch_hash_lookup(const unsigned long long* hkeys, const double* hvals,
                               uint64_t cap, const unsigned long long* q, uint64_t nq,
                               double* out, uint8_t* found, int* err_flag,
                               cudaStream_t stream);
cudaError_t launch_optimum(const double* fit, const uint8_t* ok, uint32_t n,
                           double* part_f, unsigned long long* part_r, double* f_opt,
                           unsigned long long* rank, int* has, cudaStream_t stream);
// final argmin over nparts (fitness, rank) partials (rank ~0 = empty partial)
cudaError_t launch_optimum_final(const double* part_f, const unsigned long long* part_r,
                                 int nparts, double* f_opt, unsigned long long* rank, int* has,
                                 cudaStream_t stream);

// ---- FFG ---------------------------------------------------------------------
struct BuildArgs {
    const double* fit;
    const uint8_t* ok;
    void* inm;            // in-mask (u32 or u64 per node) -- not packed mode
    uint8_t* odeg;        // out-degree -- not packed mode
    uint32_t* pw;         // packed word -- packed mode
    uint8_t* flags;       // bit0 sink, bit1 ok&&sink, bit2 strict minimum, bit3 ok
    unsigned long long* offsets;  // N+1 (emit)
    uint32_t* targets;            // E (emit)
    uint32_t* minima;             // M
    unsigned long long* e_status; // per tile
    unsigned long long* m_status; // per tile
    unsigned int* tile_counter;
    unsigned long long* totals;   // [0] E, [1] M, [2] strict minima, [3] ok nodes
    uint32_t ntiles;
    // two-pass staged build (count -> tile scan -> fill)
    uint32_t* om;                 // canonical out-mask per rank
    uint32_t* tile_e;             // per-tile edge count   (count pass)
    uint32_t* tile_m;             // per-tile minima count (count pass)
    unsigned long long* ebase;    // exclusive scan of tile_e, [ntiles] = E
    unsigned long long* mbase;    // exclusive scan of tile_m, [ntiles] = M
    // f_opt fused into the count pass: per-block (fitness, rank) argmin over ok ranks
    double* opt_part_f;
    unsigned long long* opt_part_r;
    double* f_opt;                // final reduction target (device)
    unsigned long long* opt_rank;
    int* opt_has;
    uint32_t tile_lo;             // first tile of this shard (0 unsharded)
};

// Key-range shard of a multi-GPU run: this device owns ranks
// [lo, hi); c replicas of every rank (own included) for both parities.
constexpr int kMaxShards = 8;
struct ShardInfo {
    int nranks;          // 1 = unsharded
    int self;
    uint32_t lo, hi;
    unsigned long long chunk_magic;  // fdiv magic of the chunk length
    double* peer_c[2][kMaxShards];   // [parity][rank] replica base pointers
    const uint32_t* edges_om;        // non-null: push along out-edges only (out-masks)
};
constexpr int kBuildThreads = 256;
cudaError_t launch_ffg_build(const DevShape& s, int mode, bool wide, bool emit,
                             const BuildArgs& a, int num_sms, cudaStream_t stream);

// flags & mask != 0 -> ascending u64 ranks (generic compaction, look-back)
cudaError_t launch_compact_flags(const uint8_t* flags, uint8_t mask, uint32_t n,
                                 unsigned long long* out, unsigned long long* status,
                                 unsigned int* tile_counter, uint32_t ntiles,
                                 int num_sms, cudaStream_t stream);
cudaError_t launch_flags_to_sink(const uint8_t* flags, uint32_t n, uint8_t* is_sink,
                                 cudaStream_t stream);

// ---- CSR transpose (tk_pagerank_csr) -------------------------------------
cudaError_t launch_csr_prepare(uint32_t n, const unsigned long long* offsets,
                               const uint32_t* targets, uint64_t e, uint32_t* odeg32,
                               uint32_t* indeg, cudaStream_t stream);
cudaError_t launch_exclusive_scan_u32(const uint32_t* in, uint32_t n,
                                      unsigned long long* out /* n+1 */,
                                      unsigned long long* status, unsigned int* tile_counter,
                                      uint32_t ntiles, int num_sms, cudaStream_t stream);
cudaError_t launch_csr_scatter(uint32_t n, const unsigned long long* offsets,
                               const uint32_t* targets, const unsigned long long* in_off,
                               uint32_t* cursor, uint32_t* src, cudaStream_t stream);
cudaError_t launch_csr_sort_rows(uint32_t n, const unsigned long long* in_off, uint32_t* src,
                                 cudaStream_t stream);

// ---- PageRank ----------------------------------------------------------------
struct PrArgs {
    uint32_t n;
    double inv_n;      // 1.0 / N
    double nd;         // (double) N
    double teleport;   // (1 - d) / N
    double damping;
    double tol;
    long long max_iter;
    const uint32_t* pw;            // MODE_ADJ_PACKED
    const void* inm;               // MODE_ADJ_ORDERED / MODE_HAM
    const uint8_t* odeg;           // idem
    const unsigned long long* in_off;  // MODE_CSR
    const uint32_t* src;               // MODE_CSR
    const uint32_t* odeg32;            // MODE_CSR
    double* r0;
    double* r1;
    double* c0;
    double* c1;
    double* part;                  // [2][grid][3]
    long long* out_iter;
    double* out_res;
    double* out_sum;
    int* out_parity;               // buffer index holding the result
    int* out_status;               // 0 converged, 1 max_iter
};
constexpr int kPrThreads = 256;
// grid_out receives the cooperative grid size used.
cudaError_t launch_pagerank(const DevShape& s, int mode, bool wide, const PrArgs& a,
                            int num_sms, int* grid_out, cudaStream_t stream);
int pagerank_max_grid(int mode, bool wide, int num_sms);
// Hamming: tiled contribution-only kernel (tk_hamming.cu) for shapes whose
// digits align with 512-rank tiles; cudaErrorNotSupported otherwise
bool ham_tiled_supported(const DevShape& s);
// Adjacent: ring kernel (tk_ring.cu) -- per-CTA shared-memory ring of c over
// chunks of consecutive tiles; far ranges staged per tile
bool ring_plan_available(const DevShape& s, int smem_budget, int num_sms);
cudaError_t launch_pagerank_ring(const DevShape& s, const PrArgs& a, int smem_budget, int num_sms,
                                 int* grid_out, cudaStream_t stream);
// Hamming: staged kernel (tk_hamming.cu) -- outer lines streamed through a
// shared-memory ring with TMA bulk copies, inner lines from a block copy
struct HamStagePlanOut {
    int k;        // outer dims
    uint32_t B;   // block ranks (s_{k-1})
    int R;        // outer ranges per tile
    int C;        // ranges per ring stage
    int stages;   // ring stages
};
bool ham_staged_plan(const DevShape& s, int smem_budget, HamStagePlanOut* out);
cudaError_t launch_pagerank_ham_staged(const DevShape& s, bool wide, const HamStagePlanOut& p,
                                       const PrArgs& a, int num_sms, int* grid_out,
                                       cudaStream_t stream);
cudaError_t launch_pagerank_ham_tiled(const DevShape& s, bool wide, const PrArgs& a, int num_sms,
                                      int* grid_out, cudaStream_t stream);
// Hamming: in-edge sum split by dimension groups (tk_hamsplit.cu): one
// shared-memory window pass per group and iteration, the partial sum carried in
// r1 / acc1 between passes.  Runs to convergence (host-driven chunks); the
// result lands in a.r0 like the cooperative kernels'.  ws: at least
// ham_split_workspace_bytes() of device memory.
bool ham_split_available(const DevShape& s);
size_t ham_split_workspace_bytes(const DevShape& s);
cudaError_t launch_pagerank_ham_split(const DevShape& s, bool wide, const PrArgs& a, double* acc1,
                                      void* ws, int num_sms, int* grid_out, cudaStream_t stream);

// ---- TMA-staged Adjacent kernels (tk_staged.cu) ------------------------------
// A tile is T consecutive ranks [v0, v0+T).  The Adjacent neighbours of the tile
// along dimension i are the contiguous ranges [v0 - s_i, v0 - s_i + T) and
// [v0 + s_i, v0 + s_i + T), so the block stages, per tile, one "near window"
// [v0 - H, v0 + T + H) covering every dimension with s_i <= H plus one range
// per far slot, each with a single cp.async.bulk into shared memory.
struct StagePlan {
    int T;           // ranks per tile (= threads per block)
    int stages;      // pipeline depth
    int H;           // near halo (elements)
    int nfar;        // far ranges
    long long far_off[2 * kMaxDims];  // element offset of far range f from v0
    int lo_src[kMaxDims];  // f64 smem index (plus t) of the lower neighbour of dim i
    int hi_src[kMaxDims];  // ... upper neighbour
    int own_src;           // ... of the node itself
    int lo_off[kMaxDims];  // the same as byte offsets (8 * src)
    int hi_off[kMaxDims];
    int own_off;
    int near_len;          // elements in the near window (even)
    int far_len;           // elements per far range (even)
    int aux_bytes;         // bytes before the f64 region (pw + r for PageRank, ok for FFG)
    int stage_bytes;
    unsigned int far_ef;   // far ranges whose L2 lines are loaded evict-first (bit f)
    // FFG count digit classes (bit i = dim i), tile T at rank v0, P_i = s_i * m_i:
    //   dim_inv:  P_i divides T -> x_i = (t mod P_i) / s_i, fixed per thread
    //   dim_uni:  T divides s_i -> x_i constant over the tile; its border bits
    //             are staged per tile in the stage header
    //   dim_tile: T divides P_i otherwise -> x_i = ((v0 mod P_i) + t) / s_i with
    //             v0 mod P_i staged in the header
    //   the rest: decoded per rank from the rank
    unsigned int dim_inv, dim_uni, dim_tile;
    unsigned long long npad2;  // f64 arrays hold at least this many elements (even)
    unsigned long long npad16; // u8/u32 arrays are padded to this many elements
    int fast;                  // FFG count: table is clean (finite, no -0): DADD-sign compares
};
// kind_pr: PageRank layout (u32 pw[T], f64 r[T], window) vs FFG (u8 ok[T], window)
// stage_r: PageRank stages the old ranks too (the sharded step); the single-GPU
// kernel stores contributions only and stages pw + window
bool make_stage_plan(const DevShape& s, bool kind_pr, int smem_budget, StagePlan* plan,
                     bool stage_r = true);
// count (staged) -> tile scans -> fill; a.e_status/m_status/tile_counter are the
// scan scratch (>= ceil(ntiles/256) tiles), totals[0..1] are written by the scan.
size_t fused_seg_bytes();
cudaError_t launch_ffg_build_fused(const DevShape& s, const StagePlan& p, const BuildArgs& a,
                                   int num_sms, cudaStream_t stream);
cudaError_t launch_ffg_build_staged(const DevShape& s, const StagePlan& p, bool emit,
                                    const BuildArgs& a, int num_sms, cudaStream_t stream);
cudaError_t launch_pagerank_staged(const DevShape& s, const StagePlan& p, const PrArgs& a,
                                   int num_sms, int* grid_out, cudaStream_t stream);
// Shard steps (one launch per PageRank iteration, no grid barrier): ranks
// [sh.lo, sh.hi); c' is stored into the local replica and, for ranks with an
// out-neighbour owned by another shard, into that shard's replica.
// Contribution-only: no rank vector is stored per step (c = r / outdeg, r for
// a sink).  init: c0 (parity 0) + dangling partial;  step: reads parity `cur`,
// writes parity cur^1.  Partials land in out3[0..2] (res, dangling, sum).
cudaError_t launch_pagerank_shard_init(const DevShape& s, const ShardInfo& sh, const PrArgs& a,
                                       const uint32_t* om, double* part, double* out3,
                                       int num_sms, cudaStream_t stream);
// dtot (optional, device): previous step's all-reduced totals; D/N is formed
// on the device from dtot[1] instead of taking dn
cudaError_t launch_pagerank_shard_step(const DevShape& s, const StagePlan& p, const ShardInfo& sh,
                                       const PrArgs& a, int cur, double dn,
                                       double* part, double* out3, int num_sms,
                                       cudaStream_t stream, const double* dtot = nullptr);
// r[v] over the shard's ranks [lo, hi) from its contributions c (shard_materialize_kernel)
cudaError_t launch_shard_materialize(uint64_t lo, uint64_t hi, const uint32_t* pw, const double* c,
                                    double* r, int num_sms, cudaStream_t stream);

// ---- row-tiled Adjacent PageRank (tk_rows.cu) --------------------------------
// For spaces whose trailing dims span exactly 16 ranks (a "row") and N % 512 == 0.
// Non-row dims split into far dims 0..nfar-1 (one staged 32-row range per
// direction and tile) and window dims nfar..nfar+nwin-1 (served from a per-CTA
// ring of the column's rows).  A column (super-column) is col_rows consecutive
// rows, a whole number of 32-row tiles; columns are dealt round-robin to CTAs.
struct RowPlan {
    int dims;                   // effective dims (DevShape::dims)
    int nrow_dims;              // trailing dims inside a row
    int row_radix[4];           // their radices, most significant first
    int nfar, nwin;             // far dims / window dims
    int ahead;                  // A = ceil(largest window stride in rows / 32)
    uint32_t rows;              // N / 16
    uint32_t col_rows, ncols, tiles_per_col;
    unsigned long long tpc_magic;                 // fdiv magic of tiles_per_col
    int win_rows[kMaxDims];                       // row stride of window dim nfar + k
    uint32_t far_rows[kMaxDims];                  // row stride of far dim d
    uint32_t far_radix[kMaxDims];
    unsigned long long far_magic[kMaxDims];       // fdiv magic of far_rows[d]
    unsigned long long far_rmagic[kMaxDims];      // fdiv magic of far_radix[d]
    int far_span[kMaxDims];                       // a 32-row tile spans several digits
    uint32_t far_ef;                              // far dims loaded L2 evict-first (bit d)
    int far_per_col;                              // columns are whole tiles: far digits per column
};
// TMA tensor maps of the rank-vector buffers viewed as [rows][16] f64 (SWIZZLE_128B)
// and of the packed words as [rows][16] u32 (SWIZZLE_64B), 32-row boxes.
struct alignas(64) RowMaps {
    CUtensorMap c[2];
    CUtensorMap r0;
    CUtensorMap pw;
};
bool make_row_plan(const DevShape& s, int num_sms, RowPlan* plan);
cudaError_t launch_pagerank_rows(const DevShape& s, const RowPlan& p, const PrArgs& a,
                                 int num_sms, int* grid_out, cudaStream_t stream);

// ---- C_p and report -------------------------------------------------------
constexpr int kCpBlocks = 148 * 8;  // enough warps to hide the dependent minima -> (f, r) gathers
// minima == nullptr: fit/r are already per-minimum arrays of length m.
// raw: c_p_out receives n_p numerators then the denominator (n_p + 1 values).
cudaError_t launch_centrality(const uint32_t* minima, uint64_t m, const double* fit,
                              const double* r, const double* p, int n_p, double f_opt,
                              double* part, double* c_p_out, int* degenerate,
                              cudaStream_t stream, bool raw = false);
cudaError_t launch_report(const uint32_t* minima, uint64_t m, const double* fit,
                          const double* r, double f_opt, unsigned long long* ranks,
                          double* fitness, double* fraction, double* pr,
                          cudaStream_t stream);
cudaError_t launch_gather_values(const uint32_t* idx, uint64_t m, const double* src,
                                 double* dst, cudaStream_t stream);

// ---- batches of small spaces (tk_batch.cu) --------------------------------------
constexpr uint64_t kBatchMaxNodes = 1ull << 20;
struct BatchOut {
    unsigned long long n_nodes, n_edges, n_minima, opt_rank;
    unsigned long long row_base;  // first row of this space's report rows (compact region)
    double f_opt;
    long long iterations;
    double residual, pagerank_sum;
    double c_p[TK_MAX_CP];
    int status;
};
struct BatchParams {
    int kind;
    double damping, tol;
    long long max_iter;
    int n_p;
    double onep[TK_MAX_CP];  // 1 + p (host IEEE), the band f < (1 + p) f_opt
    int zero[TK_MAX_CP];     // p == 0: f <= f_opt
};
bool batch_item_supported(uint32_t dims, const uint32_t* radix, int kind, uint64_t* n_out);
size_t batch_desc_bytes();
size_t batch_workspace_bytes(uint32_t n, uint32_t slots);
uint32_t batch_slots(uint32_t dims, const uint32_t* radix, int kind);
void batch_fill_desc(void* desc_host, const double* fit, const uint8_t* ok, uint32_t n,
                     uint32_t slots, uint32_t dims_in, const uint32_t* radix_in, uint8_t* ws,
                     unsigned int* bar, double* part, BatchOut* out, double* rows,
                     unsigned long long* row_cursor);
cudaError_t launch_batch_analyze(const void* descs_dev, uint32_t n_items, const BatchParams& P,
                                 int num_sms, cudaStream_t stream);
int batch_group_max();
size_t batch_group_state_bytes();  // per space: group barrier + member partials
int batch_group_max_np();
size_t batch_job_bytes();
int batch_group_resident(int num_sms);
void batch_set_job(void* jobs_host, size_t idx, int item, int member, int g);
cudaError_t launch_batch_group(const void* descs_dev, const void* jobs_dev, int waves, int grid,
                               const BatchParams& P, cudaStream_t stream);

// ---- random-walk validator (tk_descent.cu) ------------------------------------
constexpr int kMaxDescentSlots = 256;
struct DescentArgs {
    const double* fit;                 // rank-indexed fitness (failed = kFailFitness)
    unsigned long long n;              // nodes
    int dims;                          // the space's own dims (radix-1 dims included)
    int kind;                          // TK_HAMMING / TK_ADJACENT
    int slots;                         // build_slots size (<= kMaxDescentSlots)
    int restart_scan;
    unsigned long long walkers, seed;
    uint32_t radix[kMaxDims];
    unsigned long long stride[kMaxDims];
    uint8_t slot_dim[kMaxDescentSlots];
    int16_t slot_alt[kMaxDescentSlots];
    uint32_t* counts;                  // N arrivals per end rank (zeroed by the caller)
    unsigned long long* evaluations;   // fitness lookups (zeroed by the caller)
};
cudaError_t launch_descents(const DescentArgs& a, int num_sms, cudaStream_t stream);
cudaError_t launch_gather_counts(const uint32_t* idx, uint64_t m, const uint32_t* counts,
                                 unsigned long long* out, cudaStream_t stream);

}  // namespace tk
