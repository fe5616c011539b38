// tk_kernels.cu -- sm_100a kernels for the FFG / PageRank / C_p hot path.
//
// Reference semantics (paths relative to /root/reference/proj):
//   neighbour order       src/space.cpp:167-187      (Adjacent: x-1 then x+1)
//   FFG edge rule         include/tunekit/landscape.hpp:26-29
//   PageRank              include/tunekit/landscape.hpp:47-52
//   C_p                   include/tunekit/landscape.hpp:54-58
//   f_opt                 src/cache.cpp:55-72
//   hash_uniform          src/generators.cpp:11-23
// and the pinned decisions of SURVEY.md Appendix A.  All floating point uses
// explicit _rn intrinsics (no FMA contraction) so per-node results round
// exactly like oracle/oracle.c; only global reductions differ in order.
#include <cooperative_groups.h>

#include "tk_kernels.cuh"

namespace cg = cooperative_groups;

namespace tk {

namespace {

// ------------------------------------------------------------------ helpers --

__device__ __forceinline__ int popc(uint32_t x) { return __popc(x); }
__device__ __forceinline__ int popc(unsigned long long x) { return __popcll(x); }
__device__ __forceinline__ int lowbit(uint32_t x) { return __ffs(x) - 1; }
__device__ __forceinline__ int lowbit(unsigned long long x) { return __ffsll(x) - 1; }

// src/generators.cpp:11-16
__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// src/generators.cpp:20-23 -- exact: integer mix, u64->f64 of a 53-bit value,
// multiply by 2^-53.
__device__ __forceinline__ double hash_uniform(unsigned long long seed, unsigned long long rank,
                                               unsigned long long slot) {
    const unsigned long long h = mix64(seed ^ mix64(rank * 0x2545f4914f6cdd1dULL + slot));
    return __dmul_rn(__ull2double_rn(h >> 11), 0x1.0p-53);
}

constexpr unsigned long long kEmpty = ~0ull;

// Open-addressing probe sequence of the valid-set hash table (tk_land_lookup).
// Probes 0..3 keep the locality-preserving pattern: 32 consecutive keys share
// one hashed 32-slot run, so a warp probing consecutive ranks reads one
// contiguous 256 B segment of keys, and a taken slot moves to the same
// position of the next run, so a displaced group moves together.  Those
// probes never leave the key's residue class mod 32, and constraint-shaped
// valid sets (trailing parameters fixed, keys = 0 mod 4 or mod 32) fill a
// class long before the table is full -- so from probe 4 on the sequence is
// double hashing over the whole table: h1 + j*h2 with h2 odd and the capacity
// a power of two visits every slot once in cap probes.  The table is sized to
// >= 2x its keys, so build and lookup always meet an empty slot; kProbeCap
// only guards the loops against a corrupted table (error flag, no spin).
__device__ __forceinline__ unsigned long long hprobe(unsigned long long key, unsigned long long j,
                                                    unsigned long long mask) {
    if (j < 4) return (((mix64(key >> 5) + j) << 5) | (key & 31ull)) & mask;
    const unsigned long long h1 = mix64(key ^ 0x6a09e667f3bcc909ULL);
    const unsigned long long h2 = mix64(key + 0xbb67ae8584caa73bULL) | 1ull;
    return (h1 + (j - 4) * h2) & mask;
}

template <typename T>
__device__ __forceinline__ T grid_stride_begin() {
    return static_cast<T>(blockIdx.x) * blockDim.x + threadIdx.x;
}

int grid_for(uint64_t n, int threads, int cap) {
    uint64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > static_cast<uint64_t>(cap)) b = cap;
    return static_cast<int>(b);
}

// ------------------------------------------------------------- ingestion --

__global__ void generate_kernel(int gen, uint32_t n, double q, unsigned long long seed,
                                double* __restrict__ fit, uint8_t* __restrict__ ok) {
    for (uint64_t r = grid_stride_begin<uint64_t>(); r < n;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const bool good = !(hash_uniform(seed, r, 0) < q);
        double f = kFailFitness;
        if (good) {
            const double u1 = hash_uniform(seed, r, 1);
            f = gen == TK_GEN_IID ? __dadd_rn(1.0, u1) : __ddiv_rn(1.0, __dsub_rn(1.0, u1));
        }
        fit[r] = f;
        ok[r] = good ? 1 : 0;
    }
}

struct EncodeParams {
    int dims;
    uint32_t radix[kMaxDims];
    unsigned long long stride[kMaxDims];
};

// space.cpp:72-78 rank_of (with require_valid, space.cpp:55-70)
__global__ void encode_kernel(const int32_t* __restrict__ cfg, uint64_t nv, EncodeParams p,
                              unsigned long long* __restrict__ keys, int* err) {
    for (uint64_t i = grid_stride_begin<uint64_t>(); i < nv;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        unsigned long long k = 0;
        bool bad = false;
        for (int d = 0; d < p.dims; ++d) {
            const int32_t x = cfg[i * p.dims + d];
            bad |= x < 0 || static_cast<uint32_t>(x) >= p.radix[d];
            k += static_cast<unsigned long long>(x) * p.stride[d];
        }
        if (bad) atomicExch(err, 1);
        keys[i] = bad ? kEmpty : k;
    }
}

// ---- valid set -> dense rank-indexed table (load_sparse / load_configs) ----
// Keys are mixed-radix ranks < N (space.cpp:72-78), so the rank-indexed
// table the FFG reads anyway is a perfect hash of the valid set: the load
// fills every rank with the failed entry (cache.hpp:15) and scatters the
// valid pairs straight into it.  A bitmap of N bits (L2-resident: 14 MB at
// C5) claims each key with one atomicOr, which detects duplicates.

__global__ void fill_failed_kernel(uint32_t n, double* __restrict__ fit) {
    for (uint64_t u = grid_stride_begin<uint64_t>(); u < n;
         u += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        fit[u] = kFailFitness;
}

// A fitness the FFG count kernel's sign-of-difference compares cannot take:
// not finite (NaN, +-inf) or -0 (tk_land::fit_clean, err bit 16).
__device__ __forceinline__ bool unclean(double f) {
    const unsigned long long b = __double_as_longlong(f);
    return ((b >> 52) & 0x7ff) == 0x7ff || b == 0x8000000000000000ull;
}

// err bits: 1 key outside the space, 2 duplicate key, 4 mean >= kFailFitness
// (decision A11: an ok mean must order below every failed point), 16 a mean
// that is not finite or is -0 (unclean)
__global__ void valid_scatter_kernel(const unsigned long long* __restrict__ keys,
                                     const double* __restrict__ vals, uint64_t nv, uint64_t n,
                                     double* __restrict__ fit, uint8_t* __restrict__ ok,
                                     unsigned int* __restrict__ claimed, int* err) {
    for (uint64_t i = grid_stride_begin<uint64_t>(); i < nv;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long k = keys[i];
        const double v = vals[i];
        if (k >= n) {
            atomicOr(err, 1);
            continue;
        }
        if (v >= kFailFitness) atomicOr(err, 4);
        if (unclean(v)) atomicOr(err, 16);
        const unsigned int bit = 1u << (k & 31);
        const unsigned int old = atomicOr(claimed + (k >> 5), bit);
        if (old & bit) {
            atomicOr(err, 2);
            continue;
        }
        fit[k] = v;
        ok[k] = 1;
    }
}

// load_dense: failed entries are forced to kFailFitness (cache.cpp:49-53
// set_failed) and an ok mean >= kFailFitness is rejected (A11).
__global__ void normalize_dense_kernel(uint32_t n, double* __restrict__ fit,
                                       const uint8_t* __restrict__ ok, int* err) {
    bool bad = false, dirty = false;
    for (uint64_t u = grid_stride_begin<uint64_t>(); u < n;
         u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double f = fit[u];
        if (ok[u]) {
            bad |= f >= kFailFitness;
            dirty |= unclean(f);
        } else if (!(f == kFailFitness)) {
            fit[u] = kFailFitness;
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 4);
    if (__any_sync(0xffffffffu, dirty) && (threadIdx.x & 31) == 0) atomicOr(err, 16);
}

__global__ void count_ok_kernel(const uint8_t* __restrict__ ok, uint32_t n,
                                unsigned long long* count) {
    unsigned int c = 0;
    for (uint64_t u = grid_stride_begin<uint64_t>(); u < n;
         u += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        c += ok[u] ? 1u : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, static_cast<unsigned long long>(c));
}

// ---- open-addressing hash table of the valid set (tk_land_lookup) ----
// Built from the dense table's ok ranks; every probe loop is bounded.
constexpr unsigned long long kProbeCap = 1ull << 40;

__global__ void hash_build_kernel(const double* __restrict__ fit, const uint8_t* __restrict__ ok,
                                  uint32_t n, unsigned long long* hkeys, double* hvals,
                                  unsigned long long mask, int* err) {
    for (uint64_t u = grid_stride_begin<uint64_t>(); u < n;
         u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (!ok[u]) continue;
        const unsigned long long k = u;
        const unsigned long long limit = 4 + mask + 1;
        unsigned long long j = 0;
        for (; j < limit && j < kProbeCap; ++j) {
            const unsigned long long s = hprobe(k, j, mask);
            const unsigned long long prev = atomicCAS(hkeys + s, kEmpty, k);
            if (prev == kEmpty) {
                hvals[s] = fit[u];
                break;
            }
        }
        if (j == limit) atomicOr(err, 8);  // table full: cannot happen at cap >= 2 * keys
    }
}

__global__ void hash_lookup_kernel(const unsigned long long* __restrict__ hkeys,
                                   const double* __restrict__ hvals, unsigned long long mask,
                                   const unsigned long long* __restrict__ q, uint64_t nq,
                                   double* __restrict__ out, uint8_t* __restrict__ found,
                                   int* err) {
    for (uint64_t i = grid_stride_begin<uint64_t>(); i < nq;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long key = q[i];
        double f = kFailFitness;
        uint8_t hit = 0;
        if (key != kEmpty) {
            const unsigned long long limit = 4 + mask + 1;
            unsigned long long j = 0;
            for (; j < limit; ++j) {
                const unsigned long long s = hprobe(key, j, mask);
                const unsigned long long k = hkeys[s];
                if (k == key) {
                    f = hvals[s];
                    hit = 1;
                    break;
                }
                if (k == kEmpty) break;
            }
            if (j == limit) atomicOr(err, 8);
        }
        out[i] = f;
        found[i] = hit;
    }
}

// cache.cpp:55-72: minimum over ok entries, strict <, lowest rank on ties.
struct ArgMin {
    double f;
    unsigned long long r;  // ~0 = none
};
__device__ __forceinline__ ArgMin amin(ArgMin a, ArgMin b) {
    if (b.r == kEmpty) return a;
    if (a.r == kEmpty) return b;
    if (b.f < a.f || (b.f == a.f && b.r < a.r)) return b;
    return a;
}
__device__ __forceinline__ ArgMin amin_shfl(ArgMin a, int o) {
    ArgMin b;
    b.f = __shfl_xor_sync(0xffffffffu, a.f, o);
    b.r = __shfl_xor_sync(0xffffffffu, a.r, o);
    return amin(a, b);
}

template <int THREADS>
__device__ ArgMin block_amin(ArgMin a) {
    __shared__ double sf[THREADS / 32];
    __shared__ unsigned long long sr[THREADS / 32];
    for (int o = 16; o; o >>= 1) a = amin_shfl(a, o);
    if ((threadIdx.x & 31) == 0) {
        sf[threadIdx.x >> 5] = a.f;
        sr[threadIdx.x >> 5] = a.r;
    }
    __syncthreads();
    ArgMin t{0.0, kEmpty};
    for (int w = 0; w < THREADS / 32; ++w) t = amin(t, ArgMin{sf[w], sr[w]});
    __syncthreads();
    return t;
}

__global__ void __launch_bounds__(256) optimum_partial_kernel(
    const double* __restrict__ fit, const uint8_t* __restrict__ ok, uint32_t n,
    double* part_f, unsigned long long* part_r) {
    ArgMin a{0.0, kEmpty};
    for (uint64_t u = grid_stride_begin<uint64_t>(); u < n;
         u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (ok[u]) a = amin(a, ArgMin{fit[u], u});
    }
    a = block_amin<256>(a);
    if (threadIdx.x == 0) {
        part_f[blockIdx.x] = a.f;
        part_r[blockIdx.x] = a.r;
    }
}

__global__ void __launch_bounds__(256) optimum_final_kernel(
    const double* part_f, const unsigned long long* part_r, int nparts, double* f_opt,
    unsigned long long* rank, int* has) {
    ArgMin a{0.0, kEmpty};
    for (int i = threadIdx.x; i < nparts; i += 256) a = amin(a, ArgMin{part_f[i], part_r[i]});
    a = block_amin<256>(a);
    if (threadIdx.x == 0) {
        *has = a.r != kEmpty;
        *f_opt = a.f;
        *rank = a.r;
    }
}

// ------------------------------------------------------------------- FFG --
//
// One fused pass per node u (one thread), tiles taken in ticket order:
//   * probe every neighbour slot (space.cpp:167-187 order), compare fitness;
//   * out-mask (canonical slot order) -> out-degree, sink, minimum flags;
//   * in-mask for pull PageRank: Adjacent uses the *ordered* layout (bit j =
//     j-th in-neighbour in ascending rank), Hamming the canonical layout;
//   * block scans + decoupled look-back give each row its CSR offset and each
//     minimum its slot; the row's targets are emitted in canonical order.
template <int KIND, typename MW, bool PACKED, bool EMIT>
__global__ void __launch_bounds__(kBuildThreads) ffg_build_kernel(const DevShape s,
                                                                  const BuildArgs a) {
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_ebase, s_mbase;
    __shared__ uint32_t s_scan_e[kBuildThreads / 32];
    __shared__ uint32_t s_scan_m[kBuildThreads / 32];
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counter, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= a.ntiles) return;
        const uint32_t u = tile * kBuildThreads + threadIdx.x;
        const bool valid = u < s.n;
        MW om = 0, im = 0;
        bool notgt = false;  // some neighbour not strictly greater (== or NaN)
        uint8_t okv = 0;
        if (valid) {
            const double fu = a.fit[u];
            okv = a.ok[u];
            uint32_t rem = u;
            if (KIND == TK_ADJACENT) {
                const int d2 = 2 * s.dims - 1;
#pragma unroll 4
                for (int i = 0; i < s.dims; ++i) {
                    const uint32_t st = s.stride[i];
                    const uint32_t x = fdiv(rem, s.magic[i]);
                    rem -= x * st;
                    const bool lo = x > 0, hi = x + 1 < s.radix[i];
                    const double fl = lo ? a.fit[u - st] : fu;
                    const double fh = hi ? a.fit[u + st] : fu;
                    om |= (static_cast<MW>(fl < fu) << (2 * i)) |
                          (static_cast<MW>(fh < fu) << (2 * i + 1));
                    im |= (static_cast<MW>(fl > fu) << i) |
                          (static_cast<MW>(fh > fu) << (d2 - i));
                    notgt |= (lo && !(fl > fu)) || (hi && !(fh > fu));
                }
            } else {
                for (int i = 0; i < s.dims; ++i) {
                    const uint32_t st = s.stride[i];
                    const uint32_t x = fdiv(rem, s.magic[i]);
                    rem -= x * st;
                    const uint32_t m = s.radix[i];
                    const uint32_t row = u - x * st;
                    int b = s.base[i];
#pragma unroll 4
                    for (uint32_t j = 0; j < m; ++j) {
                        if (j == x) continue;
                        const double f = a.fit[row + j * st];
                        om |= static_cast<MW>(f < fu) << b;
                        im |= static_cast<MW>(f > fu) << b;
                        notgt |= !(f > fu);
                        ++b;
                    }
                }
            }
        }
        const uint32_t deg = valid ? static_cast<uint32_t>(popc(om)) : 0u;
        const bool sink = valid && deg == 0;
        const bool fmin = sink && okv;
        // census minimum: ok and every neighbour strictly greater
        const bool strict = fmin && !notgt;
        uint32_t etot = 0, mtot = 0;
        uint32_t epos = 0;
        if (EMIT) epos = block_exclusive_scan<kBuildThreads, uint32_t>(deg, etot, s_scan_e);
        const uint32_t mpos =
            block_exclusive_scan<kBuildThreads, uint32_t>(fmin ? 1u : 0u, mtot, s_scan_m);
        const int scount = __syncthreads_count(strict);
        const int okcount = __syncthreads_count(valid && okv);
        uint32_t esum = 0;
        if (!EMIT) {
            // edge total only: warp sums + one atomic per warp
            uint32_t w = deg;
            for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
            esum = w;
        }
        if (threadIdx.x == 0) {
            s_ebase = EMIT ? lookback(a.e_status, tile, etot) : 0ull;
            s_mbase = lookback(a.m_status, tile, mtot);
            if (scount) atomicAdd(a.totals + 2, static_cast<unsigned long long>(scount));
            if (okcount) atomicAdd(a.totals + 3, static_cast<unsigned long long>(okcount));
        }
        if (!EMIT && (threadIdx.x & 31) == 0 && esum)
            atomicAdd(a.totals, static_cast<unsigned long long>(esum));
        __syncthreads();
        if (valid) {
            if (PACKED) {
                a.pw[u] = static_cast<uint32_t>(im) | (deg << kPackedSlots);
            } else {
                static_cast<MW*>(a.inm)[u] = im;
                a.odeg[u] = static_cast<uint8_t>(deg);
            }
            a.flags[u] = static_cast<uint8_t>((sink ? 1 : 0) | (fmin ? 2 : 0) |
                                              (strict ? 4 : 0) | (okv ? 8 : 0));
            if (EMIT) {
                const unsigned long long off = s_ebase + epos;
                a.offsets[u] = off;
                uint32_t* t = a.targets + off;
                if (KIND == TK_ADJACENT) {
                    MW mm = om;
                    while (mm) {
                        const int b = lowbit(mm);
                        mm &= mm - 1;
                        const uint32_t st = s.stride[b >> 1];
                        *t++ = (b & 1) ? u + st : u - st;
                    }
                } else {
                    uint32_t rem = u;
                    for (int i = 0; i < s.dims && om; ++i) {
                        const uint32_t st = s.stride[i];
                        const uint32_t x = fdiv(rem, s.magic[i]);
                        rem -= x * st;
                        const int m1 = static_cast<int>(s.radix[i]) - 1;
                        const MW fmask = m1 >= static_cast<int>(sizeof(MW) * 8)
                                             ? ~static_cast<MW>(0)
                                             : ((static_cast<MW>(1) << m1) - 1);
                        MW field = (om >> s.base[i]) & fmask;
                        const uint32_t row = u - x * st;
                        while (field) {
                            const uint32_t k = static_cast<uint32_t>(lowbit(field));
                            field &= field - 1;
                            const uint32_t j = k < x ? k : k + 1;
                            *t++ = row + j * st;
                        }
                    }
                }
            }
            if (fmin) a.minima[s_mbase + mpos] = u;
            if (u == s.n - 1) {
                if (EMIT) {
                    const unsigned long long e = s_ebase + epos + deg;
                    a.offsets[s.n] = e;
                    a.totals[0] = e;
                }
                a.totals[1] = s_mbase + mpos + (fmin ? 1 : 0);
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) compact_flags_kernel(
    const uint8_t* __restrict__ flags, uint8_t mask, uint32_t n,
    unsigned long long* __restrict__ out, unsigned long long* status,
    unsigned int* tile_counter, uint32_t ntiles) {
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_base;
    __shared__ uint32_t s_scan[8];
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= ntiles) return;
        const uint32_t u = tile * 256 + threadIdx.x;
        const uint32_t f = (u < n && (flags[u] & mask)) ? 1u : 0u;
        uint32_t tot;
        const uint32_t pos = block_exclusive_scan<256, uint32_t>(f, tot, s_scan);
        if (threadIdx.x == 0) s_base = lookback(status, tile, tot);
        __syncthreads();
        if (f) out[s_base + pos] = u;
        __syncthreads();
    }
}

__global__ void flags_to_sink_kernel(const uint8_t* __restrict__ flags, uint32_t n,
                                     uint8_t* __restrict__ is_sink) {
    for (uint64_t u = grid_stride_begin<uint64_t>(); u < n;
         u += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        is_sink[u] = flags[u] & 1;
}

// --------------------------------------------------------- CSR transpose --

__global__ void csr_prepare_kernel(uint32_t n, const unsigned long long* __restrict__ off,
                                   const uint32_t* __restrict__ tg, uint64_t e,
                                   uint32_t* __restrict__ odeg, uint32_t* indeg) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t u = grid_stride_begin<uint64_t>(); u < n; u += stride)
        odeg[u] = static_cast<uint32_t>(off[u + 1] - off[u]);
    for (uint64_t i = grid_stride_begin<uint64_t>(); i < e; i += stride)
        atomicAdd(indeg + tg[i], 1u);
}

__global__ void __launch_bounds__(256) scan_u32_kernel(
    const uint32_t* __restrict__ in, uint32_t n, unsigned long long* __restrict__ out,
    unsigned long long* status, unsigned int* tile_counter, uint32_t ntiles) {
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_base;
    __shared__ unsigned long long s_scan[8];
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= ntiles) return;
        const uint32_t u = tile * 256 + threadIdx.x;
        const unsigned long long v = u < n ? in[u] : 0ull;
        unsigned long long tot;
        const unsigned long long pos = block_exclusive_scan<256, unsigned long long>(v, tot, s_scan);
        if (threadIdx.x == 0) s_base = lookback(status, tile, tot);
        __syncthreads();
        if (u < n) out[u] = s_base + pos;
        if (u == n - 1) out[n] = s_base + pos + v;
        __syncthreads();
    }
}

__global__ void csr_scatter_kernel(uint32_t n, const unsigned long long* __restrict__ off,
                                   const uint32_t* __restrict__ tg,
                                   const unsigned long long* __restrict__ in_off,
                                   uint32_t* cursor, uint32_t* __restrict__ src) {
    for (uint64_t u = grid_stride_begin<uint64_t>(); u < n;
         u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        for (unsigned long long i = off[u]; i < off[u + 1]; ++i) {
            const uint32_t t = tg[i];
            const uint32_t p = atomicAdd(cursor + t, 1u);
            src[in_off[t] + p] = static_cast<uint32_t>(u);
        }
    }
}

// rows of an FFG in-CSR hold at most 64 sources; shell sort keeps large rows
// of arbitrary graphs correct (ascending source order = push order).
__global__ void csr_sort_rows_kernel(uint32_t n, const unsigned long long* __restrict__ in_off,
                                     uint32_t* __restrict__ src) {
    for (uint64_t v = grid_stride_begin<uint64_t>(); v < n;
         v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t* a = src + in_off[v];
        const long long len = static_cast<long long>(in_off[v + 1] - in_off[v]);
        for (long long gap = len / 2; gap > 0; gap /= 2)
            for (long long i = gap; i < len; ++i) {
                const uint32_t x = a[i];
                long long j = i;
                for (; j >= gap && a[j - gap] > x; j -= gap) a[j] = a[j - gap];
                a[j] = x;
            }
    }
}

// -------------------------------------------------------------- PageRank --
//
// Persistent cooperative kernel: the whole power iteration in one launch.
// Per iteration and node v (pull):
//   r'[v] = (1-d)/N + d * (sum_{u->v} c[u] + D/N),  c[u] = r[u] / outdeg(u)
// with the in-edge sum in ascending source rank (bit-identical to the
// oracle's push order), then c'[v] = r'[v] / outdeg(v) (sinks feed D).
// Residual, dangling mass and sum are reduced per block, published, and after
// one grid barrier every block reduces the per-block partials in the same
// fixed order, so all blocks take the same stop decision.

template <int MODE, typename MW>
__device__ __forceinline__ uint32_t pr_degree(const PrArgs& a, uint32_t v) {
    if (MODE == MODE_ADJ_PACKED) return __ldg(a.pw + v) >> kPackedSlots;
    if (MODE == MODE_CSR) return __ldg(a.odeg32 + v);
    return __ldg(a.odeg + v);
}

template <int MODE, typename MW>
__device__ __forceinline__ double pr_gather(const DevShape& s, const PrArgs& a, uint32_t v,
                                            const double* c, uint32_t& deg) {
    double acc = 0.0;
    if (MODE == MODE_ADJ_PACKED) {
        const uint32_t w = __ldg(a.pw + v);
        deg = w >> kPackedSlots;
        const uint32_t mask = w & ((1u << kPackedSlots) - 1);
        double vals[kPackedSlots];
#pragma unroll
        for (int j = 0; j < kPackedSlots; ++j)
            vals[j] = ((mask >> j) & 1u) ? c[v + s.nbo[j]] : 0.0;
#pragma unroll
        for (int j = 0; j < kPackedSlots; ++j)
            if ((mask >> j) & 1u) acc = __dadd_rn(acc, vals[j]);
    } else if (MODE == MODE_ADJ_ORDERED) {
        const MW mask = __ldg(static_cast<const MW*>(a.inm) + v);
        deg = __ldg(a.odeg + v);
        const int S = s.slots;
        for (int j0 = 0; j0 < S; j0 += 8) {
            double vals[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int j = j0 + k;
                vals[k] = (j < S && ((mask >> j) & 1)) ? c[v + s.nbo[j]] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int j = j0 + k;
                if (j < S && ((mask >> j) & 1)) acc = __dadd_rn(acc, vals[k]);
            }
        }
    } else if (MODE == MODE_HAM) {
        const MW mask = __ldg(static_cast<const MW*>(a.inm) + v);
        deg = __ldg(a.odeg + v);
        if (mask) {
            uint32_t x[kMaxDims];
            uint32_t rem = v;
            for (int i = 0; i < s.dims; ++i) {
                x[i] = fdiv(rem, s.magic[i]);
                rem -= x[i] * s.stride[i];
            }
            // lower neighbours: dims ascending, values ascending (ranks ascending)
            for (int i = 0; i < s.dims; ++i) {
                const uint32_t st = s.stride[i];
                const uint32_t row = v - x[i] * st;
                const int b0 = s.base[i];
#pragma unroll 4
                for (uint32_t j = 0; j < x[i]; ++j)
                    if ((mask >> (b0 + j)) & 1) acc = __dadd_rn(acc, c[row + j * st]);
            }
            // upper neighbours: dims descending, values ascending
            for (int i = s.dims - 1; i >= 0; --i) {
                const uint32_t st = s.stride[i];
                const uint32_t row = v - x[i] * st;
                const int b0 = s.base[i] - 1;  // value j > x sits at bit base + j - 1
#pragma unroll 4
                for (uint32_t j = x[i] + 1; j < s.radix[i]; ++j)
                    if ((mask >> (b0 + j)) & 1) acc = __dadd_rn(acc, c[row + j * st]);
            }
        }
    } else {  // MODE_CSR
        deg = __ldg(a.odeg32 + v);
        const unsigned long long b = __ldg(a.in_off + v), e = __ldg(a.in_off + v + 1);
        for (unsigned long long i = b; i < e; ++i) acc = __dadd_rn(acc, c[__ldg(a.src + i)]);
    }
    return acc;
}

__device__ __forceinline__ double reduce_parts(const double* part, int nblocks, int k,
                                               double* s_red) {
    double t = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += kPrThreads) t = __dadd_rn(t, part[b * 3 + k]);
    return block_sum<kPrThreads>(t, s_red);
}

template <int MODE, typename MW>
__global__ void __launch_bounds__(kPrThreads) pagerank_kernel(const DevShape s,
                                                              const PrArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double s_red[kPrThreads / 32];
    const uint32_t G = gridDim.x;
    const uint64_t gsize = static_cast<uint64_t>(G) * kPrThreads;
    const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * kPrThreads + threadIdx.x;

    // r_0 = 1/N, c_0 = r_0 / outdeg, D_0 = sum over sinks
    double dang = 0.0;
    for (uint64_t v = gtid; v < a.n; v += gsize) {
        const uint32_t deg = pr_degree<MODE, MW>(a, static_cast<uint32_t>(v));
        a.r0[v] = a.inv_n;
        if (deg) {
            a.c0[v] = __ddiv_rn(a.inv_n, static_cast<double>(deg));
        } else {
            a.c0[v] = 0.0;
            dang = __dadd_rn(dang, a.inv_n);
        }
    }
    dang = block_sum<kPrThreads>(dang, s_red);
    if (threadIdx.x == 0) a.part[blockIdx.x * 3 + 1] = dang;
    grid.sync();
    double D = reduce_parts(a.part, G, 1, s_red);

    int cur = 0;
    long long it = 0;
    double res = 0.0, sum = 0.0;
    int status = 1;
    while (it < a.max_iter) {
        const double dn = __ddiv_rn(D, a.nd);
        const double* rc = cur ? a.r1 : a.r0;
        const double* cc = cur ? a.c1 : a.c0;
        double* rn = cur ? a.r0 : a.r1;
        double* cn = cur ? a.c0 : a.c1;
        double lres = 0.0, ldang = 0.0, lsum = 0.0;
        for (uint64_t v = gtid; v < a.n; v += gsize) {
            uint32_t deg;
            const double acc = pr_gather<MODE, MW>(s, a, static_cast<uint32_t>(v), cc, deg);
            const double x = __dadd_rn(a.teleport, __dmul_rn(a.damping, __dadd_rn(acc, dn)));
            lres = __dadd_rn(lres, fabs(__dsub_rn(x, rc[v])));
            lsum = __dadd_rn(lsum, x);
            rn[v] = x;
            if (deg) {
                cn[v] = __ddiv_rn(x, static_cast<double>(deg));
            } else {
                cn[v] = 0.0;
                ldang = __dadd_rn(ldang, x);
            }
        }
        lres = block_sum<kPrThreads>(lres, s_red);
        ldang = block_sum<kPrThreads>(ldang, s_red);
        lsum = block_sum<kPrThreads>(lsum, s_red);
        double* part = a.part + static_cast<size_t>((it + 1) & 1) * G * 3;
        if (threadIdx.x == 0) {
            part[blockIdx.x * 3 + 0] = lres;
            part[blockIdx.x * 3 + 1] = ldang;
            part[blockIdx.x * 3 + 2] = lsum;
        }
        grid.sync();
        res = reduce_parts(part, G, 0, s_red);
        D = reduce_parts(part, G, 1, s_red);
        sum = reduce_parts(part, G, 2, s_red);
        ++it;
        cur ^= 1;
        if (res < a.tol) {
            status = 0;
            break;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.out_iter = it;
        *a.out_res = res;
        *a.out_sum = sum;
        *a.out_parity = cur;
        *a.out_status = status;
    }
}

// ---------------------------------------------------------------- C_p --

struct CpParams {
    int n_p;
    double f_opt;
    double thr[TK_MAX_CP];
    int zero[TK_MAX_CP];
};

// One pass over the minima per block row: row y accumulates p = 16y .. 16y+15
// in registers, row 0 also the denominator (stored at p index n_p).
constexpr int kCpPerRow = 16;
__global__ void __launch_bounds__(256) cp_partial_kernel(
    const uint32_t* __restrict__ minima, uint64_t m, const double* __restrict__ fit,
    const double* __restrict__ r, const CpParams P, double* __restrict__ part) {
    __shared__ double s_red[8];
    const int p0 = blockIdx.y * kCpPerRow;
    double acc[kCpPerRow];
#pragma unroll
    for (int j = 0; j < kCpPerRow; ++j) acc[j] = 0.0;
    double den = 0.0;
    for (uint64_t i = grid_stride_begin<uint64_t>(); i < m;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t idx = minima ? __ldg(minima + i) : i;
        const double f = __ldg(fit + idx);
        const double pr = __ldg(r + idx);
        den = __dadd_rn(den, pr);
#pragma unroll
        for (int j = 0; j < kCpPerRow; ++j) {
            const int p = p0 + j;
            if (p < P.n_p && (P.zero[p] ? (f <= P.f_opt) : (f < P.thr[p])))
                acc[j] = __dadd_rn(acc[j], pr);
        }
    }
#pragma unroll
    for (int j = 0; j < kCpPerRow; ++j) {
        const double s = block_sum<256>(acc[j], s_red);
        if (threadIdx.x == 0 && p0 + j < P.n_p)
            part[static_cast<size_t>(p0 + j) * gridDim.x + blockIdx.x] = s;
    }
    den = block_sum<256>(den, s_red);
    if (threadIdx.x == 0 && blockIdx.y == 0)
        part[static_cast<size_t>(P.n_p) * gridDim.x + blockIdx.x] = den;
}

// raw = 1 writes the sums (n_p numerators, then the denominator) instead of
// the ratios: a shard's partials for the cross-GPU sum.
// One block per p (block n_p: the denominator only): each block sums the
// partial row of its p and the denominator row with a fixed thread-strided
// assignment and a fixed tree, so the result is deterministic run to run.
__global__ void __launch_bounds__(256) cp_final_kernel(const double* __restrict__ part, int n_p,
                                                       int nblocks, double* __restrict__ c_p,
                                                       int* degenerate, int raw) {
    __shared__ double s_red[8];
    const int p = blockIdx.x;
    double num = 0.0, den = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += 256) {
        den = __dadd_rn(den, part[static_cast<size_t>(n_p) * nblocks + b]);
        if (p < n_p) num = __dadd_rn(num, part[static_cast<size_t>(p) * nblocks + b]);
    }
    den = block_sum<256>(den, s_red);
    num = block_sum<256>(num, s_red);
    if (threadIdx.x == 0) {
        if (p == n_p) {
            *degenerate = !(den > 0.0);
            if (raw) c_p[n_p] = den;
        } else {
            c_p[p] = raw ? num : __ddiv_rn(num, den);
        }
    }
}

__global__ void report_kernel(const uint32_t* __restrict__ minima, uint64_t m,
                              const double* __restrict__ fit, const double* __restrict__ r,
                              double f_opt, unsigned long long* __restrict__ ranks,
                              double* __restrict__ fitness, double* __restrict__ fraction,
                              double* __restrict__ pr) {
    for (uint64_t i = grid_stride_begin<uint64_t>(); i < m;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t u = minima[i];
        const double f = fit[u];
        if (ranks) ranks[i] = u;
        if (fitness) fitness[i] = f;
        if (fraction) fraction[i] = __ddiv_rn(f_opt, f);  // cache.cpp:100-106
        if (pr) pr[i] = r[u];
    }
}

__global__ void gather_values_kernel(const uint32_t* __restrict__ idx, uint64_t m,
                                     const double* __restrict__ src, double* __restrict__ dst) {
    for (uint64_t i = grid_stride_begin<uint64_t>(); i < m;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[idx[i]];
}

}  // namespace

// =============================================================== launchers ==

cudaError_t launch_generate(int gen, uint32_t n, double q, uint64_t seed, double* fit,
                            uint8_t* ok, cudaStream_t stream) {
    generate_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, stream>>>(gen, n, q, seed, fit, ok);
    return cudaGetLastError();
}

cudaError_t launch_encode_configs(const int32_t* configs, uint64_t n_valid, int dims_in,
                                  const uint32_t* radix_in, const unsigned long long* strides_in,
                                  unsigned long long* keys_out, int* err_flag,
                                  cudaStream_t stream) {
    EncodeParams p{};
    p.dims = dims_in;
    for (int i = 0; i < dims_in; ++i) {
        p.radix[i] = radix_in[i];
        p.stride[i] = strides_in[i];
    }
    encode_kernel<<<grid_for(n_valid, 256, 148 * 16), 256, 0, stream>>>(configs, n_valid, p,
                                                                        keys_out, err_flag);
    return cudaGetLastError();
}

// ---- bucketed ingest: the valid pairs partitioned by rank slice first, so the
// scatter into the dense table touches one L2-resident slice at a time ----
//
// The direct scatter (valid_scatter_kernel) writes 8- and 1-byte words at
// random ranks: every write is a 32-byte sector read-modify-write that misses
// L2 (14.8 GB of DRAM traffic for the 2.65 GB the C5 valid set needs).  Here
//   1. bucket_count_kernel   histogram of the keys' slices (2^ingest_shift ranks)
//   2. (host-side tiny scan of the bucket counts on the device, one block)
//   3. bucket_partition_kernel  (key, mean) pairs appended to their slice's run
//   4. valid_scatter_kernel over the partitioned pairs in order: the grid works
//      on one or two slices (~1.2 MB of table) at a time, so the sector
//      read-modify-writes hit L2.
constexpr int kIngestMaxBuckets = 1024;
// slices of >= 2^17 ranks (1.2 MB of fitness + ok), at most kIngestMaxBuckets of them
int ingest_shift(uint32_t n) {
    int sh = 17;
    while ((static_cast<uint64_t>(n) >> sh) + 1 > static_cast<uint64_t>(kIngestMaxBuckets)) ++sh;
    return sh;
}

__global__ void __launch_bounds__(256) bucket_count_kernel(
    const unsigned long long* __restrict__ keys, uint64_t nv, uint64_t n, int shift, uint32_t nb,
    unsigned int* __restrict__ counts, int* err) {
    __shared__ unsigned int h[kIngestMaxBuckets];
    for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) h[i] = 0;
    __syncthreads();
    bool bad = false;
    for (uint64_t i = grid_stride_begin<uint64_t>(); i < nv;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long k = keys[i];
        if (k >= n) {
            bad = true;
            continue;
        }
        atomicAdd(&h[k >> shift], 1u);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x)
        if (h[i]) atomicAdd(counts + i, h[i]);
}

// exclusive scan of nb <= 4096 counts into cursors (one block)
__global__ void __launch_bounds__(1024) bucket_scan_kernel(const unsigned int* __restrict__ counts,
                                                           uint32_t nb,
                                                           unsigned long long* __restrict__ cursor) {
    __shared__ unsigned long long s_warp[32];
    __shared__ unsigned long long s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < nb; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const unsigned long long v = i < nb ? counts[i] : 0ull;
        unsigned long long tot;
        const unsigned long long ex = block_exclusive_scan<1024, unsigned long long>(v, tot, s_warp);
        if (i < nb) cursor[i] = s_carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += tot;
        __syncthreads();
    }
}

// One 4096-pair chunk per block iteration: positions within the chunk from
// shared-memory atomics, one global cursor reservation per non-empty bucket
// and chunk (the per-pair global atomics of a naive partition serialise on the
// ~1,000 cursors).
constexpr int kPartPer = 16;  // pairs per thread and chunk
__global__ void __launch_bounds__(256) bucket_partition_kernel(
    const unsigned long long* __restrict__ keys, const double* __restrict__ vals, uint64_t nv,
    uint64_t n, int shift, uint32_t nb, unsigned long long* __restrict__ cursor,
    unsigned long long* __restrict__ out_keys, double* __restrict__ out_vals) {
    __shared__ unsigned int s_cnt[kIngestMaxBuckets];
    __shared__ unsigned long long s_base[kIngestMaxBuckets];
    constexpr uint64_t kChunk = 256ull * kPartPer;
    for (uint64_t c0 = static_cast<uint64_t>(blockIdx.x) * kChunk; c0 < nv;
         c0 += static_cast<uint64_t>(gridDim.x) * kChunk) {
        for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) s_cnt[i] = 0;
        __syncthreads();
        unsigned long long k[kPartPer];
        unsigned int r[kPartPer];
#pragma unroll
        for (int j = 0; j < kPartPer; ++j) {
            const uint64_t i = c0 + static_cast<uint64_t>(j) * 256 + threadIdx.x;
            k[j] = i < nv ? keys[i] : ~0ull;
            r[j] = k[j] < n ? atomicAdd(&s_cnt[k[j] >> shift], 1u) : 0u;
        }
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x)
            if (s_cnt[b]) s_base[b] = atomicAdd(cursor + b, static_cast<unsigned long long>(s_cnt[b]));
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kPartPer; ++j) {
            if (k[j] >= n) continue;  // out of range (reported by the count pass) or past the end
            const uint64_t i = c0 + static_cast<uint64_t>(j) * 256 + threadIdx.x;
            const unsigned long long pos = s_base[k[j] >> shift] + r[j];
            out_keys[pos] = k[j];
            out_vals[pos] = vals[i];
        }
        __syncthreads();
    }
}

uint32_t ingest_buckets(uint32_t n) { return (n >> ingest_shift(n)) + 1; }

cudaError_t launch_load_valid(const unsigned long long* keys, const double* vals,
                              uint64_t n_valid, uint32_t n, double* fit, uint8_t* ok,
                              unsigned int* claimed, int* err_flag, cudaStream_t stream,
                              void* scratch) {
    cudaError_t e = cudaMemsetAsync(ok, 0, n, stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(claimed, 0, ((n + 31ull) / 32) * 4, stream);
    if (e != cudaSuccess) return e;
    fill_failed_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, stream>>>(n, fit);
    if (!n_valid) return cudaGetLastError();
    const uint32_t nb = ingest_buckets(n);
    const int shift = ingest_shift(n);
    if (scratch && nb <= static_cast<uint32_t>(kIngestMaxBuckets)) {
        // scratch: nb u32 counts, nb u64 cursors, n_valid keys, n_valid means
        unsigned int* counts = static_cast<unsigned int*>(scratch);
        unsigned long long* cursor =
            reinterpret_cast<unsigned long long*>(counts + ((nb + 1) & ~1u));
        unsigned long long* pk = cursor + nb;
        double* pv = reinterpret_cast<double*>(pk + n_valid);
        e = cudaMemsetAsync(counts, 0, nb * 4, stream);
        if (e != cudaSuccess) return e;
        bucket_count_kernel<<<grid_for(n_valid, 256, 148 * 4), 256, 0, stream>>>(
            keys, n_valid, n, shift, nb, counts, err_flag);
        bucket_scan_kernel<<<1, 1024, 0, stream>>>(counts, nb, cursor);
        bucket_partition_kernel<<<grid_for(n_valid, 256 * kPartPer, 148 * 4), 256, 0, stream>>>(
            keys, vals, n_valid, n, shift, nb, cursor, pk, pv);
        keys = pk;
        vals = pv;
    }
    valid_scatter_kernel<<<grid_for(n_valid, 256, 148 * 16), 256, 0, stream>>>(
        keys, vals, n_valid, n, fit, ok, claimed, err_flag);
    return cudaGetLastError();
}

size_t load_valid_scratch_bytes(uint64_t n_valid, uint32_t n) {
    const uint32_t nb = ingest_buckets(n);
    return static_cast<size_t>((nb + 1) & ~1u) * 4 + static_cast<size_t>(nb) * 8 +
           static_cast<size_t>(n_valid) * 16;
}

cudaError_t launch_normalize_dense(uint32_t n, double* fit, const uint8_t* ok, int* err_flag,
                                   cudaStream_t stream) {
    normalize_dense_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, stream>>>(n, fit, ok, err_flag);
    return cudaGetLastError();
}

cudaError_t launch_count_ok(const uint8_t* ok, uint32_t n, unsigned long long* count,
                            cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(count, 0, 8, stream);
    if (e != cudaSuccess) return e;
    count_ok_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, stream>>>(ok, n, count);
    return cudaGetLastError();
}

cudaError_t launch_hash_build(const double* fit, const uint8_t* ok, uint32_t n,
                              unsigned long long* hkeys, double* hvals, uint64_t cap,
                              int* err_flag, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(hkeys, 0xFF, cap * 8, stream);
    if (e != cudaSuccess) return e;
    hash_build_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, stream>>>(fit, ok, n, hkeys, hvals,
                                                                     cap - 1, err_flag);
    return cudaGetLastError();
}

cudaError_t launch_hash_lookup(const unsigned long long* hkeys, const double* hvals,
                               uint64_t cap, const unsigned long long* q, uint64_t nq,
                               double* out, uint8_t* found, int* err_flag, cudaStream_t stream) {
    hash_lookup_kernel<<<grid_for(nq, 256, 148 * 16), 256, 0, stream>>>(hkeys, hvals, cap - 1,
                                                                       q, nq, out, found,
                                                                       err_flag);
    return cudaGetLastError();
}

cudaError_t launch_optimum(const double* fit, const uint8_t* ok, uint32_t n, double* part_f,
                           unsigned long long* part_r, double* f_opt,
                           unsigned long long* rank, int* has, cudaStream_t stream) {
    const int g = grid_for(n, 256, 148 * 4);
    optimum_partial_kernel<<<g, 256, 0, stream>>>(fit, ok, n, part_f, part_r);
    optimum_final_kernel<<<1, 256, 0, stream>>>(part_f, part_r, g, f_opt, rank, has);
    return cudaGetLastError();
}

cudaError_t launch_optimum_final(const double* part_f, const unsigned long long* part_r,
                                 int nparts, double* f_opt, unsigned long long* rank, int* has,
                                 cudaStream_t stream) {
    optimum_final_kernel<<<1, 256, 0, stream>>>(part_f, part_r, nparts, f_opt, rank, has);
    return cudaGetLastError();
}

template <int KIND, typename MW, bool PACKED, bool EMIT>
static cudaError_t build_one(const DevShape& s, const BuildArgs& a, int num_sms,
                             cudaStream_t stream) {
    auto k = ffg_build_kernel<KIND, MW, PACKED, EMIT>;
    int bps = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, kBuildThreads, 0);
    if (e != cudaSuccess) return e;
    const int g = grid_for(a.ntiles, 1, (bps > 0 ? bps : 1) * num_sms);
    k<<<g, kBuildThreads, 0, stream>>>(s, a);
    return cudaGetLastError();
}

template <bool EMIT>
static cudaError_t build_dispatch(const DevShape& s, int mode, bool wide, const BuildArgs& a,
                                  int num_sms, cudaStream_t stream) {
    using u32 = uint32_t;
    using u64 = unsigned long long;
    if (mode == MODE_ADJ_PACKED) return build_one<TK_ADJACENT, u32, true, EMIT>(s, a, num_sms, stream);
    if (mode == MODE_ADJ_ORDERED)
        return wide ? build_one<TK_ADJACENT, u64, false, EMIT>(s, a, num_sms, stream)
                    : build_one<TK_ADJACENT, u32, false, EMIT>(s, a, num_sms, stream);
    return wide ? build_one<TK_HAMMING, u64, false, EMIT>(s, a, num_sms, stream)
                : build_one<TK_HAMMING, u32, false, EMIT>(s, a, num_sms, stream);
}

cudaError_t launch_ffg_build(const DevShape& s, int mode, bool wide, bool emit,
                             const BuildArgs& a, int num_sms, cudaStream_t stream) {
    return emit ? build_dispatch<true>(s, mode, wide, a, num_sms, stream)
                : build_dispatch<false>(s, mode, wide, a, num_sms, stream);
}

cudaError_t launch_compact_flags(const uint8_t* flags, uint8_t mask, uint32_t n,
                                 unsigned long long* out, unsigned long long* status,
                                 unsigned int* tile_counter, uint32_t ntiles, int num_sms,
                                 cudaStream_t stream) {
    compact_flags_kernel<<<grid_for(ntiles, 1, num_sms * 8), 256, 0, stream>>>(
        flags, mask, n, out, status, tile_counter, ntiles);
    return cudaGetLastError();
}

cudaError_t launch_flags_to_sink(const uint8_t* flags, uint32_t n, uint8_t* is_sink,
                                 cudaStream_t stream) {
    flags_to_sink_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, stream>>>(flags, n, is_sink);
    return cudaGetLastError();
}

cudaError_t launch_csr_prepare(uint32_t n, const unsigned long long* offsets,
                               const uint32_t* targets, uint64_t e, uint32_t* odeg32,
                               uint32_t* indeg, cudaStream_t stream) {
    csr_prepare_kernel<<<grid_for(n > e ? n : e, 256, 148 * 16), 256, 0, stream>>>(
        n, offsets, targets, e, odeg32, indeg);
    return cudaGetLastError();
}

// Wide variant for long inputs (the N/32 warp-slot counts of the FFG build):
// 4096 elements per look-back tile (16 per thread), so the serial look-back
// chain is 16x shorter than with one element per thread.
constexpr int kScanItems = 16;
__global__ void __launch_bounds__(256) scan_u32_wide_kernel(
    const uint32_t* __restrict__ in, uint32_t n, unsigned long long* __restrict__ out,
    unsigned long long* status, unsigned int* tile_counter, uint32_t ntiles) {
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_base;
    __shared__ unsigned long long s_scan[8];
    constexpr uint32_t kSpan = 256 * kScanItems;
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= ntiles) return;
        const uint32_t u0 = tile * kSpan + threadIdx.x * kScanItems;
        uint32_t v[kScanItems];
        unsigned long long sum = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            v[k] = u0 + k < n ? __ldg(in + u0 + k) : 0u;
            sum += v[k];
        }
        unsigned long long tot;
        const unsigned long long pos = block_exclusive_scan<256, unsigned long long>(sum, tot, s_scan);
        if (threadIdx.x == 0) s_base = lookback(status, tile, tot);
        __syncthreads();
        unsigned long long run = s_base + pos;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            if (u0 + k < n) out[u0 + k] = run;
            if (u0 + k == n - 1) out[n] = run + v[k];
            run += v[k];
        }
        __syncthreads();
    }
}

cudaError_t launch_exclusive_scan_u32(const uint32_t* in, uint32_t n, unsigned long long* out,
                                      unsigned long long* status, unsigned int* tile_counter,
                                      uint32_t ntiles, int num_sms, cudaStream_t stream) {
    if (n > 65536) {  // `ntiles` (and the status array) were sized for 256-element tiles
        const uint32_t wt = (n + 256 * kScanItems - 1) / (256 * kScanItems);
        scan_u32_wide_kernel<<<grid_for(wt, 1, num_sms * 8), 256, 0, stream>>>(
            in, n, out, status, tile_counter, wt);
        return cudaGetLastError();
    }
    scan_u32_kernel<<<grid_for(ntiles, 1, num_sms * 8), 256, 0, stream>>>(in, n, out, status,
                                                                          tile_counter, ntiles);
    return cudaGetLastError();
}

cudaError_t launch_csr_scatter(uint32_t n, const unsigned long long* offsets,
                               const uint32_t* targets, const unsigned long long* in_off,
                               uint32_t* cursor, uint32_t* src, cudaStream_t stream) {
    csr_scatter_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, stream>>>(n, offsets, targets,
                                                                      in_off, cursor, src);
    return cudaGetLastError();
}

cudaError_t launch_csr_sort_rows(uint32_t n, const unsigned long long* in_off, uint32_t* src,
                                 cudaStream_t stream) {
    csr_sort_rows_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, stream>>>(n, in_off, src);
    return cudaGetLastError();
}

template <int MODE, typename MW>
static void* pr_kernel_ptr() {
    return reinterpret_cast<void*>(pagerank_kernel<MODE, MW>);
}

static void* pr_select(int mode, bool wide) {
    using u32 = uint32_t;
    using u64 = unsigned long long;
    switch (mode) {
        case MODE_ADJ_PACKED: return pr_kernel_ptr<MODE_ADJ_PACKED, u32>();
        case MODE_ADJ_ORDERED:
            return wide ? pr_kernel_ptr<MODE_ADJ_ORDERED, u64>() : pr_kernel_ptr<MODE_ADJ_ORDERED, u32>();
        case MODE_HAM:
            return wide ? pr_kernel_ptr<MODE_HAM, u64>() : pr_kernel_ptr<MODE_HAM, u32>();
        default: return pr_kernel_ptr<MODE_CSR, u32>();
    }
}

int pagerank_max_grid(int mode, bool wide, int num_sms) {
    int bps = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, pr_select(mode, wide), kPrThreads, 0) !=
        cudaSuccess)
        return 0;
    return bps * num_sms;
}

cudaError_t launch_pagerank(const DevShape& s, int mode, bool wide, const PrArgs& a,
                            int num_sms, int* grid_out, cudaStream_t stream) {
    const int maxg = pagerank_max_grid(mode, wide, num_sms);
    if (maxg <= 0) return cudaErrorInvalidConfiguration;
    const uint64_t want = (static_cast<uint64_t>(a.n) + kPrThreads - 1) / kPrThreads;
    int g = static_cast<int>(want < static_cast<uint64_t>(maxg) ? want : maxg);
    if (g < 1) g = 1;
    *grid_out = g;
    DevShape sc = s;
    PrArgs ac = a;
    void* args[] = {&sc, &ac};
    return cudaLaunchCooperativeKernel(pr_select(mode, wide), dim3(g), dim3(kPrThreads), args, 0,
                                       stream);
}

cudaError_t launch_centrality(const uint32_t* minima, uint64_t m, const double* fit,
                              const double* r, const double* p, int n_p, double f_opt,
                              double* part, double* c_p_out, int* degenerate,
                              cudaStream_t stream, bool raw) {
    CpParams P{};
    P.n_p = n_p;
    P.f_opt = f_opt;
    for (int i = 0; i < n_p; ++i) {
        P.thr[i] = (1.0 + p[i]) * f_opt;  // host IEEE, same expression as the oracle
        P.zero[i] = p[i] == 0.0;
    }
    dim3 grid(kCpBlocks, (n_p + kCpPerRow - 1) / kCpPerRow);
    cp_partial_kernel<<<grid, 256, 0, stream>>>(minima, m, fit, r, P, part);
    cp_final_kernel<<<n_p + 1, 256, 0, stream>>>(part, n_p, kCpBlocks, c_p_out, degenerate,
                                                 raw ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_report(const uint32_t* minima, uint64_t m, const double* fit,
                          const double* r, double f_opt, unsigned long long* ranks,
                          double* fitness, double* fraction, double* pr,
                          cudaStream_t stream) {
    report_kernel<<<grid_for(m, 256, 148 * 16), 256, 0, stream>>>(minima, m, fit, r, f_opt,
                                                                 ranks, fitness, fraction, pr);
    return cudaGetLastError();
}

cudaError_t launch_gather_values(const uint32_t* idx, uint64_t m, const double* src,
                                 double* dst, cudaStream_t stream) {
    gather_values_kernel<<<grid_for(m, 256, 148 * 16), 256, 0, stream>>>(idx, m, src, dst);
    return cudaGetLastError();
}

}  // namespace tk
