/*
 * oracle.c -- CPU restatement of the reference's FFG / PageRank / C_p path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): the checker for the CUDA product
 * and the CPU baseline timed beside it.  Plain C99 + optional OpenMP.
 * Compiled with -ffp-contract=off so every floating-point expression rounds
 * exactly as written (the GPU side uses explicit _rn intrinsics to match).
 *
 * Every function cites the reference file:line it restates.  Paths are
 * relative to /root/reference/proj.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_FAIL_FITNESS 1.0e10 /* include/tunekit/cache.hpp:15 kFailFitness */
#define OR_MAX_DIMS 64

/* ---------------------------------------------------------------- space -- */

/* src/space.cpp:48-53: strides_[i] = prod_{j>i} m_j, size = strides_[0]*m_0 */
uint64_t or_space_strides(uint32_t dims, const uint32_t* radix, uint64_t* strides) {
    uint64_t s = 1;
    for (uint32_t i = dims; i-- > 0;) {
        strides[i] = s;
        s *= radix[i];
    }
    return s;
}

/* src/space.cpp:189-197 */
uint32_t or_max_neighbours(uint32_t dims, const uint32_t* radix, int kind) {
    uint32_t n = 0;
    for (uint32_t i = 0; i < dims; ++i) {
        uint32_t m1 = radix[i] - 1;
        n += kind == OR_HAMMING ? m1 : (m1 < 2 ? m1 : 2);
    }
    return n;
}

/* src/space.cpp:167-187: dimension ascending, then index ascending; Adjacent
 * emits x-1 before x+1.  Rank arithmetic base + j*stride. */
static uint32_t nbr_ranks(uint32_t dims, const uint32_t* radix, const uint64_t* strides,
                          uint64_t rank, int kind, uint64_t* out) {
    uint32_t k = 0;
    uint64_t rest = rank;
    for (uint32_t i = 0; i < dims; ++i) {
        const uint64_t s = strides[i];
        const int64_t xi = (int64_t)(rest / s);
        rest %= s;
        const int64_t m = radix[i];
        const uint64_t base = rank - (uint64_t)xi * s;
        if (kind == OR_HAMMING) {
            for (int64_t j = 0; j < m; ++j)
                if (j != xi) out[k++] = base + (uint64_t)j * s;
        } else {
            if (xi > 0) out[k++] = base + (uint64_t)(xi - 1) * s;
            if (xi + 1 < m) out[k++] = base + (uint64_t)(xi + 1) * s;
        }
    }
    return k;
}

uint32_t or_neighbour_ranks(uint32_t dims, const uint32_t* radix, uint64_t rank,
                            int kind, uint64_t* out) {
    uint64_t strides[OR_MAX_DIMS];
    or_space_strides(dims, radix, strides);
    return nbr_ranks(dims, radix, strides, rank, kind, out);
}

static int check_space(uint32_t dims, const uint32_t* radix, int kind) {
    if (dims == 0 || dims > OR_MAX_DIMS) return OR_EINVAL;
    if (kind != OR_HAMMING && kind != OR_ADJACENT) return OR_EINVAL;
    for (uint32_t i = 0; i < dims; ++i)
        if (radix[i] == 0) return OR_EINVAL;
    return OR_OK;
}

/* ------------------------------------------------------------------ FFG -- */

/* landscape.hpp:26-45.  A1: nodes are all N ranks (failed
 * ranks carry 1e10).  A2: u->v iff v in N(u) and f(v) < f(u), strict.
 * A3: row order is neighbour_ranks order.  A4: minima = ok && outdeg == 0,
 * ascending.  A9: N > node_limit -> InvalidArgument (OR_ELIMIT). */
/* Per-thread static chunk [lo, hi) of the node range. */
static void chunk_of(uint64_t n, int nt, int t, uint64_t* lo, uint64_t* hi) {
    const uint64_t q = n / (uint64_t)nt, r = n % (uint64_t)nt;
    *lo = (uint64_t)t * q + ((uint64_t)t < r ? (uint64_t)t : r);
    *hi = *lo + q + ((uint64_t)t < r ? 1 : 0);
}

/* nbr_ranks with the digits of `rank` already known (an odometer walks them
 * through a chunk, so the per-node div/mod of src/space.cpp:171-173 happens
 * once per chunk); same order as nbr_ranks. */
static uint32_t nbr_ranks_digits(uint32_t dims, const uint32_t* radix, const uint64_t* strides,
                                 uint64_t rank, const uint32_t* x, int kind, uint64_t* out) {
    uint32_t k = 0;
    for (uint32_t i = 0; i < dims; ++i) {
        const uint64_t s = strides[i];
        const uint32_t xi = x[i], m = radix[i];
        const uint64_t base = rank - (uint64_t)xi * s;
        if (kind == OR_HAMMING) {
            for (uint32_t j = 0; j < m; ++j)
                if (j != xi) out[k++] = base + (uint64_t)j * s;
        } else {
            if (xi > 0) out[k++] = rank - s;
            if (xi + 1 < m) out[k++] = rank + s;
        }
    }
    return k;
}

static void digits_of(uint32_t dims, const uint64_t* strides, const uint32_t* radix,
                      uint64_t rank, uint32_t* x) {
    for (uint32_t i = 0; i < dims; ++i) x[i] = (uint32_t)((rank / strides[i]) % radix[i]);
}

static void odometer_next(uint32_t dims, const uint32_t* radix, uint32_t* x) {
    for (uint32_t i = dims; i-- > 0;) {
        if (++x[i] < radix[i]) return;
        x[i] = 0;
    }
}

/* Out-degree of every node into deg[u] (deg may alias offsets + 1). */
static void ffg_degrees(uint32_t dims, const uint32_t* radix, const uint64_t* strides, uint64_t n,
                        const double* fit, int kind, uint32_t maxnb, uint64_t* deg, int nt) {
#ifdef _OPENMP
#pragma omp parallel num_threads(nt)
#endif
    {
        int t = 0, T = 1;
#ifdef _OPENMP
        t = omp_get_thread_num();
        T = omp_get_num_threads();
#endif
        uint64_t lo, hi;
        chunk_of(n, T, t, &lo, &hi);
        uint64_t* nb = (uint64_t*)malloc(sizeof(uint64_t) * (maxnb + 1));
        uint32_t x[OR_MAX_DIMS];
        if (lo < hi) digits_of(dims, strides, radix, lo, x);
        for (uint64_t u = lo; u < hi; ++u) {
            const uint32_t k = nbr_ranks_digits(dims, radix, strides, u, x, kind, nb);
            uint64_t d = 0;
            const double fu = fit[u];
            for (uint32_t j = 0; j < k; ++j) d += fit[nb[j]] < fu;
            deg[u] = d;
            odometer_next(dims, radix, x);
        }
        free(nb);
    }
}

/* landscape.hpp:26-45.  A1: nodes are all N ranks (failed
 * ranks carry 1e10).  A2: u->v iff v in N(u) and f(v) < f(u), strict.
 * A3: row order is neighbour_ranks order.  A4: minima = ok && outdeg == 0,
 * ascending.  A9: N > node_limit -> InvalidArgument (OR_ELIMIT). */
int or_ffg_count(uint32_t dims, const uint32_t* radix, const double* fit,
                 const uint8_t* ok, int kind, uint64_t node_limit,
                 uint64_t* n_edges, uint64_t* n_minima, int nthreads) {
    if (check_space(dims, radix, kind)) return OR_EINVAL;
    uint64_t strides[OR_MAX_DIMS];
    const uint64_t n = or_space_strides(dims, radix, strides);
    if (n > node_limit || n > 0xffffffffull) return OR_ELIMIT;
    const uint32_t maxnb = or_max_neighbours(dims, radix, kind);
    const int nt = nthreads > 0 ? nthreads : 1;
    uint64_t edges = 0, minima = 0;
#ifdef _OPENMP
#pragma omp parallel num_threads(nt) reduction(+ : edges, minima)
#endif
    {
        int t = 0, T = 1;
#ifdef _OPENMP
        t = omp_get_thread_num();
        T = omp_get_num_threads();
#endif
        uint64_t lo, hi;
        chunk_of(n, T, t, &lo, &hi);
        uint64_t* nb = (uint64_t*)malloc(sizeof(uint64_t) * (maxnb + 1));
        uint32_t x[OR_MAX_DIMS];
        if (lo < hi) digits_of(dims, strides, radix, lo, x);
        for (uint64_t u = lo; u < hi; ++u) {
            const uint32_t k = nbr_ranks_digits(dims, radix, strides, u, x, kind, nb);
            uint64_t deg = 0;
            const double fu = fit[u];
            for (uint32_t j = 0; j < k; ++j) deg += fit[nb[j]] < fu;
            edges += deg;
            minima += (deg == 0 && ok[u]);
            odometer_next(dims, radix, x);
        }
        free(nb);
    }
    *n_edges = edges;
    *n_minima = minima;
    return OR_OK;
}

int or_ffg_fill(uint32_t dims, const uint32_t* radix, const double* fit,
                const uint8_t* ok, int kind, uint64_t* offsets, uint32_t* targets,
                uint8_t* is_sink, uint32_t* minima, int nthreads) {
    if (check_space(dims, radix, kind)) return OR_EINVAL;
    uint64_t strides[OR_MAX_DIMS];
    const uint64_t n = or_space_strides(dims, radix, strides);
    const uint32_t maxnb = or_max_neighbours(dims, radix, kind);
    const int nt = nthreads > 0 ? nthreads : 1;
    /* pass 1: out-degrees into offsets[u+1] */
    offsets[0] = 0;
    ffg_degrees(dims, radix, strides, n, fit, kind, maxnb, offsets + 1, nt);
    /* exclusive scan -> CSR offsets; minima compaction in ascending rank
     * (two-level: per-chunk totals, then each chunk rescans from its base) */
    uint64_t part_e[257], part_m[257];
    const int T = nt < 256 ? nt : 256;
#ifdef _OPENMP
#pragma omp parallel for num_threads(T) schedule(static, 1)
#endif
    for (int t = 0; t < T; ++t) {
        uint64_t lo, hi, e = 0, m = 0;
        chunk_of(n, T, t, &lo, &hi);
        for (uint64_t u = lo; u < hi; ++u) {
            e += offsets[u + 1];
            m += offsets[u + 1] == 0 && ok[u];
        }
        part_e[t + 1] = e;
        part_m[t + 1] = m;
    }
    part_e[0] = part_m[0] = 0;
    for (int t = 0; t < T; ++t) {
        part_e[t + 1] += part_e[t];
        part_m[t + 1] += part_m[t];
    }
#ifdef _OPENMP
#pragma omp parallel for num_threads(T) schedule(static, 1)
#endif
    for (int t = 0; t < T; ++t) {
        uint64_t lo, hi, e = part_e[t], m = part_m[t];
        chunk_of(n, T, t, &lo, &hi);
        for (uint64_t u = lo; u < hi; ++u) {
            const uint64_t deg = offsets[u + 1];
            offsets[u + 1] = e + deg;
            e += deg;
            is_sink[u] = deg == 0;
            if (deg == 0 && ok[u]) minima[m++] = (uint32_t)u;
        }
    }
    /* pass 2: targets in neighbour_ranks order */
#ifdef _OPENMP
#pragma omp parallel num_threads(nt)
#endif
    {
        int t = 0, Tn = 1;
#ifdef _OPENMP
        t = omp_get_thread_num();
        Tn = omp_get_num_threads();
#endif
        uint64_t lo, hi;
        chunk_of(n, Tn, t, &lo, &hi);
        uint64_t* nb = (uint64_t*)malloc(sizeof(uint64_t) * (maxnb + 1));
        uint32_t x[OR_MAX_DIMS];
        if (lo < hi) digits_of(dims, strides, radix, lo, x);
        for (uint64_t u = lo; u < hi; ++u) {
            const uint32_t k = nbr_ranks_digits(dims, radix, strides, u, x, kind, nb);
            uint64_t o = offsets[u];
            const double fu = fit[u];
            for (uint32_t j = 0; j < k; ++j)
                if (fit[nb[j]] < fu) targets[o++] = (uint32_t)nb[j];
            odometer_next(dims, radix, x);
        }
        free(nb);
    }
    return OR_OK;
}

/* ------------------------------------------------------------- PageRank -- */

/* landscape.hpp:47-52, pinned as SURVEY.md A7:
 *   r_0 = 1/N;  D = sum_{outdeg(s)=0} r[s];
 *   r'[v] = (1-d)/N + d * (sum_{u->v} r[u]/outdeg(u) + D/N)
 *   residual = sum_v |r'[v] - r[v]|; return r' at the first iteration with
 *   residual < tol; NonConvergence(max_iter, residual) otherwise.
 * The in-edge sum runs over sources in ascending rank, which is the order a
 * push loop "for u ascending: distribute r[u]/deg(u) over targets" produces
 * (SURVEY.md s3 stack A, HOT LOOP 2).  The pull form with a stable transpose
 * keeps that order and parallelises over rows. */
int or_pagerank(uint64_t n, const uint64_t* offsets, const uint32_t* targets,
                double damping, double tol, int64_t max_iter, double* r_out,
                int64_t* iterations, double* residual, int nthreads,
                int64_t fixed_iters) {
    if (n == 0) return OR_EINVAL;
    if (!(damping >= 0.0 && damping <= 1.0) || !(tol > 0.0) || max_iter < 1)
        return OR_EINVAL;
    const int nt = nthreads > 0 ? nthreads : 1;
    const uint64_t e = offsets[n];
    /* stable transpose: in-CSR with sources ascending inside each row */
    uint64_t* in_off = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
    uint32_t* src = (uint32_t*)malloc(sizeof(uint32_t) * (e ? e : 1));
    double* c = (double*)malloc(sizeof(double) * n);
    double* r = (double*)malloc(sizeof(double) * n);
    double* rn = (double*)malloc(sizeof(double) * n);
    uint64_t* cursor = (uint64_t*)malloc(sizeof(uint64_t) * n);
    if (!in_off || !src || !c || !r || !rn || !cursor) {
        free(in_off); free(src); free(c); free(r); free(rn); free(cursor);
        return OR_EINVAL;
    }
    /* parallel stable transpose: count in-degrees (atomic), scan, scatter
     * with an atomic cursor per row, then sort each (short) row so the
     * sources come out ascending -- the result equals the serial transpose */
#ifdef _OPENMP
#pragma omp parallel for num_threads(nt) schedule(static)
#endif
    for (int64_t i = 0; i < (int64_t)e; ++i)
        __atomic_fetch_add(&in_off[targets[i] + 1], 1, __ATOMIC_RELAXED);
    {
        uint64_t part[257];
        const int T = nt < 256 ? nt : 256;
#ifdef _OPENMP
#pragma omp parallel for num_threads(T) schedule(static, 1)
#endif
        for (int t = 0; t < T; ++t) {
            uint64_t lo, hi, acc = 0;
            chunk_of(n, T, t, &lo, &hi);
            for (uint64_t v = lo; v < hi; ++v) acc += in_off[v + 1];
            part[t + 1] = acc;
        }
        part[0] = 0;
        for (int t = 0; t < T; ++t) part[t + 1] += part[t];
#ifdef _OPENMP
#pragma omp parallel for num_threads(T) schedule(static, 1)
#endif
        for (int t = 0; t < T; ++t) {
            uint64_t lo, hi, acc = part[t];
            chunk_of(n, T, t, &lo, &hi);
            for (uint64_t v = lo; v < hi; ++v) {
                acc += in_off[v + 1];
                in_off[v + 1] = acc;
            }
        }
    }
#ifdef _OPENMP
#pragma omp parallel for num_threads(nt) schedule(static)
#endif
    for (int64_t vi = 0; vi < (int64_t)n; ++vi) cursor[vi] = in_off[vi];
#ifdef _OPENMP
#pragma omp parallel for num_threads(nt) schedule(static)
#endif
    for (int64_t ui = 0; ui < (int64_t)n; ++ui)
        for (uint64_t i = offsets[ui]; i < offsets[ui + 1]; ++i)
            src[__atomic_fetch_add(&cursor[targets[i]], 1, __ATOMIC_RELAXED)] = (uint32_t)ui;
    free(cursor);
#ifdef _OPENMP
#pragma omp parallel for num_threads(nt) schedule(static)
#endif
    for (int64_t vi = 0; vi < (int64_t)n; ++vi) {
        uint32_t* row = src + in_off[vi];
        const uint64_t len = in_off[vi + 1] - in_off[vi];
        for (uint64_t a = 1; a < len; ++a) {
            const uint32_t key = row[a];
            uint64_t b = a;
            while (b > 0 && row[b - 1] > key) {
                row[b] = row[b - 1];
                --b;
            }
            row[b] = key;
        }
    }

    const double nd = (double)n;
    const double teleport = (1.0 - damping) / nd;
    for (uint64_t v = 0; v < n; ++v) r[v] = 1.0 / nd;
    int status = OR_ENOCONV;
    double res = 0.0;
    int64_t it = 0;
    const int64_t limit = fixed_iters > 0 ? fixed_iters : max_iter;
    while (it < limit) {
        double dangling = 0.0;
#ifdef _OPENMP
#pragma omp parallel for num_threads(nt) schedule(static) reduction(+ : dangling)
#endif
        for (int64_t ui = 0; ui < (int64_t)n; ++ui) {
            const uint64_t u = (uint64_t)ui;
            const uint64_t deg = offsets[u + 1] - offsets[u];
            if (deg == 0) {
                dangling += r[u];
                c[u] = 0.0;
            } else {
                c[u] = r[u] / (double)deg;
            }
        }
        const double dn = dangling / nd;
        res = 0.0;
#ifdef _OPENMP
#pragma omp parallel for num_threads(nt) schedule(static) reduction(+ : res)
#endif
        for (int64_t vi = 0; vi < (int64_t)n; ++vi) {
            const uint64_t v = (uint64_t)vi;
            double acc = 0.0;
            for (uint64_t i = in_off[v]; i < in_off[v + 1]; ++i) acc += c[src[i]];
            const double x = teleport + damping * (acc + dn);
            rn[v] = x;
            res += fabs(x - r[v]);
        }
        double* t = r; r = rn; rn = t;
        ++it;
        if (fixed_iters <= 0 && res < tol) {
            status = OR_OK;
            break;
        }
    }
    if (fixed_iters > 0) status = OR_OK;
    memcpy(r_out, r, sizeof(double) * n);
    *iterations = it;
    *residual = res;
    free(in_off); free(src); free(c); free(r); free(rn);
    return status;
}

/* landscape.hpp:54-58; pinned as SURVEY.md A8:
 * p == 0 -> include f <= f_opt; p > 0 -> include f < (1.0 + p) * f_opt.
 * Sums run over minima in ascending rank.  Zero denominator -> Error. */
int or_proportion_of_centrality(uint64_t n_minima, const uint32_t* minima,
                                const double* fit, const double* pr, double f_opt,
                                double p, double* out) {
    const double thr = (1.0 + p) * f_opt;
    double num = 0.0, den = 0.0;
    for (uint64_t i = 0; i < n_minima; ++i) {
        const uint32_t m = minima[i];
        const double f = fit[m];
        den += pr[m];
        if (p == 0.0 ? (f <= f_opt) : (f < thr)) num += pr[m];
    }
    if (!(den > 0.0)) return OR_EDEGEN;
    *out = num / den;
    return OR_OK;
}

/* src/cache.cpp:55-72 */
int or_optimum(uint64_t n, const double* fit, const uint8_t* ok, double* f_opt,
               uint64_t* rank) {
    int has = 0;
    double best = OR_FAIL_FITNESS;
    uint64_t br = 0;
    for (uint64_t r = 0; r < n; ++r) {
        if (!ok[r]) continue;
        if (!has || fit[r] < best) {
            best = fit[r];
            br = r;
            has = 1;
        }
    }
    if (!has) return OR_ENOFEAS;
    *f_opt = best;
    *rank = br;
    return OR_OK;
}

/* landscape.hpp:12-24, SPEC.md:379-387 (A5): local minimum iff ok and every
 * neighbour has strictly greater fitness. */
int or_census(uint32_t dims, const uint32_t* radix, const double* fit,
              const uint8_t* ok, int kind, uint64_t* fail_points,
              uint64_t* local_minima, uint64_t* interior, uint64_t* minima_ranks) {
    if (check_space(dims, radix, kind)) return OR_EINVAL;
    uint64_t strides[OR_MAX_DIMS];
    const uint64_t n = or_space_strides(dims, radix, strides);
    const uint32_t maxnb = or_max_neighbours(dims, radix, kind);
    uint64_t* nb = (uint64_t*)malloc(sizeof(uint64_t) * (maxnb + 1));
    uint64_t fails = 0, mins = 0, oks = 0;
    for (uint64_t u = 0; u < n; ++u) {
        if (!ok[u]) {
            ++fails;
            continue;
        }
        ++oks;
        const uint32_t k = nbr_ranks(dims, radix, strides, u, kind, nb);
        int strict = 1;
        for (uint32_t j = 0; j < k; ++j)
            if (!(fit[nb[j]] > fit[u])) { strict = 0; break; }
        if (strict) {
            if (minima_ranks) minima_ranks[mins] = u;
            ++mins;
        }
    }
    free(nb);
    *fail_points = fails;
    *local_minima = mins;
    *interior = oks - mins;
    return OR_OK;
}

/* ----------------------------------------------------------- generators -- */

/* src/generators.cpp:11-16 */
static uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* src/generators.cpp:20-23 */
double or_hash_uniform(uint64_t seed, uint64_t rank, uint64_t slot) {
    const uint64_t h = mix64(seed ^ mix64(rank * 0x2545f4914f6cdd1dULL + slot));
    return (double)(h >> 11) * 0x1.0p-53;
}

/* G_iid: ok iff hash_uniform(seed,r,0) >= q; f = 1 + u1 */
void or_gen_iid(uint64_t n, double q, uint64_t seed, double* fit, uint8_t* ok,
                int nthreads) {
    (void)nthreads;
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads > 0 ? nthreads : 1) schedule(static)
#endif
    for (int64_t ri = 0; ri < (int64_t)n; ++ri) {
        const uint64_t r = (uint64_t)ri;
        const int good = !(or_hash_uniform(seed, r, 0) < q);
        ok[r] = (uint8_t)good;
        fit[r] = good ? 1.0 + or_hash_uniform(seed, r, 1) : OR_FAIL_FITNESS;
    }
}

/* G_heavy: Pareto(1) runtimes f = 1 / (1 - u1) */
void or_gen_heavy(uint64_t n, double q, uint64_t seed, double* fit, uint8_t* ok,
                  int nthreads) {
    (void)nthreads;
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads > 0 ? nthreads : 1) schedule(static)
#endif
    for (int64_t ri = 0; ri < (int64_t)n; ++ri) {
        const uint64_t r = (uint64_t)ri;
        const int good = !(or_hash_uniform(seed, r, 0) < q);
        ok[r] = (uint8_t)good;
        fit[r] = good ? 1.0 / (1.0 - or_hash_uniform(seed, r, 1)) : OR_FAIL_FITNESS;
    }
}

/* mt19937_64 (the engine behind include/tunekit/rng.hpp:14-79) */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t y = (g->mt[i] & 0xffffffff80000000ULL) |
                               (g->mt[(i + 1) % 312] & 0x7fffffffULL);
            uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1) v ^= 0xb5026f5aa96619e9ULL;
            g->mt[i] = v;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71d67fffeda60000ULL;
    x ^= (x << 37) & 0xfff7eee000000000ULL;
    x ^= x >> 43;
    return x;
}

/* rng.hpp:21-25 */
static double rng_u01(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }
static double rng_uniform(mt64* g, double lo, double hi) { return lo + (hi - lo) * rng_u01(g); }

/* src/generators.cpp:89-145, mean-only: identical draws, identical
 * expression order, 32 jittered samples accumulated left to right from 0.0
 * (std::accumulate, cache.cpp:33-34) and divided by 32. */
int or_gen_synthetic(uint32_t dims, const uint32_t* radix, double fail_fraction,
                     double ridge_strength, double noise, double jitter,
                     uint64_t seed, double* fit, uint8_t* ok, int nthreads) {
    if (!(fail_fraction >= 0.0 && fail_fraction < 1.0)) return OR_EINVAL;
    if (dims == 0 || dims > OR_MAX_DIMS) return OR_EINVAL;
    uint64_t strides[OR_MAX_DIMS];
    const uint64_t n = or_space_strides(dims, radix, strides);
    mt64 g;
    mt64_seed(&g, mix64(seed)); /* rng.hpp:16,70-76: engine seeded with mix(seed) */
    const double scale = rng_uniform(&g, 0.5, 5.0);
    double weight[OR_MAX_DIMS], center[OR_MAX_DIMS], ra[OR_MAX_DIMS], rp[OR_MAX_DIMS];
    for (uint32_t d = 0; d < dims; ++d) {
        weight[d] = rng_uniform(&g, 0.5, 2.0);
        center[d] = rng_u01(&g);
    }
    for (uint32_t d = 0; d < dims; ++d) {
        ra[d] = rng_uniform(&g, 1.0, 3.0);
        rp[d] = rng_uniform(&g, 0.0, 3.141592653589793);
    }
    (void)nthreads;
#ifdef _OPENMP
#pragma omp parallel for num_threads(nthreads > 0 ? nthreads : 1) schedule(static)
#endif
    for (int64_t ri = 0; ri < (int64_t)n; ++ri) {
        const uint64_t rank = (uint64_t)ri;
        if (or_hash_uniform(seed, rank, 0) < fail_fraction) {
            ok[rank] = 0;
            fit[rank] = OR_FAIL_FITNESS;
            continue;
        }
        double u[OR_MAX_DIMS];
        uint64_t rest = rank;
        for (uint32_t d = 0; d < dims; ++d) {
            const int32_t x = (int32_t)(rest / strides[d]);
            rest %= strides[d];
            u[d] = (x + 0.5) / (int32_t)radix[d];
        }
        double f = 1.0;
        for (uint32_t d = 0; d < dims; ++d)
            f += weight[d] * (u[d] - center[d]) * (u[d] - center[d]);
        for (uint32_t d = 0; d + 1 < dims; ++d) {
            const double s = sin(3.141592653589793 *
                                 (ra[d] * u[d] - ra[d + 1] * u[d + 1] + rp[d]));
            f += ridge_strength * s * s;
        }
        f += noise * or_hash_uniform(seed, rank, 1);
        f *= scale;
        double acc = 0.0;
        for (int s = 0; s < 32; ++s)
            acc += f * (1.0 + jitter * (or_hash_uniform(seed, rank, 2 + (uint64_t)s) - 0.5));
        ok[rank] = 1;
        fit[rank] = acc / 32.0;
    }
    return OR_OK;
}

/* ------------------------------------------------ randomized descents --
 * hillclimb.cpp:48-87 climb_random_first.  Slot universe (build_slots,
 * hillclimb.cpp:26-38): per dimension ascending, Adjacent {-1, +1} when
 * m > 1, Hamming the m-1 alternatives a (index a < x ? a : a + 1,
 * resolve_slot :41-46).  The scan walks a random permutation of the slots
 * cyclically; the first strictly better neighbour (fp64 <) is taken, and with
 * restart_scan a fresh permutation starts after every move.  The descent
 * stops after a full cycle without an improvement.
 *
 * Draws (shared with the device validator, tk_descent.cu): walker w owns the
 * splitmix64 stream s_0 = sm(seed ^ sm(w)), next() = sm-step; uniform(k) =
 * mulhi64(next(), k).  The start rank is the first draw; a permutation is
 * Fisher-Yates from the identity, i = S-1 .. 1, swap(p[i], p[uniform(i+1)]). */
static inline uint64_t or_sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t or_sm_next(uint64_t* s) {
    *s += 0x9E3779B97F4A7C15ULL;
    return or_sm_mix(*s);
}
static inline uint64_t or_uniform(uint64_t* s, uint64_t k) {
    return (uint64_t)(((unsigned __int128)or_sm_next(s) * k) >> 64);
}

int or_descents(uint32_t dims, const uint32_t* radix, const double* fit, int kind,
                uint64_t walkers, uint64_t seed, int restart_scan, uint32_t* counts,
                uint64_t* evaluations, int nthreads) {
    uint64_t strides[64];
    if (dims > 64) return OR_EINVAL;
    const uint64_t n = or_space_strides(dims, radix, strides);
    uint8_t sdim[256];
    int16_t salt[256];
    int S = 0;
    for (uint32_t i = 0; i < dims; ++i) {
        const int m = (int)radix[i];
        if (kind == OR_HAMMING) {
            for (int a = 0; a + 1 < m; ++a) {
                if (S == 256) return OR_EINVAL;
                sdim[S] = (uint8_t)i, salt[S++] = (int16_t)a;
            }
        } else if (m > 1) {
            if (S + 2 > 256) return OR_EINVAL;
            sdim[S] = (uint8_t)i, salt[S++] = -1;
            sdim[S] = (uint8_t)i, salt[S++] = +1;
        }
    }
    memset(counts, 0, n * sizeof(uint32_t));
    uint64_t evals = 0;
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : evals)
    for (int64_t w = 0; w < (int64_t)walkers; ++w) {
        uint64_t st = or_sm_mix(seed ^ or_sm_mix((uint64_t)w));
        uint64_t rank = or_uniform(&st, n);
        double f = fit[rank];
        if (S) {
            int x[64];
            uint64_t rem = rank;
            for (uint32_t i = 0; i < dims; ++i) x[i] = (int)(rem / strides[i]), rem %= strides[i];
            uint8_t order[256];
            for (int i = 0; i < S; ++i) order[i] = (uint8_t)i;
            for (int i = S - 1; i > 0; --i) {
                const int j = (int)or_uniform(&st, (uint64_t)i + 1);
                const uint8_t t = order[i]; order[i] = order[j]; order[j] = t;
            }
            int pos = 0, since = 0;
            while (since < S) {
                const int sl = order[pos];
                pos = pos + 1 == S ? 0 : pos + 1;
                const int d = sdim[sl], m = (int)radix[d], cur = x[d];
                const int j = kind == OR_HAMMING ? (salt[sl] < cur ? salt[sl] : salt[sl] + 1)
                                                 : cur + salt[sl];
                if (j < 0 || j >= m) {
                    ++since;
                    continue;
                }
                const uint64_t nb = rank + (uint64_t)((int64_t)(j - cur) * (int64_t)strides[d]);
                const double fn = fit[nb];
                ++evals;
                if (fn < f) {
                    x[d] = j, rank = nb, f = fn, since = 0;
                    if (restart_scan) {
                        for (int i = 0; i < S; ++i) order[i] = (uint8_t)i;
                        for (int i = S - 1; i > 0; --i) {
                            const int r = (int)or_uniform(&st, (uint64_t)i + 1);
                            const uint8_t t = order[i]; order[i] = order[r]; order[r] = t;
                        }
                        pos = 0;
                    }
                } else {
                    ++since;
                }
            }
        }
#pragma omp atomic
        counts[rank] += 1;
    }
    if (evaluations) *evaluations = evals;
    return OR_OK;
}
