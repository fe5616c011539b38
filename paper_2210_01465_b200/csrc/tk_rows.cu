// tk_rows.cu -- row-tiled PageRank for Adjacent spaces whose trailing
// dimensions span exactly 16 ranks (landscape.hpp:47-52).
//
// Why a second PageRank kernel.  pagerank_staged_kernel (tk_staged.cu) is
// bound by the shared-memory crossbar (128 B/clk/SM): per rank it fills
// ~112 B by TMA (a near window + 12 far ranges) and reads 25 fp64 values
// (~200 B) with LDS -- and warp shuffles share the same crossbar
// (scripts/mb_shfl.cu: LDS+SHFL time = LDS time + SHFL time).  This kernel
// moves fewer bytes through that port per rank:
//
//  * a row = 16 consecutive ranks = the trailing dimensions whose radices
//    multiply to 16 (C5: dims 9-11, radix 4,2,2).  One consumer lane owns a
//    row: its 16 own contributions stay in registers and serve every
//    neighbour inside the row (6 of the 24 directions at C5), and every other
//    neighbour of element j of row r is element j of row r +- s_i/16.  So a
//    lane reads 1 own row + 1 row per out-of-row direction (19 instead of 25
//    values per rank), 128-byte rows swizzled by TMA (SWIZZLE_128B) so that
//    eight lanes' 16-byte loads cover all 32 banks;
//  * a tile = 32 rows (512 ranks) = one consumer warp.  Each CTA walks whole
//    "columns" (the sub-grid of the row dims and the next "window" dims,
//    C5: dims 5-11, 384 rows = 12 tiles) in rank order and keeps a ring of
//    the last/next tiles' rows in shared memory, so the window dims'
//    neighbours (C5: dims 5-8, strides <= 64 rows) come from rows staged once
//    as the column streams past: 8 B of TMA fill per rank instead of 16 per
//    direction;
//  * the remaining "far" dims (C5: 0-4) are staged as one 32-row range per
//    direction, and only for directions that exist for the tile (the far
//    digits are constant over a tile): 8.6 instead of 10 ranges per tile at C5;
//  * c' leaves through a swizzled shared-memory tile and one TMA store.
//
// Columns are dealt round-robin to the CTAs, so at any time the CTAs work on
// ~148 adjacent columns and the far ranges of dims 1-4 are L2 hits, as in the
// staged kernel (dim 0 misses: evict-first).  Per-rank arithmetic is the
// staged kernel's (contribution-only iteration, div_small, closing r' pass):
// every rank is bit-identical to the oracle's, only the global sums differ in
// summation order.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tk_kernels.cuh"

namespace cg = cooperative_groups;

namespace tk {
namespace {

constexpr int kRowLen = 16;                      // ranks per row (one lane)
constexpr int kTileRows = 32;                    // rows per tile (one consumer warp)
#ifndef TK_ROW_WARPS
#define TK_ROW_WARPS 8
#endif
constexpr int kRW = TK_ROW_WARPS;                // consumer warps = tiles in flight
constexpr int kRingTiles = 16;                   // c ring: 16 tiles of 32 rows (64 KB)
constexpr int kRingRows = kRingTiles * kTileRows;
constexpr int kPwTiles = 8;                      // packed-word ring (2 KB per tile)
#ifndef TK_ROW_FAR_SLOTS
#define TK_ROW_FAR_SLOTS 3
#endif
constexpr int kFarSlots = TK_ROW_FAR_SLOTS;      // far ranges in flight per consumer warp
// consumer warps 0..kRW-1 (warp w: tiles i = w mod kRW, lane t = row t of the
// tile, all 16 ranks of the row) and kRW/2 producer warps whose lanes 0 and 16
// serve consumer warps 2p and 2p+1
constexpr int kProdWarps = kRW / 2;
constexpr int kRowThreads = (kRW + kProdWarps) * 32;
static_assert(kRingTiles % kRW == 0 && kPwTiles % kRW == 0, "ring slots per producer");
constexpr int kTileBytes = kTileRows * kRowLen * 8;  // 4 KB
constexpr int kPwTileBytes = kTileRows * kRowLen * 4;

// dynamic shared memory map (1024-byte aligned regions: SWIZZLE_128B)
constexpr int kOffRing = 0;
constexpr int kOffFar = kOffRing + kRingTiles * kTileBytes;
constexpr int kOffOut = kOffFar + kRW * kFarSlots * kTileBytes;
constexpr int kOffPw = kOffOut + kRW * kTileBytes;
constexpr int kOffDesc = kOffPw + kPwTiles * kPwTileBytes;
constexpr int kOffBar = kOffDesc + kPwTiles * 16;
constexpr int kNumBars = 2 * kRingTiles + 2 * kPwTiles + 2 * kRW * kFarSlots;
constexpr int kRowSmem = kOffBar + kNumBars * 8 + 1024;  // + alignment slack
static_assert(kRowSmem <= 232448 - 512, "shared memory");

__device__ __forceinline__ uint32_t saddr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b, uint32_t count = 1) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(saddr(b)), "r"(parity)
            : "memory");
    }
}
// producer-side wait: the thread sleeps in try_wait (suspend hint) instead of
// spinning, so a waiting producer does not take issue slots from the consumer
// warp on its SM sub-partition
__device__ __forceinline__ void bar_wait_sleep(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t ns = 64;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(saddr(b)), "r"(parity), "r"(0x100000u)
            : "memory");
        if (!done) __nanosleep(ns);
    }
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// 2-D tensor tile (32 rows x one 128- or 64-byte row) -> shared memory
__device__ __forceinline__ void tma_load_rows(void* dst, const CUtensorMap* map, int row,
                                              uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(saddr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(row), "r"(saddr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store_rows(const CUtensorMap* map, int row, const void* src,
                                               uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], "
        "%4;" ::"l"(reinterpret_cast<uint64_t>(map)),
        "r"(0), "r"(row), "r"(saddr(src)), "l"(pol)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_half(const CUtensorMap* map, int col, int row,
                                               const void* src, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], "
        "%4;" ::"l"(reinterpret_cast<uint64_t>(map)),
        "r"(col), "r"(row), "r"(saddr(src)), "l"(pol)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void lds2(uint32_t a, double& x, double& y) {
    // volatile: never hoisted above the mbarrier wait that guards the data
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a) : "memory");
}
__device__ __forceinline__ void sts2(uint32_t a, double x, double y) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void lds4u(uint32_t a, uint32_t& x, uint32_t& y, uint32_t& z,
                                      uint32_t& w) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                 : "r"(a)
                 : "memory");
}

// Reads the 16 values of a swizzled 128-byte row at shared address `row_addr`
// whose SWIZZLE_128B phase is `key` (= shared row index & 7).
__device__ __forceinline__ void ld_row(uint32_t row_addr, uint32_t key, double (&v)[16]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) lds2(row_addr + ((q ^ key) << 4), v[2 * q], v[2 * q + 1]);
}

__device__ __forceinline__ double div_small_r(double x, double d, double y) {
    const double q0 = __dmul_rn(x, y);
    const double r = __fma_rn(-q0, d, x);
    return __fma_rn(r, y, q0);
}

// compile-time in-row structure: radices of the row dims, most significant first
template <int M0, int M1, int M2, int M3>
struct RowShape {
    static constexpr int nd = (M0 > 1) + (M1 > 1) + (M2 > 1) + (M3 > 1);
    __host__ __device__ static constexpr int radix(int k) {
        return k == 0 ? M0 : k == 1 ? M1 : k == 2 ? M2 : M3;
    }
    __host__ __device__ static constexpr int stride(int k) {  // in-row stride of row dim k
        int s = 1;
        for (int i = nd - 1; i > k; --i) s *= radix(i);
        return s;
    }
    __host__ __device__ static constexpr int digit(int j, int k) { return (j / stride(k)) % radix(k); }
};

struct PrScalars {
    double teleport, damping;
};
struct SweepState {
    uint32_t ring_base;  // global ring index of the sweep's entry 0
    uint32_t tile_base;  // block tiles of earlier sweeps (packed-word ring)
    uint32_t far_ctr;    // far-slot counter of a consumer warp and its producer lane
};

struct RowCtx {
    uint64_t* c_full;
    uint64_t* c_empty;
    uint64_t* pw_full;
    uint64_t* pw_empty;
    uint64_t* far_full;   // [kRW][kFarSlots]
    uint64_t* far_empty;
    uint8_t* ring;
    uint8_t* far;
    uint8_t* out;
    uint8_t* pwr;
    uint4* desc;          // [kPwTiles] per tile: first row, far lo / hi directions
};

// first row of sweep-local tile i of this block
__device__ __forceinline__ uint32_t tile_row(const RowPlan& p, uint32_t i) {
    const uint32_t k = fdiv(i, p.tpc_magic);
    const uint32_t w = i - k * p.tiles_per_col;
    return (blockIdx.x + k * gridDim.x) * p.col_rows + w * kTileRows;
}
__device__ __forceinline__ uint32_t block_tiles(const RowPlan& p) {
    const uint32_t cols = p.ncols > blockIdx.x ? (p.ncols - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    return cols * p.tiles_per_col;
}
// far directions of the tile at row r: bit d of lo = neighbour v - s_d exists
// for some row of the tile, of hi = v + s_d exists
__device__ __forceinline__ void far_dirs(const RowPlan& p, uint32_t r, uint32_t& lo, uint32_t& hi) {
    lo = hi = 0;
    const uint32_t r1 = r + kTileRows - 1;
    for (int d = 0; d < p.nfar; ++d) {
        const uint32_t m = p.far_radix[d];
        const uint32_t qa = fdiv(r, p.far_magic[d]), qb = fdiv(r1, p.far_magic[d]);
        const uint32_t a = qa - fdiv(qa, p.far_rmagic[d]) * m;
        const uint32_t b = qb - fdiv(qb, p.far_rmagic[d]) * m;
        if (p.far_span[d] || !(a == 0 && b == 0)) lo |= 1u << d;
        if (p.far_span[d] || !(a == m - 1 && b == m - 1)) hi |= 1u << d;
    }
}
// far_dirs of a producer's tiles, recomputed only when the tile moves to
// another column (when columns are whole tiles, every tile of a column has
// the same far digits)
struct FarCache {
    uint32_t col = ~0u, lo = 0, hi = 0;
    __device__ __forceinline__ void get(const RowPlan& p, uint32_t i, uint32_t r, uint32_t& flo,
                                        uint32_t& fhi) {
        const uint32_t c = p.far_per_col ? fdiv(i, p.tpc_magic) : i;
        if (c != col) {
            far_dirs(p, r, lo, hi);
            col = c;
        }
        flo = lo;
        fhi = hi;
    }
};

// acc += v if (m & bit), as acc = fma(v, s, acc) with s = 1.0 or 0.0: the
// product is exact and fma(v, 1, acc) == RN(acc + v) bit for bit, so this is
// the in-edge add; v is always finite (c values, TMA zero fill, the
// zero-initialised ring), so 0 * v adds +0.  Two integer ops + one DFMA per
// term instead of the DADD + two FSEL the compiler makes of a guarded add.
__device__ __forceinline__ void cadd(double& acc, double v, uint32_t m, uint32_t bit) {
    const uint32_t hi = (m & bit) ? 0x3FF00000u : 0u;
    acc = __fma_rn(v, __hiloint2double(static_cast<int>(hi), 0), acc);
}
// the 16 values of a 128-byte row: chunk q at base + off[q], one predicate
// for all eight loads (lanes with p == 0 issue no wavefront)
__device__ __forceinline__ void ld_row16(uint32_t base, const uint32_t (&off)[8], double (&v)[16],
                                         uint32_t p) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.ne.b32 q, %24, 0;\n\t"
        "@q ld.shared.v2.f64 {%0, %1}, [%16];\n\t"
        "@q ld.shared.v2.f64 {%2, %3}, [%17];\n\t"
        "@q ld.shared.v2.f64 {%4, %5}, [%18];\n\t"
        "@q ld.shared.v2.f64 {%6, %7}, [%19];\n\t"
        "@q ld.shared.v2.f64 {%8, %9}, [%20];\n\t"
        "@q ld.shared.v2.f64 {%10, %11}, [%21];\n\t"
        "@q ld.shared.v2.f64 {%12, %13}, [%22];\n\t"
        "@q ld.shared.v2.f64 {%14, %15}, [%23];\n\t}"
        : "+d"(v[0]), "+d"(v[1]), "+d"(v[2]), "+d"(v[3]), "+d"(v[4]), "+d"(v[5]), "+d"(v[6]),
          "+d"(v[7]), "+d"(v[8]), "+d"(v[9]), "+d"(v[10]), "+d"(v[11]), "+d"(v[12]), "+d"(v[13]),
          "+d"(v[14]), "+d"(v[15])
        : "r"(base + off[0]), "r"(base + off[1]), "r"(base + off[2]), "r"(base + off[3]),
          "r"(base + off[4]), "r"(base + off[5]), "r"(base + off[6]), "r"(base + off[7]), "r"(p)
        : "memory");
}

// One consumer warp handles tile i: lane t owns row r = r0 + t (16 ranks).
// The producer lane of this warp left the tile's first row and far
// directions in the packed-word slot's descriptor.
template <class RS, bool FINAL>
__device__ __forceinline__ void row_tile(const RowPlan& p, const RowMaps& maps, const RowCtx& cx,
                                         const PrScalars& a, uint32_t i, uint32_t e_i,
                                         uint32_t pw_idx, uint32_t& far_ctr, int w, int t,
                                         const uint32_t (&lo)[8], double dn, int out_map,
                                         double& lres, double& ldang, double& lsum,
                                         const double* s_rcp, uint64_t pol_out) {
    const int D = p.dims;
    const int A = p.ahead;
    uint32_t m[16];
    uint32_t r0, flo, fhi, any;
    {
        const uint32_t ps = pw_idx % kPwTiles;
        bar_wait(cx.pw_full + ps, (pw_idx / kPwTiles) & 1u);
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r0), "=r"(flo), "=r"(fhi), "=r"(any)
                     : "r"(saddr(cx.desc + ps))
                     : "memory");
        const uint32_t base = saddr(cx.pwr + ps * kPwTileBytes) + t * 64;
        const uint32_t key = (t >> 1) & 3;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            lds4u(base + ((q ^ key) << 4), m[4 * q], m[4 * q + 1], m[4 * q + 2], m[4 * q + 3]);
        __syncwarp();
        if (t == 0) bar_arrive(cx.pw_empty + ps);
    }
    any = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) any |= m[j];
    // ring tiles i-A .. i+A; the sweep's first A tiles have no tiles before
    // them (their lower window neighbours do not exist)
    const int k0 = static_cast<int>(i) >= A ? -A : -static_cast<int>(i);
    for (int k = k0; k <= A; ++k) {
        const uint32_t e = e_i + k;
        bar_wait(cx.c_full + (e % kRingTiles), (e / kRingTiles) & 1u);
    }
    const uint32_t ring = saddr(cx.ring);
    const uint32_t rrow0 = (e_i % kRingTiles) * kTileRows;  // ring row of lane 0's row
    const uint32_t far_w = saddr(cx.far + w * kFarSlots * kTileBytes);
    uint64_t* ffull = cx.far_full + w * kFarSlots;
    uint64_t* fempty = cx.far_empty + w * kFarSlots;
    uint32_t fs = far_ctr % kFarSlots, fph = (far_ctr / kFarSlots) & 1u;

    double acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0;
    double v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = 0.0;
    auto addv = [&](uint32_t bit) {
#pragma unroll
        for (int j = 0; j < 16; ++j) cadd(acc[j], v[j], m[j], bit);
    };
    // a far range: wait for its slot, read this lane's row, release it
    auto far_take = [&](uint32_t bit) {
        bar_wait(ffull + fs, fph);
        ld_row16(far_w + fs * kTileBytes, lo, v, any & bit);
        __syncwarp();
        if (t == 0) bar_arrive(fempty + fs);
        if (++fs == kFarSlots) {
            fs = 0;
            fph ^= 1u;
        }
    };
    // a window direction: ring row of lane t = rrow0 + t + drow
    auto win_take = [&](int drow, uint32_t bit) {
        const uint32_t pred = any & bit;
        const uint32_t rr = (rrow0 + t + kRingRows + drow) % kRingRows;
        if ((drow & 7) == 0) {  // same swizzle phase as the lane's own row
            ld_row16(ring + rr * 128 - t * 128, lo, v, pred);
        } else {
            const uint32_t key = rr & 7;
            uint32_t o2[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) o2[q] = (q ^ key) << 4;
            ld_row16(ring + rr * 128, o2, v, pred);
        }
    };
    // ---- lower neighbours (ascending rank): far dims, then window dims
#pragma unroll 1
    for (uint32_t rem = flo; rem; rem &= rem - 1) {
        const uint32_t bit = rem & (0u - rem);
        far_take(bit);
        addv(bit);
    }
#pragma unroll 1
    for (int wk = 0; wk < p.nwin; ++wk) {
        const uint32_t bit = 1u << (p.nfar + wk);
        win_take(-p.win_rows[wk], bit);
        addv(bit);
    }
    // ---- in-row neighbours from the own row: lower (ascending dim), then
    // upper (descending dim)
    double own[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) own[j] = 0.0;
    ld_row16(ring + rrow0 * 128, lo, own, 1u);
    {
        const int d0 = D - RS::nd;  // first row dim
#pragma unroll
        for (int k = 0; k < RS::nd; ++k) {
            const uint32_t bit = 1u << (d0 + k);
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (RS::digit(j, k) > 0)
                    cadd(acc[j], own[RS::digit(j, k) > 0 ? j - RS::stride(k) : j], m[j], bit);
        }
#pragma unroll
        for (int k = RS::nd - 1; k >= 0; --k) {
            const uint32_t bit = 1u << (2 * D - 1 - (d0 + k));
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (RS::digit(j, k) < RS::radix(k) - 1)
                    cadd(acc[j], own[RS::digit(j, k) < RS::radix(k) - 1 ? j + RS::stride(k) : j],
                         m[j], bit);
        }
    }
    // ---- upper neighbours (ascending rank): window dims (descending), far dims (descending)
#pragma unroll 1
    for (int wk = p.nwin - 1; wk >= 0; --wk) {
        const uint32_t bit = 1u << (2 * D - 1 - (p.nfar + wk));
        win_take(p.win_rows[wk], bit);
        addv(bit);
    }
#pragma unroll 1
    for (uint32_t rem = fhi; rem;) {
        const int d = 31 - __clz(rem);
        rem ^= 1u << d;
        const uint32_t bit = 1u << (2 * D - 1 - d);
        far_take(bit);
        addv(bit);
    }
    far_ctr += __popc(flo) + __popc(fhi);
    // release the ring tiles this tile read (their missing users before the
    // sweep's first / after its last tile were arrived for by the producer)
    __syncwarp();
    if (t == 0)
        for (int k = k0; k <= A; ++k) bar_arrive(cx.c_empty + ((e_i + k) % kRingTiles));
    // ---- epilogue: r' per rank, residual terms, c' (or r') out via one TMA store
    const uint32_t ob = saddr(cx.out + w * kTileBytes);
    if (t == 0) tma_store_wait_read();  // the previous store from this buffer has read it
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        double o[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = 2 * q + h;
            const uint32_t deg = m[j] >> kPackedSlots;
            const double x = __dadd_rn(a.teleport, __dmul_rn(a.damping, __dadd_rn(acc[j], dn)));
            if (FINAL) {
                o[h] = x;
            } else {
                double qv, dv;
                if (deg) {
                    const double dd = static_cast<double>(deg);
                    qv = div_small_r(x, dd, s_rcp[deg]);
                    dv = fabs(__fma_rn(own[j], dd, -x));
                } else {
                    qv = x;  // a sink's slot carries its rank (no pull reads it)
                    dv = fabs(__dsub_rn(x, own[j]));
                    ldang = __dadd_rn(ldang, x);
                }
                lres = __dadd_rn(lres, dv);
                lsum = __dadd_rn(lsum, x);
                o[h] = qv;
            }
        }
        sts2(ob + lo[q], o[0], o[1]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (t == 0) {
        const CUtensorMap* om = out_map == 2 ? &maps.r0 : &maps.c[out_map];
        tma_store_rows(om, static_cast<int>(r0), cx.out + w * kTileBytes, pol_out);
    }
}

// Producer lane of consumer warp w: for each of its tiles i, ring entry i + A
// (the tile A ahead enters the c window), the packed words + descriptor of
// tile i, and its far ranges.  Ring / packed-word slots are multiples of kRW
// apart, so a slot's loads always come from one producer lane, in order.
// Ring entry j (sweep-local) has 2A+1 users (tiles j-A..j+A); the users that
// do not exist (before tile 0, after tile L-1) are arrived for here.
__device__ __forceinline__ void row_produce(const RowPlan& p, const RowMaps& maps,
                                            const RowCtx& cx, uint32_t L, uint32_t LE,
                                            uint32_t ring_base, uint32_t tile_base,
                                            uint32_t& far_ctr, int w, int in_map) {
    const uint64_t pol = policy_evict_normal();
    const uint64_t pol_ef = policy_evict_first();
    const CUtensorMap* cm = &maps.c[in_map];
    const int A = p.ahead;
    uint8_t* far_w = cx.far + w * kFarSlots * kTileBytes;
    uint64_t* ffull = cx.far_full + w * kFarSlots;
    uint64_t* fempty = cx.far_empty + w * kFarSlots;
    uint32_t fc = far_ctr;
    uint32_t fs = fc % kFarSlots, fph = (fc / kFarSlots) & 1u;
    FarCache fcache;
    auto ring_entry = [&](uint32_t j) {
        const uint32_t e = ring_base + j;
        const uint32_t slot = e % kRingTiles;
        if (e >= kRingTiles) bar_wait_sleep(cx.c_empty + slot, ((e / kRingTiles) + 1) & 1u);
        // users j-A..j+A outside [0, L)
        const int lo_missing = static_cast<int>(j) < A ? A - static_cast<int>(j) : 0;
        const int hi_missing = static_cast<int>(j + A) >= static_cast<int>(L)
                                   ? static_cast<int>(j + A) - static_cast<int>(L) + 1
                                   : 0;
        const int missing = min(lo_missing + hi_missing, 2 * A + 1);
        if (missing) bar_arrive(cx.c_empty + slot, static_cast<uint32_t>(missing));
        if (j < L) {
            bar_expect(cx.c_full + slot, kTileBytes);
            tma_load_rows(cx.ring + slot * kTileBytes, cm, static_cast<int>(tile_row(p, j)),
                          cx.c_full + slot, pol);
        } else {
            bar_arrive(cx.c_full + slot);  // overhang entry: nothing to load
        }
    };
    auto issue = [&](int row, int d) {
        if (fc >= kFarSlots) bar_wait_sleep(fempty + fs, fph ^ 1u);
        bar_expect(ffull + fs, kTileBytes);
        tma_load_rows(far_w + fs * kTileBytes, cm, row, ffull + fs,
                      ((p.far_ef >> d) & 1u) ? pol_ef : pol);
        ++fc;
        if (++fs == kFarSlots) {
            fs = 0;
            fph ^= 1u;
        }
    };
    if (w < A && static_cast<uint32_t>(w) < LE) ring_entry(w);  // the sweep's first A entries
    for (uint32_t i = w; i < L; i += kRW) {
        ring_entry(i + A);
        const uint32_t r = tile_row(p, i);
        const uint32_t pi = tile_base + i;
        const uint32_t ps = pi % kPwTiles;
        uint32_t lo, hi;
        fcache.get(p, i, r, lo, hi);
        if (pi >= kPwTiles) bar_wait_sleep(cx.pw_empty + ps, ((pi / kPwTiles) + 1) & 1u);
        cx.desc[ps] = make_uint4(r, lo, hi, 0);  // released by the arrive below
        bar_expect(cx.pw_full + ps, kPwTileBytes);
        tma_load_rows(cx.pwr + ps * kPwTileBytes, &maps.pw, static_cast<int>(r), cx.pw_full + ps,
                      pol_ef);
        for (uint32_t rem = lo; rem; rem &= rem - 1) {
            const int d = __ffs(rem) - 1;
            issue(static_cast<int>(r) - static_cast<int>(p.far_rows[d]), d);
        }
        for (uint32_t rem = hi; rem;) {
            const int d = 31 - __clz(rem);
            rem ^= 1u << d;
            issue(static_cast<int>(r + p.far_rows[d]), d);
        }
    }
    far_ctr = fc;
}

template <class RS, bool FINAL>
__device__ __forceinline__ void row_sweep(const RowPlan& p, const RowMaps& maps, const RowCtx& cx,
                                          const PrScalars& sc, uint32_t L, uint32_t LE,
                                          SweepState& ss, int in_map, int out_map, double dn,
                                          double& lres_out, double& ldang_out, double& lsum_out,
                                          const double* s_rcp) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double lres = 0.0, ldang = 0.0, lsum = 0.0;
    if (warp >= kRW) {  // producer warps: lanes 0 and 16 serve consumer warps 2p, 2p+1
        if ((lane & 15) == 0)
            row_produce(p, maps, cx, L, LE, ss.ring_base, ss.tile_base, ss.far_ctr,
                        2 * (warp - kRW) + (lane >> 4), in_map);
    } else {
        const uint64_t pol_out = policy_evict_first();
        uint32_t lo[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) lo[q] = lane * 128 + ((q ^ (lane & 7)) << 4);
        for (uint32_t i = warp; i < L; i += kRW)
            row_tile<RS, FINAL>(p, maps, cx, sc, i, ss.ring_base + i, ss.tile_base + i, ss.far_ctr,
                                warp, lane, lo, dn, out_map, lres, ldang, lsum, s_rcp, pol_out);
        if (lane == 0) {
            tma_store_wait_all();  // c' complete before the grid barrier
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        __syncwarp();
    }
    ss.ring_base += LE;
    ss.tile_base += L;
    lres_out = __dadd_rn(lres_out, lres);
    ldang_out = __dadd_rn(ldang_out, ldang);
    lsum_out = __dadd_rn(lsum_out, lsum);
}

__device__ __forceinline__ double reduce_parts_r(const double* part, int nblocks, int k,
                                                 double* s_red) {
    double acc = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += kRowThreads) acc = __dadd_rn(acc, part[b * 3 + k]);
    return block_sum<kRowThreads>(acc, s_red);
}

// Persistent cooperative kernel, one CTA per SM: the whole power iteration
// (same iteration, stop rule and closing r' pass as pagerank_staged_kernel).
template <class RS>
__global__ void __launch_bounds__(kRowThreads, 1)
    pagerank_rows_kernel(const __grid_constant__ RowMaps maps, const __grid_constant__ RowPlan p,
                         const __grid_constant__ PrArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    __shared__ double s_red[kRowThreads / 32];
    __shared__ double s_rcp[kPackedSlots + 1];
    const int t = threadIdx.x;
    if (t <= kPackedSlots) s_rcp[t] = t ? __drcp_rn(static_cast<double>(t)) : 0.0;
    RowCtx cx;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
    cx.c_full = bars;
    cx.c_empty = cx.c_full + kRingTiles;
    cx.pw_full = cx.c_empty + kRingTiles;
    cx.pw_empty = cx.pw_full + kPwTiles;
    cx.far_full = cx.pw_empty + kPwTiles;
    cx.far_empty = cx.far_full + kRW * kFarSlots;
    cx.ring = smem + kOffRing;
    cx.far = smem + kOffFar;
    cx.out = smem + kOffOut;
    cx.pwr = smem + kOffPw;
    cx.desc = reinterpret_cast<uint4*>(smem + kOffDesc);
    // the ring starts zeroed: the first sweep's first tiles read (and multiply
    // by 0) ring rows that were never loaded
    for (int k = t; k < kRingTiles * kTileBytes / 16; k += kRowThreads)
        reinterpret_cast<uint4*>(cx.ring)[k] = make_uint4(0, 0, 0, 0);
    if (t == 0) {
        for (int k = 0; k < kRingTiles; ++k) {
            bar_init(cx.c_full + k, 1);
            bar_init(cx.c_empty + k, 2 * p.ahead + 1);
        }
        for (int k = 0; k < kPwTiles; ++k) {
            bar_init(cx.pw_full + k, 1);
            bar_init(cx.pw_empty + k, 1);
        }
        for (int k = 0; k < kRW * kFarSlots; ++k) {
            bar_init(cx.far_full + k, 1);
            bar_init(cx.far_empty + k, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeroed ring before TMA writes
    if (t < 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.c[0])) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.c[1])) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.pw)) : "memory");
    }
    __syncthreads();
    cg::grid_group grid = cg::this_grid();
    const uint32_t G = gridDim.x;

    // r_0 = 1/N: c_0 = r_0 / outdeg (r_0 for sinks), D_0 = sum over sinks
    double dang = 0.0;
    const uint64_t gsize = static_cast<uint64_t>(G) * kRowThreads;
    for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * kRowThreads + t; v < a.n; v += gsize) {
        const uint32_t deg = __ldg(a.pw + v) >> kPackedSlots;
        if (deg) {
            a.c0[v] = __ddiv_rn(a.inv_n, static_cast<double>(deg));
        } else {
            a.c0[v] = a.inv_n;
            dang = __dadd_rn(dang, a.inv_n);
        }
    }
    dang = block_sum<kRowThreads>(dang, s_red);
    if (t == 0) a.part[blockIdx.x * 3 + 1] = dang;
    asm volatile("fence.proxy.async;" ::: "memory");  // c0 (generic stores) before TMA reads
    grid.sync();
    double D = reduce_parts_r(a.part, G, 1, s_red);

    const uint32_t L = block_tiles(p);       // tiles per sweep of this block
    const uint32_t LE = L + p.ahead;         // ring entries per sweep (A overhang)
    SweepState ss{0, 0, 0};                  // running counters (continue across sweeps)
    long long it = 0;
    int cur = 0;
    double res = 0.0, sum = 0.0, dn_last = 0.0;
    int status = 1;
    const PrScalars sc{a.teleport, a.damping};

    while (it < a.max_iter) {
        const double dn = __ddiv_rn(D, a.nd);
        double lres = 0.0, ldang = 0.0, lsum = 0.0;
        row_sweep<RS, false>(p, maps, cx, sc, L, LE, ss, cur, cur ^ 1, dn, lres, ldang, lsum, s_rcp);
        lres = block_sum<kRowThreads>(lres, s_red);
        ldang = block_sum<kRowThreads>(ldang, s_red);
        lsum = block_sum<kRowThreads>(lsum, s_red);
        double* part = a.part + static_cast<size_t>((it + 1) & 1) * G * 3;
        if (t == 0) {
            part[blockIdx.x * 3 + 0] = lres;
            part[blockIdx.x * 3 + 1] = ldang;
            part[blockIdx.x * 3 + 2] = lsum;
        }
        grid.sync();
        res = reduce_parts_r(part, G, 0, s_red);
        D = reduce_parts_r(part, G, 1, s_red);
        sum = reduce_parts_r(part, G, 2, s_red);
        dn_last = dn;
        ++it;
        cur ^= 1;
        if (res < a.tol) {
            status = 0;
            break;
        }
    }
    // r' of the last iteration from the contributions it read (buffer cur ^ 1)
    {
        double l0 = 0.0, l1 = 0.0, l2 = 0.0;
        row_sweep<RS, true>(p, maps, cx, sc, L, LE, ss, cur ^ 1, 2, dn_last, l0, l1, l2, s_rcp);
    }
    if (blockIdx.x == 0 && t == 0) {
        *a.out_iter = it;
        *a.out_res = res;
        *a.out_sum = sum;
        *a.out_parity = 0;
        *a.out_status = status;
    }
}

// ------------------------------------------------------------------ host --

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

// rows x (16 elements of 8 or 4 bytes) tensor, 32-row boxes of `width` elements
bool encode_rows(CUtensorMap* m, const void* base, uint64_t rows, bool f64, int width = 16) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {16, rows};
    const cuuint64_t strides[1] = {f64 ? 128ull : 64ull};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(width), kTileRows};
    const cuuint32_t es[2] = {1, 1};
    return fn(m, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2,
              const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              (f64 && width == 16) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class RS>
void* rows_kernel() {
    return reinterpret_cast<void*>(pagerank_rows_kernel<RS>);
}

// row dims (radices, most significant first) -> kernel instance
void* rows_kernel_for(const int* rm, int nd) {
    auto is = [&](int a, int b, int c, int d) {
        const int want[4] = {a, b, c, d};
        for (int k = 0; k < 4; ++k)
            if ((k < nd ? rm[k] : 1) != want[k]) return false;
        return true;
    };
    if (is(4, 2, 2, 1)) return rows_kernel<RowShape<4, 2, 2, 1>>();
    if (is(2, 2, 2, 2)) return rows_kernel<RowShape<2, 2, 2, 2>>();
    if (is(4, 4, 1, 1)) return rows_kernel<RowShape<4, 4, 1, 1>>();
    if (is(2, 4, 2, 1)) return rows_kernel<RowShape<2, 4, 2, 1>>();
    if (is(2, 2, 4, 1)) return rows_kernel<RowShape<2, 2, 4, 1>>();
    if (is(8, 2, 1, 1)) return rows_kernel<RowShape<8, 2, 1, 1>>();
    if (is(2, 8, 1, 1)) return rows_kernel<RowShape<2, 8, 1, 1>>();
    if (is(16, 1, 1, 1)) return rows_kernel<RowShape<16, 1, 1, 1>>();
    return nullptr;
}

}  // namespace

bool make_row_plan(const DevShape& s, int num_sms, RowPlan* out) {
    // experimental until it beats pagerank_staged_kernel on C5: TK_PR_ROWS=1 selects it
    const char* env = std::getenv("TK_PR_ROWS");
    if (!env || std::strcmp(env, "1") != 0) return false;
    if (s.kind != TK_ADJACENT || 2 * s.dims > kPackedSlots || s.dims < 3) return false;
    if (s.n % (kRowLen * kTileRows) != 0) return false;
    // row dims: trailing dims whose radices multiply to exactly 16
    int nd = 0;
    uint64_t prod = 1;
    while (nd < s.dims && prod < 16) prod *= s.radix[s.dims - 1 - nd++];
    if (prod != 16 || nd > 4) return false;
    RowPlan p{};
    p.dims = s.dims;
    p.nrow_dims = nd;
    for (int k = 0; k < nd; ++k) p.row_radix[k] = static_cast<int>(s.radix[s.dims - nd + k]);
    if (!rows_kernel_for(p.row_radix, nd)) return false;
    const int dr = s.dims - nd;  // non-row dims 0..dr-1, row stride = stride / 16
    if (dr < 1) return false;
    const uint64_t rows = s.n / kRowLen;
    // window: dims F..dr-1 (the largest suffix) with lookahead A = ceil(stride_rows(F) / 32)
    // small enough for the ring (2A + kRW + 2 <= kRingTiles), at least 2 columns per
    // CTA, and a column-group ("super-column", a whole number of 32-row tiles) length
    int maxA = (kRingTiles - kRW - 2) / 2;
    if (const char* e = std::getenv("TK_ROW_MAXA")) maxA = std::max(0, std::min(maxA, std::atoi(e)));
    uint64_t min_cols = static_cast<uint64_t>(2 * num_sms);  // keep every SM busy
    if (const char* e = std::getenv("TK_ROW_MINCOLS")) min_cols = std::strtoull(e, nullptr, 0);
    int bestF = -1;
    for (int F = 1; F <= dr; ++F) {
        const uint64_t srow = s.stride[F - 1] / kRowLen;  // rows per column (dims F..)
        const uint64_t wmax = F < dr ? s.stride[F] / kRowLen : 0;
        const int A = static_cast<int>((wmax + kTileRows - 1) / kTileRows);
        if (A > maxA) continue;
        // super-column: lcm(srow, 32) rows
        uint64_t g = srow, b = kTileRows;
        while (b) {
            const uint64_t r = g % b;
            g = b;
            b = r;
        }
        const uint64_t sc = srow / g * kTileRows;
        if (rows % sc) continue;
        if (rows / sc < min_cols && F < dr) continue;
        bestF = F;
        p.col_rows = static_cast<uint32_t>(sc);
        p.far_per_col = sc == srow ? 1 : 0;  // one column per super-column
        p.ahead = A;
        break;
    }
    if (bestF < 0) return false;
    p.nfar = bestF;
    p.nwin = dr - bestF;
    p.ncols = static_cast<uint32_t>(rows / p.col_rows);
    p.tiles_per_col = p.col_rows / kTileRows;
    p.tpc_magic = p.tiles_per_col > 1 ? (~0ull / p.tiles_per_col + 1) : 0;
    p.rows = static_cast<uint32_t>(rows);
    for (int k = 0; k < p.nwin; ++k) p.win_rows[k] = static_cast<int>(s.stride[bestF + k] / kRowLen);
    // far dims: digit of row r = (r / far_rows) % radix; L2 evict-first when the
    // range's reuse distance (~2 strides of c, c' and pw: 2.5 * 16 B per row... per
    // rank 20 B) exceeds about half of L2
    const uint64_t l2_half = 60ull << 20;
    for (int d = 0; d < p.nfar; ++d) {
        const uint64_t fr = s.stride[d] / kRowLen;
        p.far_rows[d] = static_cast<uint32_t>(fr);
        p.far_radix[d] = s.radix[d];
        p.far_magic[d] = fr > 1 ? (~0ull / fr + 1) : 0;
        p.far_rmagic[d] = ~0ull / s.radix[d] + 1;
        // a tile (32 rows) may hold several digit values of this dim: stage both sides
        p.far_span[d] = fr * s.radix[d] <= static_cast<uint64_t>(kTileRows) ? 1 : 0;
        const uint64_t reuse = 2 * fr * kRowLen * 20;
        if (reuse > l2_half) p.far_ef |= 1u << d;
    }
    if (const char* e = std::getenv("TK_ROW_EF")) p.far_ef = static_cast<uint32_t>(std::strtoul(e, nullptr, 0));
    *out = p;
    return true;
}

cudaError_t launch_pagerank_rows(const DevShape& s, const RowPlan& p, const PrArgs& a,
                                 int num_sms, int* grid_out, cudaStream_t stream) {
    void* k = rows_kernel_for(p.row_radix, p.nrow_dims);
    if (!k) return cudaErrorInvalidValue;
    RowMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    const uint64_t rows = p.rows;
    if (!encode_rows(&maps.c[0], a.c0, rows, true) || !encode_rows(&maps.c[1], a.c1, rows, true) ||
        !encode_rows(&maps.pw, a.pw, rows, false) || !encode_rows(&maps.r0, a.r0, rows, true))
        return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmem);
    if (e != cudaSuccess) return e;
    int bps = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, kRowThreads, kRowSmem);
    if (e != cudaSuccess) return e;
    if (bps < 1) return cudaErrorInvalidConfiguration;
    uint64_t g = static_cast<uint64_t>(num_sms);
    if (g > p.ncols) g = p.ncols;
    *grid_out = static_cast<int>(g);
    if (std::getenv("TK_DEBUG")) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, k);
        std::fprintf(stderr,
                     "[tk] pagerank_rows row_dims=%d far=%d win=%d A=%d col_rows=%u ncols=%u "
                     "far_ef=0x%x smem=%d static=%zu regs=%d grid=%llu\n",
                     p.nrow_dims, p.nfar, p.nwin, p.ahead, p.col_rows, p.ncols, p.far_ef, kRowSmem,
                     fa.sharedSizeBytes, fa.numRegs, static_cast<unsigned long long>(g));
    }
    RowPlan pc = p;
    PrArgs ac = a;
    void* args[] = {&maps, &pc, &ac};
    return cudaLaunchCooperativeKernel(k, dim3(static_cast<unsigned>(g)), dim3(kRowThreads), args,
                                       kRowSmem, stream);
}

}  // namespace tk
