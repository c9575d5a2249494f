// TMA-staged sum-check round (sm_100a): the large-table form of k_round
// (sumcheck.hpp:118-144 round_poly_over + fold_over, mle.hpp:75-85) for the
// GKR layer sum-check's pair (V, H) plus the G table (sumcheck.hpp:368-440).
//
// Why: the register-fed k_round runs at 2 CTAs/SM (112 registers) with one
// output pair in flight per thread, so HBM latency is exposed (ncu r1: 24%
// warps active, 35-53% issue active, long-scoreboard the top stall on the
// fold rounds). Here every warp streams its own tables into its own
// shared-memory ring with cp.async.bulk.tensor (TMA): lane 0 refills a stage
// as soon as the warp has read it, so loads run ahead of the field
// arithmetic without costing registers and no warp ever waits for another.
// (A CTA-wide ring refilled by one thread measured slower: the refill had
// to wait for the slowest warp. A dedicated producer warp would cap the
// registers at 96 -- 5 warps on some SM sub-partitions -- and spill.)
//
// Layout: every table is viewed as a 2-D tensor of 128-byte rows (4 field
// elements) with the 128-byte swizzle, so each consumer's 16-byte shared
// loads are bank-conflict free in all three access patterns:
//   kScan     (round 1)   index i = elements (2i, 2i+1): tile = 128 rows
//   kFoldNat  (round 2)   index i = elements 4i..4i+3:   tile = 256 rows
//   kFoldRev  (rounds>=3) index i = elements i, i+P, i+2P, i+3P of the
//                         bit-reversed table: 4 boxes of 64 rows per tile
// A warp-tile is 32 output pairs; one ring stage holds one table's part of a
// warp-tile, so a warp-tile is ntab stages.
#pragma once

#include <cuda.h>  // CUtensorMap (the map is built on the host by cuTensorMapEncodeTiled)

constexpr int kTmaWarps = 8;
constexpr int kTmaThreads = 32 * kTmaWarps;
constexpr int kTmaWarpRing = 12 * 1024;  // per warp: 3 fold stages of 4 KB (6 scan stages of 2 KB)
constexpr int kTmaRingBytes = kTmaWarps * kTmaWarpRing;
constexpr int kTmaMaxTabs = 3;
constexpr int kTmaTile = 32;  // output pairs per warp-tile

struct RoundTmaParams {
    CUtensorMap map[kTmaMaxTabs];  // input tables, 2-D {32 x u32, rows}, SWIZZLE_128B
    Fe* out[kTmaMaxTabs];          // fold outputs (unused by kScan)
    std::uint64_t n_out_pairs;     // P (a multiple of kTmaTile)
    int log_p;
    int ntab;
    Fe* partials;
    unsigned* counter;
    Fe* result;
    FoldConst k;  // fold challenge (kernel-parameter space: IMAD constant operands)
    // debug (DGKR_TMA_VERIFY): every staged element is compared with a
    // direct global load of in[t]; mismatches counted in dbg[0], first one in dbg[1..4]
    const Fe* in[kTmaMaxTabs];
    unsigned* dbg;
};

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
/// TMA: box at (c0, c1) of *map -> dst (shared-window address), completion on bar (tx bytes)
__device__ __forceinline__ void tma_load_2d(std::uint32_t dst, const CUtensorMap* map, std::uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

/// 16 bytes from shared memory at a 32-bit shared-window address (LDS.128;
/// a generic pointer here compiles to LD.E through the generic path)
__device__ __forceinline__ uint4 lds128(std::uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
    return v;
}

/// element at (row, first 16-byte chunk c0) of a SWIZZLE_128B box at shared
/// address `box` (1024-aligned): chunk c of row r sits at chunk c ^ (r & 7)
__device__ __forceinline__ Fe lds_fe_swz(std::uint32_t box, std::uint32_t row, std::uint32_t c0) {
    const std::uint32_t sw = row & 7;
    const std::uint32_t r = box + row * 128;
    const uint4 lo = lds128(r + ((c0 ^ sw) << 4));
    const uint4 hi = lds128(r + (((c0 + 1) ^ sw) << 4));
    Fe x;
    x.v[0] = lo.x; x.v[1] = lo.y; x.v[2] = lo.z; x.v[3] = lo.w;
    x.v[4] = hi.x; x.v[5] = hi.y; x.v[6] = hi.z; x.v[7] = hi.w;
    return x;
}

template <int MODE>
struct TmaShape {
    static constexpr int kStageBytes = MODE == kScan ? kTmaTile * 64 : kTmaTile * 128;
    static constexpr int kStages = kTmaWarpRing / kStageBytes;
    // rows of one TMA box: kScan 2 pairs per row, kFoldNat 1, kFoldRev 4 boxes of 4 elements per row
    static constexpr int kBoxRows = MODE == kScan ? kTmaTile / 2 : (MODE == kFoldNat ? kTmaTile : kTmaTile / 4);
};

#ifdef DGKR_TMA_DEBUG
__device__ __noinline__ void tma_verify(const RoundTmaParams& a, int t, std::uint64_t gi, const Fe& x, int mode) {
    const Fe y = fe_load(a.in[t] + gi);
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 8; ++k) ok &= x.v[k] == y.v[k];
    if (!ok && atomicAdd(a.dbg, 1u) == 0) {
        a.dbg[1] = static_cast<unsigned>(t);
        a.dbg[2] = static_cast<unsigned>(gi);
        a.dbg[3] = static_cast<unsigned>(mode);
        a.dbg[4] = blockIdx.x;
    }
}
#define TMA_VERIFY(...) \
    if (a.dbg) {        \
        __VA_ARGS__;    \
    }
#else
#define TMA_VERIFY(...)
#endif

/// Lane view of one table of one warp-tile: the pair (x0, x1) of output index
/// i = wtile * 32 + lane, folded with the challenge unless kScan; fold outputs
/// are stored as in load_pair (kFoldNat writes bit-reversed).
template <class F, int MODE>
__device__ __forceinline__ void tma_pair(std::uint32_t st, int lane, std::uint64_t i, const RoundTmaParams& a,
                                         Fe* dst, Fe& x0, Fe& x1, int t) {
    const std::uint64_t P = a.n_out_pairs;
    if (MODE == kScan) {
        const std::uint32_t row = lane >> 1, cb = (lane & 1) * 4;
        x0 = lds_fe_swz(st, row, cb);
        x1 = lds_fe_swz(st, row, cb + 2);
        TMA_VERIFY(tma_verify(a, t, 2 * i, x0, MODE); tma_verify(a, t, 2 * i + 1, x1, MODE))
    } else if (MODE == kFoldNat) {
        const Fe a0 = lds_fe_swz(st, lane, 0), a1 = lds_fe_swz(st, lane, 2);
        const Fe b0 = lds_fe_swz(st, lane, 4), b1 = lds_fe_swz(st, lane, 6);
        TMA_VERIFY(tma_verify(a, t, 4 * i, a0, MODE); tma_verify(a, t, 4 * i + 1, a1, MODE);
                   tma_verify(a, t, 4 * i + 2, b0, MODE); tma_verify(a, t, 4 * i + 3, b1, MODE))
        x0 = foldk<F>(a0, a1, a.k);
        x1 = foldk<F>(b0, b1, a.k);
        const std::uint64_t s = a.log_p ? (__brevll(i) >> (64 - a.log_p)) : 0;
        fe_store(dst + s, x0);
        fe_store(dst + s + P, x1);
    } else {
        const std::uint32_t row = lane >> 2, cb = (lane & 3) * 2;
        constexpr int seg = kTmaTile * 32;  // one box: 32 elements, 1 KB
        const Fe a0 = lds_fe_swz(st, row, cb), b0 = lds_fe_swz(st + seg, row, cb);
        const Fe a1 = lds_fe_swz(st + 2 * seg, row, cb), b1 = lds_fe_swz(st + 3 * seg, row, cb);
        TMA_VERIFY(tma_verify(a, t, i, a0, MODE); tma_verify(a, t, i + P, b0, MODE);
                   tma_verify(a, t, i + 2 * P, a1, MODE); tma_verify(a, t, i + 3 * P, b1, MODE))
        x0 = foldk<F>(a0, a1, a.k);
        x1 = foldk<F>(b0, b1, a.k);
        fe_store(dst + i, x0);
        fe_store(dst + i + P, x1);
    }
}

/// One round over the layer tables (V, H, G): S0 = sum V0 H0 + G0,
/// S2 = sum dV dH (and S1 = sum V1 H1 + G1 when S1). Grid: persistent CTAs
/// (<= 2 per SM) of 8 independent warps; warp g of G strides over warp-tiles
/// g, g + G, ...; its units (warp-tile, table) stream through its own ring.
template <class F, int MODE, bool S1>
__global__ void __launch_bounds__(kTmaThreads, 2) k_round_tma(const __grid_constant__ RoundTmaParams a) {
    using Shape = TmaShape<MODE>;
    constexpr int NS = S1 ? 3 : 2;
    constexpr int kStages = Shape::kStages;
    constexpr bool kWide = MODE == kScan && !S1;  // round 1: unreduced products, one REDC per CTA
    extern __shared__ std::uint8_t smem_raw[];
    __shared__ std::uint64_t full_all[kTmaWarps][kStages];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    std::uint64_t* full = full_all[warp];
    // this warp's ring as a 32-bit shared-window address, 1024-aligned for the swizzle
    const std::uint32_t ring = ((smem_u32(smem_raw) + 1023u) & ~1023u) + warp * kTmaWarpRing;
    const std::uint64_t P = a.n_out_pairs;
    const std::uint64_t n_wt = P / kTmaTile;
    const std::uint64_t G = static_cast<std::uint64_t>(gridDim.x) * kTmaWarps;
    const std::uint64_t g = static_cast<std::uint64_t>(blockIdx.x) * kTmaWarps + warp;
    const std::uint64_t my_wt = g < n_wt ? (n_wt - g + G - 1) / G : 0;
    const std::uint64_t n_units = my_wt * a.ntab;
    // unit u = (warp-tile g + (u / ntab) G, table u % ntab) -> stage s (lane 0 only)
    auto issue = [&](std::uint64_t u, int s) {
        const std::uint64_t wt = g + (u / a.ntab) * G;
        const int t = static_cast<int>(u % a.ntab);
        const std::uint32_t dst = ring + s * Shape::kStageBytes;
        mbar_expect_tx(&full[s], Shape::kStageBytes);
        if (MODE == kScan) {
            tma_load_2d(dst, &a.map[t], &full[s], 0, static_cast<int>(wt * (kTmaTile / 2)));
        } else if (MODE == kFoldNat) {
            tma_load_2d(dst, &a.map[t], &full[s], 0, static_cast<int>(wt * kTmaTile));
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                tma_load_2d(dst + q * (kTmaTile * 32), &a.map[t], &full[s], 0,
                            static_cast<int>((wt * kTmaTile + q * P) >> 2));
        }
    };
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < kStages && static_cast<std::uint64_t>(s) < n_units; ++s) issue(s, s);
    }
    __syncwarp();
    std::conditional_t<kWide, Acc, Fe> w[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        if constexpr (kWide) acc_zero(w[k]);
        else w[k] = fe_zero();
    }
    int s = 0;
    std::uint32_t ph = 0;
    std::uint64_t u = 0;
    // consume unit u from stage s; once the whole warp has read it, lane 0
    // refills the stage with unit u + kStages
    auto next = [&](Fe* dst, std::uint64_t i, Fe& x0, Fe& x1, int t) {
        mbar_wait(&full[s], ph);
        tma_pair<F, MODE>(ring + s * Shape::kStageBytes, lane, i, a, dst, x0, x1, t);
        __syncwarp();
        if (lane == 0 && u + kStages < n_units) {
            // the warp's generic-proxy reads of this stage before the async-proxy (TMA) refill
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(u + kStages, s);
        }
        ++u;
        if (++s == kStages) {
            s = 0;
            ph ^= 1;
        }
    };
    for (std::uint64_t k = 0; k < my_wt; ++k) {
        const std::uint64_t i = (g + k * G) * kTmaTile + lane;
        Fe f0, f1;
        // one (rolled) copy of the staged fold for the three tables keeps
        // the loop body small in the instruction cache
#pragma unroll 1
        for (int t = 0; t < 3; ++t) {
            Fe x0, x1;
            next(a.out[t], i, x0, x1, t);
            if (t == 0) {
                f0 = x0;
                f1 = x1;
            } else if (t == 1) {
                sum_prod<F>(w[0], f0, x0);
                if constexpr (S1) sum_prod<F>(w[1], f1, x1);
                sum_prod<F>(w[NS - 1], fe_sub_lazy<F>(f1, f0), fe_sub_lazy<F>(x1, x0));
            } else {
                sum_val<F>(w[0], x0);
                if constexpr (S1) sum_val<F>(w[1], x1);
            }
        }
    }
    Fe sums[NS];
    if constexpr (kWide) {
        block_sum_wide<F, NS>(w, sums);
        grid_finish<F, NS>(sums, a.partials, a.counter, a.result, true);
    } else {
#pragma unroll
        for (int k = 0; k < NS; ++k) sums[k] = w[k];
        grid_finish<F, NS>(sums, a.partials, a.counter, a.result);
    }
}
