// Device prime-field arithmetic for sm_100a: 256-bit Montgomery form
// (R = 2^256, 8 x 32-bit little-endian limbs, the same bits as the host's
// 4 x 64-bit HostField), multiplication by CIOS with 64-bit partial products
// (IMAD.WIDE on the integer pipe) and PTX carry chains for add/sub.
//
// Two modulus policies:
//   Bn254  - BN254 Fr (field.hpp:44-49) with the modulus as immediates;
//   Rt     - any odd modulus < 2^254 read from __constant__ memory, so the
//            drop-in also serves the reference tests' p=97 / Goldilocks
//            (tests/test_sumcheck.cpp:76-86, test_field.cpp:76-95).
// Values are always fully reduced (< p), so equality is bitwise and the
// canonical encoding (field.hpp:159-167) is one Montgomery reduction away.
#pragma once

#include <cstdint>

#include "fe.hpp"

namespace dgkr_b200 {

struct RtFieldConst {
    uint32_t p[8];
    uint32_t np0;
    uint32_t r2[8];
    uint32_t one[8];
};

// Runtime-modulus constants (only kernels.cu includes this header).
__constant__ RtFieldConst c_rt_field;

struct Bn254 {
    static constexpr bool kRuntime = false;
    static constexpr bool kWide = false;
    __device__ __forceinline__ static uint32_t p(int i) {
        constexpr uint32_t P[8] = {0xf0000001u, 0x43e1f593u, 0x79b97091u, 0x2833e848u,
                                   0x8181585du, 0xb85045b6u, 0xe131a029u, 0x30644e72u};
        return P[i];
    }
    __device__ __forceinline__ static uint32_t np0() { return 0xefffffffu; }
    __device__ __forceinline__ static uint32_t r2(int i) {
        constexpr uint32_t R2[8] = {0xae216da7u, 0x1bb8e645u, 0xe35c59e3u, 0x53fe3ab1u,
                                    0x53bb8085u, 0x8c49833du, 0x7f4e44a5u, 0x0216d0b1u};
        return R2[i];
    }
    __device__ __forceinline__ static uint32_t one(int i) {
        constexpr uint32_t ONE[8] = {0x4ffffffbu, 0xac96341cu, 0x9f60cd29u, 0x36fc7695u,
                                     0x7879462eu, 0x666ea36fu, 0x9a07df2fu, 0x0e0a77c1u};
        return ONE[i];
    }
};

struct Rt {
    static constexpr bool kRuntime = true;
    static constexpr bool kWide = false;
    __device__ __forceinline__ static uint32_t p(int i) { return c_rt_field.p[i]; }
    __device__ __forceinline__ static uint32_t np0() { return c_rt_field.np0; }
    __device__ __forceinline__ static uint32_t r2(int i) { return c_rt_field.r2[i]; }
    __device__ __forceinline__ static uint32_t one(int i) { return c_rt_field.one[i]; }
};

/// Runtime modulus with 2^254 <= p < 2^256 (the reference accepts any prime,
/// field.hpp:26-40): a + b may carry out of 256 bits and 4p > 2^256, so adds
/// are carry-aware, differences are fully reduced and products use the
/// 10-limb CIOS with a 257-bit final comparison.
struct RtW : Rt {
    static constexpr bool kWide = true;
};

// ---------------------------------------------------------------------------

__device__ __forceinline__ Fe fe_zero() {
    Fe r;
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = 0;
    return r;
}

template <class F>
__device__ __forceinline__ Fe fe_one() {
    Fe r;
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = F::one(i);
    return r;
}

__device__ __forceinline__ bool fe_is_zero(const Fe& a) {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) x |= a.v[i];
    return x == 0;
}

__device__ __forceinline__ Fe fe_load(const Fe* p) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
    uint4 a = q[0], b = q[1];
    Fe r;
    r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
    r.v[4] = b.x; r.v[5] = b.y; r.v[6] = b.z; r.v[7] = b.w;
    return r;
}

__device__ __forceinline__ Fe fe_load_nc(const Fe* p) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
    uint4 a = __ldg(q), b = __ldg(q + 1);
    Fe r;
    r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
    r.v[4] = b.x; r.v[5] = b.y; r.v[6] = b.z; r.v[7] = b.w;
    return r;
}

__device__ __forceinline__ void fe_store(Fe* p, const Fe& x) {
    uint4* q = reinterpret_cast<uint4*>(p);
    q[0] = make_uint4(x.v[0], x.v[1], x.v[2], x.v[3]);
    q[1] = make_uint4(x.v[4], x.v[5], x.v[6], x.v[7]);
}

// One 256-bit access per element (LDG/STG .ENL2.256, new on sm_100) for
// tables in global memory, whose elements are 32-byte aligned (cudaMalloc
// bases, Fe-strided offsets): half the load/store instructions of the
// two-uint4 forms above. DGKR_V8=0 builds the uint4 forms (A/B).
#ifndef DGKR_V8
#define DGKR_V8 1
#endif
__device__ __forceinline__ Fe fe_load_nc32(const Fe* p) {
#if DGKR_V8
    Fe r;
    asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]),
          "=r"(r.v[7])
        : "l"(p));
    return r;
#else
    return fe_load_nc(p);
#endif
}

/// L2-only (coherent within a launch) 256-bit load
__device__ __forceinline__ Fe fe_ldcg32(const Fe* p) {
    Fe r;
#if DGKR_V8
    asm volatile("ld.global.cg.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                   "=r"(r.v[6]), "=r"(r.v[7])
                 : "l"(p)
                 : "memory");
#else
    const uint4* q = reinterpret_cast<const uint4*>(p);
    uint4 a = __ldcg(q), b = __ldcg(q + 1);
    r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
    r.v[4] = b.x; r.v[5] = b.y; r.v[6] = b.z; r.v[7] = b.w;
#endif
    return r;
}

// no "memory" clobber, so later table loads can still be hoisted above it:
// nothing in a launch reads these stores back except through fe_ldcg32
// (volatile, ordered after it) or after a grid-wide sync
__device__ __forceinline__ void fe_store32(Fe* p, const Fe& x) {
#if DGKR_V8
    asm volatile("st.global.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(x.v[0]), "r"(x.v[1]),
                 "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]), "r"(x.v[6]), "r"(x.v[7]));
#else
    fe_store(p, x);
#endif
}

/// a + b mod p for 2^254 <= p < 2^256: the sum's carry-out takes part in the comparison
template <class F>
__device__ __forceinline__ Fe fe_add_wide(const Fe& a, const Fe& b) {
    Fe s, t;
    uint32_t carry, borrow;
    asm("add.cc.u32  %0, %9, %17;\n\t"
        "addc.cc.u32 %1, %10, %18;\n\t"
        "addc.cc.u32 %2, %11, %19;\n\t"
        "addc.cc.u32 %3, %12, %20;\n\t"
        "addc.cc.u32 %4, %13, %21;\n\t"
        "addc.cc.u32 %5, %14, %22;\n\t"
        "addc.cc.u32 %6, %15, %23;\n\t"
        "addc.cc.u32 %7, %16, %24;\n\t"
        "addc.u32    %8, 0, 0;"
        : "=r"(s.v[0]), "=r"(s.v[1]), "=r"(s.v[2]), "=r"(s.v[3]), "=r"(s.v[4]), "=r"(s.v[5]), "=r"(s.v[6]),
          "=r"(s.v[7]), "=r"(carry)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    asm("sub.cc.u32  %0, %9, %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;"
        : "=r"(t.v[0]), "=r"(t.v[1]), "=r"(t.v[2]), "=r"(t.v[3]), "=r"(t.v[4]), "=r"(t.v[5]), "=r"(t.v[6]),
          "=r"(t.v[7]), "=r"(borrow)
        : "r"(s.v[0]), "r"(s.v[1]), "r"(s.v[2]), "r"(s.v[3]), "r"(s.v[4]), "r"(s.v[5]), "r"(s.v[6]), "r"(s.v[7]),
          "r"(F::p(0)), "r"(F::p(1)), "r"(F::p(2)), "r"(F::p(3)), "r"(F::p(4)), "r"(F::p(5)), "r"(F::p(6)),
          "r"(F::p(7)));
    const bool keep = borrow && !carry;  // s < p and no carry: s is reduced
    Fe r;
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = keep ? s.v[i] : t.v[i];
    return r;
}

/// r = a + b mod p (a, b < p < 2^254: the raw sum never carries out).
template <class F>
__device__ __forceinline__ Fe fe_add(const Fe& a, const Fe& b) {
    if constexpr (F::kWide) return fe_add_wide<F>(a, b);
    Fe s, t;
    asm("add.cc.u32  %0, %8, %16;\n\t"
        "addc.cc.u32 %1, %9, %17;\n\t"
        "addc.cc.u32 %2, %10, %18;\n\t"
        "addc.cc.u32 %3, %11, %19;\n\t"
        "addc.cc.u32 %4, %12, %20;\n\t"
        "addc.cc.u32 %5, %13, %21;\n\t"
        "addc.cc.u32 %6, %14, %22;\n\t"
        "addc.u32    %7, %15, %23;"
        : "=r"(s.v[0]), "=r"(s.v[1]), "=r"(s.v[2]), "=r"(s.v[3]), "=r"(s.v[4]), "=r"(s.v[5]), "=r"(s.v[6]),
          "=r"(s.v[7])
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    uint32_t borrow;
    asm("sub.cc.u32  %0, %9, %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;"
        : "=r"(t.v[0]), "=r"(t.v[1]), "=r"(t.v[2]), "=r"(t.v[3]), "=r"(t.v[4]), "=r"(t.v[5]), "=r"(t.v[6]),
          "=r"(t.v[7]), "=r"(borrow)
        : "r"(s.v[0]), "r"(s.v[1]), "r"(s.v[2]), "r"(s.v[3]), "r"(s.v[4]), "r"(s.v[5]), "r"(s.v[6]), "r"(s.v[7]),
          "r"(F::p(0)), "r"(F::p(1)), "r"(F::p(2)), "r"(F::p(3)), "r"(F::p(4)), "r"(F::p(5)), "r"(F::p(6)),
          "r"(F::p(7)));
    Fe r;
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = borrow ? s.v[i] : t.v[i];
    return r;
}

/// r = a - b mod p.
template <class F>
__device__ __forceinline__ Fe fe_sub(const Fe& a, const Fe& b) {
    Fe s;
    uint32_t borrow;
    asm("sub.cc.u32  %0, %9, %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;"
        : "=r"(s.v[0]), "=r"(s.v[1]), "=r"(s.v[2]), "=r"(s.v[3]), "=r"(s.v[4]), "=r"(s.v[5]), "=r"(s.v[6]),
          "=r"(s.v[7]), "=r"(borrow)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]));
    Fe r;
    const uint32_t m0 = F::p(0) & borrow, m1 = F::p(1) & borrow, m2 = F::p(2) & borrow, m3 = F::p(3) & borrow,
                   m4 = F::p(4) & borrow, m5 = F::p(5) & borrow, m6 = F::p(6) & borrow, m7 = F::p(7) & borrow;
    asm("add.cc.u32  %0, %8, %16;\n\t"
        "addc.cc.u32 %1, %9, %17;\n\t"
        "addc.cc.u32 %2, %10, %18;\n\t"
        "addc.cc.u32 %3, %11, %19;\n\t"
        "addc.cc.u32 %4, %12, %20;\n\t"
        "addc.cc.u32 %5, %13, %21;\n\t"
        "addc.cc.u32 %6, %14, %22;\n\t"
        "addc.u32    %7, %15, %23;"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]),
          "=r"(r.v[7])
        : "r"(s.v[0]), "r"(s.v[1]), "r"(s.v[2]), "r"(s.v[3]), "r"(s.v[4]), "r"(s.v[5]), "r"(s.v[6]), "r"(s.v[7]),
          "r"(m0), "r"(m1), "r"(m2), "r"(m3), "r"(m4), "r"(m5), "r"(m6), "r"(m7));
    return r;
}

/// b - a + p in [0, 2p) without the conditional correction: for operands
/// that only feed a Montgomery product. CIOS keeps its < 2p output (and one
/// final subtraction) for inputs < 2p since 4p < R = 2^256 (p < 2^254), and
/// the constant-multiplier path accepts any 256-bit input.
template <class F>
__device__ __forceinline__ Fe fe_sub_lazy(const Fe& b, const Fe& a) {
    if constexpr (F::kWide) return fe_sub<F>(b, a);  // b - a + p may not fit 256 bits
    Fe r;
    asm("sub.cc.u32  %0, %8, %16;\n\t"
        "subc.cc.u32 %1, %9, %17;\n\t"
        "subc.cc.u32 %2, %10, %18;\n\t"
        "subc.cc.u32 %3, %11, %19;\n\t"
        "subc.cc.u32 %4, %12, %20;\n\t"
        "subc.cc.u32 %5, %13, %21;\n\t"
        "subc.cc.u32 %6, %14, %22;\n\t"
        "subc.u32    %7, %15, %23;\n\t"
        "add.cc.u32  %0, %0, %24;\n\t"
        "addc.cc.u32 %1, %1, %25;\n\t"
        "addc.cc.u32 %2, %2, %26;\n\t"
        "addc.cc.u32 %3, %3, %27;\n\t"
        "addc.cc.u32 %4, %4, %28;\n\t"
        "addc.cc.u32 %5, %5, %29;\n\t"
        "addc.cc.u32 %6, %6, %30;\n\t"
        "addc.u32    %7, %7, %31;"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]),
          "=r"(r.v[7])
        : "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]), "r"(b.v[6]), "r"(b.v[7]),
          "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(F::p(0)), "r"(F::p(1)), "r"(F::p(2)), "r"(F::p(3)), "r"(F::p(4)), "r"(F::p(5)), "r"(F::p(6)),
          "r"(F::p(7)));
    return r;
}

// ---- even/odd carry-chain rows (n = 8 limbs; a row uses x[off], x[off+2], ...) ----
// A row x[off + 2j] * y puts lo at acc[2j] and hi at acc[2j+1]: rows of even
// and of odd limbs never overlap within themselves, so each is ONE PTX
// mad/madc carry chain (IMAD / IMAD.X / IMAD.HI.X on the FMA pipe) instead of
// 64-bit partial products plus carry adds on the ALU pipe. All asm is
// volatile: the carry flag links consecutive statements.
__device__ __forceinline__ void eo_mul_row(uint32_t acc[8], const uint32_t* x, int off, uint32_t y) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
        asm volatile("mul.lo.u32 %0, %2, %3;\n\tmul.hi.u32 %1, %2, %3;"
                     : "=r"(acc[2 * j]), "=r"(acc[2 * j + 1])
                     : "r"(x[off + 2 * j]), "r"(y));
}
/// acc += row; the carry out of acc[7] is left in the carry flag
__device__ __forceinline__ void eo_mad_row(uint32_t acc[8], const uint32_t* x, int off, uint32_t y) {
    asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;"
                 : "+r"(acc[0]), "+r"(acc[1])
                 : "r"(x[off]), "r"(y));
#pragma unroll
    for (int j = 1; j < 4; ++j)
        asm volatile("madc.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;"
                     : "+r"(acc[2 * j]), "+r"(acc[2 * j + 1])
                     : "r"(x[off + 2 * j]), "r"(y));
}
/// dst[k] = row + src[k + 2] (src[8], src[9] = 0) + the carry flag at dst[0];
/// the carry out of dst[7] is 0 (every intermediate value is < 2^288)
__device__ __forceinline__ void eo_madc_row_rshift(uint32_t dst[8], const uint32_t* x, int off, uint32_t y,
                                                   const uint32_t src[8]) {
#pragma unroll
    for (int j = 0; j < 3; ++j)
        asm volatile("madc.lo.cc.u32 %0, %2, %3, %4;\n\tmadc.hi.cc.u32 %1, %2, %3, %5;"
                     : "=r"(dst[2 * j]), "=r"(dst[2 * j + 1])
                     : "r"(x[off + 2 * j]), "r"(y), "r"(src[2 * j + 2]), "r"(src[2 * j + 3]));
    asm volatile("madc.lo.cc.u32 %0, %2, %3, 0;\n\tmadc.hi.u32 %1, %2, %3, 0;"
                 : "=r"(dst[6]), "=r"(dst[7])
                 : "r"(x[off + 6]), "r"(y));
}

/// R < 2p -> R mod p (one conditional subtraction)
template <class F>
__device__ __forceinline__ Fe fe_reduce_once(const uint32_t (&t)[8]) {
    Fe d;
    uint32_t borrow;
    asm("sub.cc.u32  %0, %9, %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;"
        : "=r"(d.v[0]), "=r"(d.v[1]), "=r"(d.v[2]), "=r"(d.v[3]), "=r"(d.v[4]), "=r"(d.v[5]), "=r"(d.v[6]),
          "=r"(d.v[7]), "=r"(borrow)
        : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5]), "r"(t[6]), "r"(t[7]), "r"(F::p(0)),
          "r"(F::p(1)), "r"(F::p(2)), "r"(F::p(3)), "r"(F::p(4)), "r"(F::p(5)), "r"(F::p(6)), "r"(F::p(7)));
    Fe r;
#pragma unroll
    for (int j = 0; j < 8; ++j) r.v[j] = borrow ? t[j] : d.v[j];
    return r;
}

/// Montgomery product for 2^254 <= p < 2^256 (RtW): CIOS with a 10-limb
/// running value (< 2p < 2^257 between rows, < 2^289 inside a row) and a
/// final comparison that includes the 257th bit. Inputs < p.
template <class F>
__device__ __forceinline__ Fe fe_mul_wide(const Fe& a, const Fe& b) {
    uint32_t t[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint64_t c = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint64_t s = static_cast<uint64_t>(a.v[j]) * b.v[i] + t[j] + c;
            t[j] = static_cast<uint32_t>(s);
            c = s >> 32;
        }
        uint64_t s = static_cast<uint64_t>(t[8]) + c;
        t[8] = static_cast<uint32_t>(s);
        t[9] = static_cast<uint32_t>(s >> 32);
        const uint32_t m = t[0] * F::np0();
        c = (static_cast<uint64_t>(m) * F::p(0) + t[0]) >> 32;
#pragma unroll
        for (int j = 1; j < 8; ++j) {
            const uint64_t s2 = static_cast<uint64_t>(m) * F::p(j) + t[j] + c;
            t[j - 1] = static_cast<uint32_t>(s2);
            c = s2 >> 32;
        }
        s = static_cast<uint64_t>(t[8]) + c;
        t[7] = static_cast<uint32_t>(s);
        t[8] = t[9] + static_cast<uint32_t>(s >> 32);
    }
    Fe d;
    uint32_t borrow;
    asm("sub.cc.u32  %0, %9, %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;"
        : "=r"(d.v[0]), "=r"(d.v[1]), "=r"(d.v[2]), "=r"(d.v[3]), "=r"(d.v[4]), "=r"(d.v[5]), "=r"(d.v[6]),
          "=r"(d.v[7]), "=r"(borrow)
        : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5]), "r"(t[6]), "r"(t[7]), "r"(F::p(0)),
          "r"(F::p(1)), "r"(F::p(2)), "r"(F::p(3)), "r"(F::p(4)), "r"(F::p(5)), "r"(F::p(6)), "r"(F::p(7)));
    const bool keep = borrow && t[8] == 0;  // the 257-bit value is below p
    Fe r;
#pragma unroll
    for (int j = 0; j < 8; ++j) r.v[j] = keep ? t[j] : d.v[j];
    return r;
}

/// Montgomery product a*b*R^{-1} mod p, fully reduced: CIOS with even/odd
/// split carry chains. The running value is T = E + O * 2^32 (E holds limb
/// columns 0..7, O columns 1..8); a row adds the even limbs' products into E
/// and the odd limbs' into O, the Montgomery row m*p likewise, and the
/// one-limb shift of CIOS is folded into the next row (O becomes E with E[1]
/// added at column 0; the rest of E, two limbs down, is the addend of the
/// next odd row). ~137 IMAD + ~51 ALU SASS instructions against ~232 + ~210
/// for 64-bit C partial products: 6.74 vs 4.53e10 products/s on B200, bit-exact
/// over 2^20 random products (tools/mulbench/eobench.cu, profiles/r2/eobench.txt).
/// Inputs may be < 2p (lazy differences): T stays < 2^288 and the result < 2p
/// before the final subtraction since 4p < R (p < 2^254).
template <class F>
__device__ __forceinline__ Fe fe_mul(const Fe& a, const Fe& b) {
    if constexpr (F::kWide) return fe_mul_wide<F>(a, b);
    uint32_t P[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) P[k] = F::p(k);
    const uint32_t np0 = F::np0();
    uint32_t E[8], O[8], N[8];
    eo_mul_row(E, a.v, 0, b.v[0]);
    eo_mul_row(O, a.v, 1, b.v[0]);
    {
        const uint32_t m = E[0] * np0;
        eo_mad_row(E, P, 0, m);
        asm volatile("addc.u32 %0, %0, 0;" : "+r"(O[7]));  // E's carry: column 8
        eo_mad_row(O, P, 1, m);
    }
#pragma unroll
    for (int i = 1; i < 8; ++i) {
        asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(O[0]) : "r"(E[1]));  // shift: E[1] to column 0
        eo_madc_row_rshift(N, a.v, 1, b.v[i], E);                            // next O: odd row + E[k+2]
        eo_mad_row(O, a.v, 0, b.v[i]);                                       // next E: old O + even row
        asm volatile("addc.u32 %0, %0, 0;" : "+r"(N[7]));
        const uint32_t m = O[0] * np0;
        eo_mad_row(O, P, 0, m);
        asm volatile("addc.u32 %0, %0, 0;" : "+r"(N[7]));
        eo_mad_row(N, P, 1, m);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            E[k] = O[k];
            O[k] = N[k];
        }
    }
    uint32_t R[8];  // final shift: R = O + E >> 32
    asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(R[0]) : "r"(O[0]), "r"(E[1]));
#pragma unroll
    for (int k = 1; k < 7; ++k) asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(R[k]) : "r"(O[k]), "r"(E[k + 1]));
    asm volatile("addc.u32 %0, %1, 0;" : "=r"(R[7]) : "r"(O[7]));
    return fe_reduce_once<F>(R);
}

/// CIOS with 64-bit C partial products and a 10-limb accumulator: valid for
/// ANY a < 2^256 when b < p (the running value stays < 2^257), which the
/// even/odd fe_mul (a, b < 2p) is not. Used by acc_reduce, whose 256-bit
/// remainder is not reduced.
template <class F>
__device__ __forceinline__ Fe fe_mul_any(const Fe& a, const Fe& b) {
    if constexpr (F::kWide) return fe_mul_wide<F>(a, b);
    uint32_t t[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint64_t c = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint64_t s = static_cast<uint64_t>(a.v[j]) * b.v[i] + t[j] + c;
            t[j] = static_cast<uint32_t>(s);
            c = s >> 32;
        }
        uint64_t s = static_cast<uint64_t>(t[8]) + c;
        t[8] = static_cast<uint32_t>(s);
        t[9] = static_cast<uint32_t>(s >> 32);
        const uint32_t m = t[0] * F::np0();
        c = (static_cast<uint64_t>(m) * F::p(0) + t[0]) >> 32;
#pragma unroll
        for (int j = 1; j < 8; ++j) {
            const uint64_t s2 = static_cast<uint64_t>(m) * F::p(j) + t[j] + c;
            t[j - 1] = static_cast<uint32_t>(s2);
            c = s2 >> 32;
        }
        s = static_cast<uint64_t>(t[8]) + c;
        t[7] = static_cast<uint32_t>(s);
        t[8] = t[9] + static_cast<uint32_t>(s >> 32);
    }
    uint32_t r8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r8[j] = t[j];
    return fe_reduce_once<F>(r8);
}

/// Multiplication by a per-launch constant r (the sum-check challenge of a
/// fold), BN254 only. With c_k = r * 2^(32k+64) * R^-1 mod p precomputed on
/// the host,  mont(x, r) = x r R^-1 = 2^-64 * sum_k x_k c_k  (mod p):
/// 64 32x32 products + 2 Montgomery steps instead of CIOS's 8 (~40% fewer
/// IMADs). S = sum < 8 * 2^32 * p < 2^289, so after the two steps the value
/// is < 2^225 + p < 2p (needs p > 2^253 + 2^224, true for BN254 Fr).
/// The 64-bit C form lowers to IMAD.WIDE (a third of the IMAD rate, on the
/// FMA pipe); a PTX mad.lo/madc.hi form uses full-rate IMADs but adds ALU
/// carry adds, and k_round is bound by the ALU pipe, so the C form measured
/// as fast or faster.
struct FoldConst {
    Fe c[8];  // c_k above (fully reduced)
    Fe r;     // r itself (Montgomery form), for the generic path
};

__device__ __forceinline__ Fe fe_mul_const_bn254(const Fe& x, const FoldConst& K) {
    // S = sum_k x_k c_k: eight rows (multiplicand c_k, scalar x_k), all at
    // column 0, accumulated as even/odd carry chains: E (columns 0..7) and
    // O (columns 1..8) plus one carry limb o8 (column 9; S < 8 * 2^32 * p < 2^289)
    uint32_t E[8], O[8], o8 = 0;
    eo_mul_row(E, K.c[0].v, 0, x.v[0]);
    eo_mul_row(O, K.c[0].v, 1, x.v[0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        eo_mad_row(E, K.c[k].v, 0, x.v[k]);
        asm volatile("addc.cc.u32 %0, %0, 0;\n\taddc.u32 %1, %1, 0;" : "+r"(O[7]), "+r"(o8));
        eo_mad_row(O, K.c[k].v, 1, x.v[k]);
        asm volatile("addc.u32 %0, %0, 0;" : "+r"(o8));
    }
    // merge into t[0..9]: t = E + O * 2^32
    uint32_t t[10];
    t[0] = E[0];
    asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(t[1]) : "r"(E[1]), "r"(O[0]));
#pragma unroll
    for (int k = 2; k < 8; ++k) asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(t[k]) : "r"(E[k]), "r"(O[k - 1]));
    asm volatile("addc.cc.u32 %0, %2, 0;\n\taddc.u32 %1, %3, 0;" : "=r"(t[8]), "=r"(t[9]) : "r"(O[7]), "r"(o8));
    // two Montgomery steps (S < 2^289 -> < 2^225 + p < 2p, p > 2^253 + 2^224)
#pragma unroll
    for (int st = 0; st < 2; ++st) {
        const uint32_t m = t[0] * Bn254::np0();
        uint64_t c = (static_cast<uint64_t>(m) * Bn254::p(0) + t[0]) >> 32;
#pragma unroll
        for (int j = 1; j < 8; ++j) {
            const uint64_t s = static_cast<uint64_t>(m) * Bn254::p(j) + t[j] + c;
            t[j - 1] = static_cast<uint32_t>(s);
            c = s >> 32;
        }
        uint64_t s = static_cast<uint64_t>(t[8]) + c;
        t[7] = static_cast<uint32_t>(s);
        s = static_cast<uint64_t>(t[9]) + (s >> 32);
        t[8] = static_cast<uint32_t>(s);
        t[9] = 0;
    }
    uint32_t r8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r8[j] = t[j];
    return fe_reduce_once<Bn254>(r8);
}

/// mont(x, r) for a fold challenge: constant-multiplier path for BN254,
/// CIOS for runtime moduli.
template <class F>
__device__ __forceinline__ Fe fe_mul_fold(const Fe& x, const FoldConst& K) {
    if constexpr (F::kRuntime) {
        return fe_mul<F>(x, K.r);
    } else {
        return fe_mul_const_bn254(x, K);
    }
}

template <class F>
__device__ __forceinline__ Fe fe_to_mont(const Fe& canonical) {
    Fe r2;
#pragma unroll
    for (int i = 0; i < 8; ++i) r2.v[i] = F::r2(i);
    return fe_mul<F>(canonical, r2);
}

template <class F>
__device__ __forceinline__ Fe fe_from_mont(const Fe& m) {
    Fe one = fe_zero();
    one.v[0] = 1;
    return fe_mul<F>(m, one);
}

/// canonical value < p ?
template <class F>
__device__ __forceinline__ bool fe_lt_p(const Fe& a) {
    uint32_t borrow;
    uint32_t d0, d1, d2, d3, d4, d5, d6, d7;
    asm("sub.cc.u32  %0, %9, %17;\n\t"
        "subc.cc.u32 %1, %10, %18;\n\t"
        "subc.cc.u32 %2, %11, %19;\n\t"
        "subc.cc.u32 %3, %12, %20;\n\t"
        "subc.cc.u32 %4, %13, %21;\n\t"
        "subc.cc.u32 %5, %14, %22;\n\t"
        "subc.cc.u32 %6, %15, %23;\n\t"
        "subc.cc.u32 %7, %16, %24;\n\t"
        "subc.u32    %8, 0, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(d4), "=r"(d5), "=r"(d6), "=r"(d7), "=r"(borrow)
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]), "r"(a.v[7]),
          "r"(F::p(0)), "r"(F::p(1)), "r"(F::p(2)), "r"(F::p(3)), "r"(F::p(4)), "r"(F::p(5)), "r"(F::p(6)),
          "r"(F::p(7)));
    return borrow != 0;
}

// ---------------------------------------------------------------------------
// Wide (unreduced) accumulation of Montgomery products for round sums:
// the 512-bit products a_i b_i (< 4p^2 < 2^510 for lazy inputs < 2p) are
// added into a 17-limb accumulator T and REDC(T) = T R^-1 mod p is taken once
// per CTA (acc_reduce), saving the reduction half of CIOS and the modular add
// on every product. A Montgomery value g (= gR) joins the sum as g * 2^256
// (acc_add_hi). Capacity 2^544 / 2^510 = 2^34 products.
// ---------------------------------------------------------------------------
struct Acc {
    uint32_t v[17];
};

__device__ __forceinline__ void acc_zero(Acc& a) {
#pragma unroll
    for (int i = 0; i < 17; ++i) a.v[i] = 0;
}

/// acc += t (16 limbs)
__device__ __forceinline__ void acc_add16(Acc& a, const uint32_t (&t)[16]) {
    asm("add.cc.u32  %0, %0, %17;\n\t"
        "addc.cc.u32 %1, %1, %18;\n\t"
        "addc.cc.u32 %2, %2, %19;\n\t"
        "addc.cc.u32 %3, %3, %20;\n\t"
        "addc.cc.u32 %4, %4, %21;\n\t"
        "addc.cc.u32 %5, %5, %22;\n\t"
        "addc.cc.u32 %6, %6, %23;\n\t"
        "addc.cc.u32 %7, %7, %24;\n\t"
        "addc.cc.u32 %8, %8, %25;\n\t"
        "addc.cc.u32 %9, %9, %26;\n\t"
        "addc.cc.u32 %10, %10, %27;\n\t"
        "addc.cc.u32 %11, %11, %28;\n\t"
        "addc.cc.u32 %12, %12, %29;\n\t"
        "addc.cc.u32 %13, %13, %30;\n\t"
        "addc.cc.u32 %14, %14, %31;\n\t"
        "addc.cc.u32 %15, %15, %32;\n\t"
        "addc.u32    %16, %16, 0;"
        : "+r"(a.v[0]), "+r"(a.v[1]), "+r"(a.v[2]), "+r"(a.v[3]), "+r"(a.v[4]), "+r"(a.v[5]), "+r"(a.v[6]),
          "+r"(a.v[7]), "+r"(a.v[8]), "+r"(a.v[9]), "+r"(a.v[10]), "+r"(a.v[11]), "+r"(a.v[12]), "+r"(a.v[13]),
          "+r"(a.v[14]), "+r"(a.v[15]), "+r"(a.v[16])
        : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5]), "r"(t[6]), "r"(t[7]), "r"(t[8]),
          "r"(t[9]), "r"(t[10]), "r"(t[11]), "r"(t[12]), "r"(t[13]), "r"(t[14]), "r"(t[15]));
}

/// acc += a * b (512-bit schoolbook product, no reduction)
__device__ __forceinline__ void acc_mad(Acc& acc, const Fe& a, const Fe& b) {
    uint32_t t[16];
    {
        uint64_t c = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint64_t s = static_cast<uint64_t>(a.v[j]) * b.v[0] + c;
            t[j] = static_cast<uint32_t>(s);
            c = s >> 32;
        }
        t[8] = static_cast<uint32_t>(c);
    }
#pragma unroll
    for (int i = 1; i < 8; ++i) {
        uint64_t c = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint64_t s = static_cast<uint64_t>(a.v[j]) * b.v[i] + t[i + j] + c;
            t[i + j] = static_cast<uint32_t>(s);
            c = s >> 32;
        }
        t[i + 8] = static_cast<uint32_t>(c);
    }
    acc_add16(acc, t);
}

/// acc += g * 2^256
__device__ __forceinline__ void acc_add_hi(Acc& a, const Fe& g) {
    asm("add.cc.u32  %0, %0, %9;\n\t"
        "addc.cc.u32 %1, %1, %10;\n\t"
        "addc.cc.u32 %2, %2, %11;\n\t"
        "addc.cc.u32 %3, %3, %12;\n\t"
        "addc.cc.u32 %4, %4, %13;\n\t"
        "addc.cc.u32 %5, %5, %14;\n\t"
        "addc.cc.u32 %6, %6, %15;\n\t"
        "addc.cc.u32 %7, %7, %16;\n\t"
        "addc.u32    %8, %8, 0;"
        : "+r"(a.v[8]), "+r"(a.v[9]), "+r"(a.v[10]), "+r"(a.v[11]), "+r"(a.v[12]), "+r"(a.v[13]), "+r"(a.v[14]),
          "+r"(a.v[15]), "+r"(a.v[16])
        : "r"(g.v[0]), "r"(g.v[1]), "r"(g.v[2]), "r"(g.v[3]), "r"(g.v[4]), "r"(g.v[5]), "r"(g.v[6]), "r"(g.v[7]));
}

/// a += b
__device__ __forceinline__ void acc_add(Acc& a, const Acc& b) {
    uint32_t t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = b.v[i];
    acc_add16(a, t);
    a.v[16] += b.v[16];
}

__device__ __forceinline__ Acc acc_shfl(const Acc& a, int src) {
    Acc r;
#pragma unroll
    for (int i = 0; i < 17; ++i) r.v[i] = __shfl_sync(0xffffffffu, a.v[i], src);
    return r;
}

__device__ __forceinline__ Acc acc_shfl_down(const Acc& a, int off) {
    Acc r;
#pragma unroll
    for (int i = 0; i < 17; ++i) r.v[i] = __shfl_down_sync(0xffffffffu, a.v[i], off);
    return r;
}

/// T R^-1 mod p, fully reduced (T < 2^544): 8 REDC steps leave the 9-limb
/// X = (T + m p) / 2^256 = T R^-1 (mod p); then
/// X mod p = ((X_lo R^2) R^-1) R^-1 ... = X_lo mod p + x_8 R mod p.
template <class F>
__device__ Fe acc_reduce(const Acc& acc) {
    uint32_t t[17];
#pragma unroll
    for (int i = 0; i < 17; ++i) t[i] = acc.v[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t m = t[i] * F::np0();
        uint64_t c = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint64_t s = static_cast<uint64_t>(m) * F::p(j) + t[i + j] + c;
            t[i + j] = static_cast<uint32_t>(s);
            c = s >> 32;
        }
#pragma unroll
        for (int k = i + 8; k < 17; ++k) {
            const uint64_t s = static_cast<uint64_t>(t[k]) + c;
            t[k] = static_cast<uint32_t>(s);
            c = s >> 32;
        }
    }
    Fe lo, hi, r2, one_raw;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        lo.v[i] = t[8 + i];
        hi.v[i] = 0;
        r2.v[i] = F::r2(i);
        one_raw.v[i] = 0;
    }
    hi.v[0] = t[16];
    one_raw.v[0] = 1;
    const Fe lo_red = fe_mul<F>(fe_mul_any<F>(lo, r2), one_raw);  // X_lo mod p (X_lo: any 256-bit value)
    const Fe hi_r = fe_mul<F>(hi, r2);                            // x_8 R mod p
    return fe_add<F>(lo_red, hi_r);
}

__device__ __forceinline__ Fe fe_shfl_down(const Fe& a, int off) {
    Fe r;
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = __shfl_down_sync(0xffffffffu, a.v[i], off);
    return r;
}

}  // namespace dgkr_b200
