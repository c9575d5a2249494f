// Microbenchmark: BN254 Montgomery product with even/odd split carry chains
// (the product a*b_i and m*p rows accumulate into two arrays -- even-indexed
// limb products in E, odd-indexed in O, one limb apart -- so every row is a
// single PTX mad/madc carry chain; the limb shift of CIOS is folded into the
// next row's madc addends). Checked bit-exact against fe_mul<Bn254> on random
// inputs, then timed like dgkr_bench_mul_peak (4 independent chains/thread).
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_2404_10404_b200/csrc
//        -o eobench eobench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "field.cuh"

using namespace dgkr_b200;

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
            std::exit(1);                                                                      \
        }                                                                                      \
    } while (0)

// ---- row primitives (n = 8 limbs; a row uses limbs a[off], a[off+2], ...) ----
// acc[0..7] (+)= sum_{j} x[off + 2j] * y placed lo/hi at acc[2j], acc[2j+1]
__device__ __forceinline__ void mul_row(uint32_t acc[8], const uint32_t* x, int off, uint32_t y) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
        asm volatile("mul.lo.u32 %0, %2, %3;\n\tmul.hi.u32 %1, %2, %3;"
            : "=r"(acc[2 * j]), "=r"(acc[2 * j + 1])
            : "r"(x[off + 2 * j]), "r"(y));
}
// acc += row, carry out of acc[7] left in CC
__device__ __forceinline__ void mad_row(uint32_t acc[8], const uint32_t* x, int off, uint32_t y) {
    asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;"
        : "+r"(acc[0]), "+r"(acc[1])
        : "r"(x[off]), "r"(y));
#pragma unroll
    for (int j = 1; j < 4; ++j)
        asm volatile("madc.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;"
            : "+r"(acc[2 * j]), "+r"(acc[2 * j + 1])
            : "r"(x[off + 2 * j]), "r"(y));
}
// dst[k] = row + src[k + 2] (src[8], src[9] = 0) + CC-in at dst[0]; carry out dropped (bounded)
__device__ __forceinline__ void madc_row_rshift(uint32_t dst[8], const uint32_t* x, int off, uint32_t y,
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

/// Montgomery product a*b*2^-256 mod p, fully reduced (inputs < 2p as fe_mul).
/// Invariant: T = E + O * 2^32 (E: limb columns 0..7, O: columns 1..8).
__device__ __forceinline__ Fe fe_mul_eo(const Fe& a, const Fe& b) {
    uint32_t P[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) P[k] = Bn254::p(k);
    const uint32_t np0 = Bn254::np0();
    uint32_t E[8], O[8], E2[8];
    // row 0
    mul_row(E, a.v, 0, b.v[0]);
    mul_row(O, a.v, 1, b.v[0]);
    {
        const uint32_t m = E[0] * np0;
        mad_row(E, P, 0, m);
        asm volatile("addc.u32 %0, %0, 0;" : "+r"(O[7]));  // E's carry: column 8
        mad_row(O, P, 1, m);                      // carry out of column 9: 0 (T < 2^288)
    }
#pragma unroll
    for (int i = 1; i < 8; ++i) {
        // shift by one limb: T' = O + E >> 32 (E[0] = 0): new E = O with E[1]
        // added at column 0, new O[k] = E[k + 2]; the add's carry (column 1)
        // enters the new O row's first madc
        asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(O[0]) : "r"(E[1]));
        madc_row_rshift(E2, a.v, 1, b.v[i], E);  // new O (odd products) + E[k+2]
        // new E = old O (+ even products of row i)
        mad_row(O, a.v, 0, b.v[i]);
        asm volatile("addc.u32 %0, %0, 0;" : "+r"(E2[7]));
        const uint32_t m = O[0] * np0;
        mad_row(O, P, 0, m);
        asm volatile("addc.u32 %0, %0, 0;" : "+r"(E2[7]));
        mad_row(E2, P, 1, m);
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // roles: E <- O (even-aligned), O <- E2 (odd-aligned)
            E[k] = O[k];
            O[k] = E2[k];
        }
    }
    // final shift: R = O + E >> 32
    uint32_t R[8];
    asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(R[0]) : "r"(O[0]), "r"(E[1]));
#pragma unroll
    for (int k = 1; k < 7; ++k) asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(R[k]) : "r"(O[k]), "r"(E[k + 1]));
    asm volatile("addc.u32 %0, %1, 0;" : "=r"(R[7]) : "r"(O[7]));
    // R < 2p: one conditional subtraction
    Fe d;
    uint32_t borrow;
    asm volatile("sub.cc.u32  %0, %9, %17;\n\t"
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
        : "r"(R[0]), "r"(R[1]), "r"(R[2]), "r"(R[3]), "r"(R[4]), "r"(R[5]), "r"(R[6]), "r"(R[7]), "r"(P[0]),
          "r"(P[1]), "r"(P[2]), "r"(P[3]), "r"(P[4]), "r"(P[5]), "r"(P[6]), "r"(P[7]));
    Fe r;
#pragma unroll
    for (int j = 0; j < 8; ++j) r.v[j] = borrow ? R[j] : d.v[j];
    return r;
}

__global__ void k_check(const Fe* a, const Fe* b, int n, unsigned* bad, Fe* first) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const Fe x = fe_mul<Bn254>(a[i], b[i]), y = fe_mul_eo(a[i], b[i]);
        bool eq = true;
        for (int k = 0; k < 8; ++k) eq &= x.v[k] == y.v[k];
        if (!eq && atomicAdd(bad, 1u) == 0) {
            first[0] = a[i];
            first[1] = b[i];
            first[2] = x;
            first[3] = y;
        }
    }
}

// the previous constant multiplier (64-bit C partial products), the reference for field.cuh's
__device__ __forceinline__ Fe const_old(const Fe& x, const FoldConst& K) {
    uint32_t t[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        uint64_t c = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint64_t s = static_cast<uint64_t>(x.v[k]) * K.c[k].v[j] + t[j] + c;
            t[j] = static_cast<uint32_t>(s);
            c = s >> 32;
        }
        const uint64_t s = static_cast<uint64_t>(t[8]) + c;
        t[8] = static_cast<uint32_t>(s);
        t[9] += static_cast<uint32_t>(s >> 32);
    }
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
    for (int j = 0; j < 8; ++j) r8[j] = t[j];
    return fe_reduce_once<Bn254>(r8);
}

__constant__ uint32_t c_pow[8][8];  // canonical 2^(32k+64) mod p

/// field.cuh fe_mul on lazy inputs in [0, 2p) vs fe_mul_any; field.cuh's
/// constant multiplier vs const_old on any 256-bit x (challenge r = b[i])
__global__ void k_check2(const Fe* a, const Fe* b, int n, unsigned* bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        // lazy operands: a + p, b + p when they stay below 2p
        Fe la = a[i], lb = b[i];
        if (i & 1) la = fe_sub_lazy<Bn254>(a[i], fe_zero());  // a + p
        if (i & 2) lb = fe_sub_lazy<Bn254>(b[i], fe_zero());
        const Fe x = fe_mul<Bn254>(la, lb), y = fe_mul_any<Bn254>(la, lb);
        bool eq = true;
        for (int k = 0; k < 8; ++k) eq &= x.v[k] == y.v[k];
        FoldConst K;
        for (int k = 0; k < 8; ++k) {
            Fe pw;
            for (int j = 0; j < 8; ++j) pw.v[j] = c_pow[k][j];
            K.c[k] = fe_mul_any<Bn254>(b[i], pw);
        }
        K.r = b[i];
        Fe xr = a[i];
        xr.v[7] ^= (i & 4) ? 0xc0000000u : 0u;  // any 256-bit input
        const Fe u = fe_mul_const_bn254(xr, K), v = const_old(xr, K);
        for (int k = 0; k < 8; ++k) eq &= u.v[k] == v.v[k];
        if (!eq) atomicAdd(bad, 1u);
    }
}

template <int V>
__global__ void __launch_bounds__(256) k_peak(int iters, Fe* sink, unsigned never) {
    Fe a[4], b;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[k].v[i] = (threadIdx.x * 0x9e3779b9u + k * 0x85ebca6bu + i) & 0x0fffffffu;
#pragma unroll
    for (int i = 0; i < 8; ++i) b.v[i] = (blockIdx.x * 0x27d4eb2fu + i) & 0x0fffffffu;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) a[k] = V == 0 ? fe_mul<Bn254>(a[k], b) : fe_mul_eo(a[k], b);
    }
    Fe s = fe_add<Bn254>(fe_add<Bn254>(a[0], a[1]), fe_add<Bn254>(a[2], a[3]));
    if (s.v[0] == never) fe_store(sink, s);
}

int main() {
    const int n = 1 << 20;
    std::mt19937_64 rng(12345);
    // random values < p (top limb below p's), including edge values
    const uint32_t P7 = 0x30644e72u;
    std::vector<Fe> ha(n), hb(n);
    for (int i = 0; i < n; ++i) {
        for (int k = 0; k < 8; ++k) {
            ha[i].v[k] = static_cast<uint32_t>(rng());
            hb[i].v[k] = static_cast<uint32_t>(rng());
        }
        ha[i].v[7] %= P7;
        hb[i].v[7] %= P7;
        if (i < 16) {  // extremes: 0, 1, all-ones low limbs
            for (int k = 0; k < 8; ++k) ha[i].v[k] = (i & 1) ? 0xffffffffu : 0u;
            ha[i].v[7] = (i & 2) ? P7 - 1 : 0;
        }
    }
    Fe *da, *db, *dfirst;
    unsigned* dbad;
    CK(cudaMalloc(&da, n * sizeof(Fe)));
    CK(cudaMalloc(&db, n * sizeof(Fe)));
    CK(cudaMalloc(&dfirst, 4 * sizeof(Fe)));
    CK(cudaMalloc(&dbad, sizeof(unsigned)));
    CK(cudaMemset(dbad, 0, sizeof(unsigned)));
    CK(cudaMemcpy(da, ha.data(), n * sizeof(Fe), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, hb.data(), n * sizeof(Fe), cudaMemcpyHostToDevice));
    k_check<<<1184, 256>>>(da, db, n, dbad, dfirst);
    unsigned bad = 0;
    CK(cudaMemcpy(&bad, dbad, sizeof(unsigned), cudaMemcpyDeviceToHost));
    std::printf("{\"check\": \"fe_mul_eo vs fe_mul on %d random products\", \"mismatches\": %u}\n", n, bad);
    {
        const uint32_t pw[8][8] = {
            {0x00000000u, 0x00000000u, 0x00000001u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u},
            {0x00000000u, 0x00000000u, 0x00000000u, 0x00000001u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u},
            {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000001u, 0x00000000u, 0x00000000u, 0x00000000u},
            {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000001u, 0x00000000u, 0x00000000u},
            {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000001u, 0x00000000u},
            {0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000000u, 0x00000001u},
            {0x4ffffffbu, 0xac96341cu, 0x9f60cd29u, 0x36fc7695u, 0x7879462eu, 0x666ea36fu, 0x9a07df2fu, 0x0e0a77c1u},
            {0x15b8b9dau, 0x93e78865u, 0xb05ea154u, 0x16df2426u, 0x302ab839u, 0x1271b743u, 0xec6c226eu, 0x06bc037eu}};
        CK(cudaMemcpyToSymbol(c_pow, pw, sizeof(pw)));
        CK(cudaMemset(dbad, 0, sizeof(unsigned)));
        k_check2<<<1184, 256>>>(da, db, n, dbad);
        unsigned bad2 = 0;
        CK(cudaMemcpy(&bad2, dbad, sizeof(unsigned), cudaMemcpyDeviceToHost));
        std::printf("{\"check\": \"field.cuh fe_mul on lazy [0,2p) operands vs 10-limb CIOS, and the constant "
                    "multiplier vs the previous one on 256-bit inputs, %d cases\", \"mismatches\": %u}\n", n, bad2);
        bad += bad2;
    }
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int iters = 4096, blocks = sms * 8;
    for (int v = 0; v < 2; ++v) {
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaEventRecord(e0));
            if (v == 0) k_peak<0><<<blocks, 256>>>(iters, da, 0xffffffffu);
            else k_peak<1><<<blocks, 256>>>(iters, da, 0xffffffffu);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
        }
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double muls = 4.0 * iters * blocks * 256.0;
        std::printf("{\"probe\": \"%s\", \"mul_per_s\": %.4e}\n", v ? "fe_mul_eo (even/odd madc chains)" : "fe_mul (CIOS, 64-bit C products)",
                    muls / (ms * 1e-3));
    }
    return bad ? 1 : 0;
}
