// Microbenchmark: BN254 Montgomery multiplication variants on sm_100a.
//   imad      : 32-bit mad.lo.u32 throughput (independent chains)
//   imadwide  : mad.wide.u32 (32x32+64 -> 64) throughput
//   cios      : fe_mul<Bn254> (8 x 32-bit CIOS with PTX carry chains)
//   r26       : radix-2^26 product scanning with 64-bit column accumulators
//               (one mad.wide per partial product, no carry chains),
//               Montgomery reduction by 2^256 = 9 x 26-bit + 1 x 22-bit steps
// r26 is checked against cios on random inputs before timing.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_2404_10404_b200/csrc
//        -o r26bench r26bench.cu
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "field.cuh"

using namespace dgkr_b200;

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(1);                                                           \
        }                                                                           \
    } while (0)

// BN254 Fr in 26-bit digits (digit 9 holds bits 234..253)
struct P26 {
    static constexpr uint32_t kMask = (1u << 26) - 1;
};
__constant__ uint32_t c_p26[10];
__constant__ uint32_t c_np26;  // -p^-1 mod 2^26
__constant__ uint32_t c_np22;  // -p^-1 mod 2^22

__device__ __forceinline__ uint64_t madw(uint32_t a, uint32_t b, uint64_t c) {
    uint64_t d;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}

__device__ __forceinline__ void to26(const Fe& x, uint32_t d[10]) {
    // bits [26i, 26i+26)
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const int lo = 26 * i, w = lo >> 5, s = lo & 31;
        uint32_t v = x.v[w] >> s;
        if (s > 6 && w + 1 < 8) v |= x.v[w + 1] << (32 - s);
        d[i] = v & P26::kMask;
    }
}

__device__ __forceinline__ Fe mul_r26(const Fe& a, const Fe& b) {
    uint32_t x[10], y[10];
    to26(a, x);
    to26(b, y);
    uint64_t c[20];
#pragma unroll
    for (int k = 0; k < 20; ++k) c[k] = 0;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
#pragma unroll
        for (int j = 0; j < 10; ++j) c[i + j] = madw(x[i], y[j], c[i + j]);
    }
    // 9 reduction steps of 26 bits
#pragma unroll
    for (int s = 0; s < 9; ++s) {
        const uint32_t m = (static_cast<uint32_t>(c[s]) * c_np26) & P26::kMask;
#pragma unroll
        for (int j = 0; j < 10; ++j) c[s + j] = madw(m, c_p26[j], c[s + j]);
        c[s + 1] += c[s] >> 26;
    }
    // last step: 22 bits
    {
        const uint32_t m = (static_cast<uint32_t>(c[9]) * c_np22) & ((1u << 22) - 1);
#pragma unroll
        for (int j = 0; j < 10; ++j) c[9 + j] = madw(m, c_p26[j], c[9 + j]);
    }
    // value = sum_{k>=9} c_k 2^(26(k-9)) >> 22; normalise the 26-bit digits
    uint32_t d[11];
    uint64_t carry = 0;
#pragma unroll
    for (int j = 0; j < 10; ++j) {
        const uint64_t v = c[9 + j] + carry;
        d[j] = static_cast<uint32_t>(v) & P26::kMask;
        carry = v >> 26;
    }
    d[10] = static_cast<uint32_t>(carry);
    // pack bits [22, 22+256) of the digit string into 8 x 32-bit limbs
    Fe t;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int lo = 22 + 32 * i;  // bit position in the digit string
        const int k = lo / 26, s = lo % 26;
        uint64_t v = (static_cast<uint64_t>(d[k]) >> s) | (static_cast<uint64_t>(d[k + 1]) << (26 - s));
        if (k + 2 <= 10) v |= static_cast<uint64_t>(d[k + 2]) << (52 - s);
        t.v[i] = static_cast<uint32_t>(v);
    }
    // conditional subtraction (t < 2p)
    Fe s_;
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
        : "=r"(s_.v[0]), "=r"(s_.v[1]), "=r"(s_.v[2]), "=r"(s_.v[3]), "=r"(s_.v[4]), "=r"(s_.v[5]), "=r"(s_.v[6]),
          "=r"(s_.v[7]), "=r"(borrow)
        : "r"(t.v[0]), "r"(t.v[1]), "r"(t.v[2]), "r"(t.v[3]), "r"(t.v[4]), "r"(t.v[5]), "r"(t.v[6]), "r"(t.v[7]),
          "r"(Bn254::p(0)), "r"(Bn254::p(1)), "r"(Bn254::p(2)), "r"(Bn254::p(3)), "r"(Bn254::p(4)),
          "r"(Bn254::p(5)), "r"(Bn254::p(6)), "r"(Bn254::p(7)));
    Fe r;
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = borrow ? t.v[i] : s_.v[i];
    return r;
}

constexpr int kThreads = 256;

// CIOS with 64-bit C partial products (IMAD.WIDE)
__device__ __forceinline__ Fe mul_wide(const Fe& a, const Fe& b) {
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
        const uint32_t m = t[0] * Bn254::np0();
        c = (static_cast<uint64_t>(m) * Bn254::p(0) + t[0]) >> 32;
#pragma unroll
        for (int j = 1; j < 8; ++j) {
            const uint64_t s2 = static_cast<uint64_t>(m) * Bn254::p(j) + t[j] + c;
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
        : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(t[5]), "r"(t[6]), "r"(t[7]), "r"(Bn254::p(0)),
          "r"(Bn254::p(1)), "r"(Bn254::p(2)), "r"(Bn254::p(3)), "r"(Bn254::p(4)), "r"(Bn254::p(5)), "r"(Bn254::p(6)),
          "r"(Bn254::p(7)));
    Fe r;
#pragma unroll
    for (int j = 0; j < 8; ++j) r.v[j] = borrow ? t[j] : d.v[j];
    return r;
}

// constant-multiplier throughput: K in kernel-parameter space (as k_round) or
// staged in shared memory (a per-block multiplier)
__global__ void __launch_bounds__(kThreads) k_const_param(int iters, Fe* sink, unsigned never,
                                                          const __grid_constant__ FoldConst K) {
    Fe a[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[k].v[i] = (threadIdx.x * 0x9e3779b9u + k * 0x85ebca6bu + i) & 0x0fffffffu;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) a[k] = fe_mul_const_bn254(a[k], K);
    }
    Fe s = fe_add<Bn254>(fe_add<Bn254>(a[0], a[1]), fe_add<Bn254>(a[2], a[3]));
    if (s.v[0] == never) fe_store(sink, s);
}

__global__ void __launch_bounds__(kThreads) k_const_smem(int iters, Fe* sink, unsigned never, const FoldConst* Kg) {
    __shared__ FoldConst K;
    if (threadIdx.x < sizeof(FoldConst) / 4)
        reinterpret_cast<uint32_t*>(&K)[threadIdx.x] = reinterpret_cast<const uint32_t*>(Kg)[threadIdx.x];
    __syncthreads();
    Fe a[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[k].v[i] = (threadIdx.x * 0x9e3779b9u + k * 0x85ebca6bu + i) & 0x0fffffffu;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) a[k] = fe_mul_const_bn254(a[k], K);
    }
    Fe s = fe_add<Bn254>(fe_add<Bn254>(a[0], a[1]), fe_add<Bn254>(a[2], a[3]));
    if (s.v[0] == never) fe_store(sink, s);
}

template <int V>
__global__ void __launch_bounds__(kThreads) k_bench(int iters, Fe* sink, unsigned never) {
    Fe a[4], b;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[k].v[i] = (threadIdx.x * 0x9e3779b9u + k * 0x85ebca6bu + i) & 0x0fffffffu;
#pragma unroll
    for (int i = 0; i < 8; ++i) b.v[i] = (blockIdx.x * 0x27d4eb2fu + i) & 0x0fffffffu;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) a[k] = V == 0 ? fe_mul<Bn254>(a[k], b) : V == 1 ? mul_r26(a[k], b) : mul_wide(a[k], b);
    }
    Fe s = fe_add<Bn254>(fe_add<Bn254>(a[0], a[1]), fe_add<Bn254>(a[2], a[3]));
    if (s.v[0] == never) fe_store(sink, s);
}

// raw pipe probes: 16 independent accumulators per thread, 256 ops per iteration
__global__ void __launch_bounds__(kThreads) k_imad(int iters, uint32_t* sink, unsigned never) {
    uint32_t acc[16];
    const uint32_t x = threadIdx.x | 1, y = blockIdx.x * 2654435761u;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = x + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int k = 0; k < 16; ++k) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(acc[k]) : "r"(y), "r"(x));
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s ^= acc[k];
    if (s == never) *sink = s;
}

__global__ void __launch_bounds__(kThreads) k_imadwide(int iters, uint64_t* sink, unsigned never) {
    uint64_t acc[16];
    const uint32_t x = threadIdx.x | 1, y = blockIdx.x * 2654435761u;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = x + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int k = 0; k < 16; ++k)
                asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[k]) : "r"(static_cast<uint32_t>(acc[(k + 1) & 15])), "r"(y));
    }
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s ^= acc[k];
    if (s == never) *sink = s;
}

__global__ void k_check(const Fe* a, const Fe* b, Fe* out0, Fe* out1, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out0[i] = fe_mul<Bn254>(a[i], b[i]);
    out1[i] = mul_r26(a[i], b[i]);
    const Fe w = mul_wide(a[i], b[i]);
    for (int j = 0; j < 8; ++j)
        if (w.v[j] != out0[i].v[j]) out1[i].v[0] ^= 0x80000000u;
}

static void set_consts() {
    // p in 26-bit digits and -p^-1 mod 2^26 / 2^22 (computed on the host)
    const uint32_t P[8] = {0xf0000001u, 0x43e1f593u, 0x79b97091u, 0x2833e848u,
                           0x8181585du, 0xb85045b6u, 0xe131a029u, 0x30644e72u};
    uint32_t d[10];
    for (int i = 0; i < 10; ++i) {
        uint64_t v = 0;
        for (int b = 0; b < 26; ++b) {
            const int bit = 26 * i + b;
            if (bit < 256 && (P[bit >> 5] >> (bit & 31) & 1)) v |= 1ull << b;
        }
        d[i] = static_cast<uint32_t>(v);
    }
    // inverse of p mod 2^32 by Newton, then negate
    uint32_t inv = 1;
    for (int k = 0; k < 6; ++k) inv *= 2 - P[0] * inv;
    const uint32_t np = 0u - inv;
    const uint32_t np26 = np & ((1u << 26) - 1), np22 = np & ((1u << 22) - 1);
    CK(cudaMemcpyToSymbol(c_p26, d, sizeof(d)));
    CK(cudaMemcpyToSymbol(c_np26, &np26, 4));
    CK(cudaMemcpyToSymbol(c_np22, &np22, 4));
}

int main() {
    set_consts();
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    // correctness: random canonical values < p (top limb masked below p's)
    const int n = 1 << 16;
    std::mt19937_64 rng(1);
    std::vector<Fe> ha(n), hb(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < 8; ++j) {
            ha[i].v[j] = static_cast<uint32_t>(rng());
            hb[i].v[j] = static_cast<uint32_t>(rng());
        }
    for (int i = 0; i < n; ++i) {
        ha[i].v[7] &= 0x2fffffffu;
        hb[i].v[7] &= 0x2fffffffu;
    }
    Fe *da, *db, *o0, *o1;
    CK(cudaMalloc(&da, n * sizeof(Fe)));
    CK(cudaMalloc(&db, n * sizeof(Fe)));
    CK(cudaMalloc(&o0, n * sizeof(Fe)));
    CK(cudaMalloc(&o1, n * sizeof(Fe)));
    CK(cudaMemcpy(da, ha.data(), n * sizeof(Fe), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, hb.data(), n * sizeof(Fe), cudaMemcpyHostToDevice));
    k_check<<<n / 256, 256>>>(da, db, o0, o1, n);
    CK(cudaDeviceSynchronize());
    std::vector<Fe> r0(n), r1(n);
    CK(cudaMemcpy(r0.data(), o0, n * sizeof(Fe), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r1.data(), o1, n * sizeof(Fe), cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < n; ++i) bad += std::memcmp(&r0[i], &r1[i], sizeof(Fe)) != 0;
    std::printf("{\"check\": \"r26 and cios_wide vs cios on %d random products\", \"mismatches\": %d}\n", n, bad);

    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    Fe* sink;
    CK(cudaMalloc(&sink, 64));
    const int blocks = sms * 8, iters = 2000;
    auto timeit = [&](auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        return ms;
    };
    const double thr = static_cast<double>(blocks) * kThreads;
    float ms = timeit([&] { k_imad<<<blocks, kThreads>>>(iters, reinterpret_cast<uint32_t*>(sink), 0xffffffffu); });
    std::printf("{\"probe\": \"imad\", \"ops_per_s\": %.4g, \"per_clk_per_sm_at_1965MHz\": %.2f}\n",
                thr * iters * 256 / (ms * 1e-3), thr * iters * 256 / (ms * 1e-3) / sms / 1.965e9);
    ms = timeit([&] { k_imadwide<<<blocks, kThreads>>>(iters, reinterpret_cast<uint64_t*>(sink), 0xffffffffu); });
    std::printf("{\"probe\": \"imad.wide\", \"ops_per_s\": %.4g, \"per_clk_per_sm_at_1965MHz\": %.2f}\n",
                thr * iters * 256 / (ms * 1e-3), thr * iters * 256 / (ms * 1e-3) / sms / 1.965e9);
    const int miters = 200;
    ms = timeit([&] { k_bench<0><<<blocks, kThreads>>>(miters, sink, 0xffffffffu); });
    std::printf("{\"probe\": \"cios\", \"mul_per_s\": %.4g}\n", thr * miters * 4 / (ms * 1e-3));
    ms = timeit([&] { k_bench<1><<<blocks, kThreads>>>(miters, sink, 0xffffffffu); });
    std::printf("{\"probe\": \"r26\", \"mul_per_s\": %.4g}\n", thr * miters * 4 / (ms * 1e-3));
    ms = timeit([&] { k_bench<2><<<blocks, kThreads>>>(miters, sink, 0xffffffffu); });
    std::printf("{\"probe\": \"cios_wide\", \"mul_per_s\": %.4g}\n", thr * miters * 4 / (ms * 1e-3));
    FoldConst hk;
    for (int k = 0; k < 8; ++k)
        for (int i = 0; i < 8; ++i) hk.c[k].v[i] = static_cast<uint32_t>(rng()) & (i == 7 ? 0x2fffffffu : ~0u);
    hk.r = hk.c[0];
    FoldConst* dk;
    CK(cudaMalloc(&dk, sizeof(FoldConst)));
    CK(cudaMemcpy(dk, &hk, sizeof(FoldConst), cudaMemcpyHostToDevice));
    ms = timeit([&] { k_const_param<<<blocks, kThreads>>>(miters, sink, 0xffffffffu, hk); });
    std::printf("{\"probe\": \"const_param\", \"mul_per_s\": %.4g}\n", thr * miters * 4 / (ms * 1e-3));
    ms = timeit([&] { k_const_smem<<<blocks, kThreads>>>(miters, sink, 0xffffffffu, dk); });
    std::printf("{\"probe\": \"const_smem\", \"mul_per_s\": %.4g}\n", thr * miters * 4 / (ms * 1e-3));
    return 0;
}
