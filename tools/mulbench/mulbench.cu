#include "field.cuh"
using namespace dgkr_b200;
// F1: plain C CIOS with 64-bit accumulation
__device__ __forceinline__ Fe mul_c64(const Fe& a, const Fe& b) {
    constexpr uint32_t P[8] = {0xf0000001u, 0x43e1f593u, 0x79b97091u, 0x2833e848u, 0x8181585du, 0xb85045b6u, 0xe131a029u, 0x30644e72u};
    uint32_t t[10] = {0};
    #pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint64_t c = 0;
        #pragma unroll
        for (int j = 0; j < 8; ++j) { uint64_t s = (uint64_t)a.v[j] * b.v[i] + t[j] + c; t[j] = (uint32_t)s; c = s >> 32; }
        uint64_t s = (uint64_t)t[8] + c; t[8] = (uint32_t)s; t[9] = (uint32_t)(s >> 32);
        uint32_t m = t[0] * 0xefffffffu;
        c = ((uint64_t)m * P[0] + t[0]) >> 32;
        #pragma unroll
        for (int j = 1; j < 8; ++j) { uint64_t s2 = (uint64_t)m * P[j] + t[j] + c; t[j-1] = (uint32_t)s2; c = s2 >> 32; }
        s = (uint64_t)t[8] + c; t[7] = (uint32_t)s; t[8] = t[9] + (uint32_t)(s >> 32);
    }
    Fe r; 
    // final subtract
    uint32_t d[8]; uint64_t br = 0;
    #pragma unroll
    for (int j = 0; j < 8; ++j) { uint64_t s = (uint64_t)t[j] - P[j] - br; d[j] = (uint32_t)s; br = (s >> 63); }
    #pragma unroll
    for (int j = 0; j < 8; ++j) r.v[j] = br ? t[j] : d[j];
    return r;
}
__global__ void k_ptx(int iters, Fe* sink, unsigned never) {
    Fe a[4], b; for (int k=0;k<4;++k) for (int i=0;i<8;++i) a[k].v[i]=(threadIdx.x*0x9e3779b9u+k*77+i)&0x0fffffff;
    for (int i=0;i<8;++i) b.v[i]=(blockIdx.x*0x27d4eb2fu+i)&0x0fffffff;
    for (int it=0; it<iters; ++it) { for (int k=0;k<4;++k) a[k]=fe_mul<Bn254>(a[k],b); }
    if (a[0].v[0]==never) { fe_store(sink,a[0]); fe_store(sink+1,a[1]); fe_store(sink+2,a[2]); fe_store(sink+3,a[3]); }
}
__global__ void k_c64(int iters, Fe* sink, unsigned never) {
    Fe a[4], b; for (int k=0;k<4;++k) for (int i=0;i<8;++i) a[k].v[i]=(threadIdx.x*0x9e3779b9u+k*77+i)&0x0fffffff;
    for (int i=0;i<8;++i) b.v[i]=(blockIdx.x*0x27d4eb2fu+i)&0x0fffffff;
    for (int it=0; it<iters; ++it) { for (int k=0;k<4;++k) a[k]=mul_c64(a[k],b); }
    if (a[0].v[0]==never) { fe_store(sink,a[0]); fe_store(sink+1,a[1]); fe_store(sink+2,a[2]); fe_store(sink+3,a[3]); }
}
__global__ void one_ptx(const Fe* x, Fe* y) { y[threadIdx.x] = fe_mul<Bn254>(x[threadIdx.x], x[threadIdx.x+256]); }
__global__ void one_c64(const Fe* x, Fe* y) { y[threadIdx.x] = mul_c64(x[threadIdx.x], x[threadIdx.x+256]); }
__global__ void one_nop(const Fe* x, Fe* y) { y[threadIdx.x] = x[threadIdx.x]; }
#include <cstdio>
// CIOS with 64-bit accumulation, but interleaving the a*b_i and m*p rows per limb
__device__ __forceinline__ Fe mul_c64b(const Fe& a, const Fe& b) {
    constexpr uint32_t P[8] = {0xf0000001u, 0x43e1f593u, 0x79b97091u, 0x2833e848u, 0x8181585du, 0xb85045b6u, 0xe131a029u, 0x30644e72u};
    uint32_t t[9] = {0};
    #pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint64_t s = (uint64_t)a.v[0] * b.v[i] + t[0];
        const uint32_t m = (uint32_t)s * 0xefffffffu;
        uint64_t c1 = s >> 32;
        uint64_t s2 = (uint64_t)m * P[0] + (uint32_t)s;
        uint64_t c2 = s2 >> 32;
        #pragma unroll
        for (int j = 1; j < 8; ++j) {
            s = (uint64_t)a.v[j] * b.v[i] + t[j] + c1;
            c1 = s >> 32;
            s2 = (uint64_t)m * P[j] + (uint32_t)s + c2;
            c2 = s2 >> 32;
            t[j - 1] = (uint32_t)s2;
        }
        s = (uint64_t)t[8] + c1 + c2;
        t[7] = (uint32_t)s;
        t[8] = (uint32_t)(s >> 32);
    }
    Fe r; uint32_t d[8]; uint64_t br = 0;
    #pragma unroll
    for (int j = 0; j < 8; ++j) { uint64_t s = (uint64_t)t[j] - P[j] - br; d[j] = (uint32_t)s; br = (s >> 63); }
    #pragma unroll
    for (int j = 0; j < 8; ++j) r.v[j] = br ? t[j] : d[j];
    return r;
}
__global__ void k_c64b(int iters, Fe* sink, unsigned never) {
    Fe a[4], b; for (int k=0;k<4;++k) for (int i=0;i<8;++i) a[k].v[i]=(threadIdx.x*0x9e3779b9u+k*77+i)&0x0fffffff;
    for (int i=0;i<8;++i) b.v[i]=(blockIdx.x*0x27d4eb2fu+i)&0x0fffffff;
    for (int it=0; it<iters; ++it) { for (int k=0;k<4;++k) a[k]=mul_c64b(a[k],b); }
    if (a[0].v[0]==never) { fe_store(sink,a[0]); fe_store(sink+1,a[1]); fe_store(sink+2,a[2]); fe_store(sink+3,a[3]); }
}
__global__ void k_check(const Fe* x, Fe* y, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    Fe a = x[i], b = x[i + n];
    Fe r0 = fe_mul<Bn254>(a, b), r1 = mul_c64(a, b), r2 = mul_c64b(a, b);
    y[3*i] = r0; y[3*i+1] = r1; y[3*i+2] = r2;
}
int main() {
    Fe* sink; cudaMalloc(&sink, 4 * sizeof(Fe));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = 148 * 8, iters = 2048;
    auto run = [&](const char* name, void (*k)(int, Fe*, unsigned)) {
        k<<<blocks, 256>>>(64, sink, 0xffffffffu);
        cudaEventRecord(e0); k<<<blocks, 256>>>(iters, sink, 0xffffffffu); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-8s %.3e mults/s  (%s)\n", name, (double)blocks * 256 * iters * 4 / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    };
    run("ptx", k_ptx); run("c64", k_c64); run("c64b", k_c64b);
    // correctness: random inputs < p (top limb masked)
    const int n = 1 << 16; Fe* hx = new Fe[2 * n]; unsigned s = 1;
    for (int i = 0; i < 2 * n; ++i) for (int j = 0; j < 8; ++j) { s = s * 1664525u + 1013904223u; hx[i].v[j] = s; }
    for (int i = 0; i < 2 * n; ++i) hx[i].v[7] &= 0x0fffffff;
    Fe *dx, *dy; cudaMalloc(&dx, 2 * n * sizeof(Fe)); cudaMalloc(&dy, 3 * n * sizeof(Fe));
    cudaMemcpy(dx, hx, 2 * n * sizeof(Fe), cudaMemcpyHostToDevice);
    k_check<<<n / 256, 256>>>(dx, dy, n);
    Fe* hy = new Fe[3 * n]; cudaMemcpy(hy, dy, 3 * n * sizeof(Fe), cudaMemcpyDeviceToHost);
    int bad1 = 0, bad2 = 0;
    for (int i = 0; i < n; ++i) { for (int j = 0; j < 8; ++j) { if (hy[3*i].v[j] != hy[3*i+1].v[j]) { bad1++; break; } } for (int j = 0; j < 8; ++j) { if (hy[3*i].v[j] != hy[3*i+2].v[j]) { bad2++; break; } } }
    printf("mismatch c64 %d c64b %d of %d\n", bad1, bad2, n);
    return 0;
}
