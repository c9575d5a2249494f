// Host <-> device round-trip latency on this box: (a) a resident kernel and a
// host thread ping-ponging through pinned mapped memory (the tail kernel's
// mailbox), in several flavours; (b) the per-round launch path: tiny kernel +
// 96-byte D2H + stream sync + 32-byte H2D. Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mailbox_probe mailbox_probe.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            std::printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); \
            return 1;                                                           \
        }                                                                       \
    } while (0)

struct alignas(128) Box {
    volatile unsigned d;
    unsigned pad0[31];
    volatile unsigned h;
    unsigned pad1[31];
};

template <int MODE>
__global__ void pingpong(Box* b, int n, unsigned* dev_flag) {
    if (threadIdx.x != 0) return;
    for (int i = 1; i <= n; ++i) {
        if (MODE == 0) {
            __threadfence_system();
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(&b->d), "r"(i) : "memory");
        } else {
            b->d = i;
        }
        for (;;) {
            unsigned h;
            if (MODE == 0) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(h) : "l"(&b->h) : "memory");
            else h = b->h;
            if (h == static_cast<unsigned>(i)) break;
            if (MODE == 2) __nanosleep(100);
        }
    }
}

__global__ void tiny(unsigned* x) {
    if (threadIdx.x == 0) x[0] += 1;
}

int main() {
    Box* b;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&b), sizeof(Box), cudaHostAllocMapped));
    Box* bd;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&bd), b, 0));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const int n = 2000;
    const char* names[3] = {"release/acquire.sys, spin", "volatile, spin", "volatile, nanosleep(100)"};
    for (int mode = 0; mode < 3; ++mode) {
        b->d = 0;
        b->h = 0;
        if (mode == 0) pingpong<0><<<1, 32, 0, st>>>(bd, n, nullptr);
        if (mode == 1) pingpong<1><<<1, 32, 0, st>>>(bd, n, nullptr);
        if (mode == 2) pingpong<2><<<1, 32, 0, st>>>(bd, n, nullptr);
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 1; i <= n; ++i) {
            if (i == 11) t0 = std::chrono::steady_clock::now();
            while (__atomic_load_n(const_cast<unsigned*>(&b->d), __ATOMIC_ACQUIRE) != static_cast<unsigned>(i)) {
            }
            __atomic_store_n(const_cast<unsigned*>(&b->h), static_cast<unsigned>(i), __ATOMIC_RELEASE);
        }
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        CK(cudaStreamSynchronize(st));
        std::printf("{\"probe\": \"mailbox round trip (%s)\", \"us\": %.2f}\n", names[mode], us / (n - 10));
    }
    unsigned* x;
    CK(cudaMalloc(&x, 256));
    unsigned* hx;
    CK(cudaMallocHost(&hx, 256));
    for (int variant = 0; variant < 2; ++variant) {
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < n; ++i) {
            if (i == 10) t0 = std::chrono::steady_clock::now();
            tiny<<<1, 32, 0, st>>>(x);
            if (variant == 1) {
                CK(cudaMemcpyAsync(hx, x, 96, cudaMemcpyDeviceToHost, st));
            }
            CK(cudaStreamSynchronize(st));
            if (variant == 1) CK(cudaMemcpyAsync(x + 32, hx + 32, 32, cudaMemcpyHostToDevice, st));
        }
        CK(cudaStreamSynchronize(st));
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        std::printf("{\"probe\": \"%s\", \"us\": %.2f}\n",
                    variant ? "launch + 96 B D2H + sync + 32 B H2D" : "launch + sync", us / (n - 10));
    }
    return 0;
}
