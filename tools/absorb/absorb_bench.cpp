// Host absorb-chain throughput probe (the C2 output absorb, gkr.hpp:189-190):
// ns per absorb for one chain, K chains interleaved in one thread, and T
// threads at once. Checks the interleaved chains against the single chain.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "../../paper_2404_10404_b200/csrc/host_core.hpp"

using namespace dgkr_b200;
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main(int argc, char** argv) {
    const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : (1u << 20);
    std::vector<std::uint8_t> data(32 * n * 4);
    for (std::size_t i = 0; i < data.size(); ++i) data[i] = static_cast<std::uint8_t>(i * 2654435761u >> 13);
    std::uint8_t ref[4][32] = {};
    double t0 = now();
    for (int k = 0; k < 4; ++k) absorb_chain32(ref[k], data.data() + 32 * n * k, n);
    const double t1 = (now() - t0) / 4;
    std::printf("{\"probe\": \"single\", \"ns_per_absorb\": %.2f}\n", 1e9 * t1 / n);
    for (int K = 2; K <= 4; ++K) {
        std::uint8_t st[4][32] = {};
        std::uint8_t* sp[4] = {st[0], st[1], st[2], st[3]};
        const std::uint8_t* ep[4];
        for (int k = 0; k < 4; ++k) ep[k] = data.data() + 32 * n * k;
        t0 = now();
        absorb_chain32_multi(sp, ep, K, n);
        const double t = now() - t0;
        bool ok = true;
        for (int k = 0; k < K; ++k) ok &= std::memcmp(st[k], ref[k], 32) == 0;
        std::printf("{\"probe\": \"interleaved\", \"K\": %d, \"ns_per_absorb_per_chain\": %.2f, \"speedup\": %.2f, \"equal\": %s}\n", K,
                    1e9 * t / n / K, t1 * K / t, ok ? "true" : "false");
    }
    const unsigned T = std::thread::hardware_concurrency();
    for (int K : {1, 2, 3, 4}) {
        std::vector<std::thread> th;
        t0 = now();
        for (unsigned j = 0; j < T; ++j)
            th.emplace_back([&, K] {
                std::uint8_t st[4][32] = {};
                std::uint8_t* sp[4] = {st[0], st[1], st[2], st[3]};
                const std::uint8_t* ep[4];
                for (int k = 0; k < 4; ++k) ep[k] = data.data() + 32 * n * k;
                absorb_chain32_multi(sp, ep, K, n);
            });
        for (auto& x : th) x.join();
        const double t = now() - t0;
        std::printf("{\"probe\": \"threads\", \"threads\": %u, \"K\": %d, \"absorbs_per_s\": %.3e}\n", T, K, T * K * n / t);
    }
    return 0;
}
