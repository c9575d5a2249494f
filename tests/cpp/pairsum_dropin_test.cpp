// The reference's PairSumSession API (sumcheck.hpp:152-221) on the B200 prover
// through the header-level drop-in (include/dropin/dgkr/sumcheck.hpp), built
// by oracle/Makefile with include/dropin first on the include path and run by
// tests/test_gpu_dropin.py. Checks, over BN254 / Goldilocks / p = 97:
//   1. the device session against the reference's own session (renamed
//      PairSumSessionCpuReference by the drop-in) step by step: total(),
//      every round_poly(), final_values(), and the reference exceptions;
//   2. the reference's OWN dist_sumcheck (renamed dist_sumcheck_cpu_reference,
//      cluster.hpp:228-320) -- which now drives one device session per worker
//      plus the master tail -- against the single-machine reference proof over
//      the concatenated tables (the equality cluster.hpp:220-227 claims) and
//      against the drop-in dist_sumcheck (C ABI); TrafficStats JSON equal.
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "dgkr/cluster.hpp"
#include "dgkr/sumcheck.hpp"

using namespace dgkr;

static int failures = 0, checks = 0;
#define EXPECT(c)                                                                    \
    do {                                                                             \
        ++checks;                                                                    \
        if (!(c)) {                                                                  \
            ++failures;                                                              \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);      \
        }                                                                            \
    } while (0)

static MultilinearTable rand_table(const FieldConfigPtr& cfg, std::size_t vars, std::mt19937_64& rng) {
    std::vector<FieldElement> v;
    for (std::size_t i = 0; i < (std::size_t{1} << vars); ++i) v.push_back(random_element(cfg, rng));
    return MultilinearTable(cfg, vars, std::move(v));
}

template <class E, class Fn>
static bool throws_as(Fn&& fn) {
    try {
        fn();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static void session_case(const FieldConfigPtr& cfg, std::size_t vars, std::size_t n_pairs, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::vector<sumcheck::ProductPair> pairs;
    for (std::size_t k = 0; k < n_pairs; ++k) pairs.push_back({rand_table(cfg, vars, rng), rand_table(cfg, vars, rng)});
    sumcheck::PairSumSession dev(pairs);
    sumcheck::PairSumSessionCpuReference ref(pairs);
    EXPECT(dev.vars_left() == ref.vars_left());
    EXPECT(dev.pair_count() == ref.pair_count());
    EXPECT(dev.total() == ref.total());
    for (std::size_t j = 0; j < vars; ++j) {
        const auto a = dev.round_poly(), b = ref.round_poly();
        for (int c = 0; c < 4; ++c) EXPECT(a.coeffs[c] == b.coeffs[c]);
        EXPECT(throws_as<std::logic_error>([&] { (void)dev.final_values(); }));
        const FieldElement r = random_element(cfg, rng);
        dev.fold(r);
        ref.fold(r);
        EXPECT(dev.vars_left() == ref.vars_left());
        EXPECT(dev.total() == ref.total());
    }
    const auto fa = dev.final_values(), fb = ref.final_values();
    EXPECT(fa.size() == fb.size());
    for (std::size_t i = 0; i < fa.size() && i < fb.size(); ++i) EXPECT(fa[i] == fb[i]);
    EXPECT(throws_as<std::logic_error>([&] { (void)dev.round_poly(); }));
    EXPECT(throws_as<std::logic_error>([&] { dev.fold(FieldElement::zero(cfg)); }));
}

static void dist_case(const FieldConfigPtr& cfg, std::size_t n_workers, std::size_t vars, std::size_t n_pairs,
                      std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::vector<sumcheck::ProductPair> pairs;
    for (std::size_t k = 0; k < n_pairs; ++k) pairs.push_back({rand_table(cfg, vars, rng), rand_table(cfg, vars, rng)});
    const auto topo = cluster::ClusterTopology::plan(n_workers);
    const auto shares = cluster::shard_pairs(pairs, n_workers);
    Transcript t_single("pairsum.dist", cfg), t_ref("pairsum.dist", cfg), t_abi("pairsum.dist", cfg);
    const auto single = sumcheck::prove_product_sum_cpu_reference(pairs, t_single);
    cluster::TrafficStats s_ref, s_abi;
    const auto via_sessions = cluster::dist_sumcheck_cpu_reference(topo, shares, t_ref, s_ref);
    const auto via_abi = cluster::dist_sumcheck(topo, shares, t_abi, s_abi);
    EXPECT(via_sessions.to_bytes() == single.to_bytes());
    EXPECT(via_abi.to_bytes() == single.to_bytes());
    EXPECT(t_ref.state() == t_single.state());
    EXPECT(t_abi.state() == t_single.state());
    EXPECT(s_ref.to_json().dump() == s_abi.to_json().dump());
}

int main() {
    const std::vector<FieldConfigPtr> fields = {FieldConfig::bn254(), FieldConfig::goldilocks(),
                                                FieldConfig::make_small_prime(BigInt(97), "p97")};
    std::uint64_t seed = 1;
    for (const auto& cfg : fields) {
        for (std::size_t vars : {0u, 1u, 2u, 3u, 6u, 11u})
            for (std::size_t np : {1u, 3u}) session_case(cfg, vars, np, seed++);
        for (std::size_t n : {1u, 2u, 4u, 8u})
            for (std::size_t np : {1u, 2u}) dist_case(cfg, n, 5, np, seed++);
    }
    // the reference's constructor errors (sumcheck.hpp:155-166)
    EXPECT(throws_as<std::invalid_argument>([] { sumcheck::PairSumSession s(std::span<const sumcheck::ProductPair>{}); }));
    {
        std::mt19937_64 rng(9);
        const auto& cfg = fields[0];
        std::vector<sumcheck::ProductPair> bad = {{rand_table(cfg, 3, rng), rand_table(cfg, 2, rng)}};
        EXPECT(throws_as<std::invalid_argument>([&] { sumcheck::PairSumSession s(bad); }));
    }
    std::printf("pairsum drop-in: %d checks, %d failures\n", checks, failures);
    return failures ? 1 : 0;
}
