// GPU test (built by oracle/Makefile into oracle/_ref/binding_test): the
// reference library's own types and calls, routed through the B200 binding
// (include/dgkr/b200_binding.hpp), must produce the same proofs as the
// reference prover itself. Exit code 0 = all equal.
#include <cstdio>
#include <random>

#include "dgkr/b200_binding.hpp"
#include "dgkr/circuit.hpp"
#include "dgkr/gkr.hpp"
#include "dgkr/pcs.hpp"
#include "dgkr/sumcheck.hpp"

using namespace dgkr;

static std::vector<std::uint8_t> gkr_bytes(const gkr::GkrProof& p) {
    std::vector<std::uint8_t> out;
    for (const auto& e : p.claimed_outputs) e.append_bytes(out);
    for (const auto& lp : p.layers) {
        for (const auto& a : lp.alphas) a.append_bytes(out);
        auto b = lp.sum.to_bytes();
        out.insert(out.end(), b.begin(), b.end());
    }
    return out;
}

int main() {
    int failures = 0;
    for (auto cfg : {FieldConfig::bn254(), FieldConfig::goldilocks()}) {
        b200::Device dev(cfg);
        std::mt19937_64 rng(77);
        for (int trial = 0; trial < 8; ++trial) {
            circuit::RandomCircuitParams p;
            p.input_size = 5 + trial;
            p.depth = 2 + trial % 4;
            p.max_gates_per_layer = 24;
            p.max_nested = 3;
            auto c = circuit::random_general_circuit(rng, p);
            std::vector<FieldElement> inputs;
            for (std::size_t i = 0; i < p.input_size; ++i) inputs.push_back(random_element(cfg, rng));
            Transcript ref_tr("binding.gkr", cfg);
            ref_tr.absorb_u64(static_cast<std::uint64_t>(trial));
            auto ts = b200::TranscriptState::from(ref_tr, 0);
            auto want = gkr::gkr_prove(c, inputs, cfg, ref_tr);
            b200::Circuit dc(dev, c);
            auto got = b200::gkr_prove(dev, dc, inputs, ts);
            const auto st = ref_tr.state();
            if (gkr_bytes(got) != gkr_bytes(want) || std::memcmp(st.data(), ts.t.state, 32) != 0) {
                std::printf("gkr mismatch (%s, trial %d)\n", cfg->name().c_str(), trial);
                ++failures;
            }
            Transcript vtr("binding.gkr", cfg);
            vtr.absorb_u64(static_cast<std::uint64_t>(trial));
            if (!gkr::gkr_verify(c, c.outputs(inputs, cfg), got, cfg, vtr).accept) {
                std::printf("reference verifier rejected the GPU proof (trial %d)\n", trial);
                ++failures;
            }
        }
        for (std::size_t vars : {0u, 3u, 9u}) {
            std::vector<sumcheck::ProductPair> pairs;
            for (int k = 0; k < 2; ++k) {
                std::vector<FieldElement> f, g;
                for (std::size_t i = 0; i < (std::size_t{1} << vars); ++i) {
                    f.push_back(random_element(cfg, rng));
                    g.push_back(random_element(cfg, rng));
                }
                pairs.push_back({MultilinearTable(cfg, vars, f), MultilinearTable(cfg, vars, g)});
            }
            Transcript ref_tr("binding.sum", cfg);
            auto ts = b200::TranscriptState::from(ref_tr, 0);
            auto want = sumcheck::prove_product_sum(pairs, ref_tr);
            auto got = b200::prove_product_sum(dev, pairs, ts);
            if (got.to_bytes() != want.to_bytes()) {
                std::printf("product sum mismatch (vars %zu)\n", vars);
                ++failures;
            }
        }
        std::vector<FieldElement> data;
        for (int i = 0; i < 4 * 64; ++i) data.push_back(random_element(cfg, rng));
        pcs::EvalMatrix m(cfg, 4, 64, data);
        if (b200::pcs_commit(dev, m).root != pcs::commit(m).root) {
            std::printf("pcs root mismatch\n");
            ++failures;
        }
        try {  // error mapping: mixed table sizes -> std::invalid_argument (sumcheck.hpp:161-163)
            std::vector<sumcheck::ProductPair> bad{{MultilinearTable::zeros(cfg, 1), MultilinearTable::zeros(cfg, 1)},
                                                   {MultilinearTable::zeros(cfg, 2), MultilinearTable::zeros(cfg, 2)}};
            Transcript t("x", cfg);
            auto ts = b200::TranscriptState::from(t, 0);
            b200::prove_product_sum(dev, bad, ts);
            ++failures;
        } catch (const std::invalid_argument&) {
        }
    }
    std::printf(failures ? "binding FAILED (%d)\n" : "binding ok\n", failures);
    return failures ? 1 : 0;
}
