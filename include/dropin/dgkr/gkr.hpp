// Drop-in dgkr/gkr.hpp: the reference header with gkr_prove (gkr.hpp:182) on
// the B200 prover. Same name, signature, proof (bit-exact) and exceptions;
// gkr_verify and the claim helpers remain the reference's.
#pragma once
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "dgkr/circuit.hpp"
#include "dgkr/field.hpp"
#include "dgkr/mle.hpp"
#include "dgkr/sumcheck.hpp"
#include "dgkr/transcript.hpp"

#define gkr_prove gkr_prove_cpu_reference
#include_next <dgkr/gkr.hpp>
#undef gkr_prove

#include "dgkr/b200_dropin_core.hpp"

namespace dgkr::gkr {

inline GkrProof gkr_prove(const circuit::GeneralCircuit& c, std::span<const FieldElement> inputs,
                          const FieldConfigPtr& cfg, Transcript& transcript) {
    namespace B = dgkr::b200_dropin;
    c.require_valid();  // gkr.hpp:185 (logic_error when not validated)
    if (inputs.size() != c.input_size()) throw std::invalid_argument("input count does not match the circuit");
    // the circuit as the C ABI's flat CSR (include/dgkr_b200.h), padding kept
    std::vector<std::uint64_t> lgs{0}, gns{0}, minp;
    std::vector<std::uint32_t> nested;
    for (std::size_t li = 1; li <= c.depth(); ++li) {
        for (const auto& g : c.gates(li)) {
            for (const auto& ng : g.nested)
                nested.insert(nested.end(), {ng.kind == circuit::GateKind::mul ? 1u : 0u, ng.left.layer,
                                             ng.left.gate, ng.right.layer, ng.right.gate});
            gns.push_back(nested.size() / 5);
        }
        lgs.push_back(gns.size() - 1);
    }
    for (std::size_t l = 0; l <= c.depth(); ++l) minp.push_back(c.padded_size(l));
    B::Device& dev = B::device(cfg);
    dgkr_circuit* dc = nullptr;
    B::check(dgkr_circuit_create(dev.ctx(), static_cast<std::uint32_t>(c.input_size()),
                                 static_cast<std::uint32_t>(c.depth()), lgs.data(), gns.data(),
                                 nested.empty() ? nullptr : nested.data(), minp.data(), 1, &dc));
    struct Free {
        dgkr_circuit* c;
        ~Free() { dgkr_circuit_destroy(c); }
    } guard{dc};
    const auto in = B::canonical(inputs);
    std::vector<std::uint8_t> out(dgkr_gkr_proof_bound(dc, dev.field()));
    std::size_t len = 0;
    dgkr_transcript t = B::load(transcript);
    B::check(dgkr_gkr_prove(dev.ctx(), dc, dev.field(), in.data(), &t, out.data(), out.size(), &len));
    B::store(transcript, t);
    // GkrProof from the ABI layout: u32 n_out | outputs | u32 n_layers | per layer (alphas, SumcheckProof)
    const std::uint8_t* p = out.data();
    GkrProof proof;
    const std::uint32_t n_out = B::take_u32(p);
    for (std::uint32_t i = 0; i < n_out; ++i) proof.claimed_outputs.push_back(B::take_elem(p, cfg));
    const std::uint32_t n_layers = B::take_u32(p);
    for (std::uint32_t l = 0; l < n_layers; ++l) {
        GkrLayerProof lp;
        const std::uint32_t na = B::take_u32(p);
        for (std::uint32_t i = 0; i < na; ++i) lp.alphas.push_back(B::take_elem(p, cfg));
        const std::uint32_t sl = B::take_u32(p);
        lp.sum = sumcheck::SumcheckProof::from_bytes(std::span<const std::uint8_t>(p, sl), cfg);
        p += sl;
        proof.layers.push_back(std::move(lp));
    }
    return proof;
}

}  // namespace dgkr::gkr
