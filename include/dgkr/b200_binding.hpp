// Reference-side binding: routes the reference library's prover calls
// (dgkr::gkr::gkr_prove, dgkr::sumcheck::prove_product_sum,
// dgkr::pcs::commit / open, dgkr::cluster::dist_sumcheck) to the B200 C ABI
// (include/dgkr_b200.h), taking and returning the REFERENCE's own types.
//
// Include it after the reference headers (/root/reference/proj/include). It is
// header-only and links against paper_2404_10404_b200/libdgkr_b200.so.
//
// Transcript hand-off: dgkr::Transcript keeps {state_, draws_} private
// (transcript.hpp:127-129). The binding reads the state through
// Transcript::state() and takes the draw counter from the caller (0 for a
// freshly constructed transcript plus absorbs, the pattern every reference
// caller uses); it returns the advanced {state, draws}. A maintainer adopting
// the binding adds the two accessors shown in INTEGRATION.md so the
// transcript object itself can be advanced in place.
#pragma once

#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "dgkr/circuit.hpp"
#include "dgkr/field.hpp"
#include "dgkr/gkr.hpp"
#include "dgkr/pcs.hpp"
#include "dgkr/sumcheck.hpp"
#include "dgkr/transcript.hpp"
#include "dgkr_b200.h"

namespace dgkr::b200 {

[[noreturn]] inline void rethrow(int rc) {
    const std::string msg = dgkr_last_error();
    switch (rc) {  // same exception types as the reference
        case DGKR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case DGKR_DOMAIN_ERROR: throw std::domain_error(msg);
        case DGKR_OUT_OF_RANGE: throw std::out_of_range(msg);
        case DGKR_LOGIC_ERROR: throw std::logic_error(msg);
        default: throw std::runtime_error("dgkr_b200: " + msg);
    }
}
inline void check(int rc) {
    if (rc != DGKR_OK) rethrow(rc);
}

/// One device context + field handle per (device, modulus).
class Device {
public:
    explicit Device(const FieldConfigPtr& cfg, int device = 0) : cfg_(cfg) {
        std::vector<std::uint8_t> mod;
        boost::multiprecision::export_bits(cfg->modulus(), std::back_inserter(mod), 8, false);
        check(dgkr_field_create(mod.data(), mod.size(), &field_));
        check(dgkr_ctx_create(device, &ctx_));
    }
    ~Device() {
        dgkr_ctx_destroy(ctx_);
        dgkr_field_destroy(field_);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    dgkr_ctx* ctx() const { return ctx_; }
    dgkr_field* field() const { return field_; }
    const FieldConfigPtr& config() const { return cfg_; }

private:
    FieldConfigPtr cfg_;
    dgkr_field* field_ = nullptr;
    dgkr_ctx* ctx_ = nullptr;
};

struct TranscriptState {
    dgkr_transcript t{};
    static TranscriptState from(const Transcript& tr, std::uint64_t draws) {
        TranscriptState s;
        const Digest d = tr.state();
        std::memcpy(s.t.state, d.data(), 32);
        s.t.draws = draws;
        return s;
    }
};

inline std::vector<std::uint8_t> canonical(std::span<const FieldElement> v, std::size_t width) {
    std::vector<std::uint8_t> out;
    out.reserve(v.size() * width);
    for (const auto& e : v) e.append_bytes(out);
    return out;
}

inline FieldElement take_elem(const std::uint8_t*& p, const FieldConfigPtr& cfg) {
    auto e = FieldElement::from_bytes(std::span<const std::uint8_t>(p, cfg->byte_width()), cfg);
    p += cfg->byte_width();
    return e;
}
inline std::uint32_t take_u32(const std::uint8_t*& p) {
    std::uint32_t v = 0;
    for (int i = 3; i >= 0; --i) v = (v << 8) | p[i];
    p += 4;
    return v;
}

/// dgkr_circuit_create from a reference GeneralCircuit (flat CSR layout).
class Circuit {
public:
    Circuit(const Device& dev, const circuit::GeneralCircuit& c) {
        std::vector<std::uint64_t> lgs{0}, gns{0}, minp;
        std::vector<std::uint32_t> nested;
        for (std::size_t li = 1; li <= c.depth(); ++li) {
            for (const auto& g : c.gates(li)) {
                for (const auto& ng : g.nested) {
                    nested.insert(nested.end(), {ng.kind == circuit::GateKind::mul ? 1u : 0u, ng.left.layer,
                                                 ng.left.gate, ng.right.layer, ng.right.gate});
                }
                gns.push_back(nested.size() / 5);
            }
            lgs.push_back(gns.size() - 1);
        }
        for (std::size_t l = 0; l <= c.depth(); ++l) minp.push_back(c.padded_size(l));
        check(dgkr_circuit_create(dev.ctx(), static_cast<std::uint32_t>(c.input_size()),
                                  static_cast<std::uint32_t>(c.depth()), lgs.data(), gns.data(),
                                  nested.empty() ? nullptr : nested.data(), minp.data(), 1, &h_));
    }
    ~Circuit() { dgkr_circuit_destroy(h_); }
    Circuit(const Circuit&) = delete;
    Circuit& operator=(const Circuit&) = delete;
    dgkr_circuit* handle() const { return h_; }

private:
    dgkr_circuit* h_ = nullptr;
};

/// gkr::gkr_prove (gkr.hpp:182) on the GPU; returns the reference GkrProof.
inline gkr::GkrProof gkr_prove(const Device& dev, const Circuit& circ, std::span<const FieldElement> inputs,
                               TranscriptState& ts) {
    const auto& cfg = dev.config();
    auto in = canonical(inputs, cfg->byte_width());
    std::vector<std::uint8_t> out(dgkr_gkr_proof_bound(circ.handle(), dev.field()));
    std::size_t len = 0;
    check(dgkr_gkr_prove(dev.ctx(), circ.handle(), dev.field(), in.data(), &ts.t, out.data(), out.size(), &len));
    const std::uint8_t* p = out.data();
    gkr::GkrProof proof;
    const std::uint32_t n_out = take_u32(p);
    for (std::uint32_t i = 0; i < n_out; ++i) proof.claimed_outputs.push_back(take_elem(p, cfg));
    const std::uint32_t n_layers = take_u32(p);
    for (std::uint32_t l = 0; l < n_layers; ++l) {
        gkr::GkrLayerProof lp;
        const std::uint32_t na = take_u32(p);
        for (std::uint32_t i = 0; i < na; ++i) lp.alphas.push_back(take_elem(p, cfg));
        const std::uint32_t sl = take_u32(p);
        lp.sum = sumcheck::SumcheckProof::from_bytes(std::span<const std::uint8_t>(p, sl), cfg);
        p += sl;
        proof.layers.push_back(std::move(lp));
    }
    return proof;
}

/// sumcheck::prove_product_sum (sumcheck.hpp:226) on the GPU.
inline sumcheck::SumcheckProof prove_product_sum(const Device& dev, std::span<const sumcheck::ProductPair> pairs,
                                                 TranscriptState& ts) {
    if (pairs.empty()) throw std::invalid_argument("product sum needs at least one pair");
    const auto& cfg = dev.config();
    std::vector<std::uint8_t> tabs;
    for (const auto& pr : pairs) {
        if (pr.f.num_vars() != pairs.front().f.num_vars() || pr.g.num_vars() != pairs.front().f.num_vars())
            throw std::invalid_argument("mixed table sizes in product sum");
        auto a = canonical(pr.f.evals(), cfg->byte_width()), b = canonical(pr.g.evals(), cfg->byte_width());
        tabs.insert(tabs.end(), a.begin(), a.end());
        tabs.insert(tabs.end(), b.begin(), b.end());
    }
    const std::size_t vars = pairs.front().f.num_vars();
    std::vector<std::uint8_t> out(64 + (vars + 2) * 4 * cfg->byte_width() + 2 * pairs.size() * cfg->byte_width());
    std::size_t len = 0;
    check(dgkr_prove_product_sum(dev.ctx(), dev.field(), pairs.size(), vars, tabs.data(), &ts.t, out.data(),
                                 out.size(), &len));
    return sumcheck::SumcheckProof::from_bytes(std::span<const std::uint8_t>(out.data(), len), cfg);
}

/// pcs::commit (pcs.hpp:105) on the GPU.
inline pcs::Commitment pcs_commit(const Device& dev, const pcs::EvalMatrix& m) {
    std::vector<std::uint8_t> data;
    for (std::size_t i = 0; i < m.rows(); ++i) {
        auto r = canonical(m.row(i), dev.config()->byte_width());
        data.insert(data.end(), r.begin(), r.end());
    }
    pcs::Commitment com;
    com.rows = m.rows();
    com.cols = m.cols();
    check(dgkr_pcs_commit(dev.ctx(), dev.field(), m.rows(), m.cols(), data.data(), com.root.data()));
    return com;
}

}  // namespace dgkr::b200
