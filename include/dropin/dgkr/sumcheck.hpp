// Drop-in dgkr/sumcheck.hpp: the reference header with PairSumSession
// (sumcheck.hpp:152-221), prove_product_sum (:226) and prove_layer_sum (:342)
// on the B200 prover. Same names, signatures, proofs (bit-exact) and
// exception types. The reference's own PairSumSession is renamed
// PairSumSessionCpuReference (it still backs the renamed CPU provers), so
// reference code that drives sessions itself -- cluster::dist_sumcheck
// (cluster.hpp:250-316) -- runs one device session per worker.
#pragma once
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "dgkr/counters.hpp"
#include "dgkr/field.hpp"
#include "dgkr/mle.hpp"
#include "dgkr/transcript.hpp"

#define prove_product_sum prove_product_sum_cpu_reference
#define prove_layer_sum prove_layer_sum_cpu_reference
#define PairSumSession PairSumSessionCpuReference
#include_next <dgkr/sumcheck.hpp>
#undef prove_product_sum
#undef prove_layer_sum
#undef PairSumSession

#include <memory>

#include "dgkr/b200_dropin_core.hpp"

namespace dgkr::sumcheck {

/// PairSumSession (sumcheck.hpp:152-221) on the device (dgkr_pairsum_*):
/// the tables are copied to the GPU at construction; round_poly / fold /
/// final_values / total are device launches. Copies share one session.
class PairSumSession {
public:
    explicit PairSumSession(std::span<const ProductPair> pairs) {
        namespace B = dgkr::b200_dropin;
        if (pairs.empty()) throw std::invalid_argument("product sum needs at least one pair");  // :155-157
        cfg_ = pairs.front().f.config();
        const std::size_t vars = pairs.front().f.num_vars();
        std::vector<std::uint8_t> tabs;
        for (const auto& p : pairs) {  // :160-169
            if (p.f.num_vars() != vars || p.g.num_vars() != vars)
                throw std::invalid_argument("mixed table sizes in product sum");
            if (p.f.config()->modulus() != cfg_->modulus() || p.g.config()->modulus() != cfg_->modulus())
                throw std::invalid_argument("mixed field configs in product sum");
            auto a = B::canonical(p.f.evals()), b = B::canonical(p.g.evals());
            tabs.insert(tabs.end(), a.begin(), a.end());
            tabs.insert(tabs.end(), b.begin(), b.end());
        }
        n_pairs_ = pairs.size();
        B::Device& dev = B::device(cfg_);
        dgkr_pairsum* h = nullptr;
        B::check(dgkr_pairsum_begin(dev.ctx(), dev.field(), n_pairs_, vars, tabs.data(), &h));
        h_ = std::shared_ptr<dgkr_pairsum>(h, dgkr_pairsum_end);
    }

    const FieldConfigPtr& config() const { return cfg_; }
    std::size_t vars_left() const { return dgkr_pairsum_vars_left(h_.get()); }
    std::size_t pair_count() const { return n_pairs_; }

    FieldElement total() const {
        std::vector<std::uint8_t> b(cfg_->byte_width());
        dgkr::b200_dropin::check(dgkr_pairsum_total(h_.get(), b.data()));
        const std::uint8_t* p = b.data();
        return dgkr::b200_dropin::take_elem(p, cfg_);
    }

    RoundPolynomial round_poly() const {
        std::vector<std::uint8_t> b(4 * cfg_->byte_width());
        dgkr::b200_dropin::check(dgkr_pairsum_round(h_.get(), b.data()));
        const std::uint8_t* p = b.data();
        FieldElement c0 = dgkr::b200_dropin::take_elem(p, cfg_);
        FieldElement c1 = dgkr::b200_dropin::take_elem(p, cfg_);
        FieldElement c2 = dgkr::b200_dropin::take_elem(p, cfg_);
        FieldElement c3 = dgkr::b200_dropin::take_elem(p, cfg_);
        return RoundPolynomial{{c0, c1, c2, c3}};
    }

    void fold(const FieldElement& r) {
        std::vector<std::uint8_t> b;
        r.append_bytes(b);
        dgkr::b200_dropin::check(dgkr_pairsum_fold(h_.get(), b.data()));
    }

    std::vector<FieldElement> final_values() const {
        std::vector<std::uint8_t> b(2 * n_pairs_ * cfg_->byte_width());
        dgkr::b200_dropin::check(dgkr_pairsum_finals(h_.get(), b.data()));
        const std::uint8_t* p = b.data();
        std::vector<FieldElement> out;
        for (std::size_t i = 0; i < 2 * n_pairs_; ++i) out.push_back(dgkr::b200_dropin::take_elem(p, cfg_));
        return out;
    }

private:
    FieldConfigPtr cfg_;
    std::size_t n_pairs_ = 0;
    std::shared_ptr<dgkr_pairsum> h_;
};

inline SumcheckProof prove_product_sum(std::span<const ProductPair> pairs, Transcript& transcript) {
    namespace B = dgkr::b200_dropin;
    if (pairs.empty()) throw std::invalid_argument("product sum needs at least one pair");  // sumcheck.hpp:155-157
    const FieldConfigPtr& cfg = pairs.front().f.config();
    const std::size_t vars = pairs.front().f.num_vars();
    std::vector<std::uint8_t> tabs;
    for (const auto& pr : pairs) {
        if (pr.f.num_vars() != vars || pr.g.num_vars() != vars)
            throw std::invalid_argument("mixed table sizes in product sum");
        auto a = B::canonical(pr.f.evals()), b = B::canonical(pr.g.evals());
        tabs.insert(tabs.end(), a.begin(), a.end());
        tabs.insert(tabs.end(), b.begin(), b.end());
    }
    B::Device& dev = B::device(cfg);
    std::vector<std::uint8_t> out(64 + (vars + 2) * 4 * cfg->byte_width() + 2 * pairs.size() * cfg->byte_width());
    std::size_t len = 0;
    dgkr_transcript t = B::load(transcript);
    B::check(dgkr_prove_product_sum(dev.ctx(), dev.field(), pairs.size(), vars, tabs.data(), &t, out.data(),
                                    out.size(), &len));
    B::store(transcript, t);
    return SumcheckProof::from_bytes(std::span<const std::uint8_t>(out.data(), len), cfg);
}

inline LayerProveResult prove_layer_sum(const LayerInstance& inst, const FieldElement& claimed,
                                        Transcript& transcript) {
    namespace B = dgkr::b200_dropin;
    const FieldConfigPtr& cfg = claimed.config();
    const std::size_t w = cfg->byte_width(), ns = inst.slot_tables.size();
    std::vector<std::uint8_t> tabs;
    for (const auto& t : inst.slot_tables) {  // sumcheck.hpp:349-353
        if (t.num_vars() != inst.side_vars) throw std::invalid_argument("slot table not padded to side_vars");
        auto b = B::canonical(t.evals());
        tabs.insert(tabs.end(), b.begin(), b.end());
    }
    const std::uint64_t table_size = std::uint64_t{1} << inst.side_vars;
    for (const auto& wi : inst.wires)  // sumcheck.hpp:354-359
        if (wi.x_slot >= ns || wi.y_slot >= ns || wi.x_index >= table_size || wi.y_index >= table_size)
            throw std::invalid_argument("layer wire index out of range");
    std::vector<std::uint32_t> meta;
    std::vector<std::uint64_t> idx;
    std::vector<std::uint8_t> weights;
    for (const auto& wi : inst.wires) {
        meta.insert(meta.end(), {wi.is_mul ? 1u : 0u, wi.x_slot, wi.y_slot});
        idx.insert(idx.end(), {wi.x_index, wi.y_index});
        wi.weight.append_bytes(weights);
    }
    std::vector<std::uint8_t> cl;
    claimed.append_bytes(cl);
    B::Device& dev = B::device(cfg);
    const std::size_t side = inst.side_vars;
    std::vector<std::uint8_t> out(64 + (2 * side + 2) * 4 * w + 2 * ns * w + w), xp(std::max<std::size_t>(side, 1) * w),
        yp(std::max<std::size_t>(side, 1) * w);
    std::size_t len = 0;
    dgkr_transcript t = B::load(transcript);
    B::check(dgkr_prove_layer_sum(dev.ctx(), dev.field(), side, ns, tabs.data(), inst.wires.size(),
                                  meta.empty() ? nullptr : meta.data(), idx.empty() ? nullptr : idx.data(),
                                  weights.empty() ? nullptr : weights.data(), cl.data(), &t, out.data(), out.size(),
                                  &len, xp.data(), yp.data()));
    B::store(transcript, t);
    LayerProveResult res;
    res.proof = SumcheckProof::from_bytes(std::span<const std::uint8_t>(out.data(), len), cfg);
    const std::uint8_t* px = xp.data();
    const std::uint8_t* py = yp.data();
    for (std::size_t k = 0; k < side; ++k) {
        res.x_point.push_back(B::take_elem(px, cfg));
        res.y_point.push_back(B::take_elem(py, cfg));
    }
    return res;
}

}  // namespace dgkr::sumcheck
