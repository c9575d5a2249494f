// Shared pieces of the header-level drop-in (include/dropin/dgkr/*.hpp):
// device/field registry, transcript hand-off, canonical byte conversions.
//
// Put include/dropin FIRST on the include path, the reference's include dir
// after it: the wrapped headers (sumcheck.hpp, gkr.hpp, pcs.hpp) pull in the
// reference header with #include_next, rename its prover function out of the
// way, and define the reference's own name and signature on top of the B200
// C ABI (include/dgkr_b200.h). Verifiers, circuits, fields and transcripts
// stay the reference's code; unchanged reference tests then exercise the GPU
// prover (tests/cpp via oracle/Makefile "dropin" targets).
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "dgkr/field.hpp"
#include "dgkr/transcript.hpp"
#include "dgkr_b200.h"

namespace dgkr::b200_dropin {

[[noreturn]] inline void rethrow(int rc) {
    const std::string msg = dgkr_last_error();
    switch (rc) {  // the reference's exception types
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

// Transcript keeps {state_, draws_} private (transcript.hpp:127-129). An
// explicit template instantiation may name private members (access checks do
// not apply there), which lets the drop-in read and advance the caller's
// transcript in place without changing the reference header.
template <class Tag, typename Tag::type M>
struct Access {
    friend typename Tag::type member(Tag) { return M; }
};
struct StateTag {
    using type = Digest Transcript::*;
    friend type member(StateTag);
};
struct DrawsTag {
    using type = std::uint64_t Transcript::*;
    friend type member(DrawsTag);
};
template struct Access<StateTag, &Transcript::state_>;
template struct Access<DrawsTag, &Transcript::draws_>;

inline dgkr_transcript load(const Transcript& tr) {
    dgkr_transcript t{};
    std::memcpy(t.state, (tr.*member(StateTag{})).data(), 32);
    t.draws = tr.*member(DrawsTag{});
    return t;
}
inline void store(Transcript& tr, const dgkr_transcript& t) {
    std::memcpy((tr.*member(StateTag{})).data(), t.state, 32);
    tr.*member(DrawsTag{}) = t.draws;
}

/// one device context + field handle per modulus (device 0), process-wide
class Device {
public:
    explicit Device(const FieldConfigPtr& cfg) : cfg_(cfg) {
        std::vector<std::uint8_t> mod;
        boost::multiprecision::export_bits(cfg->modulus(), std::back_inserter(mod), 8, false);
        check(dgkr_field_create(mod.data(), mod.size(), &field_));
        check(dgkr_ctx_create(0, &ctx_));
    }
    ~Device() {
        dgkr_ctx_destroy(ctx_);
        dgkr_field_destroy(field_);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    dgkr_ctx* ctx() const { return ctx_; }
    dgkr_field* field() const { return field_; }

private:
    FieldConfigPtr cfg_;
    dgkr_field* field_ = nullptr;
    dgkr_ctx* ctx_ = nullptr;
};

inline Device& device(const FieldConfigPtr& cfg) {
    static std::mutex mu;
    static std::map<std::string, std::unique_ptr<Device>> devs;
    std::lock_guard<std::mutex> lk(mu);
    auto& d = devs[cfg->modulus().str()];
    if (!d) d = std::make_unique<Device>(cfg);
    return *d;
}

inline std::vector<std::uint8_t> canonical(std::span<const FieldElement> v) {
    std::vector<std::uint8_t> out;
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

}  // namespace dgkr::b200_dropin
