// Drop-in dgkr/pcs.hpp: the reference header with commit (pcs.hpp:105) and
// open (:212) on the B200 prover. Same names, signatures, roots and opening
// bytes; verify remains the reference's. Everything pcs.hpp includes is
// included first, so the renaming macros only touch pcs.hpp itself.
#pragma once
#include <algorithm>
#include <array>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "dgkr/field.hpp"
#include "dgkr/merkle.hpp"
#include "dgkr/mle.hpp"
#include "dgkr/sha256.hpp"
#include "dgkr/transcript.hpp"

#define commit commit_cpu_reference
#define open open_cpu_reference
#include_next <dgkr/pcs.hpp>
#undef commit
#undef open

#include "dgkr/b200_dropin_core.hpp"

namespace dgkr::pcs {

inline std::vector<std::uint8_t> b200_matrix_bytes(const EvalMatrix& m) {
    std::vector<std::uint8_t> data;
    for (std::size_t i = 0; i < m.rows(); ++i) {
        auto r = dgkr::b200_dropin::canonical(m.row(i));
        data.insert(data.end(), r.begin(), r.end());
    }
    return data;
}

inline Commitment commit(const EvalMatrix& m) {
    namespace B = dgkr::b200_dropin;
    B::Device& dev = B::device(m.config());
    const auto data = b200_matrix_bytes(m);
    Commitment com;
    com.rows = m.rows();
    com.cols = m.cols();
    B::check(dgkr_pcs_commit(dev.ctx(), dev.field(), m.rows(), m.cols(), data.data(), com.root.data()));
    return com;
}

inline Opening open(const EvalMatrix& m, std::span<const FieldElement> r, Transcript& transcript,
                    std::size_t q = 32) {
    namespace B = dgkr::b200_dropin;
    const FieldConfigPtr& cfg = m.config();
    const std::size_t w = cfg->byte_width();
    B::Device& dev = B::device(cfg);
    const auto data = b200_matrix_bytes(m);
    const auto rb = B::canonical(r);
    std::size_t depth = 0;
    while ((std::size_t{1} << depth) < m.cols()) ++depth;
    const std::size_t nq = std::min(q, m.cols());
    std::vector<std::uint8_t> out(64 + (r.size() + 2 + m.rows() + m.cols()) * w + nq * (4 + m.rows() * w + 32 * depth));
    std::size_t len = 0;
    dgkr_transcript t = B::load(transcript);
    B::check(dgkr_pcs_open(dev.ctx(), dev.field(), m.rows(), m.cols(), data.data(), rb.empty() ? nullptr : rb.data(),
                           r.size(), q, &t, out.data(), out.size(), &len));
    B::store(transcript, t);
    // Opening::to_bytes layout (pcs.hpp:135-156)
    const std::uint8_t* p = out.data();
    Opening op;
    const std::uint32_t nr = B::take_u32(p);
    for (std::uint32_t i = 0; i < nr; ++i) op.point.push_back(B::take_elem(p, cfg));
    op.value = B::take_elem(p, cfg);
    const std::uint32_t rows = B::take_u32(p);
    for (std::uint32_t i = 0; i < rows; ++i) op.row_evals.push_back(B::take_elem(p, cfg));
    const std::uint32_t cols = B::take_u32(p);
    for (std::uint32_t i = 0; i < cols; ++i) op.combined_row.push_back(B::take_elem(p, cfg));
    const std::uint32_t ns = B::take_u32(p);
    for (std::uint32_t k = 0; k < ns; ++k) {
        op.spot_indices.push_back(B::take_u32(p));
        std::vector<FieldElement> col;
        for (std::uint32_t i = 0; i < rows; ++i) col.push_back(B::take_elem(p, cfg));
        op.spot_columns.push_back(std::move(col));
        std::vector<Digest> path;
        for (std::size_t d = 0; d < depth; ++d) {
            Digest dg;
            std::memcpy(dg.data(), p, 32);
            p += 32;
            path.push_back(dg);
        }
        op.spot_paths.push_back(std::move(path));
    }
    return op;
}

}  // namespace dgkr::pcs
