// Drop-in dgkr/cluster.hpp: the reference header with dist_sumcheck
// (cluster.hpp:228-320) on the B200 prover. Same name, signature, proof bytes
// and exceptions; the caller's TrafficStats receives the reference's message
// sequence (fully determined by workers, local variables, pairs and element
// width). DistPc stays the reference's class; its pcs::commit / open calls
// resolve to the drop-in pcs.hpp.
#pragma once
#include <cstdint>
#include <functional>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

#include "dgkr/field.hpp"
#include "dgkr/mle.hpp"
#include "dgkr/pcs.hpp"
#include "dgkr/sumcheck.hpp"
#include "dgkr/transcript.hpp"

#define dist_sumcheck dist_sumcheck_cpu_reference
#include_next <dgkr/cluster.hpp>
#undef dist_sumcheck

#include "dgkr/b200_dropin_core.hpp"

namespace dgkr::cluster {

inline sumcheck::SumcheckProof dist_sumcheck(const ClusterTopology& topo, std::span<const WorkerShare> shares,
                                             Transcript& transcript, TrafficStats& stats) {
    namespace B = dgkr::b200_dropin;
    if (shares.size() != topo.n_workers) throw std::invalid_argument("share count must match topology");
    const std::size_t n_pairs = shares.front().pairs.size();
    const std::size_t local_vars = shares.front().pairs.front().f.num_vars();
    for (const auto& s : shares) {  // cluster.hpp:237-246
        if (s.pairs.size() != n_pairs) throw std::invalid_argument("inconsistent share dimensions");
        for (const auto& p : s.pairs)
            if (p.f.num_vars() != local_vars || p.g.num_vars() != local_vars)
                throw std::invalid_argument("inconsistent share dimensions");
    }
    const FieldConfigPtr cfg = shares.front().pairs.front().f.config();
    const std::size_t width = cfg->byte_width(), n = topo.n_workers;
    std::size_t index_vars = 0;
    while ((std::size_t{1} << index_vars) < n) ++index_vars;
    // full tables (worker = high variables, shard_pairs' row-major chunks), f_k then g_k
    std::vector<std::uint8_t> tabs;
    for (std::size_t k = 0; k < n_pairs; ++k) {
        for (int side = 0; side < 2; ++side)
            for (const auto& s : shares) {
                auto b = B::canonical(side ? s.pairs[k].g.evals() : s.pairs[k].f.evals());
                tabs.insert(tabs.end(), b.begin(), b.end());
            }
    }
    B::Device& dev = B::device(cfg);
    const std::size_t vars = local_vars + index_vars;
    std::vector<std::uint8_t> out(64 + (vars + 2) * 4 * width + 2 * n_pairs * width);
    std::vector<char> js(1 << 16);
    std::size_t len = 0;
    dgkr_transcript t = B::load(transcript);
    B::check(dgkr_dist_sumcheck(dev.ctx(), dev.field(), n, n_pairs, vars, tabs.data(), &t, out.data(), out.size(),
                                &len, js.data(), js.size()));
    B::store(transcript, t);
    // the reference's messages, in its order (cluster.hpp:258-299)
    for (std::size_t i = 0; i < n; ++i) stats.record_message(i, topo.master, topo.master, width);
    for (std::size_t j = 0; j < local_vars; ++j) {
        for (std::size_t i = 0; i < n; ++i) stats.record_message(i, topo.master, topo.master, 4 * width);
        for (std::size_t i = 0; i < n; ++i) stats.record_message(topo.master, i, topo.master, width);
    }
    for (std::size_t i = 0; i < n; ++i) stats.record_message(i, topo.master, topo.master, 2 * n_pairs * width);
    return sumcheck::SumcheckProof::from_bytes(std::span<const std::uint8_t>(out.data(), len), cfg);
}

}  // namespace dgkr::cluster
