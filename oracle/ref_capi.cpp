// ORACLE TEST INFRASTRUCTURE — not product code.
//
// extern "C" wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/dgkr/*.hpp, compiled against the Boost shim in
// oracle/shim). Built by oracle/Makefile into oracle/_ref/libdgkr_ref.so. Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
// load it, as the checker and the CPU baseline — never as the product path.
//
// Conventions shared with the product C-ABI (include/dgkr_b200.h):
//  * field elements cross as canonical little-endian bytes of width
//    ceil(bits(p)/8) (field.hpp:159-187);
//  * a transcript is created as Transcript(label, cfg) followed by
//    absorb_u64(pre[i]) for each prefix word (the pattern every reference test
//    uses, e.g. tests/test_sumcheck.cpp:29-33);
//  * circuits use the flat CSR layout documented in include/dgkr_b200.h;
//  * GkrProof bytes use the layout documented there (the reference has no
//    GkrProof serializer; gkr.hpp:86-95).

#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "dgkr/circuit.hpp"
#include "dgkr/beacon.hpp"
#include "dgkr/cluster.hpp"
#include "dgkr/distinct.hpp"
#include "dgkr/field.hpp"
#include "dgkr/gkr.hpp"
#include "dgkr/pcs.hpp"
#include "dgkr/sumcheck.hpp"
#include "dgkr/transcript.hpp"

using namespace dgkr;

namespace {

thread_local std::string g_err;

enum Status { OK = 0, INVALID = 1, LOGIC = 2, DOMAIN = 3, RANGE = 4, OTHER = 5, CAPACITY = 6 };

template <class F>
int guard(F&& f) {
    try {
        return f();
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return INVALID;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return DOMAIN;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return RANGE;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return LOGIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return OTHER;
    }
}

FieldConfigPtr field_from(const std::uint8_t* mod, std::size_t len) {
    BigInt m = 0;
    boost::multiprecision::import_bits(m, mod, mod + len, 8, false);
    if (m == FieldConfig::bn254()->modulus()) return FieldConfig::bn254();
    if (m == FieldConfig::goldilocks()->modulus()) return FieldConfig::goldilocks();
    return FieldConfig::make_small_prime(m, "custom");
}

std::vector<FieldElement> read_elems(const std::uint8_t* p, std::size_t n, const FieldConfigPtr& cfg) {
    const std::size_t w = cfg->byte_width();
    std::vector<FieldElement> out;
    out.reserve(n);
    for (std::size_t i = 0; i < n; ++i) {
        out.push_back(FieldElement::from_bytes(std::span<const std::uint8_t>(p + i * w, w), cfg));
    }
    return out;
}

Transcript make_transcript(const char* label, const std::uint64_t* pre, std::size_t n_pre,
                           const FieldConfigPtr& cfg) {
    Transcript tr(label, cfg);
    for (std::size_t i = 0; i < n_pre; ++i) tr.absorb_u64(pre[i]);
    return tr;
}

int emit(const std::vector<std::uint8_t>& bytes, std::uint8_t* out, std::size_t cap, std::size_t* len) {
    *len = bytes.size();
    if (bytes.size() > cap) {
        g_err = "output buffer too small";
        return CAPACITY;
    }
    if (!bytes.empty()) std::memcpy(out, bytes.data(), bytes.size());
    return OK;
}

void put32(std::vector<std::uint8_t>& out, std::uint32_t v) {
    for (int i = 0; i < 4; ++i) out.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
}

circuit::GeneralCircuit build_circuit(std::uint32_t input_size, std::uint32_t depth,
                                      const std::uint64_t* layer_gate_start,
                                      const std::uint64_t* gate_nested_start,
                                      const std::uint32_t* nested, const std::uint64_t* min_padded) {
    std::vector<std::vector<circuit::AccumulationGate>> layers(depth);
    for (std::uint32_t li = 0; li < depth; ++li) {
        for (std::uint64_t g = layer_gate_start[li]; g < layer_gate_start[li + 1]; ++g) {
            circuit::AccumulationGate ag;
            for (std::uint64_t k = gate_nested_start[g]; k < gate_nested_start[g + 1]; ++k) {
                const std::uint32_t* e = nested + 5 * k;
                circuit::NestedGate ng;
                ng.kind = e[0] ? circuit::GateKind::mul : circuit::GateKind::add;
                ng.left = circuit::WireRef{e[1], e[2]};
                ng.right = circuit::WireRef{e[3], e[4]};
                ag.nested.push_back(ng);
            }
            layers[li].push_back(std::move(ag));
        }
    }
    circuit::GeneralCircuit c(input_size, std::move(layers));
    if (min_padded) {
        for (std::uint32_t l = 0; l <= depth; ++l) c.reserve_padding(l, min_padded[l]);
    }
    auto v = c.validate();
    if (!v.empty()) throw std::invalid_argument("invalid circuit: " + v.front());
    return c;
}

std::vector<std::uint8_t> gkr_proof_bytes(const gkr::GkrProof& p) {
    std::vector<std::uint8_t> out;
    put32(out, static_cast<std::uint32_t>(p.claimed_outputs.size()));
    for (const auto& e : p.claimed_outputs) e.append_bytes(out);
    put32(out, static_cast<std::uint32_t>(p.layers.size()));
    for (const auto& lp : p.layers) {
        put32(out, static_cast<std::uint32_t>(lp.alphas.size()));
        for (const auto& a : lp.alphas) a.append_bytes(out);
        auto sb = lp.sum.to_bytes();
        put32(out, static_cast<std::uint32_t>(sb.size()));
        out.insert(out.end(), sb.begin(), sb.end());
    }
    return out;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_field_width(const std::uint8_t* mod, std::size_t mod_len, std::size_t* width) {
    return guard([&] {
        *width = field_from(mod, mod_len)->byte_width();
        return OK;
    });
}

/// Transcript(label) + absorb_u64(pre...) ; then absorb each element in
/// `elems`, then draw n_chal challenges (written to chal_out); final state.
int ref_transcript_run(const std::uint8_t* mod, std::size_t mod_len, const char* label,
                       const std::uint64_t* pre, std::size_t n_pre, const std::uint8_t* elems,
                       std::size_t n_elems, std::size_t n_chal, std::uint8_t* chal_out,
                       std::size_t n_idx, std::uint64_t idx_bound, std::uint64_t* idx_out,
                       std::uint8_t* state_out) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        Transcript tr = make_transcript(label, pre, n_pre, cfg);
        for (const auto& e : read_elems(elems, n_elems, cfg)) tr.absorb(e);
        const std::size_t w = cfg->byte_width();
        for (std::size_t i = 0; i < n_chal; ++i) {
            auto b = tr.challenge().to_bytes();
            std::memcpy(chal_out + i * w, b.data(), w);
        }
        for (std::size_t i = 0; i < n_idx; ++i) idx_out[i] = tr.challenge_index(idx_bound);
        auto st = tr.state();
        std::memcpy(state_out, st.data(), 32);
        return OK;
    });
}

/// prove_product_sum (sumcheck.hpp:226). tables: pairs in order f0,g0,f1,g1..
/// each 2^vars elements.
int ref_prove_product_sum(const std::uint8_t* mod, std::size_t mod_len, const char* label,
                          const std::uint64_t* pre, std::size_t n_pre, std::size_t n_pairs,
                          std::size_t vars, const std::uint8_t* tables, std::uint8_t* proof_out,
                          std::size_t cap, std::size_t* proof_len, std::uint8_t* state_out) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        const std::size_t n = std::size_t{1} << vars;
        const std::size_t w = cfg->byte_width();
        std::vector<sumcheck::ProductPair> pairs;
        for (std::size_t k = 0; k < n_pairs; ++k) {
            auto f = read_elems(tables + (2 * k) * n * w, n, cfg);
            auto g = read_elems(tables + (2 * k + 1) * n * w, n, cfg);
            pairs.push_back(sumcheck::ProductPair{MultilinearTable(cfg, vars, std::move(f)),
                                                  MultilinearTable(cfg, vars, std::move(g))});
        }
        Transcript tr = make_transcript(label, pre, n_pre, cfg);
        auto proof = sumcheck::prove_product_sum(pairs, tr);
        auto st = tr.state();
        std::memcpy(state_out, st.data(), 32);
        return emit(proof.to_bytes(), proof_out, cap, proof_len);
    });
}

/// prove_layer_sum (sumcheck.hpp:342). wires: n_wires x {is_mul, x_slot,
/// y_slot} (u32) + x_index,y_index (u64) + weights (field bytes).
int ref_prove_layer_sum(const std::uint8_t* mod, std::size_t mod_len, const char* label,
                        const std::uint64_t* pre, std::size_t n_pre, std::size_t side_vars,
                        std::size_t n_slots, const std::uint8_t* slot_tables, std::size_t n_wires,
                        const std::uint32_t* wire_meta, const std::uint64_t* wire_idx,
                        const std::uint8_t* wire_weights, const std::uint8_t* claimed,
                        std::uint8_t* proof_out, std::size_t cap, std::size_t* proof_len,
                        std::uint8_t* state_out) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        const std::size_t n = std::size_t{1} << side_vars;
        const std::size_t w = cfg->byte_width();
        sumcheck::LayerInstance inst;
        inst.side_vars = side_vars;
        for (std::size_t m = 0; m < n_slots; ++m) {
            inst.slot_tables.emplace_back(cfg, side_vars, read_elems(slot_tables + m * n * w, n, cfg));
        }
        auto weights = read_elems(wire_weights, n_wires, cfg);
        for (std::size_t i = 0; i < n_wires; ++i) {
            sumcheck::LayerWire lw;
            lw.is_mul = wire_meta[3 * i] != 0;
            lw.x_slot = wire_meta[3 * i + 1];
            lw.y_slot = wire_meta[3 * i + 2];
            lw.x_index = wire_idx[2 * i];
            lw.y_index = wire_idx[2 * i + 1];
            lw.weight = weights[i];
            inst.wires.push_back(lw);
        }
        auto cl = read_elems(claimed, 1, cfg).front();
        Transcript tr = make_transcript(label, pre, n_pre, cfg);
        auto res = sumcheck::prove_layer_sum(inst, cl, tr);
        auto st = tr.state();
        std::memcpy(state_out, st.data(), 32);
        return emit(res.proof.to_bytes(), proof_out, cap, proof_len);
    });
}

/// gkr_prove (gkr.hpp:182) on a flat circuit; proof in the GkrProof layout.
int ref_gkr_prove(const std::uint8_t* mod, std::size_t mod_len, const char* label,
                  const std::uint64_t* pre, std::size_t n_pre, std::uint32_t input_size,
                  std::uint32_t depth, const std::uint64_t* layer_gate_start,
                  const std::uint64_t* gate_nested_start, const std::uint32_t* nested,
                  const std::uint64_t* min_padded, const std::uint8_t* inputs,
                  std::uint8_t* proof_out, std::size_t cap, std::size_t* proof_len,
                  std::uint8_t* state_out) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        auto c = build_circuit(input_size, depth, layer_gate_start, gate_nested_start, nested, min_padded);
        auto in = read_elems(inputs, input_size, cfg);
        Transcript tr = make_transcript(label, pre, n_pre, cfg);
        auto proof = gkr::gkr_prove(c, in, cfg, tr);
        auto st = tr.state();
        std::memcpy(state_out, st.data(), 32);
        return emit(gkr_proof_bytes(proof), proof_out, cap, proof_len);
    });
}

/// gkr_verify + check_input_claims on the proof bytes emitted above. Returns
/// OK and *accept in {0,1}.
int ref_gkr_verify(const std::uint8_t* mod, std::size_t mod_len, const char* label,
                   const std::uint64_t* pre, std::size_t n_pre, std::uint32_t input_size,
                   std::uint32_t depth, const std::uint64_t* layer_gate_start,
                   const std::uint64_t* gate_nested_start, const std::uint32_t* nested,
                   const std::uint64_t* min_padded, const std::uint8_t* inputs,
                   const std::uint8_t* proof, std::size_t proof_len, int* accept) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        const std::size_t w = cfg->byte_width();
        auto c = build_circuit(input_size, depth, layer_gate_start, gate_nested_start, nested, min_padded);
        std::size_t pos = 0;
        auto take32 = [&]() {
            if (pos + 4 > proof_len) throw std::invalid_argument("truncated gkr proof");
            std::uint32_t v = 0;
            for (int i = 3; i >= 0; --i) v = (v << 8) | proof[pos + static_cast<std::size_t>(i)];
            pos += 4;
            return v;
        };
        auto take_elem = [&]() {
            if (pos + w > proof_len) throw std::invalid_argument("truncated gkr proof");
            auto e = FieldElement::from_bytes(std::span<const std::uint8_t>(proof + pos, w), cfg);
            pos += w;
            return e;
        };
        gkr::GkrProof p;
        const std::uint32_t n_out = take32();
        for (std::uint32_t i = 0; i < n_out; ++i) p.claimed_outputs.push_back(take_elem());
        const std::uint32_t n_layers = take32();
        for (std::uint32_t l = 0; l < n_layers; ++l) {
            gkr::GkrLayerProof lp;
            const std::uint32_t na = take32();
            for (std::uint32_t i = 0; i < na; ++i) lp.alphas.push_back(take_elem());
            const std::uint32_t sl = take32();
            if (pos + sl > proof_len) throw std::invalid_argument("truncated gkr proof");
            lp.sum = sumcheck::SumcheckProof::from_bytes(std::span<const std::uint8_t>(proof + pos, sl), cfg);
            pos += sl;
            p.layers.push_back(std::move(lp));
        }
        auto in = read_elems(inputs, input_size, cfg);
        auto outputs = c.outputs(in, cfg);
        Transcript tr = make_transcript(label, pre, n_pre, cfg);
        auto res = gkr::gkr_verify(c, outputs, p, cfg, tr);
        bool ok = res.accept;
        if (ok) {
            std::vector<FieldElement> padded = in;
            padded.resize(c.padded_size(0), FieldElement::zero(cfg));
            MultilinearTable table(cfg, c.padded_log2(0), padded);
            ok = gkr::check_input_claims(res.input_claims, table);
        }
        *accept = ok ? 1 : 0;
        return OK;
    });
}

/// circuit::random_general_circuit (circuit.hpp:342) seeded with
/// std::mt19937_64(seed), exported in the flat layout. Buffers must be large
/// enough for depth*max_gates gates and depth*max_gates*max_nested entries.
int ref_random_general_circuit(std::uint64_t seed, std::size_t input_size, std::size_t depth,
                               std::size_t max_gates, std::size_t max_nested, unsigned mul_percent,
                               std::uint64_t* layer_gate_start, std::uint64_t* gate_nested_start,
                               std::uint32_t* nested, std::uint64_t* n_gates_out,
                               std::uint64_t* n_nested_out) {
    return guard([&] {
        std::mt19937_64 rng(seed);
        circuit::RandomCircuitParams p;
        p.input_size = input_size;
        p.depth = depth;
        p.max_gates_per_layer = max_gates;
        p.max_nested = max_nested;
        p.mul_percent = mul_percent;
        auto c = circuit::random_general_circuit(rng, p);
        std::uint64_t g = 0, k = 0;
        layer_gate_start[0] = 0;
        gate_nested_start[0] = 0;
        for (std::size_t li = 1; li <= c.depth(); ++li) {
            for (const auto& gate : c.gates(li)) {
                for (const auto& ng : gate.nested) {
                    std::uint32_t* e = nested + 5 * k;
                    e[0] = ng.kind == circuit::GateKind::mul ? 1u : 0u;
                    e[1] = ng.left.layer;
                    e[2] = ng.left.gate;
                    e[3] = ng.right.layer;
                    e[4] = ng.right.gate;
                    ++k;
                }
                ++g;
                gate_nested_start[g] = k;
            }
            layer_gate_start[li] = g;
        }
        *n_gates_out = g;
        *n_nested_out = k;
        return OK;
    });
}

/// pcs::commit (pcs.hpp:105): root of the rows x cols matrix (row-major).
int ref_pcs_commit(const std::uint8_t* mod, std::size_t mod_len, std::size_t rows, std::size_t cols,
                   const std::uint8_t* data, std::uint8_t* root_out) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        pcs::EvalMatrix m(cfg, rows, cols, read_elems(data, rows * cols, cfg));
        auto com = pcs::commit(m);
        std::memcpy(root_out, com.root.data(), 32);
        return OK;
    });
}

/// pcs::open (pcs.hpp:212) -> Opening::to_bytes.
int ref_pcs_open(const std::uint8_t* mod, std::size_t mod_len, const char* label,
                 const std::uint64_t* pre, std::size_t n_pre, std::size_t rows, std::size_t cols,
                 const std::uint8_t* data, const std::uint8_t* r, std::size_t r_len, std::size_t q,
                 std::uint8_t* out, std::size_t cap, std::size_t* out_len, std::uint8_t* state_out) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        pcs::EvalMatrix m(cfg, rows, cols, read_elems(data, rows * cols, cfg));
        auto point = read_elems(r, r_len, cfg);
        Transcript tr = make_transcript(label, pre, n_pre, cfg);
        auto op = pcs::open(m, point, tr, q);
        auto st = tr.state();
        std::memcpy(state_out, st.data(), 32);
        return emit(op.to_bytes(), out, cap, out_len);
    });
}

/// pcs::verify_open (pcs.hpp:256) on a fresh commit of `data` and an opening
/// given in Opening::to_bytes layout. *accept in {0,1}.
int ref_pcs_verify(const std::uint8_t* mod, std::size_t mod_len, const char* label,
                   const std::uint64_t* pre, std::size_t n_pre, std::size_t rows, std::size_t cols,
                   const std::uint8_t* root, const std::uint8_t* r, std::size_t r_len,
                   const std::uint8_t* op_bytes, std::size_t op_len, std::size_t q, int* accept) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        const std::size_t w = cfg->byte_width();
        pcs::Commitment com;
        std::memcpy(com.root.data(), root, 32);
        com.rows = rows;
        com.cols = cols;
        std::size_t pos = 0;
        auto take32 = [&]() {
            if (pos + 4 > op_len) throw std::invalid_argument("truncated opening");
            std::uint32_t v = 0;
            for (int i = 3; i >= 0; --i) v = (v << 8) | op_bytes[pos + static_cast<std::size_t>(i)];
            pos += 4;
            return v;
        };
        auto take_elem = [&]() {
            if (pos + w > op_len) throw std::invalid_argument("truncated opening");
            auto e = FieldElement::from_bytes(std::span<const std::uint8_t>(op_bytes + pos, w), cfg);
            pos += w;
            return e;
        };
        pcs::Opening op;
        std::uint32_t n = take32();
        for (std::uint32_t i = 0; i < n; ++i) op.point.push_back(take_elem());
        op.value = take_elem();
        n = take32();
        for (std::uint32_t i = 0; i < n; ++i) op.row_evals.push_back(take_elem());
        n = take32();
        for (std::uint32_t i = 0; i < n; ++i) op.combined_row.push_back(take_elem());
        n = take32();
        for (std::uint32_t k = 0; k < n; ++k) {
            op.spot_indices.push_back(take32());
            std::vector<FieldElement> col;
            for (std::size_t i = 0; i < rows; ++i) col.push_back(take_elem());
            op.spot_columns.push_back(std::move(col));
            std::size_t depth = 0;
            while ((std::size_t{1} << depth) < cols) ++depth;
            std::vector<Digest> path(depth);
            for (auto& d : path) {
                if (pos + 32 > op_len) throw std::invalid_argument("truncated opening");
                std::memcpy(d.data(), op_bytes + pos, 32);
                pos += 32;
            }
            op.spot_paths.push_back(std::move(path));
        }
        auto point = read_elems(r, r_len, cfg);
        Transcript tr = make_transcript(label, pre, n_pre, cfg);
        *accept = pcs::verify_open(com, point, op, tr, cfg, q) ? 1 : 0;
        return OK;
    });
}

/// cluster::shard_pairs + dist_sumcheck (cluster.hpp:190, :228). tables are
/// the FULL pairs (f0,g0,f1,g1,... each 2^vars). Also returns
/// TrafficStats::to_json().dump() (phase "sumcheck").
int ref_dist_sumcheck(const std::uint8_t* mod, std::size_t mod_len, const char* label,
                      const std::uint64_t* pre, std::size_t n_pre, std::size_t n_workers,
                      std::size_t n_pairs, std::size_t vars, const std::uint8_t* tables,
                      std::uint8_t* proof_out, std::size_t cap, std::size_t* proof_len,
                      std::uint8_t* state_out, char* traffic_json, std::size_t json_cap) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        const std::size_t n = std::size_t{1} << vars;
        const std::size_t w = cfg->byte_width();
        std::vector<sumcheck::ProductPair> pairs;
        for (std::size_t k = 0; k < n_pairs; ++k) {
            auto f = read_elems(tables + (2 * k) * n * w, n, cfg);
            auto g = read_elems(tables + (2 * k + 1) * n * w, n, cfg);
            pairs.push_back(sumcheck::ProductPair{MultilinearTable(cfg, vars, std::move(f)),
                                                  MultilinearTable(cfg, vars, std::move(g))});
        }
        auto shares = cluster::shard_pairs(pairs, n_workers);
        auto topo = cluster::ClusterTopology::plan(n_workers);
        cluster::TrafficStats stats;
        stats.begin_phase("sumcheck");
        Transcript tr = make_transcript(label, pre, n_pre, cfg);
        auto proof = cluster::dist_sumcheck(topo, shares, tr, stats);
        auto st = tr.state();
        std::memcpy(state_out, st.data(), 32);
        const std::string js = stats.to_json().dump();
        if (js.size() + 1 > json_cap) throw std::invalid_argument("json buffer too small");
        std::memcpy(traffic_json, js.c_str(), js.size() + 1);
        return emit(proof.to_bytes(), proof_out, cap, proof_len);
    });
}

/// cluster::DistPc commit + open (cluster.hpp:336, :386). rows: n_workers rows
/// of 2^row_vars elements. Outputs K roots (32 B each), the concatenated
/// cluster Opening::to_bytes (each prefixed by u32 length), the combined
/// value, and TrafficStats json (phases "commit" and "open").
int ref_distpc(const std::uint8_t* mod, std::size_t mod_len, std::size_t n_workers,
               std::size_t n_clusters, std::size_t row_vars, const std::uint8_t* rows,
               const std::uint8_t* r, std::size_t r_len, std::size_t q, std::uint8_t* roots_out,
               std::size_t* n_roots, std::uint8_t* open_out, std::size_t cap, std::size_t* open_len,
               std::uint8_t* combined_out, char* traffic_json, std::size_t json_cap) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        const std::size_t n = std::size_t{1} << row_vars;
        const std::size_t w = cfg->byte_width();
        std::vector<MultilinearTable> tabs;
        for (std::size_t i = 0; i < n_workers; ++i) {
            tabs.emplace_back(cfg, row_vars, read_elems(rows + i * n * w, n, cfg));
        }
        auto topo = n_clusters ? cluster::ClusterTopology::plan(n_workers, n_clusters)
                               : cluster::ClusterTopology::plan(n_workers);
        cluster::DistPc pc(topo, cfg);
        cluster::TrafficStats stats;
        stats.begin_phase("commit");
        auto coms = pc.commit(tabs, stats);
        *n_roots = coms.size();
        for (std::size_t c = 0; c < coms.size(); ++c) std::memcpy(roots_out + 32 * c, coms[c].root.data(), 32);
        stats.begin_phase("open");
        auto point = read_elems(r, r_len, cfg);
        auto op = pc.open(point, stats, q);
        std::vector<std::uint8_t> bytes;
        for (const auto& o : op.cluster_openings) {
            auto b = o.to_bytes();
            put32(bytes, static_cast<std::uint32_t>(b.size()));
            bytes.insert(bytes.end(), b.begin(), b.end());
        }
        auto cb = op.combined_value.to_bytes();
        std::memcpy(combined_out, cb.data(), w);
        const std::string js = stats.to_json().dump();
        if (js.size() + 1 > json_cap) throw std::invalid_argument("json buffer too small");
        std::memcpy(traffic_json, js.c_str(), js.size() + 1);
        return emit(bytes, open_out, cap, open_len);
    });
}

/// GeneralCircuit::to_json (circuit.hpp:227-248) of a flat circuit, dumped
/// compactly; from_json (:250-277) round trip checked by re-dumping.
int ref_circuit_json(std::uint32_t input_size, std::uint32_t depth, const std::uint64_t* layer_gate_start,
                     const std::uint64_t* gate_nested_start, const std::uint32_t* nested, char* out, std::size_t cap,
                     std::size_t* len) {
    return guard([&] {
        auto c = build_circuit(input_size, depth, layer_gate_start, gate_nested_start, nested, nullptr);
        const std::string js = c.to_json().dump();
        auto c2 = circuit::GeneralCircuit::from_json(nlohmann::json::parse(js));
        if (c2.to_json().dump() != js) throw std::logic_error("from_json/to_json round trip differs");
        *len = js.size();
        if (js.size() + 1 > cap) {
            g_err = "output buffer too small";
            return static_cast<int>(CAPACITY);
        }
        std::memcpy(out, js.c_str(), js.size() + 1);
        return static_cast<int>(OK);
    });
}

// --- beacon.hpp (config C3); records cross as ValidatorRecord::encode() ---
namespace {
std::vector<beacon::ValidatorRecord> decode_records(const std::uint8_t* recs, std::size_t n) {
    std::vector<beacon::ValidatorRecord> out(n);
    for (std::size_t i = 0; i < n; ++i) {
        const std::uint8_t* q = recs + 64 * i;
        std::copy(q, q + 48, out[i].pubkey.begin());
        std::uint64_t idx = 0;
        for (int b = 0; b < 8; ++b) idx |= static_cast<std::uint64_t>(q[48 + b]) << (8 * b);
        out[i].index = idx;
        out[i].active = q[56] != 0;
    }
    return out;
}
}  // namespace

int ref_beacon_gen(std::size_t n, std::uint64_t seed, std::uint8_t* recs) {
    return guard([&] {
        auto v = beacon::gen_validators(n, seed);
        for (std::size_t i = 0; i < n; ++i) {
            auto e = v[i].encode();
            std::memcpy(recs + 64 * i, e.data(), 64);
        }
        return static_cast<int>(OK);
    });
}

int ref_beacon_root(const std::uint8_t* recs, std::size_t n, std::size_t depth, std::uint8_t* root) {
    return guard([&] {
        auto v = decode_records(recs, n);
        beacon::BeaconTree t(v, depth);
        std::memcpy(root, t.root().data(), 32);
        return static_cast<int>(OK);
    });
}

int ref_beacon_prove(const std::uint8_t* recs, std::size_t n, std::size_t depth, std::uint64_t index,
                     std::uint8_t* leaf, std::uint8_t* siblings, std::size_t* active_log2) {
    return guard([&] {
        auto v = decode_records(recs, n);
        beacon::BeaconTree t(v, depth);
        auto p = t.prove_membership(index);
        std::memcpy(leaf, p.leaf.data(), 32);
        for (std::size_t k = 0; k < p.siblings.size(); ++k) std::memcpy(siblings + 32 * k, p.siblings[k].data(), 32);
        *active_log2 = p.active_log2;
        return static_cast<int>(OK);
    });
}

int ref_beacon_verify(const std::uint8_t* root, const std::uint8_t* rec, const std::uint8_t* leaf,
                      const std::uint8_t* siblings, std::size_t active_log2, std::uint64_t index, std::size_t depth,
                      int* ok) {
    return guard([&] {
        auto r = decode_records(rec, 1)[0];
        beacon::MembershipPath p;
        std::memcpy(p.leaf.data(), leaf, 32);
        for (std::size_t k = 0; k < active_log2; ++k) {
            Digest d;
            std::memcpy(d.data(), siblings + 32 * k, 32);
            p.siblings.push_back(d);
        }
        p.index = index;
        p.depth = depth;
        p.active_log2 = active_log2;
        Digest rt;
        std::memcpy(rt.data(), root, 32);
        *ok = beacon::BeaconTree::verify_membership(rt, r, p) ? 1 : 0;
        return static_cast<int>(OK);
    });
}

/// distinct::ah (distinct.hpp:37-44)
int ref_distinct_ah(const std::uint8_t* mod, std::size_t mod_len, const std::uint8_t* items, std::size_t n,
                    std::uint8_t* out) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        auto v = read_elems(items, n, cfg);
        auto b = distinct::ah(std::span<const FieldElement>(v), cfg).to_bytes();
        std::memcpy(out, b.data(), b.size());
        return OK;
    });
}

/// distinct::pairwise_distinct_check (distinct.hpp:53-68)
int ref_distinct_check(const std::uint8_t* mod, std::size_t mod_len, const std::uint8_t* a, std::size_t n_a,
                       const std::uint8_t* a_sorted, std::size_t n_sorted, int* ok) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        auto va = read_elems(a, n_a, cfg);
        auto vs = read_elems(a_sorted, n_sorted, cfg);
        *ok = distinct::pairwise_distinct_check(va, vs, cfg) ? 1 : 0;
        return OK;
    });
}

/// distinct::chain_update (distinct.hpp:82-92)
int ref_distinct_chain_update(const std::uint8_t* mod, std::size_t mod_len, const std::uint8_t* h,
                              std::uint64_t n_max, const std::uint8_t* items, std::size_t n, std::uint8_t* h_out) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        distinct::ChainState st{read_elems(h, 1, cfg)[0], n_max};
        distinct::IndexList block{cfg, read_elems(items, n, cfg), n_max};
        auto b = distinct::chain_update(st, block).h.to_bytes();
        std::memcpy(h_out, b.data(), b.size());
        return OK;
    });
}

/// distinct::bitchange_experiment (distinct.hpp:112-145): per-bit set counts
int ref_distinct_bitchange(const std::uint8_t* mod, std::size_t mod_len, std::size_t count, std::uint64_t* set_counts,
                           std::size_t* bits) {
    return guard([&] {
        auto cfg = field_from(mod, mod_len);
        auto res = distinct::bitchange_experiment(count, cfg);
        *bits = res.probabilities.size();
        for (std::size_t k = 0; k < res.probabilities.size(); ++k)
            set_counts[k] = static_cast<std::uint64_t>(res.probabilities[k] * static_cast<double>(count) + 0.5);
        return OK;
    });
}

}  // extern "C"
