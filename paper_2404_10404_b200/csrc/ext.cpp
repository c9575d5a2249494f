// C ABI beyond the GKR prover: distinct.hpp (AH, pairwise-distinct check,
// chain update, bit-change experiment; config C4), beacon.hpp (validator
// tree, membership paths; config C3), and Reed-Solomon / NTT / FRI
// (north-star "Virgo/FRI"; no reference exists).
#include <cstring>
#include <memory>
#include <vector>

#include <string>
#include <thread>

#include "comm.hpp"
#include "dgkr_b200.h"
#include "host_core.hpp"
#include "kernels.hpp"
#include "runtime.hpp"

namespace {

// ---------------------------------------------------------------------------
// Reed-Solomon / NTT / FRI (north-star "Virgo/FRI"; no reference exists, see
// pinned by the Python restatement oracle/fri_oracle.py).
// ---------------------------------------------------------------------------
void pow_table(Lane* ctx, const dgkr_field* f, const U256& base, std::uint64_t n, Fe* out, DBuf<Fe>& scratch) {
    std::uint64_t na = 1;
    while (na * na < n) na <<= 1;
    scratch.ensure(na + n / na + 2);
    launch_pow_table(ctx->use(f), to_fe(base), n, out, scratch.p, ctx->st);
    ctx->launched(2);
}

/// evaluations (natural order) on c * <w_N> of the polynomial with
/// coefficients `coeff` (n_in <= N entries, rest zero): a := NTT(coset-scaled, bit-reversed coeff)
void coset_ntt(Lane* ctx, const dgkr_field* f, const Fe* coeff, std::uint64_t n_in, unsigned log_n, const U256& c,
               bool apply_coset, Fe* a, DBuf<Fe>& tw, DBuf<Fe>& cpow, DBuf<Fe>& scratch) {
    const FieldKind kind = ctx->use(f);
    const std::uint64_t N = std::uint64_t{1} << log_n;
    const U256 w = f->root_of_unity(log_n);
    tw.ensure(std::max<std::uint64_t>(N / 2, 1));
    if (N >= 2) pow_table(ctx, f, w, N / 2, tw.p, scratch);
    const Fe* scale = nullptr;
    if (apply_coset) {
        cpow.ensure(n_in);
        pow_table(ctx, f, c, n_in, cpow.p, scratch);
        scale = cpow.p;
    }
    ctx->tbeg();
    launch_bitrev_scale(kind, coeff, scale, a, static_cast<int>(log_n), n_in, ctx->st);
    launch_ntt(kind, a, static_cast<int>(log_n), tw.p, ctx->st);
    ctx->tend(ctx->prof.ntt_ms);
    ctx->launched(1 + ntt_launches(static_cast<int>(log_n)));  // bit-reverse/scale + the transform
}

/// FRI over the RS codeword of `coeffs` (protocol in include/dgkr_b200.h)
/// comm != nullptr: distributed FRI: this rank folds its own
/// chunk; per layer every rank's root is all-gathered and absorbed in rank
/// order (one shared beta), the final layers likewise, the query positions
/// are shared, and the proof carries every rank's roots and final layer plus
/// this rank's openings (format in include/dgkr_b200.h).
std::vector<std::uint8_t> fri_prove(Lane* ctx, const dgkr_field* f, const std::uint8_t* coeffs, std::uint64_t n,
                                    unsigned blowup_log, unsigned final_log, std::size_t q, Transcript& tr,
                                    dgkr_comm* comm = nullptr) {
    const std::size_t world = comm ? static_cast<std::size_t>(comm->world) : 1;
    const HostField& F = f->f;
    const FieldKind kind = ctx->use(f);
    const std::size_t w = F.width();
    if (n == 0 || (n & (n - 1)) != 0) fail(DGKR_INVALID_ARGUMENT, "coefficient count must be a power of two");
    const unsigned log_n0 = log2_exact(n) + blowup_log;
    if (final_log > log_n0) fail(DGKR_INVALID_ARGUMENT, "final layer larger than the codeword");
    const unsigned L = log_n0 - final_log;
    const std::uint64_t N0 = std::uint64_t{1} << log_n0;
    NttWs& ws = ctx->nttws();
    auto& stage = ws.stage;
    auto& cf = ws.x;
    auto& tw = ws.tw;
    auto& cpow = ws.cpow;
    auto& scratch = ws.scratch;
    auto& twinv = ws.twinv;
    cf.ensure(n);
    ctx->upload_elems(f, coeffs, n, cf.p, stage);
    // layer 0: RS encoding on the coset g<w_N0>
    auto& layer = ws.layer;
    auto& tree = ws.tree;
    if (layer.size() < L + 1) layer.resize(L + 1);
    if (tree.size() < L) tree.resize(L);
    for (unsigned l = 0; l <= L; ++l) {
        if (!layer[l]) layer[l] = std::make_unique<DBuf<Fe>>();
        layer[l]->ensure(N0 >> l);
    }
    coset_ntt(ctx, f, cf.p, n, log_n0, f->coset, true, layer[0]->p, tw, cpow, scratch);
    // inverse twiddles w^-i for the fold's 1/x
    twinv.ensure(std::max<std::uint64_t>(N0 / 2, 1));
    if (N0 >= 2) pow_table(ctx, f, F.inv(f->root_of_unity(log_n0)), N0 / 2, twinv.p, scratch);
    std::vector<Digest> roots(L);
    std::vector<std::uint8_t> all_roots;  // distributed: L x world roots, layer-major, rank order
    U256 ginv = f->coset_inv;  // (g^(2^l))^-1
    for (unsigned l = 0; l < L; ++l) {
        const std::uint64_t Nl = N0 >> l;
        if (!tree[l]) tree[l] = std::make_unique<DBuf<std::uint8_t>>();
        tree[l]->ensure(2 * Nl * 32);
        ctx->tbeg();
        launch_column_digests(kind, layer[l]->p, Nl, 1, static_cast<int>(w), tree[l]->p + Nl * 32, ctx->st);
        launch_merkle(tree[l]->p, Nl, ctx->st);
        ctx->tend(ctx->prof.merkle_ms);
        ctx->launched(2);
        ctx->d2h(roots[l].data(), tree[l]->p + 32, 32);
        ctx->sync();
        if (comm) {
            std::vector<std::uint8_t> rl(world * 32);
            comm->allgather_to_host(tree[l]->p + 32, rl.data(), 32, ctx);
            for (std::size_t r = 0; r < world; ++r) tr.absorb_bytes(rl.data() + 32 * r, 32);
            all_roots.insert(all_roots.end(), rl.begin(), rl.end());
        } else {
            tr.absorb_bytes(roots[l].data(), 32);
        }
        const U256 beta = tr.challenge();
        U256 bk[9];
        f->fold_const(beta, bk);
        Fe gi = to_fe(ginv);
        ctx->tbeg();
        launch_fri_fold(kind, layer[l]->p, Nl, twinv.p, std::uint64_t{1} << l, &gi, bk, layer[l + 1]->p, ctx->st);
        ctx->tend(ctx->prof.fold_ms);
        ctx->launched();
        ginv = F.mul(ginv, ginv);
    }
    // final layer, absorbed element by element
    const std::uint64_t NL = N0 >> L;
    std::vector<std::uint8_t> fin(NL * w);
    stage.ensure(NL * w);
    launch_to_canonical(kind, layer[L]->p, stage.p, static_cast<int>(w), NL, ctx->st);
    ctx->d2h(fin.data(), stage.p, NL * w);
    ctx->sync();
    std::vector<std::uint8_t> all_fin;  // distributed: world final layers, rank order
    if (comm) {
        all_fin.resize(world * NL * w);
        comm->allgather_to_host(stage.p, all_fin.data(), NL * w, ctx);
        tr.absorb_many(all_fin.data(), world * NL, w);
    } else {
        tr.absorb_many(fin.data(), NL, w);
    }
    // queries on the first layer's half domain (distinct, like pcs.hpp:199-206)
    const std::uint64_t H = N0 / 2;
    std::vector<std::uint64_t> qi;
    if (L > 0) {
        if (q >= H) {
            for (std::uint64_t i = 0; i < H; ++i) qi.push_back(i);
        } else {
            std::vector<bool> seen(H, false);
            while (qi.size() < q) {
                const std::uint64_t j = tr.challenge_index(H);
                if (!seen[j]) {
                    seen[j] = true;
                    qi.push_back(j);
                }
            }
        }
    }
    // gather opened values and Merkle paths on the device, one D2H per layer
    std::vector<std::uint8_t> out;
    if (comm) {
        put32(out, static_cast<std::uint32_t>(world));
        put32(out, static_cast<std::uint32_t>(comm->rank));
        put32(out, L);
        out.insert(out.end(), all_roots.begin(), all_roots.end());
        put32(out, static_cast<std::uint32_t>(NL));
        out.insert(out.end(), all_fin.begin(), all_fin.end());
    } else {
        put32(out, L);
        for (const auto& r : roots) out.insert(out.end(), r.begin(), r.end());
        put32(out, static_cast<std::uint32_t>(NL));
        out.insert(out.end(), fin.begin(), fin.end());
    }
    put32(out, static_cast<std::uint32_t>(qi.size()));
    std::vector<std::vector<std::uint8_t>> vals(L), paths(L);
    std::vector<unsigned> depth(L);
    auto& didx = ws.didx;
    auto& dbuf = ws.dbuf;
    for (unsigned l = 0; l < L; ++l) {
        const std::uint64_t Nl = N0 >> l, hl = Nl / 2;
        depth[l] = log2_exact(Nl);
        std::vector<std::uint64_t> vidx, pidx;
        for (std::uint64_t i : qi) {
            const std::uint64_t il = i % hl;
            vidx.push_back(il);
            vidx.push_back(il + hl);
            for (std::uint64_t leaf : {il, il + hl}) {
                std::uint64_t node = Nl + leaf;
                while (node > 1) {
                    pidx.push_back(node ^ 1);
                    node >>= 1;
                }
            }
        }
        const std::size_t nv = vidx.size(), np = pidx.size();
        didx.ensure(nv + np);
        dbuf.ensure((nv + np) * 32 + nv * w + 32);
        ctx->h2d(didx.p, vidx.data(), nv * 8);
        if (np) ctx->h2d(didx.p + nv, pidx.data(), np * 8);
        launch_gather32(layer[l]->p, didx.p, nv, dbuf.p, ctx->st);
        launch_to_canonical(kind, reinterpret_cast<const Fe*>(dbuf.p), dbuf.p + (nv + np) * 32, static_cast<int>(w), nv,
                            ctx->st);
        launch_gather32(tree[l]->p, didx.p + nv, np, dbuf.p + nv * 32, ctx->st);
        ctx->launched(3);
        vals[l].resize(nv * w);
        paths[l].resize(np * 32);
        ctx->d2h(vals[l].data(), dbuf.p + (nv + np) * 32, nv * w);
        if (np) ctx->d2h(paths[l].data(), dbuf.p + nv * 32, np * 32);
    }
    ctx->sync();
    for (std::size_t k = 0; k < qi.size(); ++k) {
        put32(out, static_cast<std::uint32_t>(qi[k]));
        for (unsigned l = 0; l < L; ++l) {
            const std::uint8_t* v = vals[l].data() + 2 * k * w;
            out.insert(out.end(), v, v + 2 * w);
            const std::uint8_t* pth = paths[l].data() + 2 * k * depth[l] * 32;
            out.insert(out.end(), pth, pth + 2 * depth[l] * 32);
        }
    }
    return out;
}

}  // namespace

int dgkr_field_ntt_info(const dgkr_field* f, unsigned* two_adicity, std::uint8_t* root, std::uint8_t* coset) {
    return guard([&] {
        *two_adicity = f->two_adicity;
        if (root) f->f.to_bytes(f->root, root);
        if (coset) f->f.to_bytes(f->coset, coset);
    });
}

// ---------------------------------------------------------------------------
// distinct.hpp (config C4): AH, pairwise-distinct check, chain update,
// bit-change experiment. One host sync per call: the encoding error flag, the
// predicate flags and the sums come back in one pinned read.
// ---------------------------------------------------------------------------
namespace {

struct AhPass {
    std::uint64_t n = 0;
    Fe* x = nullptr;
    const std::uint8_t* canon = nullptr;  // device canonical bytes
};

/// upload + validate + AH of one list; the sum lands in h_small[slot] after sync
AhPass ah_enqueue(Lane* ctx, const dgkr_field* f, const std::uint8_t* items, std::uint64_t n, DBuf<std::uint8_t>& stage,
                  DBuf<Fe>& x, int slot) {
    const FieldKind kind = ctx->use(f);
    const std::size_t w = f->f.width();
    AhPass a;
    a.n = n;
    x.ensure(std::max<std::uint64_t>(n, 1));
    stage.ensure(std::max<std::size_t>(n * w, 1));
    if (n) {
        ctx->h2d_large(stage.p, items, n * w);
        launch_from_canonical(kind, stage.p, static_cast<int>(w), x.p, n, ctx->d_err.p, ctx->st);
        ctx->launched();
    }
    const U256 off = f->f.from_u64(4294967295ull);  // distinct.hpp:20
    Fe offe = to_fe(off);
    launch_ah(kind, x.p, n, &offe, ctx->ws, ctx->st);
    ctx->launched();
    ctx->d2h(ctx->h_small + slot, ctx->ws.result, sizeof(Fe));
    a.x = x.p;
    a.canon = stage.p;
    return a;
}

/// read back error + flags (ints at h_small[kGatherOff]) with one sync
void distinct_finish(Lane* ctx, int* flags_out) {
    int* hf = reinterpret_cast<int*>(ctx->h_small + Lane::kGatherOff);
    ctx->d2h(hf, ctx->d_err.p, sizeof(int));
    ctx->d2h(hf + 1, ctx->d_flag.p, 2 * sizeof(int));
    ctx->sync();
    if (hf[0]) {
        CK(cudaMemsetAsync(ctx->d_err.p, 0, sizeof(int), ctx->st));
        fail(DGKR_INVALID_ARGUMENT, "non-canonical field element encoding (index list)");
    }
    if (flags_out) {
        flags_out[0] = hf[1];
        flags_out[1] = hf[2];
    }
}

}  // namespace

int dgkr_distinct_ah(dgkr_ctx* ctx, const dgkr_field* f, const std::uint8_t* items, std::size_t n,
                     std::uint8_t* out) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        NttWs& ws = ctx->nttws();
        CK(cudaMemsetAsync(ctx->d_flag.p, 0, 2 * sizeof(int), ctx->st));
        ah_enqueue(ctx, f, items, n, ws.stage, ws.x, 1);
        distinct_finish(ctx, nullptr);
        f->f.to_bytes(to_u256(ctx->h_small[1]), out);
        ctx->end_call();
    });
}

int dgkr_distinct_check(dgkr_ctx* ctx, const dgkr_field* f, const std::uint8_t* a, std::size_t n_a,
                        const std::uint8_t* a_sorted, std::size_t n_sorted, int* ok) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        NttWs& ws = ctx->nttws();
        CK(cudaMemsetAsync(ctx->d_flag.p, 0, 2 * sizeof(int), ctx->st));
        ah_enqueue(ctx, f, a, n_a, ws.stage, ws.x, 1);
        AhPass s = ah_enqueue(ctx, f, a_sorted, n_sorted, ws.dbuf, ws.a, 2);
        launch_strict_ascent(s.canon, static_cast<int>(f->f.width()), n_sorted, ctx->d_flag.p, ctx->st);
        ctx->launched();
        int flags[2];
        distinct_finish(ctx, flags);
        const bool same = std::memcmp(&ctx->h_small[1], &ctx->h_small[2], sizeof(Fe)) == 0;  // distinct.hpp:57-59
        *ok = (same && !flags[0]) ? 1 : 0;
        ctx->end_call();
    });
}

int dgkr_distinct_chain_update(dgkr_ctx* ctx, const dgkr_field* f, const std::uint8_t* h, std::uint64_t n_max,
                               const std::uint8_t* items, std::size_t n, std::uint8_t* h_out) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        const HostField& F = f->f;
        const U256 hv = F.from_bytes(h);  // throws DGKR_INVALID_ARGUMENT on >= p
        NttWs& ws = ctx->nttws();
        CK(cudaMemsetAsync(ctx->d_flag.p, 0, 2 * sizeof(int), ctx->st));
        AhPass p = ah_enqueue(ctx, f, items, n, ws.stage, ws.x, 1);
        launch_bound_check(p.canon, static_cast<int>(F.width()), n, n_max, ctx->d_flag.p, ctx->st);
        ctx->launched();
        int flags[2];
        distinct_finish(ctx, flags);
        if (flags[0]) fail(DGKR_OUT_OF_RANGE, "validator index above bound");  // distinct.hpp:86-88
        F.to_bytes(F.add(hv, to_u256(ctx->h_small[1])), h_out);
        ctx->end_call();
    });
}

int dgkr_distinct_bitchange(dgkr_ctx* ctx, const dgkr_field* f, std::size_t count, std::uint64_t* set_counts) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        if (count < 10000) fail(DGKR_INVALID_ARGUMENT, "bit-change experiment needs count >= 10^4");  // :116-118
        const int bits = static_cast<int>(f->f.bits());
        if (bits > 256) fail(DGKR_UNSUPPORTED, "field too wide");
        DBuf<unsigned long long> d;
        d.ensure(bits);
        CK(cudaMemsetAsync(d.p, 0, bits * sizeof(unsigned long long), ctx->st));
        Fe offe = to_fe(f->f.from_u64(4294967295ull));
        launch_bitchange(ctx->use(f), 1, count, bits, &offe, d.p, ctx->st);
        ctx->launched();
        std::vector<unsigned long long> h(bits);
        ctx->d2h(h.data(), d.p, bits * sizeof(unsigned long long));
        ctx->sync();
        for (int k = 0; k < bits; ++k) set_counts[k] = h[k];
        ctx->end_call();
    });
}

// ---------------------------------------------------------------------------
// Beacon validator tree (beacon.hpp; config C3): root, membership paths and
// batched verify_membership on the device. Records cross as their 64-byte
// ValidatorRecord::encode() (beacon.hpp:27-37).
// ---------------------------------------------------------------------------
namespace {

/// zero_cache (beacon.hpp:66-83): z_0 = H(64 zero bytes), z_k = H(z_{k-1} || z_{k-1})
std::vector<Digest> zero_cache_host(unsigned depth) {
    std::vector<Digest> z;
    std::uint8_t zero[64] = {};
    z.push_back(sha256(zero, 64));
    for (unsigned k = 1; k <= depth; ++k) {
        std::uint8_t buf[64];
        std::memcpy(buf, z.back().data(), 32);
        std::memcpy(buf + 32, z.back().data(), 32);
        z.push_back(sha256(buf, 64));
    }
    return z;
}

unsigned active_log2_of(std::uint64_t n) {
    unsigned a = 0;
    while ((std::uint64_t{1} << a) < n) ++a;
    return a;
}

/// builds the active-subtree heap in ws.b_nodes (leaves at [2^a, 2^(a+1))); returns a
unsigned beacon_build(Lane* ctx, NttWs& ws, const std::uint8_t* records, std::uint64_t n, unsigned depth,
                      const std::vector<Digest>& zc) {
    const unsigned a = active_log2_of(n);
    if (a > depth) fail(DGKR_INVALID_ARGUMENT, "validator set exceeds tree capacity");  // beacon.hpp:113-115
    const std::uint64_t cap = std::uint64_t{1} << a;
    ws.b_recs.ensure(std::max<std::uint64_t>(n, 1) * 64);
    if (n) ctx->h2d_large(ws.b_recs.p, records, n * 64);
    ws.b_zc.ensure((depth + 1) * 32);
    ctx->h2d(ws.b_zc.p, zc.data(), (depth + 1) * 32);
    ws.b_nodes.ensure(2 * cap * 32);
    ctx->tbeg();
    launch_beacon_leaves(ws.b_recs.p, n, cap, ws.b_zc.p, ws.b_nodes.p + cap * 32, ctx->st);
    launch_merkle(ws.b_nodes.p, cap, ctx->st);
    ctx->tend(ctx->prof.merkle_ms);
    ctx->launched(2);
    return a;
}

}  // namespace

int dgkr_beacon_root(dgkr_ctx* ctx, const std::uint8_t* records, std::size_t n, unsigned depth, std::uint8_t* root) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        const auto zc = zero_cache_host(depth);
        NttWs& ws = ctx->nttws();
        const unsigned a = beacon_build(ctx, ws, records, n, depth, zc);
        Digest h;
        ctx->d2h(h.data(), ws.b_nodes.p + 32, 32);
        ctx->sync();
        for (unsigned k = a; k < depth; ++k) {  // left spine (beacon.hpp:128-131)
            std::uint8_t buf[64];
            std::memcpy(buf, h.data(), 32);
            std::memcpy(buf + 32, zc[k].data(), 32);
            h = sha256(buf, 64);
        }
        std::memcpy(root, h.data(), 32);
        ctx->end_call();
    });
}

int dgkr_beacon_prove(dgkr_ctx* ctx, const std::uint8_t* records, std::size_t n, unsigned depth,
                      const std::uint64_t* indices, std::size_t m, std::uint8_t* leaves, std::uint8_t* siblings,
                      unsigned* active_log2) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        for (std::size_t i = 0; i < m; ++i)
            if (indices[i] >= n) fail(DGKR_OUT_OF_RANGE, "inactive validator index");  // beacon.hpp:138-140
        const auto zc = zero_cache_host(depth);
        NttWs& ws = ctx->nttws();
        const unsigned a = beacon_build(ctx, ws, records, n, depth, zc);
        ws.didx.ensure(std::max<std::size_t>(m, 1));
        ws.b_leaves.ensure(std::max<std::size_t>(m, 1) * 32);
        ws.b_sib.ensure(std::max<std::size_t>(m * a, 1) * 32);
        if (m) {
            ctx->h2d(ws.didx.p, indices, m * 8);
            launch_beacon_paths(ws.b_nodes.p, static_cast<int>(a), ws.didx.p, m, ws.b_leaves.p, ws.b_sib.p, ctx->st);
            ctx->launched();
            ctx->d2h_large(leaves, ws.b_leaves.p, m * 32);
            if (a) ctx->d2h_large(siblings, ws.b_sib.p, m * a * 32);
        }
        ctx->sync();
        *active_log2 = a;
        ctx->end_call();
    });
}

int dgkr_beacon_verify(dgkr_ctx* ctx, const std::uint8_t* root, const std::uint8_t* records, const std::uint8_t* leaves,
                       const std::uint8_t* siblings, const std::uint64_t* indices, std::size_t m, unsigned depth,
                       unsigned active_log2, std::uint8_t* ok) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        if (active_log2 > 64) fail(DGKR_INVALID_ARGUMENT, "active_log2 out of range");
        if (m == 0) {
            ctx->end_call();
            return;
        }
        NttWs& ws = ctx->nttws();
        const unsigned a = active_log2;
        // paths claiming a > depth have no zero-cache tail; verify_membership walks a siblings then none
        const unsigned zdepth = std::max(depth, a);
        const auto zc = zero_cache_host(zdepth);
        ws.b_root.ensure(32);
        ws.b_recs.ensure(m * 64);
        ws.b_leaves.ensure(m * 32);
        ws.b_sib.ensure(std::max<std::size_t>(m * a, 1) * 32);
        ws.didx.ensure(m);
        ws.b_zc.ensure((zdepth + 1) * 32);
        ws.b_ok.ensure(m);
        ctx->h2d(ws.b_root.p, root, 32);
        ctx->h2d_large(ws.b_recs.p, records, m * 64);
        ctx->h2d_large(ws.b_leaves.p, leaves, m * 32);
        if (a) ctx->h2d_large(ws.b_sib.p, siblings, m * a * 32);
        ctx->h2d(ws.didx.p, indices, m * 8);
        ctx->h2d(ws.b_zc.p, zc.data(), (zdepth + 1) * 32);
        ctx->tbeg();
        launch_beacon_verify(ws.b_root.p, ws.b_recs.p, ws.b_leaves.p, ws.b_sib.p, ws.didx.p, m, static_cast<int>(a),
                             static_cast<int>(depth), ws.b_zc.p, ws.b_ok.p, ctx->st);
        ctx->tend(ctx->prof.merkle_ms);
        ctx->launched();
        ctx->d2h(ok, ws.b_ok.p, m);
        ctx->sync();
        ctx->end_call();
    });
}

int dgkr_ntt(dgkr_ctx* ctx, const dgkr_field* f, const std::uint8_t* in, unsigned log_n, int inverse,
             std::uint8_t* out) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        const HostField& F = f->f;
        const FieldKind kind = ctx->use(f);
        const std::uint64_t N = std::uint64_t{1} << log_n;
        const std::size_t w = F.width();
        NttWs& ws = ctx->nttws();
        auto& stage = ws.stage;
        auto& x = ws.x;
        auto& a = ws.a;
        auto& tw = ws.tw;
        auto& scratch = ws.scratch;
        x.ensure(N);
        a.ensure(N);
        ctx->upload_elems(f, in, N, x.p, stage);
        const U256 root = f->root_of_unity(log_n);
        tw.ensure(std::max<std::uint64_t>(N / 2, 1));
        if (N >= 2) pow_table(ctx, f, inverse ? F.inv(root) : root, N / 2, tw.p, scratch);
        ctx->tbeg();
        launch_bitrev_scale(kind, x.p, nullptr, a.p, static_cast<int>(log_n), N, ctx->st);
        launch_ntt(kind, a.p, static_cast<int>(log_n), tw.p, ctx->st);
        ctx->tend(ctx->prof.ntt_ms);
        if (inverse) {
            U256 k[9];
            f->fold_const(F.inv(F.from_u64(N)), k);
            launch_scale(kind, a.p, N, k, ctx->st);
        }
        stage.ensure(N * w);
        launch_to_canonical(kind, a.p, stage.p, static_cast<int>(w), N, ctx->st);
        ctx->d2h_large(out, stage.p, N * w);
        ctx->end_call();
    });
}

int dgkr_rs_encode(dgkr_ctx* ctx, const dgkr_field* f, const std::uint8_t* coeffs, std::size_t n,
                   unsigned blowup_log, std::uint8_t* out) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        if (n == 0 || (n & (n - 1)) != 0) fail(DGKR_INVALID_ARGUMENT, "coefficient count must be a power of two");
        const unsigned log_n = log2_exact(n) + blowup_log;
        const std::uint64_t N = std::uint64_t{1} << log_n;
        const std::size_t w = f->f.width();
        NttWs& ws = ctx->nttws();
        auto& stage = ws.stage;
        auto& cf = ws.x;
        auto& a = ws.a;
        auto& tw = ws.tw;
        auto& cpow = ws.cpow;
        auto& scratch = ws.scratch;
        cf.ensure(n);
        a.ensure(N);
        ctx->upload_elems(f, coeffs, n, cf.p, stage);
        coset_ntt(ctx, f, cf.p, n, log_n, f->coset, true, a.p, tw, cpow, scratch);
        stage.ensure(N * w);
        launch_to_canonical(ctx->use(f), a.p, stage.p, static_cast<int>(w), N, ctx->st);
        ctx->d2h_large(out, stage.p, N * w);
        ctx->end_call();
    });
}

int dgkr_fri_prove(dgkr_ctx* ctx, const dgkr_field* f, const std::uint8_t* coeffs, std::size_t n,
                   unsigned blowup_log, unsigned final_log, std::size_t queries, dgkr_transcript* t,
                   std::uint8_t* proof, std::size_t cap, std::size_t* len) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        Transcript tr(&f->f, t->state, t->draws);
        auto bytes = fri_prove(ctx, f, coeffs, n, blowup_log, final_log, queries, tr);
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        ctx->end_call();
        emit(bytes, proof, cap, len);
    });
}

int dgkr_fri_prove_dist(dgkr_ctx* ctx, dgkr_comm* comm, const dgkr_field* f, const std::uint8_t* coeffs, std::size_t n,
                        unsigned blowup_log, unsigned final_log, std::size_t queries, dgkr_transcript* t,
                        std::uint8_t* proof, std::size_t cap, std::size_t* len) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        if (!comm) fail(DGKR_INVALID_ARGUMENT, "communicator must not be NULL");
        Transcript tr(&f->f, t->state, t->draws);
        auto bytes = fri_prove(ctx, f, coeffs, n, blowup_log, final_log, queries, tr, comm);
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        ctx->end_call();
        emit(bytes, proof, cap, len);
    });
}

int dgkr_fri_prove_dist_emulated(dgkr_ctx* ctx, const dgkr_field* f, int world, const std::uint8_t* const* coeffs,
                                 std::size_t n, unsigned blowup_log, unsigned final_log, std::size_t queries,
                                 dgkr_transcript* t, std::uint8_t* const* proofs, const std::size_t* caps,
                                 std::size_t* lens) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (world < 1 || world > 64) fail(DGKR_INVALID_ARGUMENT, "world must be 1..64");
        std::vector<Lane*> lanes(world);
        for (int r = 0; r < world; ++r) {
            lanes[r] = ctx->lane(r);
            lanes[r]->profile_on = ctx->profile_on;
        }
        ctx->use(f);
        ThreadGroup group;
        group.world = world;
        std::vector<ThreadComm> comms(world);
        std::vector<dgkr_transcript> ts(world, *t);
        std::vector<int> codes(world, DGKR_OK);
        std::vector<std::string> errs(world);
        for (int r = 0; r < world; ++r) {
            comms[r].rank = r;
            comms[r].world = world;
            comms[r].g = &group;
        }
        auto work = [&](int r) {
            try {
                CK(cudaSetDevice(ctx->device));
                Lane* L = lanes[r];
                L->begin_call();
                Transcript tr(&f->f, ts[r].state, ts[r].draws);
                auto bytes = fri_prove(L, f, coeffs[r], n, blowup_log, final_log, queries, tr, &comms[r]);
                std::memcpy(ts[r].state, tr.state().data(), 32);
                ts[r].draws = tr.draws();
                L->end_call();
                emit(bytes, proofs[r], caps[r], &lens[r]);
            } catch (const Error& e) {
                codes[r] = e.code;
                errs[r] = e.what();
                group.abort();
            } catch (const std::exception& e) {
                codes[r] = DGKR_LOGIC_ERROR;
                errs[r] = e.what();
                group.abort();
            }
        };
        std::vector<std::thread> th;
        for (int r = 1; r < world; ++r) th.emplace_back(work, r);
        work(0);
        for (auto& x : th) x.join();
        for (int r = 0; r < world; ++r)
            if (codes[r] != DGKR_OK) fail(codes[r], "rank " + std::to_string(r) + ": " + errs[r]);
        for (int r = 1; r < world; ++r)
            if (std::memcmp(ts[r].state, ts[0].state, 32) != 0 || ts[r].draws != ts[0].draws)
                fail(DGKR_LOGIC_ERROR, "ranks disagree on the transcript");
        *t = ts[0];
    });
}

