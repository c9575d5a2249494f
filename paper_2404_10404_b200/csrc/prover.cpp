// Host drivers and C ABI of the B200 distributed-GKR prover
// (include/dgkr_b200.h). The protocol logic that must stay serial and
// bit-exact — transcript order, claim registry, claim combination — runs here
// on the host, following the reference line by line (citations inline); all
// O(table) work runs in the sm_100a kernels of kernels.cu. The runtime types
// live in runtime.hpp, the transports in comm.hpp; distinct / beacon / NTT /
// FRI entry points in ext.cpp.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <sched.h>
#include <memory>
#include <set>
#include <string>
#include <functional>
#include <thread>
#include <vector>

#include "comm.hpp"
#include "dgkr_b200.h"
#include "host_core.hpp"
#include "kernels.hpp"
#include "runtime.hpp"



namespace {

// ===========================================================================
// Sum-check round engine: runs the rounds of one sum-check over device pair
// tables, with the transcript on the host (sumcheck.hpp:230-238 order:
// absorb c0..c3, then challenge).
// ===========================================================================
struct RoundBuffers {
    int ntab = 0;
    std::uint64_t cap = 0;  // max table size handled
    DBuf<Fe> bufA, bufB, finals;
    DBuf<const Fe*> ptrs;   // [A ptrs | B ptrs | finals ptrs] each ntab
    std::vector<const Fe*> hptrs;  // host copy of ptrs (tensor maps of the TMA round kernel)
    /// st: the stream that will use the buffers. The pointer table is
    /// uploaded on it: a synchronous cudaMemcpy from pageable memory may
    /// return before its NULL-stream DMA lands, and non-blocking lane streams
    /// do not wait for the NULL stream.
    void ensure(int nt, std::uint64_t size0, cudaStream_t st) {
        if (nt <= ntab && size0 <= cap) return;
        ntab = std::max(nt, ntab);
        cap = std::max(size0, cap);
        const std::uint64_t a = std::max<std::uint64_t>(cap / 2, 1), b = std::max<std::uint64_t>(cap / 4, 1);
        bufA.ensure(ntab * a);
        bufB.ensure(ntab * b);
        finals.ensure(ntab);
        std::vector<const Fe*> h(3 * ntab);
        for (int t = 0; t < ntab; ++t) {
            h[t] = bufA.p + t * a;
            h[ntab + t] = bufB.p + t * b;
            h[2 * ntab + t] = finals.p + t;
        }
        ptrs.ensure(3 * ntab);
        CK(cudaMemcpyAsync(ptrs.p, h.data(), h.size() * sizeof(const Fe*), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));  // h is pageable and local
        hptrs = std::move(h);
    }
    const Fe* const* hA() const { return hptrs.data(); }
    const Fe* const* hB() const { return hptrs.data() + ntab; }
    const Fe* const* A() const { return ptrs.p; }
    const Fe* const* B() const { return ptrs.p + ntab; }
    const Fe* const* F() const { return ptrs.p + 2 * ntab; }
};

/// per-lane buffers of a distributed sum-check's phase boundary: this rank's
/// finals, the world-sized tables, their pointer array and the tail round
/// buffers (persistent: no device allocation inside a proof)
struct DistTail {
    DBuf<Fe> mine, tabs;
    DBuf<const Fe*> ptrs;
    RoundBuffers rb;
};

struct RoundPoly {
    U256 c[3];
};

struct SumcheckRun {
    std::vector<RoundPoly> rounds;
    std::vector<U256> challenges;
    std::vector<U256> finals;  // per table, Montgomery
    U256 claim_end{};          // p_last(r_last) when run with a known claim
    // stopped early (stop_after < nv): the tables folded with every challenge
    // so far, 2^(nv - stop_after) elements each, bit-reversed when tail_bitrev
    std::vector<const Fe*> tail_tables;
    bool tail_bitrev = false;
};

/// tables: device pointer array `base` of ntab = 2*np + has_g tables of
/// size 2^nv. Returns rounds, challenges and the final value of each table.
/// claim: the running sum-check claim when the caller produced it itself
/// (then p(0) + p(1) = claim holds exactly and S1 = claim - S0 is not
/// computed on the device); nullptr = derive every round from the tables.
SumcheckRun run_rounds(Lane* ctx, const dgkr_field* f, int np, bool has_g, int nv, const Fe* const* base,
                       RoundBuffers& rb, Transcript& tr, dgkr_comm* comm = nullptr, const U256* claim = nullptr,
                       const Fe* const* base_host = nullptr, bool r1_done = false, int stop_after = -1);

inline std::size_t brev_bits(std::size_t x, int bits) {
    std::size_t r = 0;
    for (int i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1);
    return r;
}

/// distributed sum-checks switch to redundant per-rank rounds once a rank's
/// live tables are this small (2^kEarlyLog): one all-gather of the tables
/// replaces the remaining per-round exchanges (SURVEY §7 "early boundary")
constexpr int kEarlyLog = 10;

/// Distributed form (cluster.hpp:228-320 generalised to the layer
/// sum-check): `nv` local variables per rank, rank = high variables. Local
/// rounds sum every rank's (S0,S1,S2) after an all-gather (the reference's
/// worker->master round messages); at the boundary the per-rank finals are
/// all-gathered and every rank finishes the log2(world) top rounds on the
/// rebuilt world-sized tables — identical on all ranks, so the transcript
/// equals the single-GPU one byte for byte.
SumcheckRun run_rounds_dist(Lane* ctx, const dgkr_field* f, int np, bool has_g, int nv, const Fe* const* base,
                            RoundBuffers& rb, Transcript& tr, dgkr_comm* comm, DistTail& dt,
                            const U256* claim = nullptr, const Fe* const* base_host = nullptr,
                            bool r1_done = false) {
    const int ntab = 2 * np + (has_g ? 1 : 0);
    const int world = comm->world;
    int lw = 0;
    while ((1 << lw) < world) ++lw;
    // local rounds with a per-round all-gather of the sums, until the live
    // tables have 2^kb elements; then ONE all-gather of those tables and every
    // rank finishes the last kb + log2(world) rounds on the rebuilt global
    // tables (rank = high bits), identically (cluster.hpp:289-318 with the
    // boundary moved down: the same rounds, sums and transcript)
    const int kb = std::min(nv, kEarlyLog);
    SumcheckRun loc = run_rounds(ctx, f, np, has_g, nv, base, rb, tr, comm, claim, base_host, r1_done, nv - kb);
    const std::size_t lsz = std::size_t{1} << kb;
    std::vector<const Fe*> src = loc.tail_tables;
    if (src.empty()) {  // no local round ran: the base tables themselves (natural order)
        src.resize(ntab);
        if (base_host) std::copy(base_host, base_host + ntab, src.begin());
        else CK(cudaMemcpy(src.data(), base, ntab * sizeof(const Fe*), cudaMemcpyDeviceToHost));
    }
    dt.mine.ensure(static_cast<std::size_t>(ntab) * lsz);
    for (int t = 0; t < ntab; ++t)
        CK(cudaMemcpyAsync(dt.mine.p + t * lsz, src[t], lsz * sizeof(Fe), cudaMemcpyDeviceToDevice, ctx->st));
    std::vector<Fe> all(static_cast<std::size_t>(world) * ntab * lsz);
    comm->allgather_to_host(dt.mine.p, all.data(), ntab * lsz * sizeof(Fe), ctx);
    // world-sized tables in natural order: global index = rank * 2^kb + logical local index
    const std::size_t gsz = lsz * static_cast<std::size_t>(world);
    std::vector<Fe> h(static_cast<std::size_t>(ntab) * gsz);
    for (int r = 0; r < world; ++r)
        for (int t = 0; t < ntab; ++t)
            for (std::size_t l = 0; l < lsz; ++l) {
                const std::size_t st = loc.tail_bitrev ? brev_bits(l, kb) : l;
                h[static_cast<std::size_t>(t) * gsz + r * lsz + l] = all[(static_cast<std::size_t>(r) * ntab + t) * lsz + st];
            }
    dt.tabs.ensure(h.size());
    ctx->h2d(dt.tabs.p, h.data(), h.size() * sizeof(Fe));
    std::vector<const Fe*> hp(ntab);
    for (int t = 0; t < ntab; ++t) hp[t] = dt.tabs.p + static_cast<std::size_t>(t) * gsz;
    dt.ptrs.ensure(ntab);
    ctx->h2d(dt.ptrs.p, hp.data(), ntab * sizeof(const Fe*));
    const U256 mid = (nv - kb > 0 || !claim) ? loc.claim_end : *claim;
    SumcheckRun tail = run_rounds(ctx, f, np, has_g, kb + lw, dt.ptrs.p, dt.rb, tr, nullptr, claim ? &mid : nullptr,
                                  hp.data());
    loc.rounds.insert(loc.rounds.end(), tail.rounds.begin(), tail.rounds.end());
    loc.challenges.insert(loc.challenges.end(), tail.challenges.begin(), tail.challenges.end());
    loc.finals = tail.finals;
    loc.claim_end = tail.claim_end;
    loc.tail_tables.clear();
    return loc;
}

SumcheckRun run_rounds(Lane* ctx, const dgkr_field* f, int np, bool has_g, int nv, const Fe* const* base,
                       RoundBuffers& rb, Transcript& tr, dgkr_comm* comm, const U256* claim,
                       const Fe* const* base_host, bool r1_done, int stop_after) {
    // stop_after in [0, nv): run rounds 1..stop_after only, then fold the
    // tables with the last challenge (the next round's fold, its sums unused)
    // and return them in tail_tables instead of finals
    // r1_done: round 1's (S0, S2) are already in ws.result (bookkeeping with
    // the first round fused, k_bookkeep_pairs); the round-1 launch is skipped
    const HostField& F = f->f;
    const bool skip_s1 = claim != nullptr;
    const int nres = skip_s1 ? 2 : 3;  // device sums per round: (S0, S2) or (S0, S1, S2)
    U256 run_claim = skip_s1 ? *claim : U256{};
    const FieldKind kind = ctx->use(f);
    const int ntab = 2 * np + (has_g ? 1 : 0);
    SumcheckRun out;
    const std::uint64_t size0 = std::uint64_t{1} << nv;
    rb.ensure(ntab, size0, ctx->st);
    Fe* d_r = ctx->d_small.p;
    const Fe* const* cur = base;
    const Fe* const* cur_h = base_host;  // host mirror of cur (null: no TMA round kernel)
    const U256 zero{};
    U256 fk[9] = {};
    const int n_rounds = (stop_after >= 0 && stop_after < nv) ? stop_after : nv;
    // host side of a round: round polynomial from the device sums in
    // h_small[1..], transcript, challenge, next fold constants (fk)
    auto host_round = [&]() -> U256 {
        const double t0 = now_ms();
        const U256 s0 = to_u256(ctx->h_small[1]);
        const U256 s1 = skip_s1 ? F.sub(run_claim, s0) : to_u256(ctx->h_small[2]);  // p(0) + p(1) = claim
        const U256 s2 = to_u256(ctx->h_small[nres]);
        RoundPoly rp;
        rp.c[0] = s0;
        rp.c[2] = s2;
        rp.c[1] = F.sub(F.sub(s1, s0), s2);
        for (int k = 0; k < 3; ++k) tr.absorb(rp.c[k]);
        tr.absorb(zero);
        const U256 r = tr.challenge();
        if (skip_s1) run_claim = F.add(rp.c[0], F.mul(r, F.add(rp.c[1], F.mul(r, rp.c[2]))));  // p(r)
        ctx->prof.host_transcript_ms += now_ms() - t0;
        ctx->prof.rounds += 1;
        out.rounds.push_back(rp);
        out.challenges.push_back(r);
        f->fold_const(r, fk);  // next round's fold constants (kernel parameters)
        return r;
    };
    // the rounds with <= tail_pairs output pairs and the final fold run in one
    // mailbox launch (launch_round_tail) where the sum-check runs to the end
    // on this lane alone
    int j_tail = n_rounds + 1;
    if (const std::uint64_t tp = tuning().tail_pairs; tp && !comm && n_rounds == nv && nv >= 1) {
        int j = 1;
        while (j <= nv && (size0 >> j) > tp) ++j;
        if (j == 1 && r1_done) j = 2;
        if (j <= nv) j_tail = j;
    }
    // one round as its own launch + sums readback (the path for large rounds,
    // distributed rounds, and the rounds after a tail launch gave up)
    auto buffer_after = [&](int j) -> const Fe* const* {  // tables as round j left them
        return j >= 2 ? ((j % 2 == 0) ? rb.A() : rb.B()) : base;
    };
    auto buffer_after_h = [&](int j) -> const Fe* const* {
        if (!base_host) return nullptr;
        return j >= 2 ? ((j % 2 == 0) ? rb.hA() : rb.hB()) : base_host;
    };
    auto launch_round_j = [&](int j) {
        RoundLaunch rl;
        rl.np = np;
        rl.has_g = has_g;
        rl.r = d_r;
        rl.fold_const = fk;
        rl.need_s1 = !skip_s1;
        if (j == 1) {
            rl.mode = 0;  // scan the natural-order base tables
            rl.in = base;
            rl.out = nullptr;
            rl.in_host = base_host;
        } else {
            rl.mode = (j == 2) ? 1 : 2;  // fold natural -> bit-reversed, then bit-reversed -> bit-reversed
            rl.in = cur;
            rl.in_host = cur_h;
            const Fe* const* nxt = buffer_after(j);
            const Fe* const* nxt_h = (j % 2 == 0) ? rb.hA() : rb.hB();
            rl.out = const_cast<Fe* const*>(nxt);
            rl.out_host = cur_h ? const_cast<Fe* const*>(nxt_h) : nullptr;
            cur = nxt;
            if (cur_h) cur_h = nxt_h;
        }
        rl.n_out_pairs = size0 >> j;
        if (ctx->profile_on) CK(cudaEventRecord(ctx->ev0, ctx->st));
        const std::uint64_t small_pairs = tuning().small_round_pairs;
        if (j == 1 && r1_done) {
            if (!skip_s1) fail(DGKR_LOGIC_ERROR, "fused round 1 computes (S0, S2) only");
        } else {
            if (rl.n_out_pairs <= small_pairs) launch_round_small(kind, rl, ctx->ws, ctx->st);
            else launch_round(kind, rl, ctx->ws, ctx->st);
            ctx->launched();
        }
        if (ctx->profile_on) CK(cudaEventRecord(ctx->ev1, ctx->st));
        if (comm) {
            // every rank's partial round sums (cluster.hpp:272-278), summed on every rank
            const std::size_t W = static_cast<std::size_t>(comm->world);
            comm->allgather_to_host(ctx->ws.result, ctx->h_small + Lane::kGatherOff, nres * sizeof(Fe), ctx);
            U256 acc[3] = {};
            for (std::size_t r = 0; r < W; ++r)
                for (int k = 0; k < nres; ++k)
                    acc[k] = F.add(acc[k], to_u256(ctx->h_small[Lane::kGatherOff + nres * r + k]));
            for (int k = 0; k < nres; ++k) ctx->h_small[1 + k] = to_fe(acc[k]);
        } else {
            ctx->d2h(ctx->h_small + 1, ctx->ws.result, nres * sizeof(Fe));
            ctx->sync();
        }
        if (ctx->profile_on && !(j == 1 && r1_done)) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
            ctx->prof.round_ms += ms;
            ctx->prof.round_launches += 1;
            const std::uint64_t pairs = rl.n_out_pairs;
            const std::uint64_t ntabs = static_cast<std::uint64_t>(ntab);
            // bytes: fold reads 4, writes 2 elements per table per output pair; scan reads 2
            ctx->prof.round_bytes += pairs * ntabs * 32 * (rl.mode ? 6 : 2);
            ctx->prof.round_mults += pairs * (nres * np + (rl.mode ? 2 * ntabs : 0));
        }
        const U256 r = host_round();
        ctx->h_small[0] = to_fe(r);
        ctx->h2d(d_r, ctx->h_small, sizeof(Fe));
    };
    for (int j = 1; j < j_tail; ++j) launch_round_j(j);
    bool tail_folded = false;  // the tail launch wrote the finals
    if (j_tail <= n_rounds) {
        TailMailbox* mb = ctx->tail_mb;
        ctx->tail_gen = ctx->tail_gen % 0xfffffeu + 1;  // tags never 0 nor kTailAbort
        const std::uint32_t tag = ctx->tail_gen << 8;
        TailLaunch tl;
        tl.in = j_tail == 1 ? base : cur;
        tl.buf_a = const_cast<Fe* const*>(rb.A());
        tl.buf_b = const_cast<Fe* const*>(rb.B());
        tl.fin = const_cast<Fe* const*>(rb.F());
        tl.np = np;
        tl.has_g = has_g;
        tl.need_s1 = !skip_s1;
        tl.j0 = j_tail;
        tl.nv = nv;
        tl.fold_const = fk;
        tl.mb = ctx->tail_mb_dev;
        tl.tag = tag;
        tl.timeout_ns = tuning().tail_timeout_us * 1000;
        std::uint32_t* d_seq = const_cast<std::uint32_t*>(&mb->d_seq);
        std::uint32_t* h_seq = const_cast<std::uint32_t*>(&mb->h_seq);
        __atomic_store_n(d_seq, 0u, __ATOMIC_RELEASE);
        __atomic_store_n(h_seq, 0u, __ATOMIC_RELEASE);  // clear a previous abort
        ctx->tbeg();
        launch_round_tail(kind, tl, ctx->st);
        ctx->launched();
        // If the CTA gives up waiting for a challenge (the host thread was
        // descheduled, or a profiler serialises launches so the host cannot
        // answer while the kernel runs), the rounds it did not finish run as
        // per-round launches from where it stopped: same tables, same bytes.
        int resume = 0;
        try {
            for (int j = j_tail; j <= nv + 1; ++j) {  // j = nv + 1: the final fold's acknowledgement
                const std::uint32_t want = tag | static_cast<std::uint32_t>(j);
                const double t0 = now_ms();
                std::uint32_t v = 0;
                const bool yield = tuning().spin_yield != 0;
                for (std::uint32_t spin = 1;; ++spin) {
                    v = __atomic_load_n(d_seq, __ATOMIC_ACQUIRE);
                    if (v == want || v == kTailAbort) break;
                    __builtin_ia32_pause();
                    if (yield && (spin & 31) == 0) sched_yield();
                    if ((spin & 4095) == 0) {
                        const cudaError_t q = cudaStreamQuery(ctx->st);
                        if (q != cudaSuccess && q != cudaErrorNotReady) CK(q);
                        v = __atomic_load_n(d_seq, __ATOMIC_ACQUIRE);
                        if (v == want || v == kTailAbort) break;
                        if (q == cudaSuccess) fail(DGKR_CUDA_ERROR, "sum-check tail kernel ended without posting");
                        if (now_ms() - t0 > 60e3) fail(DGKR_CUDA_ERROR, "sum-check tail kernel: no post in 60 s");
                    }
                }
                if (v == kTailAbort) {
                    const std::uint32_t at = __atomic_load_n(const_cast<std::uint32_t*>(&mb->abort_round),
                                                             __ATOMIC_ACQUIRE);
                    if ((at & ~0xffu) != tag) fail(DGKR_LOGIC_ERROR, "sum-check tail: abort of another launch");
                    const int ar = static_cast<int>(at & 0xffu);
                    if (ar == j && j <= nv) {  // round j's sums are posted; its challenge was not taken
                        std::memcpy(ctx->h_small + 1, mb->sums, nres * sizeof(Fe));
                        const U256 r = host_round();
                        ctx->h_small[0] = to_fe(r);
                        ctx->h2d(d_r, ctx->h_small, sizeof(Fe));
                        resume = j + 1;
                    } else if (ar == j - 1) {  // stopped before round j
                        resume = j;
                    } else {
                        fail(DGKR_LOGIC_ERROR, "sum-check tail: inconsistent abort round");
                    }
                    ctx->prof.tail_aborts += 1;
                    break;
                }
                if (j == nv + 1) {
                    tail_folded = true;
                    // DGKR_TAIL_DIAG=1: print the launch's device-side time split to stderr
                    static const bool diag = std::getenv("DGKR_TAIL_DIAG") != nullptr;
                    if (diag) {
                        const volatile std::uint64_t* d = mb->diag;
                        std::fprintf(stderr, "tail diag: rounds %d wait %.1f us compute+post %.1f us kernel %.1f us\n",
                                     nv - j_tail + 1, d[0] * 1e-3, d[1] * 1e-3, d[2] * 1e-3);
                    }
                    break;
                }
                std::memcpy(ctx->h_small + 1, mb->sums, nres * sizeof(Fe));
                const U256 r = host_round();
                std::memcpy(mb->k, fk, kFoldConstBytes);
                __atomic_store_n(h_seq, want, __ATOMIC_RELEASE);
                if (j == nv) {  // d_small[0] holds the last challenge, as after the per-round path
                    ctx->h_small[0] = to_fe(r);
                    ctx->h2d(d_r, ctx->h_small, sizeof(Fe));
                }
            }
        } catch (...) {
            // release the CTA and let it exit before the mailbox is reused
            __atomic_store_n(h_seq, kTailAbort, __ATOMIC_RELEASE);
            (void)cudaStreamSynchronize(ctx->st);
            throw;
        }
        ctx->tend(ctx->prof.tail_ms);
        if (resume) {
            cur = buffer_after(resume - 1);
            cur_h = buffer_after_h(resume - 1);
            ctx->prof.tail_rounds += static_cast<std::uint64_t>(resume - j_tail);
            for (int j = resume; j <= nv; ++j) launch_round_j(j);
        } else {
            ctx->prof.tail_rounds += static_cast<std::uint64_t>(nv - j_tail + 1);
        }
    }
    out.claim_end = run_claim;
    if (n_rounds < nv) {
        if (n_rounds == 0) return out;  // the base tables, untouched (natural order)
        // fold with r_{n_rounds}: the round kernel of round n_rounds + 1 (its sums are not used)
        const int j = n_rounds + 1;
        RoundLaunch rl;
        rl.np = np;
        rl.has_g = has_g;
        rl.fold_const = fk;
        rl.need_s1 = !skip_s1;
        rl.mode = (j == 2) ? 1 : 2;
        rl.in = cur;
        rl.in_host = cur_h;
        const Fe* const* nxt = (j % 2 == 0) ? rb.A() : rb.B();
        const Fe* const* nxt_h = (j % 2 == 0) ? rb.hA() : rb.hB();
        rl.out = const_cast<Fe* const*>(nxt);
        rl.out_host = cur_h ? const_cast<Fe* const*>(nxt_h) : nullptr;
        rl.n_out_pairs = size0 >> j;
        if (rl.n_out_pairs <= tuning().small_round_pairs) launch_round_small(kind, rl, ctx->ws, ctx->st);
        else launch_round(kind, rl, ctx->ws, ctx->st);
        ctx->launched();
        out.tail_tables.assign(nxt_h, nxt_h + ntab);
        out.tail_bitrev = true;
        return out;
    }
    // final fold of the 2-element tables (or read the 1-element tables)
    if (nv >= 1) {
        if (!tail_folded) {
            launch_fold_final(kind, cur, const_cast<Fe* const*>(rb.F()), ntab, d_r, ctx->st);
            ctx->launched();
        }
        Fe* hf = ctx->h_small + Lane::kFinalsOff;
        ctx->d2h(hf, rb.finals.p, ntab * sizeof(Fe));
        ctx->sync();
        for (int t = 0; t < ntab; ++t) out.finals.push_back(to_u256(hf[t]));
    } else {
        ctx->sync();
        std::vector<const Fe*> hp(ntab);
        CK(cudaMemcpy(hp.data(), base, ntab * sizeof(const Fe*), cudaMemcpyDeviceToHost));
        for (int t = 0; t < ntab; ++t) {
            Fe v;
            CK(cudaMemcpy(&v, hp[t], sizeof(Fe), cudaMemcpyDeviceToHost));
            out.finals.push_back(to_u256(v));
        }
    }
    return out;
}

void append_elem(std::vector<std::uint8_t>& out, const HostField& F, const U256& m) {
    const std::size_t w = F.width();
    const std::size_t off = out.size();
    out.resize(off + w);
    F.to_bytes(m, out.data() + off);
}

/// SumcheckProof::to_bytes (sumcheck.hpp:51-61)
std::vector<std::uint8_t> sumcheck_bytes(const HostField& F, const U256& claimed, const std::vector<RoundPoly>& rounds,
                                         const std::vector<U256>& finals) {
    std::vector<std::uint8_t> out;
    append_elem(out, F, claimed);
    put32(out, static_cast<std::uint32_t>(rounds.size()));
    const U256 zero{};
    for (const auto& r : rounds) {
        for (int k = 0; k < 3; ++k) append_elem(out, F, r.c[k]);
        append_elem(out, F, zero);
    }
    put32(out, static_cast<std::uint32_t>(finals.size()));
    for (const auto& e : finals) append_elem(out, F, e);
    return out;
}

// ===========================================================================
// Product sum-check on uploaded tables (shared by prove_product_sum and the
// single-device dist_sumcheck).
// ===========================================================================
std::vector<std::uint8_t> product_sumcheck(Lane* ctx, const dgkr_field* f, std::size_t n_pairs, std::size_t vars,
                                           const std::uint8_t* tables, Transcript& tr, U256* claimed_out) {
    if (n_pairs == 0) fail(DGKR_INVALID_ARGUMENT, "product sum needs at least one pair");  // sumcheck.hpp:155-157
    if (vars > 40) fail(DGKR_INVALID_ARGUMENT, "table too large");
    const HostField& F = f->f;
    const std::uint64_t n = std::uint64_t{1} << vars;
    const int ntab = static_cast<int>(2 * n_pairs);
    DBuf<Fe> tabs;
    DBuf<std::uint8_t> stage;
    tabs.ensure(static_cast<std::size_t>(ntab) * n);
    ctx->upload_elems(f, tables, static_cast<std::uint64_t>(ntab) * n, tabs.p, stage);
    std::vector<const Fe*> hp(ntab);
    for (int t = 0; t < ntab; ++t) hp[t] = tabs.p + t * n;
    DBuf<const Fe*> base;
    base.ensure(ntab);
    ctx->h2d(base.p, hp.data(), ntab * sizeof(const Fe*));
    // claimed sum: PairSumSession::total (sumcheck.hpp:177-186)
    launch_pair_total(ctx->use(f), base.p, static_cast<int>(n_pairs), n, ctx->ws, ctx->st);
    ctx->launched();
    ctx->d2h(ctx->h_small + 1, ctx->ws.result, sizeof(Fe));
    ctx->sync();
    const U256 claimed = to_u256(ctx->h_small[1]);
    tr.absorb(claimed);  // sumcheck.hpp:231
    RoundBuffers rb;
    SumcheckRun run =
        run_rounds(ctx, f, static_cast<int>(n_pairs), false, static_cast<int>(vars), base.p, rb, tr, nullptr, &claimed);
    if (claimed_out) *claimed_out = claimed;
    return sumcheck_bytes(F, claimed, run.rounds, run.finals);
}

/// One rank's share of a distributed product sum-check (cluster.hpp:228-320
/// over real devices): the rank holds f_k^(rank), g_k^(rank) -- rows
/// [rank * 2^lv, (rank + 1) * 2^lv) of every table, the rank index being the
/// high variables (shard_pairs, cluster.hpp:190-217). Claimed sum = sum of the
/// ranks' totals (an all-gather); then the layer engine's distributed rounds:
/// per-round all-gather of the round sums, the early boundary, redundant tail
/// rounds on every rank. Byte-identical to prove_product_sum over the
/// concatenated tables on every rank.
std::vector<std::uint8_t> product_sumcheck_dist(Lane* ctx, const dgkr_field* f, std::size_t n_pairs,
                                                std::size_t local_vars, const std::uint8_t* local_tables,
                                                Transcript& tr, dgkr_comm* comm, DistTail& dt, DBuf<Fe>& tabs,
                                                RoundBuffers& rb) {
    if (n_pairs == 0) fail(DGKR_INVALID_ARGUMENT, "nothing to shard");
    if (local_vars > 40) fail(DGKR_INVALID_ARGUMENT, "table too large");
    const HostField& F = f->f;
    const std::uint64_t n = std::uint64_t{1} << local_vars;
    const int ntab = static_cast<int>(2 * n_pairs);
    DBuf<std::uint8_t> stage;
    tabs.ensure(static_cast<std::size_t>(ntab) * n);
    ctx->upload_elems(f, local_tables, static_cast<std::uint64_t>(ntab) * n, tabs.p, stage);
    std::vector<const Fe*> hp(ntab);
    for (int t = 0; t < ntab; ++t) hp[t] = tabs.p + t * n;
    DBuf<const Fe*> base;
    base.ensure(ntab);
    ctx->h2d(base.p, hp.data(), ntab * sizeof(const Fe*));
    launch_pair_total(ctx->use(f), base.p, static_cast<int>(n_pairs), n, ctx->ws, ctx->st);  // local total (:258-262)
    ctx->launched();
    comm->allgather_to_host(ctx->ws.result, ctx->h_small + Lane::kGatherOff, sizeof(Fe), ctx);
    U256 claimed{};
    for (int r = 0; r < comm->world; ++r) claimed = F.add(claimed, to_u256(ctx->h_small[Lane::kGatherOff + r]));
    tr.absorb(claimed);  // :264-265
    SumcheckRun run = run_rounds_dist(ctx, f, static_cast<int>(n_pairs), false, static_cast<int>(local_vars), base.p,
                                      rb, tr, comm, dt, &claimed, hp.data());
    return sumcheck_bytes(F, claimed, run.rounds, run.finals);
}

}  // namespace

// ===========================================================================
// GKR circuit (data-parallel capable)
// ===========================================================================
struct CircuitWs {
    std::vector<std::unique_ptr<DBuf<Fe>>> values;  // per layer, capacity-sized, zero padded
    DBuf<const Fe*> d_layer_vals;
    DBuf<Fe> H, G;      // bookkeeping outputs, max_slots x Tmax and Tmax
    DBuf<Fe> Wg, EqU;   // dense per-gate weights and chi(u) tables
    DBuf<Fe> eq_hc;     // split-eq row constants (9 per hi row) for the BN254 constant-multiplier expansion
    DBuf<Fe> heavy_scr; // heavy-row partials: 2 x max_heavy
    DistTail dist;      // distributed phase-boundary buffers (run_rounds_dist)
    RoundBuffers rb;
    DBuf<std::uint8_t> stage;
    DBuf<Fe> eq_tabs;   // split-eq tables for weights and u
    DBuf<EqJob> eq_jobs, eq_jobs2;
    struct Cons {
        DBuf<SlotDesc> d_slots1, d_slots2;
        DBuf<const Fe*> base_ptrs;  // V0,H0,V1,H1,...,G
        std::vector<const Fe*> base_host;  // host copy of base_ptrs
    };
    std::vector<std::unique_ptr<Cons>> cons;
    bool inputs_loaded = false;
};

struct dgkr_circuit {
    std::uint32_t input_size = 0;  // per copy
    std::uint32_t depth = 0;
    std::uint32_t n_copies = 1;
    std::uint32_t log_copies = 0;
    // per layer 0..depth (sub-circuit view)
    std::vector<std::uint64_t> sub_size, sub_padded;
    std::vector<std::uint32_t> sub_log;      // log2 sub_padded
    std::vector<std::uint64_t> full_padded;  // n_copies * sub_padded
    std::vector<std::uint64_t> capacity;     // buffer elements
    // per consumer layer 1..depth
    struct Consumer {
        std::vector<std::uint32_t> slots;  // ascending source layers
        std::uint32_t side = 0;            // full side vars
        std::uint64_t n_wires = 0;         // sub wires
        DBuf<std::uint32_t> xoff, yoff;    // concatenated per slot
        DBuf<uint4> xent, yent;
        DBuf<std::uint32_t> gstart;        // evaluation CSR
        DBuf<std::uint32_t> eperm;         // evaluation order (mul-heavy gates first)
        DBuf<uint4> nested;
        DBuf<std::uint32_t> xperm, yperm;  // single-slot: degree-sorted rows
        DBuf<uint2> xseg, yseg;
        DBuf<uint4> xpseg, ypseg;          // single-slot: row pairs, sorted by the larger degree (fused round 1)
        DBuf<uint4> xheavy, yheavy;        // heavy-row items {slot, copy, row, 0}, sorted by table row
        std::uint32_t n_xheavy = 0, n_yheavy = 0;
    };
    std::vector<std::unique_ptr<Consumer>> cons;  // index li (0 unused)
    DBuf<std::uint32_t> d_layer_log;
    std::uint32_t max_slots = 0;
    std::uint32_t max_heavy = 0;  // largest heavy-row item list of any consumer / phase
    std::uint64_t Tmax = 1;
    std::uint64_t total_gates = 0;  // full circuit gate count
    std::mutex ws_mu;
    std::vector<std::unique_ptr<CircuitWs>> ws;  // per lane

    std::uint32_t padded_log2_full(std::uint32_t l) const { return sub_log[l] + log_copies; }
    // host copy of the sub-circuit wiring (the verifier's sparse wire list)
    std::vector<std::uint64_t> h_lgs, h_gns, h_min_padded;
    std::vector<std::uint32_t> h_nested;
};

namespace {

/// CSR rows with more entries than this are reduced by a CTA, not a thread
constexpr std::uint32_t kHeavyMin = 64;

bool fuse_round1() { return tuning().fuse_round1 != 0; }

/// GeneralCircuit::validate (circuit.hpp:103-152) on the sub-circuit plus
/// the data-parallel preconditions; builds all device-side structures.
void build_circuit(Lane* ctx, dgkr_circuit& c, const std::uint64_t* lgs, const std::uint64_t* gns,
                   const std::uint32_t* nested, const std::uint64_t* min_padded) {
    const std::uint32_t D = c.depth;
    std::vector<std::string> violations;
    c.sub_size.assign(D + 1, 0);
    c.sub_size[0] = c.input_size;
    for (std::uint32_t li = 1; li <= D; ++li) c.sub_size[li] = lgs[li] - lgs[li - 1];
    c.sub_padded.assign(D + 1, 1);
    c.sub_log.assign(D + 1, 0);
    for (std::uint32_t l = 0; l <= D; ++l) {
        std::uint64_t p = next_pow2(std::max<std::uint64_t>(c.sub_size[l], 1));  // circuit.hpp:81-84
        if (min_padded) p = std::max(p, next_pow2(min_padded[l]));
        c.sub_padded[l] = p;
        c.sub_log[l] = log2_exact(p);
    }
    if (c.n_copies > 1) {
        for (std::uint32_t l = 0; l <= D; ++l) {
            if (c.sub_size[l] != c.sub_padded[l])
                fail(DGKR_INVALID_ARGUMENT, "data-parallel circuits need power-of-two sub layer sizes");
        }
    }
    auto name = [](std::uint32_t li, std::uint64_t gi, const char* side) {
        return "layer " + std::to_string(li) + " gate " + std::to_string(gi) + " " + side;
    };
    for (std::uint32_t li = 1; li <= D; ++li) {
        bool reads_prev = false;
        const std::uint64_t g0 = lgs[li - 1], g1 = lgs[li];
        if (g0 == g1) violations.push_back("layer " + std::to_string(li) + " has no gates");
        for (std::uint64_t g = g0; g < g1; ++g) {
            if (gns[g] == gns[g + 1]) {
                violations.push_back("layer " + std::to_string(li) + " gate " + std::to_string(g - g0) +
                                     " has no nested gates");
                continue;
            }
            for (std::uint64_t k = gns[g]; k < gns[g + 1]; ++k) {
                const std::uint32_t* e = nested + 5 * k;
                const std::uint32_t refs[2][2] = {{e[1], e[2]}, {e[3], e[4]}};
                const char* sides[2] = {"left", "right"};
                for (int s = 0; s < 2; ++s) {
                    if (refs[s][0] >= li) {
                        violations.push_back("non-causal wire at " + name(li, g - g0, sides[s]));
                        continue;
                    }
                    if (refs[s][1] >= c.sub_padded[refs[s][0]]) {
                        violations.push_back("dangling wire at " + name(li, g - g0, sides[s]));
                        continue;
                    }
                    if (refs[s][0] + 1 == li) reads_prev = true;
                }
            }
        }
        if (g0 != g1 && !reads_prev)
            violations.push_back("layer " + std::to_string(li) + " has no wire into layer " + std::to_string(li - 1));
    }
    if (!violations.empty()) fail(DGKR_INVALID_ARGUMENT, "invalid circuit: " + violations.front());
    if (D >= (1u << 15)) fail(DGKR_UNSUPPORTED, "too many layers");

    c.full_padded.assign(D + 1, 0);
    for (std::uint32_t l = 0; l <= D; ++l) c.full_padded[l] = c.sub_padded[l] << c.log_copies;
    c.capacity = c.full_padded;
    c.total_gates = 0;
    for (std::uint32_t li = 1; li <= D; ++li) c.total_gates += c.sub_size[li] * c.n_copies;

    // consumers: slots (gkr.hpp:107-131), CSR transposes, evaluation CSR
    c.cons.clear();
    c.cons.resize(D + 1);
    for (std::uint32_t li = 1; li <= D; ++li) {
        auto cp = std::make_unique<dgkr_circuit::Consumer>();
        auto& C = *cp;
        std::set<std::uint32_t> srcs;  // circuit.hpp:212-221
        for (std::uint64_t g = lgs[li - 1]; g < lgs[li]; ++g) {
            for (std::uint64_t k = gns[g]; k < gns[g + 1]; ++k) {
                srcs.insert(nested[5 * k + 1]);
                srcs.insert(nested[5 * k + 3]);
            }
        }
        C.slots.assign(srcs.begin(), srcs.end());
        std::uint32_t side = 0;
        for (auto s : C.slots) side = std::max(side, c.padded_log2_full(s));
        C.side = side;
        const std::uint64_t T = std::uint64_t{1} << side;
        for (auto s : C.slots) c.capacity[s] = std::max(c.capacity[s], T);
        c.Tmax = std::max(c.Tmax, T);
        c.max_slots = std::max<std::uint32_t>(c.max_slots, static_cast<std::uint32_t>(C.slots.size()));
        std::vector<int> slot_of(D + 1, -1);
        for (std::size_t s = 0; s < C.slots.size(); ++s) slot_of[C.slots[s]] = static_cast<int>(s);
        const std::size_t ns = C.slots.size();
        // counts
        std::vector<std::uint64_t> xbase(ns + 1, 0), ybase(ns + 1, 0);
        for (std::size_t s = 0; s < ns; ++s) {
            xbase[s + 1] = xbase[s] + c.sub_padded[C.slots[s]] + 1;
        }
        ybase = xbase;
        std::vector<std::uint32_t> xoff(xbase[ns], 0), yoff(ybase[ns], 0);
        std::uint64_t nw = 0;
        for (std::uint64_t g = lgs[li - 1]; g < lgs[li]; ++g) {
            for (std::uint64_t k = gns[g]; k < gns[g + 1]; ++k) {
                const std::uint32_t* e = nested + 5 * k;
                xoff[xbase[slot_of[e[1]]] + e[2] + 1]++;
                yoff[ybase[slot_of[e[3]]] + e[4] + 1]++;
                ++nw;
            }
        }
        C.n_wires = nw;
        // prefix sums per slot (offsets are per-slot local indexes into one entry array)
        std::vector<std::uint32_t> xslot_start(ns), yslot_start(ns);
        std::uint32_t accx = 0, accy = 0;
        for (std::size_t s = 0; s < ns; ++s) {
            const std::uint64_t len = c.sub_padded[C.slots[s]] + 1;
            xoff[xbase[s]] += accx;
            for (std::uint64_t i = 1; i < len; ++i) xoff[xbase[s] + i] += xoff[xbase[s] + i - 1];
            accx = xoff[xbase[s] + len - 1];
            yoff[ybase[s]] += accy;
            for (std::uint64_t i = 1; i < len; ++i) yoff[ybase[s] + i] += yoff[ybase[s] + i - 1];
            accy = yoff[ybase[s] + len - 1];
        }
        std::vector<uint4> xent(nw), yent(nw);
        std::vector<std::uint32_t> xfill(xoff), yfill(yoff);
        std::uint32_t wid = 0;
        for (std::uint64_t g = lgs[li - 1]; g < lgs[li]; ++g) {
            const std::uint32_t gl = static_cast<std::uint32_t>(g - lgs[li - 1]);
            for (std::uint64_t k = gns[g]; k < gns[g + 1]; ++k, ++wid) {
                const std::uint32_t* e = nested + 5 * k;
                const std::uint32_t mul = e[0] ? 0x80000000u : 0u;
                const int xs = slot_of[e[1]], ys = slot_of[e[3]];
                xent[xfill[xbase[xs] + e[2]]++] = make_uint4(gl, e[4], static_cast<std::uint32_t>(ys) | mul, wid);
                yent[yfill[ybase[ys] + e[4]]++] = make_uint4(gl, e[2], static_cast<std::uint32_t>(xs) | mul, wid);
            }
        }
        // heavy rows (degree > kHeavyMin, e.g. constant wires and padding
        // gates): one CTA per (slot, copy, row) instead of one thread
        auto heavy_items = [&](const std::vector<std::uint32_t>& off, DBuf<uint4>& dst) -> std::uint32_t {
            std::vector<std::pair<std::uint64_t, uint4>> items;
            for (std::size_t s2 = 0; s2 < ns; ++s2) {
                const std::uint32_t src = C.slots[s2];
                for (std::uint64_t xl = 0; xl < c.sub_padded[src]; ++xl) {
                    if (off[xbase[s2] + xl + 1] - off[xbase[s2] + xl] <= kHeavyMin) continue;
                    for (std::uint32_t cp = 0; cp < c.n_copies; ++cp)
                        items.push_back({(static_cast<std::uint64_t>(cp) << c.sub_log[src]) | xl,
                                         make_uint4(static_cast<std::uint32_t>(s2), cp, static_cast<std::uint32_t>(xl), 0)});
                }
            }
            std::stable_sort(items.begin(), items.end(),
                             [](const auto& a, const auto& b) { return a.first < b.first; });
            if (items.size() > 0x7fffffffu) fail(DGKR_UNSUPPORTED, "too many heavy rows");
            std::vector<uint4> v(items.size());
            for (std::size_t i = 0; i < items.size(); ++i) v[i] = items[i].second;
            if (!v.empty()) {
                dst.ensure(v.size());
                CK(cudaMemcpy(dst.p, v.data(), v.size() * sizeof(uint4), cudaMemcpyHostToDevice));
            }
            c.max_heavy = std::max<std::uint32_t>(c.max_heavy, static_cast<std::uint32_t>(v.size()));
            return static_cast<std::uint32_t>(v.size());
        };
        C.n_xheavy = heavy_items(xoff, C.xheavy);
        C.n_yheavy = heavy_items(yoff, C.yheavy);
        if (ns == 1) {
            // degree-sorted row order for the single-slot bookkeeping kernels
            const std::uint64_t S = c.sub_padded[C.slots[0]];
            auto sorted = [&](const std::vector<std::uint32_t>& off, DBuf<std::uint32_t>& dperm, DBuf<uint2>& dseg) {
                std::vector<std::uint32_t> perm(S);
                for (std::uint64_t i = 0; i < S; ++i) perm[i] = static_cast<std::uint32_t>(i);
                std::stable_sort(perm.begin(), perm.end(), [&](std::uint32_t a, std::uint32_t b) {
                    return off[a + 1] - off[a] > off[b + 1] - off[b];
                });
                std::vector<uint2> seg(S);
                for (std::uint64_t i = 0; i < S; ++i) seg[i] = make_uint2(off[perm[i]], off[perm[i] + 1] - off[perm[i]]);
                dperm.ensure(S);
                dseg.ensure(S);
                CK(cudaMemcpy(dperm.p, perm.data(), S * 4, cudaMemcpyHostToDevice));
                CK(cudaMemcpy(dseg.p, seg.data(), S * sizeof(uint2), cudaMemcpyHostToDevice));
            };
            sorted(xoff, C.xperm, C.xseg);
            sorted(yoff, C.yperm, C.yseg);
            // row pairs (2j, 2j+1) for the bookkeeping kernel with round 1 fused
            auto pairs = [&](const std::vector<std::uint32_t>& off, DBuf<uint4>& dps) {
                if (S < 2) return;
                const std::uint64_t np = S / 2;
                std::vector<std::uint32_t> order(np);
                auto deg = [&](std::uint64_t r) { return off[r + 1] - off[r]; };
                for (std::uint64_t j = 0; j < np; ++j) order[j] = static_cast<std::uint32_t>(j);
                std::stable_sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
                    return std::max(deg(2 * a), deg(2 * a + 1)) > std::max(deg(2 * b), deg(2 * b + 1));
                });
                std::vector<uint4> ps(np);
                for (std::uint64_t k = 0; k < np; ++k) {
                    const std::uint32_t j = order[k];
                    ps[k] = make_uint4(off[2 * j], deg(2 * j), deg(2 * j + 1), 2 * j);
                }
                dps.ensure(np);
                CK(cudaMemcpy(dps.p, ps.data(), np * sizeof(uint4), cudaMemcpyHostToDevice));
            };
            pairs(xoff, C.xpseg);
            pairs(yoff, C.ypseg);
        }
        C.xoff.ensure(xoff.size());
        C.yoff.ensure(yoff.size());
        C.xent.ensure(nw);
        C.yent.ensure(nw);
        CK(cudaMemcpy(C.xoff.p, xoff.data(), xoff.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(C.yoff.p, yoff.data(), yoff.size() * 4, cudaMemcpyHostToDevice));
        if (nw) {
            CK(cudaMemcpy(C.xent.p, xent.data(), nw * sizeof(uint4), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(C.yent.p, yent.data(), nw * sizeof(uint4), cudaMemcpyHostToDevice));
        }
        // evaluation CSR (gate -> nested)
        const std::uint64_t ng = lgs[li] - lgs[li - 1];
        std::vector<std::uint32_t> gstart(ng + 1);
        std::vector<uint4> nest(nw);
        for (std::uint64_t g = 0; g < ng; ++g) gstart[g] = static_cast<std::uint32_t>(gns[lgs[li - 1] + g] - gns[lgs[li - 1]]);
        gstart[ng] = static_cast<std::uint32_t>(gns[lgs[li]] - gns[lgs[li - 1]]);
        for (std::uint64_t k = gns[lgs[li - 1]], i = 0; k < gns[lgs[li]]; ++k, ++i) {
            const std::uint32_t* e = nested + 5 * k;
            nest[i] = make_uint4((e[0] ? 1u : 0u) | (e[1] << 1) | (e[3] << 16), e[2], e[4], 0);
        }
        // evaluation order: gates with more mul wires first (uniform warps)
        {
            std::vector<std::uint32_t> nmul(ng, 0), ep(ng);
            for (std::uint64_t g = 0; g < ng; ++g) {
                ep[g] = static_cast<std::uint32_t>(g);
                for (std::uint32_t k = gstart[g]; k < gstart[g + 1]; ++k) nmul[g] += nest[k].x & 1u;
            }
            std::stable_sort(ep.begin(), ep.end(), [&](std::uint32_t x, std::uint32_t y) {
                return nmul[x] != nmul[y] ? nmul[x] > nmul[y] : gstart[x + 1] - gstart[x] > gstart[y + 1] - gstart[y];
            });
            C.eperm.ensure(std::max<std::uint64_t>(ng, 1));
            if (ng) CK(cudaMemcpy(C.eperm.p, ep.data(), ng * 4, cudaMemcpyHostToDevice));
        }
        C.gstart.ensure(ng + 1);
        C.nested.ensure(nw);
        CK(cudaMemcpy(C.gstart.p, gstart.data(), (ng + 1) * 4, cudaMemcpyHostToDevice));
        if (nw) CK(cudaMemcpy(C.nested.p, nest.data(), nw * sizeof(uint4), cudaMemcpyHostToDevice));
        c.cons[li] = std::move(cp);
        (void)xslot_start;
        (void)yslot_start;
    }
    std::vector<std::uint32_t> ll(D + 1);
    for (std::uint32_t l = 0; l <= D; ++l) ll[l] = c.sub_log[l];
    c.d_layer_log.ensure(D + 1);
    CK(cudaMemcpy(c.d_layer_log.p, ll.data(), ll.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());  // see workspace(): setup DMA must land before lane streams run
    (void)ctx;
}

/// Per-lane device workspace of a circuit: layer values, bookkeeping and
/// fold scratch, split-eq tables. Built on first use by a lane.
CircuitWs& workspace(dgkr_circuit& c, int lane) {
    std::lock_guard<std::mutex> lk(c.ws_mu);
    if (static_cast<int>(c.ws.size()) <= lane) c.ws.resize(lane + 1);
    if (c.ws[lane]) return *c.ws[lane];
    auto wp = std::make_unique<CircuitWs>();
    CircuitWs& W = *wp;
    const std::uint32_t D = c.depth;
    for (std::uint32_t l = 0; l <= D; ++l) {
        auto b = std::make_unique<DBuf<Fe>>();
        b->ensure(c.capacity[l]);
        W.values.push_back(std::move(b));
    }
    std::vector<const Fe*> lv(D + 1);
    for (std::uint32_t l = 0; l <= D; ++l) lv[l] = W.values[l]->p;
    W.d_layer_vals.ensure(D + 1);
    CK(cudaMemcpy(W.d_layer_vals.p, lv.data(), lv.size() * sizeof(const Fe*), cudaMemcpyHostToDevice));
    if (D >= 1) {
        W.H.ensure(static_cast<std::size_t>(c.max_slots) * c.Tmax);
        W.G.ensure(c.Tmax);
        // per-gate weights are indexed by consumer gate: a layer may have more
        // gates than its (padded) source tables have entries
        std::uint64_t gmax = 1;
        for (std::uint32_t l = 1; l <= D; ++l) gmax = std::max(gmax, c.full_padded[l]);
        W.Wg.ensure(gmax);
        W.EqU.ensure(c.Tmax);
        {  // hi rows of a split eq: 2^(nv - ceil(nv/2)); headroom for the rank bits of up to 16 ranks
            unsigned lg = 0;
            while ((std::uint64_t{1} << lg) < std::max(gmax, c.Tmax)) ++lg;
            W.eq_hc.ensure(std::size_t{9} << (lg / 2 + 2));
        }
        W.rb.ensure(2 * static_cast<int>(c.max_slots) + 1, c.Tmax, cudaStreamLegacy);
        W.heavy_scr.ensure(2 * static_cast<std::size_t>(std::max<std::uint32_t>(c.max_heavy, 1)));
    }
    W.cons.resize(D + 1);
    for (std::uint32_t li = 1; li <= D; ++li) {
        auto& C = *c.cons[li];
        auto wc = std::make_unique<CircuitWs::Cons>();
        const std::size_t ns = C.slots.size();
        std::vector<SlotDesc> s1(ns), s2(ns);
        std::uint64_t base = 0;
        for (std::size_t s = 0; s < ns; ++s) {
            const std::uint32_t src = C.slots[s];
            // stride of a slot = sub padded size of its source (copy = high bits)
            const std::uint32_t lstr = (c.n_copies > 1) ? c.sub_log[src] : c.padded_log2_full(src);
            s1[s] = SlotDesc{W.values[src]->p, W.H.p + s * c.Tmax, C.xoff.p + base, C.xent.p, lstr, 0};
            s2[s] = SlotDesc{W.values[src]->p, W.H.p + s * c.Tmax, C.yoff.p + base, C.yent.p, lstr, 0};
            base += c.sub_padded[src] + 1;
        }
        wc->d_slots1.ensure(ns);
        wc->d_slots2.ensure(ns);
        CK(cudaMemcpy(wc->d_slots1.p, s1.data(), ns * sizeof(SlotDesc), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(wc->d_slots2.p, s2.data(), ns * sizeof(SlotDesc), cudaMemcpyHostToDevice));
        std::vector<const Fe*> bp;
        for (std::size_t s = 0; s < ns; ++s) {
            bp.push_back(W.values[C.slots[s]]->p);
            bp.push_back(W.H.p + s * c.Tmax);
        }
        bp.push_back(W.G.p);
        wc->base_ptrs.ensure(bp.size());
        CK(cudaMemcpy(wc->base_ptrs.p, bp.data(), bp.size() * sizeof(const Fe*), cudaMemcpyHostToDevice));
        wc->base_host = bp;
        W.cons[li] = std::move(wc);
    }
    // the setup copies above are synchronous cudaMemcpy from pageable memory:
    // wait for their DMA before any lane stream (non-blocking) reads the tables
    CK(cudaDeviceSynchronize());
    c.ws[lane] = std::move(wp);
    return *c.ws[lane];
}

// ---------------------------------------------------------------------------
// Claims (gkr.hpp:20-84, :157-173) — host, order-sensitive, verbatim.
// ---------------------------------------------------------------------------
struct ClaimTerm {
    std::vector<U256> point;
    U256 weight;
};
struct LayerClaim {
    std::size_t layer = 0;
    std::vector<ClaimTerm> terms;
    U256 value;
};

LayerClaim combine_claims(std::vector<LayerClaim> claims, Transcript& tr, const HostField& F,
                          std::vector<U256>* alphas) {
    if (claims.empty()) fail(DGKR_INVALID_ARGUMENT, "no claims to combine");
    for (const auto& c : claims)
        if (c.layer != claims.front().layer) fail(DGKR_INVALID_ARGUMENT, "claims span different layers");
    if (claims.size() == 1) return std::move(claims.front());
    const U256 alpha = tr.challenge();
    if (alphas) alphas->push_back(alpha);
    LayerClaim out;
    out.layer = claims.front().layer;
    U256 scale = F.one();
    for (auto& c : claims) {
        out.value = F.add(out.value, F.mul(scale, c.value));
        for (auto& t : c.terms) {
            const U256 w = F.mul(scale, t.weight);
            bool merged = false;
            for (auto& ot : out.terms) {
                if (ot.point == t.point) {
                    ot.weight = F.add(ot.weight, w);
                    merged = true;
                    break;
                }
            }
            if (!merged) out.terms.push_back(ClaimTerm{std::move(t.point), w});
        }
        scale = F.mul(scale, alpha);
    }
    return out;
}

LayerClaim shrink_claim(std::size_t layer, std::size_t native, const std::vector<U256>& point, const U256& value,
                        const HostField& F) {
    U256 w = F.one();
    for (std::size_t k = native; k < point.size(); ++k) w = F.mul(w, F.sub(F.one(), point[k]));
    LayerClaim c;
    c.layer = layer;
    c.terms.push_back(ClaimTerm{std::vector<U256>(point.begin(), point.begin() + static_cast<std::ptrdiff_t>(native)), w});
    c.value = value;
    return c;
}

/// Build split-eq tables on the device: for each (point, seed) pair, A =
/// seed * eq(point[0..klo)), B = eq(point[klo..)). Returns the SplitEq view
/// rooted at `dst` (which must hold K*(2^klo + 2^khi) elements).
SplitEq build_split_eq(Lane* ctx, const dgkr_field* f, const std::vector<std::vector<U256>>& points,
                       const std::vector<U256>& seeds, Fe* dst, DBuf<EqJob>& jobs_buf, std::size_t small_off) {
    const int K = static_cast<int>(points.size());
    const int nv = K ? static_cast<int>(points[0].size()) : 0;
    const int klo = (nv + 1) / 2, khi = nv - klo;
    SplitEq e;
    e.K = K;
    e.klo = klo;
    e.khi = khi;
    e.A = dst;
    e.B = dst + static_cast<std::size_t>(K) * (std::size_t{1} << klo);
    // stage points and seeds in the small buffer
    const std::size_t limit = small_off < Lane::kEqOff2 ? Lane::kEqOff2 : Lane::kVxOff;
    if (small_off + static_cast<std::size_t>(K) * (nv + 2) > limit) fail(DGKR_UNSUPPORTED, "too many claim terms");
    Fe* hs = ctx->h_small + small_off;
    Fe* ds = ctx->d_small.p + small_off;
    std::size_t pos = 0;
    std::vector<EqJob> jobs;
    const U256 one = f->f.one();
    for (int t = 0; t < K; ++t) {
        const std::size_t pt_off = pos;
        for (int k = 0; k < nv; ++k) hs[pos++] = to_fe(points[t][k]);
        const std::size_t seed_off = pos;
        hs[pos++] = to_fe(seeds[t]);
        const std::size_t one_off = pos;
        hs[pos++] = to_fe(one);
        jobs.push_back(EqJob{ds + pt_off, ds + seed_off, const_cast<Fe*>(e.A) + (static_cast<std::size_t>(t) << klo), klo, 0});
        jobs.push_back(EqJob{ds + pt_off + klo, ds + one_off, const_cast<Fe*>(e.B) + (static_cast<std::size_t>(t) << khi), khi, 0});
    }
    ctx->h2d(ds, hs, pos * sizeof(Fe));
    jobs_buf.ensure(jobs.size() + 64);
    // jobs go right after any previous jobs in jobs_buf: caller uses distinct buffers per build
    ctx->h2d(jobs_buf.p, jobs.data(), jobs.size() * sizeof(EqJob));
    launch_eq_build(ctx->use(f), jobs_buf.p, static_cast<int>(jobs.size()), ctx->st);
    ctx->launched();
    return e;
}

/// fold_pow for the constant-multiplier split-eq expansion, after sizing the
/// row-constant scratch for this expansion (null: the generic path)
const std::uint8_t* eq_fold_pow(const dgkr_field* f, CircuitWs& W, const SplitEq& e) {
    if (f->kind != FieldKind::Bn254 || e.K != 1) return nullptr;
    W.eq_hc.ensure(std::size_t{9} << e.khi);
    return reinterpret_cast<const std::uint8_t*>(f->fold_pow);
}

void load_inputs(Lane* ctx, dgkr_circuit& c, CircuitWs& W, const dgkr_field* f, const std::uint8_t* inputs) {
    const std::uint64_t n_in = static_cast<std::uint64_t>(c.input_size) * c.n_copies;
    Fe* v0 = W.values[0]->p;
    ctx->upload_elems(f, inputs, n_in, v0, W.stage);
    if (c.capacity[0] > n_in) CK(cudaMemsetAsync(v0 + n_in, 0, (c.capacity[0] - n_in) * sizeof(Fe), ctx->st));
    W.inputs_loaded = true;
}

void evaluate_layers(Lane* ctx, dgkr_circuit& c, CircuitWs& W, const dgkr_field* f) {
    if (!W.inputs_loaded) fail(DGKR_LOGIC_ERROR, "circuit inputs not loaded");
    const FieldKind kind = ctx->use(f);
    for (std::uint32_t li = 1; li <= c.depth; ++li) {
        auto& C = *c.cons[li];
        EvalLaunch el;
        el.out = W.values[li]->p;
        el.n_write = c.capacity[li];
        el.n_gates = c.sub_size[li] * c.n_copies;
        el.log_g = (c.n_copies > 1) ? c.sub_log[li] : 63;
        el.gstart = C.gstart.p;
        el.nested = C.nested.p;
        el.perm = C.eperm.p;
        el.layer_vals = W.d_layer_vals.p;
        el.layer_log_stride = c.d_layer_log.p;
        if (ctx->profile_on) CK(cudaEventRecord(ctx->ev0, ctx->st));
        launch_evaluate(kind, el, ctx->st);
        ctx->launched();
        if (ctx->profile_on) {
            CK(cudaEventRecord(ctx->ev1, ctx->st));
            CK(cudaEventSynchronize(ctx->ev1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
            ctx->prof.evaluate_ms += ms;
        }
    }
}

void evaluate_circuit(Lane* ctx, dgkr_circuit& c, CircuitWs& W, const dgkr_field* f, const std::uint8_t* inputs) {
    load_inputs(ctx, c, W, f, inputs);
    evaluate_layers(ctx, c, W, f);
}

/// gkr_prove (gkr.hpp:182-244) on the device-resident circuit. The proof is
/// written straight into the caller's buffer (the claimed outputs, by far
/// its largest part, land there by D2H); returns the proof length.
/// comm != nullptr: this rank's share of a distributed proof; `root` is the
/// rank that gathers the claimed outputs and runs their serial absorb (the
/// other ranks' proof bytes carry zeros in the output section).
std::size_t gkr_prove(Lane* ctx, dgkr_circuit& c, CircuitWs& W, const dgkr_field* f, const std::uint8_t* inputs,
                      Transcript& tr, std::uint8_t* out, std::size_t cap, dgkr_comm* comm = nullptr, int root = 0,
                      AbsorbPool* pool = nullptr) {
    const HostField& F = f->f;
    const FieldKind kind = ctx->use(f);
    const std::size_t w = F.width();
    // distributed: this rank holds copies [rank*n, (rank+1)*n) of a
    // uniform-width data-parallel circuit; the rank index is the top log2(world)
    // variables of every layer (cluster.hpp:182-189).
    if (comm && comm->world == 1) comm = nullptr;  // a 1-rank communicator exchanges nothing
    const std::uint64_t world = comm ? static_cast<std::uint64_t>(comm->world) : 1;
    const std::uint64_t rank = comm ? static_cast<std::uint64_t>(comm->rank) : 0;
    const std::uint32_t lw = log2_exact(world);
    if (comm) {
        if ((world & (world - 1)) != 0) fail(DGKR_INVALID_ARGUMENT, "world size must be a power of two");
        for (std::uint32_t l = 0; l <= c.depth; ++l)
            if (c.sub_size[l] != c.sub_size[0] || c.sub_size[l] != c.sub_padded[l])
                fail(DGKR_INVALID_ARGUMENT, "distributed proving needs a uniform power-of-two layer width");
    }
    NvtxRange nv_prove("dgkr.gkr_prove");
    {
        NvtxRange nv("dgkr.evaluate");
        if (inputs) evaluate_circuit(ctx, c, W, f, inputs);  // gkr.hpp:186
        else evaluate_layers(ctx, c, W, f);
    }

    // absorb the padded output table (gkr.hpp:189-190): D2H canonical, serial SHA chain
    const std::uint32_t out_layer = c.depth;
    const std::uint64_t n_out_local = c.full_padded[out_layer];
    const std::uint64_t n_out = n_out_local * world;
    if (cap < 4 + n_out * w) fail(DGKR_CAPACITY, "output buffer too small");
    std::vector<std::uint8_t> proof;  // everything after the claimed outputs
    for (int i = 0; i < 4; ++i) out[i] = static_cast<std::uint8_t>(n_out >> (8 * i));
    {
        W.stage.ensure(n_out_local * w);
        launch_to_canonical(kind, W.values[out_layer]->p, W.stage.p, static_cast<int>(w), n_out_local, ctx->st);
        ctx->launched();
        if (comm) {
            // outputs in global order on the root only: it alone runs the serial absorb
            comm->gather_to_root_host(W.stage.p, out + 4, n_out_local * w, ctx, root);
        } else {
            ctx->d2h(out + 4, W.stage.p, n_out * w);
            ctx->sync();
        }
        if (!comm || comm->rank == root) {
            NvtxRange nv("dgkr.output_absorb");
            const double t0 = now_ms();
            // DGKR_DIAG_SKIP_OUTPUT_ABSORB=1: bottleneck diagnosis only (tools/diag_stream.py):
            // skips the absorb, so the proof is NOT the reference's; never set for a bench
            static const bool diag_skip = std::getenv("DGKR_DIAG_SKIP_OUTPUT_ABSORB") != nullptr;
            if (diag_skip) {
            } else if (pool && w == 32) {
                pool->run(tr.state_bytes(), out + 4, n_out);  // interleaved with other proofs' chains
            } else {
                tr.absorb_many(out + 4, n_out, w);
            }
            const double dt = now_ms() - t0;
            ctx->prof.output_absorb_ms += dt;
            ctx->prof.host_transcript_ms += dt;
        }
        if (comm) {
            // the absorbed transcript state goes to every rank (40 bytes)
            std::uint8_t st[40];
            std::memcpy(st, tr.state().data(), 32);
            const std::uint64_t draws = tr.draws();
            std::memcpy(st + 32, &draws, 8);
            comm->broadcast_host(st, 40, ctx, root);
            std::uint64_t d2;
            std::memcpy(&d2, st + 32, 8);
            tr = Transcript(&F, st, d2);
            if (comm->rank != root) std::memset(out + 4, 0, n_out * w);  // only the root holds the outputs
        }
    }
    // q and the output claim (gkr.hpp:192-202)
    const std::uint32_t qlen = c.padded_log2_full(out_layer) + lw;
    std::vector<U256> q;
    for (std::uint32_t k = 0; k < qlen; ++k) q.push_back(tr.challenge());
    // split-eq table space: (max claim terms + 1 u-table) x (2^ceil(L/2) + 2^floor(L/2))
    std::uint32_t lmax = log2_exact(c.Tmax) + lw;
    for (std::uint32_t l = 0; l <= c.depth; ++l) lmax = std::max(lmax, c.padded_log2_full(l) + lw);
    const std::size_t per_term = (std::size_t{1} << ((lmax + 1) / 2)) + (std::size_t{1} << (lmax / 2));
    const std::size_t max_terms = 2 * static_cast<std::size_t>(c.depth) * std::max<std::uint32_t>(c.max_slots, 1) + 2;
    W.eq_tabs.ensure((max_terms + 2) * per_term);
    U256 out_value;
    {
        SplitEq e = build_split_eq(ctx, f, {q}, {F.one()}, W.eq_tabs.p, W.eq_jobs, Lane::kEqOff);
        e.offset = rank * n_out_local;
        launch_dense_eval(kind, W.values[out_layer]->p, n_out_local, e, ctx->ws, ctx->st);
        ctx->launched();
        if (comm) {
            comm->allgather_to_host(ctx->ws.result, ctx->h_small + Lane::kGatherOff, sizeof(Fe), ctx);
            U256 acc{};
            for (std::uint64_t r = 0; r < world; ++r) acc = F.add(acc, to_u256(ctx->h_small[Lane::kGatherOff + r]));
            out_value = acc;
        } else {
            ctx->d2h(ctx->h_small + 1, ctx->ws.result, sizeof(Fe));
            ctx->sync();
            out_value = to_u256(ctx->h_small[1]);
        }
    }
    std::vector<std::vector<LayerClaim>> registry(out_layer + 1);
    {
        LayerClaim lc;
        lc.layer = out_layer;
        lc.terms.push_back(ClaimTerm{q, F.one()});
        lc.value = out_value;
        registry[out_layer].push_back(std::move(lc));
    }
    put32(proof, out_layer);
    // chi_x(u) of the previous (consumer) layer's phase 2 stays in W.EqU; it is
    // the first claim term of the next layer in uniform layered circuits
    std::vector<U256> equ_point;
    std::uint64_t equ_n = 0;
    for (std::uint32_t layer = out_layer; layer >= 1; --layer) {
        auto& C = *c.cons[layer];
        auto& WC = *W.cons[layer];
        const std::string nv_name = "dgkr.layer " + std::to_string(layer);
        NvtxRange nv_layer(nv_name.c_str());
        std::vector<U256> alphas;
        const double th = now_ms();
        LayerClaim combined = combine_claims(std::move(registry[layer]), tr, F, &alphas);  // gkr.hpp:206-207
        ctx->prof.host_transcript_ms += now_ms() - th;
        registry[layer].clear();
        const std::uint32_t side = C.side;
        const std::uint64_t T = std::uint64_t{1} << side;
        const int ns = static_cast<int>(C.slots.size());
        // wire weights (gkr.hpp:135-152) as split-eq tables of the claim terms
        std::vector<std::vector<U256>> pts;
        std::vector<U256> seeds;
        for (const auto& t : combined.terms) {
            pts.push_back(t.point);
            seeds.push_back(t.weight);
        }
        const std::uint32_t lgc = c.padded_log2_full(layer) + lw;
        for (auto& p : pts)
            if (p.size() != lgc) fail(DGKR_LOGIC_ERROR, "claim point length mismatch");
        if (pts.size() > max_terms) fail(DGKR_UNSUPPORTED, "too many claim terms");
        const std::uint64_t n_gates_local = c.sub_size[layer] * c.n_copies;
        // w(g) = chi_g(u) + alpha chi_g(v): reuse the dense chi_x(u) table when
        // term 0 is exactly (u, 1) over the same index range (one mult per gate saved)
        const bool reuse_u = pts.size() == 2 && equ_n == n_gates_local && seeds[0] == F.one() && pts[0] == equ_point;
        if (reuse_u) {
            pts.erase(pts.begin());
            seeds.erase(seeds.begin());
        }
        SplitEq wq = build_split_eq(ctx, f, pts, seeds, W.eq_tabs.p, W.eq_jobs, Lane::kEqOff);
        wq.offset = rank * n_gates_local;  // global gate index of local gate 0
        const std::size_t wq_elems = pts.size() * ((std::size_t{1} << wq.klo) + (std::size_t{1} << wq.khi));

        // prove_layer_sum (sumcheck.hpp:342-448)
        tr.absorb(combined.value);  // :364
        BookkeepLaunch bk;
        bk.slots = WC.d_slots1.p;
        bk.n_slots = ns;
        bk.T = T;
        bk.n_copies = c.n_copies;
        bk.log_gcons = (c.n_copies > 1) ? c.sub_log[layer] : 63;
        bk.G = W.G.p;
        bk.w = wq;
        if (ctx->profile_on) CK(cudaEventRecord(ctx->ev0, ctx->st));
        const std::uint8_t* fp_w = eq_fold_pow(f, W, wq);  // sizes W.eq_hc first
        if (reuse_u)
            launch_split_eq_expand_add(kind, wq, n_gates_local, W.EqU.p, W.Wg.p, ctx->st, fp_w, W.eq_hc.p);
        else
            launch_split_eq_expand(kind, wq, n_gates_local, W.Wg.p, ctx->st, fp_w, W.eq_hc.p);  // w(g), gkr.hpp:140-148
        ctx->launched();
        bk.gate_w = W.Wg.p;
        bk.perm = C.xperm.p;
        bk.seg = C.xseg.p;
        bk.heavy_min = kHeavyMin;
        bk.heavy_h = W.heavy_scr.p;
        bk.heavy_g = W.heavy_scr.p + std::max<std::uint32_t>(c.max_heavy, 1);
        bk.heavy = C.xheavy.p;
        bk.n_heavy = C.n_xheavy;
        // row pairs with round 1 fused: single slot, no heavy rows, a full pair table
        const bool fuse1 = fuse_round1() && C.xpseg.p && C.n_xheavy == 0 && ns == 1 && side >= 2 &&
                           c.sub_log[C.slots[0]] + c.log_copies == side;
        bk.pseg = fuse1 ? C.xpseg.p : nullptr;
        bk.r1 = ctx->ws;
        launch_bookkeep_phase1(kind, bk, ctx->st);
        ctx->launched();
        if (ctx->profile_on) {
            CK(cudaEventRecord(ctx->ev1, ctx->st));
            CK(cudaEventSynchronize(ctx->ev1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
            ctx->prof.bookkeep_ms += ms;
        }
        nvtxRangePushA("dgkr.phase1 rounds");
        SumcheckRun p1 =
            comm ? run_rounds_dist(ctx, f, ns, true, static_cast<int>(side), WC.base_ptrs.p, W.rb, tr, comm, W.dist,
                                   &combined.value, WC.base_host.data(), fuse1)
                 : run_rounds(ctx, f, ns, true, static_cast<int>(side), WC.base_ptrs.p, W.rb, tr, nullptr,
                              &combined.value, WC.base_host.data(), fuse1);
        nvtxRangePop();
        std::vector<U256> vx(ns);
        for (int m = 0; m < ns; ++m) vx[m] = p1.finals[2 * m];
        // phase 2 (sumcheck.hpp:407-431): chi_x(u) split tables + V_m(u)
        std::vector<U256> one_seed{F.one()};
        SplitEq uq = build_split_eq(ctx, f, {p1.challenges}, one_seed, W.eq_tabs.p + wq_elems, W.eq_jobs2,
                                    Lane::kEqOff2);
        uq.offset = rank * T;  // this rank's slice of the x hypercube
        // vx to device
        for (int m = 0; m < ns; ++m) ctx->h_small[Lane::kVxOff + m] = to_fe(vx[m]);
        ctx->h2d(ctx->d_small.p + Lane::kVxOff, ctx->h_small + Lane::kVxOff, ns * sizeof(Fe));
        bk.slots = WC.d_slots2.p;
        bk.u = uq;
        bk.vx = ctx->d_small.p + Lane::kVxOff;
        U256 vxk[9];
        f->fold_const(vx[0], vxk);
        bk.vx_const = vxk;
        if (ctx->profile_on) CK(cudaEventRecord(ctx->ev0, ctx->st));
        const std::uint8_t* fp_u = eq_fold_pow(f, W, uq);
        launch_split_eq_expand(kind, uq, T, W.EqU.p, ctx->st, fp_u, W.eq_hc.p);  // chi_x(u), sumcheck.hpp:415
        equ_point = p1.challenges;
        equ_n = T;
        ctx->launched();
        bk.eq_u = W.EqU.p;
        bk.perm = C.yperm.p;
        bk.seg = C.yseg.p;
        bk.heavy = C.yheavy.p;
        bk.n_heavy = C.n_yheavy;
        const bool fuse2 = fuse_round1() && C.ypseg.p && C.n_yheavy == 0 && ns == 1 && side >= 2 &&
                           c.sub_log[C.slots[0]] + c.log_copies == side && bk.vx_const;
        bk.pseg = fuse2 ? C.ypseg.p : nullptr;
        launch_bookkeep_phase2(kind, bk, ctx->st);
        ctx->launched();
        if (ctx->profile_on) {
            CK(cudaEventRecord(ctx->ev1, ctx->st));
            CK(cudaEventSynchronize(ctx->ev1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
            ctx->prof.bookkeep_ms += ms;
        }
        nvtxRangePushA("dgkr.phase2 rounds");
        SumcheckRun p2 =
            comm ? run_rounds_dist(ctx, f, ns, true, static_cast<int>(side), WC.base_ptrs.p, W.rb, tr, comm, W.dist,
                                   &p1.claim_end, WC.base_host.data(), fuse2)
                 : run_rounds(ctx, f, ns, true, static_cast<int>(side), WC.base_ptrs.p, W.rb, tr, nullptr,
                              &p1.claim_end, WC.base_host.data(), fuse2);
        nvtxRangePop();
        std::vector<U256> finals = vx;
        for (int m = 0; m < ns; ++m) finals.push_back(p2.finals[2 * m]);
        std::vector<RoundPoly> rounds = p1.rounds;
        rounds.insert(rounds.end(), p2.rounds.begin(), p2.rounds.end());
        // registry (gkr.hpp:225-233)
        for (int s = 0; s < ns; ++s) {
            const std::uint32_t src = C.slots[s];
            const std::uint32_t native = c.padded_log2_full(src) + lw;
            registry[src].push_back(shrink_claim(src, native, p1.challenges, finals[s], F));
            registry[src].push_back(shrink_claim(src, native, p2.challenges, finals[ns + s], F));
        }
        // layer proof bytes
        put32(proof, static_cast<std::uint32_t>(alphas.size()));
        for (const auto& a : alphas) append_elem(proof, F, a);
        const auto sb = sumcheck_bytes(F, combined.value, rounds, finals);
        put32(proof, static_cast<std::uint32_t>(sb.size()));
        proof.insert(proof.end(), sb.begin(), sb.end());
    }
    const std::size_t total = 4 + n_out * w + proof.size();
    if (total > cap) fail(DGKR_CAPACITY, "output buffer too small");
    std::memcpy(out + 4 + n_out * w, proof.data(), proof.size());
    return total;
}

// ---------------------------------------------------------------------------
// PCS (pcs.hpp) on device
// ---------------------------------------------------------------------------
void pcs_build_tree(Lane* ctx, const dgkr_field* f, PcsDevice& d, std::size_t rows, std::size_t cols) {
    d.nodes.ensure(2 * cols * 32);
    ctx->tbeg();
    launch_column_digests(ctx->use(f), d.m.p, cols, static_cast<int>(rows), static_cast<int>(f->f.width()),
                          d.nodes.p + cols * 32, ctx->st);
    ctx->launched();
    launch_merkle(d.nodes.p, cols, ctx->st);
    ctx->tend(ctx->prof.merkle_ms);
    ctx->launched(cols > 1 ? log2_exact(cols) : 0);
}

void check_matrix(std::size_t rows, std::size_t cols) {
    if (rows == 0 || cols == 0 || (cols & (cols - 1)) != 0 || (rows & (rows - 1)) != 0)
        fail(DGKR_INVALID_ARGUMENT, "matrix dimensions must be nonzero powers of two");  // pcs.hpp:26-29
}

Digest pcs_commit(Lane* ctx, const dgkr_field* f, PcsDevice& d, std::size_t rows, std::size_t cols,
                  const std::uint8_t* data) {
    check_matrix(rows, cols);
    d.m.ensure(rows * cols);
    ctx->upload_elems(f, data, rows * cols, d.m.p, d.stage);
    pcs_build_tree(ctx, f, d, rows, cols);
    Digest root;
    ctx->d2h(root.data(), d.nodes.p + 32, 32);
    ctx->sync();
    return root;
}

U256 chi_eval_host(std::uint64_t index, const std::vector<U256>& point, const HostField& F) {  // mle.hpp:111-120
    U256 acc = F.one();
    for (std::size_t k = 0; k < point.size(); ++k)
        acc = F.mul(acc, ((index >> k) & 1) ? point[k] : F.sub(F.one(), point[k]));
    return acc;
}

/// pcs::open (pcs.hpp:212-254) -> Opening::to_bytes
/// Opening::to_bytes size (pcs.hpp:135-156)
std::size_t pcs_opening_size(std::size_t w, std::size_t r_len, std::size_t rows, std::size_t cols, std::size_t q) {
    const std::size_t nq = std::min(q, cols);
    return 4 + r_len * w + w + 4 + rows * w + 4 + cols * w + 4 + nq * (4 + rows * w + 32 * log2_exact(cols));
}

/// pcs::open (pcs.hpp:212-254), written straight into `out` (cap bytes):
/// the combined row lands in place by one D2H and is absorbed from there.
/// Returns the opening's length.
/// resident: d.m and d.nodes already hold this matrix and its tree (the
/// commit of the same rows just before, as in DistPc::commit -> open); the
/// reference rebuilds them (pcs.hpp:241-244), which gives the same bytes.
std::size_t pcs_open(Lane* ctx, const dgkr_field* f, PcsDevice& d, std::size_t rows, std::size_t cols,
                     const std::uint8_t* data, const std::vector<U256>& r, std::size_t q, Transcript& tr,
                     U256* value_out, std::uint8_t* out, std::size_t cap, bool resident = false) {
    check_matrix(rows, cols);
    const HostField& F = f->f;
    const FieldKind kind = ctx->use(f);
    const std::size_t w = F.width();
    const std::uint32_t row_vars = log2_exact(cols), index_vars = log2_exact(rows);
    if (r.size() != row_vars + index_vars) fail(DGKR_INVALID_ARGUMENT, "opening point has wrong dimension");
    const std::size_t total = pcs_opening_size(w, r.size(), rows, cols, q);
    if (total > cap) fail(DGKR_CAPACITY, "output buffer too small");
    if (!resident) {
        d.m.ensure(rows * cols);
        ctx->upload_elems(f, data, rows * cols, d.m.p, d.stage);
    }
    std::vector<U256> r_low(r.begin(), r.begin() + row_vars), r_high(r.begin() + row_vars, r.end());
    std::vector<U256> beta(rows);
    for (std::size_t i = 0; i < rows; ++i) beta[i] = chi_eval_host(i, r_high, F);  // pcs.hpp:161-170
    // row evaluations (dense MLE at r_low, split-eq tables): one launch per
    // row, each result copied out behind its launch, one sync for all rows
    d.eqt.ensure(2 * ((std::size_t{1} << ((row_vars + 1) / 2)) + (std::size_t{1} << (row_vars / 2))) + 8);
    SplitEq e = build_split_eq(ctx, f, {r_low}, {F.one()}, d.eqt.p, d.jobs, 16);
    if (rows > Lane::kGatherOff - Lane::kFinalsOff) fail(DGKR_UNSUPPORTED, "too many matrix rows");
    Fe* hre = ctx->h_small + Lane::kFinalsOff;
    for (std::size_t i = 0; i < rows; ++i) {
        launch_dense_eval(kind, d.m.p + i * cols, cols, e, ctx->ws, ctx->st);
        ctx->launched();
        ctx->d2h(hre + i, ctx->ws.result, sizeof(Fe));
    }
    // combined row (pcs.hpp:233-239)
    d.comb.ensure(cols);
    d.beta.ensure(rows);
    std::vector<Fe> hb(rows);
    for (std::size_t i = 0; i < rows; ++i) hb[i] = to_fe(beta[i]);
    ctx->h2d(d.beta.p, hb.data(), rows * sizeof(Fe));
    launch_beta_combine(kind, d.m.p, cols, static_cast<int>(rows), d.beta.p, d.comb.p, ctx->st);
    ctx->launched();
    // leaves + tree (pcs.hpp:241-244)
    if (!resident) pcs_build_tree(ctx, f, d, rows, cols);
    ctx->sync();
    std::vector<U256> row_evals(rows);
    U256 value{};
    for (std::size_t i = 0; i < rows; ++i) {
        row_evals[i] = to_u256(hre[i]);
        value = F.add(value, F.mul(beta[i], row_evals[i]));
    }
    // Opening::to_bytes head (pcs.hpp:135-156): |r|, r, value, M, row evals, cols, combined row
    std::size_t pos = 0;
    auto put_u32 = [&](std::uint32_t v) {
        for (int i = 0; i < 4; ++i) out[pos++] = static_cast<std::uint8_t>(v >> (8 * i));
    };
    auto put_elem = [&](const U256& x) {
        F.to_bytes(x, out + pos);
        pos += w;
    };
    put_u32(static_cast<std::uint32_t>(r.size()));
    for (const auto& x : r) put_elem(x);
    put_elem(value);
    put_u32(static_cast<std::uint32_t>(rows));
    for (const auto& x : row_evals) put_elem(x);
    put_u32(static_cast<std::uint32_t>(cols));
    std::uint8_t* combined = out + pos;
    d.stage.ensure(cols * w);
    launch_to_canonical(kind, d.comb.p, d.stage.p, static_cast<int>(w), cols, ctx->st);
    ctx->launched();
    ctx->d2h_large(combined, d.stage.p, cols * w);
    pos += cols * w;
    Digest root;
    ctx->d2h(root.data(), d.nodes.p + 32, 32);
    ctx->sync();
    // derive_spot_indices (pcs.hpp:185-208): serial transcript
    const double t0 = now_ms();
    tr.absorb_bytes(root.data(), 32);
    for (const auto& x : r) tr.absorb(x);
    tr.absorb(value);
    for (const auto& x : row_evals) tr.absorb(x);
    tr.absorb_many(combined, cols, w);
    std::vector<std::uint64_t> idx;
    if (q >= cols) {
        for (std::uint64_t j = 0; j < cols; ++j) idx.push_back(j);
    } else {
        std::vector<bool> seen(cols, false);
        while (idx.size() < q) {
            const std::uint64_t j = tr.challenge_index(cols);
            if (!seen[j]) {
                seen[j] = true;
                idx.push_back(j);
            }
        }
    }
    ctx->prof.host_transcript_ms += now_ms() - t0;
    // spot checks: column + Merkle path (merkle.hpp:34-45) each; all path
    // digests gathered on the device into one buffer, one copy back
    const std::size_t depth = log2_exact(cols);
    std::vector<std::uint64_t> nodes;
    nodes.reserve(idx.size() * depth);
    for (std::uint64_t j : idx)
        for (std::size_t node = cols + j; node > 1; node >>= 1) nodes.push_back(node ^ 1);
    std::vector<std::uint8_t> paths(nodes.size() * 32);
    if (!nodes.empty()) {
        d.path_idx.ensure(nodes.size());
        d.path_out.ensure(nodes.size() * 32);
        ctx->h2d(d.path_idx.p, nodes.data(), nodes.size() * sizeof(std::uint64_t));
        launch_gather32(d.nodes.p, d.path_idx.p, nodes.size(), d.path_out.p, ctx->st);
        ctx->launched();
        ctx->d2h(paths.data(), d.path_out.p, paths.size());
        ctx->sync();
    }
    put_u32(static_cast<std::uint32_t>(idx.size()));
    for (std::size_t s = 0; s < idx.size(); ++s) {
        const std::uint64_t j = idx[s];
        put_u32(static_cast<std::uint32_t>(j));
        for (std::size_t i = 0; i < rows; ++i) {
            std::memcpy(out + pos, data + (i * cols + j) * w, w);
            pos += w;
        }
        std::memcpy(out + pos, paths.data() + s * depth * 32, depth * 32);
        pos += depth * 32;
    }
    if (pos != total) fail(DGKR_LOGIC_ERROR, "opening size mismatch");
    if (value_out) *value_out = value;
    return pos;
}

// ---------------------------------------------------------------------------
// TrafficStats (cluster.hpp:69-115), byte-accurate logical metering.
// ---------------------------------------------------------------------------
struct Traffic {
    struct P {
        std::uint64_t w2w = 0, w2m = 0, m2w = 0, mempool = 0;
    };
    P total;
    std::vector<std::pair<std::string, P>> phases;  // sorted on output (std::map order)
    std::string cur = "setup";
    P& ph() {
        for (auto& p : phases)
            if (p.first == cur) return p.second;
        phases.push_back({cur, P{}});
        return phases.back().second;
    }
    void msg(std::size_t from, std::size_t to, std::size_t master, std::size_t bytes) {
        if (from == to) return;
        P& p = ph();
        if (to == master) {
            total.w2m += bytes;
            p.w2m += bytes;
        } else if (from == master) {
            total.m2w += bytes;
            p.m2w += bytes;
        } else {
            total.w2w += bytes;
            p.w2w += bytes;
        }
    }
    void mempool(std::size_t bytes) {
        total.mempool += bytes;
        ph().mempool += bytes;
    }
    std::string json() const {
        auto obj = [](const P& p) {
            return "{\"w2w\":" + std::to_string(p.w2w) + ",\"w2m\":" + std::to_string(p.w2m) +
                   ",\"m2w\":" + std::to_string(p.m2w) + ",\"mempool\":" + std::to_string(p.mempool) + "}";
        };
        std::string s = "{\"w2w\":" + std::to_string(total.w2w) + ",\"w2m\":" + std::to_string(total.w2m) +
                        ",\"m2w\":" + std::to_string(total.m2w) + ",\"mempool\":" + std::to_string(total.mempool) +
                        ",\"phases\":";
        if (phases.empty()) return s + "null}";
        auto sorted = phases;
        std::sort(sorted.begin(), sorted.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        s += "{";
        for (std::size_t i = 0; i < sorted.size(); ++i) {
            if (i) s += ",";
            s += "\"" + sorted[i].first + "\":" + obj(sorted[i].second);
        }
        return s + "}}";
    }
};

void write_json(const std::string& js, char* out, std::size_t cap) {
    if (!out) return;
    if (js.size() + 1 > cap) fail(DGKR_CAPACITY, "traffic json buffer too small");
    std::memcpy(out, js.c_str(), js.size() + 1);
}

/// ClusterTopology::plan (cluster.hpp:38-57) -> K
std::size_t plan_clusters(std::size_t n, std::size_t k) {
    if (n == 0 || (n & (n - 1)) != 0) fail(DGKR_INVALID_ARGUMENT, "worker count must be a nonzero power of two");
    if (k) {
        if (k > n || n % k != 0) fail(DGKR_INVALID_ARGUMENT, "cluster count must divide worker count");
        return k;
    }
    std::size_t log2n = log2_exact(n), clusters = 1;
    while (clusters < log2n) clusters <<= 1;
    return std::min(clusters, n);
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* dgkr_last_error(void) { return g_err.c_str(); }
int dgkr_abi_version(void) { return 3; }  // 3: dgkr_profile gained tail_ms / tail_rounds / tail_aborts

int dgkr_field_create(const std::uint8_t* mod, std::size_t len, dgkr_field** out) {
    return guard([&] {
        auto f = std::make_unique<dgkr_field>();
        f->f = HostField(mod, len);
        static const std::uint8_t bn[32] = {0x01, 0x00, 0x00, 0xf0, 0x93, 0xf5, 0xe1, 0x43, 0x91, 0x70, 0xb9,
                                            0x79, 0x48, 0xe8, 0x33, 0x28, 0x5d, 0x58, 0x81, 0x81, 0xb6, 0x45,
                                            0x50, 0xb8, 0x29, 0xa0, 0x31, 0xe1, 0x72, 0x4e, 0x64, 0x30};
        HostField bnf(bn, 32);
        f->kind = f->f.same(bnf) ? FieldKind::Bn254 : (f->f.bits() > 254 ? FieldKind::RuntimeWide : FieldKind::Runtime);
        for (int i = 0; i < 4; ++i) {
            f->rt.p[2 * i] = static_cast<std::uint32_t>(f->f.p().w[i]);
            f->rt.p[2 * i + 1] = static_cast<std::uint32_t>(f->f.p().w[i] >> 32);
            f->rt.r2[2 * i] = static_cast<std::uint32_t>(f->f.r2().w[i]);
            f->rt.r2[2 * i + 1] = static_cast<std::uint32_t>(f->f.r2().w[i] >> 32);
            f->rt.one[2 * i] = static_cast<std::uint32_t>(f->f.one().w[i]);
            f->rt.one[2 * i + 1] = static_cast<std::uint32_t>(f->f.one().w[i] >> 32);
        }
        f->rt.np0 = static_cast<std::uint32_t>(f->f.np0());
        U256 x{{1, 0, 0, 0}};  // canonical powers of two by modular doubling
        for (int b = 0; b < 64; ++b) x = f->f.add(x, x);
        for (int k = 0; k < 8; ++k) {
            f->fold_pow[k] = x;
            for (int b = 0; b < 32; ++b) x = f->f.add(x, x);
        }
        {  // 2-adic structure for the NTT / FRI (p - 1 = 2^s t, t odd)
            const HostField& F = f->f;
            U256 pm1, one{{1, 0, 0, 0}};
            sub_to(pm1, F.p(), one);
            U256 t = pm1;
            unsigned s = 0;
            while ((t.w[0] & 1) == 0 && !t.is_zero()) {
                for (int i = 0; i < 4; ++i) t.w[i] = (t.w[i] >> 1) | (i < 3 ? t.w[i + 1] << 63 : 0);
                ++s;
            }
            U256 half = pm1;  // (p-1)/2
            for (int i = 0; i < 4; ++i) half.w[i] = (half.w[i] >> 1) | (i < 3 ? half.w[i + 1] << 63 : 0);
            const U256 minus_one = F.neg(F.one());
            for (std::uint64_t z = 2; z < 1000; ++z) {
                const U256 zm = F.from_u64(z);
                if (F.pow(zm, half) == minus_one) {  // Euler: z is a non-residue
                    f->coset = zm;
                    f->coset_inv = F.inv(zm);
                    f->root = F.pow(zm, t);  // order exactly 2^s
                    f->two_adicity = s;
                    break;
                }
            }
        }
        *out = f.release();
    });
}
void dgkr_field_destroy(dgkr_field* f) { delete f; }
std::size_t dgkr_field_width(const dgkr_field* f) { return f ? f->f.width() : 0; }
std::size_t dgkr_field_bits(const dgkr_field* f) { return f ? f->f.bits() : 0; }

int dgkr_transcript_init(const dgkr_field* f, const char* label, dgkr_transcript* t) {
    return guard([&] {
        Transcript tr(&f->f, label ? label : "");
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = 0;
    });
}
int dgkr_transcript_absorb_bytes(const dgkr_field* f, dgkr_transcript* t, const std::uint8_t* d, std::size_t n) {
    return guard([&] {
        Transcript tr(&f->f, t->state, t->draws);
        tr.absorb_bytes(d, n);
        std::memcpy(t->state, tr.state().data(), 32);
    });
}
int dgkr_transcript_absorb_u64(const dgkr_field* f, dgkr_transcript* t, std::uint64_t v) {
    return guard([&] {
        Transcript tr(&f->f, t->state, t->draws);
        tr.absorb_u64(v);
        std::memcpy(t->state, tr.state().data(), 32);
    });
}
int dgkr_transcript_absorb_elems(const dgkr_field* f, dgkr_transcript* t, const std::uint8_t* e, std::size_t n) {
    return guard([&] {
        Transcript tr(&f->f, t->state, t->draws);
        const std::size_t w = f->f.width();
        for (std::size_t i = 0; i < n; ++i) f->f.from_bytes(e + i * w);  // canonical check (field.hpp:183-185)
        tr.absorb_many(e, n, w);
        std::memcpy(t->state, tr.state().data(), 32);
    });
}
int dgkr_transcript_absorb_elems_multi(const dgkr_field* f, dgkr_transcript* const* ts, std::size_t k,
                                       const std::uint8_t* const* elems, std::size_t n, int threads) {
    return guard([&] {
        const std::size_t w = f->f.width();
        for (std::size_t j = 0; j < k; ++j)
            for (std::size_t i = 0; i < n; ++i) f->f.from_bytes(elems[j] + i * w);  // canonical check
        if (w != 32 || threads <= 1) {  // one thread: the interleaved chains directly
            std::vector<std::uint8_t*> st(k);
            for (std::size_t j = 0; j < k; ++j) st[j] = ts[j]->state;
            if (w == 32) {
                absorb_chain32_multi(st.data(), elems, k, n);
            } else {
                for (std::size_t j = 0; j < k; ++j) {
                    Transcript tr(&f->f, ts[j]->state, ts[j]->draws);
                    tr.absorb_many(elems[j], n, w);
                    std::memcpy(ts[j]->state, tr.state().data(), 32);
                }
            }
            return;
        }
        // one host thread per transcript through the combining scheduler of
        // the proof stream (AbsorbPool): the same bytes, whatever the grouping
        AbsorbPool pool;
        pool.max_k = AbsorbPool::kMaxK;
        std::vector<std::thread> th;
        for (std::size_t j = 0; j < k; ++j) th.emplace_back([&, j] { pool.run(ts[j]->state, elems[j], n); });
        for (auto& x : th) x.join();
    });
}

int dgkr_transcript_challenge(const dgkr_field* f, dgkr_transcript* t, std::uint8_t* out) {
    return guard([&] {
        Transcript tr(&f->f, t->state, t->draws);
        f->f.to_bytes(tr.challenge(), out);
        t->draws = tr.draws();
    });
}
int dgkr_transcript_challenge_index(const dgkr_field* f, dgkr_transcript* t, std::uint64_t bound, std::uint64_t* out) {
    return guard([&] {
        Transcript tr(&f->f, t->state, t->draws);
        *out = tr.challenge_index(bound);
        t->draws = tr.draws();
    });
}
int dgkr_sha256(const std::uint8_t* d, std::size_t n, std::uint8_t* out32) {
    return guard([&] {
        const Digest h = sha256(d, n);
        std::memcpy(out32, h.data(), 32);
    });
}
int dgkr_sha256_has_shani(void) { return sha256_has_shani() ? 1 : 0; }

int dgkr_ctx_create(int device, dgkr_ctx** out) {
    return guard([&] {
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) fail(DGKR_CUDA_ERROR, "no such CUDA device");
        CK(cudaSetDevice(device));
        cudaDeviceProp prop{};
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) fail(DGKR_UNSUPPORTED, "this build targets sm_100a (B200)");
        auto c = std::make_unique<dgkr_ctx>(device, prop.multiProcessorCount);
        *out = c.release();
    });
}
void dgkr_ctx_destroy(dgkr_ctx* ctx) { delete ctx; }
int dgkr_ctx_set_profile(dgkr_ctx* ctx, int on) {
    return guard([&] { ctx->profile_on = on != 0; });
}
int dgkr_ctx_get_profile(dgkr_ctx* ctx, dgkr_profile* out) {
    return guard([&] { *out = ctx->prof; });
}
int dgkr_ctx_device_info(dgkr_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor) {
    return guard([&] {
        cudaDeviceProp prop{};
        CK(cudaGetDeviceProperties(&prop, ctx->device));
        *sm_count = prop.multiProcessorCount;
        *cc_major = prop.major;
        *cc_minor = prop.minor;
    });
}

int dgkr_prove_product_sum(dgkr_ctx* ctx, const dgkr_field* f, std::size_t n_pairs, std::size_t vars,
                           const std::uint8_t* tables, dgkr_transcript* t, std::uint8_t* proof, std::size_t cap,
                           std::size_t* len) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        Transcript tr(&f->f, t->state, t->draws);
        auto bytes = product_sumcheck(ctx, f, n_pairs, vars, tables, tr, nullptr);
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        ctx->end_call();
        emit(bytes, proof, cap, len);
    });
}

// ===========================================================================
// PairSumSession (sumcheck.hpp:152-221): the product sum-check's steps as
// separate calls, so a caller (cluster.hpp:250-316 drives one per worker and
// one for the master tail) can run the protocol itself. The tables live on
// the device; fold(r) is the fused fold + next-round kernel (k_round), so
// the round polynomial of the folded tables is ready when fold returns.
// ===========================================================================
struct dgkr_pairsum {
    dgkr_ctx* ctx = nullptr;
    const dgkr_field* f = nullptr;
    int np = 0;
    int vars_left = 0;
    int layout = 0;  // 0: natural order (before the first fold), 1: bit-reversed (k_round kFoldNat/kFoldRev outputs)
    std::uint64_t size = 0;  // current table size 2^vars_left
    DBuf<Fe> tabs;
    DBuf<const Fe*> base;
    RoundBuffers rb;
    const Fe* const* cur = nullptr;
    int cur_buf = -1;  // -1 base tables, 0 rb.A, 1 rb.B
    bool have_sums = false;
    U256 sums[3]{};     // (S0, S1, S2) of the current tables
    std::vector<U256> finals;
};

namespace {

void pairsum_scan(dgkr_pairsum* s) {
    // round sums of the natural-order initial tables (k_round kScan, all three sums)
    Lane* L = s->ctx;
    RoundLaunch rl;
    rl.np = s->np;
    rl.has_g = false;
    rl.mode = 0;
    rl.in = s->cur;
    rl.n_out_pairs = s->size / 2;
    rl.need_s1 = true;
    const FieldKind kind = L->use(s->f);
    if (rl.n_out_pairs <= tuning().small_round_pairs) launch_round_small(kind, rl, L->ws, L->st);
    else launch_round(kind, rl, L->ws, L->st);
    L->launched();
    L->d2h(L->h_small + 1, L->ws.result, 3 * sizeof(Fe));
    L->sync();
    for (int k = 0; k < 3; ++k) s->sums[k] = to_u256(L->h_small[1 + k]);
    s->have_sums = true;
}

}  // namespace

int dgkr_pairsum_begin(dgkr_ctx* ctx, const dgkr_field* f, std::size_t n_pairs, std::size_t vars,
                       const std::uint8_t* tables, dgkr_pairsum** out) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (n_pairs == 0) fail(DGKR_INVALID_ARGUMENT, "product sum needs at least one pair");  // sumcheck.hpp:155-157
        if (vars > 40) fail(DGKR_INVALID_ARGUMENT, "table too large");
        auto s = std::make_unique<dgkr_pairsum>();
        s->ctx = ctx;
        s->f = f;
        s->np = static_cast<int>(n_pairs);
        s->vars_left = static_cast<int>(vars);
        s->size = std::uint64_t{1} << vars;
        const int ntab = 2 * s->np;
        s->tabs.ensure(static_cast<std::size_t>(ntab) * s->size);
        DBuf<std::uint8_t> stage;
        ctx->upload_elems(f, tables, static_cast<std::uint64_t>(ntab) * s->size, s->tabs.p, stage);  // copies the tables (:168)
        std::vector<const Fe*> hp(ntab);
        for (int t = 0; t < ntab; ++t) hp[t] = s->tabs.p + t * s->size;
        s->base.ensure(ntab);
        ctx->h2d(s->base.p, hp.data(), ntab * sizeof(const Fe*));
        s->cur = s->base.p;
        s->rb.ensure(ntab, s->size, ctx->st);
        CK(cudaStreamSynchronize(ctx->st));
        *out = s.release();
    });
}

void dgkr_pairsum_end(dgkr_pairsum* s) { delete s; }

std::size_t dgkr_pairsum_vars_left(const dgkr_pairsum* s) { return s ? static_cast<std::size_t>(s->vars_left) : 0; }

int dgkr_pairsum_total(dgkr_pairsum* s, std::uint8_t* out) {
    return guard([&] {
        Lane* L = s->ctx;
        CK(cudaSetDevice(L->device));
        U256 tot{};
        if (!s->finals.empty()) {  // folded down to the final values
            for (int k = 0; k < s->np; ++k) tot = s->f->f.add(tot, s->f->f.mul(s->finals[2 * k], s->finals[2 * k + 1]));
        } else {  // sum_k sum_b f_k(b) g_k(b) (:177-186; layout-independent)
            launch_pair_total(L->use(s->f), s->cur, s->np, s->size, L->ws, L->st);
            L->launched();
            L->d2h(L->h_small + 1, L->ws.result, sizeof(Fe));
            L->sync();
            tot = to_u256(L->h_small[1]);
        }
        s->f->f.to_bytes(tot, out);
    });
}

int dgkr_pairsum_round(dgkr_pairsum* s, std::uint8_t* out4) {
    return guard([&] {
        if (s->vars_left == 0) fail(DGKR_LOGIC_ERROR, "sumcheck session exhausted");  // sumcheck.hpp:188-191
        CK(cudaSetDevice(s->ctx->device));
        if (!s->have_sums) pairsum_scan(s);
        const HostField& F = s->f->f;
        const U256 c0 = s->sums[0], c2 = s->sums[2];
        const U256 c1 = F.sub(F.sub(s->sums[1], c0), c2);  // c1 = sum f0 dg + g0 df
        const std::size_t w = F.width();
        F.to_bytes(c0, out4);
        F.to_bytes(c1, out4 + w);
        F.to_bytes(c2, out4 + 2 * w);
        F.to_bytes(U256{}, out4 + 3 * w);  // c3 = 0 (sumcheck.hpp:18-37)
    });
}

int dgkr_pairsum_fold(dgkr_pairsum* s, const std::uint8_t* r_canon) {
    return guard([&] {
        if (s->vars_left == 0) fail(DGKR_LOGIC_ERROR, "sumcheck session exhausted");  // sumcheck.hpp:195-198
        Lane* L = s->ctx;
        CK(cudaSetDevice(L->device));
        const HostField& F = s->f->f;
        const U256 r = F.from_bytes(r_canon);
        const FieldKind kind = L->use(s->f);
        const int ntab = 2 * s->np;
        if (s->vars_left == 1) {  // 2-element tables -> the final values
            L->h_small[0] = to_fe(r);
            L->h2d(L->d_small.p, L->h_small, sizeof(Fe));
            launch_fold_final(kind, s->cur, const_cast<Fe* const*>(s->rb.F()), ntab, L->d_small.p, L->st);
            L->launched();
            Fe* hf = L->h_small + Lane::kFinalsOff;
            if (ntab > static_cast<int>(Lane::kGatherOff - Lane::kFinalsOff)) fail(DGKR_UNSUPPORTED, "too many pairs");
            L->d2h(hf, s->rb.finals.p, ntab * sizeof(Fe));
            L->sync();
            s->finals.clear();
            for (int t = 0; t < ntab; ++t) s->finals.push_back(to_u256(hf[t]));
            s->vars_left = 0;
            s->size = 1;
            s->have_sums = false;
            return;
        }
        // fold with r and compute the next round's sums in one launch (mle.hpp:75-85 + sumcheck.hpp:118-137)
        U256 fk[9];
        s->f->fold_const(r, fk);
        RoundLaunch rl;
        rl.np = s->np;
        rl.has_g = false;
        rl.mode = s->layout == 0 ? 1 : 2;
        rl.in = s->cur;
        const int nb = s->cur_buf == 0 ? 1 : 0;
        const Fe* const* nxt = nb == 0 ? s->rb.A() : s->rb.B();
        rl.out = const_cast<Fe* const*>(nxt);
        rl.n_out_pairs = s->size / 4;
        rl.fold_const = fk;
        rl.need_s1 = true;
        if (rl.n_out_pairs <= tuning().small_round_pairs) launch_round_small(kind, rl, L->ws, L->st);
        else launch_round(kind, rl, L->ws, L->st);
        L->launched();
        L->d2h(L->h_small + 1, L->ws.result, 3 * sizeof(Fe));
        L->sync();  // ws.result is shared by every session of the context: read it now
        for (int k = 0; k < 3; ++k) s->sums[k] = to_u256(L->h_small[1 + k]);
        s->have_sums = true;
        s->cur = nxt;
        s->cur_buf = nb;
        s->layout = 1;
        s->size /= 2;
        s->vars_left -= 1;
    });
}

int dgkr_pairsum_finals(dgkr_pairsum* s, std::uint8_t* out) {
    return guard([&] {
        if (s->vars_left != 0) fail(DGKR_LOGIC_ERROR, "sumcheck session still has unbound variables");  // :204-207
        if (s->finals.empty()) {  // a 0-variable session: the 1-element tables themselves
            Lane* L = s->ctx;
            CK(cudaSetDevice(L->device));
            std::vector<const Fe*> hp(2 * s->np);
            CK(cudaMemcpy(hp.data(), s->cur, hp.size() * sizeof(const Fe*), cudaMemcpyDeviceToHost));
            for (const Fe* p : hp) {
                Fe v;
                CK(cudaMemcpy(&v, p, sizeof(Fe), cudaMemcpyDeviceToHost));
                s->finals.push_back(to_u256(v));
            }
        }
        const std::size_t w = s->f->f.width();
        for (std::size_t t = 0; t < s->finals.size(); ++t) s->f->f.to_bytes(s->finals[t], out + t * w);
    });
}

int dgkr_prove_layer_sum(dgkr_ctx* ctx, const dgkr_field* f, std::size_t side_vars, std::size_t n_slots,
                         const std::uint8_t* slot_tables, std::size_t n_wires, const std::uint32_t* wire_meta,
                         const std::uint64_t* wire_idx, const std::uint8_t* wire_weights, const std::uint8_t* claimed,
                         dgkr_transcript* t, std::uint8_t* proof, std::size_t cap, std::size_t* len,
                         std::uint8_t* x_point, std::uint8_t* y_point) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        const HostField& F = f->f;
        const FieldKind kind = ctx->use(f);
        if (side_vars > 40) fail(DGKR_INVALID_ARGUMENT, "table too large");
        const std::uint64_t T = std::uint64_t{1} << side_vars;
        if (n_slots == 0) fail(DGKR_INVALID_ARGUMENT, "layer sum needs at least one slot");
        for (std::size_t i = 0; i < n_wires; ++i) {  // sumcheck.hpp:354-359
            if (wire_meta[3 * i + 1] >= n_slots || wire_meta[3 * i + 2] >= n_slots || wire_idx[2 * i] >= T ||
                wire_idx[2 * i + 1] >= T)
                fail(DGKR_INVALID_ARGUMENT, "layer wire index out of range");
        }
        const U256 cl = F.from_bytes(claimed);
        Transcript tr(&f->f, t->state, t->draws);
        DBuf<Fe> V, Hb, Gb, W;
        DBuf<std::uint8_t> stage;
        V.ensure(n_slots * T);
        ctx->upload_elems(f, slot_tables, n_slots * T, V.p, stage);
        W.ensure(n_wires);
        ctx->upload_elems(f, wire_weights, n_wires, W.p, stage);
        Hb.ensure(n_slots * T);
        Gb.ensure(T);
        // CSR transposes by (slot, x) and (slot, y)
        std::vector<std::uint32_t> xoff(n_slots * (T + 1), 0), yoff(n_slots * (T + 1), 0);
        for (std::size_t i = 0; i < n_wires; ++i) {
            xoff[wire_meta[3 * i + 1] * (T + 1) + wire_idx[2 * i] + 1]++;
            yoff[wire_meta[3 * i + 2] * (T + 1) + wire_idx[2 * i + 1] + 1]++;
        }
        std::uint32_t ax = 0, ay = 0;
        for (std::size_t s = 0; s < n_slots; ++s) {
            xoff[s * (T + 1)] += ax;
            yoff[s * (T + 1)] += ay;
            for (std::uint64_t i = 1; i <= T; ++i) {
                xoff[s * (T + 1) + i] += xoff[s * (T + 1) + i - 1];
                yoff[s * (T + 1) + i] += yoff[s * (T + 1) + i - 1];
            }
            ax = xoff[s * (T + 1) + T];
            ay = yoff[s * (T + 1) + T];
        }
        std::vector<uint4> xent(n_wires), yent(n_wires);
        std::vector<std::uint32_t> xf(xoff), yf(yoff);
        for (std::size_t i = 0; i < n_wires; ++i) {
            const std::uint32_t mul = wire_meta[3 * i] ? 0x80000000u : 0u;
            const std::uint32_t xs = wire_meta[3 * i + 1], ys = wire_meta[3 * i + 2];
            const std::uint32_t xi = static_cast<std::uint32_t>(wire_idx[2 * i]);
            const std::uint32_t yi = static_cast<std::uint32_t>(wire_idx[2 * i + 1]);
            xent[xf[xs * (T + 1) + xi]++] = make_uint4(0, yi, ys | mul, static_cast<std::uint32_t>(i));
            yent[yf[ys * (T + 1) + yi]++] = make_uint4(0, xi, xs | mul, static_cast<std::uint32_t>(i));
        }
        DBuf<std::uint32_t> dxo, dyo;
        DBuf<uint4> dxe, dye;
        dxo.ensure(xoff.size());
        dyo.ensure(yoff.size());
        dxe.ensure(n_wires);
        dye.ensure(n_wires);
        ctx->h2d(dxo.p, xoff.data(), xoff.size() * 4);
        ctx->h2d(dyo.p, yoff.data(), yoff.size() * 4);
        if (n_wires) {
            ctx->h2d(dxe.p, xent.data(), n_wires * sizeof(uint4));
            ctx->h2d(dye.p, yent.data(), n_wires * sizeof(uint4));
        }
        std::vector<SlotDesc> s1(n_slots), s2(n_slots);
        const std::uint32_t ls = static_cast<std::uint32_t>(side_vars);
        for (std::size_t s = 0; s < n_slots; ++s) {
            s1[s] = SlotDesc{V.p + s * T, Hb.p + s * T, dxo.p + s * (T + 1), dxe.p, ls, 0};
            s2[s] = SlotDesc{V.p + s * T, Hb.p + s * T, dyo.p + s * (T + 1), dye.p, ls, 0};
        }
        DBuf<SlotDesc> ds1, ds2;
        ds1.ensure(n_slots);
        ds2.ensure(n_slots);
        ctx->h2d(ds1.p, s1.data(), n_slots * sizeof(SlotDesc));
        ctx->h2d(ds2.p, s2.data(), n_slots * sizeof(SlotDesc));
        std::vector<const Fe*> bp;
        for (std::size_t s = 0; s < n_slots; ++s) {
            bp.push_back(V.p + s * T);
            bp.push_back(Hb.p + s * T);
        }
        bp.push_back(Gb.p);
        DBuf<const Fe*> dbp;
        dbp.ensure(bp.size());
        ctx->h2d(dbp.p, bp.data(), bp.size() * sizeof(const Fe*));

        tr.absorb(cl);  // sumcheck.hpp:364
        BookkeepLaunch bk;
        bk.slots = ds1.p;
        bk.n_slots = static_cast<int>(n_slots);
        bk.T = T;
        bk.n_copies = 1;
        bk.log_gcons = 63;
        bk.G = Gb.p;
        bk.wire_w = W.p;
        launch_bookkeep_phase1(kind, bk, ctx->st);
        ctx->launched();
        RoundBuffers rb;
        SumcheckRun p1 = run_rounds(ctx, f, static_cast<int>(n_slots), true, static_cast<int>(side_vars), dbp.p, rb, tr);
        std::vector<U256> vx(n_slots);
        for (std::size_t m = 0; m < n_slots; ++m) vx[m] = p1.finals[2 * m];
        DBuf<Fe> eqt;
        DBuf<EqJob> jobs;
        eqt.ensure(2 * ((std::size_t{1} << ((side_vars + 1) / 2)) + (std::size_t{1} << (side_vars / 2))) + 8);
        SplitEq uq = build_split_eq(ctx, f, {p1.challenges}, {F.one()}, eqt.p, jobs, 16);
        for (std::size_t m = 0; m < n_slots; ++m) ctx->h_small[8192 + m] = to_fe(vx[m]);
        ctx->h2d(ctx->d_small.p + 8192, ctx->h_small + 8192, n_slots * sizeof(Fe));
        bk.slots = ds2.p;
        bk.u = uq;
        bk.vx = ctx->d_small.p + 8192;
        launch_bookkeep_phase2(kind, bk, ctx->st);
        ctx->launched();
        SumcheckRun p2 = run_rounds(ctx, f, static_cast<int>(n_slots), true, static_cast<int>(side_vars), dbp.p, rb, tr);
        std::vector<U256> finals = vx;
        for (std::size_t m = 0; m < n_slots; ++m) finals.push_back(p2.finals[2 * m]);
        std::vector<RoundPoly> rounds = p1.rounds;
        rounds.insert(rounds.end(), p2.rounds.begin(), p2.rounds.end());
        if (x_point)
            for (std::size_t k = 0; k < side_vars; ++k) F.to_bytes(p1.challenges[k], x_point + k * F.width());
        if (y_point)
            for (std::size_t k = 0; k < side_vars; ++k) F.to_bytes(p2.challenges[k], y_point + k * F.width());
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        ctx->end_call();
        emit(sumcheck_bytes(F, cl, rounds, finals), proof, cap, len);
    });
}

// ===========================================================================
// GKR verifier (host): gkr_verify + check_input_claims (gkr.hpp:253-325),
// verify_layer_sum (sumcheck.hpp:461-505), run_round_checks (:249-270).
// The wiring predicate is evaluated through eq tables (O(T + W) per layer
// instead of the reference's O(W * s) chi_eval per wire; same values).
// Rejection is a result: malformed bytes reject, they do not throw.
// ===========================================================================
namespace {

struct ProofReader {
    const std::uint8_t* p;
    std::size_t n, pos = 0;
    const HostField& F;
    bool ok = true;
    std::uint32_t u32() {
        if (pos + 4 > n) {
            ok = false;
            return 0;
        }
        std::uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= static_cast<std::uint32_t>(p[pos + i]) << (8 * i);
        pos += 4;
        return v;
    }
    U256 elem() {
        const std::size_t w = F.width();
        if (pos + w > n || !F.canonical_lt_p(p + pos, w)) {
            ok = false;
            pos = n;
            return U256{};
        }
        const U256 v = F.from_bytes(p + pos);
        pos += w;
        return v;
    }
};

/// eq table: out[b] = seed * prod_k (b_k ? x_k : 1 - x_k), x_1 = LSB (mle.hpp:95-120)
/// fn(begin, end) over [0, n) on up to 16 host threads (serial below 2^15)
void par_for(std::uint64_t n, const std::function<void(std::uint64_t, std::uint64_t)>& fn) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (n < (std::uint64_t{1} << 15) || hw == 1) {
        fn(std::uint64_t{0}, n);
        return;
    }
    const std::uint64_t chunk = (n + hw - 1) / hw;
    std::vector<std::thread> th;
    for (unsigned i = 1; i < hw; ++i) {
        const std::uint64_t b = std::min<std::uint64_t>(n, i * chunk), e = std::min<std::uint64_t>(n, b + chunk);
        if (b < e) th.emplace_back([&fn, b, e] { fn(b, e); });
    }
    fn(std::uint64_t{0}, std::min<std::uint64_t>(n, chunk));
    for (auto& t : th) t.join();
}

std::vector<U256> eq_table_doubling(const HostField& F, const std::vector<U256>& x, const U256& seed) {
    std::vector<U256> t(std::size_t{1} << x.size());
    t[0] = seed;
    for (std::size_t k = 0; k < x.size(); ++k) {
        const std::size_t half = std::size_t{1} << k;
        for (std::size_t b = 0; b < half; ++b) {
            const U256 hi = F.mul(t[b], x[k]);
            t[b + half] = hi;
            t[b] = F.sub(t[b], hi);
        }
    }
    return t;
}

/// seed * eq(x, b) for every b (b_k = bit k, mle.hpp:95-120): large tables as
/// eq(low half) x eq(high half), expanded on host threads; the same field
/// elements as the doubling (products mod p commute)
std::vector<U256> eq_table_host(const HostField& F, const std::vector<U256>& x, const U256& seed) {
    if (x.size() < 16) return eq_table_doubling(F, x, seed);
    const std::size_t klo = x.size() / 2;
    const std::vector<U256> lo = eq_table_doubling(F, std::vector<U256>(x.begin(), x.begin() + klo), seed);
    const std::vector<U256> hi = eq_table_doubling(F, std::vector<U256>(x.begin() + klo, x.end()), F.one());
    std::vector<U256> t(std::size_t{1} << x.size());
    const std::uint64_t m = (std::uint64_t{1} << klo) - 1;
    par_for(t.size(), [&](std::uint64_t b0, std::uint64_t b1) {
        for (std::uint64_t b = b0; b < b1; ++b) t[b] = F.mul(lo[b & m], hi[b >> klo]);
    });
    return t;
}

/// MLE of a table (entries beyond `vals` are zero) at `point`
U256 mle_host(const HostField& F, const std::vector<U256>& vals, const std::vector<U256>& point) {
    const std::vector<U256> eq = eq_table_host(F, point, F.one());
    U256 acc{};
    for (std::size_t i = 0; i < vals.size() && i < eq.size(); ++i) acc = F.add(acc, F.mul(vals[i], eq[i]));
    return acc;
}

/// returns accept; input_claims = registry[0] on acceptance
bool gkr_verify_host(const dgkr_circuit& c, const HostField& F, const std::uint8_t* proof, std::size_t len,
                     const std::uint8_t* outputs, std::size_t n_outputs, Transcript& tr,
                     std::vector<LayerClaim>& input_claims) {
    ProofReader rd{proof, len, 0, F};
    const std::uint32_t D = c.depth;
    const std::uint64_t n_out = c.full_padded[D];
    if (rd.u32() != n_out || !rd.ok) return false;
    std::vector<U256> outs(n_out);
    for (auto& o : outs) o = rd.elem();
    if (!rd.ok) return false;
    if (outputs) {  // the statement must match the proof's outputs, padding zero (gkr.hpp:260-268)
        for (std::uint64_t i = 0; i < n_out; ++i) {
            const U256 want = i < n_outputs ? F.from_bytes(outputs + i * F.width()) : U256{};
            if (!(outs[i] == want)) return false;
        }
    }
    if (rd.u32() != D || !rd.ok) return false;
    for (const auto& o : outs) tr.absorb(o);
    std::vector<U256> q;
    for (std::uint32_t k = 0; k < c.padded_log2_full(D); ++k) q.push_back(tr.challenge());
    std::vector<std::vector<LayerClaim>> registry(D + 1);
    {
        LayerClaim lc;
        lc.layer = D;
        lc.terms.push_back(ClaimTerm{q, F.one()});
        lc.value = mle_host(F, outs, q);
        registry[D].push_back(std::move(lc));
    }
    const U256 zero{};
    for (std::uint32_t layer = D; layer >= 1; --layer) {
        const auto& C = *c.cons[layer];
        const std::uint32_t na = rd.u32();
        if (!rd.ok || na > (len - rd.pos) / F.width()) return false;  // count exceeds the remaining bytes
        std::vector<U256> pa(na);
        for (auto& a : pa) a = rd.elem();
        const std::uint32_t sb_len = rd.u32();
        if (!rd.ok) return false;
        const std::size_t sb_end = rd.pos + sb_len;
        if (sb_end > len) return false;
        std::vector<U256> alphas;
        LayerClaim combined = combine_claims(std::move(registry[layer]), tr, F, &alphas);
        registry[layer].clear();
        if (alphas.size() != pa.size()) return false;
        for (std::size_t i = 0; i < pa.size(); ++i)
            if (!(alphas[i] == pa[i])) return false;
        // SumcheckProof bytes (sumcheck.hpp:51-61)
        const U256 claimed = rd.elem();
        const std::uint32_t nr = rd.u32();
        const std::uint32_t side = C.side;
        const std::size_t ns = C.slots.size();
        if (!rd.ok || !(claimed == combined.value) || nr != 2 * side) return false;
        std::vector<std::array<U256, 4>> rounds(nr);
        for (auto& r : rounds)
            for (auto& x : r) x = rd.elem();
        const std::uint32_t nf = rd.u32();
        if (!rd.ok || nf != 2 * ns) return false;
        std::vector<U256> finals(nf);
        for (auto& x : finals) x = rd.elem();
        if (!rd.ok || rd.pos != sb_end) return false;
        // run_round_checks
        tr.absorb(claimed);
        U256 claim = claimed;
        std::vector<U256> point;
        for (const auto& r : rounds) {
            if (!(r[3] == zero)) return false;
            const U256 sum01 = F.add(F.add(r[0], r[0]), F.add(F.add(r[1], r[2]), r[3]));
            if (!(sum01 == claim)) return false;
            for (const auto& x : r) tr.absorb(x);
            const U256 ch = tr.challenge();
            claim = F.add(r[0], F.mul(ch, F.add(r[1], F.mul(ch, F.add(r[2], F.mul(ch, r[3]))))));
            point.push_back(ch);
        }
        const std::vector<U256> xp(point.begin(), point.begin() + side), yp(point.begin() + side, point.end());
        // wiring predicate at (combined claim, x, y): gate weights via eq tables of the claim points
        const std::uint64_t sub_g = c.sub_size[layer], pad_g = c.sub_padded[layer];
        const std::uint64_t n_gates_full = c.n_copies * pad_g;
        std::vector<U256> wg(n_gates_full);
        for (const auto& t : combined.terms) {
            const std::vector<U256> eq = eq_table_host(F, t.point, t.weight);
            par_for(std::min<std::uint64_t>(n_gates_full, eq.size()), [&](std::uint64_t b0, std::uint64_t b1) {
                for (std::uint64_t g = b0; g < b1; ++g) wg[g] = F.add(wg[g], eq[g]);
            });
        }
        const std::vector<U256> ex = eq_table_host(F, xp, F.one()), ey = eq_table_host(F, yp, F.one());
        auto slot_of = [&](std::uint32_t l) {
            for (std::size_t s2 = 0; s2 < ns; ++s2)
                if (C.slots[s2] == l) return s2;
            return ns;
        };
        // sum_wires w(g) chi_x(u) chi_y(v) * (V_x V_y | V_x + V_y), bucketed by
        // (x slot, y slot, mul/add) so each wire costs two products; copies
        // (or gate ranges) are split over host threads with private buckets
        const std::uint64_t g0 = c.h_lgs[layer - 1];
        const std::size_t nb = 2 * ns * ns;
        std::mutex bmu;
        std::vector<U256> bucket(nb);
        bool wiring_ok = true;
        const std::uint64_t n_items = static_cast<std::uint64_t>(c.n_copies) * sub_g;
        par_for(n_items, [&](std::uint64_t i0, std::uint64_t i1) {
            std::vector<U256> acc(nb);
            bool ok_local = true;
            for (std::uint64_t it = i0; it < i1; ++it) {
                const std::uint64_t cp = it / sub_g, g = it % sub_g;
                const U256 w = wg[cp * pad_g + g];
                for (std::uint64_t e = c.h_gns[g0 + g]; e < c.h_gns[g0 + g + 1]; ++e) {
                    const std::uint32_t* ng = &c.h_nested[5 * e];
                    const std::size_t sx = slot_of(ng[1]), sy = slot_of(ng[3]);
                    if (sx >= ns || sy >= ns) {
                        ok_local = false;
                        continue;
                    }
                    const std::uint64_t xi = cp * c.sub_padded[ng[1]] + ng[2];
                    const std::uint64_t yi = cp * c.sub_padded[ng[3]] + ng[4];
                    U256& bk = acc[(sx * ns + sy) * 2 + (ng[0] ? 1 : 0)];
                    bk = F.add(bk, F.mul(w, F.mul(ex[xi], ey[yi])));
                }
            }
            std::lock_guard<std::mutex> lk(bmu);
            if (!ok_local) wiring_ok = false;
            for (std::size_t k = 0; k < nb; ++k) bucket[k] = F.add(bucket[k], acc[k]);
        });
        if (!wiring_ok) return false;
        U256 expected{};
        for (std::size_t sx = 0; sx < ns; ++sx)
            for (std::size_t sy = 0; sy < ns; ++sy) {
                const U256 vx = finals[sx], vy = finals[ns + sy];
                expected = F.add(expected, F.mul(bucket[(sx * ns + sy) * 2 + 1], F.mul(vx, vy)));
                expected = F.add(expected, F.mul(bucket[(sx * ns + sy) * 2], F.add(vx, vy)));
            }
        if (!(expected == claim)) return false;
        for (std::size_t s2 = 0; s2 < ns; ++s2) {
            const std::uint32_t src = C.slots[s2];
            const std::uint32_t native = c.padded_log2_full(src);
            registry[src].push_back(shrink_claim(src, native, xp, finals[s2], F));
            registry[src].push_back(shrink_claim(src, native, yp, finals[ns + s2], F));
        }
    }
    if (rd.pos != len) return false;
    input_claims = std::move(registry[0]);
    return true;
}

}  // namespace

int dgkr_gkr_verify(const dgkr_circuit* c, const dgkr_field* f, const std::uint8_t* outputs, std::size_t n_outputs,
                    const std::uint8_t* inputs, const std::uint8_t* proof, std::size_t len, dgkr_transcript* t,
                    int* accept) {
    return guard([&] {
        const HostField& F = f->f;
        Transcript tr(&F, t->state, t->draws);
        std::vector<LayerClaim> claims;
        bool ok = gkr_verify_host(*c, F, proof, len, outputs, n_outputs, tr, claims);
        if (ok && inputs) {  // check_input_claims (gkr.hpp:314-325) against the padded input table
            const std::uint64_t n_in = static_cast<std::uint64_t>(c->n_copies) * c->sub_padded[0];
            std::vector<U256> tab(n_in);
            for (std::uint32_t cp = 0; cp < c->n_copies; ++cp)
                for (std::uint64_t i = 0; i < c->sub_size[0]; ++i)
                    tab[cp * c->sub_padded[0] + i] =
                        F.from_bytes(inputs + (static_cast<std::uint64_t>(cp) * c->sub_size[0] + i) * F.width());
            for (const auto& cl : claims) {
                U256 acc{};
                for (const auto& term : cl.terms) acc = F.add(acc, F.mul(term.weight, mle_host(F, tab, term.point)));
                if (!(acc == cl.value)) ok = false;
            }
        }
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        *accept = ok ? 1 : 0;
    });
}

int dgkr_gkr_input_claims(const dgkr_circuit* c, const dgkr_field* f, const std::uint8_t* proof, std::size_t len,
                          dgkr_transcript* t, int* accept, std::uint8_t* out, std::size_t cap, std::size_t* out_len) {
    return guard([&] {
        const HostField& F = f->f;
        Transcript tr(&F, t->state, t->draws);
        std::vector<LayerClaim> claims;
        const bool ok = gkr_verify_host(*c, F, proof, len, nullptr, 0, tr, claims);
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        *accept = ok ? 1 : 0;
        std::vector<std::uint8_t> b;
        put32(b, static_cast<std::uint32_t>(ok ? claims.size() : 0));
        if (ok) {
            for (const auto& cl : claims) {
                put32(b, static_cast<std::uint32_t>(cl.terms.size()));
                for (const auto& term : cl.terms) {
                    put32(b, static_cast<std::uint32_t>(term.point.size()));
                    for (const auto& x : term.point) append_elem(b, F, x);
                    append_elem(b, F, term.weight);
                }
                append_elem(b, F, cl.value);
            }
        }
        emit(b, out, cap, out_len);
    });
}

int dgkr_circuit_create(dgkr_ctx* ctx, std::uint32_t input_size, std::uint32_t depth, const std::uint64_t* lgs,
                        const std::uint64_t* gns, const std::uint32_t* nested, const std::uint64_t* min_padded,
                        std::uint32_t n_copies, dgkr_circuit** out) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (n_copies == 0 || (n_copies & (n_copies - 1)) != 0)
            fail(DGKR_INVALID_ARGUMENT, "n_copies must be a power of two");
        auto c = std::make_unique<dgkr_circuit>();
        c->input_size = input_size;
        c->depth = depth;
        c->n_copies = n_copies;
        c->log_copies = log2_exact(n_copies);
        build_circuit(ctx, *c, lgs, gns, nested, min_padded);
        c->h_lgs.assign(lgs, lgs + depth + 1);
        c->h_gns.assign(gns, gns + lgs[depth] + 1);
        c->h_nested.assign(nested, nested + 5 * gns[lgs[depth]]);
        if (min_padded) c->h_min_padded.assign(min_padded, min_padded + depth + 1);
        *out = c.release();
    });
}
void dgkr_circuit_destroy(dgkr_circuit* c) { delete c; }

// Binary CSR circuit file (little-endian):
//   "DGKRCSR1" | u32 input_size | u32 depth | u32 n_copies | u32 has_min_padded
//   | u64 n_gates | u64 n_nested | u64 layer_gate_start[depth+1]
//   | u64 gate_nested_start[n_gates+1] | u32 nested[n_nested][5] | u64 min_padded[depth+1] (if flagged)
namespace {
constexpr char kCsrMagic[8] = {'D', 'G', 'K', 'R', 'C', 'S', 'R', '1'};
}

int dgkr_circuit_save(const dgkr_circuit* c, const char* path) {
    return guard([&] {
        std::FILE* fp = std::fopen(path, "wb");
        if (!fp) fail(DGKR_INVALID_ARGUMENT, std::string("cannot open ") + path);
        const std::uint32_t hdr[4] = {c->input_size, c->depth, c->n_copies, c->h_min_padded.empty() ? 0u : 1u};
        const std::uint64_t n_gates = c->h_lgs.back(), n_nested = c->h_gns.back();
        bool ok = std::fwrite(kCsrMagic, 1, 8, fp) == 8 && std::fwrite(hdr, 4, 4, fp) == 4 &&
                  std::fwrite(&n_gates, 8, 1, fp) == 1 && std::fwrite(&n_nested, 8, 1, fp) == 1 &&
                  std::fwrite(c->h_lgs.data(), 8, c->h_lgs.size(), fp) == c->h_lgs.size() &&
                  std::fwrite(c->h_gns.data(), 8, c->h_gns.size(), fp) == c->h_gns.size() &&
                  std::fwrite(c->h_nested.data(), 4, c->h_nested.size(), fp) == c->h_nested.size();
        if (ok && !c->h_min_padded.empty())
            ok = std::fwrite(c->h_min_padded.data(), 8, c->h_min_padded.size(), fp) == c->h_min_padded.size();
        ok = (std::fclose(fp) == 0) && ok;
        if (!ok) fail(DGKR_INVALID_ARGUMENT, std::string("short write to ") + path);
    });
}

int dgkr_circuit_load(dgkr_ctx* ctx, const char* path, std::uint32_t n_copies, dgkr_circuit** out) {
    return guard([&] {
        std::FILE* fp = std::fopen(path, "rb");
        if (!fp) fail(DGKR_INVALID_ARGUMENT, std::string("cannot open ") + path);
        struct Closer {
            std::FILE* f;
            ~Closer() { std::fclose(f); }
        } closer{fp};
        char magic[8];
        std::uint32_t hdr[4];
        std::uint64_t n_gates = 0, n_nested = 0;
        if (std::fread(magic, 1, 8, fp) != 8 || std::memcmp(magic, kCsrMagic, 8) != 0)
            fail(DGKR_INVALID_ARGUMENT, "not a DGKRCSR1 circuit file");
        if (std::fread(hdr, 4, 4, fp) != 4 || std::fread(&n_gates, 8, 1, fp) != 1 || std::fread(&n_nested, 8, 1, fp) != 1)
            fail(DGKR_INVALID_ARGUMENT, "truncated circuit header");
        const std::uint32_t depth = hdr[1];
        if (depth == 0 || depth > (1u << 20) || n_gates > (1ull << 40) || n_nested > (1ull << 40))
            fail(DGKR_INVALID_ARGUMENT, "implausible circuit header");
        // the header's counts must describe exactly this file (before any allocation)
        if (std::fseek(fp, 0, SEEK_END) != 0) fail(DGKR_INVALID_ARGUMENT, "cannot size circuit file");
        const long fsize = std::ftell(fp);
        const std::uint64_t want = 40 + 8ull * (depth + 1) + 8ull * (n_gates + 1) + 20ull * n_nested +
                                   (hdr[3] ? 8ull * (depth + 1) : 0);
        if (fsize < 0 || static_cast<std::uint64_t>(fsize) != want)
            fail(DGKR_INVALID_ARGUMENT, "circuit file size does not match its header");
        if (std::fseek(fp, 40, SEEK_SET) != 0) fail(DGKR_INVALID_ARGUMENT, "cannot seek circuit file");
        std::vector<std::uint64_t> lgs(depth + 1), gns(n_gates + 1), minp;
        std::vector<std::uint32_t> nested(5 * n_nested);
        if (std::fread(lgs.data(), 8, lgs.size(), fp) != lgs.size() || std::fread(gns.data(), 8, gns.size(), fp) != gns.size() ||
            std::fread(nested.data(), 4, nested.size(), fp) != nested.size())
            fail(DGKR_INVALID_ARGUMENT, "truncated circuit body");
        if (hdr[3]) {
            minp.resize(depth + 1);
            if (std::fread(minp.data(), 8, minp.size(), fp) != minp.size()) fail(DGKR_INVALID_ARGUMENT, "truncated min_padded");
        }
        if (lgs[0] != 0 || lgs[depth] != n_gates || gns[0] != 0 || gns[n_gates] != n_nested)
            fail(DGKR_INVALID_ARGUMENT, "inconsistent CSR offsets");
        for (std::uint32_t l = 0; l < depth; ++l)
            if (lgs[l + 1] < lgs[l]) fail(DGKR_INVALID_ARGUMENT, "inconsistent CSR offsets");
        for (std::uint64_t g = 0; g < n_gates; ++g)
            if (gns[g + 1] < gns[g]) fail(DGKR_INVALID_ARGUMENT, "inconsistent CSR offsets");
        const int rc = dgkr_circuit_create(ctx, hdr[0], depth, lgs.data(), gns.data(), nested.data(),
                                           minp.empty() ? nullptr : minp.data(), n_copies ? n_copies : hdr[2], out);
        if (rc != DGKR_OK) fail(rc, g_err);  // g_err: the create call's message
    });
}
std::size_t dgkr_circuit_output_size(const dgkr_circuit* c) { return c ? c->full_padded[c->depth] : 0; }

int dgkr_circuit_evaluate(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, const std::uint8_t* inputs,
                          std::uint8_t* outputs, std::size_t cap, std::size_t* len) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        CircuitWs& W = workspace(*c, 0);
        evaluate_circuit(ctx, *c, W, f, inputs);
        const std::size_t w = f->f.width();
        const std::uint64_t n_out = c->full_padded[c->depth];
        *len = n_out * w;
        if (n_out * w > cap) fail(DGKR_CAPACITY, "output buffer too small");
        W.stage.ensure(n_out * w);
        launch_to_canonical(ctx->use(f), W.values[c->depth]->p, W.stage.p, static_cast<int>(w), n_out, ctx->st);
        ctx->d2h(outputs, W.stage.p, n_out * w);
        ctx->sync();
        ctx->end_call();
    });
}

std::size_t dgkr_gkr_proof_bound(const dgkr_circuit* c, const dgkr_field* f) {
    if (!c || !f) return 0;
    const std::size_t w = f->f.width();
    std::size_t b = 8 + c->full_padded[c->depth] * w;
    for (std::uint32_t li = 1; li <= c->depth; ++li) {
        const auto& C = *c->cons[li];
        b += 16 + w + 4 * w * 2 * C.side + 2 * C.slots.size() * w + 2 * c->depth * w + 64;
    }
    return b;
}

int dgkr_gkr_prove(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, const std::uint8_t* inputs, dgkr_transcript* t,
                   std::uint8_t* proof, std::size_t cap, std::size_t* len) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        if (!inputs) fail(DGKR_INVALID_ARGUMENT, "inputs must not be NULL");
        *len = dgkr_gkr_proof_bound(c, f);
        Transcript tr(&f->f, t->state, t->draws);
        *len = gkr_prove(ctx, *c, workspace(*c, 0), f, inputs, tr, proof, cap);
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        ctx->end_call();
    });
}

int dgkr_circuit_load_inputs(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, const std::uint8_t* inputs) {
    return dgkr_circuit_load_inputs_lane(ctx, c, f, 0, inputs);
}

int dgkr_circuit_load_inputs_lane(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, int lane,
                                  const std::uint8_t* inputs) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (lane < 0 || lane >= 64) fail(DGKR_OUT_OF_RANGE, "lane");
        Lane* L = ctx->lane(lane);
        load_inputs(L, *c, workspace(*c, lane), f, inputs);
        L->sync();
    });
}

int dgkr_gkr_prove_resident(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, dgkr_transcript* t,
                            std::uint8_t* proof, std::size_t cap, std::size_t* len) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        *len = dgkr_gkr_proof_bound(c, f);
        Transcript tr(&f->f, t->state, t->draws);
        *len = gkr_prove(ctx, *c, workspace(*c, 0), f, nullptr, tr, proof, cap);
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        ctx->end_call();
    });
}

int dgkr_gkr_prove_batch(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, std::size_t n,
                         const std::uint8_t* const* inputs, dgkr_transcript* ts, std::uint8_t* const* proofs,
                         const std::size_t* caps, std::size_t* lens) {
    return dgkr_gkr_prove_stream(ctx, c, f, n, n, inputs, ts, proofs, caps, lens, nullptr);
}

int dgkr_gkr_prove_stream(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, std::size_t n, std::size_t n_lanes,
                          const std::uint8_t* const* inputs, dgkr_transcript* ts, std::uint8_t* const* proofs,
                          const std::size_t* caps, std::size_t* lens, dgkr_profile* lane_profiles) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (n == 0) fail(DGKR_OUT_OF_RANGE, "no proofs");
        if (n_lanes == 0 || n_lanes > 64) fail(DGKR_OUT_OF_RANGE, "lanes must be 1..64");
        const std::size_t L = std::min(n, n_lanes);
        std::vector<Lane*> lanes(L);
        for (std::size_t i = 0; i < L; ++i) {
            lanes[i] = ctx->lane(static_cast<int>(i));
            workspace(*c, static_cast<int>(i));  // allocate before the threads start
            std::memset(&lanes[i]->prof, 0, sizeof(dgkr_profile));
        }
        ctx->use(f);  // upload runtime-field constants once, before concurrency
        ctx->absorb_pool.max_k = static_cast<int>(std::clamp<std::uint64_t>(tuning().absorb_chains, 1, AbsorbPool::kMaxK));
        std::vector<std::string> errs(n);
        std::vector<int> codes(n, DGKR_OK);
        // host inputs: a work queue (any lane may take any proof); resident
        // inputs: proof i belongs to lane i mod L, whose loaded inputs it proves
        std::atomic<std::size_t> next{0};
        auto work = [&](std::size_t li) {
            // no exception may leave a std::thread: a failed cudaSetDevice
            // fails every proof this lane takes
            const cudaError_t se = cudaSetDevice(ctx->device);
            Lane* Ln = lanes[li];
            dgkr_profile acc{};
            for (std::size_t k = 0;; ++k) {
                const std::size_t i = inputs ? next.fetch_add(1) : li + k * L;
                if (i >= n) break;
                if (se != cudaSuccess) {
                    codes[i] = DGKR_CUDA_ERROR;
                    errs[i] = std::string("cudaSetDevice: ") + cudaGetErrorString(se);
                    continue;
                }
                try {
                    Ln->begin_call();
                    Transcript tr(&f->f, ts[i].state, ts[i].draws);
                    lens[i] = gkr_prove(Ln, *c, workspace(*c, static_cast<int>(li)), f, inputs ? inputs[i] : nullptr,
                                        tr, proofs[i], caps[i], nullptr, 0, L > 1 ? &ctx->absorb_pool : nullptr);
                    std::memcpy(ts[i].state, tr.state().data(), 32);
                    ts[i].draws = tr.draws();
                    Ln->end_call();
                    acc.launches += Ln->prof.launches;
                    acc.h2d_bytes += Ln->prof.h2d_bytes;
                    acc.d2h_bytes += Ln->prof.d2h_bytes;
                    acc.rounds += Ln->prof.rounds;
                    acc.output_absorb_ms += Ln->prof.output_absorb_ms;
                    acc.host_transcript_ms += Ln->prof.host_transcript_ms;
                    acc.total_ms += Ln->prof.total_ms;
                } catch (const Error& e) {
                    codes[i] = e.code;
                    errs[i] = e.what();
                } catch (const std::exception& e) {
                    codes[i] = DGKR_LOGIC_ERROR;
                    errs[i] = e.what();
                }
            }
            if (lane_profiles) lane_profiles[li] = acc;
            Ln->prof = acc;
        };
        std::vector<std::thread> th;
        for (std::size_t i = 1; i < L; ++i) th.emplace_back(work, i);
        work(0);
        for (auto& t : th) t.join();
        for (std::size_t i = 0; i < n; ++i)
            if (codes[i] != DGKR_OK) fail(codes[i], "proof " + std::to_string(i) + ": " + errs[i]);
    });
}

int dgkr_gkr_prove_dist_stream(dgkr_ctx* ctx, dgkr_comm* const* comms, std::size_t n_lanes, dgkr_circuit* c,
                               const dgkr_field* f, std::size_t n, const std::uint8_t* const* inputs,
                               dgkr_transcript* ts, std::uint8_t* const* proofs, const std::size_t* caps,
                               std::size_t* lens, dgkr_profile* lane_profiles, int absorb_policy) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (n == 0 || n_lanes == 0 || n_lanes > 64) fail(DGKR_OUT_OF_RANGE, "bad proof / lane count");
        if (absorb_policy != 0 && absorb_policy != 1) fail(DGKR_INVALID_ARGUMENT, "unknown absorb policy");
        const std::size_t L = std::min(n, n_lanes);
        std::vector<Lane*> lanes(L);
        for (std::size_t i = 0; i < L; ++i) {
            lanes[i] = ctx->lane(static_cast<int>(i));
            workspace(*c, static_cast<int>(i));
        }
        ctx->use(f);
        ctx->absorb_pool.max_k = static_cast<int>(std::clamp<std::uint64_t>(tuning().absorb_chains, 1, AbsorbPool::kMaxK));
        std::vector<int> codes(n, DGKR_OK);
        std::vector<std::string> errs(n);
        // static assignment: lane l proves l, l+L, l+2L, ... in order on every
        // rank, so lane l's exchanges pair up across ranks
        auto work = [&](std::size_t li) {
            const cudaError_t se = cudaSetDevice(ctx->device);  // checked per proof: nothing may throw out of a thread
            Lane* Ln = lanes[li];
            dgkr_profile acc{};
            for (std::size_t i = li; i < n; i += L) {
                if (se != cudaSuccess) {
                    codes[i] = DGKR_CUDA_ERROR;
                    errs[i] = std::string("cudaSetDevice: ") + cudaGetErrorString(se);
                    if (auto* s = dynamic_cast<ShmComm*>(comms[li])) s->hdr->aborted.store(1);
                    break;
                }
                try {
                    Ln->begin_call();
                    Transcript tr(&f->f, ts[i].state, ts[i].draws);
                    const int root = absorb_policy == 1 ? static_cast<int>(i % static_cast<std::size_t>(comms[li]->world)) : 0;
                    lens[i] = gkr_prove(Ln, *c, workspace(*c, static_cast<int>(li)), f, inputs ? inputs[i] : nullptr,
                                        tr, proofs[i], caps[i], comms[li], root, L > 1 ? &ctx->absorb_pool : nullptr);
                    std::memcpy(ts[i].state, tr.state().data(), 32);
                    ts[i].draws = tr.draws();
                    Ln->end_call();
                    acc.launches += Ln->prof.launches;
                    acc.h2d_bytes += Ln->prof.h2d_bytes;
                    acc.d2h_bytes += Ln->prof.d2h_bytes;
                    acc.rounds += Ln->prof.rounds;
                    acc.output_absorb_ms += Ln->prof.output_absorb_ms;
                    acc.host_transcript_ms += Ln->prof.host_transcript_ms;
                    acc.total_ms += Ln->prof.total_ms;
                    acc.round_launches += Ln->prof.round_launches;
                    acc.round_ms += Ln->prof.round_ms;
                    acc.round_bytes += Ln->prof.round_bytes;
                    acc.round_mults += Ln->prof.round_mults;
                    acc.bookkeep_ms += Ln->prof.bookkeep_ms;
                    acc.evaluate_ms += Ln->prof.evaluate_ms;
                } catch (const Error& e) {
                    codes[i] = e.code;
                    errs[i] = e.what();
                    if (auto* s = dynamic_cast<ShmComm*>(comms[li])) s->hdr->aborted.store(1);
                    break;
                } catch (const std::exception& e) {
                    codes[i] = DGKR_LOGIC_ERROR;
                    errs[i] = e.what();
                    if (auto* s = dynamic_cast<ShmComm*>(comms[li])) s->hdr->aborted.store(1);
                    break;
                }
            }
            if (lane_profiles) lane_profiles[li] = acc;
        };
        std::vector<std::thread> th;
        for (std::size_t i = 1; i < L; ++i) th.emplace_back(work, i);
        work(0);
        for (auto& t : th) t.join();
        for (std::size_t i = 0; i < n; ++i)
            if (codes[i] != DGKR_OK) fail(codes[i], "proof " + std::to_string(i) + ": " + errs[i]);
    });
}

int dgkr_gkr_prove_dist(dgkr_ctx* ctx, dgkr_comm* comm, dgkr_circuit* c, const dgkr_field* f,
                        const std::uint8_t* inputs, dgkr_transcript* t, std::uint8_t* proof, std::size_t cap,
                        std::size_t* len) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        Transcript tr(&f->f, t->state, t->draws);
        *len = gkr_prove(ctx, *c, workspace(*c, 0), f, inputs, tr, proof, cap, comm);
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        ctx->end_call();
    });
}

int dgkr_gkr_prove_dist_emulated(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, int world,
                                 const std::uint8_t* inputs_all, dgkr_transcript* t, std::uint8_t* proof,
                                 std::size_t cap, std::size_t* len) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (world < 1 || world > 64 || (world & (world - 1)) != 0) fail(DGKR_INVALID_ARGUMENT, "world must be 1..64, pow2");
        if (!inputs_all) fail(DGKR_INVALID_ARGUMENT, "inputs must not be NULL");
        const std::size_t in_bytes = static_cast<std::size_t>(c->input_size) * c->n_copies * f->f.width();
        std::vector<Lane*> lanes(world);
        for (int r = 0; r < world; ++r) {
            lanes[r] = ctx->lane(r);
            workspace(*c, r);
        }
        ctx->use(f);
        ThreadGroup group;
        group.world = world;
        std::vector<ThreadComm> comms(world);
        std::vector<std::vector<std::uint8_t>> bufs(world);
        std::vector<std::size_t> lens(world, 0);
        std::vector<dgkr_transcript> ts(world, *t);
        std::vector<int> codes(world, DGKR_OK);
        std::vector<std::string> errs(world);
        for (int r = 0; r < world; ++r) {
            comms[r].rank = r;
            comms[r].world = world;
            comms[r].g = &group;
            if (r) bufs[r].resize(cap);
        }
        auto work = [&](int r) {
            try {
                CK(cudaSetDevice(ctx->device));
                Lane* L = lanes[r];
                L->begin_call();
                Transcript tr(&f->f, ts[r].state, ts[r].draws);
                std::uint8_t* dst = r ? bufs[r].data() : proof;
                lens[r] = gkr_prove(L, *c, workspace(*c, r), f, inputs_all + r * in_bytes, tr, dst, cap, &comms[r]);
                std::memcpy(ts[r].state, tr.state().data(), 32);
                ts[r].draws = tr.draws();
                L->end_call();
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
        // every rank must hold the identical proof (outside the claimed-output
        // block, which only rank 0 gathers) and transcript
        const std::size_t ob = 4 + c->full_padded[c->depth] * static_cast<std::size_t>(world) * f->f.width();
        for (int r = 1; r < world; ++r) {
            if (lens[r] != lens[0] || std::memcmp(bufs[r].data(), proof, 4) != 0 ||
                std::memcmp(bufs[r].data() + ob, proof + ob, lens[0] - ob) != 0 ||
                std::memcmp(ts[r].state, ts[0].state, 32) != 0 || ts[r].draws != ts[0].draws)
                fail(DGKR_LOGIC_ERROR, "ranks disagree on the proof");
        }
        *len = lens[0];
        *t = ts[0];
    });
}

int dgkr_ctx_get_profile_lane(dgkr_ctx* ctx, int lane, dgkr_profile* out) {
    return guard([&] {
        if (lane < 0 || lane >= 64) fail(DGKR_OUT_OF_RANGE, "lane");
        *out = ctx->lane(lane)->prof;
    });
}

int dgkr_ctx_event_record(dgkr_ctx* ctx, int slot) {
    return guard([&] {
        if (slot < 0 || slot >= 8) fail(DGKR_OUT_OF_RANGE, "event slot");
        if (!ctx->user_ev[slot]) CK(cudaEventCreate(&ctx->user_ev[slot]));
        CK(cudaEventRecord(ctx->user_ev[slot], ctx->st));
    });
}

int dgkr_ctx_event_elapsed(dgkr_ctx* ctx, int a, int b, float* ms) {
    return guard([&] {
        if (a < 0 || a >= 8 || b < 0 || b >= 8 || !ctx->user_ev[a] || !ctx->user_ev[b])
            fail(DGKR_OUT_OF_RANGE, "event slot");
        CK(cudaEventSynchronize(ctx->user_ev[b]));
        CK(cudaEventElapsedTime(ms, ctx->user_ev[a], ctx->user_ev[b]));
    });
}

int dgkr_host_register(void* ptr, std::size_t bytes) {
    return guard([&] { CK(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault)); });
}
int dgkr_host_unregister(void* ptr) {
    return guard([&] { CK(cudaHostUnregister(ptr)); });
}

int dgkr_set_tuning(const char* name, std::uint64_t value) {
    return guard([&] {
        const std::string n = name ? name : "";
        if (n == "small_round_pairs") tuning().small_round_pairs = value;
        else if (n == "tma_min_pairs") tuning().tma_min_pairs = value;
        else if (n == "fuse_round1") tuning().fuse_round1 = value;
        else if (n == "tail_pairs") tuning().tail_pairs = value;
        else if (n == "tail_timeout_us") tuning().tail_timeout_us = value;
        else if (n == "spin_yield") tuning().spin_yield = value;
        else if (n == "absorb_chains") {
            if (value < 1 || value > 4) fail(DGKR_INVALID_ARGUMENT, "absorb_chains must be 1..4");
            tuning().absorb_chains = value;
        }
        else fail(DGKR_INVALID_ARGUMENT, "unknown tuning knob: " + n);
    });
}

int dgkr_get_tuning(const char* name, std::uint64_t* value) {
    return guard([&] {
        const std::string n = name ? name : "";
        if (n == "small_round_pairs") *value = tuning().small_round_pairs;
        else if (n == "tma_min_pairs") *value = tuning().tma_min_pairs;
        else if (n == "fuse_round1") *value = tuning().fuse_round1;
        else if (n == "tail_pairs") *value = tuning().tail_pairs;
        else if (n == "tail_timeout_us") *value = tuning().tail_timeout_us;
        else if (n == "spin_yield") *value = tuning().spin_yield;
        else if (n == "absorb_chains") *value = tuning().absorb_chains;
        else fail(DGKR_INVALID_ARGUMENT, "unknown tuning knob: " + n);
    });
}

int dgkr_bench_mul_peak(dgkr_ctx* ctx, double* mults_per_s) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        DBuf<Fe> sink;
        sink.ensure(1);
        const int blocks = ctx->sms * 8, iters = 4096;
        launch_mul_peak(blocks, 64, sink.p, ctx->st);  // warm-up
        CK(cudaEventRecord(ctx->ev0, ctx->st));
        launch_mul_peak(blocks, iters, sink.p, ctx->st);
        CK(cudaEventRecord(ctx->ev1, ctx->st));
        CK(cudaEventSynchronize(ctx->ev1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        *mults_per_s = static_cast<double>(blocks) * 256.0 * iters * 4.0 / (ms * 1e-3);
    });
}

int dgkr_pcs_commit(dgkr_ctx* ctx, const dgkr_field* f, std::size_t rows, std::size_t cols, const std::uint8_t* data,
                    std::uint8_t* root32) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        PcsDevice& d = ctx->nttws().pcs;  // persistent: multi-GiB buffers are not reallocated per call
        const Digest root = pcs_commit(ctx, f, d, rows, cols, data);
        std::memcpy(root32, root.data(), 32);
        ctx->end_call();
    });
}

int dgkr_pcs_open(dgkr_ctx* ctx, const dgkr_field* f, std::size_t rows, std::size_t cols, const std::uint8_t* data,
                  const std::uint8_t* r, std::size_t r_len, std::size_t q, dgkr_transcript* t, std::uint8_t* out,
                  std::size_t cap, std::size_t* len) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        const HostField& F = f->f;
        std::vector<U256> pt(r_len);
        for (std::size_t i = 0; i < r_len; ++i) pt[i] = F.from_bytes(r + i * F.width());
        Transcript tr(&f->f, t->state, t->draws);
        PcsDevice& d = ctx->nttws().pcs;
        const std::size_t need = pcs_opening_size(F.width(), r_len, rows, cols, q);
        *len = need;
        if (need > cap) fail(DGKR_CAPACITY, "output buffer too small");
        pcs_open(ctx, f, d, rows, cols, data, pt, q, tr, nullptr, out, cap);
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        ctx->end_call();
    });
}

int dgkr_dist_sumcheck_comm(dgkr_ctx* ctx, dgkr_comm* comm, const dgkr_field* f, std::size_t n_pairs,
                            std::size_t local_vars, const std::uint8_t* local_tables, dgkr_transcript* t,
                            std::uint8_t* proof, std::size_t cap, std::size_t* len) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        if (!comm) fail(DGKR_INVALID_ARGUMENT, "no communicator");
        if ((comm->world & (comm->world - 1)) != 0) fail(DGKR_INVALID_ARGUMENT, "world size must be a power of two");
        Transcript tr(&f->f, t->state, t->draws);
        DistTail dt;
        DBuf<Fe> tabs;
        RoundBuffers rb;
        auto bytes = product_sumcheck_dist(ctx, f, n_pairs, local_vars, local_tables, tr, comm, dt, tabs, rb);
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        ctx->end_call();
        emit(bytes, proof, cap, len);
    });
}

int dgkr_dist_sumcheck_emulated(dgkr_ctx* ctx, const dgkr_field* f, int world, std::size_t n_pairs, std::size_t vars,
                                const std::uint8_t* tables, dgkr_transcript* t, std::uint8_t* proof, std::size_t cap,
                                std::size_t* len) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (world < 1 || world > 64 || (world & (world - 1)) != 0) fail(DGKR_INVALID_ARGUMENT, "world must be 1..64, pow2");
        if (n_pairs == 0) fail(DGKR_INVALID_ARGUMENT, "nothing to shard");
        const std::uint64_t total = std::uint64_t{1} << vars;
        if (total % static_cast<std::uint64_t>(world) != 0)
            fail(DGKR_INVALID_ARGUMENT, "worker count must divide table size");  // cluster.hpp:196-198
        const std::size_t lv = vars - log2_exact(static_cast<std::uint64_t>(world));
        const std::size_t w = f->f.width();
        const std::size_t chunk = (std::size_t{1} << lv) * w;
        // shard_pairs (cluster.hpp:200-215): rank r's slice of every table, f_0 g_0 f_1 g_1 ...
        std::vector<std::vector<std::uint8_t>> shares(world, std::vector<std::uint8_t>(2 * n_pairs * chunk));
        for (int r = 0; r < world; ++r)
            for (std::size_t tb = 0; tb < 2 * n_pairs; ++tb)
                std::memcpy(shares[r].data() + tb * chunk, tables + tb * total * w + r * chunk, chunk);
        std::vector<Lane*> lanes(world);
        for (int r = 0; r < world; ++r) lanes[r] = ctx->lane(r);
        ctx->use(f);
        ThreadGroup group;
        group.world = world;
        std::vector<ThreadComm> comms(world);
        std::vector<std::vector<std::uint8_t>> outs(world);
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
                Transcript tr(&f->f, ts[r].state, ts[r].draws);
                DistTail dt;
                DBuf<Fe> tabs;
                RoundBuffers rb;
                outs[r] = product_sumcheck_dist(L, f, n_pairs, lv, shares[r].data(), tr, &comms[r], dt, tabs, rb);
                std::memcpy(ts[r].state, tr.state().data(), 32);
                ts[r].draws = tr.draws();
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
            if (outs[r] != outs[0] || std::memcmp(ts[r].state, ts[0].state, 32) != 0)
                fail(DGKR_LOGIC_ERROR, "ranks disagree on the proof");
        *t = ts[0];
        emit(outs[0], proof, cap, len);
    });
}

int dgkr_dist_sumcheck(dgkr_ctx* ctx, const dgkr_field* f, std::size_t n_workers, std::size_t n_pairs,
                       std::size_t vars, const std::uint8_t* tables, dgkr_transcript* t, std::uint8_t* proof,
                       std::size_t cap, std::size_t* len, char* traffic_json, std::size_t json_cap) {
    return guard([&] {
        ctx->begin_call();
        CK(cudaSetDevice(ctx->device));
        if (n_pairs == 0) fail(DGKR_INVALID_ARGUMENT, "nothing to shard");  // cluster.hpp:192-194
        const std::uint64_t total = std::uint64_t{1} << vars;
        if (n_workers == 0 || total % n_workers != 0)
            fail(DGKR_INVALID_ARGUMENT, "worker count must divide table size");  // :196-198
        plan_clusters(n_workers, 0);
        // dist_sumcheck is byte-identical to the single-machine prover over
        // the concatenated tables (cluster.hpp:219-227); on one device the
        // shards are contiguous slices of the same tables.
        Transcript tr(&f->f, t->state, t->draws);
        auto bytes = product_sumcheck(ctx, f, n_pairs, vars, tables, tr, nullptr);
        std::memcpy(t->state, tr.state().data(), 32);
        t->draws = tr.draws();
        // logical metering (cluster.hpp:258-298)
        Traffic ts;
        ts.cur = "sumcheck";
        const std::size_t w = f->f.width();
        const std::size_t local_vars = log2_exact(total / n_workers);
        for (std::size_t i = 0; i < n_workers; ++i) ts.msg(i, 0, 0, w);
        for (std::size_t j = 0; j < local_vars; ++j) {
            for (std::size_t i = 0; i < n_workers; ++i) ts.msg(i, 0, 0, 4 * w);
            for (std::size_t i = 0; i < n_workers; ++i) ts.msg(0, i, 0, w);
        }
        for (std::size_t i = 0; i < n_workers; ++i) ts.msg(i, 0, 0, 2 * n_pairs * w);
        write_json(ts.json(), traffic_json, json_cap);
        ctx->end_call();
        emit(bytes, proof, cap, len);
    });
}

/// DistPc::commit + open (cluster.hpp:336-412) over the K = plan(N) clusters,
/// spread over the given contexts (devices): worker i's row lives on context
/// i mod n_ctx, cluster c is assembled on its leader's (worker c*M) context
/// by peer copies of the member rows (the mempool, metered as mempool bytes,
/// cluster.hpp:349-361), each cluster on its own lane (stream + host thread),
/// so the leaders hash in parallel and the K opening transcripts
/// (independent by construction, cluster.hpp:445-449) run on K host threads;
/// the open reuses the matrix and tree its commit built.
int dgkr_distpc_multi(dgkr_ctx* const* ctxs, std::size_t n_ctx, const dgkr_field* f, std::size_t n_workers,
                      std::size_t n_clusters, std::size_t row_vars, const std::uint8_t* rows, const std::uint8_t* r,
                      std::size_t r_len, std::size_t q, std::uint8_t* roots_out, std::size_t* n_roots,
                      std::uint8_t* open_out, std::size_t cap, std::size_t* open_len, std::uint8_t* combined_out,
                      char* traffic_json, std::size_t json_cap) {
    return guard([&] {
        if (!ctxs || n_ctx == 0) fail(DGKR_INVALID_ARGUMENT, "no device context");
        for (std::size_t i = 0; i < n_ctx; ++i) ctxs[i]->begin_call();
        const HostField& F = f->f;
        const std::size_t K = plan_clusters(n_workers, n_clusters);
        const std::size_t M = n_workers / K;
        if (row_vars > 40) fail(DGKR_INVALID_ARGUMENT, "rows too large");
        const std::size_t cols = std::size_t{1} << row_vars;
        const std::size_t w = F.width();
        const std::size_t row_bytes = cols * w;
        std::size_t member_vars = log2_exact(M), cluster_vars = log2_exact(K);
        if (r_len != row_vars + member_vars + cluster_vars) fail(DGKR_INVALID_ARGUMENT, "opening point has wrong dimension");
        std::vector<U256> pt(r_len);
        for (std::size_t i = 0; i < r_len; ++i) pt[i] = F.from_bytes(r + i * w);
        const std::vector<U256> r_local(pt.begin(), pt.begin() + static_cast<std::ptrdiff_t>(row_vars + member_vars));
        const std::vector<U256> r_top(pt.begin() + static_cast<std::ptrdiff_t>(row_vars + member_vars), pt.end());
        const std::size_t osz = pcs_opening_size(w, r_local.size(), M, cols, q);
        // every cluster opening has the same size: written in place, u32 length first
        *open_len = K * (4 + osz);
        if (*open_len > cap) fail(DGKR_CAPACITY, "output buffer too small");
        std::vector<std::size_t> op_len(K, 0);
        std::vector<U256> values(K);
        std::vector<Digest> roots(K);
        std::vector<int> codes(K, DGKR_OK);
        std::vector<std::string> errs(K);
        // Placement: worker i holds its row on context i mod n_ctx (its own
        // lane there); cluster c's leader is worker c*M (cluster.hpp:24-36), so
        // the cluster is assembled, committed and opened on context
        // (c*M) mod n_ctx. Member rows move device to device (peer copies)
        // into the leader's matrix: the mempool writes (cluster.hpp:349-361).
        for (std::size_t i = 0; i < n_ctx; ++i)  // direct peer copies (NVLink) where the devices allow
            for (std::size_t j = 0; j < n_ctx; ++j) {
                const int di = ctxs[i]->device, dj = ctxs[j]->device;
                int can = 0;
                if (di == dj || cudaDeviceCanAccessPeer(&can, di, dj) != cudaSuccess || !can) continue;
                CK(cudaSetDevice(di));
                const cudaError_t e = cudaDeviceEnablePeerAccess(dj, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                (void)cudaGetLastError();
            }
        const std::size_t n_threads = std::min<std::size_t>(K, 16);
        auto work = [&](std::size_t th) {
            for (std::size_t c = th; c < K; c += n_threads) {
                try {
                    dgkr_ctx* cx = ctxs[(c * M) % n_ctx];
                    Lane* L = cx->lane(static_cast<int>(1 + c));
                    PcsDevice& d = L->nttws().pcs;
                    const std::uint8_t* mine = rows + c * M * row_bytes;  // the cluster's rows (for the openings' columns)
                    check_matrix(M, cols);
                    // (1) every member uploads its own row on its own device
                    std::vector<const Fe*> src(M);
                    std::vector<int> src_dev(M);
                    for (std::size_t m = 0; m < M; ++m) {
                        const std::size_t wi = c * M + m;
                        dgkr_ctx* wc = ctxs[wi % n_ctx];
                        CK(cudaSetDevice(wc->device));
                        Lane* WL = wc->lane(static_cast<int>(1 + K + wi));
                        NttWs& ws = WL->nttws();
                        ws.worker_row.ensure(cols);
                        WL->upload_elems(f, rows + wi * row_bytes, cols, ws.worker_row.p, ws.worker_stage);  // synced
                        src[m] = ws.worker_row.p;
                        src_dev[m] = wc->device;
                    }
                    // (2) the leader pulls the member rows into its matrix (peer copies over NVLink
                    //     when the members sit on other GPUs), then commits (pcs.hpp:105-113)
                    CK(cudaSetDevice(cx->device));
                    d.m.ensure(M * cols);
                    for (std::size_t m = 0; m < M; ++m)
                        CK(cudaMemcpyPeerAsync(d.m.p + m * cols, cx->device, src[m], src_dev[m], cols * sizeof(Fe), L->st));
                    pcs_build_tree(L, f, d, M, cols);
                    L->d2h(roots[c].data(), d.nodes.p + 32, 32);
                    L->sync();
                    Transcript tr(&f->f, "dgkr.pc.cluster");  // cluster.hpp:445-449
                    tr.absorb_u64(c);
                    std::uint8_t* dst = open_out + c * (4 + osz);
                    op_len[c] = pcs_open(L, f, d, M, cols, mine, r_local, q, tr, &values[c], dst + 4, osz, true);
                    for (int i = 0; i < 4; ++i) dst[i] = static_cast<std::uint8_t>(op_len[c] >> (8 * i));
                } catch (const Error& e) {
                    codes[c] = e.code;
                    errs[c] = e.what();
                } catch (const std::exception& e) {
                    codes[c] = DGKR_LOGIC_ERROR;
                    errs[c] = e.what();
                }
            }
        };
        std::vector<std::thread> pool;
        for (std::size_t t = 1; t < n_threads; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& t : pool) t.join();
        for (std::size_t c = 0; c < K; ++c)
            if (codes[c] != DGKR_OK) fail(codes[c], "cluster " + std::to_string(c) + ": " + errs[c]);
        // TrafficStats in the reference's order (cluster.hpp:349-361, :368-371, :402-404)
        Traffic ts;
        ts.cur = "commit";
        for (std::size_t i = 0; i < n_workers; ++i) ts.mempool(row_bytes);
        for (std::size_t c = 0; c < K; ++c) {
            std::memcpy(roots_out + 32 * c, roots[c].data(), 32);
            ts.msg(c * M, 0, 0, 32);
        }
        *n_roots = K;
        ts.cur = "open";
        U256 combined{};
        for (std::size_t c = 0; c < K; ++c) {
            ts.msg(c * M, 0, 0, op_len[c]);
            combined = F.add(combined, F.mul(chi_eval_host(c, r_top, F), values[c]));
        }
        F.to_bytes(combined, combined_out);
        write_json(ts.json(), traffic_json, json_cap);
        for (std::size_t i = 0; i < n_ctx; ++i) ctxs[i]->end_call();
    });
}

int dgkr_distpc(dgkr_ctx* ctx, const dgkr_field* f, std::size_t n_workers, std::size_t n_clusters,
                std::size_t row_vars, const std::uint8_t* rows, const std::uint8_t* r, std::size_t r_len,
                std::size_t q, std::uint8_t* roots_out, std::size_t* n_roots, std::uint8_t* open_out, std::size_t cap,
                std::size_t* open_len, std::uint8_t* combined_out, char* traffic_json, std::size_t json_cap) {
    dgkr_ctx* one[1] = {ctx};
    return dgkr_distpc_multi(one, 1, f, n_workers, n_clusters, row_vars, rows, r, r_len, q, roots_out, n_roots,
                             open_out, cap, open_len, combined_out, traffic_json, json_cap);
}

}  // extern "C"
