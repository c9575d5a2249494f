// Host-visible launcher interface for the sm_100a kernels in kernels.cu.
// Every launcher enqueues on `st` and never synchronises; the drivers in
// prover.cpp own ordering and host<->device traffic.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dgkr_b200 {

struct Fe;  // 8 x u32 Montgomery limbs (fe.hpp)

/// Which field policy a launch uses: the BN254 specialisation, the
/// runtime-modulus path for p < 2^254 (constants uploaded with
/// upload_rt_field()), or the wide runtime path for 2^254 <= p < 2^256
/// (carry-aware adds, no lazy differences, 10-limb products).
enum class FieldKind : int { Bn254 = 0, Runtime = 1, RuntimeWide = 2 };

struct RtFieldHost {
    std::uint32_t p[8];
    std::uint32_t np0;
    std::uint32_t r2[8];
    std::uint32_t one[8];
};

void upload_rt_field(const RtFieldHost& f, cudaStream_t st);

// canonical LE (width bytes/element) -> Montgomery; *err set to 1 on a value >= p
void launch_from_canonical(FieldKind k, const std::uint8_t* in, int width, Fe* out, std::uint64_t n, int* err,
                           cudaStream_t st);
void launch_to_canonical(FieldKind k, const Fe* in, std::uint8_t* out, int width, std::uint64_t n, cudaStream_t st);

/// Reduction workspace shared by all "sum to a few field elements" kernels.
struct ReduceWs {
    Fe* partials = nullptr;      // [max_blocks * 3]
    unsigned* counter = nullptr; // zero-initialised, self-resetting
    Fe* result = nullptr;        // [3] (device)
    int max_blocks = 0;
    int num_sms = 0;
};

/// One sum-check round over pair tables (f_k, g_k) (+ optional G paired with
/// the implicit all-ones table). With fold=true the inputs are the previous
/// round's tables (size 4*n_out_pairs) folded with r into `out`
/// (size 2*n_out_pairs); with fold=false the inputs themselves are scanned.
/// Writes (S0, S1, S2) = (sum f0 g0, sum f1 g1, sum df dg) (+G terms into
/// S0/S1) to ws.result; the host forms c0=S0, c2=S2, c1=S1-S0-S2.
struct RoundLaunch {
    const Fe* const* in = nullptr;  // device array [2*np + has_g]
    Fe* const* out = nullptr;       // device array [2*np + has_g]
    int np = 0;
    bool has_g = false;
    int mode = 0;  // 0 scan (round 1), 1 fold natural->bit-reversed (round 2), 2 fold bit-reversed (rounds >= 3)
    std::uint64_t n_out_pairs = 0;
    const Fe* r = nullptr;          // device pointer to the fold challenge (unused by the round kernels)
    // host pointer to the fold constants {c_0..c_7, r} (9 x 32 bytes, field.cuh
    // FoldConst): c_k = r * 2^(32k+64) * R^-1 mod p; passed as kernel parameters
    const void* fold_const = nullptr;
    // false: compute only (S0, S2) into result[0..2) (S1 = claim - S0 on the host)
    bool need_s1 = true;
    // host copies of the in/out pointer arrays: enable the TMA-staged round
    // kernel (round_tma.cuh) for the layer tables (np = 1 with G) on large
    // rounds; null keeps the register-fed k_round
    const Fe* const* in_host = nullptr;
    Fe* const* out_host = nullptr;
};
constexpr std::size_t kFoldConstBytes = 9 * 32;
void launch_round(FieldKind k, const RoundLaunch& a, const ReduceWs& ws, cudaStream_t st);

/// Same as launch_round, but for small tables: one CTA, no grid reduction
/// (the tail rounds of every sum-check phase are latency-bound).
void launch_round_small(FieldKind k, const RoundLaunch& a, const ReduceWs& ws, cudaStream_t st);
constexpr std::uint64_t kSmallRoundPairs = 256;

/// Host <-> device mailbox of the tail kernel (pinned, mapped host memory,
/// one per lane). The two directions sit on separate 128-byte lines; each
/// side posts a tag (generation << 8 | round) after its payload and waits
/// for the other side's tag of the same round.
struct alignas(128) TailMailbox {
    volatile std::uint32_t d_seq;  // device -> host: sums of round (d_seq & 255) posted (nv + 1: finals
                                   // folded); kTailAbort when the CTA gave up waiting
    volatile std::uint32_t abort_round;  // with kTailAbort: tag | the round whose challenge it waited for
    std::uint32_t pad0[30];
    std::uint32_t sums[3][8];      // (S0, S1, S2) or (S0, S2), Montgomery form
    std::uint64_t diag[4];         // the launch's device time (ns): waiting for the host, computing + posting, total
    volatile std::uint32_t h_seq;  // host -> device: fold constants of the challenge of round (h_seq & 255) posted
    std::uint32_t pad2[31];
    std::uint8_t k[kFoldConstBytes];  // FoldConst of that challenge
};
constexpr std::uint32_t kTailAbort = 0xffffffffu;
/// how long the tail CTA waits for a challenge before it gives up (the host
/// then runs the remaining rounds as per-round launches): long against the
/// host's microseconds per round, short enough that a profiler serialising
/// launches (the host cannot answer while the kernel runs) costs little
constexpr std::uint64_t kTailTimeoutUs = 20000;

/// The last rounds of a sum-check (round j0..nv, every one with <=
/// tuning().tail_pairs output pairs) and the final fold in ONE launch of one
/// CTA: after each round the CTA posts its sums to `mb`, spins until the
/// host posts the fold constants of the challenge, and goes on (no launch,
/// copy or stream sync per round). Round j0's constants come in `fold_const`
/// (unused when j0 == 1). Tables ping-pong in A/B exactly like the
/// per-round launches (round j writes A when j is even), finals go to fin.
/// The kernel gives up after timeout_ns without a host answer (posts
/// abort_round and kTailAbort and exits); after the final fold it posts
/// tag | (nv + 1).
struct TailLaunch {
    const Fe* const* in = nullptr;
    Fe* const* buf_a = nullptr;
    Fe* const* buf_b = nullptr;
    Fe* const* fin = nullptr;
    int np = 0;
    bool has_g = false;
    bool need_s1 = true;
    int j0 = 1;
    int nv = 1;
    const void* fold_const = nullptr;
    TailMailbox* mb = nullptr;
    std::uint32_t tag = 0;  // generation << 8
    std::uint64_t timeout_ns = 0;
};
void launch_round_tail(FieldKind k, const TailLaunch& a, cudaStream_t st);

/// Process-wide launch tuning (dgkr_set_tuning; env DGKR_SMALL_PAIRS /
/// DGKR_TMA_MIN_PAIRS give the start values): rounds of <= small_round_pairs
/// output pairs run on one CTA; rounds of >= tma_min_pairs take the
/// TMA-staged kernel where it applies (0 disables it).
struct Tuning {
    std::uint64_t small_round_pairs;
    std::uint64_t tma_min_pairs;
    std::uint64_t fuse_round1;  // bookkeeping with round 1 fused (k_bookkeep_pairs) where it applies
    std::uint64_t absorb_chains;  // output absorbs interleaved per host thread in a proof stream (1..4)
    std::uint64_t tail_pairs;     // rounds of <= tail_pairs output pairs run in one mailbox launch (0: off)
    std::uint64_t tail_timeout_us;  // the tail CTA's wait for a challenge before it hands back to the host
    std::uint64_t spin_yield;       // host threads waiting on the GPU yield their core between polls
};
Tuning& tuning();

/// out[t][0] = in[t][0] + r (in[t][1] - in[t][0]) for each table t.
void launch_fold_final(FieldKind k, const Fe* const* in, Fe* const* out, int n_tabs, const Fe* r, cudaStream_t st);

/// sum_k sum_i f_k[i] g_k[i]  -> ws.result[0]
void launch_pair_total(FieldKind k, const Fe* const* tabs, int np, std::uint64_t n, const ReduceWs& ws,
                       cudaStream_t st);

/// eq-table jobs: out[b] = seed * chi_b(point), b < 2^nvars (one CTA per job).
struct EqJob {
    const Fe* point;
    const Fe* seed;   // device pointer to the seed value
    Fe* out;
    int nvars;
    int pad;
};
void launch_eq_build(FieldKind k, const EqJob* jobs, int n_jobs, cudaStream_t st);

/// Split-eq weight tables: w(g) = sum_t A[t][g & (2^klo - 1)] * B[t][g >> klo]
struct SplitEq {
    const Fe* A = nullptr;  // K * 2^klo
    const Fe* B = nullptr;  // K * 2^khi
    int K = 0;
    int klo = 0;
    int khi = 0;
    std::uint64_t offset = 0;  // added to every index (a rank's slice of the global hypercube)
};

/// Dense expansion of a split-eq: out[i] = sum_t A[t][i & m] * B[t][i >> klo], i < n
/// (coalesced; turns the per-wire split-eq lookups into one 32-byte gather).
/// fold_pow (8 canonical 2^(32k+64) mod p, 32 B each) and hc (>= 9 * 2^khi
/// elements of scratch) enable the BN254 single-term path: the B factor is
/// constant over 2^klo consecutive outputs, so each block multiplies by it
/// with the constant-multiplier product (field.cuh FoldConst; 1.6-1.7x CIOS).
/// Either may be null (generic CIOS path).
void launch_split_eq_expand(FieldKind k, const SplitEq& e, std::uint64_t n, Fe* out, cudaStream_t st,
                            const std::uint8_t* fold_pow = nullptr, Fe* hc = nullptr);
/// out[i] = dense[i] + sum_t seed_t A_t[lo] B_t[hi]  (one term reused from a dense chi table)
void launch_split_eq_expand_add(FieldKind k, const SplitEq& e, std::uint64_t n, const Fe* dense, Fe* out,
                                cudaStream_t st, const std::uint8_t* fold_pow = nullptr, Fe* hc = nullptr);

/// Per-slot description of a data-parallel layer: values are laid out as
/// n_copies blocks of 2^log_stride (copy = high bits).
struct SlotDesc {
    const Fe* V;             // source values (capacity >= side size, zero padded)
    Fe* out;                 // H_m (phase 1) or MA_m (phase 2), size 2^side
    const std::uint32_t* off;  // CSR offsets [2^log_stride + 1]
    const uint4* ent;        // CSR entries
    std::uint32_t log_stride;
    std::uint32_t pad;
};

struct BookkeepLaunch {
    const SlotDesc* slots = nullptr;  // device array [n_slots]
    int n_slots = 0;
    std::uint64_t T = 0;          // 2^side
    std::uint32_t n_copies = 1;
    std::uint32_t log_gcons = 0;  // consumer gate stride (log2)
    Fe* G = nullptr;              // G (phase 1) / C (phase 2)
    SplitEq w;                    // wire weights from the combined claim
    SplitEq u;                    // phase 2: chi_x(u) split tables
    const Fe* vx = nullptr;       // phase 2: V_m(u) per slot (device)
    const void* vx_const = nullptr;  // phase 2, single slot: host FoldConst of V_0(u) (kernel parameter)
    const Fe* wire_w = nullptr;   // explicit per-wire weights (entry .w = wire id), else gate_w / w
    const Fe* gate_w = nullptr;   // dense per-gate weights (global gate index), else split-eq w
    const Fe* eq_u = nullptr;     // phase 2: dense chi_x(u) table, else split-eq u
    // Single-slot fast path (layered circuits): CSR rows visited in a static
    // degree-sorted order so the 32 rows of a warp have equal length.
    const std::uint32_t* perm = nullptr;  // [2^log_stride] row (x or y local index) per position
    const uint2* seg = nullptr;           // [2^log_stride] (entry start, entry count) per position
    // Heavy rows (power-law degrees: constant wires, padding gates): CSR rows
    // with more than heavy_min entries are skipped by the one-thread-per-row
    // kernels and reduced by one CTA per (slot, copy, row) item instead;
    // items {slot, copy, local row, 0} sorted by the global row index, so the
    // merge adds partials to G without races.
    const uint4* heavy = nullptr;
    std::uint32_t n_heavy = 0;
    std::uint32_t heavy_min = 0xffffffffu;
    Fe* heavy_h = nullptr;  // scratch [n_heavy] per-item H_m / MA_m partials
    Fe* heavy_g = nullptr;  // scratch [n_heavy] per-item G / C partials
    // Row-pair path with the phase's first sum-check round fused in (single
    // slot, no heavy rows): one thread builds rows (2j, 2j+1) of a copy, the
    // pairs visited in a static order sorted by the larger row degree; then
    // it adds V0 H0 + G0 and (V1 - V0)(H1 - H0) of its pair to round 1's
    // (S0, S2) -- the sums k_round's kScan would re-read the tables for.
    const uint4* pseg = nullptr;  // [2^(log_stride-1)] {entry start of row 2j, count 2j, count 2j+1, 2j}
    ReduceWs r1{};                // round-1 sums land in r1.result[0..2)
};
/// Phase 1 / phase 2 bookkeeping; with a.pseg set (and no heavy rows) also
/// round 1 of the phase's sum-check: returns true if it was fused.
void launch_bookkeep_phase1(FieldKind k, const BookkeepLaunch& a, cudaStream_t st);
void launch_bookkeep_phase2(FieldKind k, const BookkeepLaunch& a, cudaStream_t st);

/// Layer evaluation (circuit.hpp:178-191) for a data-parallel layer.
struct EvalLaunch {
    Fe* out = nullptr;
    std::uint64_t n_write = 0;     // entries to write (gates + zero padding)
    std::uint64_t n_gates = 0;     // n_copies * sub gates
    std::uint32_t log_g = 0;       // sub gate stride (log2)
    const std::uint32_t* gstart = nullptr;  // [sub_gates + 1]
    const uint4* nested = nullptr;  // {kind | left_layer<<1 | right_layer<<16, left_gate, right_gate, 0}
    const Fe* const* layer_vals = nullptr;   // device array [depth+1]
    const std::uint32_t* layer_log_stride = nullptr;  // device array [depth+1]
    // optional [sub_gates] visit order: gates sorted by their mul-wire count so
    // a warp's threads take the same (add or mul) path
    const std::uint32_t* perm = nullptr;
};
void launch_evaluate(FieldKind k, const EvalLaunch& a, cudaStream_t st);

/// ws.result[0] = sum_g t[g] * A[g & m] * B[g >> klo]  (dense MLE evaluation, mle.hpp:51-61)
void launch_dense_eval(FieldKind k, const Fe* t, std::uint64_t n, const SplitEq& eq, const ReduceWs& ws,
                       cudaStream_t st);

/// Microbenchmark: n_blocks x 256 threads, each running `iters` dependent
/// steps of 4 independent BN254 Montgomery multiplication chains.
void launch_mul_peak(int n_blocks, int iters, Fe* sink, cudaStream_t st);

// ---- Reed-Solomon encoding (NTT) and FRI folding ------------------------
/// out[i] = A[i & (2^k - 1)] * B[i >> k] for i < n, where A[j] = base^j and
/// B[m] = base^(m 2^k) are built per thread by square-and-multiply.
void launch_pow_table(FieldKind k, const Fe& base, std::uint64_t n, Fe* out, Fe* scratch, cudaStream_t st);
/// out[brev(i)] = in[i] * (scale ? scale[i] : 1), i < 2^log_n  (scale: coset powers)
void launch_bitrev_scale(FieldKind k, const Fe* in, const Fe* scale, Fe* out, int log_n, std::uint64_t n_in,
                         cudaStream_t st);
/// in-place radix-2 DIT NTT stages on bit-reversed input; tw[i] = w_N^i, i < N/2
void launch_ntt(FieldKind k, Fe* a, int log_n, const Fe* tw, cudaStream_t st);
/// kernels launch_ntt issues for a 2^log_n transform (shared-memory stages + two-stage passes)
int ntt_launches(int log_n);
/// one FRI fold: out[i] = (f[i] + f[i+h] + beta * xinv_i * (f[i] - f[i+h])) / 2, h = n/2,
/// xinv_i = ginv * twinv[i * step]  (beta_const: host FoldConst of beta; ginv: host Fe
/// (32 bytes) of the layer's inverse coset shift)
void launch_fri_fold(FieldKind k, const Fe* f, std::uint64_t n, const Fe* twinv, std::uint64_t step,
                     const void* ginv, const void* beta_const, Fe* out, cudaStream_t st);

/// a[i] = a[i] * c for a per-launch constant (host FoldConst of c)
void launch_scale(FieldKind k, Fe* a, std::uint64_t n, const void* c_const, cudaStream_t st);
/// dst[i] = 32-byte record src[idx[i]] (Merkle nodes, field elements)
void launch_gather32(const void* src, const std::uint64_t* idx, std::uint64_t n, void* dst, cudaStream_t st);

/// Batched SHA-256 column digests (pcs.hpp:73-80): leaf[j] = SHA256(canon(m[0][j]) || ... || canon(m[M-1][j])).
void launch_column_digests(FieldKind k, const Fe* rows, std::uint64_t cols, int M, int width, std::uint8_t* leaves,
                           cudaStream_t st);
/// Merkle tree over 2^depth leaves in heap layout (merkle.hpp:16-28): nodes[i] = H(nodes[2i]||nodes[2i+1]).
void launch_merkle(std::uint8_t* nodes, std::uint64_t n_leaves, cudaStream_t st);
/// combined[j] = sum_i beta[i] * m[i][j]   (pcs.hpp:233-239)
void launch_beta_combine(FieldKind k, const Fe* rows, std::uint64_t cols, int M, const Fe* beta, Fe* out,
                         cudaStream_t st);

// ---- distinct.hpp (config C4) --------------------------------------------
/// ws.result[0] = sum_i F(items[i]) (Montgomery), F = distinct.hpp:17-27; off = Montgomery(2^32 - 1) (32 bytes)
void launch_ah(FieldKind k, const Fe* items, std::uint64_t n, const void* off, const ReduceWs& ws, cudaStream_t st);
/// *bad = 1 unless the canonical records strictly ascend
void launch_strict_ascent(const std::uint8_t* canon, int width, std::uint64_t n, int* bad, cudaStream_t st);
/// *bad = 1 if a canonical record exceeds n_max
void launch_bound_check(const std::uint8_t* canon, int width, std::uint64_t n, std::uint64_t n_max, int* bad,
                        cudaStream_t st);
/// counts[k] += #{x in [first, first+n): bit k of canonical F(x+1) - F(x) is set}, k < bits <= 256
void launch_bitchange(FieldKind k, std::uint64_t first, std::uint64_t n, int bits, const void* off,
                      unsigned long long* counts, cudaStream_t st);

// ---- beacon validator tree (beacon.hpp, config C3) -------------------------
/// leaves[i] = SHA256(64-byte record i) for i < n, the zero-leaf digest zc0 up to cap
void launch_beacon_leaves(const std::uint8_t* recs, std::uint64_t n, std::uint64_t cap, const std::uint8_t* zc0,
                          std::uint8_t* leaves, cudaStream_t st);
/// batched BeaconTree::verify_membership; siblings m x a x 32, zc = zero cache (depth+1 digests)
void launch_beacon_verify(const std::uint8_t* root, const std::uint8_t* recs, const std::uint8_t* leaves,
                          const std::uint8_t* sib, const std::uint64_t* idx, std::uint64_t m, int a, int depth,
                          const std::uint8_t* zc, std::uint8_t* ok, cudaStream_t st);
/// membership paths (leaf + a siblings) out of the active-subtree heap
void launch_beacon_paths(const std::uint8_t* nodes, int a, const std::uint64_t* idx, std::uint64_t m,
                         std::uint8_t* leaves, std::uint8_t* sib, cudaStream_t st);

}  // namespace dgkr_b200
