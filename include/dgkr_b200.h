/*
 * dgkr_b200 — C ABI of the B200 (sm_100a) Sisu distributed-GKR prover.
 *
 * This is the drop-in boundary for the reference's prover hot path
 * (/root/reference/proj/include/dgkr, a header-only C++20 library with no
 * FFI of its own). Every entry point below replaces one reference call; the
 * citation after each names it. Proof bytes, transcript state and roots are
 * bit-identical to the reference on the same inputs.
 *
 * Conventions
 *  - Field elements cross as canonical little-endian bytes of width
 *    ceil(bits(p)/8) (field.hpp:159-187): 32 B for BN254, 8 B for
 *    Goldilocks, 1 B for p = 97. Non-canonical inputs are rejected with
 *    DGKR_INVALID_ARGUMENT, as FieldElement::from_bytes throws
 *    std::invalid_argument.
 *  - A transcript is the caller-owned value {state, draws}: exactly the
 *    private state of dgkr::Transcript (transcript.hpp:127-129). Provers
 *    read and advance it in place.
 *  - Status codes mirror the reference's exception types so a C++ shim can
 *    rethrow the same type: INVALID_ARGUMENT -> std::invalid_argument,
 *    LOGIC_ERROR -> std::logic_error, DOMAIN_ERROR -> std::domain_error,
 *    OUT_OF_RANGE -> std::out_of_range. dgkr_last_error() returns the
 *    message (thread-local).
 *  - Output buffers: (out, cap, *len). *len is always set to the required
 *    size; DGKR_CAPACITY is returned when cap is too small.
 *  - No CPU fallback: provers run on the GPU or fail with DGKR_CUDA_ERROR.
 */
#ifndef DGKR_B200_H
#define DGKR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DGKR_OK 0
#define DGKR_INVALID_ARGUMENT 1
#define DGKR_LOGIC_ERROR 2
#define DGKR_DOMAIN_ERROR 3
#define DGKR_OUT_OF_RANGE 4
#define DGKR_CUDA_ERROR 5
#define DGKR_UNSUPPORTED 6
#define DGKR_CAPACITY 7
#define DGKR_COMM_ERROR 8

typedef struct dgkr_ctx dgkr_ctx;
typedef struct dgkr_field dgkr_field;
typedef struct dgkr_circuit dgkr_circuit;
typedef struct dgkr_pairsum dgkr_pairsum;

/* Transcript value: replaces the private members of dgkr::Transcript
 * (transcript.hpp:127-129). */
typedef struct dgkr_transcript {
    uint8_t state[32];
    uint64_t draws;
} dgkr_transcript;

/* Per-call profile (filled when dgkr_ctx_set_profile(ctx, 1)). */
typedef struct dgkr_profile {
    uint64_t launches;          /* kernels launched by this library */
    uint64_t round_launches;    /* fused fold+round kernels */
    double round_ms;            /* CUDA-event time inside fused round kernels */
    uint64_t round_bytes;       /* algorithmic bytes moved by round kernels */
    uint64_t round_mults;       /* algorithmic field multiplications in round kernels */
    double bookkeep_ms;         /* phase-1 + phase-2 bookkeeping kernels */
    double evaluate_ms;         /* circuit evaluation kernels */
    double total_ms;            /* wall time of the call */
    double host_transcript_ms;  /* serial host SHA-256 transcript work */
    double output_absorb_ms;    /* part of the above: absorbing the output layer */
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    uint64_t rounds;            /* sum-check rounds (host round trips) */
    double ntt_ms;              /* NTT / RS-encode kernels (bit-reverse + butterflies) */
    double merkle_ms;           /* leaf digests + Merkle tree kernels (PCS, FRI) */
    double fold_ms;             /* FRI fold kernels */
    double tail_ms;             /* sum-check tail launches (k_round_tail), incl. the host's
                                   transcript work between their rounds */
    uint64_t tail_rounds;       /* rounds run inside tail launches (not in round_ms / round_bytes) */
    uint64_t tail_aborts;       /* tail launches that gave up waiting for the host (rest run per round) */
} dgkr_profile;

const char* dgkr_last_error(void);
int dgkr_abi_version(void); /* 3 (round 2: dgkr_profile grew the tail_* fields) */

/* ---- field (field.hpp:23-80) ------------------------------------------- */
/* modulus: little-endian bytes. The GPU path supports any odd p < 2^256
 * (BN254 Fr is specialised; other moduli take the runtime-modulus path,
 * 2^254 <= p the wide variant of it). */
int dgkr_field_create(const uint8_t* modulus_le, size_t len, dgkr_field** out);
void dgkr_field_destroy(dgkr_field* f);
size_t dgkr_field_width(const dgkr_field* f);   /* field.hpp:67 byte_width() */
size_t dgkr_field_bits(const dgkr_field* f);    /* field.hpp:66 bits() */

/* ---- transcript (transcript.hpp:19-83); host-side, needs no GPU ---------- */
int dgkr_transcript_init(const dgkr_field* f, const char* label, dgkr_transcript* t);      /* ctor :19-28 */
int dgkr_transcript_absorb_bytes(const dgkr_field* f, dgkr_transcript* t, const uint8_t* data, size_t n); /* :32-37 */
int dgkr_transcript_absorb_u64(const dgkr_field* f, dgkr_transcript* t, uint64_t v);      /* :44-48 */
int dgkr_transcript_absorb_elems(const dgkr_field* f, dgkr_transcript* t, const uint8_t* elems, size_t n); /* :39-42 */
/* k independent transcripts, each absorbing its own n elements: the same
 * bytes as k calls of dgkr_transcript_absorb_elems. 32-byte fields run the
 * chains interleaved (multi-buffer SHA-NI); threads > 1 runs one host thread
 * per transcript through the proof stream's combining absorb scheduler. */
int dgkr_transcript_absorb_elems_multi(const dgkr_field* f, dgkr_transcript* const* ts, size_t k,
                                       const uint8_t* const* elems, size_t n, int threads);
int dgkr_transcript_challenge(const dgkr_field* f, dgkr_transcript* t, uint8_t* out);     /* :52-68 */
int dgkr_transcript_challenge_index(const dgkr_field* f, dgkr_transcript* t, uint64_t bound, uint64_t* out); /* :71-83 */
/* raw SHA-256 (sha256.hpp:138-151), exposed for tests */
int dgkr_sha256(const uint8_t* data, size_t n, uint8_t* out32);
int dgkr_sha256_has_shani(void);

/* ---- context -------------------------------------------------------------- */
int dgkr_ctx_create(int device, dgkr_ctx** out);
void dgkr_ctx_destroy(dgkr_ctx* ctx);
int dgkr_ctx_set_profile(dgkr_ctx* ctx, int on);
int dgkr_ctx_get_profile(dgkr_ctx* ctx, dgkr_profile* out);   /* profile of the last call */
int dgkr_ctx_device_info(dgkr_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor);

/* ---- product sum-check -----------------------------------------------------
 * prove_product_sum (sumcheck.hpp:226-241) over n_pairs pairs of 2^vars
 * tables given as f0,g0,f1,g1,... Proof = SumcheckProof::to_bytes
 * (sumcheck.hpp:51-61). */
int dgkr_prove_product_sum(dgkr_ctx* ctx, const dgkr_field* f, size_t n_pairs, size_t vars, const uint8_t* tables,
                           dgkr_transcript* t, uint8_t* proof, size_t cap, size_t* len);
/* ---- PairSumSession (sumcheck.hpp:152-221) --------------------------------------
 * The product sum-check's steps as separate calls (the cluster runtime drives
 * one session per worker, cluster.hpp:250-316). tables = f_0 g_0 f_1 g_1 ...,
 * each 2^vars canonical elements; copied to the device at begin (:168).
 * round: the round polynomial {c0, c1, c2, c3 = 0} of the current tables
 * (4 elements). fold: bind the next variable to r (canonical). finals: after
 * all folds, [f_0(r), g_0(r), f_1(r), ...] (2 n_pairs elements). Errors: the
 * reference's -- INVALID_ARGUMENT (no pairs), LOGIC_ERROR ("sumcheck session
 * exhausted" / "still has unbound variables"). */
int dgkr_pairsum_begin(dgkr_ctx* ctx, const dgkr_field* f, size_t n_pairs, size_t vars, const uint8_t* tables,
                       dgkr_pairsum** out);                                   /* PairSumSession ctor :154-171 */
void dgkr_pairsum_end(dgkr_pairsum* s);
size_t dgkr_pairsum_vars_left(const dgkr_pairsum* s);                        /* vars_left() :174 */
int dgkr_pairsum_total(dgkr_pairsum* s, uint8_t* out);                       /* total() :177-186 */
int dgkr_pairsum_round(dgkr_pairsum* s, uint8_t* out4);                      /* round_poly() :188-193 */
int dgkr_pairsum_fold(dgkr_pairsum* s, const uint8_t* r);                    /* fold(r) :195-201 */
int dgkr_pairsum_finals(dgkr_pairsum* s, uint8_t* out);                      /* final_values() :204-215 */

/* ---- layer sum-check -------------------------------------------------------
 * prove_layer_sum (sumcheck.hpp:342-448). wire_meta: n_wires x {is_mul,
 * x_slot, y_slot}; wire_idx: n_wires x {x_index, y_index}; wire_weights:
 * n_wires field elements. Proof = SumcheckProof::to_bytes; the x/y points
 * are written to x_point/y_point (side_vars elements each) when non-NULL. */
int dgkr_prove_layer_sum(dgkr_ctx* ctx, const dgkr_field* f, size_t side_vars, size_t n_slots,
                         const uint8_t* slot_tables, size_t n_wires, const uint32_t* wire_meta,
                         const uint64_t* wire_idx, const uint8_t* wire_weights, const uint8_t* claimed,
                         dgkr_transcript* t, uint8_t* proof, size_t cap, size_t* len, uint8_t* x_point,
                         uint8_t* y_point);

/* ---- circuits + GKR ----------------------------------------------------------
 * Flat layout of a GeneralCircuit (circuit.hpp:63):
 *   layer_gate_start[depth+1]  cumulative gate counts (gates of layer li, 1-based,
 *                              are [layer_gate_start[li-1], layer_gate_start[li]))
 *   gate_nested_start[G+1]     cumulative nested-gate counts per gate
 *   nested[5*N]                {kind (0 add, 1 mul), left_layer, left_gate,
 *                               right_layer, right_gate} per nested gate
 *   min_padded[depth+1]        reserve_padding() floors, or NULL
 * n_copies > 1 describes a data-parallel circuit (Sisu): the given circuit is
 * a sub-circuit replicated n_copies times, copy c of layer l occupying gates
 * [c*size_l, (c+1)*size_l) — the copy index is the high variables, as in
 * cluster.hpp:182-189. Requires n_copies and every sub layer size to be
 * powers of two. Validation follows GeneralCircuit::validate
 * (circuit.hpp:103-152); violations fail with DGKR_INVALID_ARGUMENT. */
int dgkr_circuit_create(dgkr_ctx* ctx, uint32_t input_size, uint32_t depth, const uint64_t* layer_gate_start,
                        const uint64_t* gate_nested_start, const uint32_t* nested, const uint64_t* min_padded,
                        uint32_t n_copies, dgkr_circuit** out);
void dgkr_circuit_destroy(dgkr_circuit* c);
/* padded size of the output layer of the (replicated) circuit */
size_t dgkr_circuit_output_size(const dgkr_circuit* c);
/* GeneralCircuit::evaluate (circuit.hpp:164-193): padded output layer */
int dgkr_circuit_evaluate(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, const uint8_t* inputs,
                          uint8_t* outputs, size_t cap, size_t* len);
/* gkr_prove (gkr.hpp:182-244). inputs: n_copies * input_size elements.
 * Proof bytes ("GkrProof layout"; the reference has no serializer,
 * gkr.hpp:86-95):
 *   u32 n_out || claimed_outputs || u32 n_layers ||
 *   per layer (output first): u32 n_alphas || alphas || u32 len || SumcheckProof::to_bytes */
int dgkr_gkr_prove(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, const uint8_t* inputs, dgkr_transcript* t,
                   uint8_t* proof, size_t cap, size_t* len);
size_t dgkr_gkr_proof_bound(const dgkr_circuit* c, const dgkr_field* f);
/* Split form of dgkr_gkr_prove for measurement with inputs resident in HBM:
 * load_inputs uploads + converts the inputs (not a reference call);
 * prove_resident then runs gkr_prove exactly as dgkr_gkr_prove does. */
int dgkr_circuit_load_inputs(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, const uint8_t* inputs);
int dgkr_gkr_prove_resident(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, dgkr_transcript* t,
                            uint8_t* proof, size_t cap, size_t* len);
/* n independent gkr_prove calls on the same circuit, run concurrently: proof
 * i on lane i (its own stream, workspace and host thread), so the serial
 * host transcript of one proof overlaps the GPU work of the others. Each
 * proof/transcript is exactly what dgkr_gkr_prove would produce for it.
 * inputs == NULL proves the inputs loaded with dgkr_circuit_load_inputs_lane.
 * All lanes must use the same field. */
int dgkr_gkr_prove_batch(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, size_t n,
                         const uint8_t* const* inputs, dgkr_transcript* ts, uint8_t* const* proofs,
                         const size_t* caps, size_t* lens);
/* n proofs over n_lanes lanes as a work queue (a lane takes the next proof
 * when it finishes one), so the host transcript phases of different proofs
 * stagger instead of coinciding. inputs == NULL: proof i runs on lane
 * i mod n_lanes and proves the inputs loaded there (static assignment). lane_profiles (n_lanes entries, or NULL)
 * receives each lane's accumulated counters. */
int dgkr_gkr_prove_stream(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, size_t n, size_t n_lanes,
                          const uint8_t* const* inputs, dgkr_transcript* ts, uint8_t* const* proofs,
                          const size_t* caps, size_t* lens, dgkr_profile* lane_profiles);
int dgkr_circuit_load_inputs_lane(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, int lane,
                                  const uint8_t* inputs);
int dgkr_ctx_get_profile_lane(dgkr_ctx* ctx, int lane, dgkr_profile* out);

/* Binary CSR circuit interchange (the reference's
 * JSON, circuit.hpp:227-277, is impractical at ~10^8 gates). Layout (LE):
 * "DGKRCSR1" | u32 input_size | u32 depth | u32 n_copies | u32 has_min_padded |
 * u64 n_gates | u64 n_nested | u64 layer_gate_start[depth+1] |
 * u64 gate_nested_start[n_gates+1] | u32 nested[n_nested][5] | u64 min_padded[depth+1]?
 * dgkr_circuit_load validates like dgkr_circuit_create; n_copies = 0 keeps the
 * file's copy count. */
int dgkr_circuit_save(const dgkr_circuit* c, const char* path);
int dgkr_circuit_load(dgkr_ctx* ctx, const char* path, uint32_t n_copies, dgkr_circuit** out);

/* gkr_verify + check_input_claims (gkr.hpp:253-325) on the host, for proofs in
 * the GkrProof layout above (single- or multi-GPU: the bytes are the same).
 * outputs (nullable): the claimed output statement, n_outputs canonical
 * elements, compared with the proof's padded outputs (padding must be zero);
 * inputs (nullable): the full input layer (n_copies x input_size canonical
 * elements); when given, the input-layer claims are discharged against it.
 * *accept = 1 iff everything verifies. Malformed proof bytes reject (no
 * error); the transcript is advanced like the reference verifier's. */
int dgkr_gkr_verify(const dgkr_circuit* c, const dgkr_field* f, const uint8_t* outputs, size_t n_outputs,
                    const uint8_t* inputs, const uint8_t* proof, size_t len, dgkr_transcript* t, int* accept);

/* The input-layer claims of a proof (registry[0] after gkr_verify, gkr.hpp:
 * 309-310), replayed like dgkr_gkr_verify, for composing the proof with a
 * commitment of the inputs (open the input table at each term's point and
 * check sum_t weight_t * value_t = claim value). out: u32 n_claims, per claim
 * u32 n_terms, per term (u32 n_vars, point, weight), then the value; canonical
 * elements. *accept = 0 (and no claims) when the proof does not verify. */
int dgkr_gkr_input_claims(const dgkr_circuit* c, const dgkr_field* f, const uint8_t* proof, size_t len,
                          dgkr_transcript* t, int* accept, uint8_t* out, size_t cap, size_t* out_len);

/* ---- multi-GPU data-parallel GKR (Sisu; cluster.hpp:182-320 generalised) ----
 * One process per GPU. Rank r proves copies [r*n, (r+1)*n) of a uniform-width
 * data-parallel circuit created with n_copies = n (the rank index is the top
 * log2(world) variables of every layer). Per sum-check round the only
 * traffic is an NCCL all-gather of 3 field elements per rank; at each phase
 * boundary one all-gather of the final table values; the claimed outputs are
 * all-gathered once. Every rank produces the identical proof and transcript,
 * byte-equal to the single-GPU proof of the full circuit. */
typedef struct dgkr_comm dgkr_comm;
int dgkr_comm_nccl_unique_id(uint8_t* out128);
int dgkr_comm_create_nccl(dgkr_ctx* ctx, const uint8_t* uid128, int rank, int world, dgkr_comm** out);
void dgkr_comm_destroy(dgkr_comm* comm);
/* One-node transport over POSIX shared memory (one segment per lane, named
 * e.g. "/dgkr_<token>_<lane>", same name on every rank; slot_bytes >= the
 * largest exchange, i.e. the claimed outputs of one rank). Per-lane segments
 * and barriers keep concurrently progressing lanes independent. */
int dgkr_comm_create_shm(dgkr_ctx* ctx, const char* name, int rank, int world, size_t slot_bytes,
                         dgkr_comm** out);
/* host-only all-gather through a shared-memory communicator (transport test hook) */
int dgkr_comm_allgather_host(dgkr_comm* comm, const void* in, size_t bytes, void* out);
/* n distributed proofs over n_lanes lanes, lane l using comms[l] and proving
 * l, l+n_lanes, ... in order on every rank (inputs NULL = lane-resident).
 * absorb_policy: which rank gathers proof i's claimed outputs and runs their
 * serial absorb (gkr.hpp:189-190) — 0: rank 0 for every proof; 1: rank
 * i mod world, so the host hash chains of concurrent proofs spread over all
 * ranks' cores. Every rank returns identical proof bytes except the claimed
 * output section, which only the absorbing rank fills (zeros elsewhere). */
int dgkr_gkr_prove_dist_stream(dgkr_ctx* ctx, dgkr_comm* const* comms, size_t n_lanes, dgkr_circuit* c,
                               const dgkr_field* f, size_t n, const uint8_t* const* inputs, dgkr_transcript* ts,
                               uint8_t* const* proofs, const size_t* caps, size_t* lens,
                               dgkr_profile* lane_profiles, int absorb_policy);
/* inputs: this rank's n*input_size elements, or NULL for inputs already loaded
 * with dgkr_circuit_load_inputs */
int dgkr_gkr_prove_dist(dgkr_ctx* ctx, dgkr_comm* comm, dgkr_circuit* c, const dgkr_field* f,
                        const uint8_t* inputs, dgkr_transcript* t, uint8_t* proof, size_t cap, size_t* len);
/* The same protocol with `world` ranks emulated as host threads driving
 * lanes of this one GPU (exchange through host memory); checks that every
 * rank produced the identical proof. inputs_all: world*n*input_size elements. */
int dgkr_gkr_prove_dist_emulated(dgkr_ctx* ctx, dgkr_circuit* c, const dgkr_field* f, int world,
                                 const uint8_t* inputs_all, dgkr_transcript* t, uint8_t* proof, size_t cap,
                                 size_t* len);

/* ---- measurement helpers (not reference calls) ------------------------------ */
/* CUDA events on the context's stream (slots 0..7) */
int dgkr_ctx_event_record(dgkr_ctx* ctx, int slot);
int dgkr_ctx_event_elapsed(dgkr_ctx* ctx, int slot_a, int slot_b, float* ms);
/* page-lock a caller buffer (cudaHostRegister) so proof D2H lands in place */
int dgkr_host_register(void* ptr, size_t bytes);
int dgkr_host_unregister(void* ptr);
/* Montgomery-multiplication throughput of the device (BN254), as the
 * measured integer-pipe roofline denominator: field mults per second. */
int dgkr_bench_mul_peak(dgkr_ctx* ctx, double* mults_per_s);
/* Process-wide launch tuning (no reference counterpart; proofs never depend
 * on it): "small_round_pairs" = largest round run on a single CTA (default
 * 256), "tma_min_pairs" = smallest round taking the TMA-staged round kernel
 * (default 0 = off: measured slower than the register-fed kernel on C2),
 * "fuse_round1" = 1 (default 0: measured slower) builds single-slot bookkeeping tables by row
 * pairs with round 1 of the phase fused in, "absorb_chains" = 1..4 (default
 * 1: measured best) output absorbs a host thread interleaves in a proof
 * stream, "tail_pairs" = the last rounds of a sum-check with <= this many
 * output pairs run in one launch that trades sums and challenges with the
 * host through a mapped-memory mailbox (default 256; 0 = one launch per
 * round), "tail_timeout_us" = how long that launch waits for a challenge
 * before it hands the remaining rounds back to per-round launches (default
 * 20000; a profiler that serialises launches hits it once per sum-check),
 * "spin_yield" = 1 makes host threads waiting on the GPU yield their core
 * between polls (default 0: measured no faster).
 * Unknown names -> DGKR_INVALID_ARGUMENT. */
int dgkr_set_tuning(const char* name, uint64_t value);
int dgkr_get_tuning(const char* name, uint64_t* value);

/* ---- polynomial commitment (pcs.hpp) ------------------------------------------ */
/* pcs::commit (pcs.hpp:105-113): rows x cols row-major matrix -> Merkle root */
int dgkr_pcs_commit(dgkr_ctx* ctx, const dgkr_field* f, size_t rows, size_t cols, const uint8_t* data,
                    uint8_t* root32);
/* pcs::open (pcs.hpp:212-254): Opening::to_bytes (pcs.hpp:135-156) */
int dgkr_pcs_open(dgkr_ctx* ctx, const dgkr_field* f, size_t rows, size_t cols, const uint8_t* data,
                  const uint8_t* r, size_t r_len, size_t spot_checks, dgkr_transcript* t, uint8_t* out, size_t cap,
                  size_t* len);

/* ---- Reed-Solomon encoding and FRI (north-star "Virgo/FRI" commitment) ------------
 * No reference implementation exists: the reference replaced Virgo's VPD with
 * the Merkle column commitment above. These entry points are
 * our own specification, pinned by oracle/fri_oracle.py.
 *   two-adic data: p - 1 = 2^s t; w = z^t has order 2^s where z is the smallest
 *   quadratic non-residue, which is also the coset shift g.
 *   dgkr_ntt:  out[i] = sum_j in[j] w_N^(ij)  (inverse: w^-1 and 1/N), natural order
 *   dgkr_rs_encode: out[i] = f(g w_N^i), f = coeffs (n), N = n << blowup_log
 *   dgkr_fri_prove: L = log2(N) - final_log folds of the RS codeword of coeffs;
 *     per layer l: root_l = Merkle(SHA256(canon(f_l[j]))), absorb root_l,
 *     beta_l = challenge, f_{l+1}[i] = (f_l[i] + f_l[i+h]) / 2
 *                                       + beta_l (f_l[i] - f_l[i+h]) / (2 x_i),
 *     x_i = g^(2^l) w_N^(2^l i), h = N_l / 2; absorb every element of f_L;
 *     Q = min(queries, N/2) distinct challenge_index(N/2) positions.
 *   proof = u32 L || L roots || u32 |f_L| || f_L || u32 Q || per query:
 *     u32 i || per layer l: f_l[i mod h_l] || f_l[i mod h_l + h_l] || their two Merkle paths */
/*   dgkr_fri_prove_dist: distributed FRI (BASELINE config C5 at N GPUs), rank r
 *     holding the r-th chunk of n coefficients (one polynomial per rank, shared
 *     Fiat-Shamir): per layer every rank's root is all-gathered and absorbed in
 *     rank order before beta_l is drawn; all ranks' final layers are absorbed
 *     in rank order; the Q query positions (over this rank's half domain) are
 *     shared. proof_r = u32 world || u32 rank || u32 L || L x world roots
 *     (layer-major, rank order) || u32 |f_L| || world x |f_L| final elements ||
 *     u32 Q || per query: u32 i || per layer this rank's two values + paths.
 *   dgkr_fri_prove_dist_emulated: the same with `world` ranks as host threads
 *     on lanes of one device (coeffs[r] = rank r's chunk); proofs[r], lens[r]. */
int dgkr_field_ntt_info(const dgkr_field* f, unsigned* two_adicity, uint8_t* root, uint8_t* coset);
int dgkr_ntt(dgkr_ctx* ctx, const dgkr_field* f, const uint8_t* in, unsigned log_n, int inverse, uint8_t* out);
int dgkr_rs_encode(dgkr_ctx* ctx, const dgkr_field* f, const uint8_t* coeffs, size_t n, unsigned blowup_log,
                   uint8_t* out);
int dgkr_fri_prove(dgkr_ctx* ctx, const dgkr_field* f, const uint8_t* coeffs, size_t n, unsigned blowup_log,
                   unsigned final_log, size_t queries, dgkr_transcript* t, uint8_t* proof, size_t cap, size_t* len);
int dgkr_fri_prove_dist(dgkr_ctx* ctx, dgkr_comm* comm, const dgkr_field* f, const uint8_t* coeffs, size_t n,
                        unsigned blowup_log, unsigned final_log, size_t queries, dgkr_transcript* t, uint8_t* proof,
                        size_t cap, size_t* len);
int dgkr_fri_prove_dist_emulated(dgkr_ctx* ctx, const dgkr_field* f, int world, const uint8_t* const* coeffs, size_t n,
                                 unsigned blowup_log, unsigned final_log, size_t queries, dgkr_transcript* t,
                                 uint8_t* const* proofs, const size_t* caps, size_t* lens);

/* ---- distinct indexes: associative array hash (distinct.hpp; config C4) ------------
 * F(e) = three rounds of r <- (r + e + 2^32 - 1)^3 from r = 0; AH(list) = sum F(e_i),
 * 0 for the empty list. Items cross as canonical bytes (width), non-canonical
 * encodings fail with DGKR_INVALID_ARGUMENT (FieldElement::from_bytes).
 *   dgkr_distinct_ah            distinct::ah                      distinct.hpp:37-44
 *   dgkr_distinct_check         distinct::pairwise_distinct_check distinct.hpp:53-68
 *                               (*ok = AH(a) == AH(a_sorted) and a_sorted strictly ascends)
 *   dgkr_distinct_chain_update  distinct::chain_update            distinct.hpp:82-92
 *                               (h_out = h + AH(items); DGKR_OUT_OF_RANGE if an item > n_max)
 *   dgkr_distinct_bitchange     distinct::bitchange_experiment    distinct.hpp:112-145
 *                               (set_counts[k], k < bits(p): #x in 1..count with bit k of
 *                               canonical F(x+1) - F(x) set; probability = count_k / count;
 *                               DGKR_INVALID_ARGUMENT if count < 10^4) */
int dgkr_distinct_ah(dgkr_ctx* ctx, const dgkr_field* f, const uint8_t* items, size_t n, uint8_t* out);
int dgkr_distinct_check(dgkr_ctx* ctx, const dgkr_field* f, const uint8_t* a, size_t n_a, const uint8_t* a_sorted,
                        size_t n_sorted, int* ok);
int dgkr_distinct_chain_update(dgkr_ctx* ctx, const dgkr_field* f, const uint8_t* h, uint64_t n_max,
                               const uint8_t* items, size_t n, uint8_t* h_out);
int dgkr_distinct_bitchange(dgkr_ctx* ctx, const dgkr_field* f, size_t count, uint64_t* set_counts);

/* ---- beacon validator tree (beacon.hpp; config C3) ----------------------------------
 * records: n x 64 bytes, each ValidatorRecord::encode() (pubkey | LE64 index |
 * active flag | zero pad, beacon.hpp:27-37). SSZ-style tree of `depth` over a
 * left-aligned active subtree of 2^a leaves (a = ceil log2 n), zero-cache
 * digests above it (beacon.hpp:96-132).
 *   dgkr_beacon_root    BeaconTree(validators, depth).root()
 *                       (DGKR_INVALID_ARGUMENT if a > depth)
 *   dgkr_beacon_prove   prove_membership(indices[i]) for m indices: leaves m x 32,
 *                       siblings m x a x 32 (leaf to root), *active_log2 = a
 *                       (DGKR_OUT_OF_RANGE for an index >= n, beacon.hpp:136-149)
 *   dgkr_beacon_verify  verify_membership (beacon.hpp:151-174) per path, batched:
 *                       ok[i] = 1 iff SHA256(record i) = leaf i, the index lies in
 *                       the active region and the recomputed root equals root */
int dgkr_beacon_root(dgkr_ctx* ctx, const uint8_t* records, size_t n, unsigned depth, uint8_t* root);
int dgkr_beacon_prove(dgkr_ctx* ctx, const uint8_t* records, size_t n, unsigned depth, const uint64_t* indices,
                      size_t m, uint8_t* leaves, uint8_t* siblings, unsigned* active_log2);
int dgkr_beacon_verify(dgkr_ctx* ctx, const uint8_t* root, const uint8_t* records, const uint8_t* leaves,
                       const uint8_t* siblings, const uint64_t* indices, size_t m, unsigned depth,
                       unsigned active_log2, uint8_t* ok);

/* ---- distributed runtime (cluster.hpp), N workers in one call -------------------
 * shard_pairs + dist_sumcheck (cluster.hpp:190-320) on full tables; proof
 * bytes equal the reference's, TrafficStats::to_json().dump() written to
 * traffic_json (phase "sumcheck"). */
int dgkr_dist_sumcheck(dgkr_ctx* ctx, const dgkr_field* f, size_t n_workers, size_t n_pairs, size_t vars,
                       const uint8_t* tables, dgkr_transcript* t, uint8_t* proof, size_t cap, size_t* len,
                       char* traffic_json, size_t json_cap);
/* dist_sumcheck over real devices: this rank's share (rows [rank 2^lv, (rank+1) 2^lv) of
 * every table, f_0 g_0 f_1 g_1 ..., shard_pairs cluster.hpp:190-217) on its own GPU;
 * round sums all-gathered over `comm` (NCCL / shared memory), the early boundary, tail
 * rounds redundant on every rank. Every rank returns the single-machine proof bytes. */
int dgkr_dist_sumcheck_comm(dgkr_ctx* ctx, dgkr_comm* comm, const dgkr_field* f, size_t n_pairs, size_t local_vars,
                            const uint8_t* local_tables, dgkr_transcript* t, uint8_t* proof, size_t cap, size_t* len);
/* the same with `world` ranks as host threads on lanes of one GPU (full tables in) */
int dgkr_dist_sumcheck_emulated(dgkr_ctx* ctx, const dgkr_field* f, int world, size_t n_pairs, size_t vars,
                                const uint8_t* tables, dgkr_transcript* t, uint8_t* proof, size_t cap, size_t* len);
/* DistPc commit + open (cluster.hpp:336-412): K roots (32 B each), cluster
 * openings as u32 len || Opening::to_bytes, combined value, and traffic json
 * (phases "commit", "open"). n_clusters = 0 selects ClusterTopology::plan's
 * automatic K. */
int dgkr_distpc(dgkr_ctx* ctx, const dgkr_field* f, size_t n_workers, size_t n_clusters, size_t row_vars,
                const uint8_t* rows, const uint8_t* r, size_t r_len, size_t spot_checks, uint8_t* roots_out,
                size_t* n_roots, uint8_t* open_out, size_t cap, size_t* open_len, uint8_t* combined_out,
                char* traffic_json, size_t json_cap);
/* The same over several device contexts: cluster c is committed and opened
 * on context c mod n_ctx, every cluster on its own lane (stream + host
 * thread), so the K leaders hash and open concurrently (their transcripts
 * are independent, cluster.hpp:445-449); the open reuses the matrix and the
 * Merkle tree its commit built. Output bytes equal dgkr_distpc's. */
int dgkr_distpc_multi(dgkr_ctx* const* ctxs, size_t n_ctx, const dgkr_field* f, size_t n_workers, size_t n_clusters,
                      size_t row_vars, const uint8_t* rows, const uint8_t* r, size_t r_len, size_t spot_checks,
                      uint8_t* roots_out, size_t* n_roots, uint8_t* open_out, size_t cap, size_t* open_len,
                      uint8_t* combined_out, char* traffic_json, size_t json_cap);

#ifdef __cplusplus
}
#endif

#endif /* DGKR_B200_H */
