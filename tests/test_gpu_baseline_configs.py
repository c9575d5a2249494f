"""GPU: BASELINE.json configs checked byte for byte against the compiled
reference (oracle/_ref: the unmodified reference built against oracle/shim).

  * C1 (configs[0]) at FULL scale: a single-worker GKR proof of the 2^12 x 16
    layered circuit plus the "Virgo commitment" SURVEY.md §8(d) defines for
    the reference -- pcs::commit of the input table (M = 1) and pcs::open at
    every input-claim point. Proof bytes, transcript state, root and every
    opening equal the reference's (gkr.hpp:182-244, pcs.hpp:105-254).
  * C2 (configs[1]) in its real SHAPE -- 64 data-parallel copies x 24 layers --
    at reduced width (2^8 and 2^10 gates per copy per layer): the data-parallel
    prover (copies = high variables) against the reference's gkr_prove of the
    materialised 64-copy circuit, and the emulated N = 2 / 4 / 8 rank split.
  * C5 (configs[4]) PCS commit + open at 2^16 .. 2^20 evaluations
    (pcs.hpp:105-254) and DistPc (cluster.hpp:336-412) at N = 8.
The reference runs on the GPU box's host in the test (its CPU time is the
size limit: the 64 x 2^10 x 24 C2 shape takes ~25 s there)."""
import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O
from oracle import refbind as R
from paper_2404_10404_b200 import workloads as W

pytestmark = pytest.mark.gpu

FLD = O.BN254


@pytest.fixture(scope="module", autouse=True)
def _need_reference():
    # the reference is this file's oracle: a missing build is a failure, not a skip
    assert R.available(), "oracle/_ref/libdgkr_ref.so missing (make -C oracle)"


# ---------------------------------------------------------------------------
# C1 at full scale
# ---------------------------------------------------------------------------
C1_LABEL, C1_OPEN = "dgkr.bench.c1", "dgkr.bench.c1.open"


@pytest.fixture(scope="module")
def c1(ctx):
    f = P.Field.bn254()
    insz, flat = W.layered_circuit(20240410, 12, 16)
    circ = P.Circuit(ctx, insz, *flat)
    inputs = W.random_inputs(f.p, insz, 7)
    tr = P.Transcript(f, C1_LABEL)
    proof = P.gkr_prove(ctx, circ, inputs, tr)
    return f, insz, flat, circ, inputs, proof, tr


def test_c1_gkr_proof_equals_reference(c1):
    f, insz, flat, circ, inputs, proof, tr = c1
    assert circ.n_gates == (1 << 12) * 16
    in_vals = FLD.elems_from_bytes(inputs.tobytes())
    want, want_state = R.gkr_prove(FLD, C1_LABEL, [], O.Circuit.from_flat(insz, *flat), in_vals, flat=flat)
    assert proof == want
    assert tr.state == want_state
    assert R.gkr_verify(FLD, C1_LABEL, [], O.Circuit.from_flat(insz, *flat), in_vals, proof, flat=flat)


def test_c1_commitment_and_openings_equal_reference(ctx, c1):
    f, insz, flat, circ, inputs, proof, _ = c1
    in_vals = FLD.elems_from_bytes(inputs.tobytes())
    root = P.pcs_commit(ctx, f, [inputs])
    assert root == R.pcs_commit(FLD, [in_vals])
    ok, claims = P.gkr_input_claims(circ, proof, P.Transcript(f, C1_LABEL))
    assert ok and claims
    n_open = 0
    for terms, value in claims:
        acc = 0
        for point, weight in terms:
            tr = P.Transcript(f, C1_OPEN)
            op = P.pcs_open(ctx, f, [inputs], point, tr)
            want, want_state = R.pcs_open(FLD, C1_OPEN, [], [in_vals], point)
            assert op == want
            assert tr.state == want_state
            assert R.pcs_verify(FLD, C1_OPEN, [], 1, insz, root, point, op)
            v = int.from_bytes(op[4 + len(point) * 32: 4 + (len(point) + 1) * 32], "little")  # Opening.value
            acc = (acc + weight * v) % f.p
            n_open += 1
        assert acc == value  # the committed inputs answer the proof's input claim
    assert n_open >= 2


# ---------------------------------------------------------------------------
# C2 shape (64 copies x 24 layers) at reduced width
# ---------------------------------------------------------------------------
C2_LABEL = "dgkr.c2.shape"
N_COPIES, DEPTH = 64, 24


@pytest.fixture(scope="module", params=[8, 10], ids=["64x2^8x24", "64x2^10x24"])
def c2_shape(request, ctx):
    log_w = request.param
    f = P.Field.bn254()
    insz, flat = W.layered_circuit(20240410 + log_w, log_w, DEPTH)
    circ = P.Circuit(ctx, insz, *flat, n_copies=N_COPIES)
    inputs = W.random_inputs(f.p, insz * N_COPIES, 11 + log_w)
    full_in, full_flat = W.replicate(insz, flat, N_COPIES)
    want, want_state = R.gkr_prove(FLD, C2_LABEL, [], O.Circuit.from_flat(full_in, *full_flat),
                                   FLD.elems_from_bytes(inputs.tobytes()), flat=full_flat)
    return f, insz, flat, circ, inputs, want, want_state


def test_c2_shape_equals_reference(ctx, c2_shape):
    f, insz, flat, circ, inputs, want, want_state = c2_shape
    assert circ.n_gates == N_COPIES * insz * DEPTH
    tr = P.Transcript(f, C2_LABEL)
    assert P.gkr_prove(ctx, circ, inputs, tr) == want
    assert tr.state == want_state


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c2_shape_distributed_equals_reference(ctx, c2_shape, world):
    f, insz, flat, _, inputs, want, want_state = c2_shape
    local = P.Circuit(ctx, insz, *flat, n_copies=N_COPIES // world)
    tr = P.Transcript(f, C2_LABEL)
    assert P.gkr_prove_dist_emulated(ctx, local, world, inputs, tr) == want
    assert tr.state == want_state


def test_c2_shape_stream_equals_reference(ctx, c2_shape):
    # the bench's lane stream (concurrent proofs on one GPU) proves the same bytes
    f, insz, flat, circ, inputs, want, want_state = c2_shape
    trs = [P.Transcript(f, C2_LABEL) for _ in range(4)]
    proofs = P.gkr_prove_batch(ctx, circ, [inputs] * 4, trs)
    assert all(p == want for p in proofs)
    assert all(t.state == want_state for t in trs)


# ---------------------------------------------------------------------------
# C5: PCS commit / open at 2^16 .. 2^20 evaluations, DistPc at N = 8
# ---------------------------------------------------------------------------
PCS_LABEL = "dgkr.c5.open"


@pytest.mark.parametrize("log_n,M", [(16, 1), (18, 2), (20, 1)])
def test_c5_pcs_commit_open_equals_reference(ctx, log_n, M):
    f = P.Field.bn254()
    cols = (1 << log_n) // M
    raw = W.random_inputs(f.p, 1 << log_n, 100 + log_n)
    rows_b = [raw[i * cols * 32:(i + 1) * cols * 32] for i in range(M)]
    rows = [FLD.elems_from_bytes(r.tobytes()) for r in rows_b]
    rng = np.random.default_rng(log_n)
    r = O.random_elements(FLD, log_n, rng)  # row_vars + index_vars (pcs.hpp:215)
    root = P.pcs_commit(ctx, f, rows_b)
    assert root == R.pcs_commit(FLD, rows)
    tr = P.Transcript(f, PCS_LABEL)
    op = P.pcs_open(ctx, f, rows_b, r, tr)
    want, want_state = R.pcs_open(FLD, PCS_LABEL, [], rows, r)
    assert op == want
    assert tr.state == want_state


def test_c5_distpc_n8_equals_reference(ctx):
    f = P.Field.bn254()
    n_workers, row_vars = 8, 15
    raw = W.random_inputs(f.p, n_workers << row_vars, 5)
    rows = [FLD.elems_from_bytes(raw[i * (32 << row_vars):(i + 1) * (32 << row_vars)].tobytes())
            for i in range(n_workers)]
    r = O.random_elements(FLD, row_vars + 3, np.random.default_rng(9))
    roots, ops, comb, js = P.distpc(ctx, f, rows, r)
    w_roots, w_ops, w_comb, w_js = R.distpc(FLD, rows, r)
    assert roots == w_roots and len(roots) == 4  # plan(8) = 4 clusters x 2 members (cluster.hpp:49-55)
    assert ops == w_ops
    assert comb == w_comb
    assert R.traffic_json_equal(js, w_js)


@pytest.mark.parametrize("n_ctx", [2, 3])
def test_c5_distpc_multi_context_equals_reference(ctx, n_ctx):
    """clusters spread over several contexts (dgkr_distpc_multi; cluster c on
    context c mod n_ctx, concurrently): the bytes of the single-context run and
    of the reference"""
    f = P.Field.bn254()
    n_workers, row_vars = 8, 12
    raw = W.random_inputs(f.p, n_workers << row_vars, 6)
    rows = [FLD.elems_from_bytes(raw[i * (32 << row_vars):(i + 1) * (32 << row_vars)].tobytes())
            for i in range(n_workers)]
    r = O.random_elements(FLD, row_vars + 3, np.random.default_rng(10))
    ctxs = [ctx] + [P.Context(0) for _ in range(n_ctx - 1)]
    got = P.distpc(ctxs, f, rows, r)
    want = R.distpc(FLD, rows, r)
    assert got[0] == want[0] and got[1] == want[1] and got[2] == want[2]
    assert R.traffic_json_equal(got[3], want[3])
    assert P.distpc(ctx, f, rows, r, n_clusters=8)[0] == R.distpc(FLD, rows, r, k=8)[0]
