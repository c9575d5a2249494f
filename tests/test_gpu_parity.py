"""GPU parity: the CUDA prover (through the C ABI) against the CPU oracle.

Bit-exact is the bar for every comparison (integer / byte work): proof
bytes, transcript state and draw counter, Merkle roots, openings and
TrafficStats json. Small cases compare with the pure-Python restatement
(oracle/dgkr_oracle.py); medium and full-scale cases with the compiled
reference (oracle/_ref, when present) and with size-independent properties.
"""
import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O
from paper_2404_10404_b200 import workloads as W
from paper_2404_10404_b200._lib import InvalidArgument

pytestmark = pytest.mark.gpu

FIELDS = [O.BN254_P, 97, O.GOLDILOCKS_P]


def _pairs(of, n_pairs, vars_, rng):
    return [(O.random_elements(of, 1 << vars_, rng), O.random_elements(of, 1 << vars_, rng)) for _ in range(n_pairs)]


@pytest.mark.parametrize("p", FIELDS)
@pytest.mark.parametrize("vars_,n_pairs", [(0, 1), (1, 1), (2, 2), (5, 3), (8, 2), (11, 1)])
def test_product_sum_matches_oracle(ctx, p, vars_, n_pairs):
    rng = np.random.default_rng(1000 * vars_ + n_pairs + p % 1000)
    f, of = P.Field(p), O.Field(p)
    pairs = _pairs(of, n_pairs, vars_, rng)
    tr = P.Transcript(f, "test.sumcheck", [3])
    got = P.prove_product_sum(ctx, pairs, tr)
    otr = O.Transcript("test.sumcheck", of, [3])
    want = O.prove_product_sum(pairs, otr).to_bytes(of)
    assert got == want
    assert tr.state == otr.state and tr.draws == otr.draws


def test_product_sum_kat_one_variable(ctx):
    # tests/test_sumcheck.cpp:76-86: [1,2].[3,4] -> claimed 11
    f = P.Field(97)
    tr = P.Transcript(f, "test.sumcheck", [0])
    proof = P.prove_product_sum(ctx, [([1, 2], [3, 4])], tr)
    assert proof[0] == 11


def test_product_sum_zero_tables(ctx):
    # tests/test_sumcheck.cpp:66-74
    f, of = P.Field(97), O.Field(97)
    pairs = [([0] * 8, [0] * 8)]
    tr = P.Transcript(f, "test.sumcheck", [0])
    got = P.prove_product_sum(ctx, pairs, tr)
    otr = O.Transcript("test.sumcheck", of, [0])
    assert got == O.prove_product_sum(pairs, otr).to_bytes(of)
    assert got[0] == 0


def test_product_sum_errors(ctx):
    f = P.Field(97)
    tr = P.Transcript(f, "t")
    with pytest.raises(InvalidArgument):  # sumcheck.hpp:161-163 mixed table sizes
        P.prove_product_sum(ctx, [([1, 2], [3, 4]), ([1, 2, 3, 4], [1, 2, 3, 4])], tr)
    with pytest.raises(InvalidArgument):  # field.hpp:183-185 non-canonical
        P.prove_product_sum(ctx, [(bytes([97, 1]), bytes([1, 1]))], tr)


@pytest.mark.parametrize("p", [O.BN254_P, 97])
@pytest.mark.parametrize("n_workers", [1, 2, 4, 8])
def test_dist_sumcheck_matches_oracle(ctx, p, n_workers):
    rng = np.random.default_rng(n_workers + p % 7)
    f, of = P.Field(p), O.Field(p)
    pairs = _pairs(of, 2, 5, rng)
    tr = P.Transcript(f, "dgkr.bench")
    proof, js = P.dist_sumcheck(ctx, n_workers, pairs, tr)
    otr = O.Transcript("dgkr.bench", of)
    ts = O.TrafficStats()
    ts.begin_phase("sumcheck")
    want = O.dist_sumcheck(n_workers, pairs, otr, ts).to_bytes(of)
    assert proof == want and tr.state == otr.state
    assert js == ts.to_json()


def _random_layer(of, rng, side, n_slots, n_wires):
    T = 1 << side
    tables = [O.random_elements(of, T, rng) for _ in range(n_slots)]
    wires = [O.LayerWire(bool(rng.integers(2)), O.random_elements(of, 1, rng)[0], int(rng.integers(n_slots)),
                         int(rng.integers(n_slots)), int(rng.integers(T)), int(rng.integers(T)))
             for _ in range(n_wires)]
    claimed = sum(w.weight * (tables[w.x_slot][w.x_index] * tables[w.y_slot][w.y_index] if w.is_mul else
                              tables[w.x_slot][w.x_index] + tables[w.y_slot][w.y_index]) for w in wires) % of.p
    return tables, wires, claimed


@pytest.mark.parametrize("p", FIELDS)
@pytest.mark.parametrize("side,n_slots,n_wires", [(0, 1, 1), (2, 1, 16), (3, 2, 20), (6, 3, 200)])
def test_layer_sum_matches_oracle(ctx, p, side, n_slots, n_wires):
    rng = np.random.default_rng(side * 100 + n_slots)
    f, of = P.Field(p), O.Field(p)
    tables, wires, claimed = _random_layer(of, rng, side, n_slots, n_wires)
    tr = P.Transcript(f, "test.layer")
    got, xp, yp = P.prove_layer_sum(ctx, side, tables, wires, claimed, tr)
    otr = O.Transcript("test.layer", of)
    proof, u, v = O.prove_layer_sum(side, tables, wires, claimed, otr)
    assert got == proof.to_bytes(of)
    assert xp == u and yp == v and tr.state == otr.state


def _gkr_both(ctx, p, circ: O.Circuit, inputs, label="test.gkr", pre=(0,)):
    f, of = P.Field(p), O.Field(p)
    dc = P.Circuit.from_oracle(ctx, circ)
    tr = P.Transcript(f, label, pre)
    got = P.gkr_prove(ctx, dc, inputs, tr)
    otr = O.Transcript(label, of, pre)
    outs, layers = O.gkr_prove(circ, inputs, otr)
    want = O.gkr_proof_bytes(of, outs, layers)
    return got, want, tr, otr


def test_gkr_acc4_example(ctx):
    # tests/test_gkr.cpp:17-24, :61-73: one accumulation gate adding 4 inputs -> 10
    circ = O.Circuit(4, [[[(O.ADD, (0, 0), (0, 1)), (O.ADD, (0, 2), (0, 3))]]])
    got, want, tr, otr = _gkr_both(ctx, 97, circ, [1, 2, 3, 4])
    assert got == want and tr.state == otr.state
    assert got[4] == 10  # claimed output


def test_gkr_empty_circuit(ctx):
    # tests/test_gkr.cpp:128-140: no layers, claims land on the inputs
    circ = O.Circuit(4, [])
    got, want, tr, otr = _gkr_both(ctx, 97, circ, [9, 8, 7, 6])
    assert got == want and tr.state == otr.state


def _py_random_general_circuit(rng, input_size, depth, max_gates, max_nested, mul_percent=50):
    """Same shape as circuit::random_general_circuit (circuit.hpp:342-381) with
    a numpy generator: accumulation gates, wires into any earlier layer."""
    sizes = [input_size]
    layers = []
    for li in range(1, depth + 1):
        n_gates = 1 + int(rng.integers(max_gates))
        layer = []
        reads_prev = False
        for _ in range(n_gates):
            g = []
            for _ in range(1 + int(rng.integers(max_nested))):
                kind = O.MUL if rng.integers(100) < mul_percent else O.ADD
                ll, rl = int(rng.integers(li)), int(rng.integers(li))
                g.append((kind, (ll, int(rng.integers(sizes[ll]))), (rl, int(rng.integers(sizes[rl])))))
                reads_prev |= ll + 1 == li or rl + 1 == li
            layer.append(g)
        if not reads_prev:
            k, _l, r = layer[0][0]
            layer[0][0] = (k, (li - 1, int(rng.integers(sizes[li - 1]))), r)
        sizes.append(len(layer))
        layers.append(layer)
    return O.Circuit(input_size, layers)


@pytest.mark.parametrize("p", FIELDS)
@pytest.mark.parametrize("trial", range(6))
def test_gkr_general_circuits_match_oracle(ctx, p, trial):
    rng = np.random.default_rng(trial * 31 + p % 101)
    of = O.Field(p)
    insz = 4 + trial
    circ = _py_random_general_circuit(rng, insz, 2 + trial % 4, 12, 3)
    inputs = O.random_elements(of, insz, rng)
    got, want, tr, otr = _gkr_both(ctx, p, circ, inputs, pre=(trial,))
    assert got == want and tr.state == otr.state and tr.draws == otr.draws


@pytest.mark.parametrize("seed", [1, 4, 10, 18, 21, 25, 40, 77])
def test_gkr_reference_generated_wide_consumers(ctx, seed):
    """Reference-generated circuits (circuit::random_general_circuit) whose
    consumer layers have more gates than their source tables (regression:
    the per-gate weight buffer was sized by the source tables)."""
    from oracle import refbind as R

    if not R.available():
        pytest.skip("oracle/_ref not built")
    fld = O.BN254
    insz, depth = 5 + seed % 8, 2 + seed % 4
    c = R.random_general_circuit(1000 + seed, insz, depth, 24, 3)
    inputs = O.random_elements(fld, insz, np.random.default_rng(seed))
    want, st = R.gkr_prove(fld, "h", [seed], c, inputs)
    tr = P.Transcript(P.Field(fld.p), "h", [seed])
    assert P.gkr_prove(ctx, P.Circuit.from_oracle(ctx, c), inputs, tr) == want
    assert tr.state == st


def test_gkr_layered_matches_oracle(ctx):
    insz, flat = W.layered_circuit(seed=5, log_width=6, depth=5)
    circ = O.Circuit.from_flat(insz, *flat)
    inputs = O.Field(O.BN254_P).elems_from_bytes(W.random_inputs(O.BN254_P, insz, 6).tobytes())
    got, want, tr, otr = _gkr_both(ctx, O.BN254_P, circ, inputs)
    assert got == want and tr.state == otr.state


@pytest.mark.parametrize("n_copies", [2, 4, 8])
def test_gkr_data_parallel_matches_replicated_oracle(ctx, n_copies):
    """dgkr_circuit_create(..., n_copies): copy index = high variables
    (cluster.hpp:182-189) — must equal gkr_prove on the explicit replica."""
    p = O.BN254_P
    f, of = P.Field(p), O.Field(p)
    insz, flat = W.layered_circuit(seed=11, log_width=4, depth=4)
    full_in, full_flat = W.replicate(insz, flat, n_copies)
    inputs = W.random_inputs(p, full_in, 12)
    dc = P.Circuit(ctx, insz, *flat, n_copies=n_copies)
    tr = P.Transcript(f, "dp", [1])
    got = P.gkr_prove(ctx, dc, inputs, tr)
    circ = O.Circuit.from_flat(full_in, *full_flat)
    otr = O.Transcript("dp", of, [1])
    outs, layers = O.gkr_prove(circ, of.elems_from_bytes(inputs.tobytes()), otr)
    assert got == O.gkr_proof_bytes(of, outs, layers)
    assert tr.state == otr.state


@pytest.mark.parametrize("n", [1, 3])
def test_gkr_batch_equals_single_proofs(ctx, n):
    """dgkr_gkr_prove_batch runs n proofs concurrently on n lanes; each must be
    byte-identical to the oracle's proof of the same instance."""
    p = O.BN254_P
    f, of = P.Field(p), O.Field(p)
    insz, flat = W.layered_circuit(seed=21, log_width=5, depth=4)
    dc = P.Circuit(ctx, insz, *flat, n_copies=2)
    full_in, full_flat = W.replicate(insz, flat, 2)
    circ = O.Circuit.from_flat(full_in, *full_flat)
    inputs = [W.random_inputs(p, full_in, 100 + i) for i in range(n)]
    trs = [P.Transcript(f, "batch", [i]) for i in range(n)]
    got = P.gkr_prove_batch(ctx, dc, inputs, trs)
    for i in range(n):
        otr = O.Transcript("batch", of, [i])
        outs, layers = O.gkr_prove(circ, of.elems_from_bytes(inputs[i].tobytes()), otr)
        assert got[i] == O.gkr_proof_bytes(of, outs, layers)
        assert trs[i].state == otr.state
    # resident inputs per lane
    for i in range(n):
        P.load_inputs_lane(ctx, dc, f, i, inputs[i])
    trs2 = [P.Transcript(f, "batch", [i]) for i in range(n)]
    assert P.gkr_prove_batch(ctx, dc, None, trs2) == got


def test_circuit_validation_errors(ctx):
    # circuit.hpp:103-152 violations surface as invalid_argument
    bad = O.Circuit(2, [[[(O.ADD, (1, 0), (0, 0))]]])  # non-causal
    with pytest.raises(InvalidArgument, match="non-causal"):
        P.Circuit.from_oracle(ctx, bad)
    bad = O.Circuit(2, [[[(O.ADD, (0, 9), (0, 0))]]])  # dangling
    with pytest.raises(InvalidArgument, match="dangling"):
        P.Circuit.from_oracle(ctx, bad)


@pytest.mark.parametrize("p", [O.BN254_P, 97])
@pytest.mark.parametrize("M,cols,q", [(1, 1, 32), (1, 8, 32), (2, 8, 4), (4, 16, 5), (2, 64, 32), (1, 1024, 32)])
def test_pcs_commit_open_match_oracle(ctx, p, M, cols, q):
    rng = np.random.default_rng(M * 1000 + cols)
    f, of = P.Field(p), O.Field(p)
    rows = [O.random_elements(of, cols, rng) for _ in range(M)]
    assert P.pcs_commit(ctx, f, rows) == O.pcs_commit(of, rows)
    r = O.random_elements(of, O.log2_exact(cols) + O.log2_exact(M), rng)
    tr = P.Transcript(f, "test.pcs")
    got = P.pcs_open(ctx, f, rows, r, tr, q)
    otr = O.Transcript("test.pcs", of)
    assert got == O.pcs_open(of, rows, r, otr, q)
    assert tr.state == otr.state


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_distpc_matches_oracle(ctx, N):
    p = O.BN254_P
    rng = np.random.default_rng(N)
    f, of = P.Field(p), O.Field(p)
    rows = [O.random_elements(of, 16, rng) for _ in range(N)]
    r = O.random_elements(of, 4 + O.log2_exact(N), rng)
    roots, ops, comb, js = P.distpc(ctx, f, rows, r, 4)
    ts = O.TrafficStats()
    roots2, ops2, comb2 = O.distpc(of, rows, r, 4, ts)
    assert roots == roots2 and ops == ops2 and comb == comb2
    assert js == ts.to_json()


@pytest.mark.parametrize("n_copies", [1, 4])
@pytest.mark.parametrize("multi_slot", [False, True])
def test_gkr_heavy_rows(ctx, n_copies, multi_slot):
    """CSR rows with more than 64 entries (constant wires / padding gates)
    take the CTA-per-row bookkeeping path; proofs must not change."""
    p = O.BN254_P
    f, of = P.Field(p), O.Field(p)
    rng = np.random.default_rng(31 + n_copies + 2 * multi_slot)
    w, insz = 256, 256
    layers = []
    for li in range(1, 4):
        gates = []
        for g in range(w):
            src = li - 1
            if g < 192:      # heavy x row: input 0 of the previous layer
                ng = [(int(rng.integers(0, 2)), src, 0, src, int(rng.integers(0, w)))]
            elif g < 224:    # heavy y row: gate 7 of the previous layer
                ng = [(int(rng.integers(0, 2)), src, int(rng.integers(0, w)), src, 7)]
            else:
                ng = [(int(rng.integers(0, 2)), src, int(rng.integers(0, w)), src, int(rng.integers(0, w)))]
            if multi_slot and li >= 2:  # second slot: the input layer, also heavy on x
                ng.append((int(rng.integers(0, 2)), 0, 3, li - 1, int(rng.integers(0, w))))
            gates.append(ng)
        layers.append(gates)
    lgs, gns, rows = [0], [0], []
    for gl in layers:
        for g in gl:
            rows.extend(g)
            gns.append(gns[-1] + len(g))
        lgs.append(lgs[-1] + len(gl))
    flat = (np.array(lgs, np.uint64), np.array(gns, np.uint64), np.array(rows, np.uint32).reshape(-1, 5),
            np.ones(len(layers) + 1, np.uint64))
    dc = P.Circuit(ctx, insz, *flat, n_copies=n_copies)
    full_in, full_flat = W.replicate(insz, flat, n_copies)
    inputs = W.random_inputs(p, full_in, 77)
    tr = P.Transcript(f, "heavy", [n_copies])
    got = P.gkr_prove(ctx, dc, inputs, tr)
    circ = O.Circuit.from_flat(full_in, *full_flat)
    otr = O.Transcript("heavy", of, [n_copies])
    outs, lay = O.gkr_prove(circ, of.elems_from_bytes(inputs.tobytes()), otr)
    assert got == O.gkr_proof_bytes(of, outs, lay)
    assert tr.state == otr.state


def test_runtime_moduli_alternate_across_contexts():
    """Two contexts on one device, each proving over its own runtime modulus,
    interleaved: the device's constant block is shared, so the upload cache
    must be per device (a per-context cache proved p=97 with
    Goldilocks constants after the other context had loaded them)."""
    ctx_a, ctx_b = P.Context(0), P.Context(0)
    fa, fb = P.Field(97), P.Field(O.GOLDILOCKS_P)
    oa, ob = O.Field(97), O.Field(O.GOLDILOCKS_P)
    rng = np.random.default_rng(77)
    pa, pb = _pairs(oa, 2, 6, rng), _pairs(ob, 2, 6, rng)
    for _ in range(3):
        for ctx, f, of, pairs in ((ctx_a, fa, oa, pa), (ctx_b, fb, ob, pb)):
            tr = P.Transcript(f, "alt", [1])
            otr = O.Transcript("alt", of, [1])
            assert P.prove_product_sum(ctx, pairs, tr) == O.prove_product_sum(pairs, otr).to_bytes(of)
            assert tr.state == otr.state


def test_pcs_rejects_ragged_rows(ctx):
    f = P.Field.bn254()
    a = W.random_inputs(f.p, 8, 1)
    b = W.random_inputs(f.p, 4, 2)
    with pytest.raises(InvalidArgument):
        P.pcs_commit(ctx, f, [a, b])
    with pytest.raises(InvalidArgument):
        P.pcs_commit(ctx, f, [a[:-1]])
    with pytest.raises(InvalidArgument):
        P.pcs_open(ctx, f, [a, b], [1, 2], P.Transcript(f, "x"))


@pytest.mark.parametrize("p", FIELDS)
@pytest.mark.parametrize("vars_,n_pairs", [(0, 1), (1, 2), (4, 1), (9, 3)])
def test_pairsum_session_steps_match_oracle(ctx, p, vars_, n_pairs):
    """dgkr_pairsum_* (PairSumSession, sumcheck.hpp:152-221) driven step by
    step reproduces prove_product_sum's transcript and proof bytes."""
    import ctypes as C

    from paper_2404_10404_b200._lib import LogicError, check, lib

    rng = np.random.default_rng(7000 + vars_ + 10 * n_pairs + p % 97)
    f, of = P.Field(p), O.Field(p)
    pairs = _pairs(of, n_pairs, vars_, rng)
    tabs = b"".join(f.encode(x) for pr in pairs for x in pr)
    h = C.c_void_p()
    check(lib().dgkr_pairsum_begin(ctx.handle, f.handle, C.c_size_t(n_pairs), C.c_size_t(vars_), tabs, C.byref(h)))
    try:
        w = f.width
        tr = P.Transcript(f, "sess", [1])
        buf = C.create_string_buffer(4 * w)
        check(lib().dgkr_pairsum_total(h, buf))
        out = buf.raw[:w]
        tr.absorb_bytes(buf.raw[:w])
        lib().dgkr_pairsum_vars_left.restype = C.c_size_t
        assert lib().dgkr_pairsum_vars_left(h) == vars_
        for _ in range(vars_):
            check(lib().dgkr_pairsum_round(h, buf))
            rp = buf.raw[:4 * w]
            for k in range(4):
                tr.absorb_bytes(rp[k * w:(k + 1) * w])
            out += rp
            r = tr.challenge()
            check(lib().dgkr_pairsum_fold(h, f.encode([r])))
        fin = C.create_string_buffer(2 * n_pairs * w)
        check(lib().dgkr_pairsum_finals(h, fin))
        with pytest.raises(LogicError):
            check(lib().dgkr_pairsum_round(h, buf))
    finally:
        lib().dgkr_pairsum_end(h)
    otr = O.Transcript("sess", of, [1])
    want = O.prove_product_sum(pairs, otr).to_bytes(of)
    n = len(want)
    # SumcheckProof bytes = claimed || u32 rounds || 4w per round || u32 finals || finals (sumcheck.hpp:51-61)
    got = out[:w] + vars_.to_bytes(4, "little") + out[w:] + (2 * n_pairs).to_bytes(4, "little") + fin.raw
    assert got == want and len(got) == n
    assert tr.state == otr.state
