"""GPU: moduli of 255 and 256 bits (2^255 - 19 and secp256k1's p). The
reference accepts any prime (field.hpp:26-40); the device's default runtime
path needs p < 2^254 (lazy differences, 4p < 2^256), so these run on the wide
policy (RtW: carry-aware adds, fully reduced differences, 10-limb products).
Proofs, transcripts, roots and openings against the Python oracle and the
compiled reference, byte for byte."""
import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O
from oracle import refbind as R
from paper_2404_10404_b200 import workloads as W
from paper_2404_10404_b200._lib import DgkrError

pytestmark = pytest.mark.gpu
WIDE = [2**255 - 19, 2**256 - 2**32 - 977]


def _pairs(of, n_pairs, vars_, rng):
    return [(O.random_elements(of, 1 << vars_, rng), O.random_elements(of, 1 << vars_, rng)) for _ in range(n_pairs)]


@pytest.mark.parametrize("p", WIDE)
@pytest.mark.parametrize("vars_,n_pairs", [(0, 1), (3, 2), (9, 1), (12, 2)])
def test_wide_product_sum(ctx, p, vars_, n_pairs):
    rng = np.random.default_rng(vars_ + 7 * n_pairs)
    f, of = P.Field(p), O.Field(p)
    pairs = _pairs(of, n_pairs, vars_, rng)
    pairs[0][0][0] = p - 1  # extremes: sums that carry out of 256 bits
    pairs[0][1][0] = p - 1
    tr = P.Transcript(f, "wide.sc", [1])
    got = P.prove_product_sum(ctx, pairs, tr)
    otr = O.Transcript("wide.sc", of, [1])
    assert got == O.prove_product_sum(pairs, otr).to_bytes(of)
    assert tr.state == otr.state


@pytest.mark.parametrize("p", WIDE)
@pytest.mark.parametrize("copies", [1, 4])
def test_wide_gkr_equals_reference(ctx, p, copies):
    assert R.available()
    f, of = P.Field(p), O.Field(p)
    insz, flat = W.layered_circuit(777, 7, 4)
    inputs = W.random_inputs(p, insz * copies, 3)
    circ = P.Circuit(ctx, insz, *flat, n_copies=copies)
    tr = P.Transcript(f, "wide.gkr")
    proof = P.gkr_prove(ctx, circ, inputs, tr)
    full_in, full_flat = W.replicate(insz, flat, copies) if copies > 1 else (insz, flat)
    want, want_state = R.gkr_prove(of, "wide.gkr", [], O.Circuit.from_flat(full_in, *full_flat),
                                   of.elems_from_bytes(inputs.tobytes()), flat=full_flat)
    assert proof == want and tr.state == want_state
    assert P.gkr_verify(circ, proof, P.Transcript(f, "wide.gkr"), inputs=inputs)


@pytest.mark.parametrize("p", WIDE)
def test_wide_pcs_equals_reference(ctx, p):
    f, of = P.Field(p), O.Field(p)
    rows = [O.random_elements(of, 1 << 10, np.random.default_rng(k)) for k in range(2)]
    r = O.random_elements(of, 11, np.random.default_rng(5))
    assert P.pcs_commit(ctx, f, rows) == R.pcs_commit(of, rows)
    tr = P.Transcript(f, "wide.pcs")
    op = P.pcs_open(ctx, f, rows, r, tr)
    want, st = R.pcs_open(of, "wide.pcs", [], rows, r)
    assert op == want and tr.state == st


@pytest.mark.parametrize("p", WIDE)
@pytest.mark.parametrize("world", [2, 8])
def test_wide_distributed(ctx, p, world):
    f, of = P.Field(p), O.Field(p)
    pairs = _pairs(of, 2, 8, np.random.default_rng(world))
    t1 = P.Transcript(f, "wide.dist")
    single = P.prove_product_sum(ctx, pairs, t1)
    t2 = P.Transcript(f, "wide.dist")
    assert P.prover.dist_sumcheck_emulated(ctx, world, pairs, t2) == single and t2.state == t1.state
    insz, flat = W.layered_circuit(31, 6, 3)
    inputs = W.random_inputs(p, insz * 8, 4)
    t3 = P.Transcript(f, "wide.gd")
    want = P.gkr_prove(ctx, P.Circuit(ctx, insz, *flat, n_copies=8), inputs, t3)
    t4 = P.Transcript(f, "wide.gd")
    local = P.Circuit(ctx, insz, *flat, n_copies=8 // world)
    assert P.gkr_prove_dist_emulated(ctx, local, world, inputs, t4) == want and t4.state == t3.state


@pytest.mark.parametrize("p", WIDE)
def test_wide_ntt_roundtrip(ctx, p):
    f, of = P.Field(p), O.Field(p)
    x = O.random_elements(of, 16, np.random.default_rng(1))
    try:
        y = P.ntt(ctx, f, x)
    except DgkrError:
        pytest.skip("domain larger than the field's 2-adic subgroup")
    assert P.ntt(ctx, f, y, inverse=True) == x
