"""GPU: distinct.hpp on the device (dgkr_distinct_*) against the compiled
reference's fixtures and the restatement: AH (incl. empty and large lists),
the pairwise-distinct check, chain_update with its out_of_range error, encoding
errors and the bit-change experiment."""
import json
import os

import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
FIELDS = {"bn254": O.BN254_P, "tiny97": 97, "goldilocks": O.GOLDILOCKS_P}


@pytest.mark.parametrize("case", GOLDEN["distinct"], ids=lambda c: c["field"])
def test_distinct_golden(ctx, case):
    f = P.Field(FIELDS[case["field"]])
    assert P.distinct_ah(ctx, f, case["items"]) == case["ah"]
    assert P.distinct_ah(ctx, f, []) == case["ah_empty"]
    assert P.pairwise_distinct_check(ctx, f, case["perm"], case["sorted"]) == case["check_true"]
    assert P.pairwise_distinct_check(ctx, f, case["items"], sorted(case["items"])) == case["check_dup"]
    assert P.chain_update(ctx, f, case["h0"], case["n_max"], case["items"]) == case["chain"]
    with pytest.raises(P._lib.OutOfRange):
        P.chain_update(ctx, f, case["h0"], max(case["items"]) - 1, case["items"])
    if "bitchange_10000" in case:
        counts, probs = P.bitchange_experiment(ctx, f, 10000)
        assert counts == case["bitchange_10000"]
        assert abs(probs[0] - counts[0] / 10000) < 1e-12


def test_distinct_large_vs_reference(ctx):
    """C4 scale (32,000 validator indexes) and 2^20, against the compiled reference"""
    R = pytest.importorskip("oracle.refbind")
    if not R.available():
        pytest.skip("oracle/_ref not built")
    f = P.Field.bn254()
    fld = O.BN254
    rng = np.random.default_rng(7)
    for n in (32000, 1 << 20):
        items = rng.permutation(np.arange(n, dtype=np.uint64) * 3 + 1)
        vals = [int(x) for x in items]
        b = fld.elems_to_bytes(vals)
        ah = P.distinct_ah(ctx, f, b)
        if n == 32000:
            assert ah == R.distinct_ah(fld, vals)
        else:
            half = P.distinct_ah(ctx, f, fld.elems_to_bytes(vals[: n // 2]))
            rest = P.distinct_ah(ctx, f, fld.elems_to_bytes(vals[n // 2:]))
            assert ah == (half + rest) % fld.p  # AH is additive over concatenation (associativity)
        srt = sorted(vals)
        assert P.pairwise_distinct_check(ctx, f, b, fld.elems_to_bytes(srt))
        srt[n // 3], srt[n // 3 + 1] = srt[n // 3 + 1], srt[n // 3]
        assert not P.pairwise_distinct_check(ctx, f, b, fld.elems_to_bytes(srt))  # same AH, not ascending


def test_distinct_errors(ctx):
    f = P.Field(97)
    with pytest.raises(P._lib.InvalidArgument):
        P.distinct_ah(ctx, f, bytes([97]))  # >= p
    with pytest.raises(P._lib.InvalidArgument):
        P.bitchange_experiment(ctx, f, 9999)
    # small-field bit-change against the restatement (x wraps mod p)
    counts, _ = P.bitchange_experiment(ctx, f, 10000)
    assert counts == O.bitchange_counts(10000, 97)


@pytest.mark.parametrize("k,n_items", [(4, 6), (8, 64), (16, 100)])
def test_ah_circuit_gkr_matches_reference(ctx, k, n_items):
    """§8(f) rank 3: the associative hash as a data-parallel GKR circuit
    (workloads.ah_circuit). Proof bytes equal the compiled reference's
    gkr_prove on the explicit replica, the reference verifier accepts, and the
    copies' outputs sum to distinct::ah of the list."""
    from paper_2404_10404_b200 import workloads as W
    R = pytest.importorskip("oracle.refbind")
    if not R.available():
        pytest.skip("oracle/_ref not built")
    p = O.BN254_P
    f, of = P.Field(p), O.Field(p)
    rng = np.random.default_rng(k)
    items = [int(x) for x in rng.integers(0, 1 << 20, n_items)]
    insz, flat = W.ah_circuit(k)
    inputs, copies = W.ah_inputs(p, items, k)
    dc = P.Circuit(ctx, insz, *flat, n_copies=copies)
    tr = P.Transcript(f, "ah", [k])
    got = P.gkr_prove(ctx, dc, inputs, tr)
    full_in, full_flat = W.replicate(insz, flat, copies)
    circ = O.Circuit.from_flat(full_in, *full_flat)
    ins = of.elems_from_bytes(inputs.tobytes())
    want, _ = R.gkr_prove(of, "ah", [k], circ, ins, flat=full_flat)
    assert got == want
    assert R.gkr_verify(of, "ah", [k], circ, ins, got, flat=full_flat)
    n_out = int.from_bytes(got[:4], "little")
    outs = of.elems_from_bytes(got[4:4 + n_out * of.width])
    assert sum(outs[:copies]) % p == R.distinct_ah(of, items) == P.distinct_ah(ctx, f, items)


def test_distinct_circuit_gkr_matches_reference(ctx):
    """the grand-product distinct circuit proved on the GPU: byte-equal to the
    compiled reference's gkr_prove, reference verifier accepts, outputs pass
    the final product/range check for a distinct list and fail for a duplicate"""
    from paper_2404_10404_b200 import distinct_circuit as DC
    from paper_2404_10404_b200 import workloads as W
    R = pytest.importorskip("oracle.refbind")
    if not R.available():
        pytest.skip("oracle/_ref not built")
    p = O.BN254_P
    f, of = P.Field(p), O.Field(p)
    insz, flat, L = DC.build_distinct_circuit(8)
    r, coeffs = DC.derive_challenges(p, b"gpu", L.n_constraints)
    rng = np.random.default_rng(11)
    for items, ok in ((list(rng.permutation(1 << 20)[:30]), True), ([5, 9, 5, 1, 2, 3, 4, 6, 7, 8], False)):
        items = [int(x) for x in items]
        inputs, copies = DC.distinct_witness(p, L, insz, items, sorted(items), r, coeffs)
        dc = P.Circuit(ctx, insz, *flat, n_copies=copies)
        got = P.gkr_prove(ctx, dc, inputs, P.Transcript(f, "dc"))
        n_out = int.from_bytes(got[:4], "little")
        outs = of.elems_from_bytes(got[4:4 + n_out * of.width])
        assert DC.accept(p, outs, copies) == ok
        full_in, full_flat = W.replicate(insz, flat, copies)
        circ = O.Circuit.from_flat(full_in, *full_flat)
        ins = of.elems_from_bytes(inputs.tobytes())
        want, _ = R.gkr_prove(of, "dc", [], circ, ins, flat=full_flat)
        assert got == want
        assert R.gkr_verify(of, "dc", [], circ, ins, got, flat=full_flat)
