"""GPU: the CUDA prover against the compiled reference's golden fixtures
(tests/golden/golden.json, from tests/golden/make_golden.py)."""
import json
import os

import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
FIELDS = {"bn254": O.BN254_P, "tiny97": 97, "goldilocks": O.GOLDILOCKS_P}


@pytest.mark.parametrize("case", GOLDEN["product_sum"], ids=lambda c: f'{c["field"]}-{len(c["pairs"][0][0])}')
def test_product_sum(ctx, case):
    f = P.Field(FIELDS[case["field"]])
    tr = P.Transcript(f, case["label"], case["pre"])
    assert P.prove_product_sum(ctx, [tuple(x) for x in case["pairs"]], tr).hex() == case["proof"]
    assert tr.state.hex() == case["state"]


@pytest.mark.parametrize("case", GOLDEN["layer_sum"], ids=lambda c: f'{c["field"]}-{c["side"]}')
def test_layer_sum(ctx, case):
    f = P.Field(FIELDS[case["field"]])
    tr = P.Transcript(f, case["label"])
    wires = [O.LayerWire(bool(a), b, c, d, e, g) for a, b, c, d, e, g in case["wires"]]
    proof, _, _ = P.prove_layer_sum(ctx, case["side"], case["tables"], wires, case["claimed"], tr)
    assert proof.hex() == case["proof"]
    assert tr.state.hex() == case["state"]


@pytest.mark.parametrize("case", GOLDEN["gkr"], ids=lambda c: f'{c["field"]}-{c["label"]}-{c["pre"][0]}')
def test_gkr(ctx, case):
    f = P.Field(FIELDS[case["field"]])
    cj = case["circuit"]
    circ = P.Circuit(ctx, cj["input_size"], np.array(cj["layer_gate_start"], np.uint64),
                     np.array(cj["gate_nested_start"], np.uint64), np.array(cj["nested"], np.uint32).reshape(-1, 5),
                     np.array(cj["min_padded"], np.uint64), n_copies=case["n_copies"])
    tr = P.Transcript(f, case["label"], case["pre"])
    assert P.gkr_prove(ctx, circ, case["inputs"], tr).hex() == case["proof"]
    assert tr.state.hex() == case["state"]


@pytest.mark.parametrize("case", GOLDEN["pcs"], ids=lambda c: f'{c["field"]}-{len(c["rows"])}x{len(c["rows"][0])}')
def test_pcs(ctx, case):
    f = P.Field(FIELDS[case["field"]])
    assert P.pcs_commit(ctx, f, case["rows"]).hex() == case["root"]
    tr = P.Transcript(f, case["label"])
    assert P.pcs_open(ctx, f, case["rows"], case["r"], tr, case["q"]).hex() == case["opening"]
    assert tr.state.hex() == case["state"]


@pytest.mark.parametrize("case", GOLDEN["dist_sumcheck"], ids=lambda c: f'N{c["n_workers"]}')
def test_dist_sumcheck(ctx, case):
    f = P.Field(O.BN254_P)
    tr = P.Transcript(f, case["label"])
    proof, js = P.dist_sumcheck(ctx, case["n_workers"], [tuple(x) for x in case["pairs"]], tr)
    assert proof.hex() == case["proof"] and tr.state.hex() == case["state"] and js == case["traffic"]


@pytest.mark.parametrize("case", GOLDEN["distpc"], ids=lambda c: f'N{len(c["rows"])}')
def test_distpc(ctx, case):
    f = P.Field(O.BN254_P)
    roots, ops, comb, js = P.distpc(ctx, f, case["rows"], case["r"], case["q"])
    assert [x.hex() for x in roots] == case["roots"]
    assert [x.hex() for x in ops] == case["openings"]
    assert comb == case["combined"] and js == case["traffic"]
