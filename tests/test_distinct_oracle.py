"""CPU: the distinct.hpp restatement (oracle/dgkr_oracle.py) against the
compiled reference's fixtures (tests/golden/golden.json "distinct") and the
value of f_hash(0) on BN254 derived in SURVEY.md §8(c)."""
import json
import os

import pytest

from oracle import dgkr_oracle as O

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
FIELDS = {"bn254": O.BN254_P, "tiny97": 97, "goldilocks": O.GOLDILOCKS_P}


def test_f_hash_zero_bn254():
    assert O.f_hash(0, O.BN254_P) == 1073523316353959767041899164559407182558796233967617010940674283753464237929


@pytest.mark.parametrize("case", GOLDEN["distinct"], ids=lambda c: c["field"])
def test_distinct_restatement(case):
    p = FIELDS[case["field"]]
    assert O.ah(case["items"], p) == case["ah"]
    assert O.ah([], p) == case["ah_empty"] == 0
    assert O.ah(case["perm"], p) == O.ah(case["sorted"], p)  # permutation invariance
    assert O.pairwise_distinct_check(case["perm"], case["sorted"], p) == case["check_true"]
    assert O.pairwise_distinct_check(case["items"], sorted(case["items"]), p) == case["check_dup"]
    assert O.chain_update(case["h0"], case["n_max"], case["items"], p) == case["chain"]
    with pytest.raises(IndexError):
        O.chain_update(case["h0"], min(case["items"]) - 1 if min(case["items"]) else -1, case["items"], p)
    if "bitchange_10000" in case:
        assert O.bitchange_counts(10000, p) == case["bitchange_10000"]


def test_bitchange_minimum_count():
    with pytest.raises(ValueError):
        O.bitchange_counts(9999, 97)
