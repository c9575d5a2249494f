"""CPU: the beacon.hpp restatement (oracle/dgkr_oracle.py) against the
compiled reference's fixtures (tests/golden/golden.json "beacon")."""
import json
import os

import pytest

from oracle import dgkr_oracle as O

HERE = os.path.dirname(__file__)
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def records_of(case) -> bytes:
    if "records" in case:
        return bytes.fromhex(case["records"])
    return open(os.path.join(HERE, "golden", case["records_file"]), "rb").read()


@pytest.mark.parametrize("case", GOLDEN["beacon"], ids=lambda c: f'{c["n"]}-{c["depth"]}')
def test_beacon_restatement(case):
    recs = records_of(case)
    if case["n"] <= 64:
        assert O.beacon_root(recs, case["depth"]).hex() == case["root"]
    root = bytes.fromhex(case["root"])
    for p in case["paths"]:
        sib = bytes.fromhex(p["siblings"])
        sibs = [sib[32 * k:32 * (k + 1)] for k in range(p["active_log2"])]
        rec = recs[64 * p["index"]:64 * (p["index"] + 1)]
        assert O.beacon_verify(root, rec, bytes.fromhex(p["leaf"]), sibs, p["index"], case["depth"])
        other = recs[64 * ((p["index"] + 1) % case["n"]):64 * ((p["index"] + 1) % case["n"] + 1)]
        if case["n"] > 1:
            assert not O.beacon_verify(root, other, bytes.fromhex(p["leaf"]), sibs, p["index"], case["depth"])
