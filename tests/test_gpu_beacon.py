"""GPU: beacon.hpp on the device (dgkr_beacon_root / _prove / _verify)
against the compiled reference's fixtures (tests/golden "beacon"), incl. the
C3 size (4,096 validators, depth 56), tampering and error cases."""
import json
import os

import numpy as np
import pytest

import paper_2404_10404_b200 as P

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(__file__)
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def records_of(case) -> bytes:
    if "records" in case:
        return bytes.fromhex(case["records"])
    return open(os.path.join(HERE, "golden", case["records_file"]), "rb").read()


@pytest.mark.parametrize("case", GOLDEN["beacon"], ids=lambda c: f'{c["n"]}-{c["depth"]}')
def test_beacon_golden(ctx, case):
    recs, depth, n = records_of(case), case["depth"], case["n"]
    root = P.beacon_root(ctx, recs, depth)
    assert root.hex() == case["root"]
    idx = [p["index"] for p in case["paths"]]
    leaves, sib, a = P.beacon_prove(ctx, recs, depth, idx)
    for k, p in enumerate(case["paths"]):
        assert a == p["active_log2"]
        assert leaves[32 * k:32 * (k + 1)].hex() == p["leaf"]
        assert sib[32 * a * k:32 * a * (k + 1)].hex() == p["siblings"]
    # every validator's path verifies; tampering fails per path only
    all_idx = np.arange(n, dtype=np.uint64)
    L, S, a = P.beacon_prove(ctx, recs, depth, all_idx)
    ok = P.beacon_verify(ctx, root, recs, L, S, all_idx, depth, a)
    assert ok.all()
    if n > 1 and a > 0:
        S2 = bytearray(S)
        S2[32 * a * 1 + 5] ^= 0x40  # path 1, first sibling
        recs2 = bytearray(recs)
        recs2[64 * 0 + 3] ^= 1      # record 0
        bad_idx = all_idx.copy()
        bad_idx[n - 1] = bad_idx[n - 1] | (np.uint64(1) << np.uint64(a))  # outside the active region
        ok2 = P.beacon_verify(ctx, root, bytes(recs2), L, bytes(S2), bad_idx, depth, a)
        want = np.ones(n, dtype=np.uint8)
        want[[0, 1, n - 1]] = 0
        assert np.array_equal(ok2, want)
        root2 = bytearray(root)
        root2[0] ^= 1
        assert not P.beacon_verify(ctx, bytes(root2), recs, L, S, all_idx, depth, a).any()


def test_beacon_errors(ctx):
    recs = records_of(GOLDEN["beacon"][2])  # 37 validators
    with pytest.raises(P._lib.InvalidArgument):
        P.beacon_root(ctx, recs, 5)  # 2^6 > 2^5: exceeds capacity
    with pytest.raises(P._lib.OutOfRange):
        P.beacon_prove(ctx, recs, 12, [37])
    from oracle import dgkr_oracle as O
    assert P.beacon_root(ctx, b"", 3) == O.beacon_root(b"", 3)  # empty set: the zero-cache spine
