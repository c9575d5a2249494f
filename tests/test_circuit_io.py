"""CPU: circuit interchange. The JSON mapping (paper_2404_10404_b200.circuit_io)
against the reference's own GeneralCircuit::to_json / from_json (compiled
reference, oracle/_ref), on reference-generated random circuits and the
workload circuits."""
import json

import numpy as np
import pytest

from oracle import dgkr_oracle as O
from oracle import refbind as R
from paper_2404_10404_b200 import circuit_io as IO
from paper_2404_10404_b200 import workloads as W

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def _same_flat(a, b):
    return all(np.array_equal(np.asarray(x).astype(np.uint64), np.asarray(y).astype(np.uint64)) for x, y in zip(a[:3], b[:3]))


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_json_matches_reference(seed):
    c = R.random_general_circuit(seed, input_size=5, depth=4, max_gates=7, max_nested=3)
    flat = c.to_flat()
    ref = json.loads(R.circuit_json(c, flat))
    ours = IO.to_json(c.input_size, flat)
    assert ours == ref  # same structure and key order semantics
    assert list(ours.keys()) == list(ref.keys()) == ["input_size", "layers"]
    insz, back = IO.from_json(json.dumps(ref))
    assert insz == c.input_size and _same_flat(back, flat)


def test_json_workloads_round_trip():
    for insz, flat in (W.layered_circuit(5, 4, 3), W.ah_circuit(4)):
        c = O.Circuit.from_flat(insz, *flat)
        ref = json.loads(R.circuit_json(c, flat))
        assert IO.to_json(insz, flat) == ref
        i2, f2 = IO.from_json(ref)
        assert i2 == insz and _same_flat(f2, flat)


def test_json_unknown_op():
    bad = {"input_size": 2, "layers": [[{"nested": [{"op": "xor", "left": [0, 0], "right": [0, 1]}]}]]}
    with pytest.raises(ValueError, match="unknown gate op"):
        IO.from_json(bad)
