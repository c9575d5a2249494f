"""CPU: the pairwise-distinct (grand-product) circuit of distinct_circuit.py
evaluated by the oracle: accepts exactly the distinct lists whose claimed sort
is a strictly ascending permutation (the native check is distinct.hpp:53-68)."""
import random

import pytest

from oracle import dgkr_oracle as O
from paper_2404_10404_b200 import distinct_circuit as D
from paper_2404_10404_b200 import workloads as W

P_ = O.BN254_P


@pytest.fixture(scope="module")
def circ8():
    insz, flat, L = D.build_distinct_circuit(8)
    return insz, flat, L, D.derive_challenges(P_, b"cpu", L.n_constraints)


def _run(circ8, items, srt):
    insz, flat, L, (r, R) = circ8
    inp, copies = D.distinct_witness(P_, L, insz, items, srt, r, R)
    fi, ff = W.replicate(insz, flat, copies)
    outs = O.Circuit.from_flat(fi, *ff).evaluate(O.BN254.elems_from_bytes(inp.tobytes()), P_)[-1]
    return D.accept(P_, outs, copies)


@pytest.mark.parametrize("n", [1, 7, 8, 20])
def test_distinct_lists_accept(circ8, n):
    items = random.Random(n).sample(range(10 ** 6), n)
    assert _run(circ8, items, sorted(items))
    assert O.pairwise_distinct_check(items, sorted(items), P_)


def test_rejections(circ8):
    items = random.Random(5).sample(range(1000), 20)
    dup = items[:-1] + [items[0]]
    assert not _run(circ8, dup, sorted(dup))                    # duplicate: a zero gap
    srt = sorted(items)
    swapped = srt[:]
    swapped[2], swapped[3] = swapped[3], swapped[2]
    assert not _run(circ8, items, swapped)                      # not ascending
    other = srt[:-1] + [srt[-1] + 1]
    assert not _run(circ8, items, other)                        # not a permutation
    with pytest.raises(ValueError):
        D.distinct_witness(P_, circ8[2], circ8[0], items, srt[:-1], 1, circ8[3][1])
