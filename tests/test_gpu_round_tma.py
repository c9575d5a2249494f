"""GPU: the TMA-staged round kernel (csrc/round_tma.cuh) against the register-
fed k_round and the compiled reference. The kernel takes the large rounds of
every GKR layer sum-check (np = 1 pair + G); forcing its threshold down to
256 output pairs runs it on every round shape -- round 1 scan (wide sums),
round 2 natural->bit-reversed fold, rounds >= 3 bit-reversed folds -- at
sizes the reference proves in seconds. Bit-exact is the bar."""
import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O
from oracle import refbind as R
from paper_2404_10404_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture
def tma_everywhere():
    old = P.get_tuning("tma_min_pairs")
    P.set_tuning("tma_min_pairs", 256)
    yield
    P.set_tuning("tma_min_pairs", old)


def _prove(ctx, f, insz, flat, copies, inputs, label, tma):
    old = P.get_tuning("tma_min_pairs")
    P.set_tuning("tma_min_pairs", 256 if tma else 0)
    try:
        circ = P.Circuit(ctx, insz, *flat, n_copies=copies)
        tr = P.Transcript(f, label)
        return P.gkr_prove(ctx, circ, inputs, tr), tr.state
    finally:
        P.set_tuning("tma_min_pairs", old)


@pytest.mark.parametrize("p", [O.BN254_P, O.GOLDILOCKS_P, 97])
@pytest.mark.parametrize("log_w,copies,depth", [(8, 1, 3), (9, 4, 3), (10, 16, 2), (12, 2, 2)])
def test_tma_round_equals_register_round(ctx, p, log_w, copies, depth):
    f = P.Field(p)
    insz, flat = W.layered_circuit(300 + log_w, log_w, depth)
    inputs = W.random_inputs(f.p, insz * copies, log_w + copies)
    a = _prove(ctx, f, insz, flat, copies, inputs, "tma.ab", True)
    b = _prove(ctx, f, insz, flat, copies, inputs, "tma.ab", False)
    assert a == b


def test_tma_round_equals_reference(ctx, tma_everywhere):
    assert R.available()
    f = P.Field.bn254()
    insz, flat = W.layered_circuit(4242, 9, 4)
    copies = 8
    inputs = W.random_inputs(f.p, insz * copies, 5)
    circ = P.Circuit(ctx, insz, *flat, n_copies=copies)
    tr = P.Transcript(f, "tma.ref")
    proof = P.gkr_prove(ctx, circ, inputs, tr)
    full_in, full_flat = W.replicate(insz, flat, copies)
    want, want_state = R.gkr_prove(O.BN254, "tma.ref", [], O.Circuit.from_flat(full_in, *full_flat),
                                   O.BN254.elems_from_bytes(inputs.tobytes()), flat=full_flat)
    assert proof == want and tr.state == want_state


@pytest.mark.parametrize("world", [2, 8])
def test_tma_round_distributed(ctx, tma_everywhere, world):
    f = P.Field.bn254()
    insz, flat = W.layered_circuit(77, 11, 2)
    copies = 16
    inputs = W.random_inputs(f.p, insz * copies, 3)
    tr = P.Transcript(f, "tma.dist")
    single = P.gkr_prove(ctx, P.Circuit(ctx, insz, *flat, n_copies=copies), inputs, tr)
    tr2 = P.Transcript(f, "tma.dist")
    local = P.Circuit(ctx, insz, *flat, n_copies=copies // world)
    assert P.gkr_prove_dist_emulated(ctx, local, world, inputs, tr2) == single
    assert tr2.state == tr.state


def test_tuning_rejects_unknown_knob():
    with pytest.raises(P.prover.InvalidArgument):
        P.set_tuning("no_such_knob", 1)


# ---------------------------------------------------------------------------
# bookkeeping by row pairs with round 1 fused (k_bookkeep_pairs)
# ---------------------------------------------------------------------------
def _prove_fuse(ctx, f, insz, flat, copies, inputs, label, fuse):
    old = P.get_tuning("fuse_round1")
    P.set_tuning("fuse_round1", 1 if fuse else 0)
    try:
        circ = P.Circuit(ctx, insz, *flat, n_copies=copies)
        tr = P.Transcript(f, label)
        return P.gkr_prove(ctx, circ, inputs, tr), tr.state
    finally:
        P.set_tuning("fuse_round1", old)


@pytest.mark.parametrize("p", [O.BN254_P, O.GOLDILOCKS_P, 97])
@pytest.mark.parametrize("log_w,copies,depth", [(1, 1, 3), (2, 2, 3), (8, 1, 3), (10, 8, 3)])
def test_fused_round1_equals_separate(ctx, p, log_w, copies, depth):
    f = P.Field(p)
    insz, flat = W.layered_circuit(900 + log_w, log_w, depth)
    inputs = W.random_inputs(f.p, insz * copies, 3 + log_w)
    assert _prove_fuse(ctx, f, insz, flat, copies, inputs, "fuse", True) == \
        _prove_fuse(ctx, f, insz, flat, copies, inputs, "fuse", False)


def test_fused_round1_equals_reference(ctx):
    old = P.get_tuning("fuse_round1")
    P.set_tuning("fuse_round1", 1)
    f = P.Field.bn254()
    insz, flat = W.layered_circuit(5151, 7, 5)
    copies = 4
    inputs = W.random_inputs(f.p, insz * copies, 8)
    circ = P.Circuit(ctx, insz, *flat, n_copies=copies)
    tr = P.Transcript(f, "fuse.ref")
    proof = P.gkr_prove(ctx, circ, inputs, tr)
    full_in, full_flat = W.replicate(insz, flat, copies)
    want, want_state = R.gkr_prove(O.BN254, "fuse.ref", [], O.Circuit.from_flat(full_in, *full_flat),
                                   O.BN254.elems_from_bytes(inputs.tobytes()), flat=full_flat)
    P.set_tuning("fuse_round1", old)
    assert proof == want and tr.state == want_state
