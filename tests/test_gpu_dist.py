"""GPU: the multi-GPU data-parallel protocol (rank = high variables, per-round
all-gather of 3 field elements, boundary all-gather + log2(world) tail
rounds) with ranks emulated as host threads driving lanes of one B200.

The bar (acceptance #2 SPEC.md:725; cluster.hpp:219-227): the
distributed proof is byte-identical to the single-GPU proof of the full
circuit, and every rank holds the same proof (checked inside the call).
"""
import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O
from paper_2404_10404_b200 import workloads as W
from paper_2404_10404_b200._lib import InvalidArgument

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_dist_emulated_equals_single_and_oracle(ctx, world):
    p = O.BN254_P
    f, of = P.Field(p), O.Field(p)
    n_total = 8
    insz, flat = W.layered_circuit(seed=31, log_width=4, depth=4)
    inputs = W.random_inputs(p, insz * n_total, 32)
    single = P.Circuit(ctx, insz, *flat, n_copies=n_total)
    tr1 = P.Transcript(f, "dist", [7])
    want = P.gkr_prove(ctx, single, inputs, tr1)
    local = P.Circuit(ctx, insz, *flat, n_copies=n_total // world)
    tr2 = P.Transcript(f, "dist", [7])
    got = P.gkr_prove_dist_emulated(ctx, local, world, inputs, tr2)
    assert got == want and tr2.state == tr1.state
    full_in, full_flat = W.replicate(insz, flat, n_total)
    otr = O.Transcript("dist", of, [7])
    outs, layers = O.gkr_prove(O.Circuit.from_flat(full_in, *full_flat), of.elems_from_bytes(inputs.tobytes()), otr)
    assert got == O.gkr_proof_bytes(of, outs, layers)


@pytest.mark.parametrize("world", [2, 8])
def test_dist_emulated_larger(ctx, world):
    """2^10-wide sub-circuits x 6 layers, 16 copies: single == distributed."""
    p = O.BN254_P
    f = P.Field(p)
    insz, flat = W.layered_circuit(seed=41, log_width=10, depth=6)
    inputs = W.random_inputs(p, insz * 16, 42)
    tr1 = P.Transcript(f, "dist.big")
    want = P.gkr_prove(ctx, P.Circuit(ctx, insz, *flat, n_copies=16), inputs, tr1)
    tr2 = P.Transcript(f, "dist.big")
    got = P.gkr_prove_dist_emulated(ctx, P.Circuit(ctx, insz, *flat, n_copies=16 // world), world, inputs, tr2)
    assert got == want and tr1.state == tr2.state


def test_dist_requires_uniform_width(ctx):
    p = O.BN254_P
    f = P.Field(p)
    insz, flat = W.layered_circuit(seed=1, log_width=4, depth=2, input_log=3)  # input layer narrower
    local = P.Circuit(ctx, insz, *flat, n_copies=2)
    with pytest.raises(InvalidArgument):
        P.gkr_prove_dist_emulated(ctx, local, 2, W.random_inputs(p, insz * 4, 1), P.Transcript(f, "x"))


def test_nccl_transport_world1(ctx):
    """The NCCL communicator path (dlopen'd libnccl, all-gather / send-recv
    group / broadcast) with the one rank a single GPU allows."""
    p = O.BN254_P
    f = P.Field(p)
    insz, flat = W.layered_circuit(seed=61, log_width=6, depth=4)
    inputs = W.random_inputs(p, insz * 4, 62)
    tr1 = P.Transcript(f, "nccl")
    want = P.gkr_prove(ctx, P.Circuit(ctx, insz, *flat, n_copies=4), inputs, tr1)
    comm = P.Comm(ctx, P.Comm.nccl_unique_id(), 0, 1)
    tr2 = P.Transcript(f, "nccl")
    got = P.gkr_prove_dist(ctx, comm, P.Circuit(ctx, insz, *flat, n_copies=4), inputs, tr2)
    assert got == want and tr2.state == tr1.state


@pytest.mark.parametrize("p", [O.BN254_P, O.GOLDILOCKS_P, 97])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("vars_,n_pairs", [(3, 1), (7, 2), (12, 3)])
def test_dist_sumcheck_over_comm_equals_single(ctx, p, world, vars_, n_pairs):
    """dist_sumcheck with the ranks' shards exchanging round sums through a
    communicator (dgkr_dist_sumcheck_comm's code path, ranks as threads):
    the single-machine prove_product_sum bytes on every rank (cluster.hpp:219-227)"""
    rng = np.random.default_rng(900 + world + 10 * vars_ + p % 91)
    f, of = P.Field(p), O.Field(p)
    pairs = [(O.random_elements(of, 1 << vars_, rng), O.random_elements(of, 1 << vars_, rng)) for _ in range(n_pairs)]
    t1 = P.Transcript(f, "dsc", [world])
    single = P.prove_product_sum(ctx, pairs, t1)
    t2 = P.Transcript(f, "dsc", [world])
    assert P.prover.dist_sumcheck_emulated(ctx, world, pairs, t2) == single
    assert t2.state == t1.state
