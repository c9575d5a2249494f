"""GPU: NTT, RS encoding and FRI (north-star "Virgo/FRI") against the
Python restatement of our spec (oracle/fri_oracle.py; parity vs the
reference is unpinned — the reference has no FRI) and its verifier."""
import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O
from oracle import fri_oracle as FO

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p", [O.BN254_P, O.GOLDILOCKS_P, 97])
@pytest.mark.parametrize("log_n", [0, 1, 3, 5, 11, 12])
def test_ntt_matches_oracle(ctx, p, log_n):
    fld = O.Field(p)
    if log_n > FO.two_adic(fld)[0]:
        pytest.skip("domain larger than the 2-adic subgroup")
    f = P.Field(p)
    a = O.random_elements(fld, 1 << log_n, np.random.default_rng(log_n))
    assert P.ntt(ctx, f, a) == FO.ntt_fast(fld, a)
    assert P.ntt(ctx, f, FO.ntt_fast(fld, a), inverse=True) == a


@pytest.mark.parametrize("n,blowup", [(1, 1), (8, 2), (64, 1), (1024, 2)])
def test_rs_encode_matches_oracle(ctx, n, blowup):
    fld = O.BN254
    co = O.random_elements(fld, n, np.random.default_rng(n))
    assert P.rs_encode(ctx, P.Field(fld.p), co, blowup) == FO.rs_encode(fld, co, blowup)


@pytest.mark.parametrize("n,blowup,final,q", [(8, 2, 1, 4), (16, 1, 2, 100), (4, 3, 0, 8), (256, 2, 3, 16),
                                              (1024, 1, 4, 32)])
def test_fri_prove_matches_oracle_and_verifies(ctx, n, blowup, final, q):
    fld = O.BN254
    f = P.Field(fld.p)
    co = O.random_elements(fld, n, np.random.default_rng(n * 7 + q))
    tr = P.Transcript(f, "fri", [n])
    got = P.fri_prove(ctx, f, co, blowup, final, q, tr)
    otr = O.Transcript("fri", fld, [n])
    assert got == FO.fri_prove(fld, co, blowup, final, q, otr)
    assert tr.state == otr.state
    assert FO.fri_verify(fld, got, n, blowup, final, q, O.Transcript("fri", fld, [n]))


def test_fri_large_verifies(ctx):
    """2^16 coefficients, blowup 4 (2^18 codeword): the verifier accepts."""
    fld = O.BN254
    f = P.Field(fld.p)
    n = 1 << 16
    from paper_2404_10404_b200 import workloads as W

    co = W.random_inputs(fld.p, n, 9)
    got = P.fri_prove(ctx, f, co, 2, 6, 16, P.Transcript(f, "fri.big"))
    assert FO.fri_verify(fld, got, n, 2, 6, 16, O.Transcript("fri.big", fld))
