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


@pytest.mark.parametrize("world,n,blowup,final,q", [(1, 16, 2, 1, 8), (2, 8, 2, 1, 4), (3, 16, 1, 2, 100),
                                                    (4, 256, 2, 3, 16), (8, 64, 1, 2, 12)])
def test_fri_dist_emulated_matches_oracle(ctx, world, n, blowup, final, q):
    """distributed FRI, `world` ranks as threads on lanes of one GPU: every
    rank's proof equals the oracle's, the transcript ends in the same state
    and the distributed verifier accepts"""
    fld = O.BN254
    f = P.Field(fld.p)
    rng = np.random.default_rng(world * 1000 + n)
    chunks = [O.random_elements(fld, n, rng) for _ in range(world)]
    tr = P.Transcript(f, "fri.d", [world])
    got = P.fri_prove_dist_emulated(ctx, f, chunks, blowup, final, q, tr)
    otr = O.Transcript("fri.d", fld, [world])
    assert got == FO.fri_prove_dist(fld, chunks, blowup, final, q, otr)
    assert tr.state == otr.state
    assert FO.fri_verify_dist(fld, got, n, blowup, final, q, O.Transcript("fri.d", fld, [world]))
    if world == 1:
        single = P.fri_prove(ctx, f, chunks[0], blowup, final, q, P.Transcript(f, "fri.d", [world]))
        assert got[0][8:] == single


@pytest.mark.parametrize("p", [O.GOLDILOCKS_P, 97])
def test_fri_dist_emulated_runtime_fields(ctx, p):
    fld = O.Field(p)
    f = P.Field(p)
    rng = np.random.default_rng(p % 1000)
    n = 4 if p == 97 else 64
    chunks = [O.random_elements(fld, n, rng) for _ in range(2)]
    got = P.fri_prove_dist_emulated(ctx, f, chunks, 1, 1, 6, P.Transcript(f, "fri.d"))
    assert got == FO.fri_prove_dist(fld, chunks, 1, 1, 6, O.Transcript("fri.d", fld))


def test_fri_dist_large_verifies(ctx):
    """4 ranks x 2^14 coefficients, blowup 4: the distributed verifier accepts"""
    from paper_2404_10404_b200 import workloads as W

    fld = O.BN254
    f = P.Field(fld.p)
    n = 1 << 14
    chunks = [W.random_inputs(fld.p, n, 20 + r) for r in range(4)]
    got = P.fri_prove_dist_emulated(ctx, f, chunks, 2, 5, 12, P.Transcript(f, "fri.dbig"))
    assert FO.fri_verify_dist(fld, got, n, 2, 5, 12, O.Transcript("fri.dbig", fld))


def test_fri_dist_two_process_shm(ctx, tmp_path):
    """two processes (one per rank) over the shared-memory transport: each
    rank's proof equals the emulated run's and the verifier accepts"""
    import os
    import secrets
    import subprocess
    import sys

    from paper_2404_10404_b200 import workloads as W

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    world, n, blowup, final, q = 2, 1 << 10, 2, 3, 16
    token = secrets.token_hex(4)
    out = str(tmp_path / "fri")
    worker = os.path.join(root, "tools", "fri_shm_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), token, str(n), str(blowup), str(final),
                               str(q), out], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    logs = [p.communicate(timeout=300)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    fld = O.BN254
    f = P.Field(fld.p)
    chunks = [W.random_inputs(fld.p, n, 100 + r) for r in range(world)]
    tr = P.Transcript(f, "fri.shm", [world])
    want = P.fri_prove_dist_emulated(ctx, f, chunks, blowup, final, q, tr)
    got = []
    for r in range(world):
        raw = open(f"{out}.{r}", "rb").read()
        got.append(raw[:-32])
        assert raw[-32:] == tr.state
    assert got == want
    assert FO.fri_verify_dist(fld, got, n, blowup, final, q, O.Transcript("fri.shm", fld, [world]))


def test_ntt_large_roundtrip_through_chunked_transfers(ctx):
    """2^21 elements (64 MiB each way, pageable host buffers): the upload and
    the download take the chunked pinned-staging path (Lane::h2d_large /
    d2h_large); iNTT(NTT(a)) = a byte for byte, and entry 0 of the forward
    transform is the sum of the inputs"""
    from paper_2404_10404_b200 import workloads as W

    f = P.Field.bn254()
    n_log = 21
    a = W.random_inputs(f.p, 1 << n_log, 77).tobytes()
    fwd = P.ntt(ctx, f, a)
    back = P.ntt(ctx, f, f.encode(fwd), inverse=True)
    assert f.encode(back) == a
    # the forward transform's first entry is the sum of the inputs
    fld = O.BN254
    assert fwd[0] == sum(fld.elems_from_bytes(a)) % fld.p
