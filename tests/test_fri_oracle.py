"""CPU: the NTT / RS / FRI restatement (oracle/fri_oracle.py). No reference
implementation exists (parity unpinned); these pin the spec by
algebraic properties and an honest/tampered-proof verifier."""
import numpy as np
import pytest

from oracle import dgkr_oracle as O
from oracle import fri_oracle as FO


@pytest.mark.parametrize("fld", [O.BN254, O.GOLDILOCKS, O.TINY97], ids=["bn254", "goldilocks", "p97"])
def test_two_adic_structure(fld):
    s, w, g = FO.two_adic(fld)
    p = fld.p
    assert (p - 1) % (1 << s) == 0 and ((p - 1) >> s) % 2 == 1
    assert pow(w, 1 << s, p) == 1 and pow(w, 1 << (s - 1), p) == p - 1
    assert pow(g, (p - 1) // 2, p) == p - 1  # non-residue: outside every 2-power subgroup coset-wise


@pytest.mark.parametrize("n", [1, 2, 8, 32])
def test_ntt_matches_dft_and_inverts(n):
    fld = O.BN254
    a = O.random_elements(fld, n, np.random.default_rng(n))
    assert FO.ntt_fast(fld, a) == FO.ntt(fld, a)
    assert FO.ntt_fast(fld, FO.ntt_fast(fld, a), inverse=True) == a


def test_fold_of_codeword_is_codeword():
    fld = O.BN254
    p = fld.p
    rng = np.random.default_rng(3)
    co = O.random_elements(fld, 16, rng)
    cw = FO.rs_encode(fld, co, 2)  # N = 64
    beta = O.random_elements(fld, 1, rng)[0]
    folded = FO.fri_fold(fld, cw, beta, 0, 6)
    # f'(y) = f_even(y) + beta f_odd(y) on the squared coset
    even, odd = co[0::2], co[1::2]
    want = [(e + beta * o) % p for e, o in zip(even, odd)]
    _, _, g = FO.two_adic(fld)
    g2 = g * g % p
    w2 = pow(FO.root_of_unity(fld, 6), 2, p)
    direct = [sum(c * pow(g2 * pow(w2, i, p) % p, j, p) for j, c in enumerate(want)) % p for i in range(32)]
    assert folded == direct


@pytest.mark.parametrize("n,blowup,final,q", [(8, 2, 1, 4), (16, 1, 2, 100), (4, 3, 0, 8), (32, 2, 3, 16)])
def test_fri_honest_accepts_tampered_rejects(n, blowup, final, q):
    fld = O.BN254
    co = O.random_elements(fld, n, np.random.default_rng(n + q))
    pr = FO.fri_prove(fld, co, blowup, final, q, O.Transcript("fri", fld))
    assert FO.fri_verify(fld, pr, n, blowup, final, q, O.Transcript("fri", fld))
    for k in (40, len(pr) // 2, 10):
        bad = bytearray(pr)
        bad[k] ^= 1
        assert not FO.fri_verify(fld, bytes(bad), n, blowup, final, q, O.Transcript("fri", fld))


def test_fri_dist_world1_is_single_proof_with_header():
    fld = O.BN254
    co = O.random_elements(fld, 16, np.random.default_rng(3))
    one = FO.fri_prove(fld, co, 2, 1, 8, O.Transcript("fri", fld))
    (d,) = FO.fri_prove_dist(fld, [co], 2, 1, 8, O.Transcript("fri", fld))
    assert d == (1).to_bytes(4, "little") + (0).to_bytes(4, "little") + one


@pytest.mark.parametrize("world,n,blowup,final,q", [(2, 8, 2, 1, 4), (3, 16, 1, 2, 100), (4, 4, 3, 0, 8)])
def test_fri_dist_honest_accepts_tampered_rejects(world, n, blowup, final, q):
    fld = O.BN254
    rng = np.random.default_rng(world * 100 + n)
    chunks = [O.random_elements(fld, n, rng) for _ in range(world)]
    prs = FO.fri_prove_dist(fld, chunks, blowup, final, q, O.Transcript("fri.d", fld))
    assert FO.fri_verify_dist(fld, prs, n, blowup, final, q, O.Transcript("fri.d", fld))
    # ranks swapped, a rank's proof missing, a flipped byte in the shared head or in the openings
    assert not FO.fri_verify_dist(fld, prs[::-1], n, blowup, final, q, O.Transcript("fri.d", fld))
    assert not FO.fri_verify_dist(fld, prs[:-1], n, blowup, final, q, O.Transcript("fri.d", fld))
    for r in range(world):
        for k in (20, len(prs[r]) // 2, len(prs[r]) - 3):
            bad = list(prs)
            b = bytearray(bad[r])
            b[k] ^= 1
            bad[r] = bytes(b)
            assert not FO.fri_verify_dist(fld, bad, n, blowup, final, q, O.Transcript("fri.d", fld))


def test_fri_dist_rejects_high_degree_rank():
    """a rank whose codeword is not low-degree (random word) is caught"""
    fld = O.BN254
    rng = np.random.default_rng(5)
    good = O.random_elements(fld, 8, rng)
    bad = O.random_elements(fld, 32, rng)  # 4x the degree bound on the same domain with blowup 0
    prs_good = FO.fri_prove_dist(fld, [good, good], 2, 1, 100, O.Transcript("fri.d", fld))
    assert FO.fri_verify_dist(fld, prs_good, 8, 2, 1, 100, O.Transcript("fri.d", fld))
    prs = FO.fri_prove_dist(fld, [good[:8] * 4, bad], 0, 1, 100, O.Transcript("fri.d", fld))
    assert not FO.fri_verify_dist(fld, prs, 8, 2, 1, 100, O.Transcript("fri.d", fld))
