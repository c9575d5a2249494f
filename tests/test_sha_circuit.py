"""CPU: the SHA-256 compression circuit (sha_circuit.py):
the witness chain equals hashlib, the honest witness evaluates (oracle) to all
zero outputs, and any corrupted witness bit is caught."""
import hashlib

import numpy as np
import pytest

from oracle import dgkr_oracle as O
from paper_2404_10404_b200 import sha_circuit as S


@pytest.fixture(scope="module")
def circ():
    insz, flat, L = S.build_compression_circuit()
    return insz, flat, L, O.Circuit.from_flat(insz, *flat)


def test_merkle_path_chain_matches_hashlib():
    rng = np.random.default_rng(1)
    leaf = bytes(rng.integers(0, 256, 64, dtype=np.uint8))
    sibs = [bytes(rng.integers(0, 256, 32, dtype=np.uint8)) for _ in range(3)]
    h_in, blocks, root = S.merkle_path_compressions(leaf, sibs, 5)
    h = hashlib.sha256(leaf).digest()
    node = 5
    for s in sibs:
        h = hashlib.sha256(s + h if node & 1 else h + s).digest()
        node >>= 1
    assert root == h and len(h_in) == 2 * (1 + len(sibs))


def test_honest_witness_is_all_zero(circ):
    insz, flat, L, c = circ
    rng = np.random.default_rng(2)
    h_in = rng.integers(0, 1 << 32, (3, 8), dtype=np.uint64)
    blocks = rng.integers(0, 1 << 32, (3, 16), dtype=np.uint64)
    inp, hout = S.sha256_witness(O.BN254_P, L, insz, h_in, blocks)
    fld = O.BN254
    for k in range(3):
        vals = fld.elems_from_bytes(inp[k * insz * 32:(k + 1) * insz * 32].tobytes())
        assert not any(c.evaluate(vals, fld.p)[-1])
    # digest words equal hashlib on the padded single-block message path
    msg = bytes(range(64))
    tr = S.compress_trace(S.IV[None, :], S.digest_words(msg)[None, :])
    pad = np.zeros((1, 16), np.uint64)
    pad[0, 0], pad[0, 15] = 0x80000000, 512
    d = S.compress_trace(tr["hout"], pad)["hout"][0]
    assert b"".join(int(x).to_bytes(4, "big") for x in d) == hashlib.sha256(msg).digest()


@pytest.mark.parametrize("what", ["a", "e", "w", "hout", "qa", "hin"])
def test_corrupted_witness_is_caught(circ, what):
    insz, flat, L, c = circ
    rng = np.random.default_rng(3)
    inp, _ = S.sha256_witness(O.BN254_P, L, insz, rng.integers(0, 1 << 32, (1, 8), dtype=np.uint64),
                              rng.integers(0, 1 << 32, (1, 16), dtype=np.uint64))
    vals = O.BN254.elems_from_bytes(inp.tobytes())
    idx = {"a": L.words[("a", 30)][7], "e": L.words[("e", 64)][0], "w": L.words[("w", 40)][31],
           "hout": L.words[("hout", 3)][9], "qa": L.qbits[("a", 12)][0], "hin": L.words[("hin", 0)][0]}[what]
    vals[idx] ^= 1
    assert any(c.evaluate(vals, O.BN254_P)[-1])
    vals[idx] = 2  # not a bit
    assert any(c.evaluate(vals, O.BN254_P)[-1])


def test_rlc_circuit_single_output():
    """rlc=True folds a copy's constraints into one output sum_i R_i c_i"""
    insz, flat, L = S.build_compression_circuit(rlc=True)
    c = O.Circuit.from_flat(insz, *flat)
    assert int(flat[0][-1] - flat[0][-2]) == 1 and len(L.rlc) > 7000
    R = S.rlc_coefficients(O.BN254_P, b"test", len(L.rlc))
    rng = np.random.default_rng(9)
    inp, _ = S.sha256_witness(O.BN254_P, L, insz, rng.integers(0, 1 << 32, (1, 8), dtype=np.uint64),
                              rng.integers(0, 1 << 32, (1, 16), dtype=np.uint64), rlc=R)
    vals = O.BN254.elems_from_bytes(inp.tobytes())
    assert c.evaluate(vals, O.BN254_P)[-1] == [0]
    vals[L.words[("w", 20)][0]] ^= 1
    assert c.evaluate(vals, O.BN254_P)[-1][0] != 0
    with pytest.raises(ValueError):
        S.sha256_witness(O.BN254_P, L, insz, rng.integers(0, 1 << 32, (1, 8), dtype=np.uint64),
                         rng.integers(0, 1 << 32, (1, 16), dtype=np.uint64))


def test_rlc_slots_filled_after_commit():
    """prove_compressions_rlc's host steps: a witness built with zero R_i and
    then filled by _put_rlc equals the witness built with the R_i directly,
    and the R_i depend on the seed (the challenge drawn from the root)"""
    class _F:
        width, p = 32, O.BN254_P

        def encode(self, v):
            return b"".join(int(x).to_bytes(32, "little") for x in v)

    f = _F()
    insz, _, L = S.build_compression_circuit(rlc=True)
    rng = np.random.default_rng(4)
    h_in = rng.integers(0, 1 << 32, (2, 8), dtype=np.uint64)
    blocks = rng.integers(0, 1 << 32, (2, 16), dtype=np.uint64)
    co = S.rlc_coefficients(f.p, b"seed-a", len(L.rlc))
    assert co != S.rlc_coefficients(f.p, b"seed-b", len(L.rlc))
    want, _ = S.sha256_witness(f.p, L, insz, h_in, blocks, rlc=co)
    got, _ = S.sha256_witness(f.p, L, insz, h_in, blocks, rlc=[0] * len(L.rlc))
    S._put_rlc(f, L, insz, 2, got, co)
    assert np.array_equal(got, want)
