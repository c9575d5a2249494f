"""GPU: committed-witness rlc proofs of SHA-256 compressions
(sha_circuit.prove_compressions_rlc): a Merkle path proves with every
claimed output zero and the verifier accepts; the R_i depend on the witness
commitment; a corrupted witness (with an honest commitment to it) gives a
non-zero output, and tampering with the root, the R_i or the proof is
rejected."""
import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O
from paper_2404_10404_b200 import sha_circuit as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def path_case():
    rng = np.random.default_rng(11)
    leaf = bytes(rng.integers(0, 256, 64, dtype=np.uint8))
    sibs = [bytes(rng.integers(0, 256, 32, dtype=np.uint8)) for _ in range(3)]
    return S.merkle_path_compressions(leaf, sibs, 5)  # 8 compressions


def test_rlc_commit_path_accepts(ctx, path_case):
    f = P.Field(O.BN254_P)
    h_in, blocks, root_digest = path_case
    pr, built = S.prove_compressions_rlc(ctx, f, h_in, blocks)
    n = int.from_bytes(pr.proof[:4], "little")
    assert n >= len(h_in) and not any(pr.proof[4:4 + n * f.width])
    assert b"".join(int(x).to_bytes(4, "big") for x in pr.digests[-1]) == root_digest
    assert S.verify_compressions_rlc(ctx, f, built, pr.inputs, pr.root, pr.proof)
    # deterministic
    pr2, _ = S.prove_compressions_rlc(ctx, f, h_in, blocks, built=built)
    assert (pr2.root, pr2.proof) == (pr.root, pr.proof)


def test_rlc_commit_rejects_tampering(ctx, path_case):
    f = P.Field(O.BN254_P)
    h_in, blocks, _ = path_case
    pr, built = S.prove_compressions_rlc(ctx, f, h_in, blocks)
    bad_root = bytes([pr.root[0] ^ 1]) + pr.root[1:]
    assert not S.verify_compressions_rlc(ctx, f, built, pr.inputs, bad_root, pr.proof)
    insz, _, L, _ = built
    w = f.width
    bad_r = pr.inputs.copy()
    bad_r[L.rlc[0] * w] ^= 1
    assert not S.verify_compressions_rlc(ctx, f, built, bad_r, pr.root, pr.proof)
    bad_p = bytearray(pr.proof)
    bad_p[-40] ^= 1
    assert not S.verify_compressions_rlc(ctx, f, built, pr.inputs, pr.root, bytes(bad_p))


def test_rlc_commit_wrong_witness_nonzero(ctx, path_case):
    """a wrong digest word in compression 3: the prover commits to it
    honestly, the R_i are drawn after, and copy 3's output is non-zero"""
    f = P.Field(O.BN254_P)
    h_in, blocks, _ = path_case
    blocks = blocks.copy()
    pr, built = S.prove_compressions_rlc(ctx, f, h_in, blocks)
    insz, flat, L, dc = built
    w = f.width
    # flip one witness bit of copy 3 (its round-50 e word), re-commit and re-prove
    bad = pr.inputs.copy()
    S._put_rlc(f, L, insz, len(bad) // (insz * w), bad, [0] * len(L.rlc))
    bad[(3 * insz + L.words[("e", 50)][3]) * w] ^= 1
    root = S._witness_root(ctx, f, bad)
    tr = P.Transcript(f, "sha.rlc", [len(bad) // (insz * w)])
    coeffs = S.rlc_coefficients(f.p, S._rlc_seed(tr, root), len(L.rlc))
    S._put_rlc(f, L, insz, len(bad) // (insz * w), bad, coeffs)
    proof = P.gkr_prove(ctx, dc, bad, tr)
    n = int.from_bytes(proof[:4], "little")
    outs = [int.from_bytes(proof[4 + i * w:4 + (i + 1) * w], "little") for i in range(n)]
    assert [i for i, v in enumerate(outs) if v] == [3]
    assert not S.verify_compressions_rlc(ctx, f, built, bad, root, proof)
