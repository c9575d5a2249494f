"""GPU: SHA-256 compression circuits (sha_circuit.py)
proved by the data-parallel GKR prover: byte-equal to the compiled
reference's gkr_prove of the replicated circuit, all claimed outputs zero
for honest witnesses, our and the reference's verifiers accept, and a
corrupted witness shows up as a non-zero claimed output."""
import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O
from paper_2404_10404_b200 import sha_circuit as S
from paper_2404_10404_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sha():
    return S.build_compression_circuit()


def _outs(proof, w):
    n = int.from_bytes(proof[:4], "little")
    return [int.from_bytes(proof[4 + i * w:4 + (i + 1) * w], "little") for i in range(n)]


def test_sha_circuit_matches_reference(ctx, sha):
    R = pytest.importorskip("oracle.refbind")
    if not R.available():
        pytest.skip("oracle/_ref not built")
    insz, flat, L = sha
    p = O.BN254_P
    f, of = P.Field(p), O.Field(p)
    rng = np.random.default_rng(5)
    n = 2
    inputs, _ = S.sha256_witness(p, L, insz, rng.integers(0, 1 << 32, (n, 8), dtype=np.uint64),
                                 rng.integers(0, 1 << 32, (n, 16), dtype=np.uint64))
    dc = P.Circuit(ctx, insz, *flat, n_copies=n)
    tr = P.Transcript(f, "sha", [n])
    got = P.gkr_prove(ctx, dc, inputs, tr)
    assert not any(_outs(got, f.width))
    full_in, full_flat = W.replicate(insz, flat, n)
    circ = O.Circuit.from_flat(full_in, *full_flat)
    ins = of.elems_from_bytes(inputs.tobytes())
    want, _ = R.gkr_prove(of, "sha", [n], circ, ins, flat=full_flat)
    assert got == want
    assert P.gkr_verify(dc, got, P.Transcript(f, "sha", [n]), inputs=inputs)


def test_sha_merkle_path_circuit(ctx, sha):
    """a depth-6 Merkle path: 14 compressions (16 copies with 2 dummy ones),
    all constraints zero, digest chain equals hashlib; a corrupted copy is
    visible in exactly its own outputs"""
    insz, flat, L = sha
    p = O.BN254_P
    f = P.Field(p)
    rng = np.random.default_rng(6)
    leaf = bytes(rng.integers(0, 256, 64, dtype=np.uint8))
    sibs = [bytes(rng.integers(0, 256, 32, dtype=np.uint8)) for _ in range(6)]
    h_in, blocks, root = S.merkle_path_compressions(leaf, sibs, 37)
    m = len(h_in)
    copies = 16
    h_in = np.concatenate([h_in, np.tile(S.IV, (copies - m, 1))])
    blocks = np.concatenate([blocks, np.zeros((copies - m, 16), np.uint64)])
    inputs, hout = S.sha256_witness(p, L, insz, h_in, blocks)
    dc = P.Circuit(ctx, insz, *flat, n_copies=copies)
    proof = P.gkr_prove(ctx, dc, inputs, P.Transcript(f, "path"))
    assert not any(_outs(proof, f.width))
    assert P.gkr_verify(dc, proof, P.Transcript(f, "path"), inputs=inputs)
    assert b"".join(int(x).to_bytes(4, "big") for x in hout[m - 1]) == root
    bad = inputs.copy()
    k = 9
    bad[(k * insz + L.words[("e", 50)][3]) * 32] ^= 1
    outs = _outs(P.gkr_prove(ctx, dc, bad, P.Transcript(f, "path")), f.width)
    per = dc.output_size // copies
    nz = {i // per for i, v in enumerate(outs) if v}
    assert nz == {k}


def test_sha_rlc_circuit_matches_reference(ctx):
    """the rlc=True circuit (one output per compression) proved by the GPU,
    byte-equal to the compiled reference; outputs all zero"""
    R = pytest.importorskip("oracle.refbind")
    if not R.available():
        pytest.skip("oracle/_ref not built")
    insz, flat, L = S.build_compression_circuit(rlc=True)
    p = O.BN254_P
    f, of = P.Field(p), O.Field(p)
    rng = np.random.default_rng(8)
    n = 2
    coeffs = S.rlc_coefficients(p, b"gpu", len(L.rlc))
    inputs, _ = S.sha256_witness(p, L, insz, rng.integers(0, 1 << 32, (n, 8), dtype=np.uint64),
                                 rng.integers(0, 1 << 32, (n, 16), dtype=np.uint64), rlc=coeffs)
    dc = P.Circuit(ctx, insz, *flat, n_copies=n)
    got = P.gkr_prove(ctx, dc, inputs, P.Transcript(f, "rlc"))
    assert _outs(got, f.width) == [0, 0]
    full_in, full_flat = W.replicate(insz, flat, n)
    circ = O.Circuit.from_flat(full_in, *full_flat)
    want, _ = R.gkr_prove(of, "rlc", [], circ, of.elems_from_bytes(inputs.tobytes()), flat=full_flat)
    assert got == want
