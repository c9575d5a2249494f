"""GPU: the host GKR verifier (dgkr_gkr_verify) cross-checked with the
compiled reference's prover and verifier, the binary CSR circuit file, and
the dgkr-compatible CLI (python -m paper_2404_10404_b200)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O
from oracle import refbind as R
from paper_2404_10404_b200 import circuit_io as IO
from paper_2404_10404_b200 import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _outputs(proof: bytes, w: int):
    n = int.from_bytes(proof[:4], "little")
    return [int.from_bytes(proof[4 + i * w:4 + (i + 1) * w], "little") for i in range(n)]


@pytest.mark.parametrize("seed", [3, 5, 8, 13])
def test_verifier_cross_checks_reference(ctx, seed):
    p = O.BN254_P
    f, of = P.Field(p), O.Field(p)
    circ = R.random_general_circuit(seed, input_size=6, depth=4, max_gates=9, max_nested=3)
    flat = circ.to_flat()
    dc = P.Circuit(ctx, circ.input_size, *flat)
    inputs = O.random_elements(of, circ.input_size, np.random.default_rng(seed))
    tr = P.Transcript(f, "ver", [seed])
    proof = P.gkr_prove(ctx, dc, inputs, tr)
    ref_proof, ref_state = R.gkr_prove(of, "ver", [seed], circ, inputs, flat=flat)
    assert proof == ref_proof
    outs = _outputs(proof, f.width)[: circ.layer_size(circ.depth)]
    vtr = P.Transcript(f, "ver", [seed])
    assert P.gkr_verify(dc, proof, vtr, outputs=outs, inputs=inputs)
    assert vtr.state == tr.state  # the verifier replays the prover's transcript
    assert R.gkr_verify(of, "ver", [seed], circ, inputs, proof, flat=flat)
    # rejections: wrong inputs, wrong statement, tampered round coefficient, truncation
    bad_in = list(inputs)
    bad_in[0] = (bad_in[0] + 1) % p
    assert not P.gkr_verify(dc, proof, P.Transcript(f, "ver", [seed]), outputs=outs, inputs=bad_in)
    bad_out = list(outs)
    bad_out[-1] = (bad_out[-1] + 1) % p
    assert not P.gkr_verify(dc, proof, P.Transcript(f, "ver", [seed]), outputs=bad_out)
    tam = bytearray(proof)
    tam[-40] ^= 1
    assert not P.gkr_verify(dc, bytes(tam), P.Transcript(f, "ver", [seed]))
    assert not P.gkr_verify(dc, proof[:-1], P.Transcript(f, "ver", [seed]))
    assert not P.gkr_verify(dc, proof, P.Transcript(f, "other", [seed]))


def test_verifier_data_parallel(ctx):
    p = O.BN254_P
    f = P.Field(p)
    insz, flat = W.layered_circuit(seed=2, log_width=4, depth=5)
    dc = P.Circuit(ctx, insz, *flat, n_copies=8)
    inputs = W.random_inputs(p, insz * 8, 3)
    tr = P.Transcript(f, "dpv")
    proof = P.gkr_prove(ctx, dc, inputs, tr)
    assert P.gkr_verify(dc, proof, P.Transcript(f, "dpv"), inputs=inputs)
    bad = inputs.copy()
    bad[0] ^= 1
    assert not P.gkr_verify(dc, proof, P.Transcript(f, "dpv"), inputs=bad)


def test_binary_circuit_file_round_trip(ctx, tmp_path):
    p = O.BN254_P
    f = P.Field(p)
    circ = R.random_general_circuit(21, input_size=5, depth=3, max_gates=6, max_nested=2)
    flat = circ.to_flat()
    dc = P.Circuit(ctx, circ.input_size, *flat)
    path = str(tmp_path / "c.dgkrc")
    dc.save(path)
    dc2 = P.Circuit.load(ctx, path)
    assert (dc2.depth, dc2.input_size, dc2.output_size) == (dc.depth, dc.input_size, dc.output_size)
    inputs = W.random_inputs(p, circ.input_size, 4)
    assert P.gkr_prove(ctx, dc, inputs, P.Transcript(f, "b")) == P.gkr_prove(ctx, dc2, inputs, P.Transcript(f, "b"))
    # data-parallel copy count override, and corrupt files
    insz, lf = W.layered_circuit(seed=1, log_width=3, depth=2)
    P.Circuit(ctx, insz, *lf, n_copies=4).save(path)
    assert P.Circuit.load(ctx, path).n_copies == 4
    assert P.Circuit.load(ctx, path, n_copies=2).n_copies == 2
    blob = open(path, "rb").read()
    open(path, "wb").write(blob[:-7])
    with pytest.raises(P._lib.InvalidArgument):
        P.Circuit.load(ctx, path)


def _cli(*args, cwd=None):
    env = dict(os.environ, PYTHONPATH=ROOT)
    return subprocess.run([sys.executable, "-m", "paper_2404_10404_b200", *args], capture_output=True, text=True,
                          cwd=cwd, env=env, timeout=300)


def test_cli_circuit_prove_and_convert(tmp_path):
    circ = R.random_general_circuit(9, input_size=4, depth=3, max_gates=5, max_nested=2)
    js = R.circuit_json(circ)  # written by the reference's own to_json
    path = tmp_path / "c.json"
    path.write_text(js)
    inputs = [3, 1, 4, 1]
    r = _cli("circuit", "--file", str(path), "--inputs", ",".join(map(str, inputs)), "--prove")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == f"circuit ok: {circ.depth} layers, input size {circ.input_size}"
    want = circ.evaluate(inputs, O.BN254_P)[-1][: circ.layer_size(circ.depth)]
    assert lines[1] == "outputs:" + "".join(f" {v}" for v in want)
    assert lines[2] == "proof verified"
    # validate only; wrong input count; unknown field; malformed json
    assert _cli("circuit", "--file", str(path)).returncode == 0
    r = _cli("circuit", "--file", str(path), "--inputs", "1,2")
    assert r.returncode == 2 and "expected 4 inputs" in r.stderr
    assert _cli("circuit", "--file", str(path), "--inputs", "1,2,3,4", "--field", "nope").returncode == 2
    (tmp_path / "bad.json").write_text("{not json")
    r = _cli("circuit", "--file", str(tmp_path / "bad.json"))
    assert r.returncode == 2 and "invalid circuit file" in r.stderr
    # convert to the binary format and prove from it
    binp = tmp_path / "c.dgkrc"
    assert _cli("convert", str(path), str(binp)).returncode == 0
    r2 = _cli("circuit", "--file", str(binp), "--inputs", ",".join(map(str, inputs)), "--prove")
    assert r2.returncode == 0, r2.stderr
    assert r2.stdout.splitlines() == lines


def test_cli_bitchange_matches_reference(tmp_path):
    out = tmp_path / "bc.csv"
    r = _cli("bitchange", "--field", "goldilocks", "--count", "10000", "--out", str(out))
    assert r.returncode == 0, r.stderr
    counts = R.distinct_bitchange(O.Field(O.GOLDILOCKS_P), 10000)
    want = "index,bit_change\n" + "".join(f"{i},{c / 10000:g}\n" for i, c in enumerate(counts))
    assert out.read_text() == want
    assert _cli("bitchange", "--count", "10", "--out", str(out)).returncode == 2


def test_cli_bench(tmp_path):
    out = tmp_path / "bench.csv"
    r = _cli("bench", "--workers", "1,2,4", "--vars", "8", "--out", str(out))
    assert r.returncode == 0, r.stderr
    rows = out.read_text().splitlines()
    assert rows[0] == "numval,time" and [x.split(",")[0] for x in rows[1:]] == ["1", "2", "4"]
    assert _cli("bench", "--workers", "3", "--vars", "8", "--out", str(out)).returncode == 2


def test_input_claims_match_the_inputs(ctx):
    """dgkr_gkr_input_claims: the verifier's input-layer claims, each equal to
    sum_t weight_t * MLE(inputs, point_t) (check_input_claims, gkr.hpp:314-325)"""
    p = O.BN254_P
    f, of = P.Field(p), O.Field(p)
    circ = R.random_general_circuit(17, input_size=6, depth=4, max_gates=9, max_nested=3)
    flat = circ.to_flat()
    dc = P.Circuit(ctx, circ.input_size, *flat)
    inputs = O.random_elements(of, circ.input_size, np.random.default_rng(17))
    proof = P.gkr_prove(ctx, dc, inputs, P.Transcript(f, "claims"))
    ok, claims = P.gkr_input_claims(dc, proof, P.Transcript(f, "claims"))
    assert ok and claims
    table = list(inputs) + [0] * (circ.padded_size(0) - len(inputs))
    for terms, value in claims:
        assert sum(w * O.mle_eval(table, pt, p) for pt, w in terms) % p == value
    tam = bytearray(proof)
    tam[-40] ^= 1
    assert P.gkr_input_claims(dc, bytes(tam), P.Transcript(f, "claims")) == (False, [])


def test_fuzz_verifier_and_loader(ctx, tmp_path):
    """malformed proofs reject (no exception, no crash); corrupted circuit files
    raise InvalidArgument"""
    p = O.BN254_P
    f = P.Field(p)
    insz, flat = W.layered_circuit(seed=3, log_width=4, depth=3)
    dc = P.Circuit(ctx, insz, *flat, n_copies=2)
    inputs = W.random_inputs(p, insz * 2, 5)
    proof = P.gkr_prove(ctx, dc, inputs, P.Transcript(f, "fz"))
    rng = np.random.default_rng(99)
    for trial in range(200):
        b = bytearray(proof)
        kind = trial % 4
        if kind == 0:
            for _ in range(int(rng.integers(1, 8))):
                b[int(rng.integers(0, len(b)))] ^= int(rng.integers(1, 256))
        elif kind == 1:
            b = b[: int(rng.integers(0, len(b)))]
        elif kind == 2:
            b = bytearray(rng.integers(0, 256, int(rng.integers(0, 2 * len(proof))), dtype=np.uint8).tobytes())
        else:
            b += bytes(int(rng.integers(1, 64)))
        assert not P.gkr_verify(dc, bytes(b), P.Transcript(f, "fz"), inputs=inputs)
        assert P.gkr_input_claims(dc, bytes(b), P.Transcript(f, "fz"))[0] is False
    assert P.gkr_verify(dc, proof, P.Transcript(f, "fz"), inputs=inputs)
    # binary circuit files: corrupt header fields and truncations
    path = str(tmp_path / "c.dgkrc")
    dc.save(path)
    blob = open(path, "rb").read()
    for trial in range(40):
        b = bytearray(blob)
        if trial % 2:
            off = int(rng.integers(8, 40))  # header: sizes / counts
            b[off] ^= int(rng.integers(1, 256))
        else:
            b = b[: int(rng.integers(0, len(b)))]
        open(path, "wb").write(bytes(b))
        try:
            P.Circuit.load(ctx, path)
        except P._lib.InvalidArgument:
            pass
        except P._lib.DgkrError as e:  # e.g. a header that asks for too much memory
            assert "CAPACITY" in str(e) or "UNSUPPORTED" in str(e) or "CUDA" in str(e), str(e)
