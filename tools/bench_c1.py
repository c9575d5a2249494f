"""Config C1 (BASELINE.json configs[0]): single-worker GKR proof of a
synthetic layered circuit (2^12 gates/layer x 16 layers) + "Virgo
commitment" as SURVEY.md §8(d) defines it for the reference: pcs::commit of
the input table as an M=1 EvalMatrix, and pcs::open at each input-claim point
of the proof (the claims come from dgkr_gkr_input_claims). Every byte is
checked against the compiled reference (oracle/_ref): the GKR proof, the
commitment root and each opening; the reference verifier accepts the proof
and every opening, and sum_t weight_t * value_t equals each claim.
Prints one JSON line: GPU and reference time per stage."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from oracle import dgkr_oracle as O  # noqa: E402
from oracle import refbind as R  # noqa: E402

LABEL, OPEN_LABEL = "dgkr.bench.c1", "dgkr.bench.c1.open"
ctx = P.Context(0)
f = P.Field.bn254()
fld = O.BN254
insz, flat = W.layered_circuit(20240410, 12, 16)
circ = P.Circuit(ctx, insz, *flat)
inputs = W.random_inputs(f.p, insz, 7)
in_vals = fld.elems_from_bytes(inputs.tobytes())


def pipeline():
    t = {}
    t0 = time.perf_counter()
    proof = P.gkr_prove(ctx, circ, inputs, P.Transcript(f, LABEL))
    t["prove_ms"] = 1e3 * (time.perf_counter() - t0)
    t0 = time.perf_counter()
    root = P.pcs_commit(ctx, f, [inputs.tobytes()])
    t["commit_ms"] = 1e3 * (time.perf_counter() - t0)
    t0 = time.perf_counter()
    ok, claims = P.gkr_input_claims(circ, proof, P.Transcript(f, LABEL))
    t["verify_ms"] = 1e3 * (time.perf_counter() - t0)
    assert ok
    t0 = time.perf_counter()
    openings = []
    for terms, value in claims:
        acc = 0
        for point, weight in terms:
            op = P.pcs_open(ctx, f, [inputs.tobytes()], point, P.Transcript(f, OPEN_LABEL))
            v = int.from_bytes(op[4 + len(point) * 32: 4 + (len(point) + 1) * 32], "little")  # Opening.value
            acc = (acc + weight * v) % f.p
            openings.append((point, op))
        assert acc == value, "input claim does not match the committed inputs"
    t["open_ms"] = 1e3 * (time.perf_counter() - t0)
    return proof, root, claims, openings, t


pipeline()  # warm-up
runs = [pipeline() for _ in range(5)]
proof, root, claims, openings, _ = runs[-1]
med = {k: statistics.median(r[4][k] for r in runs) for k in runs[0][4]}
line = {"config": "C1: single-worker GKR 2^12 gates/layer x 16 layers + pcs commit/open of the inputs at every "
                  "input-claim point (BN254)", "gates": circ.n_gates, "input_claims": len(claims),
        "openings": len(openings), "gpu_ms": med, "gpu_total_ms": sum(med.values())}
if R.available():
    oc = O.Circuit.from_flat(insz, *flat)
    t0 = time.perf_counter()
    want, _ = R.gkr_prove(fld, LABEL, [], oc, in_vals, flat=flat)
    t_ref_prove = time.perf_counter() - t0
    t0 = time.perf_counter()
    want_root = R.pcs_commit(fld, [in_vals])
    t_ref_commit = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref_ops = [R.pcs_open(fld, OPEN_LABEL, [], [in_vals], point)[0] for point, _ in openings]
    t_ref_open = time.perf_counter() - t0
    line["bytes_equal_reference"] = {
        "proof": want == proof, "root": want_root == root,
        "openings": all(a == b[1] for a, b in zip(ref_ops, openings))}
    line["reference_accepts"] = {
        "proof": R.gkr_verify(fld, LABEL, [], oc, in_vals, proof, flat=flat),
        "openings": all(R.pcs_verify(fld, OPEN_LABEL, [], 1, insz, root, point, op) for point, op in openings)}
    line["ref_ms"] = {"prove_ms": 1e3 * t_ref_prove, "commit_ms": 1e3 * t_ref_commit, "open_ms": 1e3 * t_ref_open}
    line["ref_total_ms"] = 1e3 * (t_ref_prove + t_ref_commit + t_ref_open)
print(json.dumps(line), flush=True)
