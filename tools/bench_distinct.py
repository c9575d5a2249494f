"""Config C4 (BASELINE.json / SURVEY.md §8(d)): associative hash over 32,000
validator indexes on one GPU, beside the compiled reference (oracle/_ref,
single-threaded as the reference is).

  * native: dgkr_distinct_check (AH of the list and of its sorted copy +
    strict-ascent scan) and dgkr_distinct_chain_update, host bytes in and out
    (latency per call, median of 20 after warm-up);
  * circuit: gkr_prove of the AH circuit (workloads.ah_circuit, k indexes per
    copy, data-parallel over the copies) for the same list.
Prints one JSON line per measurement."""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from oracle import dgkr_oracle as O  # noqa: E402
from oracle import refbind as R  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
ctx = P.Context(0)
f = P.Field.bn254()
fld = O.BN254
rng = np.random.default_rng(4)
items = [int(x) for x in rng.permutation(n)]
srt = sorted(items)
ba, bs = fld.elems_to_bytes(items), fld.elems_to_bytes(srt)


def med(fn, reps=20):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * statistics.median(ts)


gpu_check = med(lambda: P.pairwise_distinct_check(ctx, f, ba, bs))
gpu_chain = med(lambda: P.chain_update(ctx, f, 0, n, ba))
assert P.pairwise_distinct_check(ctx, f, ba, bs)
ref_check = ref_chain = None
if R.available():
    t0 = time.perf_counter()
    assert R.distinct_check(fld, items, srt)
    ref_check = 1e3 * (time.perf_counter() - t0)
    t0 = time.perf_counter()
    h = R.distinct_chain_update(fld, 0, n, items)
    ref_chain = 1e3 * (time.perf_counter() - t0)
    assert h == P.chain_update(ctx, f, 0, n, ba)
print(json.dumps({"config": f"C4 native: pairwise_distinct_check + chain_update over {n} indexes (BN254)",
                  "mults_per_list": 6 * n, "gpu_check_ms": gpu_check, "gpu_chain_update_ms": gpu_chain,
                  "ref_check_ms": ref_check, "ref_chain_update_ms": ref_chain,
                  "note": "host bytes in/out, one host sync per call"}), flush=True)

# AH as a data-parallel GKR circuit
insz, flat = W.ah_circuit(k)
inputs, copies = W.ah_inputs(fld.p, items, k)
circ = P.Circuit(ctx, insz, *flat, n_copies=copies)
gates = copies * (int(flat[0][-1]))
P.gkr_prove(ctx, circ, inputs, P.Transcript(f, "c4"))
ts = []
for _ in range(5):
    tr = P.Transcript(f, "c4")
    t0 = time.perf_counter()
    proof = P.gkr_prove(ctx, circ, inputs, tr)
    ts.append(time.perf_counter() - t0)
gpu_prove = 1e3 * statistics.median(ts)
n_out = int.from_bytes(proof[:4], "little")
outs = fld.elems_from_bytes(proof[4:4 + n_out * fld.width])
assert sum(outs) % fld.p == P.distinct_ah(ctx, f, ba)
line = {"config": f"C4 circuit: AH of {n} indexes as GKR, k={k} per copy x {copies} copies, depth {len(flat[0]) - 1}",
        "gates": gates, "gpu_prove_ms": gpu_prove, "gpu_gates_per_s": gates / (gpu_prove * 1e-3),
        "proof_bytes": len(proof)}
if R.available():
    full_in, full_flat = W.replicate(insz, flat, copies)
    oc = O.Circuit.from_flat(full_in, *full_flat)
    ins = fld.elems_from_bytes(inputs.tobytes())
    t0 = time.perf_counter()
    want, _ = R.gkr_prove(fld, "c4", [], oc, ins, flat=full_flat)
    line["ref_prove_ms"] = 1e3 * (time.perf_counter() - t0)
    line["bytes_equal_reference"] = want == proof
print(json.dumps(line), flush=True)

# pairwise-distinct check as a grand-product circuit (distinct_circuit.py)
from paper_2404_10404_b200 import distinct_circuit as DC  # noqa: E402

k = 64
dinsz, dflat, DL = DC.build_distinct_circuit(k)
r, coeffs = DC.derive_challenges(fld.p, b"bench.c4", DL.n_constraints)
t0 = time.perf_counter()
dinputs, dcopies = DC.distinct_witness(fld.p, DL, dinsz, items, srt, r, coeffs)
t_wit = time.perf_counter() - t0
dcirc = P.Circuit(ctx, dinsz, *dflat, n_copies=dcopies)
dgates = dcopies * int(dflat[0][-1])
P.gkr_prove(ctx, dcirc, dinputs, P.Transcript(f, "c4.gp"))
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    dproof = P.gkr_prove(ctx, dcirc, dinputs, P.Transcript(f, "c4.gp"))
    ts.append(time.perf_counter() - t0)
n_out = int.from_bytes(dproof[:4], "little")
douts = fld.elems_from_bytes(dproof[4:4 + n_out * fld.width])
assert DC.accept(fld.p, douts, dcopies)
line = {"config": f"C4 circuit: pairwise-distinct (grand product + strict ascent) over {n} indexes, k={k} per copy x "
                  f"{dcopies} copies, depth {len(dflat[0]) - 1}", "gates": dgates,
        "gpu_prove_ms": 1e3 * statistics.median(ts), "proof_bytes": len(dproof), "witness_gen_s": t_wit}
if R.available():
    sample = 8
    fi, ff = W.replicate(dinsz, dflat, sample)
    oc = O.Circuit.from_flat(fi, *ff)
    ins = fld.elems_from_bytes(dinputs[: sample * dinsz * fld.width].tobytes())
    t0 = time.perf_counter()
    R.gkr_prove(fld, "c4.gp", [], oc, ins, flat=ff)
    line["ref_prove_ms_extrapolated"] = 1e3 * (time.perf_counter() - t0) * dcopies / sample
    line["ref_note"] = f"compiled reference gkr_prove on {sample} copies, scaled linearly to {dcopies}"
print(json.dumps(line), flush=True)
