"""Bottleneck diagnosis for the C2 proof stream (NOT a bench; proofs made
with DGKR_DIAG_SKIP_OUTPUT_ABSORB=1 are not the reference's). Runs the bench's
stream (resident inputs, `lanes` lanes, n proofs) and prints proofs/s and
gates/s, so runs with and without the skip show whether the host output
absorb or the GPU bounds the stream. Usage: diag_stream.py lanes n_proofs."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from paper_2404_10404_b200._lib import Transcript_t, check, lib  # noqa: E402

lanes, n = int(sys.argv[1]), int(sys.argv[2])
ctx = P.Context(0)
f = P.Field.bn254()
insz, flat = W.layered_circuit(20240410, 16, 24)
circ = P.Circuit(ctx, insz, *flat, n_copies=64)
inputs = W.random_inputs(f.p, insz * 64, 7)
for i in range(lanes):
    P.load_inputs_lane(ctx, circ, f, i, inputs)
cap = circ.proof_bound(f)
bufs = [np.empty(cap, dtype=np.uint8) for _ in range(n)]


def run(k):
    tarr = (Transcript_t * k)()
    for i in range(k):
        tarr[i] = P.Transcript(f, "diag").t
    outs = (C.c_void_p * k)(*[bufs[i].ctypes.data for i in range(k)])
    caps = (C.c_size_t * k)(*([cap] * k))
    lens = (C.c_size_t * k)()
    t0 = time.perf_counter()
    check(lib().dgkr_gkr_prove_stream(ctx.handle, circ.handle, f.handle, C.c_size_t(k), C.c_size_t(lanes), None, tarr,
                                      outs, caps, lens, None))
    return time.perf_counter() - t0


run(lanes)
t = run(n)
print({"lanes": lanes, "proofs": n, "skip_absorb": os.environ.get("DGKR_DIAG_SKIP_OUTPUT_ABSORB") == "1",
       "spin_us": os.environ.get("DGKR_SPIN_US"), "proofs_per_s": round(n / t, 2),
       "gates_per_s": n * circ.n_gates / t}, flush=True)
