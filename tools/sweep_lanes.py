"""Throughput vs concurrent proofs (lanes) for a config. Exploration tool."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
lanes_list = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
n_copies, lw, depth = {"c2": (64, 16, 24), "c1": (1, 12, 16)}[cfg]
ctx = P.Context(0)
f = P.Field.bn254()
insz, flat = W.layered_circuit(20240410, lw, depth)
circ = P.Circuit(ctx, insz, *flat, n_copies=n_copies)
inputs = W.random_inputs(f.p, insz * n_copies, 7)
gates = circ.n_gates
for L in lanes_list:
    for i in range(L):
        P.load_inputs_lane(ctx, circ, f, i, inputs)
    P.gkr_prove_batch(ctx, circ, None, [P.Transcript(f, "x") for _ in range(L)])
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        P.gkr_prove_batch(ctx, circ, None, [P.Transcript(f, "x") for _ in range(L)])
        ts.append(time.perf_counter() - t0)
    dt = min(ts)
    print(f"lanes={L} batch {dt*1e3:.1f} ms  -> {L*gates/dt/1e6:.1f} Mgates/s  (per-proof {dt*1e3/L:.1f} ms)", flush=True)
