"""Steady-state throughput of a proof stream vs lanes (exploration tool)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
lanes_list = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,8,12,16").split(",")]
per_lane = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n_copies, lw, depth = {"c2": (64, 16, 24), "c1": (1, 12, 16)}[cfg]
ctx = P.Context(0); f = P.Field.bn254()
insz, flat = W.layered_circuit(20240410, lw, depth)
circ = P.Circuit(ctx, insz, *flat, n_copies=n_copies)
inputs = W.random_inputs(f.p, insz * n_copies, 7)
for L in lanes_list:
    for i in range(L):
        P.load_inputs_lane(ctx, circ, f, i, inputs)
    P.gkr_prove_stream(ctx, circ, L, L, f)
    n = L * per_lane
    t0 = time.perf_counter()
    proofs, states, profs = P.gkr_prove_stream(ctx, circ, n, L, f)
    dt = time.perf_counter() - t0
    assert len(set(states)) == 1
    print(f"lanes={L} n={n}: {dt*1e3:.0f} ms -> {n*circ.n_gates/dt/1e6:.1f} Mgates/s ({dt*1e3/n:.1f} ms/proof)", flush=True)
