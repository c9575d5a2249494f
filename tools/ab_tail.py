"""A/B of the sum-check tail: one launch per round vs the mailbox tail kernel
(tuning "tail_pairs"). Single-proof latency (median of 15, unprofiled) of
C1 and C2 and the proof's transcript state, which must agree across
settings. Usage: ab_tail.py [tail_pairs ...]. Not a bench."""
import ctypes as C
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from paper_2404_10404_b200._lib import check, lib  # noqa: E402

settings = [int(x) for x in sys.argv[1:]] or [0, 256]
ctx = P.Context(0)
f = P.Field.bn254()
for cfg, (n_copies, lw, depth) in {"c1": (1, 12, 16), "c2": (64, 16, 24)}.items():
    insz, flat = W.layered_circuit(20240410, lw, depth)
    circ = P.Circuit(ctx, insz, *flat, n_copies=n_copies)
    inputs = W.random_inputs(f.p, insz * n_copies, 7)
    check(lib().dgkr_circuit_load_inputs(ctx.handle, circ.handle, f.handle, inputs.ctypes.data_as(C.c_void_p)))
    cap = circ.proof_bound(f)
    buf = C.create_string_buffer(cap)
    ln = C.c_size_t()
    states = set()
    for tp in settings:
        P.set_tuning("tail_pairs", tp)
        ts = []
        for it in range(18):
            tr = P.Transcript(f, "dgkr.ab.tail")
            t0 = time.perf_counter()
            check(lib().dgkr_gkr_prove_resident(ctx.handle, circ.handle, f.handle, C.byref(tr.t), buf,
                                                C.c_size_t(cap), C.byref(ln)))
            if it >= 3:
                ts.append(time.perf_counter() - t0)
        states.add((tr.state.hex(), bytes(buf[:ln.value])))
        print(json.dumps({"cfg": cfg, "tail_pairs": tp, "latency_ms_median": 1e3 * statistics.median(ts),
                          "latency_ms_min": 1e3 * min(ts), "state": tr.state.hex()[:16]}), flush=True)
    print(json.dumps({"cfg": cfg, "proofs_agree": len(states) == 1}), flush=True)
