"""A/B of round-kernel variants on one C2 proof (profiled: per-launch CUDA
events around the round kernels). Usage: ab_round.py [cfg] [tma_min ...].
Prints per setting: round / bookkeeping / evaluate kernel ms per proof and
the proof's transcript state (must agree across settings). Not a bench."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from paper_2404_10404_b200._lib import check, lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
# settings: integers (tma_min_pairs) or knob=value
settings = [x if "=" in x else int(x) for x in sys.argv[2:]] or [0, 1 << 14]
n_copies, lw, depth = {"c2": (64, 16, 24), "c1": (1, 12, 16), "small": (4, 12, 4)}[cfg]
ctx = P.Context(0)
f = P.Field.bn254()
insz, flat = W.layered_circuit(20240410, lw, depth)
circ = P.Circuit(ctx, insz, *flat, n_copies=n_copies)
inputs = W.random_inputs(f.p, insz * n_copies, 7)
check(lib().dgkr_circuit_load_inputs(ctx.handle, circ.handle, f.handle, inputs.ctypes.data_as(C.c_void_p)))
cap = circ.proof_bound(f)
buf = C.create_string_buffer(cap)
ln = C.c_size_t()
states = set()
for tma in settings:
    if isinstance(tma, str):
        knob, val = tma.split("=")
        P.set_tuning(knob, int(val))
    else:
        P.set_tuning("tma_min_pairs", tma)
    for prof in (False, True, True):
        ctx.set_profile(prof)
        tr = P.Transcript(f, "dgkr.bench.c2")
        check(lib().dgkr_gkr_prove_resident(ctx.handle, circ.handle, f.handle, C.byref(tr.t), buf, C.c_size_t(cap),
                                            C.byref(ln)))
    pr = ctx.profile()
    states.add(tr.state.hex())
    print(json.dumps({"cfg": cfg, "setting": tma, "round_ms": pr["round_ms"], "bookkeep_ms": pr["bookkeep_ms"],
                      "evaluate_ms": pr["evaluate_ms"], "total_ms": pr["total_ms"],
                      "round_GBps": pr["round_bytes"] / pr["round_ms"] / 1e6, "state": tr.state.hex()[:16]}),
          flush=True)
print("states agree:", len(states) == 1)
