"""One gkr_prove step of a config (for ncu / launch lists). Not a bench."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from paper_2404_10404_b200._lib import check, lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
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
ctx.set_profile(os.environ.get("DGKR_PROFILE") == "1")
for _ in range(steps):
    tr = P.Transcript(f, "dgkr.bench.c2")
    check(lib().dgkr_gkr_prove_resident(ctx.handle, circ.handle, f.handle, C.byref(tr.t), buf, C.c_size_t(cap),
                                        C.byref(ln)))
mp = C.c_double()
check(lib().dgkr_bench_mul_peak(ctx.handle, C.byref(mp)))
print("proof", ln.value, "state", tr.state.hex()[:16], "mul_peak %.3e" % mp.value, ctx.profile())
