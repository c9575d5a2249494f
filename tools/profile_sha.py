"""One SHA-256-circuit proof (sha_circuit.py) for ncu launch lists. Not a bench."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import sha_circuit as S  # noqa: E402
from paper_2404_10404_b200._lib import check, lib  # noqa: E402

copies = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = P.Context(0)
f = P.Field.bn254()
insz, flat, L = S.build_compression_circuit()
rng = np.random.default_rng(1)
inputs, _ = S.sha256_witness(f.p, L, insz, rng.integers(0, 1 << 32, (copies, 8), dtype=np.uint64),
                             rng.integers(0, 1 << 32, (copies, 16), dtype=np.uint64))
circ = P.Circuit(ctx, insz, *flat, n_copies=copies)
check(lib().dgkr_circuit_load_inputs(ctx.handle, circ.handle, f.handle, inputs.ctypes.data_as(C.c_void_p)))
cap = circ.proof_bound(f)
buf = C.create_string_buffer(cap)
ln = C.c_size_t()
ctx.set_profile(os.environ.get("DGKR_PROFILE") == "1")
tr = P.Transcript(f, "sha")
check(lib().dgkr_gkr_prove_resident(ctx.handle, circ.handle, f.handle, C.byref(tr.t), buf, C.c_size_t(cap), C.byref(ln)))
print("proof", ln.value, ctx.profile())
