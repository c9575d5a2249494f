"""Evidence for the reference arm's sample: the compiled
reference's gkr_prove (oracle/_ref, single-threaded as the reference is) on
layered circuits of the C2 family at growing width -- 2^14, 2^16, 2^18 gates
per layer x 2 layers, 2^12 x 24, and ONE C2 sub-circuit at full depth
(2^16 x 24) -- so the per-gate cost's growth with s (SURVEY §8(a) a5:
~(3s + 30) mults per gate) and the gap between the 2-layer sample and the
real shape are measured, not assumed. Prints one JSON line per case."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import dgkr_oracle as O  # noqa: E402
from oracle import refbind as R  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402

cases = [(14, 2, 1), (16, 2, 1), (18, 2, 1), (12, 24, 1), (16, 24, 1), (16, 6, 2)]
if len(sys.argv) > 1:
    cases = cases[: int(sys.argv[1])]
for lw, depth, copies in cases:
    insz, flat = W.layered_circuit(20240410, lw, depth)
    full_in, full_flat = W.replicate(insz, flat, copies) if copies > 1 else (insz, flat)
    vals = O.BN254.elems_from_bytes(W.random_inputs(O.BN254_P, full_in, 7).tobytes())
    c = O.Circuit.from_flat(full_in, *full_flat)
    t0 = time.perf_counter()
    R.gkr_prove(O.BN254, "ref.scaling", [], c, vals, flat=full_flat)
    dt = time.perf_counter() - t0
    gates = (1 << lw) * depth * copies
    s = lw + (copies - 1).bit_length()
    print(json.dumps({"case": f"{copies} x 2^{lw} gates/layer x {depth} layers", "s": s, "gates": gates,
                      "seconds": dt, "gates_per_s": gates / dt, "ns_per_gate": 1e9 * dt / gates,
                      "model_mults_per_gate_3s_plus_30": 3 * s + 30}), flush=True)
