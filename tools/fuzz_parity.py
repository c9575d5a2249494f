"""Differential fuzz: GPU gkr_prove vs the compiled reference (oracle/_ref),
byte for byte, over three families (a GPU box with oracle/_ref built):
  * general circuits from the reference's own generator (BN254);
  * data-parallel layered circuits of 2^13..2^17 gates per layer, so the BN254
    constant-multiplier chi expansion (k_split_eq_expand_const, klo >= 8) and
    the lazy-difference round kernels run at size;
  * general circuits over the runtime-modulus path (p = 97, Goldilocks).
usage: python tools/fuzz_parity.py [general_cases] [layered_cases] [seconds]
Prints one line per family and exits 1 on any mismatch."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2404_10404_b200 as P  # noqa: E402
from oracle import dgkr_oracle as O  # noqa: E402
from oracle import refbind as R  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402

n_general = int(sys.argv[1]) if len(sys.argv) > 1 else 300
n_layered = int(sys.argv[2]) if len(sys.argv) > 2 else 16
budget = float(sys.argv[3]) if len(sys.argv) > 3 else 900.0
if not R.available():
    raise SystemExit("oracle/_ref is not built")
ctx = P.Context(0)
t_end = time.time() + budget
bad = 0


def general(fld, cases, tag):
    global bad
    f = P.Field(fld.p)
    rng = np.random.default_rng(fld.p % 100003)
    done = 0
    for seed in range(cases):
        if time.time() > t_end:
            break
        insz, depth = 5 + seed % 8, 2 + seed % 4
        c = R.random_general_circuit(7000 + seed, insz, depth, 24, 3)
        inputs = O.random_elements(fld, insz, rng)
        want, _ = R.gkr_prove(fld, tag, [seed], c, inputs)
        got = P.gkr_prove(ctx, P.Circuit.from_oracle(ctx, c), inputs, P.Transcript(f, tag, [seed]))
        if got != want:
            bad += 1
            print(f"MISMATCH {tag} p={fld.p} seed {seed}", flush=True)
        done += 1
    print(f"{tag} p={fld.p}: {done} circuits, mismatches so far {bad}", flush=True)


def layered(cases):
    global bad
    fld = O.BN254
    f = P.Field(fld.p)
    rng = np.random.default_rng(5)
    done = 0
    for k in range(cases):
        if time.time() > t_end:
            break
        lw = int(rng.integers(6, 13))
        # 2^13..2^17 gates per layer in total: from 2^15 on the split-eq row
        # factor spans >= 256 outputs (the constant-multiplier path)
        total_log = int(rng.integers(13, 18))
        copies = 1 << max(0, total_log - lw)
        depth = int(rng.integers(2, 4))
        insz, flat = W.layered_circuit(900 + k, lw, depth)
        inputs = W.random_inputs(fld.p, insz * copies, 40 + k)
        full_in, full_flat = W.replicate(insz, flat, copies)
        oc = O.Circuit.from_flat(full_in, *full_flat)
        want, _ = R.gkr_prove(fld, "fz", [k], oc, fld.elems_from_bytes(inputs.tobytes()), flat=full_flat)
        got = P.gkr_prove(ctx, P.Circuit(ctx, insz, *flat, n_copies=copies), inputs, P.Transcript(f, "fz", [k]))
        if got != want:
            bad += 1
            print(f"MISMATCH layered k={k} lw={lw} copies={copies} depth={depth}", flush=True)
        done += 1
    print(f"layered BN254 (2^13..2^17 gates/layer): {done} circuits, mismatches so far {bad}", flush=True)


general(O.BN254, n_general, "gen")
layered(n_layered)
general(O.Field(O.GOLDILOCKS_P), n_general // 3, "gen")
general(O.Field(97), n_general // 3, "gen")
print("total mismatches", bad)
sys.exit(1 if bad else 0)
