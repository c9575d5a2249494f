"""Search reference-generated general circuits for GPU/reference mismatches."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2404_10404_b200 as P
from oracle import dgkr_oracle as O, refbind as R
ctx = P.Context(0)
fld = O.BN254; f = P.Field(fld.p)
rng = np.random.default_rng(0)
bad = 0
for seed in range(300):
    insz = 5 + seed % 8; depth = 2 + seed % 4
    c = R.random_general_circuit(1000 + seed, insz, depth, 24, 3)
    inputs = O.random_elements(fld, insz, rng)
    pb, st = R.gkr_prove(fld, "h", [seed], c, inputs)
    dc = P.Circuit.from_oracle(ctx, c)
    tr = P.Transcript(f, "h", [seed])
    got = P.gkr_prove(ctx, dc, inputs, tr)
    if got != pb:
        bad += 1
        sizes = [c.layer_size(l) for l in range(c.depth + 1)]
        slots = [c.source_layers(l) for l in range(1, c.depth + 1)]
        # first differing layer
        print("MISMATCH seed", seed, "sizes", sizes, "slots", slots, "len", len(got), len(pb), flush=True)
        if bad >= 6: break
print("bad", bad)
