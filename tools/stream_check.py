"""Stream determinism check: L proofs over L lanes (resident inputs) must each
equal the single proof of the same inputs. Usage:
  stream_check.py cfg lanes [tma_min_pairs] [same|distinct]
distinct: every lane proves different inputs (exposes cross-lane mixing)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402

cfg, lanes = sys.argv[1], int(sys.argv[2])
if len(sys.argv) > 3 and sys.argv[3] != "-":
    P.set_tuning("tma_min_pairs", int(sys.argv[3]))
mode = sys.argv[4] if len(sys.argv) > 4 else "same"
n_copies, lw, depth = {"c2": (64, 16, 24), "c2q": (16, 16, 6), "small": (4, 12, 4)}[cfg]
ctx = P.Context(0)
f = P.Field.bn254()
insz, flat = W.layered_circuit(20240410, lw, depth)
circ = P.Circuit(ctx, insz, *flat, n_copies=n_copies)
ins = [W.random_inputs(f.p, insz * n_copies, 7 + (i if mode == "distinct" else 0)) for i in range(lanes)]
singles = {}
for i in range(lanes if mode == "distinct" else 1):
    tr = P.Transcript(f, "chk")
    singles[i] = P.gkr_prove(ctx, circ, ins[i], tr)
for i in range(lanes):
    P.load_inputs_lane(ctx, circ, f, i, ins[i])
trs = [P.Transcript(f, "chk") for _ in range(lanes)]
proofs = P.gkr_prove_batch(ctx, circ, None, trs)
bad = [i for i, p in enumerate(proofs) if p != singles[i if mode == "distinct" else 0]]
print(f"{cfg} {mode} lanes={lanes} tma_min={P.get_tuning('tma_min_pairs')}: {len(bad)} of {lanes} differ", bad[:8],
      flush=True)
if bad:
    p, s = proofs[bad[0]], singles[bad[0] if mode == "distinct" else 0]
    k = next(j for j in range(len(p)) if p[j] != s[j])
    print("first differing byte", k, "of", len(p))
