"""One rank of a shared-memory distributed proof on the local GPU (used by
tests/test_gpu_dist_shm.py: two processes share one GPU; they exchange only
through host shared memory, never by kernels waiting on each other)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from paper_2404_10404_b200.dist import ShmComm, prove_dist_stream, slot_bytes_for  # noqa: E402

rank, world, token, lanes, n, out = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]),
                                     int(sys.argv[5]), sys.argv[6])
spread = (len(sys.argv) > 7 and sys.argv[7] == "spread") or os.environ.get("DGKR_STRESS_SPREAD") == "1"
n_total = int(os.environ.get("DGKR_STRESS_COPIES", "8"))
ctx = P.Context(0)
f = P.Field.bn254()
insz, flat = W.layered_circuit(seed=51, log_width=int(os.environ.get("DGKR_STRESS_LW", "8")),
                               depth=int(os.environ.get("DGKR_STRESS_DEPTH", "5")))
circ = P.Circuit(ctx, insz, *flat, n_copies=n_total // world)
inputs = W.random_inputs(f.p, insz * n_total, 52)
per = insz * (n_total // world) * f.width
mine = np.ascontiguousarray(inputs[rank * per:(rank + 1) * per])
# 4 KiB slots: the claimed-output gather (32 KiB per rank) runs chunked
comms = [ShmComm(ctx, f"/dgkr_{token}_{l}", rank, world, slot_bytes_for(circ, f, cap=4096)) for l in range(lanes)]
for l in range(lanes):
    P.load_inputs_lane(ctx, circ, f, l, mine)
proofs, states, _ = prove_dist_stream(ctx, comms, circ, f, n, "shm", spread_absorb=spread)
if os.environ.get("DGKR_STRESS_LW"):
    print("rank", rank, "ok", len(set(states)) == 1)
    sys.exit(0)
if rank == 0 or spread:
    with open(out + (f".{rank}" if spread else ""), "wb") as fh:
        for p_, s in zip(proofs, states):
            fh.write(len(p_).to_bytes(8, "little") + bytes(p_) + s)
print("rank", rank, "ok")
