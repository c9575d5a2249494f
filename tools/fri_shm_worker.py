"""One rank of a distributed FRI (dgkr_fri_prove_dist) over the shared-memory
transport on the local GPU (used by tests/test_gpu_fri.py; ranks exchange
roots and final layers only through host shared memory).

usage: fri_shm_worker.py rank world token n blowup_log final_log queries out"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from paper_2404_10404_b200.dist import ShmComm  # noqa: E402

rank, world, token, n, blowup, final, q, out = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]),
                                                int(sys.argv[5]), int(sys.argv[6]), int(sys.argv[7]), sys.argv[8])
ctx = P.Context(0)
f = P.Field.bn254()
comm = ShmComm(ctx, f"/dgkr_fri_{token}", rank, world, 1 << 16)
tr = P.Transcript(f, "fri.shm", [world])
proof = P.fri_prove_dist(ctx, comm, f, W.random_inputs(f.p, n, 100 + rank), blowup, final, q, tr)
with open(f"{out}.{rank}", "wb") as fh:
    fh.write(proof + tr.state)
print("rank", rank, "ok")
