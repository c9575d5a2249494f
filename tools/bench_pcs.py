"""Config C5 sweep (BASELINE.json configs[4]): polynomial commitment over 2^e
evaluations — pcs::commit (column SHA-256 + Merkle, pcs.hpp:105) and
pcs::open (row evals, beta-combined row, serial transcript absorb of the
combined row, spot paths; pcs.hpp:212) — on the GPU, with the compiled
reference timed at the smaller sizes. Prints one JSON line per size.

usage: python tools/bench_pcs.py [e_min] [e_max] [ref_max_e]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402

e_min = int(sys.argv[1]) if len(sys.argv) > 1 else 20
e_max = int(sys.argv[2]) if len(sys.argv) > 2 else 24
ref_max = int(sys.argv[3]) if len(sys.argv) > 3 else 20
ctx = P.Context(0)
f = P.Field.bn254()
for e in range(e_min, e_max + 1):
    cols = 1 << e
    data = W.random_inputs(f.p, cols, e).tobytes()
    root = P.pcs_commit(ctx, f, [data])  # warm-up
    t0 = time.perf_counter()
    root = P.pcs_commit(ctx, f, [data])
    t_commit = time.perf_counter() - t0
    r = [int.from_bytes(W.random_inputs(f.p, 1, 1000 + k).tobytes(), "little") for k in range(e)]
    P.pcs_open(ctx, f, [data], r, P.Transcript(f, "dgkr.pc.cluster", [0]), 32)  # warm-up (workspace, pages)
    tr = P.Transcript(f, "dgkr.pc.cluster", [0])
    t0 = time.perf_counter()
    op = P.pcs_open(ctx, f, [data], r, tr, 32)
    t_open = time.perf_counter() - t0
    prof = ctx.profile()
    compressions = 2 * cols - 1  # one per 32-byte column leaf + two per inner node (leaf: 1 block)
    line = {"config": f"C5 pcs M=1 cols=2^{e}", "commit_ms": 1e3 * t_commit, "open_ms": 1e3 * t_open,
            "open_host_transcript_ms": prof["host_transcript_ms"], "commit_compressions": cols + 2 * (cols - 1),
            "commit_compressions_per_s": (cols + 2 * (cols - 1)) / t_commit, "root": root.hex()[:16],
            "opening_bytes": len(op)}
    if e <= ref_max:
        from oracle import refbind as R
        from oracle import dgkr_oracle as O

        if R.available():
            rows = [O.BN254.elems_from_bytes(data)]
            t0 = time.perf_counter()
            rroot = R.pcs_commit(O.BN254, rows)
            line["ref_commit_ms"] = 1e3 * (time.perf_counter() - t0)
            t0 = time.perf_counter()
            rop, rst = R.pcs_open(O.BN254, "dgkr.pc.cluster", [0], rows, r, 32)
            line["ref_open_ms"] = 1e3 * (time.perf_counter() - t0)
            line["bit_exact"] = bool(rroot == root and rop == op and rst == tr.state)
    print(json.dumps(line), flush=True)
