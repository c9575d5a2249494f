"""Config C5 distributed commitment (BASELINE.json configs[4]): DistPc::commit
+ open (cluster.hpp:336-412) of 2^e evaluations split into N worker rows,
K = plan(N) clusters (N=8 -> K=4 x M=2). The K clusters commit and open
concurrently on K lanes (dgkr_distpc_multi); `serial_open_absorb_ms` is what
one cluster's serial transcript absorb of its combined row costs alone, for
comparison with the wall time of all K. Prints one JSON line per size.

usage: python tools/bench_distpc.py [e_min] [e_max] [N]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402

e_min = int(sys.argv[1]) if len(sys.argv) > 1 else 22
e_max = int(sys.argv[2]) if len(sys.argv) > 2 else 26
N = int(sys.argv[3]) if len(sys.argv) > 3 else 8
ctx = P.Context(0)
f = P.Field.bn254()
for e in range(e_min, e_max + 1):
    row_vars = e - (N.bit_length() - 1)
    raw = W.random_inputs(f.p, 1 << e, e)
    rows = [raw[i * (32 << row_vars):(i + 1) * (32 << row_vars)].tobytes() for i in range(N)]
    r = [int.from_bytes(W.random_inputs(f.p, 1, 2000 + k).tobytes(), "little") for k in range(e)]
    P.distpc(ctx, f, rows, r)  # warm-up (lanes, workspaces)
    t0 = time.perf_counter()
    roots, ops, comb, js = P.distpc(ctx, f, rows, r)
    t = time.perf_counter() - t0
    K = len(roots)
    # one cluster's open transcript absorb alone (its combined row: 2^(e - log2 K) elements)
    cols = 1 << (e - (K.bit_length() - 1))
    tr = P.Transcript(f, "x")
    comb_row = W.random_inputs(f.p, cols, 1)
    t0 = time.perf_counter()
    tr.absorb_elems(comb_row.tobytes())
    t_abs = time.perf_counter() - t0
    print(json.dumps({"config": f"C5 DistPc 2^{e} evaluations, N={N} rows, K={K} clusters", "commit_open_ms": 1e3 * t,
                      "serial_open_absorb_ms_one_cluster": 1e3 * t_abs,
                      "serial_open_absorb_ms_all_clusters": 1e3 * t_abs * K,
                      "opening_bytes": sum(len(o) for o in ops)}),
          flush=True)
