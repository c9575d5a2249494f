"""Config C5 distributed commitment (BASELINE.json configs[4]): DistPc::commit
+ open (cluster.hpp:336-412) of 2^e evaluations split into N worker rows,
K = plan(N) clusters (N=8 -> K=4 x M=2). The K clusters commit and open
concurrently on K lanes (dgkr_distpc_multi). Timed: the C call alone, inputs
and output buffers prepared in host memory beforehand.
`serial_open_absorb_ms_one_cluster` is one cluster's serial transcript absorb
of its combined row alone (pcs.hpp:199-206), the floor of the open.
Prints one JSON line per size.

usage: python tools/bench_distpc.py [e_min] [e_max] [N]"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from paper_2404_10404_b200._lib import check, lib  # noqa: E402

e_min = int(sys.argv[1]) if len(sys.argv) > 1 else 22
e_max = int(sys.argv[2]) if len(sys.argv) > 2 else 26
N = int(sys.argv[3]) if len(sys.argv) > 3 else 8
ctx = P.Context(0)
f = P.Field.bn254()
for e in range(e_min, e_max + 1):
    row_vars = e - (N.bit_length() - 1)
    data = W.random_inputs(f.p, 1 << e, e)
    r = np.frombuffer(W.random_inputs(f.p, e, 2000 + e).tobytes(), np.uint8)
    K = {1: 1, 2: 1, 4: 2, 8: 4, 16: 4, 32: 8, 64: 8}[N]
    M = N // K
    cols = 1 << row_vars
    osz = 4 + (e + 2 + M + cols) * 32 + 4 * 3 + min(32, cols) * (4 + M * 32 + 32 * row_vars) + 64
    out = np.empty(K * (4 + osz), np.uint8)
    roots = np.empty(32 * N, np.uint8)
    comb = np.empty(32, np.uint8)
    js = C.create_string_buffer(8192)
    nr, ln = C.c_size_t(), C.c_size_t()

    def call():
        check(lib().dgkr_distpc(ctx.handle, f.handle, C.c_size_t(N), C.c_size_t(0), C.c_size_t(row_vars),
                                data.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p), C.c_size_t(e),
                                C.c_size_t(32), roots.ctypes.data_as(C.c_void_p), C.byref(nr),
                                out.ctypes.data_as(C.c_void_p), C.c_size_t(out.size), C.byref(ln),
                                comb.ctypes.data_as(C.c_void_p), js, C.c_size_t(8192)))

    call()  # warm-up (lanes, workspaces, pages)
    t0 = time.perf_counter()
    call()
    t = time.perf_counter() - t0
    assert nr.value == K
    tr = P.Transcript(f, "x")
    row = W.random_inputs(f.p, cols, 1)
    t0 = time.perf_counter()
    tr.absorb_elems(row.tobytes())
    t_abs = time.perf_counter() - t0
    print(json.dumps({"config": f"C5 DistPc 2^{e} evaluations, N={N} rows, K={K} clusters x M={M}",
                      "commit_open_ms": 1e3 * t, "serial_open_absorb_ms_one_cluster": 1e3 * t_abs,
                      "serial_open_absorb_ms_all_clusters": 1e3 * t_abs * K, "opening_bytes": ln.value}), flush=True)
