"""Config C3: native beacon membership paths on one GPU.
BeaconTree of depth 56 over N validators (a = log2 N); verify_membership of
every validator's path = 1 leaf digest + 56 concat hashes = 114 SHA-256
compressions per path. Reports compressions/s (kernel time from CUDA events,
and end to end through the C ABI with host buffers), beside the compiled
reference (oracle/_ref, single thread) on a bounded sample of paths."""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from oracle import refbind as R  # noqa: E402

depth = 56
ctx = P.Context(0)
HERE = os.path.join(ROOT, "tests", "golden")
for n in [int(x) for x in (sys.argv[1:] or ["4096", "1048576"])]:
    if n == 4096 and os.path.exists(os.path.join(HERE, "beacon_4096.bin")):
        recs = open(os.path.join(HERE, "beacon_4096.bin"), "rb").read()
        src = "reference gen_validators(4096, seed 4) (tests/golden/beacon_4096.bin)"
    else:
        rng = np.random.default_rng(n)
        r = np.zeros((n, 64), dtype=np.uint8)
        r[:, :48] = rng.integers(0, 256, (n, 48), dtype=np.uint8)
        r[:, 48:56] = np.arange(n, dtype=np.uint64).view(np.uint8).reshape(n, 8)
        r[:, 56] = 1
        recs = r.tobytes()
        src = "synthetic records (random pubkeys, dense indexes, active)"
    idx = np.arange(n, dtype=np.uint64)
    t0 = time.perf_counter()
    root = P.beacon_root(ctx, recs, depth)
    t_root = time.perf_counter() - t0
    L, S, a = P.beacon_prove(ctx, recs, depth, idx)
    P.beacon_verify(ctx, root, recs, L, S, idx, depth, a)  # warm-up
    walls, kers = [], []
    for _ in range(5):
        ctx.set_profile(True)
        t0 = time.perf_counter()
        ok = P.beacon_verify(ctx, root, recs, L, S, idx, depth, a)
        walls.append(time.perf_counter() - t0)
        kers.append(ctx.profile()["merkle_ms"] * 1e-3)
        ctx.set_profile(False)
    assert ok.all()
    comp = n * (2 + 2 * depth)
    line = {"config": f"C3 native: verify_membership of {n} paths, depth {depth} (a={a})", "records": src,
            "compressions": comp, "gpu_kernel_ms": 1e3 * statistics.median(kers),
            "gpu_compressions_per_s": comp / statistics.median(kers),
            "e2e_ms": 1e3 * statistics.median(walls), "e2e_compressions_per_s": comp / statistics.median(walls),
            "root_build_ms_incl_transfers": 1e3 * t_root}
    if R.available():
        sample = min(n, 512)
        t0 = time.perf_counter()
        for i in range(sample):
            assert R.beacon_verify(root, recs[64 * i:64 * (i + 1)], L[32 * i:32 * (i + 1)],
                                   S[32 * a * i:32 * a * (i + 1)], a, i, depth)
        dt = time.perf_counter() - t0
        line["ref_compressions_per_s"] = sample * (2 + 2 * depth) / dt
        line["ref_sample"] = f"{sample} paths, single thread, per-path ctypes call"
    print(json.dumps(line), flush=True)
