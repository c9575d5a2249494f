"""Config C5 (BASELINE.json configs[4]) for the Virgo/FRI path: RS-encode
(NTT) + per-layer Merkle + FRI folds over 2^e codeword evaluations, blowup 2,
on one GPU. Reports wall time of dgkr_fri_prove, the serial host transcript
share, and NTT throughput. Prints one JSON line per size."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402

e_min = int(sys.argv[1]) if len(sys.argv) > 1 else 20
e_max = int(sys.argv[2]) if len(sys.argv) > 2 else 26
ctx = P.Context(0)
f = P.Field.bn254()
for e in range(e_min, e_max + 1):
    blowup = 1
    n = 1 << (e - blowup)
    co = W.random_inputs(f.p, n, e)
    P.fri_prove(ctx, f, co, blowup, 4, 32, P.Transcript(f, "fri"))
    t0 = time.perf_counter()
    pr = P.fri_prove(ctx, f, co, blowup, 4, 32, P.Transcript(f, "fri"))
    dt = time.perf_counter() - t0
    prof = ctx.profile()
    data = W.random_inputs(f.p, 1 << e, e + 100)
    P.ntt(ctx, f, data)
    t0 = time.perf_counter()
    P.ntt(ctx, f, data)
    t_ntt = time.perf_counter() - t0
    butterflies = (1 << e) // 2 * e
    print(json.dumps({"config": f"C5 FRI codeword 2^{e} (n=2^{e - blowup}, blowup 2^{blowup})",
                      "fri_prove_ms": 1e3 * dt, "host_transcript_ms": prof["host_transcript_ms"],
                      "gpu_launches": prof["launches"], "proof_bytes": len(pr),
                      "ntt_ms_incl_transfers": 1e3 * t_ntt, "ntt_butterflies": butterflies}), flush=True)
