"""Config C5 (BASELINE.json configs[4]) for the Virgo/FRI path: RS-encode
(NTT) + per-layer Merkle + FRI folds over 2^e codeword evaluations, blowup 2,
on one GPU. Per size, after one warm-up call (workspace allocation):
  * fri_prove_ms: wall time of dgkr_fri_prove from pageable host bytes
    (includes the H2D of the coefficients and the query gathers);
  * ntt/merkle/fold_ms: CUDA-event kernel time inside that call (profile on);
  * ntt_kernel_ms: dgkr_ntt's bit-reverse + butterfly kernels for a 2^e NTT,
    with butterflies/s and the mont-mul fraction of the measured mul peak.
Prints one JSON line per size."""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from paper_2404_10404_b200._lib import check, lib  # noqa: E402

e_min = int(sys.argv[1]) if len(sys.argv) > 1 else 20
e_max = int(sys.argv[2]) if len(sys.argv) > 2 else 26
ctx = P.Context(0)
f = P.Field.bn254()
_mp = C.c_double()
check(lib().dgkr_bench_mul_peak(ctx.handle, C.byref(_mp)))
peak = _mp.value
for e in range(e_min, e_max + 1):
    blowup = 1
    n = 1 << (e - blowup)
    co = W.random_inputs(f.p, n, e).tobytes()
    P.fri_prove(ctx, f, co, blowup, 4, 32, P.Transcript(f, "fri"))
    ctx.set_profile(True)
    t0 = time.perf_counter()
    pr = P.fri_prove(ctx, f, co, blowup, 4, 32, P.Transcript(f, "fri"))
    dt = time.perf_counter() - t0
    prof = ctx.profile()
    ctx.set_profile(False)
    data = W.random_inputs(f.p, 1 << e, e + 100).tobytes()
    out = C.create_string_buffer(len(data))
    check(lib().dgkr_ntt(ctx.handle, f.handle, C.c_char_p(data), C.c_uint(e), C.c_int(0), out))
    ctx.set_profile(True)
    t0 = time.perf_counter()
    check(lib().dgkr_ntt(ctx.handle, f.handle, C.c_char_p(data), C.c_uint(e), C.c_int(0), out))
    t_ntt = time.perf_counter() - t0
    nprof = ctx.profile()
    ctx.set_profile(False)
    butterflies = (1 << e) // 2 * e
    k_ms = nprof["ntt_ms"]
    line = {"config": f"C5 FRI codeword 2^{e} (n=2^{e - blowup}, blowup 2^{blowup}, final 2^4, 32 queries)",
            "fri_prove_ms": 1e3 * dt, "fri_ntt_ms": prof["ntt_ms"], "fri_merkle_ms": prof["merkle_ms"],
            "fri_fold_ms": prof["fold_ms"], "gpu_launches": prof["launches"], "proof_bytes": len(pr),
            "ntt_call_ms": 1e3 * t_ntt, "ntt_kernel_ms": k_ms, "ntt_butterflies": butterflies,
            "ntt_butterflies_per_s": butterflies / (k_ms * 1e-3) if k_ms else None}
    if peak and k_ms:
        line["ntt_mul_frac_of_peak"] = butterflies / (k_ms * 1e-3) / peak
    print(json.dumps(line), flush=True)
