"""Config C5 at N ranks (BASELINE.json configs[4], "1/2/4/8 GPUs"): the
distributed FRI (dgkr_fri_prove_dist) of one 2^e codeword (n = 2^(e-1)
coefficients, blowup 2) split into N rank chunks of n/N coefficients, shared
Fiat-Shamir. This box has one GPU, so per N it reports
  * rank_alone_ms: fri_prove of one n/N chunk alone on the GPU (what each of N
    GPUs computes; wall time from host bytes, median of 3);
  * emulated_ms: dgkr_fri_prove_dist_emulated with all N ranks as threads on
    lanes of this one GPU (the whole protocol incl. the L+1 all-gathers; the
    ranks share one GPU, so this is not an N-GPU time);
  * collective_bytes_per_rank: what one rank contributes to the all-gathers
    (L roots x 32 B + the final layer).
Prints one JSON line per N."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402

e = int(sys.argv[1]) if len(sys.argv) > 1 else 24
worlds = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
blowup, final, q = 1, 4, 32
ctx = P.Context(0)
f = P.Field.bn254()
n = 1 << (e - blowup)


def med(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * statistics.median(ts)


for world in worlds:
    m = n // world
    chunks = [W.random_inputs(f.p, m, 300 + r).tobytes() for r in range(world)]
    alone = med(lambda: P.fri_prove(ctx, f, chunks[0], blowup, final, q, P.Transcript(f, "fri")))
    emu = med(lambda: P.fri_prove_dist_emulated(ctx, f, chunks, blowup, final, q, P.Transcript(f, "fri.d")))
    prs = P.fri_prove_dist_emulated(ctx, f, chunks, blowup, final, q, P.Transcript(f, "fri.d"))
    L = (m.bit_length() - 1 + blowup) - final
    print(json.dumps({"config": f"C5 distributed FRI: codeword 2^{e} (n=2^{e - blowup}, blowup 2) over {world} ranks",
                      "ranks": world, "rank_chunk_coeffs": m, "rank_alone_ms": alone, "emulated_ms": emu,
                      "allgathers": L + 1, "collective_bytes_per_rank": L * 32 + (1 << final) * f.width,
                      "proof_bytes_per_rank": len(prs[0])}), flush=True)
