"""§8(f) rank 2 / config C3 in-circuit: SHA-256 compressions proved as a
data-parallel GKR circuit (sha_circuit.py; one compression per copy, depth 4,
or 5 with --rlc). Merkle paths of depth 56 over 64-byte nodes (114
compressions per path incl. the leaf), padded to a power-of-two copy count.

Per batch: GPU proof time (median of 3, inputs resident), gates/s and
compressions/s, the kernel / transcript breakdown, and the compiled
reference's gkr_prove on a 2-copy sample (per compression). --rlc folds each
copy's constraints into one output (sum R_i c_i), so the reference
transcript's serial absorb covers 1 output per compression instead of 8,192.
--stream L: steady-state throughput of 2L proofs of the largest batch of at
most 1,024 copies over L lanes. C3 (4,096 validators x depth 56 = 466,944 compressions) is reported as
the time at the measured compressions/s.

usage: python tools/bench_sha_circuit.py [--rlc] [--stream L] [paths ...]"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import sha_circuit as S  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from paper_2404_10404_b200._lib import check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("paths", nargs="*", type=int, default=[1, 8, 32])
ap.add_argument("--rlc", action="store_true")
ap.add_argument("--stream", type=int, default=0)
ap.add_argument("--commit", action="store_true",
                help="also time prove_compressions_rlc (witness commit, R_i draw, proof) per batch")
args = ap.parse_args()

ctx = P.Context(0)
f = P.Field.bn254()
insz, flat, L = S.build_compression_circuit(rlc=args.rlc)
coeffs = S.rlc_coefficients(f.p, b"bench.sha", len(L.rlc)) if args.rlc else None
gates_per_copy = int(flat[0][-1])
depth = 56
C3_COMPRESSIONS = 4096 * (2 + 2 * depth) // 2  # 4,096 paths x 114 compressions
rng = np.random.default_rng(56)
ref_per_comp = None
last = None
for n_paths in args.paths:
    hs, bs = [], []
    for _ in range(n_paths):
        leaf = bytes(rng.integers(0, 256, 64, dtype=np.uint8))
        sibs = [bytes(rng.integers(0, 256, 32, dtype=np.uint8)) for _ in range(depth)]
        h, b, _ = S.merkle_path_compressions(leaf, sibs, int(rng.integers(0, 1 << 40)))
        hs.append(h)
        bs.append(b)
    h_in, blocks = np.concatenate(hs), np.concatenate(bs)
    comps = len(h_in)
    copies = 1
    while copies < comps:
        copies *= 2
    h_in = np.concatenate([h_in, np.tile(S.IV, (copies - comps, 1))])
    blocks = np.concatenate([blocks, np.zeros((copies - comps, 16), np.uint64)])
    t0 = time.perf_counter()
    inputs, _ = S.sha256_witness(f.p, L, insz, h_in, blocks, rlc=coeffs)
    t_wit = time.perf_counter() - t0
    circ = P.Circuit(ctx, insz, *flat, n_copies=copies)
    check(lib().dgkr_circuit_load_inputs(ctx.handle, circ.handle, f.handle, inputs.ctypes.data_as(C.c_void_p)))
    cap = circ.proof_bound(f)
    buf = C.create_string_buffer(cap)
    ln = C.c_size_t()
    ts = []
    for _ in range(4):
        tr = P.Transcript(f, "sha.c3")
        t0 = time.perf_counter()
        check(lib().dgkr_gkr_prove_resident(ctx.handle, circ.handle, f.handle, C.byref(tr.t), buf, C.c_size_t(cap),
                                            C.byref(ln)))
        ts.append(time.perf_counter() - t0)
    dt = statistics.median(ts[1:])
    proof = buf.raw[: ln.value]
    n_out = int.from_bytes(proof[:4], "little")
    assert not any(proof[4:4 + 32 * n_out])  # all constraints zero
    ctx.set_profile(True)
    tr = P.Transcript(f, "sha.c3")
    check(lib().dgkr_gkr_prove_resident(ctx.handle, circ.handle, f.handle, C.byref(tr.t), buf, C.c_size_t(cap),
                                        C.byref(ln)))
    prof = ctx.profile()
    ctx.set_profile(False)
    gates = copies * gates_per_copy
    line = {"config": f"SHA-256 in circuit{' (rlc)' if args.rlc else ''}: {n_paths} Merkle path(s) x depth {depth}"
                      f" = {comps} compressions ({copies} copies)", "gates": gates, "outputs": n_out,
            "gpu_prove_ms": 1e3 * dt, "gates_per_s": gates / dt, "compressions_per_s": comps / dt,
            "c3_4096_validators_s_at_this_rate": C3_COMPRESSIONS / (comps / dt), "witness_gen_s": t_wit,
            "breakdown_ms": {k: prof[k] for k in ("round_ms", "bookkeep_ms", "evaluate_ms", "host_transcript_ms",
                                                  "output_absorb_ms")}}
    if ref_per_comp is None:
        try:
            from oracle import dgkr_oracle as O
            from oracle import refbind as R
            if R.available():
                fi, ff = W.replicate(insz, flat, 2)
                oc = O.Circuit.from_flat(fi, *ff)
                ins = O.BN254.elems_from_bytes(inputs[: 2 * insz * 32].tobytes())
                t0 = time.perf_counter()
                R.gkr_prove(O.BN254, "sha.c3", [], oc, ins, flat=ff)
                ref_per_comp = (time.perf_counter() - t0) / 2
        except Exception as e:  # reported, not required
            line["ref_error"] = str(e)
    if ref_per_comp:
        line["ref_s_per_compression"] = ref_per_comp
        line["ref_compressions_per_s"] = 1 / ref_per_comp
        line["ref_note"] = "compiled reference gkr_prove on 2 copies, single thread"
    print(json.dumps(line), flush=True)
    if args.commit:
        built, ts = None, []
        for _ in range(3):
            t0 = time.perf_counter()
            pr, built = S.prove_compressions_rlc(ctx, f, h_in[:comps], blocks[:comps], built=built)
            ts.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        S._witness_root(ctx, f, pr.inputs)
        t_commit = time.perf_counter() - t0
        ok = S.verify_compressions_rlc(ctx, f, built, pr.inputs, pr.root, pr.proof)
        dt_c = statistics.median(ts[1:])
        print(json.dumps({"config": f"committed-witness rlc proof: {comps} compressions ({copies} copies)",
                          "total_ms": 1e3 * dt_c, "commit_ms": 1e3 * t_commit,
                          "compressions_per_s": comps / dt_c, "verifier_accepts": ok,
                          "note": "witness generation + pcs_commit of the input layer + R_i draw + gkr_prove"}),
              flush=True)
    if copies <= 1024:  # per-lane workspace of larger batches is tens of GB
        last = (circ, inputs, comps, copies, gates)

if args.stream and last:
    circ, inputs, comps, copies, gates = last
    lanes = args.stream
    for lane in range(lanes):
        P.load_inputs_lane(ctx, circ, f, lane, inputs)
    P.gkr_prove_stream(ctx, circ, lanes, lanes, f)  # warm-up
    n = 2 * lanes
    t0 = time.perf_counter()
    P.gkr_prove_stream(ctx, circ, n, lanes, f)
    dt = time.perf_counter() - t0
    print(json.dumps({"config": f"SHA-256 in circuit{' (rlc)' if args.rlc else ''}: stream of {n} proofs x {comps} "
                                f"compressions over {lanes} lanes", "compressions_per_s": n * comps / dt,
                      "gates_per_s": n * gates / dt,
                      "c3_4096_validators_s_at_this_rate": C3_COMPRESSIONS / (n * comps / dt)}), flush=True)
