"""Differential fuzz: GPU gkr_prove vs the compiled reference (oracle/_ref),
byte for byte, over three families (a GPU box with oracle/_ref built):
  * general circuits from the reference's own generator (BN254);
  * data-parallel layered circuits of 2^13..2^17 gates per layer, so the BN254
    constant-multiplier chi expansion (k_split_eq_expand_const, klo >= 8) and
    the lazy-difference round kernels run at size;
  * general circuits over the runtime-modulus path (p = 97, Goldilocks) and
    the wide path (255- and 256-bit primes);
  * the distributed prover (emulated ranks 2/4/8) against the single proof;
  * pcs commit roots and openings (M rows, random sizes, BN254/Goldilocks);
  every third general circuit runs with a random sum-check tail threshold and
  hand-back timeout (the mailbox tail launch and its fallback).
usage: python tools/fuzz_parity.py [general_cases] [layered_cases] [seconds]
Prints one line per family and exits 1 on any mismatch."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2404_10404_b200 as P  # noqa: E402
from oracle import dgkr_oracle as O  # noqa: E402
from oracle import refbind as R  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402

n_general = int(sys.argv[1]) if len(sys.argv) > 1 else 300
n_layered = int(sys.argv[2]) if len(sys.argv) > 2 else 16
budget = float(sys.argv[3]) if len(sys.argv) > 3 else 900.0
if not R.available():
    raise SystemExit("oracle/_ref is not built")
ctx = P.Context(0)
t_end = time.time() + budget
bad = 0


def general(fld, cases, tag):
    global bad
    f = P.Field(fld.p)
    rng = np.random.default_rng(fld.p % 100003)
    done = 0
    for seed in range(cases):
        if time.time() > t_end:
            break
        insz, depth = 5 + seed % 8, 2 + seed % 4
        c = R.random_general_circuit(7000 + seed, insz, depth, 24, 3)
        inputs = O.random_elements(fld, insz, rng)
        want, _ = R.gkr_prove(fld, tag, [seed], c, inputs)
        # every third circuit: a random tail threshold and hand-back timeout
        # (0-5 us makes the tail launch give up at varying rounds)
        if seed % 3 == 2:
            P.set_tuning("tail_pairs", [0, 1, 4, 256, 1 << 22][seed % 5])
            P.set_tuning("tail_timeout_us", [0, 2, 5, 20000][seed % 4])
        try:
            got = P.gkr_prove(ctx, P.Circuit.from_oracle(ctx, c), inputs, P.Transcript(f, tag, [seed]))
        finally:
            P.set_tuning("tail_pairs", 256)
            P.set_tuning("tail_timeout_us", 20000)
        if got != want:
            bad += 1
            print(f"MISMATCH {tag} p={fld.p} seed {seed}", flush=True)
        done += 1
    print(f"{tag} p={fld.p}: {done} circuits, mismatches so far {bad}", flush=True)


def layered(cases):
    global bad
    fld = O.BN254
    f = P.Field(fld.p)
    rng = np.random.default_rng(5)
    done = 0
    for k in range(cases):
        if time.time() > t_end:
            break
        lw = int(rng.integers(6, 13))
        # 2^13..2^17 gates per layer in total: from 2^15 on the split-eq row
        # factor spans >= 256 outputs (the constant-multiplier path)
        total_log = int(rng.integers(13, 18))
        copies = 1 << max(0, total_log - lw)
        depth = int(rng.integers(2, 4))
        insz, flat = W.layered_circuit(900 + k, lw, depth)
        inputs = W.random_inputs(fld.p, insz * copies, 40 + k)
        full_in, full_flat = W.replicate(insz, flat, copies)
        oc = O.Circuit.from_flat(full_in, *full_flat)
        want, _ = R.gkr_prove(fld, "fz", [k], oc, fld.elems_from_bytes(inputs.tobytes()), flat=full_flat)
        got = P.gkr_prove(ctx, P.Circuit(ctx, insz, *flat, n_copies=copies), inputs, P.Transcript(f, "fz", [k]))
        if got != want:
            bad += 1
            print(f"MISMATCH layered k={k} lw={lw} copies={copies} depth={depth}", flush=True)
        done += 1
    print(f"layered BN254 (2^13..2^17 gates/layer): {done} circuits, mismatches so far {bad}", flush=True)


def distributed(cases):
    """emulated ranks (threads on lanes of this GPU) vs the single-GPU proof"""
    global bad
    f = P.Field.bn254()
    rng = np.random.default_rng(11)
    done = 0
    for k in range(cases):
        if time.time() > t_end:
            break
        world = int(1 << rng.integers(1, 4))
        lw = int(rng.integers(4, 12))
        copies = world * int(1 << rng.integers(0, 3))
        depth = int(rng.integers(2, 6))
        insz, flat = W.layered_circuit(3000 + k, lw, depth)
        inputs = W.random_inputs(f.p, insz * copies, 60 + k)
        tr1, tr2 = P.Transcript(f, "fd", [k]), P.Transcript(f, "fd", [k])
        want = P.gkr_prove(ctx, P.Circuit(ctx, insz, *flat, n_copies=copies), inputs, tr1)
        got = P.gkr_prove_dist_emulated(ctx, P.Circuit(ctx, insz, *flat, n_copies=copies // world), world, inputs,
                                        tr2)
        if got != want or tr1.state != tr2.state:
            bad += 1
            print(f"MISMATCH dist k={k} world={world} lw={lw} copies={copies} depth={depth}", flush=True)
        done += 1
    print(f"distributed (emulated ranks 2/4/8) vs single: {done} circuits, mismatches so far {bad}", flush=True)


def pcs(cases):
    """pcs::commit root and pcs::open bytes vs the compiled reference"""
    global bad
    done = 0
    rng = np.random.default_rng(13)
    for k in range(cases):
        if time.time() > t_end:
            break
        fld = O.BN254 if k % 3 else O.Field(O.GOLDILOCKS_P)
        f = P.Field(fld.p)
        lm = int(rng.integers(0, 3))  # M = 1, 2, 4 rows
        M = 1 << lm
        lc = int(rng.integers(0, 13))
        rows = [O.random_elements(fld, 1 << lc, rng) for _ in range(M)]
        point = O.random_elements(fld, lc + lm, rng)
        q = int(rng.integers(1, 40))
        ok = P.pcs_commit(ctx, f, rows) == R.pcs_commit(fld, rows)
        got = P.pcs_open(ctx, f, rows, point, P.Transcript(f, "fp", [k]), q)
        want = R.pcs_open(fld, "fp", [k], rows, point, q)[0]
        if not ok or got != want:
            bad += 1
            print(f"MISMATCH pcs k={k} p={fld.p} M={M} cols=2^{lc} q={q}", flush=True)
        done += 1
    print(f"pcs commit/open: {done} instances, mismatches so far {bad}", flush=True)


general(O.BN254, n_general, "gen")
layered(n_layered)
general(O.Field(O.GOLDILOCKS_P), n_general // 3, "gen")
general(O.Field(97), n_general // 3, "gen")
general(O.Field(2**255 - 19), n_general // 6, "gen")           # wide runtime policy (255 bits)
general(O.Field(2**256 - 2**32 - 977), n_general // 6, "gen")  # wide runtime policy (256 bits)
distributed(max(8, n_layered))
pcs(max(20, n_layered * 2))
print("total mismatches", bad)
sys.exit(1 if bad else 0)
