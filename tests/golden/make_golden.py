"""Generate tests/golden/golden.json from the COMPILED REFERENCE
(oracle/_ref/libdgkr_ref.so = the unmodified reference headers built against
oracle/shim). Run in the container that has /root/reference:

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin both the Python restatement (tests/test_oracle.py, CPU) and
the CUDA prover (tests/test_gpu_golden.py, GPU) to the reference's own bytes.
Inputs are generated from fixed numpy seeds and stored in the file, so the
fixtures do not depend on this script's RNG at check time.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import dgkr_oracle as O  # noqa: E402
from oracle import refbind as R  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402

FIELDS = {"bn254": O.BN254_P, "tiny97": 97, "goldilocks": O.GOLDILOCKS_P}


def flat_json(insz, flat):
    lgs, gns, nested, minp = flat
    return {"input_size": int(insz), "layer_gate_start": [int(x) for x in lgs],
            "gate_nested_start": [int(x) for x in gns], "nested": [[int(v) for v in e] for e in nested],
            "min_padded": [int(x) for x in minp]}


def main():
    rng = np.random.default_rng(20240410)
    out = {"source": "oracle/_ref/libdgkr_ref.so (unmodified /root/reference/proj/include via oracle/shim)",
           "transcript": [], "product_sum": [], "layer_sum": [], "gkr": [], "pcs": [], "dist_sumcheck": [],
           "distpc": [], "distinct": [], "beacon": []}
    for name, p in FIELDS.items():
        fld = O.Field(p)
        el = O.random_elements(fld, 6, rng)
        ch, idx, st = R.transcript_run(fld, "golden.t", [1, 2], el, 5, 4, 1000)
        out["transcript"].append({"field": name, "label": "golden.t", "pre": [1, 2], "elems": el, "challenges": ch,
                                  "idx_bound": 1000, "indices": idx, "state": st.hex()})
        for vars_, npairs in ((0, 1), (1, 1), (3, 2), (6, 3)):
            pairs = [(O.random_elements(fld, 1 << vars_, rng), O.random_elements(fld, 1 << vars_, rng))
                     for _ in range(npairs)]
            pb, st = R.prove_product_sum(fld, "golden.s", [vars_], pairs)
            out["product_sum"].append({"field": name, "label": "golden.s", "pre": [vars_], "pairs": pairs,
                                       "proof": pb.hex(), "state": st.hex()})
        for side, ns, nw in ((1, 1, 3), (3, 2, 24)):
            T = 1 << side
            tables = [O.random_elements(fld, T, rng) for _ in range(ns)]
            wires = [[int(rng.integers(2)), O.random_elements(fld, 1, rng)[0], int(rng.integers(ns)),
                      int(rng.integers(ns)), int(rng.integers(T)), int(rng.integers(T))] for _ in range(nw)]
            lw = [O.LayerWire(bool(a), b, c, d, e, f) for a, b, c, d, e, f in wires]
            claimed = O.random_elements(fld, 1, rng)[0]
            pb, st = R.prove_layer_sum(fld, "golden.l", [], side, tables, lw, claimed)
            out["layer_sum"].append({"field": name, "label": "golden.l", "side": side, "tables": tables,
                                     "wires": wires, "claimed": claimed, "proof": pb.hex(), "state": st.hex()})
        for seed in range(3):
            c = R.random_general_circuit(100 + seed, 5 + seed, 3, 8, 3)
            inputs = O.random_elements(fld, c.input_size, rng)
            pb, st = R.gkr_prove(fld, "golden.g", [seed], c, inputs)
            acc = R.gkr_verify(fld, "golden.g", [seed], c, inputs, pb)
            out["gkr"].append({"field": name, "label": "golden.g", "pre": [seed],
                               "circuit": flat_json(c.input_size, c.to_flat()), "n_copies": 1, "inputs": inputs,
                               "proof": pb.hex(), "state": st.hex(), "ref_verifier_accepts": acc})
        for M, cols, q in ((1, 1, 32), (2, 8, 3), (4, 32, 6)):
            rows = [O.random_elements(fld, cols, rng) for _ in range(M)]
            r = O.random_elements(fld, O.log2_exact(cols) + O.log2_exact(M), rng)
            root = R.pcs_commit(fld, rows)
            ob, st = R.pcs_open(fld, "golden.p", [], rows, r, q)
            acc = R.pcs_verify(fld, "golden.p", [], M, cols, root, r, ob, q)
            out["pcs"].append({"field": name, "label": "golden.p", "rows": rows, "r": r, "q": q, "root": root.hex(),
                               "opening": ob.hex(), "state": st.hex(), "ref_verifier_accepts": acc})
    fld = O.BN254
    # data-parallel layered circuit (replicated explicitly for the reference)
    insz, flat = W.layered_circuit(seed=77, log_width=3, depth=3)
    full_in, full_flat = W.replicate(insz, flat, 4)
    circ = O.Circuit.from_flat(full_in, *full_flat)
    inputs = fld.elems_from_bytes(W.random_inputs(fld.p, full_in, 78).tobytes())
    pb, st = R.gkr_prove(fld, "golden.dp", [4], circ, inputs)
    out["gkr"].append({"field": "bn254", "label": "golden.dp", "pre": [4], "circuit": flat_json(insz, flat),
                       "n_copies": 4, "inputs": inputs, "proof": pb.hex(), "state": st.hex(),
                       "ref_verifier_accepts": R.gkr_verify(fld, "golden.dp", [4], circ, inputs, pb)})
    for N in (1, 2, 4, 8):
        pairs = [(O.random_elements(fld, 16, rng), O.random_elements(fld, 16, rng)) for _ in range(2)]
        pb, st, js = R.dist_sumcheck(fld, "dgkr.bench", [], N, pairs)
        out["dist_sumcheck"].append({"field": "bn254", "label": "dgkr.bench", "n_workers": N, "pairs": pairs,
                                     "proof": pb.hex(), "state": st.hex(), "traffic": js})
        rows = [O.random_elements(fld, 8, rng) for _ in range(N)]
        r = O.random_elements(fld, 3 + O.log2_exact(N), rng)
        roots, ops, comb, js = R.distpc(fld, rows, r, 4)
        out["distpc"].append({"field": "bn254", "rows": rows, "r": r, "q": 4, "roots": [x.hex() for x in roots],
                              "openings": [x.hex() for x in ops], "combined": comb, "traffic": js})
    # distinct.hpp (C4): AH, pairwise check (true / false cases), chain update, bit-change counts
    drng = np.random.default_rng(2404104)
    for name, p in FIELDS.items():
        fld = O.Field(p)
        bound = min(p - 1, 100000)
        items = [int(x) for x in drng.integers(0, bound + 1, 33)]
        uniq = sorted(set(items))
        perm = [uniq[i] for i in drng.permutation(len(uniq))]
        case = {"field": name, "items": items, "ah": R.distinct_ah(fld, items), "ah_empty": R.distinct_ah(fld, []),
                "perm": perm, "sorted": uniq, "check_true": R.distinct_check(fld, perm, uniq),
                "check_dup": R.distinct_check(fld, items, sorted(items)),
                "h0": 12345 % p, "n_max": bound, "chain": R.distinct_chain_update(fld, 12345 % p, bound, items)}
        if p > 1 << 20:
            case["bitchange_10000"] = R.distinct_bitchange(fld, 10000)
        out["distinct"].append(case)
    # beacon.hpp (C3): roots, membership paths and verdicts of the reference tree
    here = os.path.dirname(os.path.abspath(__file__))
    for n, depth, seed in ((1, 4, 1), (10, 8, 2), (37, 12, 3), (4096, 56, 4)):
        recs = R.beacon_gen(n, seed)
        idx = sorted({0, n - 1, n // 2, (7 * n) // 9})
        paths = []
        for i in idx:
            leaf, sib, a = R.beacon_prove(recs, depth, i)
            paths.append({"index": i, "leaf": leaf.hex(), "siblings": sib.hex(), "active_log2": a})
        case = {"n": n, "depth": depth, "seed": seed, "root": R.beacon_root(recs, depth).hex(), "paths": paths}
        if n <= 64:
            case["records"] = recs.hex()
        else:
            case["records_file"] = f"beacon_{n}.bin"
            with open(os.path.join(here, case["records_file"]), "wb") as fh:
                fh.write(recs)
        out["beacon"].append(case)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
