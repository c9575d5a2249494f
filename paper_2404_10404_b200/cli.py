"""`dgkr`-compatible command line on the B200 prover (
reference: proj/tools/dgkr.cpp). Run as ``python -m paper_2404_10404_b200 ...``.

Subcommands (same options, outputs and exit codes as the reference):
  circuit    validate / evaluate / prove + verify a circuit file
             (JSON as GeneralCircuit::from_json, or a binary DGKRCSR1 file)
             dgkr.cpp:187-243
  bench      dist_sumcheck + DistPc scaling over worker counts -> CSV
             "numval,time" dgkr.cpp:136-185
  bitchange  avalanche experiment of the associative hash -> CSV dgkr.cpp:116-128
  convert    JSON -> binary DGKRCSR1 circuit file (new; the reference's
             JSON is impractical at ~10^8 gates)
`demo` (the beacon/epoch pipeline) is outside the hot-path scope
and exits 2 with a message.

Exit codes: 0 ok; 1 verification failed / runtime error; 2 bad input
(invalid_argument, unreadable files, parse errors), as dgkr.cpp:313-331.
Logging to stderr follows DGKR_LOG=quiet|debug (dgkr.cpp:27-39).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from typing import List, Optional

from . import circuit_io as IO
from . import prover as P
from ._lib import DgkrError, InvalidArgument, OutOfRange


def _log_level() -> int:
    v = os.environ.get("DGKR_LOG")
    if v is None:
        return 1
    return {"quiet": 0, "debug": 2}.get(v, 1)


def log_info(msg: str) -> None:
    if _log_level() >= 1:
        print(f"dgkr: {msg}", file=sys.stderr)


def field_by_name(name: str) -> P.Field:
    """FieldConfig::by_name (field.hpp:58-62)"""
    if name == "bn254":
        return P.Field.bn254()
    if name == "goldilocks":
        return P.Field.goldilocks()
    raise InvalidArgument(1, f"unknown field name: {name}")


def _write(path: str, content: str) -> bool:
    try:
        with open(path, "w") as fh:
            fh.write(content)
        return True
    except OSError:
        return False


def _load_circuit_file(ctx: P.Context, path: str):
    """-> (Circuit, input_size, n_out_unpadded) or an exit code"""
    try:
        with open(path, "rb") as fh:
            head = fh.read(8)
    except OSError:
        print(f"dgkr: cannot open {path}", file=sys.stderr)
        return 2
    if head == b"DGKRCSR1":
        try:
            c = P.Circuit.load(ctx, path)
        except InvalidArgument as e:
            print(f"violation: {e}", file=sys.stderr)
            return 2
        import struct
        with open(path, "rb") as fh:
            blob = fh.read(40)
        _, depth, ncp, _, _, _ = struct.unpack("<4I2Q", blob[8:40])
        # unpadded output size of the file's circuit: read layer_gate_start tail
        with open(path, "rb") as fh:
            fh.seek(40 + 8 * (depth - 1))
            a, b = struct.unpack("<2Q", fh.read(16))
        return c, c.input_size * c.n_copies, int(b - a) * c.n_copies
    try:
        with open(path) as fh:
            obj = json.load(fh)
        insz, flat = IO.from_json(obj)
    except (ValueError, KeyError, TypeError, IndexError) as e:
        print(f"dgkr: invalid circuit file: {e}", file=sys.stderr)
        return 2
    try:
        c = P.Circuit(ctx, insz, *flat)
    except InvalidArgument as e:
        print(f"violation: {e}", file=sys.stderr)
        return 2
    return c, insz, int(flat[0][-1] - flat[0][-2])


def run_circuit(a) -> int:
    """dgkr.cpp:187-243"""
    if not os.access(a.file, os.R_OK):
        print(f"dgkr: cannot open {a.file}", file=sys.stderr)
        return 2
    ctx = P.Context(0)
    got = _load_circuit_file(ctx, a.file)
    if isinstance(got, int):
        return got
    c, n_in, n_out = got
    print(f"circuit ok: {c.depth} layers, input size {n_in}")
    if not a.inputs:
        return 0
    f = field_by_name(a.field)
    try:
        vals = [int(x) % f.p for x in a.inputs.split(",")]  # FieldElement(cfg, BigInt) reduces
    except ValueError as e:
        raise InvalidArgument(1, f"bad input value: {e}")
    if len(vals) != n_in:
        print(f"dgkr: expected {n_in} inputs", file=sys.stderr)
        return 2
    outs = c.evaluate(f, vals)
    ov = [int.from_bytes(outs[i * f.width:(i + 1) * f.width], "little") for i in range(n_out)]
    print("outputs:" + "".join(f" {v}" for v in ov))
    if not a.prove:
        return 0
    ptr = P.Transcript(f, "dgkr.cli.circuit")
    proof = P.gkr_prove(ctx, c, vals, ptr)
    vtr = P.Transcript(f, "dgkr.cli.circuit")
    ok = P.gkr_verify(c, proof, vtr, outputs=ov, inputs=vals)
    print("proof verified" if ok else "proof rejected")
    return 0 if ok else 1


def run_bench(a) -> int:
    """dgkr.cpp:136-185: per worker count N, dist_sumcheck over `pairs`
    product pairs (f0 shared, as the reference) and DistPc over the workers'
    f0 shards; wall time per N -> CSV. Tables are random canonical elements
    from seeded numpy (the reference draws mt19937_64; timing only)."""
    from . import workloads as W
    if not a.workers:
        print("dgkr: bench needs at least one worker count", file=sys.stderr)
        return 2
    f = field_by_name(a.field)
    ctx = P.Context(0)
    csv = "numval,time\n"
    n = 1 << a.vars
    for N in a.workers:
        if N == 0 or (N & (N - 1)) != 0 or n < N:
            print(f"dgkr: invalid worker count {N}", file=sys.stderr)
            return 2
        f0 = W.random_inputs(f.p, n, a.seed).tobytes()
        pairs = [(f0, W.random_inputs(f.p, n, a.seed + 1 + k).tobytes()) for k in range(a.pairs)]
        chunk = (n // N) * f.width
        rows = [f0[i * chunk:(i + 1) * chunk] for i in range(N)]
        r = [int.from_bytes(W.random_inputs(f.p, 1, a.seed + 1000 + k).tobytes(), "little") for k in range(a.vars)]
        t0 = time.perf_counter()
        P.dist_sumcheck(ctx, N, pairs, P.Transcript(f, "dgkr.bench"))
        P.distpc(ctx, f, rows, r)
        dt = time.perf_counter() - t0
        csv += f"{N},{dt:g}\n"
        log_info(f"N={N} took {dt:f}s")
    if not _write(a.out, csv):
        print(f"dgkr: cannot write {a.out}", file=sys.stderr)
        return 2
    return 0


def run_bitchange(a) -> int:
    """dgkr.cpp:116-128"""
    f = field_by_name(a.field)
    ctx = P.Context(0)
    _, probs = P.bitchange_experiment(ctx, f, a.count)
    if not _write(a.out, P.bitchange_csv(probs)):
        print(f"dgkr: cannot write {a.out}", file=sys.stderr)
        return 2
    log_info(f"wrote {len(probs)} rows to {a.out}")
    return 0


def run_convert(a) -> int:
    """JSON -> binary DGKRCSR1 (validated on the way)"""
    with open(a.input, "rb") as fh:
        head = fh.read(8)
    if head == b"DGKRCSR1":
        raise InvalidArgument(1, f"{a.input} is already a binary circuit file")
    ctx = P.Context(0)
    insz, flat = IO.load_json_file(a.input)
    P.Circuit(ctx, insz, *flat).save(a.output)
    log_info(f"wrote {a.output}")
    return 0


def _workers(s: str) -> List[int]:
    return [int(x) for x in s.split(",") if x]


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="dgkr", description="distributed sumcheck/GKR proving toolkit (B200)")
    sub = ap.add_subparsers(dest="cmd")
    sub.add_parser("demo", help="run a full demo epoch (not provided: outside the hot-path scope)")
    b = sub.add_parser("bitchange", help="bit-change probability experiment")
    b.add_argument("--field", default="bn254")
    b.add_argument("--count", type=int, default=1000000)
    b.add_argument("--out", default="index-bit_change.csv")
    be = sub.add_parser("bench", help="distributed sumcheck/commit scaling bench")
    be.add_argument("--field", default="bn254")
    be.add_argument("--workers", type=_workers, default=[])
    be.add_argument("--vars", type=int, default=10)
    be.add_argument("--pairs", type=int, default=2)
    be.add_argument("--seed", type=int, default=1)
    be.add_argument("--out", default="bench.csv")
    c = sub.add_parser("circuit", help="validate/evaluate/prove a circuit file")
    c.add_argument("--file", required=True)
    c.add_argument("--field", default="bn254")
    c.add_argument("--inputs", default="")
    c.add_argument("--prove", action="store_true")
    cv = sub.add_parser("convert", help="JSON -> binary DGKRCSR1 circuit file")
    cv.add_argument("input")
    cv.add_argument("output")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    if a.cmd is None:
        ap.print_usage(sys.stderr)
        return 2
    try:
        if a.cmd == "demo":
            print("dgkr: demo (beacon/epoch pipeline) is not part of the B200 hot path; see DESIGN.md", file=sys.stderr)
            return 2
        return {"bitchange": run_bitchange, "bench": run_bench, "circuit": run_circuit, "convert": run_convert}[a.cmd](a)
    except InvalidArgument as e:
        print(f"dgkr: {e}", file=sys.stderr)
        return 2
    except (DgkrError, OutOfRange, RuntimeError, OSError) as e:
        print(f"dgkr: error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
