#!/usr/bin/env python
"""Benchmark: GKR prover gates/sec on the BASELINE.json workload.

Default workload (N=1): config C2 — a data-parallel GKR proof of 64 identical
sub-circuits of 2^16 gates/layer x 24 layers (100,663,296 gates) over BN254,
synthetic inputs. One proof = one complete gkr_prove (gkr.hpp:182-244):
circuit evaluation, serial output-table absorb, 24 two-phase layer
sum-checks, proof bytes back to the host. One "step" = `--lanes` proofs; the
K timed steps run as one continuous stream of K*lanes proofs over `lanes`
concurrent lanes (dgkr_gkr_prove_stream), because bit-exactness forces a
~0.5 s serial host SHA-256 chain per proof that only
concurrency can hide.

  value  gates/s of the stream, inputs resident in HBM on every lane, CUDA
         events around the stream
  proof_latency_ms   one proof alone (dgkr_gkr_prove_resident)
  e2e    the same stream through the public C-ABI call with pinned host
         inputs (H2D inside) and proof bytes back to pinned host buffers
  roofline / roofline_int   fused fold+round kernel (the dominant kernel),
         from a separate profiled step (per-launch CUDA events)
  cpu_baseline   the compiled reference (oracle/_ref) on a bounded sample

`--impl reference` times the reference's own CPU prover (oracle/_ref) on a
bounded sample with all host threads. Multi-GPU: launched with torchrun, one
rank per GPU.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n_copies, log_width, depth, description)
    "c2": (64, 16, 24, "C2: 64 data-parallel sub-circuits x 2^16 gates/layer x 24 layers, BN254"),
    "c1": (1, 12, 16, "C1: single-worker 2^12 gates/layer x 16 layers, BN254"),
}
CIRCUIT_SEED = 20240410
INPUT_SEED = 7


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=5)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# Reference CPU prover (oracle/_ref) — the baseline, never the product.
# ---------------------------------------------------------------------------
_REF_CACHE = {}


def _ref_worker(args):
    """one reference gkr_prove (separate process: the reference keeps a
    shared_ptr<FieldConfig> in every FieldElement, so threads would contend on
    one atomic refcount). Circuit and inputs are generated once per worker
    process (pool initializer) and cached; copies differ by transcript prefix."""
    log_width, depth, t = args
    sys.path.insert(0, ROOT)
    from oracle import dgkr_oracle as O
    from oracle import refbind as R
    from paper_2404_10404_b200 import workloads as W

    fld = O.BN254
    key = (log_width, depth)
    if key not in _REF_CACHE:
        insz, flat = W.layered_circuit(CIRCUIT_SEED, log_width, depth)

        class _Shape:  # minimal shape for refbind.gkr_prove's capacity math
            input_size = insz

            @staticmethod
            def padded_size(l):
                return 1 << log_width

        inputs = fld.elems_from_bytes(W.random_inputs(fld.p, insz, INPUT_SEED).tobytes())
        _REF_CACHE[key] = (_Shape, flat, inputs)
    if t < 0:  # pool initializer: build the cache only
        return 0.0
    shape, flat, inputs = _REF_CACHE[key]
    t0 = time.perf_counter()
    R.gkr_prove(fld, "dgkr.bench", [t], shape, inputs, flat=flat)
    return time.perf_counter() - t0


def reference_sample(workers: int, log_width: int, depth: int, pool=None):
    """gates/s of the reference gkr_prove on `workers` independent copies of a
    (2^log_width x depth) sub-circuit of the same family, run concurrently in
    separate processes; wall time of the whole batch)."""
    gates = (1 << log_width) * depth
    if pool is None:
        dt = _ref_worker((log_width, depth, 0))
        workers = 1
    else:
        t0 = time.perf_counter()
        pool.map(_ref_worker, [(log_width, depth, t) for t in range(workers)], chunksize=1)
        dt = time.perf_counter() - t0
    return workers * gates / dt, dt, gates


def run_reference_arm(args, cfg_name):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    n_copies, lw, depth, desc = CONFIGS[cfg_name]
    from oracle import refbind as R

    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdgkr_ref.so not built"}))
        return 0
    import multiprocessing as mp

    threads = len(os.sched_getaffinity(0)) or 1
    s_depth = 2 if cfg_name == "c2" else depth
    s_lw = lw
    sample = (f"{threads} concurrent independent reference gkr_prove calls (one process per host core), each on "
              f"one 2^{s_lw} x {s_depth}-layer sub-circuit of the {cfg_name.upper()} family (BN254); "
              f"gates/s = total gates / wall time")
    vals, times = [], []
    with mp.get_context("spawn").Pool(threads, initializer=_ref_worker,
                                      initargs=((s_lw, s_depth, -1),)) as pool:
        for _ in range(args.warmup):
            reference_sample(threads, s_lw, s_depth, pool)
        for _ in range(args.steps):
            v, dt, _g = reference_sample(threads, s_lw, s_depth, pool)
            vals.append(v)
            times.append(dt)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "gkr_prover_gates_per_sec", "value": value, "unit": "gates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u256", "data": "synthetic",
        "config": config_dict(cfg_name, world),
        "cpu_baseline": {"value": value, "unit": "gates/s", "cores": threads, "kind": "reference", "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "sample_vs_workload": (
            "measured on one core of this host (tools/ref_scaling.py, profiles/r2/reference_scaling.jsonl): "
            "12.9 us/gate for the 2^16 x 2 sample, 13.3 for one full 2^16 x 24 sub-circuit, growing ~0.7-0.9 us "
            "per extra variable (SURVEY 8(a) a5: (3s+30) mults/gate); at C2's s = 22 the reference pays ~16-18 "
            "us/gate, so this sample overstates its C2 throughput by ~1.25-1.4x" if cfg_name == "c2" else None),
    }
    print(json.dumps(line))
    return 0


def config_dict(cfg_name, world):
    n_copies, lw, depth, desc = CONFIGS[cfg_name]
    return {"workload": desc, "field": "bn254", "n_copies": n_copies, "gates_per_layer_per_copy": 1 << lw,
            "depth": depth, "gates": n_copies * (1 << lw) * depth, "parallelism": f"dp{world}",
            "l2": "no flush: every layer table (2^22 x 32 B = 128 MiB) exceeds the 126 MB L2"}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(args, cfg_name):
    import paper_2404_10404_b200 as P
    from paper_2404_10404_b200 import workloads as W
    from paper_2404_10404_b200._lib import check, lib

    rank, world, local_rank = env_rank()
    n_copies, lw, depth, desc = CONFIGS[cfg_name]
    if world > 1 or os.environ.get("DGKR_FORCE_DIST") == "1":
        from paper_2404_10404_b200 import dist

        return dist.run_bench_rank(args, cfg_name, CONFIGS, CIRCUIT_SEED, INPUT_SEED,
                                   helpers={"clock_sampler": ClockSampler, "measured_peaks": measured_peaks,
                                            "proof_roofline": proof_roofline})
    ctx = P.Context(local_rank)
    field = P.Field.bn254()
    insz, flat = W.layered_circuit(CIRCUIT_SEED, lw, depth)
    circ = P.Circuit(ctx, insz, *flat, n_copies=n_copies)
    n_in = insz * n_copies
    inputs = W.random_inputs(field.p, n_in, INPUT_SEED)  # canonical bytes
    gates = circ.n_gates
    cap = circ.proof_bound(field)
    # pinned host buffers (e2e contract: H2D from pinned memory)
    in_pinned = np.empty_like(inputs)
    in_pinned[:] = inputs
    out_buf = np.empty(cap, dtype=np.uint8)
    check(lib().dgkr_host_register(in_pinned.ctypes.data_as(C.c_void_p), C.c_size_t(in_pinned.nbytes)))
    check(lib().dgkr_host_register(out_buf.ctypes.data_as(C.c_void_p), C.c_size_t(out_buf.nbytes)))
    ln = C.c_size_t()

    def prove_resident():
        tr = P.Transcript(field, "dgkr.bench.c2")
        check(lib().dgkr_gkr_prove_resident(ctx.handle, circ.handle, field.handle, C.byref(tr.t),
                                            out_buf.ctypes.data_as(C.c_void_p), C.c_size_t(cap), C.byref(ln)))
        return tr

    def prove_e2e():
        tr = P.Transcript(field, "dgkr.bench.c2")
        check(lib().dgkr_gkr_prove(ctx.handle, circ.handle, field.handle, in_pinned.ctypes.data_as(C.c_void_p),
                                   C.byref(tr.t), out_buf.ctypes.data_as(C.c_void_p), C.c_size_t(cap), C.byref(ln)))
        return tr

    # (1) single-proof latency, inputs resident in HBM (lane 0)
    check(lib().dgkr_circuit_load_inputs(ctx.handle, circ.handle, field.handle, in_pinned.ctypes.data_as(C.c_void_p)))
    for _ in range(args.warmup):
        tr_ref = prove_resident()
    state0 = tr_ref.state
    lat_ms = []
    for _ in range(args.steps):
        check(lib().dgkr_ctx_event_record(ctx.handle, 4))
        prove_resident()
        check(lib().dgkr_ctx_event_record(ctx.handle, 5))
        ms = C.c_float()
        check(lib().dgkr_ctx_event_elapsed(ctx.handle, 4, 5, C.byref(ms)))
        lat_ms.append(ms.value)
    latency_ms = statistics.median(lat_ms)

    # (2) throughput: a step is `lanes` proofs; the K timed steps run as ONE
    # continuous stream of K*lanes proofs over `lanes` lanes (work queue: a
    # lane takes the next proof when it finishes one, so the serial host
    # transcript of one proof overlaps the GPU work of the others). Inputs
    # are resident in HBM on every lane.
    lanes = args.lanes or 32
    for i in range(lanes):
        P.load_inputs_lane(ctx, circ, field, i, in_pinned)
    from paper_2404_10404_b200._lib import Profile_t, Transcript_t

    n_max = lanes * max(args.steps, args.warmup)
    bufs = [out_buf] + [np.empty(cap, dtype=np.uint8) for _ in range(n_max - 1)]
    for b in bufs[1:]:
        check(lib().dgkr_host_register(b.ctypes.data_as(C.c_void_p), C.c_size_t(b.nbytes)))

    def stream(n_proofs: int, resident: bool):
        tarr = (Transcript_t * n_proofs)()
        for i in range(n_proofs):
            tarr[i] = P.Transcript(field, "dgkr.bench.c2").t
        outs = (C.c_void_p * n_proofs)(*[bufs[i].ctypes.data for i in range(n_proofs)])
        caps = (C.c_size_t * n_proofs)(*([cap] * n_proofs))
        lens = (C.c_size_t * n_proofs)()
        in_ptrs = None if resident else (C.c_void_p * n_proofs)(*([in_pinned.ctypes.data] * n_proofs))
        profs = (Profile_t * lanes)()
        check(lib().dgkr_gkr_prove_stream(ctx.handle, circ.handle, field.handle, C.c_size_t(n_proofs),
                                          C.c_size_t(lanes), in_ptrs, tarr, outs, caps, lens, profs))
        for i in range(n_proofs):
            assert bytes(tarr[i].state) == state0, "stream proof differs from the single proof"
        tot = {"launches": 0, "h2d_bytes": 0, "d2h_bytes": 0, "output_absorb_ms": 0.0, "host_transcript_ms": 0.0,
               "rounds": 0}
        for i in range(min(lanes, n_proofs)):
            for k in tot:
                tot[k] += getattr(profs[i], k)
        return tot, lens[0]

    stream(lanes * args.warmup, True)
    clocks = ClockSampler(local_rank)
    clocks.start()
    check(lib().dgkr_ctx_event_record(ctx.handle, 0))
    tot, proof_len = stream(lanes * args.steps, True)
    check(lib().dgkr_ctx_event_record(ctx.handle, 1))
    ms = C.c_float()
    check(lib().dgkr_ctx_event_elapsed(ctx.handle, 0, 1, C.byref(ms)))
    clk = clocks.stop()
    launches = tot["launches"]
    phase = {k: tot[k] for k in ("output_absorb_ms", "host_transcript_ms", "rounds")}
    ms_per_step = ms.value / args.steps
    value = lanes * gates / (ms_per_step * 1e-3)

    # (3) e2e: the same stream through the public call with pinned host inputs
    # (H2D inside) and proof bytes back in pinned host buffers (D2H inside)
    stream(lanes, False)
    check(lib().dgkr_ctx_event_record(ctx.handle, 2))
    t0 = time.perf_counter()
    tot, _ = stream(lanes * args.steps, False)
    check(lib().dgkr_ctx_event_record(ctx.handle, 3))
    wall_e2e = (time.perf_counter() - t0) / args.steps
    check(lib().dgkr_ctx_event_elapsed(ctx.handle, 2, 3, C.byref(ms)))
    e2e_ms = ms.value / args.steps
    h2d, d2h = tot["h2d_bytes"], tot["d2h_bytes"]
    for b in bufs[1:]:
        check(lib().dgkr_host_unregister(b.ctypes.data_as(C.c_void_p)))

    # profiled step: per-launch CUDA events around the fused round kernels
    ctx.set_profile(True)
    prove_resident()
    prof = ctx.profile()
    ctx.set_profile(False)
    peak_gbs, peak_src = measured_peaks()
    mp = C.c_double()
    check(lib().dgkr_bench_mul_peak(ctx.handle, C.byref(mp)))
    round_s = prof["round_ms"] * 1e-3
    achieved_gbs = prof["round_bytes"] / round_s / 1e9 if round_s > 0 else None
    achieved_mps = prof["round_mults"] / round_s if round_s > 0 else None
    traffic, traffic_ratio = load_ncu_traffic()

    cpu = None
    if not args.no_cpu_baseline:
        try:
            from oracle import refbind as R

            if R.available():
                v, dt, g = reference_sample(1, lw, 6 if cfg_name == "c2" else depth)
                cpu = {"value": v, "unit": "gates/s", "cores": 1, "kind": "reference",
                       "sample": f"reference gkr_prove (oracle/_ref, single-threaded as the reference is) on one "
                                 f"2^{lw} x {6 if cfg_name == 'c2' else depth}-layer sub-circuit of the same family: "
                                 f"{g} gates in {dt:.1f} s", "cpu": cpu_model()}
        except Exception as e:  # baseline is reported, not required
            cpu = {"value": None, "unit": "gates/s", "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    line = {
        "metric": "gkr_prover_gates_per_sec", "value": value, "unit": "gates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u256", "data": "synthetic",
        "config": config_dict(cfg_name, world),
        "proof_latency_ms": latency_ms, "lanes": lanes,
        "e2e": {"value": lanes * gates / (e2e_ms * 1e-3), "unit": "gates/s", "ms_per_step": e2e_ms,
                "wall_ms_per_step": 1e3 * wall_e2e, "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps},
        "gpu_launches": launches,
        "breakdown_ms_per_step": {
            "host_output_absorb_per_proof": phase["output_absorb_ms"] / args.steps / lanes,
            "host_transcript_total_per_proof": phase["host_transcript_ms"] / args.steps / lanes,
            "round_kernels": prof["round_ms"], "bookkeeping_kernels": prof["bookkeep_ms"],
            "evaluate_kernels": prof["evaluate_ms"], "rounds_per_proof": phase["rounds"] // (args.steps * lanes),
            "tail_launches_incl_host_exchange": prof["tail_ms"], "tail_rounds_per_proof": prof["tail_rounds"],
            "note": "kernel times from one profiled single proof (per-launch CUDA events); round_kernels and the "
                    "roofline cover the rounds with > 256 pairs, the smaller ones run inside the tail launches"},
        "roofline": {"bound": "hbm", "kernel": "k_round (fused fold+round)", "achieved": achieved_gbs,
                     "peak": peak_gbs, "unit": "GB/s", "frac": (achieved_gbs / peak_gbs) if achieved_gbs else None,
                     "traffic": traffic, "traffic_over_algorithmic": traffic_ratio, "peak_source": peak_src,
                     "note": "algorithmic bytes: fold reads 4 + writes 2 elements (32 B) per table per output pair"},
        "roofline_int": {"bound": "imad", "kernel": "k_round (fused fold+round)",
                         "achieved": achieved_mps, "unit": "BN254 mont-mul/s",
                         "peak": HW_MUL_PEAK, "frac": (achieved_mps / HW_MUL_PEAK) if achieved_mps else None,
                         "peak_source": HW_MUL_PEAK_SOURCE,
                         "own_multiplier_peak": mp.value,
                         "own_multiplier_frac": (achieved_mps / mp.value) if achieved_mps else None,
                         "own_multiplier_source": "dgkr_bench_mul_peak: this repo's CIOS, 4 independent chains/thread "
                                                  "(a software ceiling, not the hardware's)"},
        "roofline_proof": proof_roofline(n_copies, lw, depth, ms_per_step / lanes, mp.value),
        "cpu_baseline": cpu,
        "clocks": clk,
        "proof_bytes": proof_len,
    }
    print(json.dumps(line))
    check(lib().dgkr_host_unregister(in_pinned.ctypes.data_as(C.c_void_p)))
    check(lib().dgkr_host_unregister(out_buf.ctypes.data_as(C.c_void_p)))
    return 0


# Hardware integer roofline for BN254 Montgomery products: the IMAD issue rate
# probed on this B200 (1.857e13 IMAD/s = 63.85 per clock per SM at 1965 MHz,
# profiles/mulbench_r1.jsonl) over SURVEY.md §8(d)'s 256 IMAD per product.
IMAD_PER_S = 1.857e13
HW_MUL_PEAK = IMAD_PER_S / 256
HW_MUL_PEAK_SOURCE = ("probed IMAD issue rate 1.857e13/s (profiles/mulbench_r1.jsonl) / 256 IMAD per BN254 "
                      "Montgomery product (SURVEY.md 8(d)); the SASS of this repo's CIOS has 232 IMAD, the "
                      "constant-multiplier fold 140")


def proof_roofline(n_copies, lw, depth, ms_per_proof, mul_peak):
    """Whole-proof integer roofline with SURVEY.md §8(d)'s algorithmic count:
    sum over layers of (K_l + 13) T_l + 3 W_l, plus the evaluate mul wires and
    T_out, K_l = 1 at the output layer and 2 below (layered circuit, W = T,
    half the gates mul); achieved = that count / the stream's time per proof."""
    T = n_copies << lw
    mults = sum((1 if l == depth else 2) * T + 13 * T + 3 * T for l in range(1, depth + 1)) + depth * T // 2 + T
    achieved = mults / (ms_per_proof * 1e-3)
    return {"bound": "imad", "unit": "BN254 mont-mul/s", "algorithmic_mults_per_proof": mults,
            "ms_per_proof": ms_per_proof, "achieved": achieved, "peak": HW_MUL_PEAK, "frac": achieved / HW_MUL_PEAK,
            "peak_source": HW_MUL_PEAK_SOURCE, "own_multiplier_peak": mul_peak,
            "own_multiplier_frac": achieved / mul_peak,
            "note": "survey count treats every fold as a full Montgomery multiplication"}


def load_ncu_traffic():
    """(dram bytes per launch, dram / algorithmic bytes of the same launches)
    of k_round from the committed ncu capture (profiles/ncu_round_traffic.json)"""
    path = os.path.join(ROOT, "profiles", "ncu_round_traffic.json")
    try:
        t = json.load(open(path))
        return t.get("dram_bytes_per_launch"), t.get("dram_over_algorithmic")
    except Exception:
        return None, None


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--lanes", type=int, default=None,
                    help="concurrent proofs per step (lanes; default 32 on one GPU, min(64, 32 N) on N GPUs); "
                         "the single-proof latency is reported separately")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args, args.config)
    return run_b200(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
