"""Multi-GPU data-parallel proving: one process per GPU (torchrun), rank r
proving copies [r*n, (r+1)*n) of the data-parallel circuit (the rank index is
the top log2(world) variables of every layer, cluster.hpp:182-189).

Transports (csrc/prover.cpp):
  * shared memory ("shm", default for the multi-lane stream): one POSIX
    segment per lane; per-round payloads are host-resident already, so a
    one-node host exchange is the lowest-latency path and keeps lanes
    independent;
  * NCCL ("nccl"): one communicator per process over NVLink/NVSwitch; used
    for single-lane proving (dgkr_gkr_prove_dist).

torch.distributed is the plumbing: rendezvous, the token/NCCL-id broadcast,
barriers and the max-over-ranks timing reduction.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import secrets
import statistics
import time
from typing import List, Optional, Sequence

import numpy as np

from . import prover as P
from ._lib import Profile_t, Transcript_t, check, lib


class ShmComm:
    """dgkr_comm over a shared-memory segment `name` (same on every rank)."""

    def __init__(self, ctx: Optional[P.Context], name: str, rank: int, world: int, slot_bytes: int):
        h = C.c_void_p()
        check(lib().dgkr_comm_create_shm(ctx.handle if ctx is not None else None, name.encode(), C.c_int(rank),
                                         C.c_int(world), C.c_size_t(slot_bytes), C.byref(h)))
        self._h = h
        self.rank, self.world = rank, world

    @property
    def handle(self):
        return self._h

    def allgather_host(self, data: bytes) -> List[bytes]:
        out = C.create_string_buffer(len(data) * self.world)
        check(lib().dgkr_comm_allgather_host(self._h, C.c_char_p(bytes(data)), C.c_size_t(len(data)), out))
        raw = out.raw
        return [raw[i * len(data):(i + 1) * len(data)] for i in range(self.world)]

    def __del__(self):
        try:
            if self._h:
                lib().dgkr_comm_destroy(self._h)
        except Exception:
            pass


def slot_bytes_for(circuit: P.Circuit, field: P.Field, cap: int = 1 << 20) -> int:
    """per-rank slot of a lane's segment: 1 MiB. The claimed-output gather is
    chunked through it (a C2 rank share is 2^22/N x 32 B), and it holds the
    early-boundary table gather (up to 31 tables x 2^10 elements x 32 B,
    prover.cpp kEarlyLog). 64 lanes x 8 ranks x 1 MiB = 512 MiB of /dev/shm."""
    del circuit, field
    return cap


def prove_dist_stream(ctx: P.Context, comms: Sequence, circuit: P.Circuit, field: P.Field, n: int, label: str,
                      inputs=None, out_bufs=None, spread_absorb: bool = False):
    """n distributed proofs over len(comms) lanes (lane l: proofs l, l+L, ...).
    spread_absorb: proof i's claimed outputs are gathered to and absorbed on
    rank i mod world (else rank 0); only that rank's copy of proof i carries
    the output section."""
    L = len(comms)
    cap = circuit.proof_bound(field) + (comms[0].world - 1) * circuit.output_size * field.width + 4096
    if out_bufs is None:
        out_bufs = [np.empty(cap, dtype=np.uint8) for _ in range(n)]
    # fewer buffers than proofs: proof i uses buffer i mod len (proofs i and
    # i + L run one after the other on lane i mod L, so reuse is safe when
    # len(out_bufs) is a multiple of L); the returned proofs then alias
    out_bufs = [out_bufs[i % len(out_bufs)] for i in range(n)]
    tarr = (Transcript_t * n)()
    for i in range(n):
        tarr[i] = P.Transcript(field, label).t
    outs = (C.c_void_p * n)(*[out_bufs[i].ctypes.data for i in range(n)])
    caps = (C.c_size_t * n)(*[len(out_bufs[i]) for i in range(n)])
    lens = (C.c_size_t * n)()
    carr = (C.c_void_p * L)(*[c.handle.value for c in comms])
    in_ptrs = None
    if inputs is not None:
        in_ptrs = (C.c_void_p * n)(*([inputs.ctypes.data] * n))
    profs = (Profile_t * L)()
    check(lib().dgkr_gkr_prove_dist_stream(ctx.handle, carr, C.c_size_t(L), circuit.handle, field.handle,
                                           C.c_size_t(n), in_ptrs, tarr, outs, caps, lens, profs,
                                           C.c_int(1 if spread_absorb else 0)))
    return ([out_bufs[i][: lens[i]] for i in range(n)], [bytes(tarr[i].state) for i in range(n)],
            [profs[i].as_dict() for i in range(L)])


def run_bench_rank(args, cfg_name, configs, circuit_seed, input_seed, helpers=None):
    """bench.py --gpus N under torchrun: every rank proves its share of each
    proof of a stream; rank 0 prints the JSON line (max-over-ranks timing).
    helpers (from bench.py): clock_sampler, measured_peaks, proof_roofline."""
    helpers = helpers or {}
    import torch
    import torch.distributed as dist

    from . import workloads as W

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local_rank = int(os.environ.get("LOCAL_RANK", rank))
    # DGKR_DEVICE / DGKR_DIST_BACKEND let tests run several ranks on one GPU
    # (ranks exchange only through host shared memory; no kernel waits on another)
    device = int(os.environ.get("DGKR_DEVICE", local_rank))
    backend = os.environ.get("DGKR_DIST_BACKEND", "nccl")
    # proofs in flight: the serial output absorb (~0.5 s of host time per C2
    # proof, spread over the ranks) caps throughput at lanes / 0.5 s, so lanes
    # grow with N; per-lane device memory shrinks as 1/N
    # DGKR_TRANSPORT: "shm" (default: one POSIX shared-memory segment per lane;
    # the per-round payloads are host-resident already) or "nccl" (one NCCL
    # communicator per lane over NVLink; communicator setup is heavier, so the
    # default lane count is lower)
    transport = os.environ.get("DGKR_TRANSPORT", "shm")
    if transport not in ("shm", "nccl"):
        raise SystemExit(f"DGKR_TRANSPORT={transport}: expected shm or nccl")
    lanes = args.lanes or (min(64, 32 * world) if transport == "shm" else min(16, 8 * world))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    if lanes * local_world > (os.cpu_count() or 1) and "DGKR_SPIN_US" not in os.environ:
        # more lane threads than host cores: spin briefly, then block, so
        # waiting lanes leave the cores to the lanes hashing their outputs
        os.environ["DGKR_SPIN_US"] = "200"
    torch.cuda.set_device(device)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", device))
    else:
        dist.init_process_group(backend)
    n_copies, lw, depth, desc = configs[cfg_name]
    if n_copies % world:
        raise SystemExit(f"{n_copies} copies do not shard over {world} GPUs")
    ctx = P.Context(device)
    field = P.Field.bn254()
    insz, flat = W.layered_circuit(circuit_seed, lw, depth)
    n_local = n_copies // world
    circ = P.Circuit(ctx, insz, *flat, n_copies=n_local)
    all_inputs = W.random_inputs(field.p, insz * n_copies, input_seed)
    per = insz * n_local * field.width
    mine = np.ascontiguousarray(all_inputs[rank * per:(rank + 1) * per])
    if transport == "shm":
        token = [secrets.token_hex(6) if rank == 0 else None]
        dist.broadcast_object_list(token, src=0)
        comms = [ShmComm(ctx, f"/dgkr_{token[0]}_{l}", rank, world, slot_bytes_for(circ, field))
                 for l in range(lanes)]
    else:
        uids = [[P.Comm.nccl_unique_id() for _ in range(lanes)] if rank == 0 else None]
        dist.broadcast_object_list(uids, src=0)
        comms = [P.Comm(ctx, uids[0][l], rank, world) for l in range(lanes)]
    for l in range(lanes):
        P.load_inputs_lane(ctx, circ, field, l, mine)
    cap = circ.proof_bound(field) + (world - 1) * circ.output_size * field.width + 4096
    bufs = [np.empty(cap, dtype=np.uint8) for _ in range(lanes)]  # one per lane, reused
    gates = n_copies * (1 << lw) * depth

    def timed(n, inputs=None):
        """device time of n proofs (CUDA events on the context stream around
        the call, which returns after every lane's work is done), max over ranks"""
        dist.barrier()
        torch.cuda.synchronize()
        check(lib().dgkr_ctx_event_record(ctx.handle, 4))
        proofs, states, profs = prove_dist_stream(ctx, comms, circ, field, n, "dgkr.bench.c2", inputs=inputs,
                                                  spread_absorb=True, out_bufs=bufs)
        check(lib().dgkr_ctx_event_record(ctx.handle, 5))
        ev_ms = C.c_float()
        check(lib().dgkr_ctx_event_elapsed(ctx.handle, 4, 5, C.byref(ev_ms)))
        dt = torch.tensor([ev_ms.value * 1e-3], device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)  # max over ranks
        return float(dt.item()), proofs, states, profs

    timed(lanes * args.warmup)
    sampler = helpers["clock_sampler"](device) if (rank == 0 and "clock_sampler" in helpers) else None
    if sampler:
        sampler.start()
    dt, proofs, states, profs = timed(lanes * args.steps)
    clk = sampler.stop() if sampler else None
    # e2e: the same stream with this rank's inputs read from pinned host memory
    # by every proof (H2D inside) and proof bytes written to pinned host buffers
    mine_p = np.empty_like(mine)
    mine_p[:] = mine
    pinned = [mine_p] + bufs
    for a_ in pinned:
        check(lib().dgkr_host_register(a_.ctypes.data_as(C.c_void_p), C.c_size_t(a_.nbytes)))
    timed(lanes, inputs=mine_p)
    dt_e2e, _, states_e2e, profs_e2e = timed(lanes * args.steps, inputs=mine_p)
    io = torch.tensor([sum(p_["h2d_bytes"] for p_ in profs_e2e), sum(p_["d2h_bytes"] for p_ in profs_e2e)],
                      dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
    dist.all_reduce(io, op=dist.ReduceOp.SUM)  # whole-job bytes
    for a_ in pinned:
        check(lib().dgkr_host_unregister(a_.ctypes.data_as(C.c_void_p)))
    # single-proof latency (one lane)
    lat, _, _, _ = timed(1)
    # one profiled proof (lane 0 of every rank): per-launch CUDA events around the round kernels
    ctx.set_profile(True)
    dist.barrier()
    _, _, pprof = prove_dist_stream(ctx, comms[:1], circ, field, 1, "dgkr.bench.c2", spread_absorb=True,
                                    out_bufs=bufs[:1])
    ctx.set_profile(False)
    pp = pprof[0]
    if rank == 0:
        assert len(set(states)) == 1 and set(states_e2e) == set(states)
        ms_per_step = 1e3 * dt / args.steps
        e2e_ms = 1e3 * dt_e2e / args.steps
        line = {
            "metric": "gkr_prover_gates_per_sec", "value": lanes * gates / (ms_per_step * 1e-3), "unit": "gates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u256",
            "data": "synthetic",
            "config": {"workload": desc, "field": "bn254", "n_copies": n_copies, "copies_per_gpu": n_local,
                       "gates_per_layer_per_copy": 1 << lw, "depth": depth, "gates": gates,
                       "parallelism": f"dp{world} (rank = top log2(N) variables)",
                       "transport": "shm per lane" if transport == "shm" else "NCCL communicator per lane",
                       "output_absorb": "proof i on rank i mod N",
                       "l2": "no flush: layer tables exceed L2"},
            "lanes": lanes, "proof_latency_ms": 1e3 * lat,
            "e2e": {"value": lanes * gates / (e2e_ms * 1e-3), "unit": "gates/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(io[0].item()) // args.steps,
                    "d2h_bytes_per_step": int(io[1].item()) // args.steps,
                    "note": "every rank's inputs from pinned host memory per proof, proof bytes to pinned host; "
                            "bytes summed over ranks"},
            "gpu_launches": sum(p["launches"] for p in profs),
        }
        if pp["round_ms"] > 0 and "measured_peaks" in helpers:
            peak_gbs, peak_src = helpers["measured_peaks"]()
            mp = C.c_double()
            check(lib().dgkr_bench_mul_peak(ctx.handle, C.byref(mp)))
            gbs = pp["round_bytes"] / (pp["round_ms"] * 1e-3) / 1e9
            line["roofline"] = {"bound": "hbm", "kernel": "k_round (fused fold+round), rank 0",
                                "achieved": gbs, "peak": peak_gbs, "unit": "GB/s", "frac": gbs / peak_gbs,
                                "traffic": None, "peak_source": peak_src}
            mps = pp["round_mults"] / (pp["round_ms"] * 1e-3)
            line["roofline_int"] = {"bound": "imad", "kernel": "k_round, rank 0", "achieved": mps, "peak": mp.value,
                                    "unit": "BN254 mont-mul/s", "frac": mps / mp.value}
            if "proof_roofline" in helpers:  # per GPU: each rank proves 1/N of every proof
                line["roofline_proof"] = helpers["proof_roofline"](n_copies, lw, depth,
                                                                    ms_per_step / lanes * world, mp.value)
        line["breakdown_ms_rank0_per_proof"] = {k: pp[k] for k in ("round_ms", "bookkeep_ms", "evaluate_ms",
                                                                   "output_absorb_ms", "host_transcript_ms")}
        line["clocks"] = clk
        print(json.dumps(line))
    dist.barrier()
    dist.destroy_process_group()
    return 0
