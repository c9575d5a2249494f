"""CPU, world_size 2 (gloo): the multi-GPU path's host logic.

1. The shared-memory transport of csrc/prover.cpp (per-lane segments and
   barriers) exchanges correctly between two processes (no GPU needed).
2. The distributed sum-check protocol the GPU path implements — every rank
   folds its slice (rank = high variables), partial round sums are all-gathered
   and summed, finals are all-gathered at the boundary and the top log2(world)
   rounds finish redundantly — run with real torch.distributed collectives
   over the oracle's arithmetic, reproduces the reference's single-machine
   proof byte for byte (cluster.hpp:219-227).
"""
import os
import secrets
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dgkr_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _allgather_obj(x, world):
    out = [None] * world
    dist.all_gather_object(out, x)
    return out


def _worker_shm(rank, world, port, name, q):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2404_10404_b200.dist import ShmComm

    _init(rank, world, port)
    comm = ShmComm(None, name, rank, world, 4096)
    ok = True
    for it in range(50):
        payload = bytes([(rank * 31 + it + k) & 0xFF for k in range(96)])
        got = comm.allgather_host(payload)
        want = [bytes([(r * 31 + it + k) & 0xFF for k in range(96)]) for r in range(world)]
        ok &= got == want
    dist.barrier()
    q.put((rank, ok))
    dist.destroy_process_group()


def test_shm_transport_two_processes():
    world = 2
    port = _free_port()
    name = f"/dgkr_test_{secrets.token_hex(4)}"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_shm, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(res.values()) and len(res) == world


def _dist_product_sum(rank, world, pairs, label):
    """the GPU path's distributed protocol, on the oracle's arithmetic"""
    fld = O.BN254
    p = fld.p
    n = len(pairs[0][0])
    chunk = n // world
    mine = [(f[rank * chunk:(rank + 1) * chunk], g[rank * chunk:(rank + 1) * chunk]) for f, g in pairs]
    tr = O.Transcript(label, fld)
    local_total = sum(a * b for f, g in mine for a, b in zip(f, g)) % p
    claimed = sum(_allgather_obj(local_total, world)) % p
    proof = O.SumcheckProof(claimed)
    tr.absorb(claimed)
    for _ in range(chunk.bit_length() - 1):
        parts = _allgather_obj(O.round_poly_over(mine, p), world)
        rp = tuple(sum(x[k] for x in parts) % p for k in range(3)) + (0,)
        for c in rp:
            tr.absorb(c)
        proof.rounds.append(rp)
        mine = O.fold_pairs(mine, tr.challenge(), p)
    finals = _allgather_obj([(f[0], g[0]) for f, g in mine], world)
    tail = [([finals[r][k][0] for r in range(world)], [finals[r][k][1] for r in range(world)]) for k in range(len(pairs))]
    for _ in range(world.bit_length() - 1):
        rp = O.round_poly_over(tail, p)
        for c in rp:
            tr.absorb(c)
        proof.rounds.append(rp)
        tail = O.fold_pairs(tail, tr.challenge(), p)
    proof.finals = [x for f, g in tail for x in (f[0], g[0])]
    return proof.to_bytes(fld), tr.state


def _worker_protocol(rank, world, port, q):
    import sys

    import numpy as np

    sys.path.insert(0, ROOT)
    _init(rank, world, port)
    rng = np.random.default_rng(5)
    pairs = [(O.random_elements(O.BN254, 64, rng), O.random_elements(O.BN254, 64, rng)) for _ in range(2)]
    got = _dist_product_sum(rank, world, pairs, "dgkr.bench")
    tr = O.Transcript("dgkr.bench", O.BN254)
    want = (O.prove_product_sum(pairs, tr).to_bytes(O.BN254), tr.state)
    q.put((rank, got == want))
    dist.destroy_process_group()


def test_distributed_protocol_gloo_equals_single_machine():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_protocol, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(res.values()) and len(res) == world
