"""GPU: the multi-process (one process per rank) data-parallel prover over
the shared-memory transport, two ranks sharing this one GPU. Ranks exchange
only through host shared memory (no kernel waits on another). Rank 0's
proofs must equal the single-GPU proof of the full circuit."""
import os
import secrets
import subprocess
import sys

import pytest

import paper_2404_10404_b200 as P
from paper_2404_10404_b200 import workloads as W

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("lanes,n", [(1, 1), (2, 4)])
def test_two_process_shm_equals_single(ctx, tmp_path, lanes, n):
    world = 2
    token = secrets.token_hex(4)
    out = str(tmp_path / "proofs.bin")
    worker = os.path.join(ROOT, "tools", "dist_shm_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), token, str(lanes), str(n), out],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    logs = [p.communicate(timeout=300)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    f = P.Field.bn254()
    insz, flat = W.layered_circuit(seed=51, log_width=8, depth=5)
    inputs = W.random_inputs(f.p, insz * 8, 52)
    tr = P.Transcript(f, "shm")
    want = P.gkr_prove(ctx, P.Circuit(ctx, insz, *flat, n_copies=8), inputs, tr)
    raw = open(out, "rb").read()
    pos = 0
    for _ in range(n):
        ln = int.from_bytes(raw[pos:pos + 8], "little")
        proof, state = raw[pos + 8:pos + 8 + ln], raw[pos + 8 + ln:pos + 8 + ln + 32]
        pos += 8 + ln + 32
        assert proof == want and state == tr.state


def test_two_process_shm_spread_absorb(ctx, tmp_path):
    """absorb_policy 1: proof i's outputs are gathered to and absorbed on rank
    i mod 2; that rank's copy equals the single-GPU proof, the other rank's
    copy differs only by the zeroed output section, transcripts agree."""
    world, lanes, n = 2, 2, 4
    token = secrets.token_hex(4)
    out = str(tmp_path / "proofs.bin")
    worker = os.path.join(ROOT, "tools", "dist_shm_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), token, str(lanes), str(n), out, "spread"],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    logs = [p.communicate(timeout=300)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    f = P.Field.bn254()
    insz, flat = W.layered_circuit(seed=51, log_width=8, depth=5)
    inputs = W.random_inputs(f.p, insz * 8, 52)
    tr = P.Transcript(f, "shm")
    want = P.gkr_prove(ctx, P.Circuit(ctx, insz, *flat, n_copies=8), inputs, tr)
    n_out_bytes = 4 + int.from_bytes(want[:4], "little") * f.width

    def read(path):
        raw, pos, res = open(path, "rb").read(), 0, []
        for _ in range(n):
            ln = int.from_bytes(raw[pos:pos + 8], "little")
            res.append((raw[pos + 8:pos + 8 + ln], raw[pos + 8 + ln:pos + 8 + ln + 32]))
            pos += 8 + ln + 32
        return res

    per_rank = [read(f"{out}.{r}") for r in range(world)]
    for i in range(n):
        for r in range(world):
            proof, state = per_rank[r][i]
            assert state == tr.state
            if r == i % world:
                assert proof == want
            else:
                assert proof[n_out_bytes:] == want[n_out_bytes:] and not any(proof[4:n_out_bytes])


@pytest.mark.parametrize("world,vars_,n_pairs", [(2, 9, 2), (4, 13, 1)])
def test_dist_sumcheck_processes_over_shm(ctx, tmp_path, world, vars_, n_pairs):
    """dgkr_dist_sumcheck_comm with one process per rank (all on this GPU),
    round sums and the early-boundary table gather through shared memory
    (4 KiB slots: chunked): every rank returns the single-machine proof"""
    token = secrets.token_hex(4)
    out = str(tmp_path / "dsc")
    worker = os.path.join(ROOT, "tools", "dsc_shm_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), token, str(vars_), str(n_pairs), out],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    logs = [p.communicate(timeout=300)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    f = P.Field.bn254()
    tabs = [W.random_inputs(f.p, 1 << vars_, 300 + t).tobytes() for t in range(2 * n_pairs)]
    pairs = [(tabs[2 * k], tabs[2 * k + 1]) for k in range(n_pairs)]
    tr = P.Transcript(f, "dsc.shm")
    want = P.prove_product_sum(ctx, pairs, tr)
    for r in range(world):
        raw = open(f"{out}.{r}", "rb").read()
        assert raw[:-32] == want and raw[-32:] == tr.state
