"""One rank of a multi-process distributed product sum-check over the
shared-memory transport (dgkr_dist_sumcheck_comm): this rank's shard_pairs
slice (cluster.hpp:190-217) on the local GPU, round sums through host shared
memory. Used by tests/test_gpu_dist_shm.py (ranks share this pool's one GPU).
usage: dsc_shm_worker.py rank world token vars n_pairs out"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2404_10404_b200 as P  # noqa: E402
from paper_2404_10404_b200 import workloads as W  # noqa: E402
from paper_2404_10404_b200._lib import check, lib  # noqa: E402
from paper_2404_10404_b200.dist import ShmComm  # noqa: E402

rank, world, token, vars_, n_pairs, out = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]),
                                           int(sys.argv[5]), sys.argv[6])
ctx = P.Context(0)
f = P.Field.bn254()
tabs = [W.random_inputs(f.p, 1 << vars_, 300 + t).tobytes() for t in range(2 * n_pairs)]  # f_0 g_0 f_1 g_1 ...
lv = vars_ - (world.bit_length() - 1)
chunk = (32 << lv)
mine = b"".join(t[rank * chunk:(rank + 1) * chunk] for t in tabs)
comm = ShmComm(ctx, f"/dgkr_dsc_{token}", rank, world, 4096)  # small slots: the table gather runs chunked
tr = P.Transcript(f, "dsc.shm")
cap = 64 + (vars_ + 2) * 4 * 32 + 2 * n_pairs * 32 + 64
buf = C.create_string_buffer(cap)
ln = C.c_size_t()
check(lib().dgkr_dist_sumcheck_comm(ctx.handle, comm.handle, f.handle, C.c_size_t(n_pairs), C.c_size_t(lv),
                                    C.c_char_p(mine), C.byref(tr.t), buf, C.c_size_t(cap), C.byref(ln)))
with open(f"{out}.{rank}", "wb") as fh:
    fh.write(buf.raw[: ln.value] + tr.state)
print("rank", rank, "ok")
