"""GPU: the reference's OWN unit tests (test_sumcheck.cpp, test_gkr.cpp,
test_pcs.cpp from /root/reference/proj/tests, unchanged) compiled against the
header-level drop-in (include/dropin: prove_product_sum, prove_layer_sum,
gkr_prove, pcs::commit / open on the B200 prover; oracle/Makefile
"dropin_test_*") must pass, with their verifiers and bit-level checks
running on the reference's code."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", ["sumcheck", "gkr", "pcs"])
def test_reference_suite_on_the_gpu_prover(name):
    exe = os.path.join(ROOT, "oracle", "_ref", f"dropin_test_{name}")
    if not os.path.exists(exe):
        pytest.skip("drop-in test binaries not built (make -C oracle, needs /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]


@pytest.mark.parametrize("args", [
    [],
    ["64", "3", "8", "7"],
    ["32", "4", "4", "1", "perturb-round-poly:1"],
    ["32", "4", "4", "1", "flip-sibling:2"],
    ["32", "4", "4", "1", "dup-index:0"],
    ["32", "4", "4", "1", "mempool-overwrite:3"],
])
def test_reference_epoch_pipeline_on_the_gpu_prover(args):
    """the reference's pipeline::run_epoch (pipeline.hpp) with gkr_prove and
    pcs::commit / open on the B200 prover reports exactly what the CPU
    reference reports: acceptance flags, final chain state, traffic, proof
    sizes - and rejects the same tampered blocks"""
    cpu = os.path.join(ROOT, "oracle", "_ref", "epoch_cpu")
    gpu = os.path.join(ROOT, "oracle", "_ref", "epoch_gpu")
    if not (os.path.exists(cpu) and os.path.exists(gpu)):
        pytest.skip("epoch drivers not built (make -C oracle, needs /root/reference)")
    a = subprocess.run([cpu, *args], capture_output=True, text=True, timeout=900)
    b = subprocess.run([gpu, *args], capture_output=True, text=True, timeout=900)
    assert a.returncode == 0 and b.returncode == 0, (a.stderr + b.stderr)[-3000:]
    assert a.stdout == b.stdout
    assert ('"all_accepted":true' in a.stdout) == (len(args) <= 4)


def test_pairsum_session_and_reference_dist_sumcheck_on_device_sessions():
    """PairSumSession (sumcheck.hpp:152-221) on the device through the drop-in,
    step by step against the reference's own session, and the reference's OWN
    dist_sumcheck (cluster.hpp:228-320) driving one device session per worker:
    byte-equal to the single-machine reference proof and to the C-ABI
    dist_sumcheck, N = 1..8, three fields (tests/cpp/pairsum_dropin_test.cpp)"""
    exe = os.path.join(ROOT, "oracle", "_ref", "pairsum_dropin_test")
    if not os.path.exists(exe):
        pytest.skip("pairsum drop-in test not built (make -C oracle, needs /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert ", 0 failures" in r.stdout
