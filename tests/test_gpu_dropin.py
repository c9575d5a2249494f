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
