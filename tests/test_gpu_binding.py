"""GPU: the reference library's own C++ types and calls, routed through the
reference-side binding include/dgkr/b200_binding.hpp (what INTEGRATION.md
asks a maintainer to add), prove byte-identically to the reference prover and
the reference verifier accepts the GPU proofs. The test binary is built here
from the reference headers (oracle/Makefile) and shipped prebuilt."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "binding_test")


def test_reference_types_through_binding():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/binding_test not built (needs /root/reference at build time)")
    res = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "binding ok" in res.stdout
