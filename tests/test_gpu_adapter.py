"""GPU: the reference-side C++ binding (include/okt_oklab.hpp) runs the
reference's own scenarios next to the reference itself (both linked into
oracle/_ref/adapter_parity, built where /root/reference exists) and every
result, OkState and ledger row must match."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_parity")


def test_oklab_adapter_matches_reference(gpus):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/adapter_parity not built")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failing scenarios" in out.stdout
