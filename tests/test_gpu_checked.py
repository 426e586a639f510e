"""The checked build (libokt_checked.so: device-side invariant traps, see
OKT_DCHECK in paper_2201_07598_b200/csrc/okt_device.cuh) over every step
shape — the single-rank step, the host-synchronised two-rank step and the
device-driven P2P step with two ranks on one GPU — each also checked against
the oracle.  compute-sanitizer is refused on the GPU pool (see
test_gpu_sanitizer.py), so this is the memory-safety evidence that runs there."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
CHECKED = os.path.join(os.path.dirname(HERE), "paper_2201_07598_b200", "libokt_checked.so")


@pytest.mark.parametrize("mode", ["single", "hostsync", "p2p"])
def test_checked_build_clean(gpus, mode):
    if not os.path.exists(CHECKED):
        pytest.skip("libokt_checked.so not built (make -C paper_2201_07598_b200/csrc DEBUG_CHECKS=1)")
    env = dict(os.environ, OKT_LIB_PATH=CHECKED)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_sanitize_run.py"), mode], env=env, capture_output=True,
                       text=True, timeout=900)
    out = r.stdout + r.stderr
    assert "OKT_DCHECK failed" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    assert f"ok {mode}" in out, out[-2000:]
