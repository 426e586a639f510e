"""The device-driven (NVLink P2P) step at world sizes larger than the box:
P = 8 (and 4) ranks as threads of one process, two per GPU, with the P2P path
forced on through its test hooks.  The driver's 8-GPU scaling run takes this
path with one rank per GPU; here it is checked bit for bit against the oracle
(exact-sum EF trajectory, refreshes included)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("P", [4, 8])
def test_p2p_step_two_ranks_per_gpu(gpus, P):
    G = min(gpus, P // 2)
    if G < 2 or P % G:
        pytest.skip("needs at least 2 GPUs")
    env = dict(os.environ, OKT_P2P_ALLOW_SHARED="1", OKT_P2P_GRID_DIV=str(P // G), OKT_P2P_TRACE="1")
    r = subprocess.run([sys.executable, os.path.join(HERE, "_p2p_shared_run.py"), str(P), str(G)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert f"ok {P} {G}" in r.stdout
