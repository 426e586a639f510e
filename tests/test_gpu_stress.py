"""GPU, one process per GPU (torchrun): a few hundred EF-SGD steps through the
device-driven P2P step must reproduce the host-synchronised NCCL path bit for
bit on every step (u) and in the final model (tools/stress_p2p.py; the round's
long runs are in profiles/r01_stress_p2p.jsonl)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("P", [2, 4])
def test_p2p_matches_nccl_path_over_many_steps(gpus, P):
    if gpus < P:
        pytest.skip(f"needs {P} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tools", "stress_p2p.py"), "300", "300000", "0.01"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert '"mismatched_steps": 0' in out.stdout and '"model_mismatch_ranks": 0' in out.stdout, out.stdout
