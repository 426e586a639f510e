"""compute-sanitizer over every kernel family of the path at small n:
memcheck, racecheck (shared-memory hazards) and synccheck (barrier misuse)
on the single-rank step, the host-synchronised multi-rank step and the
device-driven P2P step (two ranks on one GPU).  Each run is also an oracle
parity check (tests/_sanitize_run.py)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

CASES = [(tool, mode) for tool in ("memcheck", "racecheck", "synccheck") for mode in ("single", "hostsync", "p2p")]


@pytest.mark.parametrize("tool,mode", CASES)
def test_compute_sanitizer_clean(gpus, tool, mode):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    cmd = [SAN, f"--tool={tool}", "--error-exitcode=99", "--target-processes=all"]
    if tool == "memcheck":
        cmd.append("--leak-check=no")
    cmd += [sys.executable, os.path.join(HERE, "_sanitize_run.py"), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:  # (the GPU pool's wrapper refuses compute-sanitizer runs)
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert r.returncode == 0, out[-6000:]
    assert f"ok {mode}" in out, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-3000:]
