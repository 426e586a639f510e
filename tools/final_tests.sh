#!/usr/bin/env bash
# Round-end test pass on a box with N GPUs: the whole GPU suite + smoke.
set -u
OUT=${1:-gpurun_out/final_tests}
mkdir -p "$OUT"
timeout 2700 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest_exit=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke_exit=$?" >> "$OUT/smoke.log"
echo done
