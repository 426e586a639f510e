#!/usr/bin/env bash
# One GPU iteration: tests, smoke, the default bench line, and the N = 1 launch
# list.  usage: tools/gpu_check.sh OUTDIR [pytest -k expr]
set -u
OUT=${1:-gpurun_out/chk}
mkdir -p "$OUT"
K=${2:-}
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > "$OUT/pytest_gpu.log" 2>&1; echo "pytest_exit=$?" >> "$OUT/pytest_gpu.log"
else
  timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest_exit=$?" >> "$OUT/pytest_gpu.log"
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke_exit=$?" >> "$OUT/smoke.log"
timeout 900 python bench.py > "$OUT/bench_n1.log" 2>&1; echo "bench_exit=$?" >> "$OUT/bench_n1.log"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file "$OUT/launches_n1.csv" python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 2 \
    > "$OUT/ncu_list.log" 2>&1
echo done
