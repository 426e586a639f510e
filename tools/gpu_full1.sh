#!/usr/bin/env bash
# 1-GPU validation + evidence: the whole GPU suite, smoke, the bench line, the
# ncu launch list and full captures of the N = 1 kernels.  usage: tools/gpu_full1.sh OUTDIR
set -u
OUT=${1:-gpurun_out/full1}
mkdir -p "$OUT"
timeout 2400 python -m pytest tests -m gpu -q -x > "$OUT/pytest_gpu.log" 2>&1; echo "pytest_exit=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke_exit=$?" >> "$OUT/smoke.log"
timeout 900 python bench.py > "$OUT/bench_n1.log" 2>&1
timeout 900 python bench.py --impl reference > "$OUT/ref_n1.log" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file "$OUT/launches_n1.csv" python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 2 \
    > "$OUT/ncu_list.log" 2>&1
bash tools/ncu_n1.sh "$OUT/ncu"
echo done
