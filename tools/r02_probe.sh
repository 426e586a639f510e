#!/usr/bin/env bash
# Round-2 first probe: box facts, GPU tests, and the BERT-L-sized N=1 step of
# the round-1 code (bench line, launch list, full captures of K1 and phase B).
set -u
OUT=gpurun_out/r02a
mkdir -p "$OUT"
{ nproc; free -g; lscpu | head -20; nvidia-smi; } > "$OUT/box.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest_exit=$?" >> "$OUT/pytest_gpu.log"
BN="--n 340000000 --ring 4 --no-cpu-baseline"
timeout 600 python bench.py $BN --steps 40 --warmup 5 > "$OUT/bench_bert.log" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file "$OUT/launches_bert.csv" python bench.py $BN --steps 4 --warmup 3 > "$OUT/ncu_list.log" 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:compact_kernel --launch-skip 5 \
    --launch-count 1 -o "$OUT/compact_full" python bench.py $BN --steps 4 --warmup 3 > "$OUT/ncu_compact.log" 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k1_kernel --launch-skip 6 \
    --launch-count 1 -o "$OUT/k1_full" python bench.py $BN --steps 4 --warmup 3 > "$OUT/ncu_k1.log" 2>&1
echo done
