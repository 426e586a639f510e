#!/usr/bin/env bash
# Round-end bench lines only (okt + reference arm) at N = 1..MAXG, P2P traces,
# N = 1 launch list.   tools/final_lines.sh OUTDIR MAXG
set -u
OUT=${1:-gpurun_out/final_lines}
MAXG=${2:-4}
mkdir -p "$OUT"
timeout 900 python bench.py > "$OUT/bench_n1.log" 2>&1
timeout 900 python bench.py --impl reference > "$OUT/ref_n1.log" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 300 --csv --log-file "$OUT/launches_n1.csv" python bench.py --steps 6 --warmup 3 --no-cpu-baseline \
    --e2e-steps 2 > "$OUT/ncu_list.log" 2>&1
N=2
while [ "$N" -le "$MAXG" ]; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
  timeout 900 $TR --master-port $((29640 + N)) bench.py --gpus $N --p2p-trace "$OUT/p2p_bert_n$N" \
      > "$OUT/bench_n$N.log" 2>&1
  timeout 1500 $TR --master-port $((29650 + N)) bench.py --gpus $N --impl reference > "$OUT/ref_n$N.log" 2>&1
  N=$((N * 2))
done
echo done
