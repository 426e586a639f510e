#!/usr/bin/env bash
# Round-end multi-GPU measurement on one box with MAXG GPUs: bench lines (okt
# + reference arm) at N = 2..MAXG with per-CTA P2P traces, the per-call NCCL
# parity tool, and the sweep at N = 1..MAXG.   tools/final_multi.sh OUTDIR MAXG
set -u
OUT=${1:-gpurun_out/final_multi}
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
  timeout 900 $TR --master-port $((29600 + N)) bench.py --gpus $N --p2p-trace "$OUT/p2p_bert_n$N" \
      > "$OUT/bench_n$N.log" 2>&1
  timeout 1500 $TR --master-port $((29610 + N)) bench.py --gpus $N --impl reference > "$OUT/ref_n$N.log" 2>&1
  timeout 1200 $TR --master-port $((29620 + N)) tools/parity_configs_nccl.py --elements 14728266 --density 0.01 \
      --iters 34 --out "$OUT/parity_vgg_n$N.jsonl" > "$OUT/parity_vgg_n$N.log" 2>&1
  N=$((N * 2))
done
bash tools/sweep.sh "$OUT/sweep" "$MAXG"
echo done
