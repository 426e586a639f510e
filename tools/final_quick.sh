#!/usr/bin/env bash
# Round-end measurement on one box with MAXG GPUs, okt arm only (the reference arm's lines come from
# tools/final_lines.sh): bench lines at N = 1..MAXG with P2P traces, the N = 1 launch list, the multi-GPU tests,
# per-call NCCL parity at VGG with MAXG ranks, smoke.     tools/final_quick.sh OUTDIR MAXG
set -u
OUT=${1:-gpurun_out/final_quick}
MAXG=${2:-4}
mkdir -p "$OUT"
timeout 900 python bench.py > "$OUT/bench_n1.log" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 300 --csv --log-file "$OUT/launches_n1.csv" python bench.py --steps 6 --warmup 3 --no-cpu-baseline \
    --e2e-steps 2 > "$OUT/ncu_list.log" 2>&1
N=2
while [ "$N" -le "$MAXG" ]; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29840 + N)) bench.py --gpus $N --p2p-trace "$OUT/p2p_bert_n$N" > "$OUT/bench_n$N.log" 2>&1
  N=$((N * 2))
done
timeout 1200 python -m pytest tests -m gpu -x -q -k "nccl or p2p or stress or ddp or robustness" \
    > "$OUT/pytest_multi_n$MAXG.log" 2>&1; echo "pytest_exit=$?" >> "$OUT/pytest_multi_n$MAXG.log"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $MAXG --master-addr 127.0.0.1 \
    --master-port 29850 tools/parity_configs_nccl.py --elements 14728266 --density 0.01 --iters 34 \
    --out "$OUT/parity_vgg_n$MAXG.jsonl" > "$OUT/parity_vgg_n$MAXG.log" 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke_exit=$?" >> "$OUT/smoke.log"
echo done
