#!/usr/bin/env bash
# A/B of one environment switch at N GPUs: the BERT-L bench line and per-CTA P2P traces per value.
# usage: tools/ab_env.sh OUTDIR N VAR "v1 v2 ..." [extra bench args]     (v = none: VAR unset)
set -u
OUT=${1:-gpurun_out/ab}; N=${2:-2}; VAR=$3; VALS=$4
shift 4
mkdir -p "$OUT"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29541; i=0
for v in $VALS; do
  i=$((i+1)); tag="${i}_$v"
  if [ "$v" = none ]; then unset "$VAR"; else export "$VAR=$v"; fi
  timeout 600 $TR --master-port $port bench.py --gpus $N --no-cpu-baseline --e2e-steps 2 "$@" > "$OUT/bench_n${N}_$tag.log" 2>&1; port=$((port+1))
  timeout 600 $TR --master-port $port bench.py --gpus $N --steps 12 --no-cpu-baseline --e2e-steps 2 \
    --p2p-trace "$OUT/p2p_n${N}_$tag" "$@" > "$OUT/trace_n${N}_$tag.log" 2>&1; port=$((port+1))
done
echo done
