#!/usr/bin/env bash
# Quick multi-GPU timing: the BERT-L and VGG bench lines with per-CTA P2P traces.
# usage: tools/gpu_multi_quick.sh OUTDIR N [extra bench args]
set -u
OUT=${1:-gpurun_out/mq}
N=${2:-2}
shift 2 || true
mkdir -p "$OUT"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29521 bench.py --gpus $N --steps 12 --p2p-trace "$OUT/p2p_bert" $* > "$OUT/bench_bert_n$N.log" 2>&1
timeout 600 $TR --master-port 29522 bench.py --gpus $N --elements 14728266 --p2p-trace "$OUT/p2p_vgg" $* > "$OUT/bench_vgg_n$N.log" 2>&1
echo done
