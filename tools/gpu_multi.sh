#!/usr/bin/env bash
# Multi-GPU iteration (run with gpurun --gpus N): the multi-GPU tests, bench
# lines at BERT-L and VGG with per-CTA P2P traces, per-call NCCL parity at VGG.
# usage: tools/gpu_multi.sh OUTDIR N
set -u
OUT=${1:-gpurun_out/multi}
N=${2:-2}
mkdir -p "$OUT"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -x -q -k "nccl or p2p or stress or ddp or robustness" > "$OUT/pytest_multi.log" 2>&1
echo "pytest_exit=$?" >> "$OUT/pytest_multi.log"
timeout 900 $TR --master-port 29511 bench.py --gpus $N --p2p-trace "$OUT/p2p_bert" > "$OUT/bench_bert_n$N.log" 2>&1
timeout 900 $TR --master-port 29512 bench.py --gpus $N --elements 14728266 --p2p-trace "$OUT/p2p_vgg" > "$OUT/bench_vgg_n$N.log" 2>&1
timeout 1200 $TR --master-port 29513 tools/parity_configs_nccl.py --elements 14728266 --density 0.01 --iters 34 \
    --out "$OUT/parity_vgg_n$N.jsonl" > "$OUT/parity_vgg_n$N.log" 2>&1
echo done
