#!/usr/bin/env bash
# Interleaved A/B of a diagnostics switch on one box:  tools/ab_env.sh N REPS VAR
# (runs bench.py with VAR unset, then VAR=0)
N=${1:-2}; R=${2:-2}; V=${3:-OKT_P2P_PULL_SPEC}
run() { env $3 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 \
  bench.py --gpus $N --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', $N, round(d['ms_per_step'],4), round(d['steady_ms'],4))"; }
for i in $(seq 1 $R); do
  run $((29800 + i)) on ""
  run $((29850 + i)) off "$V=0"
done
