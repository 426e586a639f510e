#!/usr/bin/env bash
# Interleaved A/B of the argument-fed P2P EF step on one box (diagnostics):
#   tools/ab_argfed.sh N REPS
N=${1:-4}; R=${2:-2}
run() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 \
  bench.py --gpus $N --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', $N, round(d['ms_per_step'],4), round(d['steady_ms'],4), 'e2e', round(d['e2e']['value'],3), round(d['e2e']['ms_median'],3))"; }
for i in $(seq 1 $R); do
  run $((29700 + i)) argfed
  OKT_P2P_ARGFED=0 run $((29750 + i)) h2d
done
