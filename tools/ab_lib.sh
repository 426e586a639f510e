#!/usr/bin/env bash
# Interleaved A/B of two builds of the library on one box (diagnostics):
#   tools/ab_lib.sh N REPS OTHER_SO   (libokt.so vs OTHER_SO through OKT_LIB_PATH)
N=${1:-2}; R=${2:-2}; B=${3:-paper_2201_07598_b200/libokt_base.so}
run() { env $3 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 \
  bench.py --gpus $N --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', $N, round(d['ms_per_step'],4), round(d['steady_ms'],4))"; }
for i in $(seq 1 $R); do
  run $((29900 + i)) new ""
  run $((29950 + i)) base "OKT_LIB_PATH=$PWD/$B"
done
