#!/usr/bin/env bash
# SURVEY 8(d) configurations beyond the headline VGG one, at N = 1..MAXG GPUs:
# one bench line per (config, N) into OUT/sweep.jsonl (device-resident
# ms/iter with steady / refresh split, dense-equivalent GB/s, the dense NCCL
# allreduce of the same gradient, K1's HBM roofline).
#   tools/sweep.sh OUTDIR MAXGPUS
set -u
OUT=${1:-gpurun_out/sweep}
MAXG=${2:-1}
mkdir -p "$OUT"
: > "$OUT/sweep.jsonl"
run_cfg() {  # name n density ring
  local name=$1 n=$2 dens=$3 ring=$4 N=1
  while [ "$N" -le "$MAXG" ]; do
    if [ "$N" -eq 1 ]; then
      timeout 900 python bench.py --elements "$n" --density "$dens" --ring "$ring" --steps 64 --warmup 8 \
          --no-cpu-baseline > "$OUT/${name}_n$N.log" 2>&1
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
          --master-port $((29850 + N)) bench.py --gpus "$N" --elements "$n" --density "$dens" --ring "$ring" \
          --steps 64 --warmup 8 > "$OUT/${name}_n$N.log" 2>&1
    fi
    grep '^{' "$OUT/${name}_n$N.log" | sed "s/^{/{\"sweep\": \"$name\", /" >> "$OUT/sweep.jsonl"
    N=$((N * 2))
  done
}
run_cfg 1m_1pct 1000000 0.01 8
run_cfg lstm_2pct 27569568 0.02 4
run_cfg bertl_1pct 340000000 0.01 2
echo done >&2
