#!/usr/bin/env bash
# SURVEY 8(d) / BASELINE configs[4]: n = 1M..1B and density 0.1%..5% at
# N = 1..MAXG GPUs, one bench line per (config, N) into OUT/sweep.jsonl: the
# tau'-amortised ms/iter (steady / refresh split), dense-equivalent GB/s, the
# dense NCCL allreduce of the same gradient (N > 1), K1's HBM roofline, the
# NVLink bytes per phase (N > 1), and at N = 1 the reference's CPU path timed
# beside it (bounded sample: t = 1 refresh + steady iterations, one core).
#   tools/sweep.sh OUTDIR MAXGPUS [configs...]
set -u
OUT=${1:-gpurun_out/sweep}
MAXG=${2:-1}
shift 2 || true
mkdir -p "$OUT"
run_cfg() {  # name n density steps cpu_iters ring
  local name=$1 n=$2 dens=$3 steps=$4 cpui=$5 ring=$6 N=${SWEEP_MIN_N:-1}  # (SWEEP_MIN_N: first N of the doubling)
  while [ "$N" -le "$MAXG" ]; do
    if [ "$N" -eq 1 ]; then
      local cpu="--cpu-iters $cpui"
      [ -n "${SWEEP_NO_CPU:-}" ] && cpu="--no-cpu-baseline"  # (SWEEP_NO_CPU=1: skip the reference's CPU leg)
      timeout 1500 python bench.py --elements "$n" --density "$dens" --steps "$steps" --warmup 3 --ring-max "$ring" \
          $cpu --e2e-steps 3 > "$OUT/${name}_n$N.log" 2>&1
    else
      timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
          --master-port $((29850 + N)) bench.py --gpus "$N" --elements "$n" --density "$dens" --steps "$steps" \
          --warmup 3 --ring-max "$ring" --e2e-steps 3 > "$OUT/${name}_n$N.log" 2>&1
    fi
    grep '^{' "$OUT/${name}_n$N.log" | sed "s/^{/{\"sweep\": \"$name\", /" >> "$OUT/sweep.jsonl"
    N=$((N * 2))
  done
}
ALL="1m_1pct vgg_1pct lstm_2pct 100m_0p1pct 100m_1pct 100m_5pct bertl_1pct 1b_1pct"
CFGS=${*:-$ALL}
for c in $CFGS; do
  case $c in
    1m_1pct)     run_cfg 1m_1pct 1000000 0.01 34 34 24 ;;
    vgg_1pct)    run_cfg vgg_1pct 14728266 0.01 34 8 24 ;;
    lstm_2pct)   run_cfg lstm_2pct 27569568 0.02 34 6 24 ;;
    100m_0p1pct) run_cfg 100m_0p1pct 100000000 0.001 20 3 20 ;;
    100m_1pct)   run_cfg 100m_1pct 100000000 0.01 20 3 20 ;;
    100m_5pct)   run_cfg 100m_5pct 100000000 0.05 20 3 20 ;;
    bertl_1pct)  run_cfg bertl_1pct 340000000 0.01 20 3 12 ;;
    1b_1pct)     run_cfg 1b_1pct 1000000000 0.01 8 2 4 ;;
  esac
done
echo done >&2
