#!/usr/bin/env bash
# One measurement pass for the round's profiles/ (run on the GPU box from the
# repo root, with N GPUs visible):  tools/measure_round.sh OUTDIR MAXGPUS
# Bench lines (okt + reference arm) at N = 1..MAXGPUS, the ncu launch list of
# the N = 1 bench, and one `ncu --set full` capture of K1.
set -u
OUT=${1:-gpurun_out/meas}
MAXG=${2:-1}
mkdir -p "$OUT"
run() { echo "== $*" >&2; "$@"; }
run timeout 400 python bench.py > "$OUT/bench_n1.log" 2>&1
run timeout 400 python bench.py --impl reference > "$OUT/ref_n1.log" 2>&1
N=2
while [ "$N" -le "$MAXG" ]; do
  run timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
      --master-port $((29600 + N)) bench.py --gpus "$N" --p2p-trace "$OUT/p2p_n$N" > "$OUT/bench_n$N.log" 2>&1
  run timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
      --master-port $((29700 + N)) bench.py --gpus "$N" --impl reference > "$OUT/ref_n$N.log" 2>&1
  N=$((N * 2))
done
# launch list (cold-cache, serialised: shares, not absolutes) of the N = 1 bench command
run timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches_n1.csv" python bench.py --steps 4 --warmup 3 --no-cpu-baseline > "$OUT/ncu_list.log" 2>&1
# one full capture of the EF-step K1 (after warm-up)
run timeout 600 ncu --set full --import-source on --clock-control none -k regex:k1_kernel --launch-skip 12 \
    --launch-count 1 -o "$OUT/k1_full" python bench.py --steps 4 --warmup 3 --no-cpu-baseline > "$OUT/ncu_k1.log" 2>&1
echo done >&2
