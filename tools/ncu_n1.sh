#!/usr/bin/env bash
# Full ncu captures of the N = 1 step's kernels (one launch each, after
# warm-up) + a CUPTI timeline of 16 steps.  usage: tools/ncu_n1.sh OUTDIR [bench args]
set -u
OUT=${1:-gpurun_out/ncu}
shift || true
mkdir -p "$OUT"
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 2 $*"
cap() {  # name regex skip
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$2" --launch-skip "$3" \
      --launch-count 1 -o "$OUT/$1" $B > "$OUT/ncu_$1.log" 2>&1
  ncu -i "$OUT/$1.ncu-rep" --page raw --csv > "$OUT/$1_raw.csv" 2>/dev/null
}
cap k1_steady 'k1_kernel<.bool.1, .bool.1, .bool.0, .bool.1, .bool.1' 3
cap phaseb 'compact_kernel<.int.1, .bool.1>' 3
cap k1_refresh_select 'k1_kernel<.bool.0, .bool.1, .bool.0, .bool.1, .bool.1' 1
cap k1_hist 'k1_kernel<.bool.1, .bool.0, .bool.1' 1
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 2 --trace "$OUT/trace" $* > "$OUT/trace.log" 2>&1
echo done
