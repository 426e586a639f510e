#!/usr/bin/env bash
# A/B of merge ring geometries (library variants via OKT_LIB_PATH) at N GPUs.
# Build the variants first, e.g.
#   make -C paper_2201_07598_b200/csrc OUT=../libokt_s6r128.so OBJDIR=../../build/okt_s6r128 \
#        EXTRA_FLAGS="-DOKT_MERGE_STAGES_SMALL=6 -DOKT_MERGE_RING=128"
set -u
OUT=${1:-gpurun_out/abm}
N=${2:-4}
mkdir -p "$OUT"
for v in libokt libokt_s6r128 libokt_s16r64; do
  OKT_LIB_PATH=$PWD/paper_2201_07598_b200/$v.so bash tools/gpu_multi_quick.sh "$OUT/$v" "$N"
done
echo done
