set -u
O=gpurun_out/r02s; mkdir -p $O
for v in none 32 64; do
  if [ $v = none ]; then unset OKT_L2_FETCH_BYTES; else export OKT_L2_FETCH_BYTES=$v; fi
  timeout 600 python bench.py --no-cpu-baseline --e2e-steps 2 > $O/bench_l2_$v.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file $O/launches_l2_$v.csv python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/ncu_l2_$v.log 2>&1
done
echo done
