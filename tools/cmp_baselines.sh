set -x
mkdir -p gpurun_out/cmp
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 600 python tools/bench_baselines.py --steps 16 > gpurun_out/cmp/vgg_n$N.jsonl 2> gpurun_out/cmp/vgg_n$N.err;
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tools/bench_baselines.py --steps 16 > gpurun_out/cmp/vgg_n$N.jsonl 2> gpurun_out/cmp/vgg_n$N.err; fi
  cat gpurun_out/cmp/vgg_n$N.jsonl; tail -3 gpurun_out/cmp/vgg_n$N.err
done
