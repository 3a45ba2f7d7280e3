#!/bin/bash
# N=2 bench path on one device (two processes, in place so both 64-GiB shards fit), shard reblock on/off
T=gpurun_out/r02ab; mkdir -p $T
for cfg in "" "QK_NO_XREBLOCK=1"; do
  echo "== $cfg" >> $T/bench_n2.json
  env $cfg QK_INPLACE=1 QK_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29541 bench.py --gpus 2 --circuit qft33_c10_r1 --steps 2 --warmup 1 >> $T/bench_n2.json 2>> $T/bench_n2.err
done
