#!/bin/bash
# N=2 path of the driver's scaling run at HEAD (both ranks on the one device, gloo
# for the host collectives), after qk_reset stopped synchronising.
T=gpurun_out/r02bu
mkdir -p $T
QK_INPLACE=1 QK_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29541 bench.py --gpus 2 --circuit qft33_c10_r1 --steps 2 --warmup 1 > $T/bench_n2.json 2> $T/bench_n2.err
echo "rc=$?" >> $T/bench_n2.err
ls -la $T
