#!/bin/bash
# shard reblock with leaving wires kept off the low bits: parity, group and N=2 timing
T=gpurun_out/r02ac; mkdir -p $T
timeout 1200 python -m pytest tests/test_gpu_multidev.py tests/test_multiproc_gpu.py tests/test_gpu_fullsize.py -q -x -rfE > $T/tests.log 2>&1; echo "rc=$?" >> $T/tests.log
for cfg in "" "QK_NO_XREBLOCK=1"; do
  for c in qft33_c10_r1 qaoa31_c12_r1; do
    echo "== $cfg $c" >> $T/group.txt
    env $cfg QK_NO_TUNE=1 RUNS=3 timeout 600 python tools/xrs_probe.py $c >> $T/group.txt 2>&1
  done
  echo "== $cfg" >> $T/bench_n2.json
  env $cfg QK_INPLACE=1 QK_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29541 bench.py --gpus 2 --circuit qft33_c10_r1 --steps 2 --warmup 1 >> $T/bench_n2.json 2>> $T/bench_n2.err
done
