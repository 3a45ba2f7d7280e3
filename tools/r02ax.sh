#!/bin/bash
# bench lines with the full-sweep transparency measurement
T=gpurun_out/r02ax; mkdir -p $T
timeout 900 python bench.py > $T/bench_default.json 2> $T/bench_default.err
for w in qft30 bv33 h33 rzz33 u33 qft33 qaoa33r3; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu >> $T/bench_all.json 2>> $T/bench_all.err
done
