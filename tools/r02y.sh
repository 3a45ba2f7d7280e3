#!/bin/bash
# factor-order variant (bit 4) in the autotuner: per-pass times, bench lines, parity
T=gpurun_out/r02y; mkdir -p $T
for w in qaoa30 qft33 qft30; do
  echo "== $w" >> $T/times.txt
  QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py $w 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
timeout 600 python bench.py --no-cpu > $T/bench_qaoa30.json 2> $T/bench.err
for w in qft33 bv33 h33 u33; do
  timeout 400 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu >> $T/bench_all.json 2>> $T/bench_all.err
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x > $T/tests.log 2>&1; echo "rc=$?" >> $T/tests.log
