#!/bin/bash
# tile padding of scheduled passes: 12 (default) vs 10 bits
T=gpurun_out/r02av; mkdir -p $T
for w in qft33 bv33 qft30 bv30 qaoa30 h33; do
  for cfg in "" "QK_PAD=10"; do
    echo "== $cfg $w" >> $T/times.txt
    env $cfg QK_JIT_CACHE=/tmp/jitc timeout 600 python tools/pass_times.py $w 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
  done
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > $T/fullsize.log 2>&1; echo "rc=$?" >> $T/fullsize.log
