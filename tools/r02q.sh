#!/bin/bash
# QUAD factors computed while the stage's TMA load is in flight; stage cap off/on
T=gpurun_out/r02q; mkdir -p $T
for cfg in "" "QK_NO_SMAX=1" "QK_SMAX=3"; do
  echo "== $cfg" >> $T/times.txt
  env $cfg QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py qaoa30 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > $T/fullsize.log 2>&1; echo "rc=$?" >> $T/fullsize.log
