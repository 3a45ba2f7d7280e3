#!/bin/bash
# stage count sensitivity of the QAOA30 passes
T=gpurun_out/r02bg; mkdir -p $T
for cfg in "" "QK_SMAX=2" "QK_NO_SMAX=1"; do
  echo "== $cfg qaoa30" >> $T/times.txt
  env $cfg QK_JIT_CACHE=/tmp/jitc timeout 600 python tools/pass_times.py qaoa30 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
