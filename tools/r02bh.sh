#!/bin/bash
# stage cap without the dense-gate condition: default vs the old cap vs no caps
T=gpurun_out/r02bh; mkdir -p $T
for w in qaoa30 qft33 u33 bv33 qft30 qaoa33r3; do
  for cfg in "" "QK_SMAX_MAT=1" "QK_NO_SMAX=1"; do
    echo "== $cfg $w" >> $T/times.txt
    env $cfg QK_JIT_CACHE=/tmp/jitc timeout 600 python tools/pass_times.py $w 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
  done
done
