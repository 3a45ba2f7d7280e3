#!/bin/bash
# phase-count sensitivity of the QAOA30 passes (QK_EXP_MAXPH drops phases: timing only)
T=gpurun_out/r02aj; mkdir -p $T
for cfg in "" "QK_EXP_MAXPH=3" "QK_EXP_MAXPH=4" "QK_EXP_MAXPH=2"; do
  echo "== $cfg" >> $T/times.txt
  env $cfg QK_JIT_CACHE=/tmp/jitc timeout 600 python tools/pass_times.py qaoa30 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
