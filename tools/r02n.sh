#!/bin/bash
# QAOA30 per-pass times: two consumer groups at 112 registers; strided store vs contiguous store (timing only)
T=gpurun_out/r02n; mkdir -p $T
for cfg in "QK_NG2=1" "QK_NG2=1 QK_EXP_SKIP=7" "QK_EXP_SKIP=15" "QK_EXP_SKIP=8" "QK_NG2=1 QK_JIT_MAXNREG=120"; do
  echo "== $cfg" >> $T/times.txt
  env $cfg QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py qaoa30 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
