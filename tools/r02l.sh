#!/bin/bash
# Attribution of the QAOA30 pass costs (QK_EXP_SKIP drops op kinds: timing only)
# and the two-group / 8-amplitude consumer variants.
T=gpurun_out/r02l; mkdir -p $T
for cfg in "" "QK_EXP_SKIP=1" "QK_EXP_SKIP=2" "QK_EXP_SKIP=3" "QK_EXP_SKIP=7" "QK_NG2=1" "QK_NG2=1 QK_EXP_SKIP=7" "QK_M=3" "QK_NG2=1 QK_JIT_MAXNREG=96"; do
  echo "== $cfg" >> $T/times.txt
  env $cfg QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py qaoa30 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
