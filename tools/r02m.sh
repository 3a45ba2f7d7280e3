#!/bin/bash
# QAOA30 per-pass times: two consumer groups (120 registers), L2 prefetch,
# stage count and chunk order, each also with every op dropped (data movement only)
T=gpurun_out/r02m; mkdir -p $T
for cfg in "" "QK_NG2=1" "QK_NG2=1 QK_EXP_SKIP=7" "QK_EXP_SKIP=7" "QK_JIT_PREFETCH=1" "QK_JIT_PREFETCH=1 QK_EXP_SKIP=7" "QK_SMAX=2 QK_EXP_SKIP=7" "QK_NO_CORDER=1 QK_EXP_SKIP=7" "QK_NG2=1 QK_JIT_PREFETCH=1"; do
  echo "== $cfg" >> $T/times.txt
  env $cfg QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py qaoa30 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
