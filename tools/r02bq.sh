#!/bin/bash
# QFT write-only passes: stage count (L1 room for the factor tables), factor
# hoisting budget, two consumer groups; per-pass times.
T=gpurun_out/r02bq
mkdir -p $T
for w in qft30 qft33; do
  for env in "X=0" "QK_SMAX=2" "QK_QHOIST=24" "QK_QHOIST=48" "QK_NG2=1" "QK_SMAX=2 QK_QHOIST=24"; do
    echo "== $w $env" >> $T/pass_times.txt
    env $env timeout 300 python tools/pass_times.py $w 2>&1 | grep "instr.*ms$" >> $T/pass_times.txt
  done
done
ls -la $T
