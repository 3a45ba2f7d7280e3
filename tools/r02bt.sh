#!/bin/bash
# Per-pass QAOA30 times under launch-shape knobs (candidates for per-pass variants).
T=gpurun_out/r02bt
mkdir -p $T
for env in "X=0" "QK_PAIR=1" "QK_NG2=1" "QK_SMAX=2" "QK_SMAX=4"; do
  echo "== qaoa30 $env" >> $T/pass_times.txt
  env $env timeout 300 python tools/pass_times.py qaoa30 2>&1 | grep "instr.*ms$" >> $T/pass_times.txt
done
ls -la $T
