#!/bin/bash
T=gpurun_out/r02g; mkdir -p $T
for cfg in "" "QK_NG2=1" "QK_NG2=1 QK_NG2_EVEN=1"; do
  echo "== $cfg" >> $T/times.txt
  env $cfg timeout 300 python tools/pass_times.py qaoa30 2>&1 | grep "instr .* ms\|run" >> $T/times.txt
done
QK_NG2=1 timeout 600 python tools/rb_check.py qaoa24_c12_r0 qaoa26_c12_r0 >> $T/check.txt 2>&1
