#!/bin/bash
# 2-CTA cluster pairs for 128-B-row strided tiles (QK_PAIR)
T=gpurun_out/r02t; mkdir -p $T
for cfg in "" "QK_PAIR=1" "QK_EXP_SKIP=7" "QK_PAIR=1 QK_EXP_SKIP=7"; do
  echo "== $cfg" >> $T/times.txt
  env $cfg QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py qaoa30 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
for w in qft30 bv30 h30 qft33 h33; do
  echo "== $w" >> $T/times.txt
  QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py $w 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
  echo "== QK_PAIR=1 $w" >> $T/times.txt
  QK_PAIR=1 QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py $w 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
QK_PAIR=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > $T/fullsize.log 2>&1; echo "rc=$?" >> $T/fullsize.log
QK_PAIR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "random_streams or golden or strategies or lazy" > $T/parity.log 2>&1; echo "rc=$?" >> $T/parity.log
