#!/bin/bash
# five register qubits (QK_M5): timing and parity
T=gpurun_out/r02al; mkdir -p $T
for w in qaoa30 qft33 u33; do
  for cfg in "" "QK_M5=1"; do
    echo "== $cfg $w" >> $T/times.txt
    env $cfg QK_JIT_CACHE=/tmp/jitc timeout 600 python tools/pass_times.py $w 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
  done
done
QK_M5=1 timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -rfE > $T/tests_m5.log 2>&1; echo "rc=$?" >> $T/tests_m5.log
