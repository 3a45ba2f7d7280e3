#!/bin/bash
# pj constants as kernel parameters: timing A/B and parity
T=gpurun_out/r02bb; mkdir -p $T
for w in qaoa30 qft33 qft30; do
  for cfg in "" "QK_NO_PJ_CONST=1"; do
    echo "== $cfg $w" >> $T/times.txt
    env $cfg QK_JIT_CACHE=/tmp/jitc timeout 600 python tools/pass_times.py $w 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
  done
done
( time timeout 1800 python -m pytest tests -m gpu -q -x -rfE ) > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
