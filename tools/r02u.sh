#!/bin/bash
# zero-support bounded reads (every pass of a run from reset reads only below 2^zbits)
T=gpurun_out/r02u; mkdir -p $T
for w in qaoa30 qft30 bv30 h30 qft33 h33 bv33 u33; do
  for cfg in "" "QK_NO_ZBOUND=1"; do
    echo "== $cfg $w" >> $T/times.txt
    env $cfg QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py $w 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
  done
done
( time timeout 1800 python -m pytest tests -m gpu -q -x -rfE ) > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
