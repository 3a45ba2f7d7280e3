#!/bin/bash
# zero-chunk skipping in bounded passes: parity (full GPU suite) and timing
T=gpurun_out/r02ah; mkdir -p $T
( time timeout 1800 python -m pytest tests -m gpu -q -x -rfE ) > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
for w in qaoa30 qft33 bv33 qft30 bv30; do
  for cfg in "" "QK_NO_ZPLACE=1"; do
    echo "== $cfg $w" >> $T/times.txt
    env $cfg QK_JIT_CACHE=/tmp/jitc timeout 600 python tools/pass_times.py $w 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
  done
done
timeout 900 python bench.py --no-cpu > $T/bench_qaoa30.json 2> $T/bench.err
