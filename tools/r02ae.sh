#!/bin/bash
# TMA-store epilogue through an unbounded store view (bounded zero-support passes too) vs the register-store twin on bounded passes
T=gpurun_out/r02ae; mkdir -p $T
for w in qaoa30 qft33 h33 u33 bv33; do
  for cfg in "" "QK_TSTORE_TWIN=1"; do
    echo "== $cfg $w" >> $T/times.txt

    env $cfg QK_JIT_CACHE=/tmp/jitc timeout 600 python tools/pass_times.py $w 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
  done
done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_multidev.py -q -x -rfE > $T/tests.log 2>&1; echo "rc=$?" >> $T/tests.log
timeout 900 python bench.py --no-cpu > $T/bench_qaoa30.json 2> $T/bench.err
