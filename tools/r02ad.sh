#!/bin/bash
# TMA-store epilogue (variant bit 8) in the autotuner: per-pass times with/without, parity
T=gpurun_out/r02ad; mkdir -p $T
for w in qaoa30 qft33 h33 u33 bv33; do
  for cfg in "" "QK_NO_TSTORE=1"; do
    echo "== $cfg $w" >> $T/times.txt
    env $cfg QK_DUMP_TUNE=1 QK_JIT_CACHE=/tmp/jitc timeout 600 python tools/pass_times.py $w >> $T/tune_$w.log 2>&1
    env $cfg QK_JIT_CACHE=/tmp/jitc timeout 600 python tools/pass_times.py $w 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
  done
done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_multidev.py -q -x -rfE > $T/tests.log 2>&1; echo "rc=$?" >> $T/tests.log
