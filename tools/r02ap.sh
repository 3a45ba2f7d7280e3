#!/bin/bash
# M=5: repeatability and sanitizer checks
T=gpurun_out/r02ap; mkdir -p $T
for k in 1 2 3 4 5 6; do
  echo "== run $k" >> $T/log.txt
  QK_M5=1 QK_JIT_VARIANT=0 QK_NO_TUNE=1 timeout 300 python tools/one_run.py qaoa30 >> $T/log.txt 2>&1
done
QK_M5=1 QK_JIT_VARIANT=0 QK_NO_TUNE=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python tools/one_run.py qaoa24 > $T/synccheck.txt 2>&1
for cfg in "" "QK_M5=1"; do
  echo "== $cfg qaoa30" >> $T/times.txt
  env $cfg QK_JIT_CACHE=/tmp/jitc timeout 600 python tools/pass_times.py qaoa30 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
