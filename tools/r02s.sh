#!/bin/bash
# tuned per-pass times: QUAD factors of the next chunk computed before the stage wait (pending slot)
T=gpurun_out/r02s; mkdir -p $T
for cfg in "" "QK_LIB_PATH=scratch_cubins/old/libqkb200.so" "QK_EXP_SKIP=7"; do
  echo "== $cfg" >> $T/times.txt
  env $cfg QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py qaoa30 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > $T/fullsize.log 2>&1; echo "rc=$?" >> $T/fullsize.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "random_streams or golden or strategies" > $T/parity.log 2>&1; echo "rc=$?" >> $T/parity.log
