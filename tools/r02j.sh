#!/bin/bash
T=gpurun_out/r02j; mkdir -p $T
timeout 600 python tools/rb_check.py qft20_c10_r0 qaoa24_c12_r0 qft26_c10_r0 > $T/check.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q > $T/fullsize.log 2>&1; echo "rc=$?" >> $T/fullsize.log
for w in qaoa30 qft33 qft30 bv33 qaoa33r3 h33 u33; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu >> $T/bench_all.json 2>> $T/bench_all.err
done
QK_DUMP_TIMES=1 timeout 300 python tools/plan_dump.py qft33_c10_r0 33 10 > $T/times_qft33.txt 2>&1
QK_DUMP_TIMES=1 timeout 300 python tools/plan_dump.py qaoa30_c12_r0 30 12 > $T/times_qaoa30.txt 2>&1
