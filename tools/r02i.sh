#!/bin/bash
T=gpurun_out/r02i; mkdir -p $T
QK_DUMP_TIMES=1 timeout 300 python tools/plan_dump.py qft33_c10_r0 33 10 > $T/times_qft33.txt 2>&1
QK_DUMP_TIMES=1 timeout 300 python tools/plan_dump.py qaoa30_c12_r0 30 12 > $T/times_qaoa30.txt 2>&1
timeout 600 python tools/rb_check.py qaoa24_c12_r0 qft26_c10_r0 > $T/check.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qk_jit -c 1 -o /tmp/qft0 python tools/plan_dump.py qft33_c10_r0 33 10 > $T/ncu.log 2>&1
python tools/ncu_summary.py report /tmp/qft0.ncu-rep > $T/summary.txt 2>&1
ncu -i /tmp/qft0.ncu-rep --page source --csv --print-source sass > /tmp/src.csv 2>/dev/null; gzip -c /tmp/src.csv > $T/source_sass.csv.gz
ncu -i /tmp/qft0.ncu-rep --page details --csv > $T/details.csv 2>/dev/null
