#!/bin/bash
# ncu of QFT30's last (full) pass
T=gpurun_out/r02bd; mkdir -p $T
QK_NO_TUNE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_jit --launch-skip 2 -c 1 -o /tmp/q30 \
  python tools/one_run.py qft30 > $T/ncu.log 2>&1
python tools/ncu_summary.py report /tmp/q30.ncu-rep > $T/summary.txt 2>&1
ncu -i /tmp/q30.ncu-rep --page source --csv --print-source sass > /tmp/q30src.csv 2>/dev/null; gzip -c /tmp/q30src.csv > $T/source_sass.csv.gz
QK_DUMP_PHASES=1 QK_NO_TUNE=1 timeout 300 python tools/one_run.py qft30 > $T/phases.txt 2>&1
