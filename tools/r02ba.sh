#!/bin/bash
# ncu of QFT33's last (full) pass, application replay (128 GiB state)
T=gpurun_out/r02ba; mkdir -p $T
QK_NO_TUNE=1 timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:qk_jit --launch-skip 3 -c 1 -o /tmp/q33 \
  python tools/one_run.py qft33 > $T/ncu.log 2>&1
python tools/ncu_summary.py report /tmp/q33.ncu-rep > $T/summary.txt 2>&1
ncu -i /tmp/q33.ncu-rep --page source --csv --print-source sass > /tmp/q33src.csv 2>/dev/null; gzip -c /tmp/q33src.csv > $T/source_sass.csv.gz
