#!/bin/bash
# ncu evidence beyond the headline passes: QAOA30 pass 3 source-level (bank
# conflicts), one H33 pass and the QAOA33r3 fix-up SQS (application replay: the
# 128 GiB state is too large to save per kernel replay), the group exchange kernels.
T=gpurun_out/r02w; mkdir -p $T
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_jit --launch-skip 81 -c 1 -o /tmp/p3 \
  python tools/pass_times.py qaoa30 > $T/p3.log 2>&1
python tools/ncu_summary.py report /tmp/p3.ncu-rep > $T/p3_summary.txt 2>&1
ncu -i /tmp/p3.ncu-rep --page source --csv --print-source sass > /tmp/p3src.csv 2>/dev/null; gzip -c /tmp/p3src.csv > $T/p3_source_sass.csv.gz
QK_NO_TUNE=1 timeout 1500 ncu --set full --clock-control none --replay-mode application -k regex:qk_jit --launch-skip 1 -c 1 -o /tmp/h33 \
  python tools/one_run.py h33 > $T/h33.log 2>&1
python tools/ncu_summary.py report /tmp/h33.ncu-rep > $T/h33_summary.txt 2>&1
QK_NO_TUNE=1 timeout 1500 ncu --set full --clock-control none --replay-mode application -k regex:sqs -c 1 -o /tmp/sqs33 \
  python tools/one_run.py qaoa33r3 > $T/sqs33.log 2>&1
python tools/ncu_summary.py report /tmp/sqs33.ncu-rep > $T/sqs33_summary.txt 2>&1
QK_HOST_BARRIER=1 QK_NO_OVERLAP=1 QK_NO_TUNE=1 timeout 900 ncu --set full --clock-control none -k regex:swap -c 2 -o /tmp/xrs \
  python tools/xrs_probe.py qaoa31_c12_r1 > $T/xrs.log 2>&1
python tools/ncu_summary.py report /tmp/xrs.ncu-rep > $T/xrs_summary.txt 2>&1
QK_NO_TUNE=1 RUNS=3 timeout 600 python tools/xrs_probe.py qaoa31_c12_r1 > $T/xrs_times.txt 2>&1
ls -la $T
