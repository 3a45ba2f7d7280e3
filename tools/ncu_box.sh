#!/bin/bash
# Capture an ncu --set full report on the GPU box and keep only text summaries
# (the .ncu-rep of 24 passes is ~100 MB, over gpurun's copy-back limit).
#   gpurun -- 'bash tools/ncu_box.sh <tag> <kernel regex> <count> <cmd...>'
T=gpurun_out/$1; K=$2; C=$3; shift 3
mkdir -p $T
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$K -c $C -o /tmp/rep "$@" > $T/ncu.log 2>&1
python tools/ncu_summary.py report /tmp/rep.ncu-rep > $T/summary.txt 2>&1
ncu -i /tmp/rep.ncu-rep --page raw --csv > /tmp/raw.csv 2>/dev/null; gzip -c /tmp/raw.csv > $T/raw.csv.gz
ls -la $T
