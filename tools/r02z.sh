#!/bin/bash
# source-level ncu of QAOA30 pass 6 (strided 21..29, 5 phases) and pass 12 (strided 12..20, 3 phases)
# (9 tuning/warm runs x 13 launches precede the timed run)
T=gpurun_out/r02z; mkdir -p $T
for p in 6 12; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_jit --launch-skip $((117 + p)) -c 1 -o /tmp/p$p \
    python tools/pass_times.py qaoa30 > $T/p$p.log 2>&1
  python tools/ncu_summary.py report /tmp/p$p.ncu-rep > $T/p${p}_summary.txt 2>&1
  ncu -i /tmp/p$p.ncu-rep --page source --csv --print-source sass > /tmp/p${p}src.csv 2>/dev/null; gzip -c /tmp/p${p}src.csv > $T/p${p}_source_sass.csv.gz
done
ls -la $T
