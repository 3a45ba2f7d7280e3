#!/bin/bash
# ncu of the swap kernels: k_sqs (relabeled mode, QK_NO_LAZY12, in place) and
# the group exchange (device barriers; a barrier that cannot meet times out
# after 60 s with an error instead of hanging); QFT33 A/B vs the pre-pending-slot build
T=gpurun_out/r02x; mkdir -p $T
QK_NO_LAZY12=1 QK_INPLACE=1 QK_NO_TUNE=1 timeout 900 ncu --set full --clock-control none -k regex:sqs -c 2 -o /tmp/sqs \
  python tools/one_run.py qaoa30 > $T/sqs.log 2>&1
python tools/ncu_summary.py report /tmp/sqs.ncu-rep > $T/sqs_summary.txt 2>&1
QK_NO_OVERLAP=1 QK_NO_TUNE=1 timeout 600 ncu --set full --clock-control none -k regex:swap -c 2 -o /tmp/xrs \
  python tools/xrs_probe.py qaoa31_c12_r1 > $T/xrs.log 2>&1
python tools/ncu_summary.py report /tmp/xrs.ncu-rep > $T/xrs_summary.txt 2>&1
for cfg in "" "QK_LIB_PATH=scratch_cubins/old/libqkb200.so"; do
  echo "== $cfg qft33" >> $T/times.txt
  env $cfg QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py qft33 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
  echo "== $cfg qft30" >> $T/times.txt
  env $cfg QK_JIT_CACHE=/tmp/jitc timeout 300 python tools/pass_times.py qft30 2>&1 | grep "instr .* ms\|run\|rror" >> $T/times.txt
done
ls -la $T
