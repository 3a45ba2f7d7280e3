#!/bin/bash
# 256-B row segments (QK_ROWBITS=4: bits 0..3 in every tile) against 128-B rows, per workload.
T=gpurun_out/r02bn
mkdir -p $T
for w in qft30 qft33 bv33 h33 u33 rzz33 bv30 h30 qaoa30; do
  for rb in 3 4; do
    QK_ROWBITS=$rb timeout 400 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu > $T/bench_${w}_rb$rb.json 2> $T/bench_${w}_rb$rb.err
  done
done
QK_ROWBITS=4 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -rfE > $T/pytest_rb4.log 2>&1; echo "rc=$?" >> $T/pytest_rb4.log
ls -la $T
