#!/bin/bash
# Cross-block pass scheduling (reblock) + OP_QUAD: plan, parity, bench.
T=gpurun_out/r02b
mkdir -p $T/src
export QK_JIT_VERBOSE=1
QK_JIT_DUMP=$T/src QK_DUMP_PLAN=1 timeout 300 python tools/plan_dump.py qaoa30_c12_r0 30 12 > $T/plan_qaoa30.txt 2>&1
echo "rc=$?" >> $T/plan_qaoa30.txt
ls $T/src | head -3 > /dev/null
QK_DUMP_PLAN=1 timeout 300 python tools/plan_dump.py qft33_c10_r0 33 10 > $T/plan_qft33.txt 2>&1
echo "rc=$?" >> $T/plan_qft33.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > $T/fullsize.log 2>&1; echo "rc=$?" >> $T/fullsize.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $T/bench_qaoa30.json 2> $T/bench.err
for w in qft33 bv33 h33 u33 rzz33 qft30 bv30 qaoa26 qaoa33r3; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu >> $T/bench_all.json 2>> $T/bench_all.err
done
timeout 1500 python -m pytest tests -m gpu -x -q > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
