#!/bin/bash
T=gpurun_out/r02e; mkdir -p $T
timeout 600 python tools/rb_check.py qft20_c10_r0 qaoa24_c12_r0 qft26_c10_r0 qaoa26_c12_r0 > $T/rb_check.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $T/bench_qaoa30.json 2> $T/bench.err
for w in rzz33 qft33 h33 bv33 u33 qft30 qaoa33r3 qft20; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu >> $T/bench_all.json 2>> $T/bench_all.err
done
QK_DUMP_PLAN=1 timeout 300 python tools/pass_times.py qaoa30 > $T/times_qaoa30.txt 2>&1
bash tools/ncu_box.sh r02e/full_qaoa30 qk_jit 13 python tools/pass_times.py qaoa30
