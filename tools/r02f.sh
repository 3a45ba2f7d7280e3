#!/bin/bash
T=gpurun_out/r02f; mkdir -p $T
for cfg in "" "QK_NG2=1" "QK_NO_TAIL_MOVE=1"; do
  echo "== $cfg" >> $T/times.txt
  env $cfg timeout 300 python tools/pass_times.py qaoa30 2>&1 | grep "instr .* ms\|run" >> $T/times.txt
done
timeout 600 python tools/rb_check.py qaoa24_c12_r0 qft26_c10_r0 >> $T/check.txt 2>&1
QK_NG2=1 timeout 600 python tools/rb_check.py qaoa24_c12_r0 >> $T/check.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $T/bench_qaoa30.json 2> $T/bench.err
QK_NG2=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $T/bench_qaoa30_ng2.json 2>> $T/bench.err
for w in qft33 bv33 h33 rzz33; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu >> $T/bench_all.json 2>> $T/bench_all.err
done
