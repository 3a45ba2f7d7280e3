#!/bin/bash
# OP_QLITE hoisting variant (bit 4 on passes without OP_QUAD) against HEAD (ab/libqkb200_base.so), same box; GPU suite.
T=gpurun_out/r02br
mkdir -p $T
for w in qft30 qft33 qft20 bv33; do
  for v in base new; do
    if [ $v = base ]; then export QK_LIB_PATH=$PWD/ab/libqkb200_base.so; else unset QK_LIB_PATH; fi
    timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $T/bench_${w}_$v.json 2> $T/bench_${w}_$v.err
  done
done
unset QK_LIB_PATH
python tools/pass_times.py qft30 > $T/pass_times_qft30.txt 2>&1
python tools/pass_times.py qft33 > $T/pass_times_qft33.txt 2>&1
( time timeout 1800 python -m pytest tests -m gpu -q -x -rfE ) > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
ls -la $T
