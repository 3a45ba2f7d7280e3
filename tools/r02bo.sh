#!/bin/bash
# Per-thread OP_QUAD/OP_QLITE factor tables in columns (entry k of thread t at
# k*2^T + t: a warp's load is 512 contiguous bytes) against the row layout
# (HEAD library, ab/libqkb200_base.so), same box; then the GPU suite.
T=gpurun_out/r02bo
mkdir -p $T
for w in qft30 qft33 qaoa30 u33 rzz33 bv33 h33; do
  for v in base new; do
    if [ $v = base ]; then export QK_LIB_PATH=$PWD/ab/libqkb200_base.so; else unset QK_LIB_PATH; fi
    timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > $T/bench_${w}_$v.json 2> $T/bench_${w}_$v.err
  done
done
unset QK_LIB_PATH
python tools/pass_times.py qft30 > $T/pass_times_qft30.txt 2>&1
python tools/pass_times.py qft33 > $T/pass_times_qft33.txt 2>&1
( time timeout 1800 python -m pytest tests -m gpu -q -x -rfE ) > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
bash tools/ncu_box.sh r02bo/full_qft30 qk_jit 3 --launch-skip 99 python tools/pass_times.py qft30
ls -la $T
