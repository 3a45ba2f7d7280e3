#!/bin/bash
# Final evidence at HEAD (graph replay, column tables, OP_QLITE hoisting variant):
# GPU tests, smoke, headline bench, reference arm, other configs, launch list,
# ncu of the QFT30 write-only pass.
T=gpurun_out/r02bs
mkdir -p $T
nvidia-smi > $T/smi.txt 2>&1
( time timeout 1800 python -m pytest tests -m gpu -q -rfE ) > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1; echo "rc=$?" >> $T/smoke.log
timeout 900 python bench.py > $T/bench_default.json 2> $T/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $T/ref1.json 2> $T/ref1.err
for w in qft20 qft30 bv30 h30 bv33 h33 rzz33 u33 qft33 qaoa33r3; do
  timeout 400 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu >> $T/bench_all.json 2>> $T/bench_all.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $T/launches_qaoa30.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > $T/ncu_launch.log 2>&1
python tools/ncu_summary.py launches $T/launches_qaoa30.csv > $T/launches_qaoa30.txt 2>&1
bash tools/ncu_box.sh r02bs/full_qft30 qk_jit 3 --launch-skip 99 python tools/pass_times.py qft30
ls -la $T
