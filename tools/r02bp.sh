#!/bin/bash
# Evidence at HEAD (graph replay + thread columns): headline bench, reference arm,
# other configs, launch list; per-pass times of the 256-B-row schedules (QK_ROWBITS=4).
T=gpurun_out/r02bp
mkdir -p $T
nvidia-smi > $T/smi.txt 2>&1
timeout 900 python bench.py > $T/bench_default.json 2> $T/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $T/ref1.json 2> $T/ref1.err
for w in qft20 qft30 bv30 h30 bv33 h33 rzz33 u33 qft33 qaoa33r3; do
  timeout 400 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu >> $T/bench_all.json 2>> $T/bench_all.err
done
for w in qft30 qft33 bv33; do
  QK_ROWBITS=4 QK_DUMP_SCHED=1 timeout 300 python tools/pass_times.py $w > $T/pass_times_${w}_rb4.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $T/launches_qaoa30.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > $T/ncu_launch.log 2>&1
python tools/ncu_summary.py launches $T/launches_qaoa30.csv > $T/launches_qaoa30.txt 2>&1
ls -la $T
