#!/bin/bash
# Round evidence on one B200: tests, smoke, bench lines, ncu launch list and
# full captures of the block pass / cluster-exchange pass / SQS.
#   gpurun -- 'bash tools/evidence.sh <tag>'
T=gpurun_out/${1:-ev}
mkdir -p $T
nvidia-smi > $T/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1
timeout 600 python bench.py > $T/bench_default.json 2> $T/bench_default.err
for w in qft20 bv33 h33 rzz33 u33 qft33 qft30 bv30 qaoa26 qaoa33r3; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu >> $T/bench_all.json 2>> $T/bench_all.err
done
for sq in "circuit 30" "gate 30" "qubit 30"; do
  set -- $sq
  timeout 600 python -m paper_2406_14084_b200.bench --suite $1 --qubits $2 --reps 1 \
    --out $T/suite_$1$2.csv > /dev/null 2>> $T/suite.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $T/launches_qaoa30.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > $T/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_jit -c 8 -o $T/full_qaoa26 \
  python tools/pass_times.py qaoa26 > $T/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sqs -c 2 -o $T/full_sqs_qaoa26 \
  python tools/pass_times.py qaoa26 > $T/ncu_sqs.log 2>&1
ls -la $T
