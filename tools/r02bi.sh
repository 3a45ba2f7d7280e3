#!/bin/bash
# Round-2 evidence at HEAD: GPU tests, smoke, bench lines (N=1 all configs, N=2 on
# one device through torchrun/gloo), reference arm, launch list, ncu of the
# QAOA30 passes, one H33 pass, the qaoa33r3 fix-up SQS and the peer exchange.
T=gpurun_out/r02bi
mkdir -p $T
nvidia-smi > $T/smi.txt 2>&1; nproc > $T/nproc.txt
( time timeout 1800 python -m pytest tests -m gpu -q -rfE --durations=20 ) > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1
timeout 900 python bench.py > $T/bench_default.json 2> $T/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $T/ref1.json 2> $T/ref1.err
for w in qft20 qft30 bv30 h30 bv33 h33 rzz33 u33 qft33 qaoa33r3; do
  timeout 400 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu >> $T/bench_all.json 2>> $T/bench_all.err
done
# N=2 path of the driver's scaling run, both ranks on the one device (gloo for the host collectives)
QK_INPLACE=1 QK_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29531 bench.py --gpus 2 --circuit qft33_c10_r1 --steps 2 --warmup 1 > $T/bench_n2.json 2> $T/bench_n2.err
QK_INPLACE=1 QK_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29532 bench.py --impl reference --gpus 2 --circuit qft33_c10_r1 --steps 1 --warmup 1 > $T/ref_n2.json 2> $T/ref_n2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $T/launches_qaoa30.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > $T/ncu_launch.log 2>&1
python tools/ncu_summary.py launches $T/launches_qaoa30.csv > $T/launches_qaoa30.txt 2>&1
# the 13 passes of the tuned run (6 tuning/warm runs of 13 launches before it)
bash tools/ncu_box.sh r02bi/full_qaoa30 qk_jit 13 --launch-skip 429 python tools/pass_times.py qaoa30
ls -la $T
