#!/bin/bash
# CUDA-graph replay, capture on the second run from a start state: graph tests,
# QFT20 (configs[0]) with and without replay (device and e2e), GPU suite, headline.
T=gpurun_out/r02bl
mkdir -p $T
nvidia-smi > $T/smi.txt 2>&1
( timeout 600 python -m pytest tests/test_gpu_graph.py -q -rfE ) > $T/pytest_graph.log 2>&1; echo "rc=$?" >> $T/pytest_graph.log
for w in qft20; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu > $T/bench_${w}_graph.json 2> $T/bench_${w}_graph.err
  QK_NO_GRAPH=1 timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu > $T/bench_${w}_eager.json 2> $T/bench_${w}_eager.err
done
( time timeout 1800 python -m pytest tests -m gpu -q -rfE --durations=10 ) > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1; echo "rc=$?" >> $T/smoke.log
timeout 900 python bench.py > $T/bench_default.json 2> $T/bench_default.err
ls -la $T
QK_DUMP_LOAD=1 timeout 120 python tools/e2e_probe.py qft20 > $T/e2e_probe_qft20.txt 2>&1
QK_NO_GRAPH=1 timeout 120 python tools/e2e_probe.py qft20 > $T/e2e_probe_qft20_eager.txt 2>&1
