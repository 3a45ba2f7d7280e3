#!/bin/bash
# One H2D copy for the OP_QUAD/OP_QLITE pool data at load: e2e probe of QFT20
# (load breakdown), bench lines QFT20 / QAOA30, GPU suite.
T=gpurun_out/r02bv
mkdir -p $T
QK_DUMP_LOAD=1 timeout 120 python tools/e2e_probe.py qft20 > $T/e2e_probe_qft20.txt 2>&1
QK_DUMP_LOAD=1 timeout 300 python tools/e2e_probe.py qaoa30 > $T/e2e_probe_qaoa30.txt 2>&1
timeout 300 python bench.py --workload qft20 --steps 20 --warmup 3 --no-cpu > $T/bench_qft20.json 2> $T/bench_qft20.err
( time timeout 1800 python -m pytest tests -m gpu -q -x -rfE ) > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
timeout 900 python bench.py > $T/bench_default.json 2> $T/bench_default.err
ls -la $T
