#!/bin/bash
# tests (incl. the written-state run) and the e2e bench with the schedule memo
T=gpurun_out/r02ar; mkdir -p $T
( time timeout 1800 python -m pytest tests -m gpu -q -x -rfE ) > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
timeout 900 python bench.py --no-cpu > $T/bench_qaoa30.json 2> $T/bench.err
QK_DUMP_LOAD=1 timeout 300 python tools/e2e_probe.py > $T/e2e_probe.txt 2>&1
