#!/bin/bash
T=gpurun_out/r02c; mkdir -p $T
timeout 600 python tools/rb_check.py qft20_c10_r0 qaoa24_c12_r0 qft24_c10_r1 qft26_c10_r0 > $T/rb_check.txt 2>&1
QK_DUMP_PLAN=1 QK_DUMP_PHASES=1 timeout 300 python tools/rb_check.py qft20_c10_r0 > $T/plan_qft20.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_bench_suite.py::test_gate_by_gate_baseline_matches_block_mode > $T/pytest.log 2>&1; echo "rc=$?" >> $T/pytest.log
