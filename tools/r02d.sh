#!/bin/bash
T=gpurun_out/r02d; mkdir -p $T
timeout 900 python tools/rb_check2.py qft20_c10_r0 qaoa24_c12_r0 qaoa26_c12_r0 > $T/rb_check2.txt 2>&1
