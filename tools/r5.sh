mkdir -p gpurun_out/r5
QK_DUMP_TUNE=1 QK_DUMP_LOAD=1 timeout 300 python tools/variant_times.py qaoa30_c12_r0 30 12 > gpurun_out/r5/tune.txt 2>&1
grep -E "variant|tune|load" gpurun_out/r5/tune.txt | tail -30
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r5/bench.json 2>gpurun_out/r5/bench.err
cat gpurun_out/r5/bench.json
