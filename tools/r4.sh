mkdir -p gpurun_out/r4
for v in 0 1 2 3; do
  QK_JIT_VARIANT=$v timeout 300 python tools/variant_times.py qaoa30_c12_r0 30 12 > gpurun_out/r4/v$v.txt 2>&1
done
grep variant gpurun_out/r4/v*.txt
