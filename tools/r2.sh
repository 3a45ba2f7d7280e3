mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_multidev.py tests/test_multiproc_gpu.py -x -q -s > gpurun_out/r2/multi.log 2>&1
QK_DUMP_PLAN=1 QK_DEVICES=0,0 timeout 300 python -c "
import os,sys; sys.path.insert(0,'.')
from paper_2406_14084_b200 import LayoutParams, Simulator
t=open('bench_circuits/qft33_c10_r1.txt').read()
for mode in ('ovl','QK_NO_OVERLAP'):
    if mode!='ovl': os.environ[mode]='1'
    sim=Simulator(LayoutParams(n=33,c=32,r=1))
    p=sim.load_text(t,10)
    for i in range(3):
        sim.reset(); res=sim.run_loaded(p)
    st=sim.handle.stats()
    print(mode, res.timings, 'overlapped', st[12], 'xrs', st[5], st[4], flush=True)
    sim.release(); os.environ.pop(mode,None)
" > gpurun_out/r2/qft33_group.txt 2>&1
tail -5 gpurun_out/r2/multi.log; grep -v "^instr\|^relabel\|^block\|^table\|^pass\|^   " gpurun_out/r2/qft33_group.txt | tail
