mkdir -p gpurun_out/r1
nproc > gpurun_out/r1/nproc.txt; free -g >> gpurun_out/r1/nproc.txt
timeout 900 python -m pytest tests/test_multiproc_gpu.py -x -q -s > gpurun_out/r1/multiproc.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r1/bench1.json 2> gpurun_out/r1/bench1.err
QK_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 2 --circuit qft33_c10_r1 > gpurun_out/r1/bench2_qft33.json 2> gpurun_out/r1/bench2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r1/ref1.json 2> gpurun_out/r1/ref1.err
tail -5 gpurun_out/r1/multiproc.log
