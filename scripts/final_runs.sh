#!/bin/sh
# Final round-2 measurement set on one 4-GPU box: N = 4, 2, 1 bench lines
# (defaults: cfg4, K = 50), the N = 1 ncu launch list, and the GPU test-suite
# (multi-GPU tests included).
o=${1:-gpurun_out/final}
mkdir -p $o
timeout 1000 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 4 > $o/bench_n4.json 2> $o/bench_n4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29702 bench.py --gpus 2 > $o/bench_n2.json 2> $o/bench_n2.err
CUDA_VISIBLE_DEVICES=0 python bench.py > $o/bench_n1.json 2> $o/bench_n1.err
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:"k_|gemm" -c 700 --csv --log-file $o/launches_n1.csv python bench.py --steps 20 --warmup 3 --no-cpu > $o/ncu_launch.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $o/gputest.log 2>&1
cp gpurun_out/parity_report.json $o/ 2>/dev/null
