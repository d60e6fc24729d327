#!/bin/sh
# Multi-GPU check of a pre-gather change: the 2/4-GPU tests, then N = 4 and N = 2 bench lines.
o=gpurun_out/serve
mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -k "distributed or strategy" > $o/tdist.log 2>&1
timeout 1000 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 4 --no-model-centric > $o/bench_n4.json 2> $o/bench_n4.err
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29712 bench.py --gpus 2 --no-model-centric > $o/bench_n2.json 2> $o/bench_n2.err
