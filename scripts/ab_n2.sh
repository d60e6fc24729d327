#!/bin/sh
# Same-box A/B of the layer-1 feature-stream L2 policy at N = 2 (bench.py
# defaults otherwise: cfg4, K = 50, G = 10).  Round 2 also A/B'd a fused
# one-launch p2p update here (measured slower, removed).
out=${1:-gpurun_out/ab_n2}
mkdir -p $out
port=29530
for st in 1 0 1; do
  port=$((port + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus 2 --agg-stream $st --no-model-centric \
    > $out/s${st}_$port.json 2> $out/s${st}_$port.err
done
