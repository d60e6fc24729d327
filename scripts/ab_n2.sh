#!/bin/sh
# Same-box A/B of the multi-GPU update and the feature-stream policy at N = 2
# (bench.py defaults otherwise: cfg4, K = 50, G = 10).
out=${1:-gpurun_out/ab_n2}
mkdir -p $out
port=29530
for v in "fused 1" "split 1" "fused 0" "fused 1"; do
  set -- $v
  port=$((port + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus 2 --update $1 --agg-stream $2 --no-model-centric \
    > $out/u$1_s$2_$port.json 2> $out/u$1_s$2_$port.err
done
