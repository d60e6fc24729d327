#!/bin/sh
# Run-ahead group size at the driver's K = 20: auto (G = 5, 4 replays) vs G = 10 (2 replays), N = 2 and N = 1.
o=gpurun_out/ab_group
mkdir -p $o
p=29800
for r in 1 2; do
  for g in 0 10; do
    p=$((p + 1))
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $p bench.py --gpus 2 --steps 20 --warmup 5 --group $g --no-model-centric > $o/n2_g${g}_$r.json 2> $o/n2_g${g}_$r.err
    python bench.py --steps 20 --warmup 5 --group $g --no-cpu > $o/n1_g${g}_$r.json 2> $o/n1_g${g}_$r.err
  done
done
