#!/bin/sh
# L2 policy of the layer-1 feature stream inside the replayed group loop.
out=${1:-gpurun_out/sweep_stream.jsonl}
for st in 0 1; do
  for cfg in "3 3" "2 2"; do
    set -- $cfg
    timeout 200 python scripts/timeline_group.py --stream $st --build-ctas $1 --agg-ctas $2 --reps 8 >> $out
  done
  timeout 200 python scripts/timeline_group.py --stream $st --no-train --reps 8 >> $out
done
