#!/bin/sh
# Persistent step inside the replayed group loop: side-branch budgets x persist on/off.
out=${1:-gpurun_out/sweep_persist.jsonl}
for p in 0 1; do
  timeout 200 python scripts/timeline_group.py --persist $p --no-build --reps 8 >> $out
  for cfg in "3 3" "2 2" "2 1" "1 1"; do
    set -- $cfg
    timeout 200 python scripts/timeline_group.py --persist $p --build-ctas $1 --agg-ctas $2 --reps 8 >> $out
  done
done
