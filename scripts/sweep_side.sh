#!/bin/sh
# Side-branch budget sweep of the grouped loop (scripts/timeline_group.py):
# build CTAs/SM x grouped-gather CTAs/SM, with and without the training branch.
out=${1:-gpurun_out/sweep.jsonl}
for b in 2 3 4; do for a in 1 2 3; do
  timeout 300 python scripts/timeline_group.py --build-ctas $b --agg-ctas $a --reps 8 >> $out
  timeout 300 python scripts/timeline_group.py --build-ctas $b --agg-ctas $a --reps 8 --no-train >> $out
done; done
