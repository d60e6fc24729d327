"""Standalone hg_mg_build timing on the papers-shaped graph (no training in
flight).  HG_BUILD_MONO=1 selects the single-kernel build for A/B."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench
from paper_2409_00657_b200.batching import epoch_permutation
from paper_2409_00657_b200.graph import GraphSpec, generate
from paper_2409_00657_b200.rng import chain
from paper_2409_00657_b200.sampler import MicrographBuilder
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "papers"]
g = generate(GraphSpec(n=cfg["n"], avg_deg=cfg["avg_deg"], beta=cfg["beta"], p_in=cfg["p_in"],
                       n_blocks=cfg["n_blocks"], d_cap=cfg["d_cap"], seed=cfg["seed"]))
perm = epoch_permutation(0, 0, g.n_vertices)
import os
B = int(os.environ.get("HG_B", cfg["batch"]))
b = MicrographBuilder(cfg["fanout"], B)
states = torch.tensor(np.array([chain(chain(0, 6), 0, it) for it in range(64)], dtype=np.uint64).view(np.int64), device="cuda")
for it in range(5):
    b.build(g, perm[it * B:(it + 1) * B], states[it:it + 1], B)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
n = 40
for it in range(n):
    b.build(g, perm[it * B:(it + 1) * B], states[it:it + 1], B)
ev[1].record()
torch.cuda.synchronize()
print(f"build {cfg['fanout']} B={B}: {ev[0].elapsed_time(ev[1]) / n * 1000:.1f} us/batch")
b.check()
