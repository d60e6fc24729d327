"""Degree statistics of the hop-2 frontier (layer-1 vertices) of papers-shaped batches."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench
from paper_2409_00657_b200.engine import Trainer
from paper_2409_00657_b200.featstore import FeatureTable
from paper_2409_00657_b200.graph import GraphSpec, generate
from paper_2409_00657_b200.model import init_model
cfg = bench.CONFIGS["papers"]
g = generate(GraphSpec(n=cfg["n"], avg_deg=cfg["avg_deg"], beta=cfg["beta"], p_in=cfg["p_in"],
                       n_blocks=cfg["n_blocks"], d_cap=cfg["d_cap"], seed=cfg["seed"]))
t = FeatureTable(1, 128, torch.bfloat16, torch.device("cuda"), 128)
m = init_model("sage-mean", 128, 256, 2, 172, 3)
from paper_2409_00657_b200.sampler import MicrographBuilder
from paper_2409_00657_b200.batching import epoch_permutation
b = MicrographBuilder((15, 10), 1024, torch.device("cuda"))
perm = epoch_permutation(0, 0, g.n_vertices, "cuda")
off = g.offsets
allf, allr = [], []
for it in range(4):
    roots = perm[it * 1024:(it + 1) * 1024].contiguous()
    keys = torch.full((1,), 12345 + it, dtype=torch.int64, device="cuda")
    b.build(g, roots, keys, 1024, n_roots=1024)
    tt = b.tensors
    n1 = int(tt["totals"][1].item())
    ids = tt["need_ids"][1][:n1].long()
    inl = tt["in_layer"][1][:n1].bool()
    f = ids[inl]
    d = (off[f + 1] - off[f]).cpu().numpy()
    dr = (off[roots + 1] - off[roots]).cpu().numpy()
    allf.append(d); allr.append(dr)
d = np.concatenate(allf); dr = np.concatenate(allr)
print("hop-2 tasks/batch", len(d) / 4, "sum deg/batch", d.sum() / 4, "mean", d.mean(),
      "p50", np.median(d), "p90", np.percentile(d, 90), "p99", np.percentile(d, 99), "max", d.max())
for lo, hi in ((0, 10), (11, 256), (257, 1024), (1025, 4096), (4097, 1 << 20)):
    sel = (d >= lo) & (d <= hi)
    print(f"deg {lo}-{hi}: tasks {sel.sum()/4:.0f}  slots {d[sel].sum()/4:.0f}")
print("root deg mean", dr.mean(), "max", dr.max(), "sum", dr.sum() / 4)
