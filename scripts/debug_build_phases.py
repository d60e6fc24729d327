"""Per-phase clock64 breakdown of k_mg_build (needs a -DHG_BUILD_PROFILE build)."""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2409_00657_b200 import _lib
from paper_2409_00657_b200.graph import GraphSpec, generate
from paper_2409_00657_b200.sampler import MicrographBuilder
from paper_2409_00657_b200.batching import epoch_permutation
from paper_2409_00657_b200.rng import chain
g = generate(GraphSpec(n=111_000_000, avg_deg=15.6, beta=0.6, p_in=0.95, n_blocks=8, d_cap=1 << 15, seed=0))
perm = epoch_permutation(0, 0, g.n_vertices)
b = MicrographBuilder((15, 10), 1024)
for it in range(3):
    st = torch.tensor([np.uint64(chain(chain(0, 6), 0, it)).view(np.int64)], device='cuda')
    roots = perm[it * 1024:(it + 1) * 1024]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(); b.build(g, roots, st, 1024); ev1.record(); torch.cuda.synchronize()
    print("build ms", ev0.elapsed_time(ev1))
buf = (C.c_longlong * (16 * 1024))()
_lib.call("hg_debug_build_phases", buf, 1024)
a = np.array(buf, dtype=np.int64).reshape(1024, 16)
names = {0: "init", 1: "h1 counts+scan", 2: "h1 warp tasks", 3: "h1 hubs", 4: "h1 sort", 5: "h2 counts+scan",
         6: "h2 warp tasks", 7: "h2 hubs", 8: "h2 sort", 13: "need sets", 14: "outputs"}
order = [0, 1, 2, 3, 4, 5, 6, 7, 8, 13, 14]
tot = a[:, 14] - a[:, 0]
print("per-CTA cycles: mean", tot.mean(), "p50", np.median(tot), "p90", np.percentile(tot, 90), "max", tot.max())
for i in range(1, len(order)):
    d = a[:, order[i]] - a[:, order[i - 1]]
    print(f"{names[order[i]]:16s} mean {d.mean():9.0f}  p90 {np.percentile(d, 90):9.0f}  max {d.max():9.0f}")
span = (a[:, 14].max() - a[:, 0].min())
print("kernel span cycles", span)
