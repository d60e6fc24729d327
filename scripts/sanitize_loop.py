"""Driver for tests/test_sanitizer_gpu.py: a few iterations of the grouped
CUDA-graph training loop (warp-per-root build, grouped gather, tcgen05 step,
fused SGD/refresh) on a 6K-vertex graph, run under compute-sanitizer.
Argument: "loop" (memcheck of the whole loop) or "build" (racecheck of the
micrograph builds, both kernels)."""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2409_00657_b200 import _lib  # noqa: E402
from paper_2409_00657_b200.engine import Trainer  # noqa: E402
from paper_2409_00657_b200.featstore import FeatureTable  # noqa: E402
from paper_2409_00657_b200.graph import GraphSpec, generate  # noqa: E402
from paper_2409_00657_b200.model import init_model  # noqa: E402
from paper_2409_00657_b200.rng import chain  # noqa: E402
from paper_2409_00657_b200.sampler import GroupBuilder, MicrographBuilder  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "loop"
g = generate(GraphSpec(n=6000, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4, d_cap=1500, seed=21))
if what == "loop":
    for dtype, H in ((torch.bfloat16, 64), (torch.float32, 32)):
        table = FeatureTable.generated(g.n_vertices, 32, 5, dtype)
        model = init_model("sage-mean", 32, H, 2, 11, chain(5, 7))
        tr = Trainer(g, table, model, (15, 10), 96, 5, iterations=12, group=4)
        tr.begin_epoch(0)
        for it in range(tr.iters):
            tr.step(it)
        torch.cuda.synchronize()
        tr.check()
    print("loop ok")
else:
    roots = torch.randperm(6000, device="cuda")[:256].to(torch.int64)
    keys = torch.tensor(np.array([chain(3, 1), chain(3, 2)], dtype=np.uint64).view(np.int64),
                        device="cuda")
    for mode in (0, 1):
        _lib.call("hg_mg_build_mode", mode)
        for fo in ((15, 10), (10, 5, 3)):
            bs = [MicrographBuilder(fo, 128) for _ in range(2)]
            gb = GroupBuilder(bs)
            gb.roots.copy_(roots)
            gb.keys.copy_(keys)
            gb.build(g, ctas_per_sm=2)
            torch.cuda.synchronize()
            gb.check()
    _lib.call("hg_mg_build_mode", 0)
    print("build ok")
