"""One grouped build (k_mg_build_w2 on the capped persistent grid) and one
grouped layer-1 gather (k_aggregate over G = 10 batches) of the papers-shaped
cfg4 loop, launched once each after one warm-up round -- the launches
`ncu --set full -k regex:"k_mg_build_w2|k_aggregate" --launch-skip 2 -c 2`
captures for profiles/ (DRAM bytes of the gather = bench.py roofline.traffic,
warp instructions of the build = roofline_sampler issue rate)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS  # noqa: E402
from paper_2409_00657_b200.engine import Trainer  # noqa: E402
from paper_2409_00657_b200.featstore import FeatureTable  # noqa: E402
from paper_2409_00657_b200.graph import GraphSpec, generate  # noqa: E402
from paper_2409_00657_b200.model import init_model  # noqa: E402
from paper_2409_00657_b200.rng import chain  # noqa: E402

cfg = CONFIGS["papers"]
G = 10
g = generate(GraphSpec(**{k: cfg[k] for k in ("n", "avg_deg", "beta", "p_in", "n_blocks",
                                               "d_cap", "seed")}))
table = FeatureTable.generated(g.n_vertices, cfg["dim"], cfg["seed"], torch.bfloat16)
model = init_model(cfg["arch"], cfg["dim"], cfg["hidden"], 2, cfg["classes"],
                   chain(cfg["seed"], 0x07))
tr = Trainer(g, table, model, cfg["fanout"], cfg["batch"], cfg["seed"], group=G)
tr.begin_epoch(0)
for it in range(2 + 2 * G):  # eager steps + the group loop's capture
    tr.step(it, stop=2 + 2 * G)
torch.cuda.synchronize()
for rnd in range(2):  # round 0 warms up, round 1 is what ncu captures
    tr._gg.run_eager(100 + rnd * G)
    torch.cuda.synchronize()
# the grouped layer-1 gather alone, inside an NVTX range (ncu --nvtx-include "gather/")
import ctypes as C  # noqa: E402
from paper_2409_00657_b200 import _lib  # noqa: E402
s = torch.cuda.current_stream().cuda_stream
with torch.cuda.nvtx.range("gather"):
    _lib.call("hg_step_prologue_group", tr._gg.descp[0], G, 1, s)
    torch.cuda.synchronize()
tr.check()
print("profile_group ok")
