"""Timeline of one replayed group of the papers-shaped cfg4 loop (G = 10):
the GroupLoop graph re-captured with device timestamps (hg_stamp,
%globaltimer) at the branch boundaries -- side branch: stage / build /
gather; training branch: after every train step + SGD -- so the overlap of
the build with the training chain can be read from inside the replay.
    python scripts/timeline_group.py [--build-ctas N] [--reps R]"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS  # noqa: E402
from paper_2409_00657_b200 import _lib, engine  # noqa: E402
from paper_2409_00657_b200.engine import Trainer  # noqa: E402
from paper_2409_00657_b200.featstore import FeatureTable  # noqa: E402
from paper_2409_00657_b200.graph import GraphSpec, generate  # noqa: E402
from paper_2409_00657_b200.model import init_model  # noqa: E402
from paper_2409_00657_b200.rng import chain  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--build-ctas", type=int, default=engine.BUILD_CTAS_PER_SM)
ap.add_argument("--agg-ctas", type=int, default=3, help="grouped gather CTAs/SM (hg_set_side_budget)")
ap.add_argument("--reps", type=int, default=6)
ap.add_argument("--stream", type=int, default=1, help="evict-first feature loads")
ap.add_argument("--inline-gather", action="store_true",
                help="layer-1 gather of each step on the training stream (not the side branch)")
ap.add_argument("--persist", type=int, default=0, help="persistent training step (hg_set_persist)")
ap.add_argument("--no-build", action="store_true", help="training branch only")
ap.add_argument("--no-train", action="store_true", help="side branch only")
args = ap.parse_args()

_lib.call("hg_set_side_budget", args.agg_ctas, args.stream)
_lib.call("hg_set_persist", args.persist, 0, 0)
cfg = CONFIGS["papers"]
G = 10
g = generate(GraphSpec(**{k: cfg[k] for k in ("n", "avg_deg", "beta", "p_in", "n_blocks",
                                               "d_cap", "seed")}))
table = FeatureTable.generated(g.n_vertices, cfg["dim"], cfg["seed"], torch.bfloat16)
model = init_model(cfg["arch"], cfg["dim"], cfg["hidden"], 2, cfg["classes"],
                   chain(cfg["seed"], 0x07))
tr = Trainer(g, table, model, cfg["fanout"], cfg["batch"], cfg["seed"], group=G)
tr.begin_epoch(0)
stop = 4 * G + 2
for it in range(2 + 2 * G):
    tr.step(it, stop=stop)
torch.cuda.synchronize()
gl = tr._gg
B = tr.B
m = tr.model
st = torch.zeros(2, 64, dtype=torch.int64, device="cuda")
stamp = lambda x, i, s: _lib.call("hg_stamp", st[x, i:].data_ptr(), s)  # noqa: E731
graphs = []
cur = torch.cuda.current_stream()
for x in range(2):
    nxt = gl.gb[1 - x]
    gr = torch.cuda.CUDAGraph()
    cap = gl._cap
    cap.wait_stream(cur)
    with torch.cuda.graph(gr, stream=cap):
        cs = cap.cuda_stream
        stamp(x, 0, cs)
        gl.side.wait_stream(cap)
        ss = gl.side.cuda_stream
        if not args.no_build:
            with torch.cuda.stream(gl.side):
                _lib.call("hg_iter_stage_group", tr._perm_buf.data_ptr(), tr._states_buf.data_ptr(),
                          tr.iters, tr._it_dev.data_ptr(), B, G, G, G, nxt.roots.data_ptr(),
                          nxt.keys.data_ptr(), ss)
                stamp(x, 1, ss)
                nxt.build(tr.graph, stream=ss, ctas_per_sm=args.build_ctas)
                stamp(x, 2, ss)
                if not args.inline_gather:
                    _lib.call("hg_step_prologue_group", gl.descp[1 - x], G, 1, ss)
                stamp(x, 3, ss)
        if not args.no_train:
            for i, r in enumerate(gl.sets[x]):
                if args.inline_gather:  # this step's layer-1 gather on the training stream
                    _lib.call("hg_step_prologue", C.byref(r.desc), B, 1, cs)
                r.desc.lowp_fresh = 1
                _lib.call("hg_train_step_sgd", C.byref(r.desc), B, m.flat.data_ptr(),
                          m.grad.data_ptr(), m.flat.numel(), float(tr.lr), 1.0 / B, 1, cs)
                r.desc.lowp_fresh = 0
                stamp(x, 10 + i, cs)
        cap.wait_stream(gl.side)
        stamp(x, 30, cs)
    cur.wait_stream(cap)
    graphs.append(gr)
torch.cuda.synchronize()
gl.restart(0)
out = []
for rep in range(args.reps):
    x = rep & 1
    graphs[x].replay()
    torch.cuda.synchronize()
    if rep < 2:
        continue
    t = st[x].cpu().numpy().astype(np.int64)
    t0 = t[0]
    us = lambda i: round((t[i] - t0) / 1000.0, 1)  # noqa: E731
    rec = {"total_us": us(30)}
    if not args.no_build:
        rec.update(stage_us=us(1), build_end_us=us(2), gather_end_us=us(3))
    if not args.no_train:
        rec["train_steps_end_us"] = [us(10 + i) for i in range(G)]
    out.append(rec)
tr.check()
mean = {k: round(float(np.mean([r[k] for r in out])), 1) for k in out[0] if k != "train_steps_end_us"}
print(json.dumps({"build_ctas_per_sm": args.build_ctas, "agg_ctas": args.agg_ctas, "persist": args.persist, "stream": args.stream, "inline_gather": args.inline_gather, "mean": mean, "no_build": args.no_build,
                  "no_train": args.no_train, "replays": out}))
