"""Persistent training step vs the split kernels on one papers-shaped batch
(cfg4 by default): loss / gradients after one step without update, parameters
after one step with the fused SGD, and the graph-replayed step time of both.
    python scripts/check_persist.py [config] [--ctas N] [--split-w1 N]"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_00657_b200 import _lib  # noqa: E402
from paper_2409_00657_b200.batching import epoch_permutation  # noqa: E402
from paper_2409_00657_b200.featstore import FeatureTable  # noqa: E402
from paper_2409_00657_b200.graph import GraphSpec, generate  # noqa: E402
from paper_2409_00657_b200.model import LabelOracle, init_model  # noqa: E402
from paper_2409_00657_b200.rng import chain  # noqa: E402
from paper_2409_00657_b200.trainer import CellRunner  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="papers")
ap.add_argument("--ctas", type=int, default=0)
ap.add_argument("--split-w1", type=int, default=0)
ap.add_argument("--batch", type=int, default=0)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
dev = torch.device("cuda")
g = generate(GraphSpec(n=cfg["n"], avg_deg=cfg["avg_deg"], beta=cfg["beta"], p_in=cfg["p_in"],
                       n_blocks=cfg["n_blocks"], d_cap=cfg["d_cap"], seed=cfg["seed"]), dev)
table = FeatureTable.generated(g.n_vertices, cfg["dim"], cfg["seed"], torch.bfloat16, dev)
model = init_model(cfg["arch"], cfg["dim"], cfg["hidden"], len(cfg["fanout"]), cfg["classes"],
                   chain(cfg["seed"], 0x07), dev)
B = args.batch or cfg["batch"]
run = CellRunner(g, table, model, cfg["fanout"], B, LabelOracle(cfg["classes"], chain(0, 4)))
perm = epoch_permutation(0, 0, g.n_vertices, dev)
st = np.uint64(chain(chain(0, 6), 0, 0)).view(np.int64)
run.stage_roots(perm[:B], [st], B)
s = torch.cuda.current_stream().cuda_stream
run.builder.build(g, run.roots, run.keys, B, n_roots=B)
_lib.call("hg_step_prologue", C.byref(run.desc), B, 1, s)
run.desc.agg1_ready = 1
m = model
flat0 = m.flat.clone()


def refresh():
    _lib.call("hg_sgd_refresh", C.byref(run.desc), m.flat.data_ptr(), m.grad.data_ptr(),
              m.flat.numel(), 0.0, 1.0, 0, s)


def step(ss, update, lr=0.05):
    run.desc.lowp_fresh = 1
    _lib.call("hg_train_step_sgd", C.byref(run.desc), B, m.flat.data_ptr(), m.grad.data_ptr(),
              m.flat.numel(), lr, 1.0 / B, update, ss)
    run.desc.lowp_fresh = 0


def one(persist, update):
    _lib.call("hg_set_persist", persist, args.ctas, args.split_w1)
    m.flat.copy_(flat0)
    m.grad.zero_()
    refresh()
    step(s, update)
    torch.cuda.synchronize()
    run.check()
    return (run.loss[:B].clone(), m.grad.clone(), m.flat.clone(), run.h[1].clone(),
            run.h[2].clone())


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).abs().max() / max(b.abs().max().item(), 1e-30))


out = {"config": args.config, "batch": B,
       "totals": run.builder.tensors["totals"].cpu().numpy()[:3].tolist()}
la, ga, _, h1a, h2a = one(0, 0)
lb, gb_, _, h1b, h2b = one(1, 0)
n1, n2 = out["totals"][1], out["totals"][2]
out["no_update"] = {"loss": rel(lb, la), "grad": rel(gb_, ga),
                    "h1_equal": bool(torch.equal(h1a[:n1], h1b[:n1])),
                    "h2_equal": bool(torch.equal(h2a[:n2], h2b[:n2])),
                    "loss_sum": [float(la.sum()), float(lb.sum())]}
_, _, pa, _, _ = one(0, 1)
_, _, pb, _, _ = one(1, 1)
out["update"] = {"params": rel(pb - flat0, pa - flat0), "params_abs": rel(pb, pa)}
# graph-replayed step time, 10 steps per graph, both paths
for persist in (0, 1):
    _lib.call("hg_set_persist", persist, args.ctas, args.split_w1)
    m.flat.copy_(flat0)
    m.grad.zero_()
    refresh()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(gr, stream=cap):
        for _ in range(10):
            step(cap.cuda_stream, 1, 1e-4)
    torch.cuda.synchronize()
    for _ in range(3):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    run.check()
    out[f"us_per_step_{'persist' if persist else 'split'}"] = round(e0.elapsed_time(e1) * 1000 / 200, 2)
print(json.dumps(out))

# phase timeline of one persistent step (every CTA's barrier stamps)
_lib.call("hg_set_persist", 1, args.ctas, args.split_w1)
P = 148 if not args.ctas else args.ctas
tb = torch.zeros(P * 64, dtype=torch.int64, device="cuda")
_lib.call("hg_persist_trace", tb.data_ptr())
for _ in range(3):
    step(s, 1, 1e-4)
torch.cuda.synchronize()
_lib.call("hg_persist_trace", None)
t = tb.view(P, 64).cpu().numpy().astype(np.int64)
nb = 9 if t[0, 19] else 8
t0 = t[:, 0].min()
us = lambda x: round(float(x) / 1000.0, 2)  # noqa: E731
tl = {"entry_spread": us(t[:, 0].max() - t0), "setup_max": us(t[:, 1].max() - t0)}
prev_rel = t[:, 1]
phases = []
for i in range(1, nb + 1):
    arr, relz = t[:, 2 * i], t[:, 2 * i + 1]
    work = arr - prev_rel
    phases.append({"phase": i, "work_med": us(np.median(work)), "work_max": us(work.max()),
                   "end": us(arr.max() - t0), "barrier": us(relz.min() - arr.max())})
    prev_rel = relz
work = t[:, 30] - prev_rel
phases.append({"phase": nb + 1, "work_med": us(np.median(work)), "work_max": us(work.max()),
               "end": us(t[:, 30].max() - t0)})
tl["phases"] = phases
tl["exit_max"] = us(t[:, 30].max() - t0)
# phase 1 detail, CTAs with a tile: loads issued / landed, accumulator ready, stores issued
act = t[:, 20] > 0
rel1 = t[act, 1]
det = {}
for nm, i in (("issue", 20), ("land", 24)):
    for j in range(4):
        det[f"{nm}{j}"] = [us(np.median(t[act, i + j] - rel1)), us((t[act, i + j] - rel1).max())]
det["acc"] = [us(np.median(t[act, 28] - rel1)), us((t[act, 28] - rel1).max())]
det["stored"] = [us(np.median(t[act, 29] - rel1)), us((t[act, 29] - rel1).max())]
det["arrive"] = [us(np.median(t[act, 2] - rel1)), us((t[act, 2] - rel1).max())]
tl["p1_detail_med_max"] = det
c0 = int(np.argmax(act))
tl["p1_epi_cta"] = {"acc": us(t[c0, 28] - t[c0, 1]),
                    "chunks": [[us(t[c0, 32 + 4 * j + k] - t[c0, 1]) if t[c0, 32 + 4 * j + k] else None
                                for k in range(4)] for j in range(4)],
                    "stored": us(t[c0, 29] - t[c0, 1]), "complete": us(t[c0, 48] - t[c0, 1])}
print(json.dumps(tl))
