"""Train-branch latency on the papers step (no build running beside it):
one CellRunner's batch built once, then [hg_train_step + hg_sgd_refresh]
graph-replayed.  Shows what the training chain alone costs per iteration.
    python scripts/bench_train.py [config]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2409_00657_b200 import _lib
from paper_2409_00657_b200.batching import epoch_permutation
from paper_2409_00657_b200.featstore import FeatureTable
from paper_2409_00657_b200.graph import GraphSpec, generate
from paper_2409_00657_b200.model import LabelOracle, init_model
from paper_2409_00657_b200.rng import chain
from paper_2409_00657_b200.trainer import CellRunner

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "papers"]
dev = torch.device("cuda")
g = generate(GraphSpec(n=cfg["n"], avg_deg=cfg["avg_deg"], beta=cfg["beta"], p_in=cfg["p_in"],
                       n_blocks=cfg["n_blocks"], d_cap=cfg["d_cap"], seed=cfg["seed"]), dev)
table = FeatureTable.generated(g.n_vertices, cfg["dim"], cfg["seed"], torch.bfloat16, dev)
model = init_model(cfg["arch"], cfg["dim"], cfg["hidden"], len(cfg["fanout"]), cfg["classes"],
                   chain(cfg["seed"], 0x07), dev)
B = cfg["batch"]
run = CellRunner(g, table, model, cfg["fanout"], B, LabelOracle(cfg["classes"], chain(0, 4)))
perm = epoch_permutation(0, 0, g.n_vertices, dev)
st = np.uint64(chain(chain(0, 6), 0, 0)).view(np.int64)
run.stage_roots(perm[:B], [st], B)
s = torch.cuda.current_stream().cuda_stream
run.builder.build(g, run.roots, run.keys, B, n_roots=B)
_lib.call("hg_step_prologue", C.byref(run.desc), B, 1, s)
run.desc.agg1_ready = 1
m = model


def step(ss):
    run.desc.lowp_fresh = 1
    _lib.call("hg_train_step", C.byref(run.desc), B, ss)
    _lib.call("hg_sgd_refresh", C.byref(run.desc), m.flat.data_ptr(), m.grad.data_ptr(),
              m.flat.numel(), 1e-4, 1.0 / B, 1, ss)
    run.desc.lowp_fresh = 0


_lib.call("hg_sgd_refresh", C.byref(run.desc), m.flat.data_ptr(), m.grad.data_ptr(),
          m.flat.numel(), 0.0, 1.0, 0, s)
for _ in range(3):
    step(s)
torch.cuda.synchronize()
for per in (1, 10):
    gr = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(gr, stream=cap):
        for _ in range(per):
            step(cap.cuda_stream)
    torch.cuda.synchronize()
    for _ in range(3):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 200 // per
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"train chain, {per} step(s) per graph: {e0.elapsed_time(e1) * 1000 / (reps * per):.1f} us/step")
tot = run.builder.tensors["totals"].cpu().numpy()
print("batch N_k", tot[:len(cfg['fanout']) + 1].tolist(), "loss", float(run.loss[:B].sum()))
if os.environ.get("HG_TOP_TRACE"):
    tb = torch.zeros(96, dtype=torch.int64, device="cuda")
    _lib.call("hg_top_trace", tb.data_ptr())
    for _ in range(3):
        step(s)
    torch.cuda.synchronize()
    _lib.call("hg_top_trace", None)
    t = tb.cpu().numpy()
    t0 = t[72]
    rel = lambda i: round((t[i] - t0) / 1000.0, 2) if t[i] else None  # noqa: E731
    print("top trace (us from epilogue start): producer start", rel(0))
    print(" load issued", [rel(1 + i) for i in range(24)])
    print(" load landed", [rel(32 + i) for i in range(24)])
    print(" epilogue", [rel(64 + i) for i in range(8)])
    print(" softmax", [rel(73 + i) for i in range(6)])
