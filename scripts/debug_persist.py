"""Repeat the persistent step on a small batch and report which buffers ever
differ from the split kernels' (race hunting).
    python scripts/debug_persist.py [reps]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables  # noqa: E402
from oracle.rng import chain  # noqa: E402
from paper_2409_00657_b200 import _lib  # noqa: E402
from paper_2409_00657_b200.featstore import FeatureTable  # noqa: E402
from paper_2409_00657_b200.graph import Graph  # noqa: E402
from paper_2409_00657_b200.model import LabelOracle, init_model  # noqa: E402
from paper_2409_00657_b200.trainer import CellRunner  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
CASES = {"small": ("sage-mean", (10, 5), 32, 64, 8), "big": ("sage-mean", (15, 10), 128, 256, 172),
         "gcn": ("gcn", (10, 10), 64, 128, 40)}
case = CASES[sys.argv[2] if len(sys.argv) > 2 else "small"]
kw = dict(n=3000, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4, d_cap=600, seed=11)
off, tgt = build_csr(build_tables(OSpec(**kw)))
world = Graph.from_host(off, tgt)
arch, fo, D, H, Cn = case
cap, n_real = 128, 96
model = init_model(arch, D, H, 2, Cn, chain(5, 0x07))
table = FeatureTable.generated(world.n_vertices, D, 5, dtype=torch.bfloat16)
run = CellRunner(world, table, model, fo, cap, LabelOracle(Cn, chain(5, 0x04)))
roots = np.random.default_rng(3).choice(world.n_vertices, cap, replace=False).astype(np.int64)
run.stage_roots(roots, [np.uint64(chain(chain(5, 6), 0, 1)).view(np.int64)], cap)
n_dev = torch.tensor([n_real], dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
run.builder.build(world, run.roots, run.keys, cap, n_roots=cap, n_dev=n_dev.data_ptr())
_lib.call("hg_step_prologue", C.byref(run.desc), cap, 1, s)
run.desc.agg1_ready = 1
m = model
flat0 = m.flat.clone()
dagg = run.dagg


def step(persist):
    _lib.call("hg_set_persist", persist, 0, 0)
    m.flat.copy_(flat0)
    m.grad.zero_()
    run.logits.fill_(float("nan"))
    dagg.fill_(float("nan"))
    run.lowp.fill_(float("nan"))
    _lib.call("hg_sgd_refresh", C.byref(run.desc), m.flat.data_ptr(), m.grad.data_ptr(),
              m.flat.numel(), 0.0, 1.0, 0, s)
    run.desc.lowp_fresh = 1
    _lib.call("hg_train_step_sgd", C.byref(run.desc), cap, m.flat.data_ptr(), m.grad.data_ptr(),
              m.flat.numel(), 0.05, 1.0 / n_real, 0, s)
    run.desc.lowp_fresh = 0
    torch.cuda.synchronize()
    return {"loss": run.loss.clone(), "grad": m.grad.clone(), "h1": run.h[1].clone(),
            "h2": run.h[2].clone(), "agg2": run.agg[2].clone(), "dl": run.dl16.clone(),
            "logits": run.logits.clone(), "dagg": dagg.clone(), "lowp": run.lowp.clone()}


tot = run.builder.tensors["totals"].cpu().numpy()
n1, n2 = int(tot[1]), int(tot[2])
ref = step(0)
seg = {}
offs = [int(x) for x in model.offsets] if hasattr(model, "offsets") else []
bad = {}
for i in range(reps):
    got = step(1)
    for k, v in got.items():
        a = v.float()
        b = ref[k].float()
        if k in ("h1",):
            a, b = a[:n1], b[:n1]
        if k in ("h2", "agg2", "dl", "logits", "loss"):
            a, b = a[:n2], b[:n2]
        if k == "dagg":
            w = 2 * H if arch == "sage-mean" else H
            a, b = a[:n2 * w], b[:n2 * w]
        if k == "lowp":
            a, b = a[:n1], b[:n1]
        nan = int(torch.isnan(a).sum())
        diff = float((a - b).abs().nan_to_num(1e30).max())
        if nan or diff > 1e-3 * max(float(b.abs().nan_to_num(0).max()), 1e-30):
            where = torch.nonzero(torch.isnan(a) | ((a - b).abs() > 1e-3)).flatten()[:8].tolist()
            bad.setdefault(k, []).append({"rep": i, "nan": nan, "diff": diff, "where": where,
                                          "ref_nan": int(torch.isnan(b).sum())})
print(json.dumps({"n1": n1, "n2": n2, "offsets": offs, "bad": bad}))
