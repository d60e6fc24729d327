"""Debug: eager run-ahead vs no run-ahead, per-step parameter snapshots."""
import sys, os, torch, numpy as np
sys.path.insert(0, '/root/repo')
from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables
from paper_2409_00657_b200.graph import Graph
from paper_2409_00657_b200.engine import Trainer
from paper_2409_00657_b200.featstore import FeatureTable
from paper_2409_00657_b200.model import init_model
from paper_2409_00657_b200.rng import chain
N, B, IT = 6000, 96, int(os.environ.get("ITERS", "11"))
off, tgt = build_csr(build_tables(OSpec(n=N, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4, d_cap=800, seed=21)))
g = Graph.from_host(off, tgt)
def mk(graphs, run_ahead=True):
    seed, D, C = 5, 32, 11
    table = FeatureTable.generated(g.n_vertices, D, seed, torch.float32)
    model = init_model("sage-mean", D, 64, 2, C, chain(seed, 0x07))
    return Trainer(g, table, model, (15, 10), B, seed, lr=0.1, iterations=IT, graphs=graphs, run_ahead=run_ahead), model
def rel(a, b):
    return float((a.double() - b.double()).abs().max() / b.double().abs().max())
EP = 3
res = {}
for name, ra in (("ref", True), ("pl", False)):
    tr, m = mk(False, ra)
    snap = torch.empty((EP * IT, m.flat.numel()), device="cuda")
    lo = torch.empty((EP * IT,), device="cuda")
    k = 0
    info = torch.zeros((EP * IT, 8), dtype=torch.float64, device="cuda")
    for epoch in range(EP):
        iters = tr.begin_epoch(epoch)
        for it in range(iters):
            tr.step(it)
            snap[k].copy_(m.flat)
            r = tr.last_runner
            n1 = r.builder.tensors["totals"][1]
            info[k, 0] = r.loss[:B].double().sum()
            info[k, 1] = r.agg[1].double().sum()   # whole buffer incl. stale rows
            info[k, 2] = r.builder.tensors["totals"].double().sum()
            info[k, 3] = r.h[1].double().sum()
            info[k, 4] = r.roots[:B].double().sum() if not tr.run_ahead else 0
            info[k, 5] = n1.double()
            k += 1
    torch.cuda.synchronize()
    res[name] = snap
    res["offsets"] = m.offsets; res["shapes"] = m.shapes
    res[name + "_info"] = info.cpu().numpy()
bad = [i for i in range(EP * IT) if rel(res["ref"][i], res["pl"][i]) > 1e-5]
if bad:
    i = bad[0]
    np.set_printoptions(precision=10, linewidth=200)
    for j in (i - 1, i):
        print(j, "ref", res["ref_info"][j][:6], "\n  ", "pl ", res["pl_info"][j][:6])
if bad:
    i = bad[0]
    for nm in ("ref", "pl"):
        d = (res[nm][i] - res[nm][i - 1]).double().cpu()
        res[nm + "_d"] = d
    o = res["offsets"]
    for b in range(len(o) - 1):
        a, c = res["ref_d"][o[b]:o[b + 1]], res["pl_d"][o[b]:o[b + 1]]
        e = float((a - c).abs().max() / c.abs().max().clamp_min(1e-30))
        idx = int((a - c).abs().argmax())
        print("block", b, res["shapes"][b], f"delta err {e:.2e}", "at", np.unravel_index(idx, res["shapes"][b]), float(a[idx]), float(c[idx]))
print("first bad step", bad[:1], "n bad", len(bad), [f"{rel(res['ref'][i], res['pl'][i]):.1e}" for i in bad[:3]])
