"""Scratch: per-stage device vs bf16-emulating oracle, tc path, cfg4 dims."""
import sys, os, json
import numpy as np, torch
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
from oracle import kernels as OK, model as OM
from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables
from oracle.rng import chain
from oracle.sampler import sample_micrograph as o_sample, stream_key
from bf16_oracle import forward_bf16, _bf
from paper_2409_00657_b200.featstore import FeatureTable, feature_state
from paper_2409_00657_b200.graph import Graph
from paper_2409_00657_b200.model import LabelOracle, init_model
from paper_2409_00657_b200.trainer import CellRunner

kw = dict(n=3000, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4, d_cap=600, seed=11)
off, tgt = build_csr(build_tables(OSpec(**kw)))
G = Graph.from_host(off, tgt)
arch, fo, D, H, C = "sage-mean", (15, 10), 128, 256, 172
seed = 7
sseed, mseed, lseed = chain(seed, 6), chain(seed, 7), chain(seed, 4)
roots = np.random.default_rng(1).choice(3000, 96, replace=False).astype(np.int64)
model = init_model(arch, D, H, 2, C, mseed)
table = FeatureTable.generated(3000, D, seed, dtype=torch.bfloat16)
run = CellRunner(G, table, model, fo, 128, LabelOracle(C, lseed))
st = np.uint64(chain(sseed, 0, 3)).view(np.int64)
run.stage_roots(roots, [st], len(roots))
batch = run.launch()
torch.cuda.synchronize()
P = OM.init_params(arch, D, H, 2, C, mseed)
h = batch.to_host()
out = {}
def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return [float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)),
            float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))]
agg1 = run.agg[1].float().cpu().numpy(); h1 = run.h[1].float().cpu().numpy()
agg2 = run.agg[2].float().cpu().numpy(); h2 = run.h[2].float().cpu().numpy()
dl = run.logits.cpu().numpy()
lowp = run.lowp.float().cpu().numpy()
mr = run.max_rows
dz1 = lowp[:mr[1]]; dz2 = lowp[mr[1]:mr[1] + mr[2]]
errs = {k: [] for k in ("agg1", "h1", "agg2", "h2", "dl", "dz2", "dz1")}
Dp = model.Dp
for i, r in enumerate(roots.tolist()[:32]):
    m = o_sample(off, tgt, r, fo, stream_key(sseed, 0, 3, r), draw=OK.sample_frontier_nb)
    x = OK.feature_rows(m.vertices, D, feature_state(seed))
    stt = forward_bf16(m, x, P, tc=True)
    n1 = slice(h["need_off"][1][i], h["need_off"][1][i + 1])
    n2 = slice(h["need_off"][2][i], h["need_off"][2][i + 1])
    a1 = agg1[n1]; a1 = np.concatenate([a1[:, :D], a1[:, Dp:Dp + D]], 1)
    errs["agg1"].append(rel(a1, stt["aggs"][0]))
    errs["h1"].append(rel(h1[n1], stt["h"][1]))
    errs["agg2"].append(rel(agg2[n2], stt["aggs"][1]))
    errs["h2"].append(rel(h2[n2], stt["h"][2]))
    lg = stt["logits"]; e = np.exp(lg - lg.max()); d_ = e / e.sum()
    lab = int(OM.labels([r], C, lseed)[0]); d_[lab] -= 1
    errs["dl"].append(rel(dl[i, :C], d_))
    dh2 = _bf(P.Wc) @ _bf(d_)
    dz2_o = dh2 * (stt["zs"][1][0] > 0)
    errs["dz2"].append(rel(dz2[n2][0], _bf(dz2_o)))
out = {k: (np.max(np.array(v), 0).tolist() if v else None) for k, v in errs.items()}
print(json.dumps(out))
json.dump(out, open("gpurun_out/debug_bf16.json", "w"))
