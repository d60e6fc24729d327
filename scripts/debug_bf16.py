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

# --- pinpoint: device operands and the dh GEMM, in torch from the device's own buffers
n = len(roots)
Cp = run.dl16.shape[1]
dl16 = run.dl16[:n].float()
wcp = run.wcp.float()                      # [H x Cp]
dh_t = dl16 @ wcp.t()                      # torch fp32 of the same bf16 operands
h2d = run.h[2][:n].float()
dz_t = dh_t * (h2d > 0)
dz_dev = run.dh[2][:n]
pin = {"dh_gemm_vs_torch": rel(dz_dev.cpu().numpy(), dz_t.cpu().numpy()),
       "lowp2_vs_f32dz": rel(run.lowp[mr[1]:mr[1] + n].float().cpu().numpy(), dz_dev.cpu().numpy()),
       "wcp_vs_Wc": rel(wcp[:, :C].cpu().numpy(), _bf(P.Wc)),
       "wcp_pad_zero": float(wcp[:, C:].abs().max().item()) if Cp > C else 0.0,
       "dl16_vs_dlogits": rel(dl16[:, :C].cpu().numpy(), _bf(dl[:n, :C])),
       "max_rows": list(run.max_rows), "Cp": Cp}
print(json.dumps(pin))
# --- the per-micrograph shim on one root
from paper_2409_00657_b200 import micro as M
m = o_sample(off, tgt, int(roots[0]), fo, stream_key(sseed, 0, 3, int(roots[0])), draw=OK.sample_frontier_nb)
x = OK.feature_rows(m.vertices, D, feature_state(seed))
m32 = init_model(arch, D, H, 2, C, mseed)
one = M._OneRoot(m, x, m32)
one.run("hg_forward")
torch.cuda.synchronize()
r = one.runner
t = r.builder.tensors
shim = {"totals": t["totals"].cpu().tolist(), "need0": t["need_ids"][0][:8].cpu().tolist(),
        "agg1_abs": float(r.agg[1][:int(t["totals"][1])].abs().max()),
        "h1_abs": float(r.h[1][:int(t["totals"][1])].abs().max()),
        "h2_abs": float(r.h[2][:1].abs().max()), "logits": r.logits[0, :4].cpu().tolist(),
        "table_abs": float(r.table.table.abs().max()), "feat_row": r.desc.feat_row,
        "features": r.desc.features, "table_ptr": r.table.table.data_ptr(),
        "act_dtype": r.desc.act_dtype, "use_tc": r.desc.use_tc}
print(json.dumps(shim))
