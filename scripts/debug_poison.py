"""Debug: poison every runner buffer before build+train; a stale/OOB read shows as NaN or a diff."""
import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables
from paper_2409_00657_b200.graph import Graph
from paper_2409_00657_b200.batching import epoch_permutation
from paper_2409_00657_b200.rng import chain
from paper_2409_00657_b200.featstore import FeatureTable
from paper_2409_00657_b200.model import init_model, LabelOracle
from paper_2409_00657_b200.trainer import CellRunner
N, B = 6000, 96
off, tgt = build_csr(build_tables(OSpec(n=N, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4, d_cap=800, seed=21)))
g = Graph.from_host(off, tgt)
seed, D, Cc = 5, 32, 11
dtype = torch.bfloat16 if "bf16" in sys.argv else torch.float32
PRO = "pro" in sys.argv
import ctypes as C
from paper_2409_00657_b200 import _lib
table = FeatureTable.generated(g.n_vertices, D, seed, dtype)
model = init_model("sage-mean", D, 64, 2, Cc, chain(seed, 0x07))
run = CellRunner(g, table, model, (15, 10), B, LabelOracle(Cc, chain(seed, 4)))

def poison(val_f, val_i):
    for t in run.agg[1:] + run.h[1:] + run.dh[1:] + [run.dagg, run.logits, run.loss, run.lowp, run.dl16]:
        if t.dtype.is_floating_point:
            t.fill_(val_f)
    bt = run.builder.tensors
    for k, v in bt.items():
        for x in (v if isinstance(v, list) else [v]):
            if x is not None and k != "totals":
                x.fill_(val_i)
    run.builder.ws.fill_(val_i)

for epoch in range(2):
    perm = epoch_permutation(seed, epoch, g.n_vertices, "cuda")
    for it in range(11):
        roots = perm[it * B:(it + 1) * B].clone()
        st = np.uint64(chain(chain(seed, 6), epoch, it)).view(np.int64)
        out = []
        for pv in ((0.0, 0), (float("nan"), 7), (1e30, -1)):
            run.stage_roots(roots, [st], B)
            poison(*pv)
            model.grad.zero_()
            if PRO:
                run.builder.build(g, run.roots, run.keys, B, n_roots=B)
                s = torch.cuda.current_stream().cuda_stream
                _lib.call("hg_step_prologue", C.byref(run.desc), B, 1, s)
                run.desc.agg1_ready = 1
                _lib.call("hg_train_step", C.byref(run.desc), B, s)
                run.desc.agg1_ready = 0
            else:
                run.launch()
            torch.cuda.synchronize()
            out.append((model.grad.clone(), run.loss[:B].clone()))
        run.check()
        g0 = out[0][0]
        msg = []
        for i, (gr, lo) in enumerate(out[1:], 1):
            if not torch.isfinite(gr).all() or not torch.isfinite(lo).all():
                msg.append(f"poison{i}: non-finite")
            else:
                e = float((gr - g0).abs().max() / g0.abs().max())
                if e > 1e-6:
                    msg.append(f"poison{i}: err {e:.1e}")
        if msg:
            print("epoch", epoch, "it", it, msg, flush=True)
print("done")
