"""Debug: group loop vs eager run-ahead vs no run-ahead, end-of-epoch params."""
import sys, torch, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_graph_gpu as T
from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables
from paper_2409_00657_b200.graph import Graph
from paper_2409_00657_b200.engine import Trainer
from paper_2409_00657_b200.featstore import FeatureTable
from paper_2409_00657_b200.model import init_model
from paper_2409_00657_b200.rng import chain
off, tgt = build_csr(build_tables(OSpec(n=T.N, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4, d_cap=800, seed=21)))
g = Graph.from_host(off, tgt)


def mk(graphs, group, run_ahead=True):
    seed, D, C = 5, 32, 11
    table = FeatureTable.generated(g.n_vertices, D, seed, torch.float32)
    model = init_model("sage-mean", D, 64, 2, C, chain(seed, 0x07))
    tr = Trainer(g, table, model, (15, 10), T.B, seed, lr=0.1, iterations=T.G_ITERS,
                 graphs=graphs, group=group, run_ahead=run_ahead)
    return tr, model


for trial in range(int(sys.argv[1])):
    trs = {"plain": mk(False, 1, False), "ra": mk(False, 1), "g1": mk(True, 1), "g4": mk(True, 4),
           "g2": mk(True, 2)}
    out = []
    for epoch in range(3):
        for name, (tr, m) in trs.items():
            iters = tr.begin_epoch(epoch)
            for it in range(iters):
                tr.step(it)
        torch.cuda.synchronize()
        base = trs["plain"][1].flat
        out.append(" ".join(f"{n}:{T._maxrel(m.flat, base):.1e}" for n, (tr, m) in trs.items()
                            if n != "plain"))
    print(trial, " | ".join(out), flush=True)
