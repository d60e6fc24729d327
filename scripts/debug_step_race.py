"""Debug: run the train step of one batch many times; look for nondeterminism."""
import sys, torch, numpy as np, ctypes as C
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_graph_gpu as T
from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables
from paper_2409_00657_b200.graph import Graph
from paper_2409_00657_b200.batching import epoch_permutation
from paper_2409_00657_b200.rng import chain
from paper_2409_00657_b200.featstore import FeatureTable
from paper_2409_00657_b200.model import init_model, LabelOracle
from paper_2409_00657_b200.trainer import CellRunner
from paper_2409_00657_b200 import _lib
off, tgt = build_csr(build_tables(OSpec(n=T.N, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4, d_cap=800, seed=21)))
g = Graph.from_host(off, tgt)
seed, D, Cc, B = 5, 32, 11, T.B
table = FeatureTable.generated(g.n_vertices, D, seed, torch.float32)
model = init_model("sage-mean", D, 64, 2, Cc, chain(seed, 0x07))
run = CellRunner(g, table, model, (15, 10), B, LabelOracle(Cc, chain(seed, 4)))
side = torch.cuda.Stream()
for epoch, it in ((1, 10), (1, 9), (0, 10)):
    perm = epoch_permutation(seed, epoch, g.n_vertices, "cuda")
    roots = perm[it * B:(it + 1) * B].clone()
    st = np.uint64(chain(chain(seed, 6), epoch, it)).view(np.int64)
    run.stage_roots(roots, [st], B)
    ref = None
    nbad = 0
    for rep in range(300):
        model.grad.zero_()
        if rep % 2 == 0:
            with torch.cuda.stream(side):
                x = torch.randn(2048, 2048, device="cuda") @ torch.randn(2048, 2048, device="cuda")
        run.launch()
        cur = (model.grad.clone(), run.loss[:B].clone())
        torch.cuda.synchronize()
        if ref is None:
            ref = cur
            continue
        e = float((cur[0] - ref[0]).abs().max() / ref[0].abs().max())
        el = float((cur[1] - ref[1]).abs().max())
        if e > 1e-5 or el > 1e-5:
            nbad += 1
            if nbad <= 3:
                print("epoch", epoch, "it", it, "rep", rep, f"grad err {e:.2e} loss err {el:.2e}")
    run.check()
    print("epoch", epoch, "it", it, "mismatches", nbad, "of 299", flush=True)
