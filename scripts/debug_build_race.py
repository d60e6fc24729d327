"""Debug: rebuild one batch many times and look for nondeterministic roots."""
import sys, torch, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import test_graph_gpu as T
from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables
from paper_2409_00657_b200.graph import Graph
from paper_2409_00657_b200.batching import epoch_permutation
from paper_2409_00657_b200.rng import chain
from paper_2409_00657_b200.sampler import MicrographBuilder
off, tgt = build_csr(build_tables(OSpec(n=T.N, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4, d_cap=800, seed=21)))
g = Graph.from_host(off, tgt)
seed = 5
B = T.B
for epoch, it in ((1, 10), (0, 10), (1, 9)):
    perm = epoch_permutation(seed, epoch, g.n_vertices, "cuda")
    roots = perm[it * B:(it + 1) * B].clone()
    st = torch.tensor(np.array([chain(chain(seed, 6), epoch, it)], dtype=np.uint64).view(np.int64), device="cuda")
    b = MicrographBuilder((15, 10), B)
    ref = None
    nbad = 0
    side = torch.cuda.Stream()
    for rep in range(300):
        b.build(g, roots, st, B)
        if rep % 3 == 0:  # perturb: concurrent work on another stream
            with torch.cuda.stream(side):
                x = torch.randn(4096, 4096, device="cuda") @ torch.randn(4096, 4096, device="cuda")
        t = {k: (v[:] if not isinstance(v, list) else [x.clone() if x is not None else None for x in v]) for k, v in b.tensors.items()}
        tot = b.tensors["totals"].clone()
        cur = [tot] + [b.tensors[n][k].clone() for n in ("need_ids", "need_off", "nbr_off", "nbr_idx", "self_pos") for k in range(3) if b.tensors[n][k] is not None]
        torch.cuda.synchronize()
        if ref is None:
            ref = cur
            continue
        same = all(torch.equal(a, c) for a, c in zip(ref, cur))
        if not same:
            nbad += 1
            if nbad <= 3:
                diffs = [i for i, (a, c) in enumerate(zip(ref, cur)) if not torch.equal(a, c)]
                print("epoch", epoch, "it", it, "rep", rep, "differs in", diffs, "totals", ref[0].tolist(), cur[0].tolist())
    b.check()
    print("epoch", epoch, "it", it, "mismatches", nbad, "of 299")
