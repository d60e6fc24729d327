"""CUDA-graph replay of the training loop (engine.GraphLoop) against the eager
run-ahead loop, and the eager loop against the oracle's model-centric
iteration (S = 1).  Graph replay must not change the math: the same kernels
run in the same order, so parameters agree to float-atomics reordering
(fp32: 1e-5 max-relative after several SGD steps; bf16: the 1e-2 bf16 step
tolerance, since a reordered sum can flip one bf16 rounding).  The fp32 run is pinned to the
float64 oracle at the 1e-3 tolerance of tests/test_step_gpu.py."""
import numpy as np
import pytest
import torch

from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables

pytestmark = pytest.mark.gpu

N, B, ITERS = 6000, 96, 7


@pytest.fixture(scope="module")
def world():
    off, tgt = build_csr(build_tables(OSpec(n=N, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4,
                                            d_cap=800, seed=21)))
    from paper_2409_00657_b200.graph import Graph
    return off, tgt, Graph.from_host(off, tgt)


def _trainer(world, graphs, dtype, arch="sage-mean", fanout=(15, 10), hidden=64):
    from paper_2409_00657_b200.engine import Trainer
    from paper_2409_00657_b200.featstore import FeatureTable
    from paper_2409_00657_b200.model import init_model
    from paper_2409_00657_b200.rng import chain
    seed, D, C = 5, 32, 11
    g = world[2]
    table = FeatureTable.generated(g.n_vertices, D, seed, dtype)
    model = init_model(arch, D, hidden, len(fanout), C, chain(seed, 0x07))
    tr = Trainer(g, table, model, fanout, B, seed, lr=0.1, iterations=ITERS, graphs=graphs)
    return tr, model


def _maxrel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("arch,fanout,hidden", [("sage-mean", (15, 10), 64),
                                                ("gcn", (10, 10), 128)])
def test_graph_replay_matches_eager(world, dtype, arch, fanout, hidden):
    ref, m_ref = _trainer(world, False, dtype, arch, fanout, hidden)
    got, m_got = _trainer(world, True, dtype, arch, fanout, hidden)
    for epoch in range(2):
        for tr in (ref, got):
            iters = tr.begin_epoch(epoch)
            for it in range(iters):
                tr.step(it)
        torch.cuda.synchronize()
        assert got._gl is not None, "graph loop never engaged"
        err = _maxrel(m_got.flat, m_ref.flat)
        # bf16: a float-atomics reordering can flip one bf16 rounding (2^-8 relative)
        # of an operand, which SGD then carries -- the bf16 step tolerance applies
        tol = 1e-5 if dtype == torch.float32 else 1e-2
        assert err < tol, f"epoch {epoch}: params differ from eager by {err:.2e}"
    ref.check()
    got.check()


def test_graph_e2e_train_step_matches_eager(world):
    """Public train_step (pinned host roots in, loss out) through the graph loop."""
    ref, m_ref = _trainer(world, False, torch.float32)
    got, m_got = _trainer(world, True, torch.float32)
    for tr in (ref, got):
        tr.begin_epoch(0)
    roots = [ref.roots_of(it).cpu().pin_memory() for it in range(ref.iters)]
    losses = {}
    for name, tr in (("ref", ref), ("got", got)):
        out = []
        for it in range(tr.iters):
            nxt = roots[it + 1] if it + 1 < tr.iters else None
            prev = tr.train_step(roots[it], it, nxt)
            if prev is not None:
                out.append(prev)
        out.append(tr.last_loss())
        losses[name] = out
    torch.cuda.synchronize()
    assert got._gl_e2e is not None, "e2e graph loop never engaged"
    assert len(losses["got"]) == len(losses["ref"]) == ref.iters
    np.testing.assert_allclose(losses["got"], losses["ref"], rtol=1e-5)
    assert _maxrel(m_got.flat, m_ref.flat) < 1e-5


def test_eager_loop_matches_oracle(world):
    """S = 1 model-centric iterations of the oracle engine == the device loop."""
    from oracle import engine as OE
    off, tgt, _ = world
    tr, m = _trainer(world, True, torch.float32)
    tr.begin_epoch(0)
    for it in range(tr.iters):
        tr.step(it)
    torch.cuda.synchronize()
    w = OE.World(off, tgt, np.zeros(N, np.int64), 1, 5, "sage-mean", 32, 64, 11, (15, 10), B,
                 iterations=ITERS)
    P = w.fresh_params()
    for it, batches in enumerate(OE.epoch_batches(5, 0, N, 1, B, ITERS)):
        OE.model_centric_iteration(w, P, 0, it, batches)
    for i, (a, b) in enumerate(zip(m.params(), P.arrays())):
        err = float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))
        assert err < 1e-3, f"param {i}: {err:.2e}"
