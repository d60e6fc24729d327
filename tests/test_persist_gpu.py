"""Persistent training step (k_step_persist, hg_set_persist) against the split
kernels it replaces, on the same micrograph batch (model.py:213-329, L = 2,
bf16 tensor-core path).

The persistent kernel runs the split kernels' arithmetic (same bf16 operands,
rounding points and per-element accumulation order); only the order of the
atomic bias-gradient column sums and of the split-K weight-gradient
reductions differs.  So: losses and the forward activations bit-identical;
gradients and SGD-updated parameters within 1e-5 of max|ref| (float32
summation-order noise).  The split path itself is pinned to the oracle by
tests/test_step_gpu.py.  A 128-root capacity holding 96 real roots (device
root count) exercises the zeroed capacity rows.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables
from oracle.rng import chain

pytestmark = pytest.mark.gpu

# (arch, fanout, D, H, C): in_dim[1] (2D for SAGE, D for GCN) a multiple of 64,
# C a multiple of 4 (16-byte logit rows for the TMA store)
CASES = [("sage-mean", (15, 10), 128, 256, 172),
         ("sage-mean", (10, 5), 32, 64, 8),
         ("gcn", (10, 10), 64, 128, 40)]
TOL = 1e-5


@pytest.fixture(scope="module")
def world():
    kw = dict(n=3000, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4, d_cap=600, seed=11)
    off, tgt = build_csr(build_tables(OSpec(**kw)))
    from paper_2409_00657_b200.graph import Graph
    return Graph.from_host(off, tgt)


def _rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).abs().max() / max(float(b.abs().max()), 1e-30))


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-D{c[2]}-H{c[3]}-C{c[4]}")
def test_persistent_step_matches_split(world, case):
    from paper_2409_00657_b200 import _lib
    from paper_2409_00657_b200.featstore import FeatureTable
    from paper_2409_00657_b200.model import LabelOracle, init_model
    from paper_2409_00657_b200.trainer import CellRunner
    arch, fo, D, H, Cn = case
    cap, n_real = 128, 96
    model = init_model(arch, D, H, 2, Cn, chain(5, 0x07))
    table = FeatureTable.generated(world.n_vertices, D, 5, dtype=torch.bfloat16)
    run = CellRunner(world, table, model, fo, cap, LabelOracle(Cn, chain(5, 0x04)))
    roots = np.random.default_rng(3).choice(world.n_vertices, cap, replace=False).astype(np.int64)
    st = np.uint64(chain(chain(5, 6), 0, 1)).view(np.int64)
    run.stage_roots(roots, [st], cap)
    n_dev = torch.tensor([n_real], dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    run.builder.build(world, run.roots, run.keys, cap, n_roots=cap, n_dev=n_dev.data_ptr())
    _lib.call("hg_step_prologue", C.byref(run.desc), cap, 1, s)
    run.desc.agg1_ready = 1
    m = model
    flat0 = m.flat.clone()

    def step(persist, update):
        _lib.call("hg_set_persist", persist, 0, 0)
        m.flat.copy_(flat0)
        m.grad.zero_()
        _lib.call("hg_sgd_refresh", C.byref(run.desc), m.flat.data_ptr(), m.grad.data_ptr(),
                  m.flat.numel(), 0.0, 1.0, 0, s)
        run.desc.lowp_fresh = 1
        try:
            _lib.call("hg_train_step_sgd", C.byref(run.desc), cap, m.flat.data_ptr(),
                      m.grad.data_ptr(), m.flat.numel(), 0.05, 1.0 / n_real, update, s)
            torch.cuda.synchronize()
        finally:
            run.desc.lowp_fresh = 0
            _lib.call("hg_set_persist", 0, 0, 0)
        run.check()
        return (run.loss.clone(), m.grad.clone(), m.flat.clone(), run.h[1].clone(),
                run.h[2].clone(), run.dl16.clone())

    tot = run.builder.tensors["totals"].cpu().numpy()
    n1, n2 = int(tot[1]), int(tot[2])
    assert n2 == n_real
    la, ga, _, h1a, h2a, dla = step(0, 0)
    lb, gb, _, h1b, h2b, dlb = step(1, 0)
    assert torch.equal(la, lb), "losses (capacity rows included) differ"
    assert torch.equal(h1a[:n1], h1b[:n1]) and torch.equal(h2a[:n2], h2b[:n2])
    assert torch.equal(dla, dlb)
    assert float(lb[n_real:].abs().max()) == 0.0
    assert not torch.isnan(ga).any(), f"split-path gradients NaN at {torch.nonzero(torch.isnan(ga)).flatten()[:6].tolist()}"
    assert not torch.isnan(gb).any(), f"persistent gradients NaN at {torch.nonzero(torch.isnan(gb)).flatten()[:6].tolist()} offsets {list(m.offsets)}"
    assert _rel(gb, ga) <= TOL, f"gradients {_rel(gb, ga):.3e}"
    _, _, pa, _, _, _ = step(0, 1)
    _, gz, pb, _, _, _ = step(1, 1)
    # the update (lr * g / B) is ~1e-3 of the weights: its float32 difference
    # carries the weights' rounding (one ulp of |w| ~ 1e-5 of the update)
    assert _rel(pb - flat0, pa - flat0) <= 10 * TOL, "SGD updates differ"
    assert _rel(pb, pa) <= 1e-6, "updated parameters differ"
    assert float(gz.abs().max()) == 0.0, "gradients not reset by the fused SGD"
    # bf16 operand copies refreshed by the fused SGD == hg_sgd_refresh of the same parameters
    lowp = [t.clone() for t in (run.wb16, run.wct, run.wcp)]
    _lib.call("hg_sgd_refresh", C.byref(run.desc), m.flat.data_ptr(), m.grad.data_ptr(),
              m.flat.numel(), 0.0, 1.0, 0, s)
    torch.cuda.synchronize()
    for a, b in zip(lowp, (run.wb16, run.wct, run.wcp)):  # bitwise (unused slots hold garbage)
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))


def test_persist_ineligible_falls_back_to_split(world):
    """A descriptor the persistent kernel does not cover (L = 3) runs the split
    kernels through the same entry point, with identical results."""
    from paper_2409_00657_b200 import _lib
    from paper_2409_00657_b200.featstore import FeatureTable
    from paper_2409_00657_b200.model import LabelOracle, init_model
    from paper_2409_00657_b200.trainer import CellRunner
    model = init_model("gcn", 64, 64, 3, 5, 3)
    table = FeatureTable.generated(world.n_vertices, 64, 3, dtype=torch.bfloat16)
    run = CellRunner(world, table, model, (5, 5, 5), 64, LabelOracle(5, 9))
    roots = np.arange(0, 3000, 47, dtype=np.int64)[:64]
    run.stage_roots(roots, [np.uint64(chain(1, 0, 0)).view(np.int64)], 64)
    s = torch.cuda.current_stream().cuda_stream
    run.builder.build(world, run.roots, run.keys, 64, n_roots=64)
    _lib.call("hg_step_prologue", C.byref(run.desc), 64, 1, s)
    run.desc.agg1_ready = 1
    out = []
    for persist in (0, 1):
        _lib.call("hg_set_persist", persist, 0, 0)
        model.grad.zero_()
        run.desc.lowp_fresh = 0
        try:
            _lib.call("hg_train_step_sgd", C.byref(run.desc), 64, model.flat.data_ptr(),
                      model.grad.data_ptr(), model.flat.numel(), 0.0, 1.0, 0, s)
            torch.cuda.synchronize()
        finally:
            _lib.call("hg_set_persist", 0, 0, 0)
        out.append((run.loss.clone(), model.grad.clone()))
    assert torch.equal(out[0][0], out[1][0])
    assert _rel(out[1][1], out[0][1]) <= TOL
