"""The oracle against the LIVE reference (gnnsim) on randomised inputs (CPU).

gnnsim is imported from baseline/_ref (baseline/install_ref.sh) or, in the
build container, from /root/reference/pkg/src; the module is skipped where
neither exists.  Complements the golden vectors (test_oracle_golden.py) with
inputs the goldens do not hold: the benchmark generator's hub rows, random
fanouts and both architectures.  Also pins oracle/graphgen.rows_csr (the
vectorised row generator the bench-shape parity tests and the reference arm
use) to the scalar row() it restates.
"""
import os
import sys

import numpy as np
import pytest

from oracle import kernels as OK
from oracle import model as OM
from oracle.cpu_bench import LazyGraphSampler
from oracle.graphgen import GraphSpec, build_csr, build_tables, row, rows_csr
from oracle.rng import chain
from oracle.sampler import sample_micrograph as o_sample

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gnnsim():
    for path in (os.path.join(REPO, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "gnnsim")):
            os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gnnsim_numba_cache")
            if path not in sys.path:
                sys.path.insert(0, path)
            import gnnsim  # noqa: F401
            from gnnsim import graph, kernels, model, sampler  # noqa: F401
            return sys.modules["gnnsim"]
    return None


gs = _gnnsim()
needs_ref = pytest.mark.skipif(gs is None, reason="gnnsim (reference) not available")

SPEC = GraphSpec(n=5000, avg_deg=14.0, beta=0.8, p_in=0.9, n_blocks=4, d_cap=2000, seed=3)


@pytest.fixture(scope="module")
def csr():
    return build_csr(build_tables(SPEC))


def test_rows_csr_matches_row():
    for spec in (SPEC, GraphSpec(n=111_000_000, avg_deg=15.6, beta=0.6, p_in=0.95,
                                 n_blocks=8, d_cap=1 << 15, seed=0)):
        t = build_tables(spec)
        vs = np.random.default_rng(7).integers(0, spec.n, 400)
        off, tgt = rows_csr(t, vs)
        for i, v in enumerate(vs.tolist()):
            assert np.array_equal(tgt[off[i]:off[i + 1]], row(t, v))


@needs_ref
@pytest.mark.parametrize("fanout", [1, 3, 10, 25])
def test_sample_frontier_vs_gnnsim(csr, fanout):
    off, tgt = csr
    deg = np.diff(off)
    rng = np.random.default_rng(fanout)
    frontier = np.concatenate([np.argsort(-deg)[:20], rng.integers(0, SPEC.n, 200)])
    for st in (chain(1, fanout), chain(99, 2)):
        a = OK.sample_frontier(off, tgt, frontier, fanout, st)
        b = gs.kernels.sample_frontier(off, tgt, frontier, fanout, st)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@needs_ref
@pytest.mark.parametrize("fanout", [(15, 10), (10, 10, 10), (10, 10, 5, 5)])
def test_micrographs_vs_gnnsim(csr, fanout):
    off, tgt = csr
    g = gs.graph.Graph(SPEC.n, off, tgt, directed=True)
    cfg = gs.sampler.SamplerConfig(len(fanout), fanout, seed=chain(4, 6))
    lazy = LazyGraphSampler(SPEC)
    roots = np.random.default_rng(1).integers(0, SPEC.n, 40)
    keys = [gs.sampler.stream_key(cfg.seed, 0, 3, int(r)) for r in roots]
    mine = lazy.micrographs(roots, fanout, keys)
    for r, k, m in zip(roots.tolist(), keys, mine):
        ref = gs.sampler.sample_micrograph(g, r, cfg, k)
        o = o_sample(off, tgt, r, fanout, k)
        for x in (m, o):
            assert all(np.array_equal(a, b) for a, b in zip(x.layers, ref.layers))
            assert all(np.array_equal(a, c) and np.array_equal(b, d)
                       for (a, b), (c, d) in zip(x.pairs, ref.pairs))
            assert np.array_equal(x.vertices, ref.vertices)
        plan = gs.model.build_plan(ref)
        need, steps = OM.build_plan(m)
        assert all(np.array_equal(a, b) for a, b in zip(need, plan.need))
        assert all(np.array_equal(a, b) for x, y in zip(steps, plan.layers) for a, b in zip(x, y))


@needs_ref
@pytest.mark.parametrize("arch,fanout", [("sage-mean", (15, 10)), ("gcn", (10, 10, 10)),
                                         ("sage-mean", (10, 10, 5, 5))])
def test_forward_backward_sgd_vs_gnnsim(csr, arch, fanout):
    off, tgt = csr
    g = gs.graph.Graph(SPEC.n, off, tgt, directed=True)
    D, H, C, seed = 24, 16, 7, 11
    cfg = gs.sampler.SamplerConfig(len(fanout), fanout, seed=chain(seed, 6))
    ref_model = gs.model.init_model(arch, D, H, len(fanout), C, chain(seed, 7))
    P = OM.init_params(arch, D, H, len(fanout), C, chain(seed, 7))
    assert all(np.array_equal(a, b) for a, b in zip(P.arrays(), ref_model.params()))
    labels = gs.model.LabelOracle(C, chain(seed, 4))
    fstate = chain(chain(seed, 3), 0xFE)
    acc = gs.model.GradAccumulator.for_model(0, ref_model)
    G = P.zeros()
    roots = np.random.default_rng(2).integers(0, SPEC.n, 24)
    for r in roots.tolist():
        m = gs.sampler.sample_micrograph(g, r, cfg, gs.sampler.stream_key(cfg.seed, 0, 0, r))
        x = gs.kernels.feature_rows(m.vertices, D, fstate)
        assert np.array_equal(x, OK.feature_rows(m.vertices, D, fstate))
        st = gs.model.forward(m, x, ref_model)
        loss, gr = gs.model.loss_and_backward(st, labels.label(r), ref_model)
        gs.model.accumulate(acc, gr)
        ost = OM.forward(m, x, P)
        assert int(OM.labels([r], C, chain(seed, 4))[0]) == labels.label(r)
        oloss, og = OM.loss_and_grads(ost, labels.label(r), P)
        assert abs(oloss - loss) <= 1e-12 * max(1.0, abs(loss))
        OM.add_into(G, og)
    for a, b in zip(G.arrays(), acc.grads.arrays()):
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-12)
    gs.model.sync_and_update([ref_model], [acc], len(roots), 0.1)
    OM.sgd_step(P, G, len(roots), 0.1)
    for a, b in zip(P.arrays(), ref_model.params()):
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-12)
