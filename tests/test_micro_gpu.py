"""Per-micrograph model API (paper_2409_00657_b200.micro: build_plan, forward,
loss_and_backward, accumulate, sync_and_update) against gnnsim's own
(model.py:183-329), fp32 device math vs float64: 1e-3 relative."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "gnnsim")):
    pytest.skip("baseline/_ref not installed (baseline/install_ref.sh)", allow_module_level=True)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("arch,fanout,D,H,C", [("sage-mean", (15, 10), 24, 16, 7),
                                               ("gcn", (10, 10, 10), 20, 16, 5),
                                               ("sage-mean", (5, 5, 3), 13, 24, 4)])
def test_per_micrograph_api_matches_gnnsim(arch, fanout, D, H, C):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gnnsim_numba_cache")
    sys.path.insert(0, REF)
    import gnnsim.graph as gg
    import gnnsim.kernels as gk
    import gnnsim.model as gm
    import gnnsim.sampler as gsamp
    from oracle.graphgen import GraphSpec, build_csr, build_tables
    from paper_2409_00657_b200 import micro as M
    from paper_2409_00657_b200.featstore import CommLedger
    from paper_2409_00657_b200.model import init_model
    from paper_2409_00657_b200.rng import chain
    off, tgt = build_csr(build_tables(GraphSpec(n=3000, avg_deg=12.0, beta=0.7, p_in=0.9,
                                                n_blocks=4, d_cap=600, seed=11)))
    g = gg.Graph(3000, off, tgt, directed=True)
    cfg = gsamp.SamplerConfig(len(fanout), fanout, seed=chain(3, 6))
    ref = [gm.init_model(arch, D, H, len(fanout), C, chain(3, 7)) for _ in range(2)]
    mine = [init_model(arch, D, H, len(fanout), C, chain(3, 7)) for _ in range(2)]
    labels = gm.LabelOracle(C, chain(3, 4))
    accs_r = [gm.GradAccumulator.for_model(d, ref[0]) for d in range(2)]
    accs_m = [M.GradAccumulator.for_model(d, mine[0]) for d in range(2)]
    roots = np.random.default_rng(0).choice(3000, 12, replace=False)
    for i, r in enumerate(roots.tolist()):
        m = gsamp.sample_micrograph(g, r, cfg, gsamp.stream_key(cfg.seed, 0, 0, r))
        x = gk.feature_rows(m.vertices, D, chain(chain(3, 3), 0xFE))
        p_r, p_m = gm.build_plan(m), M.build_plan(m)
        assert all(np.array_equal(a, b) for a, b in zip(p_r.need, p_m.need))
        st_r = gm.forward(m, x, ref[0])
        st_m = M.forward(m, x, mine[0])
        assert _rel(st_m.logits, st_r.logits) < 1e-3
        for a, b in zip(st_m.values, st_r.values):
            assert _rel(a, b) < 1e-3
        for a, b in zip(st_m.pre_relu, st_r.pre_relu):
            assert _rel(a, b) < 1e-3
        lr_, g_r = gm.loss_and_backward(st_r, labels.label(r), ref[0])
        lm_, g_m = M.loss_and_backward(st_m, labels.label(r), mine[0])
        assert abs(lm_ - lr_) <= 1e-3 * max(1.0, abs(lr_))
        for a, b in zip(g_m.arrays(), g_r.arrays()):
            assert _rel(a, b) < 1e-3
        gm.accumulate(accs_r[i % 2], g_r)
        M.accumulate(accs_m[i % 2], g_m)
    import gnnsim.featstore as gf
    led_r, led_m = gf.CommLedger(), CommLedger()
    step_r = gm.sync_and_update(ref, accs_r, len(roots), 0.1, led_r)
    step_m = M.sync_and_update(mine, accs_m, len(roots), 0.1, led_m)
    for a, b in zip(step_m.arrays(), step_r.arrays()):
        assert _rel(a, b) < 1e-3
    for model in mine:
        for a, b in zip(model.params(), ref[0].params()):
            assert _rel(a, b) < 1e-3
    assert {k: tuple(v) for k, v in led_m.counters.items()} == \
        {k: tuple(v) for k, v in led_r.counters.items()}
