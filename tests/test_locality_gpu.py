"""Layer-wise sampling (sampler.py:109-120, shared draw by the CUDA
pick_k_smallest) and the locality report (metrics.py:23-113) against gnnsim."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "gnnsim")):
    pytest.skip("baseline/_ref not installed (baseline/install_ref.sh)", allow_module_level=True)


@pytest.fixture(scope="module")
def gs():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gnnsim_numba_cache")
    sys.path.insert(0, REF)
    import gnnsim
    import gnnsim.config, gnnsim.metrics, gnnsim.sampler, gnnsim.graph  # noqa: E401,F401
    return gnnsim


@pytest.mark.parametrize("fanout", [(4, 3), (20, 20, 10)])
def test_layer_wise_micrographs_match_gnnsim(gs, fanout):
    from paper_2409_00657_b200.graph import SbmSpec, generate_sbm
    from paper_2409_00657_b200.sampler import SamplerConfig, sample_micrograph
    from paper_2409_00657_b200.rng import chain
    spec = SbmSpec((150, 120, 90), 0.1, 0.01, chain(2, 1))
    g = generate_sbm(spec)
    rg = gs.graph.generate_sbm(gs.graph.SbmSpec(spec.block_sizes, spec.p_in, spec.p_out,
                                                spec.seed))
    cfg = SamplerConfig(len(fanout), fanout, "layer-wise", seed=chain(5, 6))
    rcfg = gs.sampler.SamplerConfig(len(fanout), fanout, "layer-wise", chain(5, 6))
    for r in range(0, 360, 17):
        k = cfg.stream_key(0, 1, r)
        a = sample_micrograph(g, r, cfg, k)
        b = gs.sampler.sample_micrograph(rg, r, rcfg, k)
        assert all(np.array_equal(x, y) for x, y in zip(a.layers, b.layers))
        assert all(np.array_equal(x, z) and np.array_equal(y, w)
                   for (x, y), (z, w) in zip(a.pairs, b.pairs))
        assert np.array_equal(a.vertices, b.vertices)


def test_locality_report_matches_gnnsim(gs):
    from paper_2409_00657_b200.locality import locality_report, write_locality_csv
    cfg = gs.config.RunConfig(graph="sbm", blocks=(120, 100, 80), p_in=0.12, p_out=0.01,
                              fanout=(3,), batch=16, seed=3)
    args = (["hash", "greedy"], ["node-wise", "layer-wise"], [2, 3], [1, 2])
    want = gs.metrics.locality_report(cfg, *args, iterations=2)
    got = locality_report(cfg, *args, iterations=2)
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert (a.n_servers, a.n_layers, a.mode, a.partitioner, a.samples) == \
            (b.n_servers, b.n_layers, b.mode, b.partitioner, b.samples)
        assert abs(a.r_micro_mean - b.r_micro_mean) <= 1e-12
        assert abs(a.r_sub_mean - b.r_sub_mean) <= 1e-12
    import io
    s1, s2 = io.StringIO(), io.StringIO()
    write_locality_csv(got, s1)
    gs.metrics.write_locality_csv(want, s2)
    got_rows = gs.metrics.read_locality_csv(io.StringIO(s1.getvalue()))  # same format
    want_rows = gs.metrics.read_locality_csv(io.StringIO(s2.getvalue()))
    for a, b in zip(got_rows, want_rows):   # means may differ in the last ulp
        assert a.samples == b.samples and abs(a.r_sub_mean - b.r_sub_mean) <= 1e-12
