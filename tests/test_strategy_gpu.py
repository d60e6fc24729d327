"""Trainer-level drop-in (paper_2409_00657_b200.strategy) against the reference
trainer itself (gnnsim from baseline/_ref): run_strategy(RunConfig) ->
EpochMetrics for every supported strategy, on SBM worlds with the hash and
greedy partitioners and a non-trivial cost model (so simulated time and the
merge controller's decisions are exercised).

Exact: graph (SBM pair pass on the GPU), partition homes (GPU greedy BFS),
ledger counters per link and category, bytes by category, miss rate, alpha,
imbalance, trained compositions, column counts, staged bytes, simulated
seconds.  Parameters after training: fp32 device math vs the reference's
float64, 1e-3 relative (north_star).
"""
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
def E():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gnnsim_numba_cache")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import gnnsim.engine as E
    return E


COST = dict(bandwidth=2e6, latency=1e-4, sync_overhead=1e-3, kernel_launch=1e-5,
            compute_rate=1e-9)


def _cfg(E, **kw):
    from gnnsim.config import RunConfig
    base = dict(graph="sbm", blocks=(300, 250, 250), p_in=0.08, p_out=0.004, servers=3,
                partitioner="hash", layers=2, fanout=(5, 3), dim=16, hidden=16, classes=5,
                arch="sage-mean", lr=0.1, batch=32, epochs=3, strategy="micrograph", seed=4,
                **COST)
    base.update(kw)
    return RunConfig(**base)


def _reference(E, cfg):
    """gnnsim's run_* with access to its trained models."""
    world = E.build_world(cfg)
    models = E.fresh_models(world)
    s = cfg.strategy
    if s == "model-centric":
        ms = [E._model_centric_epoch(world, models, e) for e in range(cfg.epochs)]
    elif s == "micrograph+pg+merge":
        ms, _, _ = E.merge_controller(cfg, world=world, models=models, pregather=True, name=s)
    elif s == "locality-optimized":
        return E.run_locality_optimized(cfg), None, world
    else:
        tt = E.TraceTable.initial(world.n_servers)
        ms = [E._micrograph_epoch(world, models, tt, e, s == "micrograph+pg", s)
              for e in range(cfg.epochs)]
    return ms, models[0], world


def _same_metrics(a, b):
    assert a.epoch == b.epoch and a.strategy == b.strategy
    assert a.steps == b.steps and a.iterations == b.iterations and a.n_columns == b.n_columns
    norm = lambda led: {k: (float(v[0]), int(v[1])) for k, v in led.counters.items()}  # noqa
    assert norm(a.ledger) == norm(b.ledger)
    assert a.bytes_by_category == b.bytes_by_category
    assert a.miss_rate == b.miss_rate and a.alpha == b.alpha and a.imbalance == b.imbalance
    assert a.staged_bytes == b.staged_bytes
    assert a.composition_diverged == b.composition_diverged
    assert len(a.trained) == len(b.trained)
    for ta, tb in zip(a.trained, b.trained):
        assert all(np.array_equal(x, y) for x, y in zip(ta, tb))
    assert abs(a.sim_seconds - b.sim_seconds) <= 1e-9 * max(1.0, abs(b.sim_seconds))
    np.testing.assert_allclose(a.busy_seconds, b.busy_seconds, rtol=1e-9)


@pytest.mark.parametrize("strategy", ["model-centric", "micrograph", "micrograph+pg",
                                      "micrograph+pg+merge", "locality-optimized"])
@pytest.mark.parametrize("partitioner", ["hash", "greedy"])
def test_run_strategy_matches_reference(E, strategy, partitioner):
    from paper_2409_00657_b200 import strategy as S
    cfg = _cfg(E, strategy=strategy, partitioner=partitioner,
               merge_k=1, epochs=4 if "merge" in strategy else 2)
    want, ref_model, ref_world = _reference(E, cfg)
    world = S.build_world(cfg)
    off, tgt = world.graph.to_host()
    assert np.array_equal(off, ref_world.graph.offsets)
    assert np.array_equal(tgt, ref_world.graph.targets)
    assert np.array_equal(world.partition.home, ref_world.partition.home)
    got = S.run_strategy(cfg, world=world)
    assert len(got) == len(want)
    for a, b in zip(got, want):
        _same_metrics(a, b)
    if ref_model is not None:
        for x, y in zip(world.model.params(), ref_model.params()):
            err = np.abs(x - y).max() / max(np.abs(y).max(), 1e-30)
            assert err < 1e-3, err


def test_greedy_partition_matches_reference_on_power_law(E):
    """The GPU greedy BFS on a 50K-vertex power-law graph (many re-seeds, cap
    cutting inside rows), slack 0 and 0.1, 2..8 parts."""
    import gnnsim.graph as gg
    from paper_2409_00657_b200.graph import GraphSpec, generate, partition_greedy_locality
    g = generate(GraphSpec(n=50_000, avg_deg=9.0, beta=0.8, p_in=0.9, n_blocks=8,
                           d_cap=3000, seed=2))
    off, tgt = g.to_host()
    rg = gg.Graph(g.n_vertices, off, tgt, directed=True)
    for S_, slack in ((2, 0.0), (3, 0.1), (8, 0.0)):
        a = partition_greedy_locality(g, S_, slack)
        b = gg.partition_greedy_locality(rg, S_, slack)
        assert np.array_equal(a.home, b.home), (S_, slack)


def test_partition_and_feature_files_roundtrip(E, tmp_path):
    import gnnsim.featstore as gf
    import gnnsim.graph as gg
    from paper_2409_00657_b200.featstore import FeatureTable, read_feature_file, write_feature_file
    from paper_2409_00657_b200.graph import PartitionMap, load_partition, save_partition
    home = np.random.default_rng(0).integers(0, 4, 1000)
    p = PartitionMap(home, 4)
    save_partition(p, tmp_path / "a.part")
    assert np.array_equal(gg.load_partition(str(tmp_path / "a.part"), 4).home, home)
    gg.save_partition(gg.PartitionMap(home, 4), str(tmp_path / "b.part"))
    assert np.array_equal(load_partition(tmp_path / "b.part", 4).home, home)
    m = np.random.default_rng(1).standard_normal((300, 13)).astype(np.float32)
    write_feature_file(m, tmp_path / "a.feat")
    assert np.array_equal(gf.read_feature_file(str(tmp_path / "a.feat")), m)
    gf.write_feature_file(m, str(tmp_path / "b.feat"))
    assert np.array_equal(read_feature_file(tmp_path / "b.feat"), m)
    t = FeatureTable.from_file(tmp_path / "b.feat")
    assert np.array_equal(t.rows(np.arange(300)), m)
