"""The drop-in boundary exercised from the reference's side (GPU).

1. Every function of the reference operator layer (gnnsim.kernels:
   sample_frontier, feature_rows, pick_k_smallest, sbm_edges) against gnnsim's
   own numba backend on randomised inputs, bit-exact.
2. gnnsim's OWN test-suite (test_kernels / test_sampler / test_graph /
   test_featstore / test_model / test_engine) run with its operator layer bound
   to libhopgnn (tests/gnnsim_cuda_plugin.py) -- the GNNSIM_KERNELS=cuda backend
   a gnnsim maintainer would add.
3. BASELINE configs[0] (cfg1: GraphSAGE-2, fanout (10, 5), hidden 128, batch
   1024, 100K-vertex power-law graph, 2 partitions) through the reference CPU
   micrograph trainer (gnnsim.engine.run_strategy) with the CUDA backend:
   ledger, metrics and trained parameters identical to the numba backend.

Needs baseline/_ref (baseline/install_ref.sh; travels with the snapshot).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
SUITE = os.path.join(REF, "gnnsim_tests")

if not os.path.isdir(os.path.join(REF, "gnnsim")):
    pytest.skip("baseline/_ref not installed (baseline/install_ref.sh)", allow_module_level=True)


@pytest.fixture(scope="module")
def gs():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gnnsim_numba_cache")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import gnnsim._kernels_nb as nb
    import gnnsim.kernels  # noqa: F401
    return nb


def test_operator_layer_matches_numba_backend(gs):
    from paper_2409_00657_b200 import kernels as K
    from paper_2409_00657_b200.graph import GraphSpec, generate
    nb = gs
    rng = np.random.default_rng(5)
    g = generate(GraphSpec(n=20000, avg_deg=20.0, beta=0.8, p_in=0.8, n_blocks=8, d_cap=5000,
                           seed=5))
    off, tgt = g.to_host()
    frontier = np.concatenate([np.argsort(-np.diff(off))[:30], rng.integers(0, 20000, 300)])
    for fo in (1, 4, 15, 40):
        st = int(rng.integers(0, 2 ** 63))
        a, b = K.sample_frontier(off, tgt, frontier, fo, st), nb.sample_frontier(off, tgt, frontier, fo, st)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    ids = np.unique(rng.integers(0, 10 ** 9, 5000))
    for k in (0, 1, 7, 100, 4999, 6000):
        st = int(rng.integers(0, 2 ** 63))
        assert np.array_equal(K.pick_k_smallest(ids, k, st), nb.pick_k_smallest(ids, k, st))
    assert np.array_equal(K.feature_rows(ids[:300], 37, 123), nb.feature_rows(ids[:300], 37, 123))
    block_of = np.sort(rng.integers(0, 5, 1500)).astype(np.int64)
    for modes in ((1, 2 ** 62, 1, 2 ** 58), (2, 0, 0, 0), (0, 0, 1, 2 ** 60), (1, 0, 2, 0)):
        st = int(rng.integers(0, 2 ** 63))
        us, vs = K.sbm_edges(block_of, *modes, st)
        ru, rv = nb.sbm_edges(block_of, modes[0], modes[1], modes[2], modes[3], st)
        assert np.array_equal(us, ru) and np.array_equal(vs, rv)


def test_reference_suite_on_cuda_backend():
    files = [os.path.join(SUITE, f) for f in ("test_kernels.py", "test_sampler.py",
                                              "test_graph.py", "test_featstore.py",
                                              "test_model.py", "test_engine.py")]
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REPO, "tests"), REPO, REF,
                                         env.get("PYTHONPATH", "")])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/gnnsim_numba_cache")
    # test_env_flag_selects_backend spawns a bare interpreter without PYTHONPATH
    # (it fails the same way on the reference's own backends); deselect it
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "gnnsim_cuda_plugin",
                        "-p", "no:cacheprovider", "-k", "not test_env_flag_selects_backend",
                        *files], capture_output=True, text=True, env=env, cwd="/tmp",
                       timeout=1800)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    line = [x for x in out.splitlines() if x.startswith("GNNSIM_CUDA_CALLS")]
    assert line, out[-2000:]
    calls = dict(kv.split("=") for kv in line[-1].split()[1:])
    assert int(calls.get("sample_frontier", 0)) > 1000, line
    assert int(calls.get("feature_rows", 0)) > 0 and int(calls.get("sbm_edges", 0)) > 0, line
    assert int(calls.get("pick_k_smallest", 0)) > 0, line


def _cfg1(path, strategy):
    from gnnsim.config import RunConfig
    return RunConfig(graph=path, servers=2, partitioner="hash", layers=2, fanout=(10, 5),
                     dim=128, hidden=128, classes=16, arch="sage-mean", lr=0.1, batch=1024,
                     epochs=1, iterations=2, strategy=strategy, seed=0)


def test_cfg1_reference_trainer_on_cuda_backend(gs, tmp_path):
    """cfg1 through gnnsim's own micrograph trainer, S = 2: CUDA backend == numba."""
    import gnnsim.engine as E
    import gnnsim.kernels as gk
    from paper_2409_00657_b200 import _kernels_cuda
    from paper_2409_00657_b200.graph import GraphSpec, generate, save_csr
    g = generate(GraphSpec(n=100_000, avg_deg=18.5, beta=0.8, p_in=0.9, n_blocks=8,
                           d_cap=1 << 14, seed=0))
    path = str(tmp_path / "cfg1.csr")
    save_csr(g, path)
    saved = {n: getattr(gk, n) for n in ("sample_frontier", "feature_rows", "pick_k_smallest",
                                         "sbm_edges", "BACKEND")}
    res = {}
    for backend in ("numba", "cuda"):
        if backend == "cuda":
            _kernels_cuda.install(gk)
        try:
            res[backend] = {s: E.run_strategy(_cfg1(path, s))
                            for s in ("micrograph+pg", "model-centric")}
        finally:
            for n, f in saved.items():
                setattr(gk, n, f)
    for s in ("micrograph+pg", "model-centric"):
        a, b = res["numba"][s][0], res["cuda"][s][0]
        assert a.ledger.counters == b.ledger.counters
        assert a.bytes_by_category == b.bytes_by_category
        assert a.miss_rate == b.miss_rate and a.alpha == b.alpha and a.imbalance == b.imbalance
        assert all(np.array_equal(x, y) for it_a, it_b in zip(a.trained, b.trained)
                   for x, y in zip(it_a, it_b))
