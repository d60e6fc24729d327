"""Multi-GPU micrograph strategy (NCCL) against the oracle engine, which is
pinned to gnnsim's ledgers and parameters (tests/test_oracle_golden.py).
Needs >= 2 GPUs (run with `gpurun --gpus 2`); skipped otherwise.
feat "pg": dedup staging over NCCL all-to-all; "peer": rows read in place
from the owner GPU over NVLink (CUDA IPC) -- both charge the reference ledger."""
import json
import os
import tempfile

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _world():
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    return min(n, 4)


@pytest.mark.parametrize("mode,dtype,feat", [("fused", "f32", "pg"), ("faithful", "f32", "pg"),
                                             ("fused", "bf16", "pg"), ("fused", "f32", "peer"),
                                             ("faithful", "f32", "peer"),
                                             ("fused", "bf16", "peer")])
def test_micrograph_strategy_matches_oracle(mode, dtype, feat):
    import dist_helpers
    world = _world()
    d = tempfile.mkdtemp()
    mp.spawn(dist_helpers.micrograph_worker,
             args=(world, os.path.join(d, "init"), os.path.join(d, "res"), mode, dtype, feat),
             nprocs=world, join=True)
    res = json.load(open(os.path.join(d, "res.0")))
    assert res["ok"], res["msg"]


@pytest.mark.parametrize("feat", ["pg", "peer"])
def test_model_centric_matches_oracle(feat):
    """Model-centric baseline (engine.py:482-507) on the GPUs: ledger exact."""
    import dist_helpers
    world = _world()
    d = tempfile.mkdtemp()
    mp.spawn(dist_helpers.micrograph_worker,
             args=(world, os.path.join(d, "init"), os.path.join(d, "res"), "fused", "f32", feat,
                   "model-centric"),
             nprocs=world, join=True)
    res = json.load(open(os.path.join(d, "res.0")))
    assert res["ok"], res["msg"]


@pytest.mark.parametrize("feat", ["pg", "peer"])
def test_merge_controller_matches_oracle(feat):
    """Merging controller (engine.py:773-833) with a forced-acceptance cost:
    decisions, merged trace tables, ledger and parameters equal the oracle's."""
    import dist_helpers
    world = _world()
    d = tempfile.mkdtemp()
    mp.spawn(dist_helpers.merge_worker,
             args=(world, os.path.join(d, "init"), os.path.join(d, "res"), feat),
             nprocs=world, join=True)
    res = json.load(open(os.path.join(d, "res.0")))
    assert res["ok"], res["msg"]


@pytest.mark.parametrize("strategy", ["micrograph", "model-centric"])
def test_graph_loop_matches_oracle(strategy):
    """Enough iterations for the CUDA-graph loop (DistGraphLoop) to engage:
    device root counts, cursor-staged roots, cursor-indexed ledger rows."""
    import dist_helpers
    world = _world()
    d = tempfile.mkdtemp()
    mp.spawn(dist_helpers.micrograph_worker,
             args=(world, os.path.join(d, "init"), os.path.join(d, "res"), "fused", "f32", "peer",
                   strategy, 7),
             nprocs=world, join=True)
    res = json.load(open(os.path.join(d, "res.0")))
    assert res["ok"], res["msg"]
    assert res["graph_used"], "graph loop never engaged"


@pytest.mark.parametrize("strategy", ["micrograph", "model-centric"])
def test_group_loop_matches_oracle(strategy):
    """DistGroupLoop (2 iterations per replay): grouped builds with per-batch
    device root counts, per-iteration pre-gathers and ledger rows, the exit
    path that trains the already pre-gathered group -- ledger and parameters
    equal the oracle's."""
    import dist_helpers
    world = _world()
    d = tempfile.mkdtemp()
    mp.spawn(dist_helpers.micrograph_worker,
             args=(world, os.path.join(d, "init"), os.path.join(d, "res"), "fused", "f32", "peer",
                   strategy, 9, 2),
             nprocs=world, join=True)
    res = json.load(open(os.path.join(d, "res.0")))
    assert res["ok"], res["msg"]
    assert res["graph_used"], "group loop never engaged"


@pytest.mark.parametrize("strategy,csr", [("micrograph", "sharded-hash"),
                                          ("micrograph", "sharded-blocks"),
                                          ("model-centric", "sharded-hash")])
def test_sharded_csr_matches_oracle(strategy, csr):
    """Partitioned CSR (north_star): every rank holds only its homed rows and
    reads peers' rows over NVLink inside the builds; grouped graph loop
    engaged.  Ledger and parameters equal the oracle's."""
    import dist_helpers
    world = _world()
    d = tempfile.mkdtemp()
    mp.spawn(dist_helpers.micrograph_worker,
             args=(world, os.path.join(d, "init"), os.path.join(d, "res"), "fused", "f32", "peer",
                   strategy, 9, 2, csr),
             nprocs=world, join=True)
    res = json.load(open(os.path.join(d, "res.0")))
    assert res["ok"], res["msg"]
    assert res["graph_used"], "group loop never engaged"


@pytest.mark.parametrize("allreduce", ["p2p", "nccl"])
def test_allreduce_paths_match_oracle(allreduce):
    """Gradient all-reduce over NVLink peer memory (hg_p2p_allreduce: push,
    signal, wait, reduce; the default) and over NCCL, both inside the grouped
    graph loop: parameters and ledger equal the oracle's."""
    import dist_helpers
    world = _world()
    d = tempfile.mkdtemp()
    mp.spawn(dist_helpers.micrograph_worker,
             args=(world, os.path.join(d, "init"), os.path.join(d, "res"), "fused", "f32", "peer",
                   "micrograph", 9, 2, "sharded-blocks", allreduce),
             nprocs=world, join=True)
    res = json.load(open(os.path.join(d, "res.0")))
    assert res["ok"], res["msg"]
    assert res["graph_used"], "group loop never engaged"
