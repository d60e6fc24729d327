"""Multi-GPU micrograph strategy (NCCL) against the oracle engine, which is
pinned to gnnsim's ledgers and parameters (tests/test_oracle_golden.py).
Needs >= 2 GPUs (run with `gpurun --gpus 2`); skipped otherwise."""
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


@pytest.mark.parametrize("mode,dtype", [("fused", "f32"), ("faithful", "f32"), ("fused", "bf16")])
def test_micrograph_strategy_matches_oracle(mode, dtype):
    import dist_helpers
    world = _world()
    d = tempfile.mkdtemp()
    mp.spawn(dist_helpers.micrograph_worker,
             args=(world, os.path.join(d, "init"), os.path.join(d, "res"), mode, dtype),
             nprocs=world, join=True)
    res = json.load(open(os.path.join(d, "res.0")))
    assert res["ok"], res["msg"]
