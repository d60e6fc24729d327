"""Merging controller decision logic (engine.py:773-833) on CPU: the epoch
runner and the next-epoch probe are stubbed, the controller itself is the
product code.  Mirrors gnnsim's test_merge_controller_* (test_engine.py:326-360);
the GPU run against the oracle is tests/test_distributed_gpu.py."""
import numpy as np
import pytest

from paper_2409_00657_b200 import distributed as D


class _Stub:
    strategy = "micrograph"

    def __init__(self, S):
        self.S = S
        self.table = None
        self.epochs = []


@pytest.fixture
def stubbed(monkeypatch):
    def run_epoch(trainer, epoch):
        trainer.table.validate()
        trainer.epochs.append((epoch, trainer.table.n_columns))
        return 1.0

    def counts(trainer, tt, epoch):
        rng = np.random.default_rng(epoch)
        return rng.integers(0, 20, size=tt.server_of.shape).astype(np.int64)

    monkeypatch.setattr(D, "run_epoch", run_epoch)
    monkeypatch.setattr(D, "counts_for_next_epoch", counts)


def test_equal_cost_keeps_all_columns(stubbed):
    tr = _Stub(4)
    tt, hist, times = D.merge_controller(tr, epochs=4, merge_k=1,
                                         cost=lambda table, sec: 0.0)
    assert tt.n_columns == 4
    assert [h.action for h in hist] == ["baseline", "rejected", "settled"]
    assert len(times) == 4


def test_sync_dominated_reaches_one_column(stubbed):
    tr = _Stub(4)
    tt, hist, _ = D.merge_controller(tr, epochs=8, merge_k=1,
                                     cost=lambda table, sec: 100.0 * table.n_columns)
    assert tt.n_columns == 1
    cols = [c for _, c in tr.epochs]
    assert cols == sorted(cols, reverse=True)
    accepted = [h.avg_seconds for h in hist if h.action in ("baseline", "accepted")]
    assert accepted == sorted(accepted, reverse=True)
    tt.validate()
    assert len(tt.removed) == 3


def test_rejected_drop_is_reverted(stubbed):
    tr = _Stub(3)
    tt, hist, _ = D.merge_controller(tr, epochs=6, merge_k=2,
                                     cost=lambda table, sec: float(10 - table.n_columns))
    assert tt.n_columns == 3 and tt.removed == ()
    assert [h.action for h in hist] == ["baseline", "rejected", "settled"]
    assert [c for _, c in tr.epochs] == [3, 3, 2, 2, 3, 3]


def test_model_centric_refuses_merging():
    tr = _Stub(2)
    tr.strategy = "model-centric"
    with pytest.raises(ValueError):
        D.merge_controller(tr, epochs=2, merge_k=1)
