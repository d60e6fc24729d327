"""Host-side logic of the multi-GPU path on CPU: trace table / merge replay
against the oracle, reference ledger accounting, and the pre-gather
all-to-all exchange run for real with world_size 2, 3 and 8 (the driver's largest N) over gloo."""
import os
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import engine as OE


def test_trace_table_matches_oracle():
    from paper_2409_00657_b200 import distributed as D
    rng = np.random.default_rng(3)
    for S in (2, 3, 4, 8):
        home = rng.integers(0, S, 400)
        batches = [rng.choice(400, 40, replace=False) for _ in range(S)]
        groups = [tuple(b[home[b] == s] for s in range(S)) for b in batches]
        tt = D.TraceTable.initial(S)
        assert np.array_equal(tt.server_of, OE.initial_table(S))
        cells = D.assign_cell_roots(tt, groups, 11)
        tt.root_counts = D.cell_counts(cells)
        tt.validate()
        removed, sv, cnt = (), OE.initial_table(S), tt.root_counts
        for _ in range(S - 1):
            col = D.find_fewest_column(tt)
            assert col == OE.fewest_column(cnt)
            tt = D.delete_column_and_redistribute(tt, col)
            sv, cnt = OE.delete_column(sv, cnt, col)
            removed = removed + (col,)
            assert np.array_equal(tt.root_counts, cnt) and np.array_equal(tt.server_of, sv)
            got = D.assign_cell_roots(tt, groups, 11)
            want = OE.assign_cells(groups, removed, 11)
            for a, b in zip(got, want):
                for x, y in zip(a, b):
                    assert np.array_equal(x, y)
            for d in range(S):  # membership conserved (test_engine.py:145-158)
                assert np.array_equal(np.sort(np.concatenate(got[d])), np.sort(batches[d]))
        assert D.find_fewest_column(tt) is None


def test_ledger_semantics():
    from paper_2409_00657_b200.errors import InvariantViolation
    from paper_2409_00657_b200.featstore import FEATURE, CommLedger
    led = CommLedger()
    led.add(1, 0, FEATURE, 400.0, 1)
    led.add(1, 0, FEATURE, 100.0, 1)
    assert led.link(1, 0, FEATURE) == (500.0, 2)
    with pytest.raises(InvariantViolation):
        led.add(2, 2, FEATURE, 1.0)
    with pytest.raises(ValueError):
        led.add(0, 1, "bogus", 1.0)
    other = CommLedger()
    other.add(0, 1, FEATURE, 8.0, 1)
    led.merge(other)
    assert led.bytes_by_category()[FEATURE] == 508.0
    assert sum(e[3] for e in led.events) == led.total_bytes()


def test_plan_pregather_matches_oracle():
    from paper_2409_00657_b200.featstore import plan_pregather
    rng = np.random.default_rng(0)
    home = rng.integers(0, 4, 300)
    sets = [rng.integers(0, 300, 30) for _ in range(5)]
    got = plan_pregather(2, sets, home)
    want = OE.pregather_plan(2, sets, home)
    assert [(h, ids.tolist()) for h, ids in got.by_source] == [(h, ids.tolist()) for h, ids in want]


@pytest.mark.parametrize("world", [2, 3, 8])
def test_pregather_all_to_all_gloo(world):
    import dist_helpers
    d = tempfile.mkdtemp()
    init = os.path.join(d, "init")
    res = os.path.join(d, "res")
    mp.spawn(dist_helpers.pregather_worker, args=(world, init, res), nprocs=world, join=True)
    for r in range(world):
        assert open(f"{res}.{r}").read() == "ok"
