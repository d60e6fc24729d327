"""Expected pre-gather outcome (restates featstore.py:226-279) — test checker."""
import numpy as np

from .engine import pregather_plan
from .kernels import feature_rows


def pregather_expect(at, vertex_sets, home, n_servers, dim, fstate):
    """(rows per home, requested ids in home-then-id order, their feature rows)."""
    plan = pregather_plan(at, [np.asarray(v, dtype=np.int64) for v in vertex_sets], home)
    counts = np.zeros(n_servers, dtype=np.int64)
    ids = []
    for h, group in plan:
        counts[h] = len(group)
        ids.append(group)
    ids = np.concatenate(ids) if ids else np.empty(0, dtype=np.int64)
    rows = feature_rows(ids, dim, fstate) if len(ids) else np.zeros((0, dim), np.float32)
    return counts, ids, rows
