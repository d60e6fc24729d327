"""CPU restatement of the reference kernel boundary ``gnnsim.kernels``.

Reference: ``kernels.py:31-34`` re-exports ``sample_frontier``,
``feature_rows`` and ``pick_k_smallest`` from ``_kernels_np.py`` /
``_kernels_nb.py``.  This file restates them twice:

* plain numpy (``sample_frontier``, ``feature_rows``, ``pick_k_smallest``):
  the checker used by the tests;
* numba (``*_nb``): the fast scalar port the CPU baseline leg of
  ``bench.py`` times, the analogue of the reference's default numba backend.

Selection rule (``_kernels_np.py:55-84``, ``_kernels_nb.py:55-86``): a
frontier vertex with degree <= fanout keeps all neighbours in CSR order;
otherwise slot j gets the key ``(mix64(mix64(state ^ v) ^ j) & HI32) | j``
and the ``fanout`` smallest keys win, emitted in ascending slot order.
"""
from __future__ import annotations

import numpy as np

from .rng import U64, keyed, mix64, mix64_array

HI32 = U64(0xFFFFFFFF00000000)


def slot_keys(state: int, v: int, deg: int) -> np.ndarray:
    """Selection keys of the deg slots of vertex v (_kernels_nb.py:77-80)."""
    hv = mix64(int(state) ^ int(v))
    slots = np.arange(deg, dtype=np.uint64)
    return (mix64_array(slots ^ U64(hv)) & HI32) | slots


def draw_slots(state: int, v: int, deg: int, fanout: int) -> np.ndarray:
    """Chosen slot indices of one frontier vertex, ascending."""
    if deg <= fanout:
        return np.arange(deg, dtype=np.int64)
    keys = slot_keys(state, v, deg)
    # keys are distinct (slot index in the low word), so "fanout smallest"
    # is well defined without a tie rule.
    cut = np.partition(keys, fanout - 1)[fanout - 1]
    return np.flatnonzero(keys <= cut).astype(np.int64)


def sample_frontier(offsets, targets, frontier, fanout: int, state: int):
    """(counts, flat) for a frontier (_kernels_np.py:55-84)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    targets = np.asarray(targets)
    frontier = np.asarray(frontier, dtype=np.int64)
    counts = np.zeros(len(frontier), dtype=np.int64)
    pieces = []
    for i, v in enumerate(frontier.tolist()):
        lo, hi = int(offsets[v]), int(offsets[v + 1])
        chosen = draw_slots(state, v, hi - lo, fanout)
        counts[i] = len(chosen)
        pieces.append(targets[lo + chosen].astype(np.int64))
    flat = np.concatenate(pieces) if pieces else np.empty(0, dtype=np.int64)
    return counts, flat


def pick_k_smallest(ids, k: int, state: int) -> np.ndarray:
    """Layer-wise shared draw (_kernels_np.py:87-98)."""
    ids = np.asarray(ids, dtype=np.int64)
    if k >= len(ids):
        return ids.copy()
    ranks = np.arange(len(ids), dtype=np.uint64)
    keys = (keyed(state, ids) & HI32) | ranks
    cut = np.partition(keys, k - 1)[k - 1]
    return ids[keys <= cut]


def feature_rows(ids, dim: int, state: int) -> np.ndarray:
    """f32 rows in [-0.5, 0.5) on a 2^-24 grid (_kernels_np.py:101-106)."""
    ids = np.asarray(ids, dtype=np.int64)
    row_key = keyed(state, ids)
    cols = np.arange(dim, dtype=np.uint64)
    h = mix64_array(row_key[:, None] ^ cols[None, :])
    top24 = (h >> U64(40)).astype(np.float64)
    return (top24 * (2.0 ** -24) - 0.5).astype(np.float32)


# ----------------------------------------------------------------------------
# numba port (CPU baseline only)
# ----------------------------------------------------------------------------
try:  # pragma: no cover - exercised by bench.py when numba is importable
    import numba as _nb

    _I = np.uint64(0x9E3779B97F4A7C15)
    _A = np.uint64(0xBF58476D1CE4E5B9)
    _B = np.uint64(0x94D049BB133111EB)
    _H = np.uint64(0xFFFFFFFF00000000)

    @_nb.njit(cache=False, inline="always")
    def _mix_nb(x):
        z = x + _I
        z = (z ^ (z >> np.uint64(30))) * _A
        z = (z ^ (z >> np.uint64(27))) * _B
        return z ^ (z >> np.uint64(31))

    @_nb.njit(cache=False)
    def _frontier_nb(offsets, targets, frontier, fanout, state):
        f = frontier.shape[0]
        counts = np.empty(f, dtype=np.int64)
        total = 0
        for i in range(f):
            d = offsets[frontier[i] + 1] - offsets[frontier[i]]
            counts[i] = d if d <= fanout else fanout
            total += counts[i]
        flat = np.empty(total, dtype=np.int64)
        pos = 0
        for i in range(f):
            v = frontier[i]
            lo = offsets[v]
            d = offsets[v + 1] - lo
            if d <= fanout:
                for j in range(d):
                    flat[pos + j] = targets[lo + j]
                pos += d
                continue
            hv = _mix_nb(state ^ np.uint64(v))
            keys = np.empty(d, dtype=np.uint64)
            for j in range(d):
                keys[j] = (_mix_nb(hv ^ np.uint64(j)) & _H) | np.uint64(j)
            cut = np.sort(keys)[fanout - 1]
            for j in range(d):
                if keys[j] <= cut:
                    flat[pos] = targets[lo + j]
                    pos += 1
        return counts, flat

    def sample_frontier_nb(offsets, targets, frontier, fanout, state):
        return _frontier_nb(np.asarray(offsets, dtype=np.int64),
                            np.asarray(targets, dtype=np.int64),
                            np.asarray(frontier, dtype=np.int64),
                            int(fanout), np.uint64(int(state)))

    HAVE_NUMBA = True
except ImportError:  # pragma: no cover
    HAVE_NUMBA = False
    sample_frontier_nb = sample_frontier
