"""Host-side scalar key folding (reference rng.py:21-42).

Only scalar keys (seeds, per-iteration states) are folded on the host; every
per-element hash runs on the device (csrc/hg_common.cuh).  ``hash_vec`` is a
small numpy helper for host-side partition tables.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


def mix64(x: int) -> int:
    z = (int(x) + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def chain(*words: int) -> int:
    h = 0
    for w in words:
        h = mix64(h ^ (int(w) & MASK64))
    return h


hash_u64 = chain


def hash_vec(state: int, values) -> np.ndarray:
    z = np.asarray(values).astype(np.uint64) ^ np.uint64(int(state) & MASK64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z
