"""Micrograph sampling and root regrouping (restates reference ``sampler.py``).

A micrograph is the per-root computation graph: ``layers[L] = [root]`` and
hop ``h = L - k`` samples ``fanout[h-1]`` neighbours of every vertex of
``layers[k+1]`` into ``layers[k]`` (sampler.py:84-106).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import kernels
from .rng import chain


def stream_key(seed: int, epoch: int, iteration: int, root: int) -> int:
    """Per-root draw key (sampler.py:52-54)."""
    return chain(seed, epoch, iteration, root)


@dataclass(frozen=True)
class Micro:
    """Same fields as the reference ``Micrograph`` (sampler.py:57-81)."""

    root: int
    layers: tuple
    pairs: tuple
    vertices: np.ndarray

    @property
    def n_layers(self) -> int:
        return len(self.layers) - 1

    @property
    def vertex_count(self) -> int:
        return len(self.vertices)


def sample_micrograph(offsets, targets, root: int, fanout: Sequence[int],
                      key: int, draw: Callable = None) -> Micro:
    """Node-wise k-hop sampling of one root (sampler.py:84-106).

    ``draw`` defaults to the numpy frontier kernel; the CPU baseline passes
    the numba port.  Layers are sorted-unique; pairs are (frontier index,
    searchsorted position) exactly like the reference.
    """
    draw = draw or kernels.sample_frontier
    n = len(offsets) - 1
    if not 0 <= root < n:
        raise ValueError(f"root {root} out of range for {n} vertices")
    L = len(fanout)
    layers = [None] * (L + 1)
    pairs = [None] * L
    layers[L] = np.array([root], dtype=np.int64)
    for k in range(L - 1, -1, -1):
        hop = L - k
        front = layers[k + 1]
        counts, flat = draw(offsets, targets, front, fanout[hop - 1], chain(key, hop))
        layers[k] = np.unique(flat)
        dst = np.repeat(np.arange(len(front), dtype=np.int64), counts)
        pairs[k] = (dst, np.searchsorted(layers[k], flat).astype(np.int64))
    vertices = np.unique(np.concatenate(layers))
    return Micro(int(root), tuple(layers), tuple(pairs), vertices)


def redistribute_roots(batches, home: np.ndarray, n_servers: int):
    """groups[d][s] = roots of batch d homed at s, order kept (sampler.py:168-177)."""
    out = []
    for b in batches:
        b = np.asarray(b, dtype=np.int64)
        h = home[b]
        out.append(tuple(b[h == s] for s in range(n_servers)))
    return tuple(out)


def load_imbalance(groups, n_servers: int) -> float:
    """(max - min) / mean of per-server totals (sampler.py:180-186)."""
    tot = np.zeros(n_servers, dtype=np.int64)
    for per_model in groups:
        for s, r in enumerate(per_model):
            tot[s] += len(r)
    mean = tot.mean() if len(tot) else 0.0
    return 0.0 if mean == 0 else float((tot.max() - tot.min()) / mean)
