"""Exact float64 GCN / SAGE-mean math of one micrograph (restates ``model.py``).

Arrays follow the reference layout: ``W_k`` is ``(in_k, H)`` with
``in_k = 2*prev`` for SAGE (model.py:69-84), biases are zero-initialised,
the classifier has no bias, ReLU is applied after every GNN layer including
the last (model.py:242-246).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .rng import chain, keyed, unit_f64

GCN = "gcn"
SAGE = "sage-mean"
BYTES_PER_ELEM = 4


@dataclass
class Params:
    arch: str
    W: list
    b: list
    Wc: np.ndarray

    def arrays(self):
        return [*self.W, *self.b, self.Wc]

    @property
    def count(self) -> int:
        return sum(a.size for a in self.arrays())

    @property
    def nbytes_ref(self) -> int:
        """Transport size under the reference convention, 4 B/elem (model.py:53-56)."""
        return self.count * BYTES_PER_ELEM

    def copy(self) -> "Params":
        return Params(self.arch, [w.copy() for w in self.W], [x.copy() for x in self.b],
                      self.Wc.copy())

    def zeros(self) -> "Params":
        return Params(self.arch, [np.zeros_like(w) for w in self.W],
                      [np.zeros_like(x) for x in self.b], np.zeros_like(self.Wc))


def glorot(rows: int, cols: int, state: int) -> np.ndarray:
    """Keyed uniform(-a, a), a = sqrt(6/(rows+cols)), row-major (model.py:87-90)."""
    a = np.sqrt(6.0 / (rows + cols))
    u = unit_f64(keyed(state, np.arange(rows * cols, dtype=np.int64)))
    return ((2.0 * u - 1.0) * a).reshape(rows, cols)


def init_params(arch: str, dim: int, hidden: int, n_layers: int, n_classes: int,
                seed: int) -> Params:
    """Deterministic init keyed on (seed, 0x11, k) / (seed, 0x12) (model.py:69-84)."""
    W, b = [], []
    width = dim
    for k in range(n_layers):
        fan_in = 2 * width if arch == SAGE else width
        W.append(glorot(fan_in, hidden, chain(seed, 0x11, k)))
        b.append(np.zeros(hidden))
        width = hidden
    return Params(arch, W, b, glorot(width, n_classes, chain(seed, 0x12)))


def labels(ids, n_classes: int, seed: int) -> np.ndarray:
    """label(v) = chain(seed, 0x1A, v) mod C (model.py:93-109)."""
    h = keyed(chain(seed, 0x1A), np.asarray(ids, dtype=np.int64))
    return (h % np.uint64(n_classes)).astype(np.int64)


def build_plan(m):
    """need sets and per-layer (self_pos, dpos, spos, deg) (model.py:183-198)."""
    L = m.n_layers
    need = [None] * (L + 1)
    need[L] = m.layers[L]
    for k in range(L - 1, -1, -1):
        need[k] = np.union1d(m.layers[k], need[k + 1])
    steps = []
    for k in range(1, L + 1):
        dst_idx, src_idx = m.pairs[k - 1]
        self_pos = np.searchsorted(need[k - 1], need[k])
        dpos = np.searchsorted(need[k], m.layers[k][dst_idx])
        spos = np.searchsorted(need[k - 1], m.layers[k - 1][src_idx])
        deg = np.bincount(dpos, minlength=len(need[k])).astype(np.float64)
        steps.append((self_pos, dpos, spos, deg))
    return need, steps


def forward(m, x_rows, P: Params):
    """Layered forward of one micrograph; x_rows aligned with m.vertices (model.py:213-247)."""
    need, steps = build_plan(m)
    x = np.asarray(x_rows, dtype=np.float64)
    h = [x[np.searchsorted(m.vertices, need[0])]]
    aggs, zs = [], []
    for k, (self_pos, dpos, spos, deg) in enumerate(steps, start=1):
        prev = h[-1]
        s = np.zeros((len(need[k]), prev.shape[1]))
        np.add.at(s, dpos, prev[spos])
        own = prev[self_pos]
        if P.arch == GCN:
            agg = (s + own) / (deg + 1.0)[:, None]
        else:
            has = (deg > 0)[:, None]
            agg = np.concatenate([own, np.where(has, s / np.maximum(deg, 1.0)[:, None], own)], 1)
        z = agg @ P.W[k - 1] + P.b[k - 1]
        aggs.append(agg)
        zs.append(z)
        h.append(np.maximum(z, 0.0))
    logits = h[-1][0] @ P.Wc
    return dict(need=need, steps=steps, h=h, aggs=aggs, zs=zs, logits=logits)


def loss_and_grads(st, label: int, P: Params):
    """Softmax-CE on the root and unscaled gradients (model.py:250-287)."""
    lg = st["logits"]
    sh = lg - lg.max()
    e = np.exp(sh)
    loss = float(np.log(e.sum()) - sh[label])
    dl = e / e.sum()
    dl[label] -= 1.0
    G = P.zeros()
    L = len(P.W)
    G.Wc += np.outer(st["h"][L][0], dl)
    dh = np.zeros_like(st["h"][L])
    dh[0] = P.Wc @ dl
    for k in range(L, 0, -1):
        self_pos, dpos, spos, deg = st["steps"][k - 1]
        dz = dh * (st["zs"][k - 1] > 0.0)
        G.W[k - 1] += st["aggs"][k - 1].T @ dz
        G.b[k - 1] += dz.sum(0)
        dagg = dz @ P.W[k - 1].T
        prev = np.zeros_like(st["h"][k - 1])
        if P.arch == GCN:
            part = dagg / (deg + 1.0)[:, None]
            prev[self_pos] += part
            np.add.at(prev, spos, part[dpos])
        else:
            w = st["h"][k - 1].shape[1]
            has = deg > 0
            prev[self_pos] += dagg[:, :w]
            np.add.at(prev, spos, np.where(has[:, None], dagg[:, w:] / np.maximum(deg, 1.0)[:, None], 0.0)[dpos])
            prev[self_pos] += np.where(has[:, None], 0.0, dagg[:, w:])
        dh = prev
    return loss, G


def add_into(acc: Params, g: Params) -> None:
    for a, b in zip(acc.arrays(), g.arrays()):
        a += b


def sgd_step(P: Params, acc_sum: Params, batch_total: int, lr: float) -> None:
    """theta -= lr * sum(acc)/batch_total (model.py:299-324)."""
    scale = 1.0 / batch_total if batch_total > 0 else 1.0
    for p, g in zip(P.arrays(), acc_sum.arrays()):
        p -= lr * (g * scale)


def ring_allreduce_bytes(n: int, param_bytes: int) -> float:
    """Per-link charge of the reference ring all-reduce (model.py:325-328)."""
    return 2.0 * (n - 1) / n * param_bytes
