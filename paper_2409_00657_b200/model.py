"""GNN parameters on the device and the batched training step.

Drop-in counterpart of reference ``gnnsim.model``: ``ModelState`` /
``init_model`` (model.py:26-90), ``LabelOracle`` (model.py:93-109),
``sync_and_update`` semantics (model.py:299-329).  The per-micrograph
float64 loops of ``forward`` / ``loss_and_backward`` become one
``hg_train_step`` launch sequence over a whole cell of roots
(csrc/hg_dense.cu).

Parameter layout: one flat fp32 buffer (master weights) holding, in order,
W_1..W_L, b_1..b_L, W_c.  W_1 is stored with padded rows when the feature
width D is padded to Dp (16-byte rows): SAGE rows [0,D) = self half,
[Dp, Dp+D) = neighbour half, padding rows are zero and stay zero (their
gradient is agg-padding(=0) x dz).  ``reference_arrays()`` returns the
reference's unpadded float64 arrays.  A bf16 shadow of the flat buffer is
refreshed by every update when activations run in bf16.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .rng import chain, hash_vec

GCN = "gcn"
SAGE_MEAN = "sage-mean"
ARCHS = (GCN, SAGE_MEAN)
BYTES_PER_ELEM = 4  # reference transport convention (featstore.py:20, model.py:53-56)


def pad8(x: int) -> int:
    return (x + 7) // 8 * 8


def glorot_device(rows: int, cols: int, state: int, dtype=torch.float64, device="cuda"):
    """Keyed Glorot uniform, bit-identical to model.py:87-90 in float64."""
    out = torch.empty((rows, cols), dtype=dtype, device=device)
    code = 0 if dtype == torch.float64 else 1
    _lib.call("hg_glorot", rows, cols, state & ((1 << 64) - 1), code, out.data_ptr(),
              torch.cuda.current_stream(out.device).cuda_stream)
    return out


class ModelState:
    """Device parameters of a small GCN / SAGE-mean GNN plus its gradient
    accumulator (the reference keeps them in ModelState + GradAccumulator)."""

    def __init__(self, arch: str, feat_dim: int, hidden: int, n_layers: int, n_classes: int,
                 device="cuda", feat_ld: int = None):
        if arch not in ARCHS:
            raise ValueError(f"unknown arch {arch!r}")
        if n_classes < 2:
            raise ValueError("need at least 2 classes")
        if hidden % 8:
            raise ValueError("hidden must be a multiple of 8 on the device")
        self.arch, self.D, self.H, self.L, self.C = arch, feat_dim, hidden, n_layers, n_classes
        self.Dp = feat_ld or pad8(feat_dim)
        self.device = torch.device(device)
        sage = arch == SAGE_MEAN
        self.in_dim = [0] * (n_layers + 1)
        self.in_ref = [0] * (n_layers + 1)
        for k in range(1, n_layers + 1):
            w = self.Dp if k == 1 else hidden
            wr = feat_dim if k == 1 else hidden
            self.in_dim[k] = 2 * w if sage else w
            self.in_ref[k] = 2 * wr if sage else wr
        shapes = [(self.in_dim[k], hidden) for k in range(1, n_layers + 1)]
        shapes += [(hidden,)] * n_layers + [(hidden, n_classes)]
        self.shapes = shapes
        sizes = [int(np.prod(s)) for s in shapes]
        self.offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        n = int(self.offsets[-1])
        self.flat = torch.zeros(n, dtype=torch.float32, device=self.device)
        self.grad = torch.zeros(n, dtype=torch.float32, device=self.device)
        self.shadow = torch.zeros(n, dtype=torch.bfloat16, device=self.device)

    # views ------------------------------------------------------------
    def _view(self, buf, i):
        return buf[self.offsets[i]:self.offsets[i + 1]].view(*self.shapes[i])

    def W(self, k, buf=None):
        return self._view(self.flat if buf is None else buf, k - 1)

    def b(self, k, buf=None):
        return self._view(self.flat if buf is None else buf, self.L + k - 1)

    def Wc(self, buf=None):
        return self._view(self.flat if buf is None else buf, 2 * self.L)

    @property
    def n_layers(self) -> int:
        return self.L

    @property
    def n_classes(self) -> int:
        return self.C

    @property
    def param_count(self) -> int:
        """Reference parameter count (unpadded), model.py:49-51."""
        return (sum(self.in_ref[k] * self.H for k in range(1, self.L + 1)) + self.L * self.H
                + self.H * self.C)

    @property
    def param_bytes(self) -> int:
        return self.param_count * BYTES_PER_ELEM

    def _ref_rows(self, k):
        """Indices of the padded W_k rows that hold reference rows."""
        if k != 1 or self.Dp == self.D:
            return np.arange(self.in_ref[k])
        if self.arch == SAGE_MEAN:
            return np.concatenate([np.arange(self.D), self.Dp + np.arange(self.D)])
        return np.arange(self.D)

    def load_reference(self, weights, biases, classifier, buf=None) -> None:
        """Set parameters (or, buf=self.grad, the accumulator) from
        reference-layout arrays (float64 ok)."""
        dst = self.flat if buf is None else buf
        dst.zero_()
        for k in range(1, self.L + 1):
            w = torch.as_tensor(np.asarray(weights[k - 1]), dtype=torch.float32)
            self.W(k, dst)[torch.as_tensor(self._ref_rows(k))] = w.to(self.device)
            self.b(k, dst).copy_(torch.as_tensor(np.asarray(biases[k - 1]), dtype=torch.float32))
        self.Wc(dst).copy_(torch.as_tensor(np.asarray(classifier), dtype=torch.float32))
        if buf is None:
            self.refresh_shadow()

    def reference_arrays(self, buf=None):
        """(weights, biases, classifier) as float64 numpy in reference layout."""
        buf = self.flat if buf is None else buf
        ws = [self.W(k, buf).cpu().numpy()[self._ref_rows(k)].astype(np.float64)
              for k in range(1, self.L + 1)]
        bs = [self.b(k, buf).cpu().numpy().astype(np.float64) for k in range(1, self.L + 1)]
        return ws, bs, self.Wc(buf).cpu().numpy().astype(np.float64)

    def params(self):
        w, b, c = self.reference_arrays()
        return [*w, *b, c]

    def grads(self):
        w, b, c = self.reference_arrays(self.grad)
        return [*w, *b, c]

    def refresh_shadow(self) -> None:
        self.shadow.copy_(self.flat.to(torch.bfloat16))

    def sgd(self, lr: float, batch_total: int, stream=None) -> None:
        """theta -= lr * acc / batch_total; acc = 0 (model.py:315-324)."""
        inv = 1.0 / batch_total if batch_total > 0 else 1.0
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        _lib.call("hg_sgd_update", self.flat.data_ptr(), self.grad.data_ptr(), None,
                  self.flat.numel(), float(lr), float(inv), s)


def init_model(arch: str, feat_dim: int, hidden: int, n_layers: int, n_classes: int,
               seed: int, device="cuda", feat_ld: int = None) -> ModelState:
    """Deterministic Glorot init keyed on (seed, 0x11, k) / (seed, 0x12) (model.py:69-84)."""
    m = ModelState(arch, feat_dim, hidden, n_layers, n_classes, device, feat_ld)
    ws = []
    width = feat_dim
    for k in range(n_layers):
        rows = 2 * width if arch == SAGE_MEAN else width
        ws.append(glorot_device(rows, hidden, chain(seed, 0x11, k), device=device).cpu().numpy())
        width = hidden
    wc = glorot_device(width, n_classes, chain(seed, 0x12), device=device).cpu().numpy()
    m.load_reference(ws, [np.zeros(hidden)] * n_layers, wc)
    return m


@dataclass(frozen=True)
class LabelOracle:
    """label(v) = chain(seed, 0x1A, v) mod C (model.py:93-109)."""

    n_classes: int
    seed: int

    def __post_init__(self):
        if self.n_classes < 2:
            raise ValueError("need at least 2 classes")

    @property
    def state(self) -> int:
        return chain(self.seed, 0x1A)

    def labels(self, ids) -> np.ndarray:
        h = hash_vec(self.state, np.asarray(ids, dtype=np.int64))
        return (h % np.uint64(self.n_classes)).astype(np.int64)

    def label(self, v: int) -> int:
        return int(self.labels(np.array([v]))[0])


StepDesc = _lib.StepDesc
