"""Per-micrograph model API of the reference, on the GPU.

gnnsim's ``model`` module trains one micrograph at a time (model.py:112-329):
``build_plan`` -> ``forward`` -> ``loss_and_backward`` -> ``accumulate`` ->
``sync_and_update``.  The batched hot path (``CellRunner`` / the trainers)
replaces those loops; this module keeps the per-micrograph names and
semantics for callers that drive them directly: a host ``Micrograph``
(sampler.py:57-81) and its feature rows are uploaded as a one-root batch
(the same device layout ``hg_mg_build`` writes) and run through the same
``hg_forward`` / ``hg_train_step`` kernels; ``sync_and_update`` applies the
summed accumulators with the device SGD (``hg_sgd_update``).  Results are
the reference's within the fp32 tolerance of the step (1e-3 relative).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InvariantViolation
from .featstore import GRADIENT, CommLedger, FeatureTable
from .model import LabelOracle, ModelState


@dataclass
class MicroPlan:
    """need sets and (self_pos, dpos, spos, deg) per layer (model.py:167-180)."""

    need: list
    layers: list


def build_plan(micro) -> MicroPlan:
    """model.py:183-198 (host index arithmetic over one micrograph)."""
    L = micro.n_layers
    need = [None] * (L + 1)
    need[L] = np.asarray(micro.layers[L], dtype=np.int64)
    for k in range(L - 1, -1, -1):
        need[k] = np.union1d(micro.layers[k], need[k + 1]).astype(np.int64)
    layers = []
    for k in range(1, L + 1):
        dst_idx, src_idx = micro.pairs[k - 1]
        self_pos = np.searchsorted(need[k - 1], need[k])
        dpos = np.searchsorted(need[k], np.asarray(micro.layers[k])[dst_idx])
        spos = np.searchsorted(need[k - 1], np.asarray(micro.layers[k - 1])[src_idx])
        deg = np.bincount(dpos, minlength=len(need[k])).astype(np.float64)
        layers.append((self_pos, dpos, spos, deg))
    return MicroPlan(need, layers)


class Gradients:
    """Parameter-shaped gradient triple in the reference layout (model.py:112-141)."""

    def __init__(self, weights, biases, classifier):
        self.weights, self.biases, self.classifier = list(weights), list(biases), classifier

    @classmethod
    def zeros_like(cls, model: ModelState) -> "Gradients":
        w, b, c = model.reference_arrays()
        return cls([np.zeros_like(x) for x in w], [np.zeros_like(x) for x in b],
                   np.zeros_like(c))

    def arrays(self):
        return [*self.weights, *self.biases, self.classifier]

    def add(self, other: "Gradients") -> None:
        for a, b in zip(self.arrays(), other.arrays()):
            if a.shape != b.shape:
                raise ValueError("gradient shape mismatch")
            a += b

    def scaled(self, factor: float) -> "Gradients":
        return Gradients([w * factor for w in self.weights], [b * factor for b in self.biases],
                         self.classifier * factor)

    def max_abs(self) -> float:
        return max(float(np.abs(a).max()) if a.size else 0.0 for a in self.arrays())


@dataclass
class GradAccumulator:
    """Running gradient sum of one logical model (model.py:144-158)."""

    model_id: int
    grads: Gradients
    count: int = 0

    @classmethod
    def for_model(cls, model_id: int, model: ModelState) -> "GradAccumulator":
        return cls(model_id, Gradients.zeros_like(model))

    def reset(self) -> None:
        for a in self.grads.arrays():
            a[:] = 0.0
        self.count = 0


def accumulate(acc: GradAccumulator, g: Gradients) -> None:
    """model.py:161-164."""
    acc.grads.add(g)
    acc.count += 1


class _OneRoot:
    """A host micrograph as a one-root device batch (hg_mg_batch layout)."""

    def __init__(self, micro, features, model: ModelState):
        from .trainer import CellRunner
        L = micro.n_layers
        if L != model.L:
            raise ValueError("micrograph depth differs from the model's layer count")
        feats = np.asarray(features, dtype=np.float32)
        if feats.shape[0] != micro.vertex_count:
            raise ValueError("need one feature row per micrograph vertex")
        plan = build_plan(micro)
        self.plan = plan
        verts = np.asarray(micro.vertices, dtype=np.int64)
        # fanout bound per hop that makes the builder layout hold this micrograph
        fo = []
        for hop in range(1, L + 1):
            k = L - hop
            d = np.bincount(micro.pairs[k][0], minlength=max(1, len(micro.layers[k + 1])))
            fo.append(max(1, int(d.max()) if d.size else 1))
        dev = model.device
        table = FeatureTable(max(len(verts), 1), model.D, torch.float32, dev, model.Dp)
        table.table[:len(verts), :model.D].copy_(torch.from_numpy(feats).to(dev))
        self.runner = CellRunner(None, table, model, tuple(fo), 1,
                                 LabelOracle(model.C, 0), use_tc=False)
        t = self.runner.builder.tensors
        i32 = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int32), device=dev)  # noqa: E731
        tot = [0] * (2 * L + 2)
        for k in range(L + 1):
            nk = len(plan.need[k])
            tot[k] = nk
            # features are addressed by position in micro.vertices (need[0] == vertices)
            ids = np.searchsorted(verts, plan.need[k])
            t["need_ids"][k][:nk].copy_(i32(ids))
            t["need_off"][k][:2].copy_(i32([0, nk]))
            inl = np.isin(plan.need[k], micro.layers[k])
            t["in_layer"][k][:nk].copy_(torch.as_tensor(inl.astype(np.int8), device=dev))
        for k in range(1, L + 1):
            self_pos, dpos, spos, deg = plan.layers[k - 1]
            nk = len(plan.need[k])
            order = np.argsort(dpos, kind="stable")
            off = np.zeros(nk + 1, dtype=np.int64)
            np.cumsum(np.bincount(dpos, minlength=nk), out=off[1:])
            t["self_pos"][k][:nk].copy_(i32(self_pos))
            t["nbr_off"][k][:nk + 1].copy_(i32(off))
            t["nbr_idx"][k][:len(spos)].copy_(i32(spos[order]))
            t["pair_off"][k][:2].copy_(i32([0, len(spos)]))
            tot[L + k] = len(spos)
        t["totals"].copy_(i32(tot))
        # the fused-gather vertex-id lists are not built for a host batch
        self.runner.desc.mg.nbr_vid1 = None
        self.runner.desc.mg.self_vid1 = None
        self.runner.desc.roots = self.runner.roots.data_ptr()
        self.runner.desc.agg1_ready = 0
        self.labels = torch.zeros(1, dtype=torch.int32, device=dev)

    def run(self, fn: str, label: int = None) -> None:
        d = self.runner.desc
        d.labels = None
        if label is not None:
            self.labels.fill_(int(label))
            d.labels = self.labels.data_ptr()
        s = torch.cuda.current_stream(self.runner.device).cuda_stream
        _lib.call(fn, C.byref(d), 1, s)


@dataclass
class ForwardState:
    """Forward artifacts (model.py:201-210): values[k] (layer-k activations of
    need[k], values[0] = inputs), aggregates, pre_relu (host float64 copies of
    the device buffers) and the root logits."""

    micro: object
    plan: MicroPlan
    values: list
    aggregates: list
    pre_relu: list
    logits: np.ndarray
    _dev: object = None


def forward(micro, features, model: ModelState) -> ForwardState:
    """model.py:213-247 on the GPU (hg_forward over a one-root batch)."""
    one = _OneRoot(micro, features, model)
    one.run("hg_forward")
    r = one.runner
    L = micro.n_layers
    torch.cuda.synchronize(model.device)
    feats = np.asarray(features, dtype=np.float64)
    values = [feats[np.searchsorted(micro.vertices, one.plan.need[0])]]
    aggs, pre = [], []
    for k in range(1, L + 1):
        nk = len(one.plan.need[k])
        values.append(r.h[k][:nk].double().cpu().numpy())
        a = r.agg[k][:nk].double().cpu().numpy()
        if k == 1 and model.Dp != model.D:  # drop the 16-byte row padding
            a = a[:, model._ref_rows(1)] if model.arch == "sage-mean" else a[:, :model.D]
        aggs.append(a)
    # the device step keeps h = ReLU(z), not z: pre-activations are re-formed from
    # the device aggregates (z_k = agg_k W_k + b_k, model.py:241-242)
    ws, bs, _ = model.reference_arrays()
    pre = [aggs[k] @ ws[k] + bs[k] for k in range(L)]
    logits = r.logits[0, :model.C].double().cpu().numpy()
    return ForwardState(micro, one.plan, values, aggs, pre, logits, one)


def loss_and_backward(state: ForwardState, label: int, model: ModelState):
    """model.py:250-287: (softmax-CE loss, unscaled Gradients) of one micrograph.
    Runs the device step (forward + backward, hg_train_step) with the explicit
    label; the model's own accumulator is left untouched."""
    one = state._dev
    saved = model.grad.clone()
    model.grad.zero_()
    one.run("hg_train_step", label)
    loss = float(one.runner.loss[0].item())
    w, b, c = model.reference_arrays(model.grad)
    model.grad.copy_(saved)
    return loss, Gradients(w, b, c)


def micrograph_loss(micro, features, label: int, model: ModelState) -> float:
    """Loss only (model.py:290-296)."""
    st = forward(micro, features, model)
    sh = st.logits - st.logits.max()
    e = np.exp(sh)
    return float(np.log(e.sum()) - sh[int(label)])


def sync_and_update(models, accs, batch_total: int, lr: float, ledger: CommLedger = None):
    """All-reduce the accumulators and step every replica (model.py:299-329):
    replicas must be identical; global = sum(accs) / batch_total; each model's
    SGD runs on the device (hg_sgd_update); ring all-reduce bytes in the ledger."""
    n = len(models)
    if n == 0:
        raise ValueError("no models")
    base = models[0]
    for m in models[1:]:
        if not torch.equal(m.flat, base.flat):
            raise InvariantViolation("replicas diverged before gradient sync")
    total = Gradients.zeros_like(base)
    for acc in accs:
        total.add(acc.grads)
    step = total.scaled(1.0 / batch_total) if batch_total > 0 else total
    for m in models:
        m.load_reference(total.weights, total.biases, total.classifier, buf=m.grad)
        m.sgd(lr, batch_total)
    if ledger is not None and n > 1:
        per_link = 2.0 * (n - 1) / n * base.param_bytes
        for s in range(n):
            ledger.add(s, (s + 1) % n, GRADIENT, per_link, 2 * (n - 1))
    return step
