"""Training drivers: single-GPU trainer and the multi-GPU micrograph strategy.

Reference: engine.py — ``epoch_batches`` (268-287), ``run_cell`` (413-448),
``_model_centric_epoch`` (485-507), ``_micrograph_epoch`` (562-623),
``TraceTable`` / ``assign_cell_roots`` (103-205), merge controller
(779-833).  With one server every strategy degenerates to model-centric
training (test_engine.py:215-225); ``Trainer`` is that case, fully
device-resident: the epoch permutation and the per-iteration stream-key
states live in HBM and each step is

    hg_mg_build (sample + dedup/relabel + plan)  ->  hg_train_step  ->  SGD

with no host synchronisation.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .batching import epoch_permutation, iterations_per_epoch
from .featstore import FeatureTable
from .graph import Graph
from .model import LabelOracle, ModelState
from .rng import chain
from .trainer import CellRunner

SEED_GRAPH, SEED_PARTITION, SEED_FEATURES, SEED_LABELS = 0x01, 0x02, 0x03, 0x04
SEED_BATCHES, SEED_SAMPLER, SEED_MODEL, SEED_MERGE = 0x05, 0x06, 0x07, 0x08


def _u64_as_i64(vals) -> np.ndarray:
    return np.asarray([int(v) & ((1 << 64) - 1) for v in vals], dtype=np.uint64).view(np.int64)


class Trainer:
    """One model on one GPU (S = 1): the reference's micrograph and
    model-centric strategies coincide here (engine.py:485-507 with N = 1)."""

    def __init__(self, graph: Graph, table: FeatureTable, model: ModelState, fanout,
                 batch: int, seed: int, lr: float = 0.1, iterations: int = 0):
        self.graph, self.table, self.model = graph, table, model
        self.fanout = tuple(fanout)
        self.B, self.seed, self.lr, self.iter_cap = int(batch), int(seed), float(lr), iterations
        self.labels = LabelOracle(model.C, chain(seed, SEED_LABELS))
        self.sampler_seed = chain(seed, SEED_SAMPLER)
        self.runner = CellRunner(graph, table, model, self.fanout, self.B, self.labels)
        self.device = model.device
        self.epoch = None
        self.stream = torch.cuda.current_stream(self.device)

    # ------------------------------------------------------------ epoch plan
    def begin_epoch(self, epoch: int) -> int:
        """Permutation + per-iteration key states for `epoch`; returns #iterations."""
        n = self.graph.n_vertices
        self.perm = epoch_permutation(self.seed, epoch, n, self.device)
        self.iters = iterations_per_epoch(n, 1, self.B, self.iter_cap)
        states = [chain(self.sampler_seed, epoch, it) for it in range(self.iters)]
        self.states = torch.from_numpy(_u64_as_i64(states)).to(self.device)
        self.epoch = epoch
        return self.iters

    def roots_of(self, it: int) -> torch.Tensor:
        lo = min(it * self.B, self.perm.numel())
        return self.perm[lo:min(lo + self.B, self.perm.numel())]

    # ------------------------------------------------------------ steps
    def step(self, it: int) -> None:
        """One iteration with inputs already resident in HBM (no host sync)."""
        roots = self.roots_of(it)
        n = roots.numel()
        s = self.stream.cuda_stream
        r = self.runner
        r.builder.build(self.graph, roots.data_ptr(), self.states.data_ptr() + 8 * it, n,
                        n_roots=n, stream=s)
        r.desc.roots = roots.data_ptr()
        _lib.call("hg_train_step", C.byref(r.desc), n, s)
        self.model.sgd(self.lr, n, stream=s)

    def train_step(self, roots_host: torch.Tensor, it: int) -> float:
        """Public end-to-end step: roots come from (pinned) host memory and the
        summed loss of the step is read back (engine.py:434-445 semantics)."""
        r = self.runner
        n = roots_host.numel()
        r.roots[:n].copy_(roots_host, non_blocking=True)
        s = self.stream.cuda_stream
        r.builder.build(self.graph, r.roots.data_ptr(), self.states.data_ptr() + 8 * it, n,
                        n_roots=n, stream=s)
        r.desc.roots = r.roots.data_ptr()
        _lib.call("hg_train_step", C.byref(r.desc), n, s)
        self.model.sgd(self.lr, n, stream=s)
        return float(r.loss[:n].sum().item())

    def check(self) -> None:
        self.runner.check()

    def batch_sizes(self):
        """(N_k, P_k) of the last built batch (synchronises)."""
        tot = self.runner.builder.tensors["totals"].cpu().numpy()
        L = len(self.fanout)
        return tot[:L + 1].tolist(), tot[L + 1:2 * L + 1].tolist()
