"""Device step runner: one cell of roots -> micrographs -> loss + gradients.

This is what the reference's ``run_cell`` (engine.py:413-448) does per
micrograph in Python; here it is two C-ABI calls on one stream
(``hg_mg_build`` then ``hg_train_step``) over buffers allocated once at
capacity, so the sequence can be captured in a CUDA graph.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .featstore import FeatureTable
from .graph import Graph
from .model import SAGE_MEAN, LabelOracle, ModelState
from .sampler import MicrographBatch, MicrographBuilder


class CellRunner:
    def __init__(self, graph: Graph, table: FeatureTable, model: ModelState, fanout,
                 max_roots: int, labels: LabelOracle, split_k: int = 0, use_tc: bool = True):
        if len(fanout) != model.L:
            raise ValueError("one fanout per layer")
        if table.ld != model.Dp:
            raise ValueError("feature row stride must equal the model's padded width")
        self.graph, self.table, self.model = graph, table, model
        self.device = model.device
        self.builder = MicrographBuilder(fanout, max_roots, self.device)
        lay = self.builder.layout
        L, H = model.L, model.H
        act = table.dtype
        dev = self.device
        self.max_roots = int(max_roots)
        self.max_rows = [max_roots * lay.cap_need[k] for k in range(L + 1)]
        self.agg = [None] + [torch.empty((self.max_rows[k], model.in_dim[k]), dtype=act, device=dev)
                             for k in range(1, L + 1)]
        self.h = [None] + [torch.empty((self.max_rows[k], H), dtype=act, device=dev)
                           for k in range(1, L + 1)]
        self.dh = [None] + [torch.zeros((self.max_rows[k], H), dtype=torch.float32, device=dev)
                            for k in range(1, L + 1)]
        dagg_rows = max([self.max_rows[k] * model.in_dim[k] for k in range(2, L + 1)] or [1])
        self.dagg = torch.empty(dagg_rows, dtype=torch.float32, device=dev)
        self.logits = torch.empty((max_roots, model.C), dtype=torch.float32, device=dev)
        self.loss = torch.zeros(max_roots, dtype=torch.float32, device=dev)
        # one bf16 dz region per layer (hg_step_desc.lowp_layered)
        self.lowp = torch.empty((sum(self.max_rows[1:]), H), dtype=torch.bfloat16, device=dev)
        self.roots = torch.zeros(max_roots, dtype=torch.int64, device=dev)
        self.keys = torch.zeros(max(max_roots, 1), dtype=torch.int64, device=dev)
        d = _lib.StepDesc()
        d.n_layers, d.arch = L, 1 if model.arch == SAGE_MEAN else 0
        d.act_dtype = table.act_dtype
        d.feat_dim, d.feat_ld, d.hidden, d.n_classes = model.D, model.Dp, H, model.C
        d.max_roots = max_roots
        for k in range(L + 1):
            d.max_rows[k] = self.max_rows[k]
            # layer k's pairs come from hop L-k+1 (fanout[L-k], sampler.py:93-98)
            d.max_deg[k] = int(fanout[L - k]) if k >= 1 else 0
            d.root_rows[k] = lay.cap_need[k]
            d.in_dim[k] = model.in_dim[k]
        d.split_k = split_k or max(1, min(64, self.max_rows[1] // 2048))
        d.use_tc = int(use_tc)
        # the step's tensor-core path (mirrors run_step's condition)
        self.tc = act == torch.bfloat16 and use_tc and H % 64 == 0 and H <= 256
        d.features = table.table.data_ptr()
        d.feat_row = table.row_of.data_ptr() if table.row_of is not None else None
        d.roots = self.roots.data_ptr()
        d.label_state = labels.state
        d.mg = self.builder.cbatch
        for k in range(1, L + 1):
            d.W[k] = model.W(k).data_ptr()
            d.b[k] = model.b(k).data_ptr()
            d.Wlp[k] = model.W(k, model.shadow).data_ptr()
            d.gW[k] = model.W(k, model.grad).data_ptr()
            d.gb[k] = model.b(k, model.grad).data_ptr()
            d.agg[k] = self.agg[k].data_ptr()
            d.h[k] = self.h[k].data_ptr()
            d.dh[k] = self.dh[k].data_ptr()
        d.Wc = model.Wc().data_ptr()
        d.Wclp = model.Wc(model.shadow).data_ptr()
        d.gWc = model.Wc(model.grad).data_ptr()
        d.dagg = self.dagg.data_ptr()
        d.logits = self.logits.data_ptr()
        d.loss = self.loss.data_ptr()
        d.lowp_scratch = self.lowp.data_ptr()
        d.lowp_layered = 1
        # bf16 operand copies of the parameters: one set per model, shared by
        # every runner (steps are serialised on the training stream), so a
        # fused SGD + refresh (hg_sgd_refresh) keeps all of them current
        if not hasattr(model, "_lowp"):
            Cp_ = (model.C + 63) // 64 * 64
            model._lowp = {
                "wb16": torch.empty(model.flat.numel(), dtype=torch.bfloat16, device=dev),
                "wct": torch.empty((model.C, H), dtype=torch.bfloat16, device=dev),
                "wcp": torch.zeros((H, Cp_), dtype=torch.bfloat16, device=dev)}
        self.wb16, self.wct, self.wcp = (model._lowp[k] for k in ("wb16", "wct", "wcp"))
        for k in range(1, L + 1):
            d.Wb[k] = self.wb16.data_ptr() + 2 * int(model.offsets[k - 1])
        Cp = (model.C + 63) // 64 * 64
        self.dl16 = torch.zeros((max_roots, Cp), dtype=torch.bfloat16, device=dev)
        d.WcT, d.Wcp, d.dl_lowp = self.wct.data_ptr(), self.wcp.data_ptr(), self.dl16.data_ptr()
        self.desc = d
        self.n_roots = 0
        self.n_dev = torch.zeros(1, dtype=torch.int32, device=dev)  # device root count (graphs)

    def stage_roots(self, roots, keys, roots_per_state: int) -> None:
        """Copy roots (int64) and iteration states / keys into the fixed buffers."""
        r = torch.as_tensor(roots, dtype=torch.int64, device=self.device)
        n = r.numel()
        if n > self.max_roots:
            raise ValueError(f"{n} roots > capacity {self.max_roots}")
        self.roots[:n].copy_(r, non_blocking=True)
        k = torch.as_tensor(keys, dtype=torch.int64, device=self.device)
        self.keys[:k.numel()].copy_(k, non_blocking=True)
        self.n_roots = n
        self.roots_per_state = roots_per_state

    def launch(self, n_roots: int = None, roots_per_state: int = None, backward: bool = True,
               stream=None) -> MicrographBatch:
        """Build micrographs for the staged roots and run forward(+backward).
        Gradients are accumulated into model.grad."""
        n = self.n_roots if n_roots is None else n_roots
        rps = self.roots_per_state if roots_per_state is None else roots_per_state
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        batch = self.builder.build(self.graph, self.roots, self.keys, rps, n_roots=n, stream=s)
        fn = "hg_train_step" if backward else "hg_forward"
        _lib.call(fn, C.byref(self.desc), n, s)
        return batch

    def check(self) -> None:
        self.builder.check()

    def losses(self, n=None) -> np.ndarray:
        return self.loss[:(self.n_roots if n is None else n)].cpu().numpy()
