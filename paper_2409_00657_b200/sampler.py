"""Micrograph sampling on the GPU (drop-in for reference ``gnnsim.sampler``).

``sample_micrograph`` keeps the reference signature (sampler.py:84-106) and
returns a host ``Micrograph`` with identical layers / pairs / vertices.  The
hot path uses ``MicrographBuilder``: one ``hg_mg_build`` launch samples,
dedups, relabels and plans a whole batch of roots into device-resident
``MicrographBatch`` tensors (layout: csrc/hg_sampler.cu, include/hopgnn.h).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .graph import Graph, PartitionMap
from .rng import chain

MAX_GROUP = _lib.MAX_GROUP

NODE_WISE = "node-wise"
LAYER_WISE = "layer-wise"


@dataclass(frozen=True)
class SamplerConfig:
    """Same fields and validation as the reference (sampler.py:28-49)."""

    n_layers: int
    fanout: tuple
    mode: str = NODE_WISE
    seed: int = 0

    def __post_init__(self):
        fo = self.fanout if isinstance(self.fanout, (tuple, list)) else (self.fanout,) * self.n_layers
        fo = tuple(int(f) for f in fo)
        if len(fo) == 1 and self.n_layers > 1:
            fo = fo * self.n_layers
        object.__setattr__(self, "fanout", fo)
        if self.n_layers < 1:
            raise ValueError("n_layers must be >= 1")
        if len(self.fanout) != self.n_layers or any(f < 1 for f in self.fanout):
            raise ValueError("need one fanout >= 1 per layer")
        if self.mode not in (NODE_WISE, LAYER_WISE):
            raise ValueError(f"unknown sampling mode {self.mode!r}")

    def stream_key(self, epoch: int, iteration: int, root: int) -> int:
        return stream_key(self.seed, epoch, iteration, root)


def stream_key(seed: int, epoch: int, iteration: int, root: int) -> int:
    """Key for one root's draw (sampler.py:52-54)."""
    return chain(seed, epoch, iteration, root)


def iteration_state(seed: int, epoch: int, iteration: int) -> int:
    """Prefix of stream_key: the device folds the root in (mix64(state ^ root))."""
    return chain(seed, epoch, iteration)


@dataclass(frozen=True)
class Micrograph:
    """Host view with the reference fields (sampler.py:57-81)."""

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


def plan_layout(fanout: Sequence[int]) -> _lib.MgLayout:
    lay = _lib.MgLayout()
    arr = (C.c_int32 * len(fanout))(*[int(f) for f in fanout])
    _lib.call("hg_mg_plan_layout", len(fanout), arr, C.byref(lay))
    return lay


class MicrographBatch:
    """Device tensors of one built batch (global row numbering, see hopgnn.h)."""

    def __init__(self, L: int, n_roots: int, t: dict):
        self.L = L
        self.n_roots = n_roots
        self.need_ids = t["need_ids"]
        self.need_off = t["need_off"]
        self.in_layer = t["in_layer"]
        self.self_pos = t["self_pos"]
        self.nbr_off = t["nbr_off"]
        self.nbr_idx = t["nbr_idx"]
        self.pair_off = t["pair_off"]
        self.totals = t["totals"]

    def sizes(self):
        """(N_k for k=0..L, P_k for k=1..L) — synchronises."""
        tot = self.totals.cpu().numpy()
        return tot[:self.L + 1].tolist(), tot[self.L + 1:2 * self.L + 1].tolist()

    def to_host(self):
        L = self.L
        h = {}
        for name in ("need_ids", "need_off", "in_layer", "self_pos", "nbr_off", "nbr_idx",
                     "pair_off"):
            h[name] = [None if x is None else x.cpu().numpy() for x in getattr(self, name)]
        return h

    def micrographs(self, roots, h: dict = None) -> list:
        """Rebuild reference ``Micrograph`` objects (parity checks)."""
        h = self.to_host() if h is None else h
        L = self.L
        out = []
        for r, root in enumerate(np.asarray(roots).tolist()):
            need = [h["need_ids"][k][h["need_off"][k][r]:h["need_off"][k][r + 1]].astype(np.int64)
                    for k in range(L + 1)]
            inl = [h["in_layer"][k][h["need_off"][k][r]:h["need_off"][k][r + 1]].astype(bool)
                   for k in range(L + 1)]
            layers = [need[k][inl[k]] for k in range(L + 1)]
            pairs = []
            for k in range(1, L + 1):
                base, pbase = h["need_off"][k][r], h["need_off"][k - 1][r]
                dst, src = [], []
                di = 0
                for a in range(len(need[k])):
                    g = base + a
                    lo, hi = h["nbr_off"][k][g], h["nbr_off"][k][g + 1]
                    if inl[k][a]:
                        srcv = need[k - 1][h["nbr_idx"][k][lo:hi] - pbase]
                        src.append(np.searchsorted(layers[k - 1], srcv))
                        dst.append(np.full(hi - lo, di, dtype=np.int64))
                        di += 1
                pairs.append((np.concatenate(dst) if dst else np.empty(0, np.int64),
                              np.concatenate(src).astype(np.int64) if src else np.empty(0, np.int64)))
            out.append(Micrograph(int(root), tuple(layers), tuple(pairs), need[0]))
        return out

    def plans(self, r: int, h: dict = None):
        """need sets and (self_pos, dpos, spos, deg) of root r in local numbering
        (h: a to_host() snapshot, reused across roots)."""
        h = self.to_host() if h is None else h
        L = self.L
        need = [h["need_ids"][k][h["need_off"][k][r]:h["need_off"][k][r + 1]].astype(np.int64)
                for k in range(L + 1)]
        steps = []
        for k in range(1, L + 1):
            base, pbase = h["need_off"][k][r], h["need_off"][k - 1][r]
            nk = len(need[k])
            sp = h["self_pos"][k][base:base + nk] - pbase
            off = h["nbr_off"][k][base:base + nk + 1]
            deg = np.diff(off).astype(np.float64)
            dpos = np.repeat(np.arange(nk), np.diff(off))
            spos = h["nbr_idx"][k][off[0]:off[-1]] - pbase
            steps.append((sp.astype(np.int64), dpos.astype(np.int64), spos.astype(np.int64), deg))
        return need, steps


class MicrographBuilder:
    """Owns the reusable workspace + output buffers of hg_mg_build for up to
    `max_roots` roots (fixed addresses, so launches can be graph-captured)."""

    def __init__(self, fanout: Sequence[int], max_roots: int, device="cuda"):
        self.fanout = tuple(int(f) for f in fanout)
        self.L = len(self.fanout)
        self.layout = plan_layout(self.fanout)
        self.max_roots = int(max_roots)
        dev = torch.device(device)
        self.device = dev
        lay = self.layout
        R = self.max_roots
        L = self.L
        i32 = dict(dtype=torch.int32, device=dev)
        self.ws = torch.empty(R * lay.ws_root_ints, **i32)
        t = {k: [None] * (L + 1) for k in ("need_ids", "need_off", "in_layer", "self_pos",
                                           "nbr_off", "nbr_idx", "pair_off")}
        for k in range(L + 1):
            cap = R * lay.cap_need[k]
            t["need_ids"][k] = torch.empty(max(cap, 1), **i32)
            t["need_off"][k] = torch.zeros(R + 1, **i32)
            t["in_layer"][k] = torch.empty(max(cap, 1), dtype=torch.int8, device=dev)
            if k >= 1:
                t["self_pos"][k] = torch.empty(max(cap, 1), **i32)
                t["nbr_off"][k] = torch.zeros(cap + 1, **i32)
                t["nbr_idx"][k] = torch.empty(max(R * lay.cap_lay[k - 1], 1), **i32)
                t["pair_off"][k] = torch.zeros(R + 1, **i32)
        t["totals"] = torch.zeros(2 * L + 2, **i32)
        t["nbr_vid1"] = torch.empty(max(R * lay.cap_lay[0], 1), **i32)
        t["self_vid1"] = torch.empty(max(R * lay.cap_need[1], 1), **i32)
        self.tensors = t
        self.err = torch.zeros(1, **i32)
        self.cbatch = _lib.MgBatch()
        for name in ("need_ids", "need_off", "in_layer", "self_pos", "nbr_off", "nbr_idx",
                     "pair_off"):
            arr = getattr(self.cbatch, name)
            for k in range(L + 1):
                x = t[name][k]
                arr[k] = x.data_ptr() if x is not None else None
        self.cbatch.totals = t["totals"].data_ptr()
        self.cbatch.nbr_vid1 = t["nbr_vid1"].data_ptr()
        self.cbatch.self_vid1 = t["self_vid1"].data_ptr()

    def build(self, g: Graph, roots: torch.Tensor, keys: torch.Tensor, roots_per_state: int,
              n_roots: int = None, stream=None, n_dev: int = None) -> MicrographBatch:
        """Launch sampling + build.  keys: uint64 (as int64) iteration states, or
        per-root final keys when roots_per_state == 0."""
        n = roots.numel() if n_roots is None else int(n_roots)
        if n > self.max_roots:
            raise ValueError(f"{n} roots > builder capacity {self.max_roots}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        rp = roots if isinstance(roots, int) else roots.data_ptr()
        kp = keys if isinstance(keys, int) else keys.data_ptr()
        if getattr(g, "shards", None) is not None:  # partitioned CSR (graph.ShardedGraph)
            _lib.call("hg_mg_build_group_sharded", C.byref(g.shards), g.n_vertices, rp, n, 1,
                      n_dev, kp, int(roots_per_state), C.byref(self.layout), self.ws.data_ptr(),
                      C.byref(self.cbatch), self.err.data_ptr(), 0, s)
            return MicrographBatch(self.L, n, self.tensors)
        if n_dev is not None:  # n is the capacity; the device count says how many are real
            _lib.call("hg_mg_build_n", g.offsets.data_ptr(), g.targets.data_ptr(), g.n_vertices,
                      rp, n, n_dev, kp, int(roots_per_state), C.byref(self.layout),
                      self.ws.data_ptr(), C.byref(self.cbatch), self.err.data_ptr(), s)
            return MicrographBatch(self.L, n, self.tensors)
        _lib.call("hg_mg_build", g.offsets.data_ptr(), g.targets.data_ptr(), g.n_vertices,
                  rp, n, kp, int(roots_per_state),
                  C.byref(self.layout), self.ws.data_ptr(), C.byref(self.cbatch),
                  self.err.data_ptr(), s)
        return MicrographBatch(self.L, n, self.tensors)

    def check(self, what="hg_mg_build"):
        code = int(self.err.item())
        if code:
            self.err.zero_()
        _lib.flag_status(code, what)


class GroupBuilder:
    """Run-ahead over several iterations in ONE build launch
    (hg_mg_build_group): batch b of the group is written into builders[b]'s
    own output buffers, exactly as builders[b].build would have written it.
    Owns the group's contiguous roots [K*R], iteration states [K] and
    workspace (fixed addresses: graph-capturable)."""

    def __init__(self, builders, per_batch: int = None):
        if not 1 <= len(builders) <= MAX_GROUP:
            raise ValueError(f"group of {len(builders)} batches (1..{MAX_GROUP})")
        self.builders = list(builders)
        b0 = self.builders[0]
        if any(b.fanout != b0.fanout or b.max_roots != b0.max_roots for b in self.builders):
            raise ValueError("grouped builders must share fanout and capacity")
        self.K, self.layout, self.device = len(builders), b0.layout, b0.device
        # roots per batch (the stride of the roots buffer; <= builder capacity)
        self.R = b0.max_roots if per_batch is None else int(per_batch)
        if not 1 <= self.R <= b0.max_roots:
            raise ValueError(f"per_batch {self.R} outside 1..{b0.max_roots}")
        i32 = dict(dtype=torch.int32, device=self.device)
        self.ws = torch.empty(self.K * self.R * self.layout.ws_root_ints, **i32)
        self.roots = torch.zeros(self.K * self.R, dtype=torch.int64, device=self.device)
        self.keys = torch.zeros(self.K, dtype=torch.int64, device=self.device)
        self.err = torch.zeros(1, **i32)
        self.n_dev = torch.zeros(self.K, **i32)  # per-batch device root counts (optional)
        self.outs = (_lib.MgBatch * self.K)(*[b.cbatch for b in self.builders])

    def roots_ptr(self, b: int) -> int:
        return self.roots.data_ptr() + 8 * b * self.R

    def build(self, g: Graph, stream=None, n_dev: int = None, ctas_per_sm: int = 0) -> None:
        """Build all K batches from self.roots / self.keys (R roots each;
        batch b keyed by iteration state keys[b]).  ctas_per_sm > 0 caps the
        resident build CTAs per SM (persistent grid) to leave room for
        concurrently running kernels."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        if getattr(g, "shards", None) is not None:  # partitioned CSR (graph.ShardedGraph)
            _lib.call("hg_mg_build_group_sharded", C.byref(g.shards), g.n_vertices,
                      self.roots.data_ptr(), self.R, self.K, n_dev, self.keys.data_ptr(), self.R,
                      C.byref(self.layout), self.ws.data_ptr(), self.outs, self.err.data_ptr(),
                      int(ctas_per_sm), s)
            return
        _lib.call("hg_mg_build_group", g.offsets.data_ptr(), g.targets.data_ptr(), g.n_vertices,
                  self.roots.data_ptr(), self.R, self.K, n_dev, self.keys.data_ptr(), self.R,
                  C.byref(self.layout), self.ws.data_ptr(), self.outs, self.err.data_ptr(),
                  int(ctas_per_sm), s)

    def check(self, what="hg_mg_build_group"):
        code = int(self.err.item())
        if code:
            self.err.zero_()
        _lib.flag_status(code, what)


_builders: dict = {}


def _as_u64_tensor(vals, device):
    arr = np.asarray([int(v) & ((1 << 64) - 1) for v in vals], dtype=np.uint64).view(np.int64)
    return torch.from_numpy(arr).to(device)


def sample_micrograph(g: Graph, root: int, cfg: SamplerConfig, key: int) -> Micrograph:
    """Sample one root's micrograph under `key` (sampler.py:84-106); node-wise
    through the batched device build, layer-wise hop by hop on the device."""
    if not 0 <= int(root) < g.n_vertices:
        raise ValueError(f"root {root} out of range for {g.n_vertices} vertices")
    if cfg.mode == LAYER_WISE:
        return _layer_wise_micrograph(g, int(root), cfg, key)
    return sample_micrographs(g, [root], cfg, [key])[0]


def layer_wise_hop(g: Graph, frontier: torch.Tensor, budget: int, state: int):
    """One layer-wise hop (sampler.py:109-120) on the device: the frontier's
    neighbour spans, their distinct ids as candidates, a shared draw of
    `budget` of them (kernels.pick_k_smallest, hg_pick_k_smallest), and the
    (dst, src) pairs whose source was drawn.  Returns device int64 tensors."""
    from .kernels import pick_k_smallest
    dev = g.device
    if frontier.numel() == 0:
        e = torch.empty(0, dtype=torch.int64, device=dev)
        return e, e
    lo, hi = g.offsets[frontier], g.offsets[frontier + 1]
    ln = hi - lo
    start = torch.zeros(frontier.numel() + 1, dtype=torch.int64, device=dev)
    torch.cumsum(ln, 0, out=start[1:])
    m = int(start[-1].item())
    dst_all = torch.repeat_interleave(torch.arange(frontier.numel(), device=dev), ln)
    flat_all = g.targets[torch.repeat_interleave(lo - start[:-1], ln) +
                         torch.arange(m, device=dev)].long() if m else dst_all
    cand = torch.unique(flat_all)
    sel = torch.as_tensor(pick_k_smallest(cand, int(budget), state), device=dev)
    keep = torch.isin(flat_all, sel)
    return dst_all[keep], flat_all[keep]


def _layer_wise_micrograph(g: Graph, root: int, cfg: SamplerConfig, key: int) -> Micrograph:
    """sample_micrograph's hop loop with layer-wise hops (sampler.py:93-106)."""
    L = cfg.n_layers
    dev = g.device
    layers = [None] * (L + 1)
    pairs = [None] * L
    layers[L] = torch.tensor([root], dtype=torch.int64, device=dev)
    for k in range(L - 1, -1, -1):
        hop = L - k
        dst, flat = layer_wise_hop(g, layers[k + 1], cfg.fanout[hop - 1], chain(key, hop))
        layers[k] = torch.unique(flat)
        pairs[k] = (dst, torch.searchsorted(layers[k], flat))
    host = [x.cpu().numpy().astype(np.int64) for x in layers]
    hp = tuple((d.cpu().numpy().astype(np.int64), s_.cpu().numpy().astype(np.int64))
               for d, s_ in pairs)
    verts = np.unique(np.concatenate(host))
    return Micrograph(int(root), tuple(host), hp, verts)


def sample_micrographs(g: Graph, roots, cfg: SamplerConfig, keys) -> list:
    """Batch version with explicit per-root stream keys (one launch)."""
    roots = np.asarray(roots, dtype=np.int64)
    if len(roots) and (roots.min() < 0 or roots.max() >= g.n_vertices):
        raise ValueError(f"root out of range for {g.n_vertices} vertices")
    bkey = (cfg.fanout, str(g.device))
    b = _builders.get(bkey)
    if b is None or b.max_roots < max(len(roots), 1):
        b = MicrographBuilder(cfg.fanout, max(len(roots), 64), g.device)
        _builders[bkey] = b
    rt = torch.from_numpy(roots).to(g.device)
    kt = _as_u64_tensor(keys, g.device)
    batch = b.build(g, rt, kt, 0)
    torch.cuda.synchronize(g.device)
    b.check()
    return batch.micrographs(roots)


# ---------------------------------------------------------------- root plans

@dataclass(frozen=True)
class MiniBatchPlan:
    """Per-model batches and their home regrouping (sampler.py:148-165)."""

    batches: tuple
    groups: tuple
    n_servers: int

    def server_totals(self) -> np.ndarray:
        tot = np.zeros(self.n_servers, dtype=np.int64)
        for per_model in self.groups:
            for s, roots in enumerate(per_model):
                tot[s] += len(roots)
        return tot


def redistribute_roots(batches, p: PartitionMap) -> MiniBatchPlan:
    """Group every batch's roots by home server, order kept (sampler.py:168-177)."""
    norm, groups = [], []
    for b in batches:
        b = np.asarray(b, dtype=np.int64)
        norm.append(b)
        h = p.home[b]
        groups.append(tuple(b[h == s] for s in range(p.n_servers)))
    return MiniBatchPlan(tuple(norm), tuple(groups), p.n_servers)


def load_imbalance(plan: MiniBatchPlan) -> float:
    tot = plan.server_totals()
    mean = tot.mean() if len(tot) else 0.0
    return 0.0 if mean == 0 else float((tot.max() - tot.min()) / mean)
