"""Locality statistics of micrographs (reference metrics.py:23-113).

R_micro: the fraction of a micrograph's vertices homed with its root;
R_sub: per root, the fraction of its mini-batch subgraph's distinct vertices
homed with it (the paper's locality argument for feature-centric training).
``locality_report`` samples the batches on the GPU (one batched build per
model batch; node-wise) and reduces the ratios there; the per-micrograph
``r_micro`` / ``r_sub`` keep the reference signatures.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Sequence

import numpy as np
import torch

from .sampler import Micrograph, NODE_WISE, SamplerConfig, sample_micrograph
from .rng import chain


@dataclass(frozen=True)
class Subgraph:
    """The micrographs of one mini-batch (sampler.py:123-141)."""

    members: tuple
    roots: np.ndarray

    @property
    def unique_vertices(self) -> np.ndarray:
        if not self.members:
            return np.empty(0, dtype=np.int64)
        return np.unique(np.concatenate([m.vertices for m in self.members]))

    @property
    def unique_vertex_count(self) -> int:
        return len(self.unique_vertices)


def build_subgraph(micros: Sequence[Micrograph]) -> Subgraph:
    roots = np.array([m.root for m in micros], dtype=np.int64)
    if len(np.unique(roots)) != len(roots):
        raise ValueError("duplicate roots in one mini-batch")
    return Subgraph(tuple(micros), roots)


def r_micro(m: Micrograph, p, include_root: bool = True) -> float:
    """metrics.py:23-34."""
    co = int(np.count_nonzero(p.home[m.vertices] == p.home[m.root]))
    if not include_root:
        co -= 1
    return co / m.vertex_count


def r_sub(sg: Subgraph, p, include_root: bool = True) -> float:
    """metrics.py:37-51."""
    if len(sg.roots) == 0:
        raise ValueError("subgraph has no roots")
    homes = p.home[sg.unique_vertices]
    total = len(homes)
    ratios = []
    for r in sg.roots:
        co = int(np.count_nonzero(homes == p.home[r]))
        if not include_root:
            co -= 1
        ratios.append(co / total)
    return float(np.mean(ratios))


@dataclass(frozen=True)
class LocalityRow:
    n_servers: int
    n_layers: int
    mode: str
    partitioner: str
    r_micro_mean: float
    r_sub_mean: float
    samples: int


def _batch_ratios(world, roots: np.ndarray, epoch: int, it: int):
    """(per-root R_micro, R_sub) of one batch, reduced on the device."""
    from .sampler import MicrographBuilder
    cfg = world.cfg
    dev = world.graph.device
    home = world.partition.home_device(dev).long()
    n = len(roots)
    if cfg.mode == NODE_WISE:
        b = MicrographBuilder(cfg.fanout, n, dev)
        st = torch.tensor([np.uint64(chain(world.sampler_seed, epoch, it)).view(np.int64)],
                          device=dev)
        batch = b.build(world.graph, torch.from_numpy(roots).to(dev), st, n)
        off = batch.need_off[0][:n + 1].long()
        verts = batch.need_ids[0][:int(off[-1])].long()
        owner = torch.repeat_interleave(torch.arange(n, device=dev), off[1:] - off[:-1])
    else:
        scfg = SamplerConfig(cfg.layers, cfg.fanout, cfg.mode, world.sampler_seed)
        ms = [sample_micrograph(world.graph, int(r), scfg, scfg.stream_key(epoch, it, int(r)))
              for r in roots]
        verts = torch.from_numpy(np.concatenate([m.vertices for m in ms])).to(dev)
        owner = torch.repeat_interleave(torch.arange(n, device=dev),
                                        torch.tensor([len(m.vertices) for m in ms], device=dev))
    rh = home[torch.from_numpy(roots).to(dev)]
    same = (home[verts] == rh[owner]).double()
    cnt = torch.bincount(owner, minlength=n).double()
    micro = torch.zeros(n, dtype=torch.float64, device=dev).index_add_(0, owner, same) / cnt
    uh = home[torch.unique(verts)]
    per_root = (uh[None, :] == rh[:, None]).sum(1).double() / uh.numel()
    return micro.cpu().numpy(), float(np.mean(per_root.cpu().numpy()))


def locality_report(world_cfg, partitioners: Sequence[str], modes: Sequence[str],
                    server_counts: Sequence[int], layer_counts: Sequence[int],
                    iterations: int = 3, batch: int = None) -> list:
    """Monte Carlo locality ratios over sampled batches (metrics.py:63-82): one
    row per (partitioner, mode, S, L) in that order; a pure function of the seed."""
    from .strategy import as_run_config, build_world, epoch_batches
    base = as_run_config(world_cfg)
    batch = batch or base.batch
    rows = []
    for partitioner in partitioners:
        for mode in modes:
            for S in server_counts:
                for L in layer_counts:
                    cfg = replace(base, partitioner=partitioner, mode=mode, servers=S, layers=L,
                                  fanout=(base.fanout[0],) * L, batch=batch)
                    rows.append(_locality_row(build_world(cfg, modes_ok=True), iterations))
    return rows


def _locality_row(world, iterations: int) -> LocalityRow:
    """metrics.py:85-103."""
    from .strategy import epoch_batches
    micro_vals, sub_vals, count = [], [], 0
    for epoch in range(iterations):
        for it_roots in epoch_batches(world, epoch)[0]:
            if len(it_roots) == 0:
                continue
            m, s = _batch_ratios(world, np.asarray(it_roots, dtype=np.int64), epoch, 0)
            micro_vals.extend(m.tolist())
            sub_vals.append(s)
            count += len(it_roots)
    cfg = world.cfg
    return LocalityRow(cfg.servers, cfg.layers, cfg.mode, cfg.partitioner,
                       float(np.mean(micro_vals)), float(np.mean(sub_vals)), count)


LOCALITY_HEADER = "servers,layers,mode,partitioner,r_micro,r_sub,samples"


def write_locality_csv(rows, sink) -> None:
    """metrics.py:109-113."""
    sink.write(LOCALITY_HEADER + "\n")
    for r in rows:
        sink.write(f"{r.n_servers},{r.n_layers},{r.mode},{r.partitioner},"
                   f"{r.r_micro_mean!r},{r.r_sub_mean!r},{r.samples}\n")
