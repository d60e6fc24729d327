"""Feature-centric micrograph training across GPUs (one process per GPU).

Reference: engine.py ``_micrograph_epoch`` (562-623), ``TraceTable`` /
``assign_cell_roots`` / merge replay (103-205), ``plan_pregather`` /
``execute_pregather`` (featstore.py:226-279), ``sync_and_update``
(model.py:299-329).  The reference *simulates* the cluster in one process
with a byte ledger; here every server is a GPU and the bytes really move:

* features are sharded by home (each GPU holds only the rows homed at it,
  plus an iteration-scoped staging area for pre-gathered remote rows);
* the CSR is replicated (6.4 GB at papers scale; SURVEY 8(e) fallback);
* every GPU samples and trains the micrographs of the cells the trace table
  assigns to it — with the initial table, exactly the roots homed on it;
* pre-gathering is one deduplicated all-to-all per iteration (ids, then
  bf16 rows) over NCCL;
* model hop (``mode="faithful"``): after every trace-table column the model
  (parameters + gradient accumulator) is ring-shifted to the next server with
  NCCL send/recv, exactly the reference's migration schedule;
  ``mode="fused"`` skips the hops: parameters are replicated and unchanged
  within an iteration, so summing every server's gradients in the final
  all-reduce yields the identical update — the performance mode;
* the final gradient all-reduce (NCCL) is followed by the fused SGD kernel.

The ``CommLedger`` keeps the reference's accounting (4 B/element, identical
categories and messages) so byte counts compare one for one with gnnsim;
``actual`` records the bytes this implementation put on NVLink.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .batching import epoch_permutation, iterations_per_epoch
from .errors import InvariantViolation
from .featstore import (BYTES_PER_ELEM, FEATURE, GRADIENT, MODEL, CommLedger, FeatureTable,
                        FetchStats, feature_state)
from .graph import Graph, PartitionMap
from .model import LabelOracle, ModelState
from .rng import chain, hash_vec
from .trainer import CellRunner

SEED_LABELS, SEED_SAMPLER, SEED_MERGE = 0x04, 0x06, 0x08


# ---------------------------------------------------------------- trace table

def even_split(count: int, parts: int) -> list:
    """Split as evenly as possible, remainder to low indices (engine.py:156-159)."""
    base, rem = divmod(count, parts)
    return [base + (1 if i < rem else 0) for i in range(parts)]


def keyed_shuffle(state: int, values: np.ndarray) -> np.ndarray:
    values = np.asarray(values)
    keys = hash_vec(state, np.arange(len(values), dtype=np.int64))
    return values[np.argsort(keys, kind="stable")]


@dataclass
class TraceTable:
    """Model -> server placement per column plus per-cell root counts
    (engine.py:103-145).  server_of[d, j] = server of model d in column j."""

    server_of: np.ndarray
    root_counts: np.ndarray
    removed: tuple = ()

    @classmethod
    def initial(cls, n: int) -> "TraceTable":
        d = np.arange(n, dtype=np.int64)[:, None]
        t = np.arange(n, dtype=np.int64)[None, :]
        return cls((d + t) % n, np.zeros((n, n), dtype=np.int64))

    @property
    def n_models(self) -> int:
        return self.server_of.shape[0]

    @property
    def n_columns(self) -> int:
        return self.server_of.shape[1]

    def model_at(self, server: int, col: int) -> int:
        return int(np.flatnonzero(self.server_of[:, col] == server)[0])

    def validate(self) -> None:
        n = self.n_models
        for j in range(self.n_columns):
            if not np.array_equal(np.sort(self.server_of[:, j]), np.arange(n)):
                raise InvariantViolation(f"column {j} is not a bijection")
        if self.root_counts.shape != self.server_of.shape:
            raise InvariantViolation("root_counts shape mismatch")
        if np.any(self.root_counts < 0):
            raise InvariantViolation("negative root count")

    def copy(self) -> "TraceTable":
        return TraceTable(self.server_of.copy(), self.root_counts.copy(), self.removed)


def find_fewest_column(tt: TraceTable):
    """Column with the smallest root total, ties low; None below 2 columns (engine.py:148-153)."""
    if tt.n_columns < 2:
        return None
    return int(np.argmin(tt.root_counts.sum(axis=0)))


def delete_column_and_redistribute(tt: TraceTable, col: int) -> TraceTable:
    """Drop a column, spreading each model's roots over its survivors (engine.py:162-178)."""
    if tt.n_columns < 2:
        raise ValueError("cannot remove the last column")
    keep = [j for j in range(tt.n_columns) if j != col]
    counts = tt.root_counts[:, keep].copy()
    for d in range(tt.n_models):
        for i, extra in enumerate(even_split(int(tt.root_counts[d, col]), len(keep))):
            counts[d, i] += extra
    return TraceTable(tt.server_of[:, keep].copy(), counts, tt.removed + (col,))


def assign_cell_roots(tt: TraceTable, groups, key: int):
    """cells[d][j] root lists with the merge history replayed (engine.py:181-205)."""
    n = tt.n_models
    cells = [[groups[d][(d + t) % n] for t in range(n)] for d in range(n)]
    for ordinal, pos in enumerate(tt.removed):
        for d in range(n):
            row = cells[d]
            moved = keyed_shuffle(chain(key, ordinal, d), row.pop(pos))
            start = 0
            for i, size in enumerate(even_split(len(moved), len(row))):
                if size:
                    row[i] = np.concatenate([row[i], moved[start:start + size]])
                start += size
    return cells


def cell_counts(cells) -> np.ndarray:
    return np.array([[len(c) for c in row] for row in cells], dtype=np.int64)


# ---------------------------------------------------------------- sharded features

class ShardedFeatures:
    """This GPU's feature rows (home == rank) plus a staging area for the
    iteration's pre-gathered remote rows, in one HBM table indexed through
    ``row_of`` (int32[n]: local row, staging row, or -1)."""

    def __init__(self, part: PartitionMap, rank: int, dim: int, seed: int, staging_rows: int,
                 dtype=torch.bfloat16, device="cuda"):
        dev = torch.device(device)
        local = np.flatnonzero(part.home == rank).astype(np.int64)
        self.n_local = len(local)
        self.table = FeatureTable(self.n_local + staging_rows, dim, dtype, dev)
        self.staging_cap = staging_rows
        st = feature_state(seed)
        contiguous = self.n_local > 0 and local[-1] - local[0] + 1 == self.n_local
        if contiguous:
            self.table.fill_generated(int(local[0]), self.n_local, st)
        elif self.n_local:
            self.table.fill_generated(0, self.n_local, st, ids=torch.from_numpy(local).to(dev))
        row_of = torch.full((part.n_vertices,), -1, dtype=torch.int32, device=dev)
        if self.n_local:
            if contiguous:
                row_of[int(local[0]):int(local[-1]) + 1] = torch.arange(
                    self.n_local, dtype=torch.int32, device=dev)
            else:
                row_of[torch.from_numpy(local).to(dev)] = torch.arange(
                    self.n_local, dtype=torch.int32, device=dev)
        self.table.row_of = row_of
        self.home = part.home_device(dev)
        self.rank = rank
        self.S = part.n_servers
        self.device = dev


@dataclass
class Traffic:
    """Bytes this implementation moved between GPUs (not the reference's accounting)."""

    feature_rows: int = 0
    feature_bytes: int = 0
    request_bytes: int = 0
    hop_bytes: int = 0
    allreduce_bytes: float = 0.0

    def total(self) -> float:
        return self.feature_bytes + self.request_bytes + self.hop_bytes + self.allreduce_bytes


def pregather(feats: ShardedFeatures, need_ids: list, group=None):
    """Iteration-scoped pre-gathering (featstore.py:226-279): dedup the remote
    vertices of every micrograph this GPU trains, request them from their
    homes with one all-to-all, receive the rows with a second one into the
    staging area, and point ``row_of`` at them.  Returns (rows per home
    (np.int64[S]), staged rows, actual bytes moved in, request bytes out)."""
    S, rank, dev = feats.S, feats.rank, feats.device
    ids = torch.cat([x.long() for x in need_ids]) if need_ids else torch.empty(0, dtype=torch.long, device=dev)
    h = feats.home[ids].long()
    uniq = torch.unique(ids[h != rank])
    hu = feats.home[uniq].long()
    order = torch.argsort(hu, stable=True)
    req = uniq[order]
    send_counts = torch.bincount(hu, minlength=S).to(torch.int64)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    sc = send_counts.cpu().tolist()
    rc = recv_counts.cpu().tolist()
    n_req = int(sum(sc))
    if n_req > feats.staging_cap:
        raise InvariantViolation(f"pre-gather needs {n_req} rows > staging {feats.staging_cap}")
    incoming = torch.empty(int(sum(rc)), dtype=torch.int64, device=dev)
    dist.all_to_all_single(incoming, req, output_split_sizes=rc, input_split_sizes=sc, group=group)
    tab = feats.table
    out_rows = tab.table[feats.table.row_of[incoming].long()] if len(incoming) else \
        torch.empty((0, tab.ld), dtype=tab.dtype, device=dev)
    staged = tab.table[feats.n_local:feats.n_local + n_req]
    dist.all_to_all_single(staged, out_rows.contiguous(), output_split_sizes=sc,
                           input_split_sizes=rc, group=group)
    if n_req:
        tab.row_of[req] = torch.arange(feats.n_local, feats.n_local + n_req, dtype=torch.int32,
                                       device=dev)
    row_bytes = tab.ld * tab.table.element_size()
    return np.asarray(sc, dtype=np.int64), n_req, n_req * row_bytes, n_req * 8


# ---------------------------------------------------------------- trainer

class MicrographTrainer:
    """One rank of the HopGNN micrograph strategy (+ pre-gathering)."""

    def __init__(self, graph: Graph, part: PartitionMap, model: ModelState, fanout, batch: int,
                 seed: int, lr: float = 0.1, dtype=torch.bfloat16, mode: str = "fused",
                 iterations: int = 0, group=None, use_tc: bool = True):
        if mode not in ("fused", "faithful"):
            raise ValueError("mode must be 'fused' or 'faithful'")
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.S = part.n_servers
        if dist.is_initialized() and dist.get_world_size(group) != self.S:
            raise ValueError("one rank per server: world size must equal n_servers")
        self.graph, self.part, self.model = graph, part, model
        self.fanout, self.B, self.seed, self.lr = tuple(fanout), int(batch), int(seed), float(lr)
        self.mode, self.iter_cap = mode, iterations
        self.device = model.device
        self.labels = LabelOracle(model.C, chain(seed, SEED_LABELS))
        self.sampler_seed = chain(seed, SEED_SAMPLER)
        from .sampler import plan_layout
        lay = plan_layout(self.fanout)
        cap_roots = self.B * self.S if mode == "fused" else self.B
        staging = max(1, cap_roots * lay.cap_need[0] * (1 if mode == "fused" else self.S))
        staging = min(staging, part.n_vertices)
        self.feats = ShardedFeatures(part, self.rank, model.D, seed, staging, dtype, self.device)
        n_runners = 1 if mode == "fused" else self.S
        self.runners = [CellRunner(graph, self.feats.table, model, self.fanout, cap_roots,
                                   self.labels, use_tc=use_tc) for _ in range(n_runners)]
        self.table = TraceTable.initial(self.S)
        self.ledger = CommLedger()
        self.stats = FetchStats()
        self.traffic = Traffic()
        self.flat_bytes = model.flat.numel() * 4
        self._recv_p = torch.empty_like(model.flat) if mode == "faithful" else None
        self._recv_g = torch.empty_like(model.grad) if mode == "faithful" else None

    # ------------------------------------------------------------ epoch
    def begin_epoch(self, epoch: int) -> int:
        n = self.graph.n_vertices
        perm = epoch_permutation(self.seed, epoch, n, self.device)
        self.perm = perm.cpu().numpy()
        self.epoch = epoch
        self.iters = iterations_per_epoch(n, self.S, self.B, self.iter_cap)
        return self.iters

    def batches(self, it: int):
        n = len(self.perm)
        out = []
        for d in range(self.S):
            lo = min((it * self.S + d) * self.B, n)
            out.append(self.perm[lo:min(lo + self.B, n)])
        return out

    def _stage(self, runner: CellRunner, roots: np.ndarray, it: int) -> int:
        st = np.uint64(chain(self.sampler_seed, self.epoch, it)).view(np.int64)
        runner.stage_roots(torch.from_numpy(np.ascontiguousarray(roots)), [st], max(len(roots), 1))
        return len(roots)

    # ------------------------------------------------------------ iteration
    def step(self, it: int) -> float:
        """One iteration (engine.py:569-622).  Returns this rank's summed loss."""
        S, rank = self.S, self.rank
        batches = self.batches(it)
        home = self.part.home
        groups = [tuple(b[home[b] == s] for s in range(S)) for b in batches]
        cells = assign_cell_roots(self.table, groups, chain(self.seed, SEED_MERGE, self.epoch, it))
        self.table.root_counts = cell_counts(cells)
        tt = self.table
        cols = tt.n_columns
        mine = []  # (column, model, roots) trained on this GPU
        for j in range(cols):
            d = tt.model_at(rank, j)
            mine.append((j, d, cells[d][j]))
        s = torch.cuda.current_stream(self.device).cuda_stream
        loss = 0.0
        if self.mode == "fused":
            r = self.runners[0]
            roots = np.concatenate([c for _, _, c in mine]) if mine else np.empty(0, np.int64)
            n = self._stage(r, roots, it)
            if n:
                r.builder.build(self.graph, r.roots, r.keys, n, n_roots=n, stream=s)
            self._exchange([r] if n else [], [n])
            if n:
                _lib.call("hg_train_step", C.byref(r.desc), n, s)
                loss = float(r.loss[:n].sum().item())
        else:
            active = []
            for (j, d, roots), r in zip(mine, self.runners):
                n = self._stage(r, roots, it)
                if n:
                    r.builder.build(self.graph, r.roots, r.keys, n, n_roots=n, stream=s)
                active.append(n)
            self._exchange([r for r, n in zip(self.runners, active) if n],
                           [n for n in active if n])
            for idx, ((j, d, roots), r) in enumerate(zip(mine, self.runners)):
                n = active[idx]
                if n:
                    _lib.call("hg_train_step", C.byref(r.desc), n, s)
                    loss += float(r.loss[:n].sum().item())
                if j + 1 < cols:
                    self._hop(int(tt.server_of[0, j + 1] - tt.server_of[0, j]) % S)
        self._account_hops_and_sync()
        # synchronous update: all-reduce the accumulators, then SGD (model.py:299-324)
        if S > 1:
            dist.all_reduce(self.model.grad, group=self.group)
            self.traffic.allreduce_bytes += 2.0 * (S - 1) / S * self.flat_bytes
        self.model.sgd(self.lr, sum(len(b) for b in batches), stream=s)
        return loss

    def _exchange(self, runners, counts):
        need = []
        for r in runners:
            n0 = int(r.builder.tensors["totals"][0].item())
            need.append(r.builder.tensors["need_ids"][0][:n0])
        if self.S == 1:
            return
        per_home, n_req, nbytes, req_bytes = pregather(self.feats, need, self.group)
        for h, c in enumerate(per_home.tolist()):
            if c:
                self.ledger.add(h, self.rank, FEATURE, c * self.model.D * BYTES_PER_ELEM, 1)
        self.stats.transferred += n_req
        self.traffic.feature_rows += n_req
        self.traffic.feature_bytes += nbytes
        self.traffic.request_bytes += req_bytes

    def _hop(self, delta: int):
        """Shift of (parameters, accumulator) by `delta` servers (engine.py:610-618):
        every trace-table column is a uniform shift, so each hop is a ring
        permutation over NVSwitch."""
        S, rank = self.S, self.rank
        nxt, prv = (rank + delta) % S, (rank - delta) % S
        ops = [dist.P2POp(dist.isend, self.model.flat, nxt, self.group),
               dist.P2POp(dist.isend, self.model.grad, nxt, self.group),
               dist.P2POp(dist.irecv, self._recv_p, prv, self.group),
               dist.P2POp(dist.irecv, self._recv_g, prv, self.group)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        if not torch.equal(self._recv_p, self.model.flat):
            raise InvariantViolation("replicas diverged during migration")
        self.model.grad.copy_(self._recv_g)
        self.traffic.hop_bytes += 2 * self.flat_bytes

    def _account_hops_and_sync(self):
        """Reference ledger entries this rank owns: MODEL+GRADIENT per hop
        arriving here (engine.py:610-618) and the ring all-reduce link leaving
        here (model.py:325-328)."""
        tt, S, rank = self.table, self.S, self.rank
        pb = self.model.param_bytes
        for j in range(tt.n_columns - 1):
            for d in range(tt.n_models):
                if int(tt.server_of[d, j + 1]) == rank:
                    src = int(tt.server_of[d, j])
                    self.ledger.add(src, rank, MODEL, pb, 1)
                    self.ledger.add(src, rank, GRADIENT, pb, 1)
        if S > 1:
            self.ledger.add(rank, (rank + 1) % S, GRADIENT, 2.0 * (S - 1) / S * pb, 2 * (S - 1))

    def global_ledger(self) -> CommLedger:
        """Merge every rank's ledger (collective)."""
        if not dist.is_initialized() or self.S == 1:
            return self.ledger
        parts = [None] * self.S
        dist.all_gather_object(parts, self.ledger.counters, group=self.group)
        out = CommLedger()
        for p in parts:
            other = CommLedger()
            other.counters = p
            out.merge(other)
        return out


def model_centric_feature_rows(trainer: MicrographTrainer, it: int):
    """Bytes denominator: rows model d = rank would fetch under model-centric
    training (engine.py:490-498: fetch unique remote vertices of its whole
    batch).  Returns rows per home (np.int64[S])."""
    S, rank = trainer.S, trainer.rank
    b = trainer.batches(it)[rank]
    r = trainer.runners[0]
    n = trainer._stage(r, b, it)
    s = torch.cuda.current_stream(trainer.device).cuda_stream
    r.builder.build(trainer.graph, r.roots, r.keys, n, n_roots=n, stream=s)
    n0 = int(r.builder.tensors["totals"][0].item())
    ids = torch.unique(r.builder.tensors["need_ids"][0][:n0].long())
    h = trainer.feats.home[ids].long()
    counts = torch.bincount(h, minlength=S).cpu().numpy()
    counts[rank] = 0
    return counts
