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


class PeerFeatures:
    """Feature shards mapped across GPUs through CUDA IPC (no staging copies).

    Each rank owns the rows homed on it in a raw cudaMalloc allocation; IPC
    handles are all-gathered and every rank maps every peer's shard, so the
    layer-1 gather (k_aggregate) reads a remote row directly from its owner's
    HBM over NVLink/NVSwitch: address = peers[home[v]] + local_row[v] * ld.
    """

    def __init__(self, part: PartitionMap, rank: int, dim: int, seed: int, dtype=torch.bfloat16,
                 device="cuda", group=None):
        dev = torch.device(device)
        self.dim, self.ld = dim, (dim + 7) // 8 * 8
        self.dtype, self.device = dtype, dev
        self.rank, self.S = rank, part.n_servers
        self.group = group
        esz = 2 if dtype == torch.bfloat16 else 4
        home = part.home
        local = np.flatnonzero(home == rank).astype(np.int64)
        self.n_local = len(local)
        ptr = C.c_void_p()
        _lib.call("hg_alloc", max(self.n_local, 1) * self.ld * esz, C.byref(ptr))
        self.ptr = ptr.value
        st = feature_state(seed)
        code = 1 if dtype == torch.bfloat16 else 0
        stream = torch.cuda.current_stream(dev).cuda_stream
        if self.n_local:
            contiguous = local[-1] - local[0] + 1 == self.n_local
            ids = None if contiguous else torch.from_numpy(local).to(dev)
            _lib.call("hg_feature_table", ids.data_ptr() if ids is not None else None,
                      int(local[0]) if contiguous else 0, self.n_local, dim, self.ld,
                      st & ((1 << 64) - 1), code, self.ptr, stream)
        # local_row[v] = position of v inside its home's shard (ascending ids)
        local_row = np.empty(len(home), dtype=np.int32)
        for h in range(self.S):
            idx = np.flatnonzero(home == h)
            local_row[idx] = np.arange(len(idx), dtype=np.int32)
        self.local_row = torch.from_numpy(local_row).to(dev)
        self.home = part.home_device(dev)
        torch.cuda.synchronize(dev)
        handle = (C.c_char * 64)()
        _lib.call("hg_ipc_handle", self.ptr, handle)
        handles = [None] * self.S
        if dist.is_initialized() and self.S > 1:
            dist.all_gather_object(handles, bytes(handle), group=group)
        else:
            handles = [bytes(handle)]
        self.opened = []
        ptrs = []
        for h, hb in enumerate(handles):
            if h == rank:
                ptrs.append(self.ptr)
                continue
            p = C.c_void_p()
            buf = (C.c_char * 64).from_buffer_copy(hb)
            _lib.call("hg_ipc_open", buf, C.byref(p))
            self.opened.append(p.value)
            ptrs.append(p.value)
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=dev)
        self.bitmap = torch.zeros((len(home) + 31) // 32, dtype=torch.int32, device=dev)

    def bind(self, runner: CellRunner) -> None:
        """Peer-read mode: the gather kernel loads remote rows over NVLink."""
        d = runner.desc
        d.features = self.ptr
        d.feat_row = self.local_row.data_ptr()
        d.feat_peers = self.peers.data_ptr()
        d.feat_home = self.home.data_ptr()
        d.stage_base = None
        d.stage_row = None
        d.row_handle = None
        d.rank = self.rank

    def alloc_mailbox(self, stage_cap: int) -> None:
        """Allocate this rank's mailbox (signal counters, request list, staging
        rows) and map every peer's (collective: all ranks call it together, at
        trainer setup -- never lazily behind a per-rank root count)."""
        if not hasattr(self, "mbox"):
            dev = self.device
            S, row = self.S, self.ld * (2 if self.dtype == torch.bfloat16 else 4)
            cap = int(stage_cap)
            up = lambda x: (x + 255) // 256 * 256  # noqa: E731
            o_flags, o_done = 0, 8 * S
            o_count = up(16 * S)
            o_list = up(o_count + 16)
            o_staging = up(o_list + 4 * cap)
            total = o_staging + cap * row
            ptr = C.c_void_p()
            _lib.call("hg_alloc", total, C.byref(ptr))
            self.mbox = ptr.value
            self.mb_off = (o_flags, o_done, o_count, o_list, o_staging)
            handle = (C.c_char * 64)()
            _lib.call("hg_ipc_handle", self.mbox, handle)
            handles = [None] * S
            if dist.is_initialized() and S > 1:
                dist.all_gather_object(handles, bytes(handle), group=self.group)
            else:
                handles = [bytes(handle)]
            boxes = []
            for h, hb in enumerate(handles):
                if h == self.rank:
                    boxes.append(self.mbox)
                    continue
                p = C.c_void_p()
                _lib.call("hg_ipc_open", (C.c_char * 64).from_buffer_copy(hb), C.byref(p))
                self.opened.append(p.value)
                boxes.append(p.value)
            self.boxes = torch.tensor(boxes, dtype=torch.int64, device=dev)
            self.stage_cap = cap
            self.row_bytes = row
            self.stage_row = torch.zeros(len(self.local_row), dtype=torch.int32, device=dev)
            self.seq = torch.zeros(1, dtype=torch.int64, device=dev)
            self.stamp = torch.zeros(len(self.local_row), dtype=torch.int32, device=dev)
            self.err = torch.zeros(1, dtype=torch.int32, device=dev)

    def bind_staged(self, runner: CellRunner, stage_cap: int) -> None:
        """Staged mode: remote rows are pre-gathered into local HBM (the staging
        rows of this rank's mailbox) by hg_pregather_push, the gather reads HBM
        only.  The mailbox must already exist (alloc_mailbox)."""
        if not hasattr(self, "mbox"):
            raise InvariantViolation("bind_staged before alloc_mailbox (collective setup)")
        if int(stage_cap) > self.stage_cap:
            raise ValueError(f"staging capacity {stage_cap} > mailbox {self.stage_cap}")
        d = runner.desc
        d.features = self.ptr
        d.feat_row = self.local_row.data_ptr()
        d.feat_peers = None
        d.feat_home = self.home.data_ptr()
        d.stage_base = self.mbox + self.mb_off[4]
        d.stage_row = self.stage_row.data_ptr()
        d.rank = self.rank
        # per-batch row handles of the need[0] entries, resolved after every
        # pre-gather (hg_resolve_rows): the layer-1 gather then does one
        # L2-resident lookup per source row instead of home + staging-row
        # lookups by vertex id
        if getattr(runner, "row_handle", None) is None:
            cap0 = runner.builder.tensors["need_ids"][0].numel()
            runner.row_handle = torch.zeros(cap0, dtype=torch.int32, device=self.device)
        d.row_handle = runner.row_handle.data_ptr()

    def pregather(self, runner: CellRunner, uniq_row_ptr: int, total_ptr: int, stream,
                  it_dev_ptr=None, empty: bool = False) -> None:
        """Owner-side push pre-gather of the runner's remote rows (every rank
        calls it in lock-step).  Ledger counts go to uniq_row_ptr (plus
        *it_dev * S rows when a device cursor is given)."""
        t = runner.builder.tensors
        o = self.mb_off
        if not hasattr(self, "_zero"):
            self._zero = torch.zeros(1, dtype=torch.int32, device=self.device)
        n_ptr = self._zero.data_ptr() if empty else t["totals"].data_ptr()
        _lib.call("hg_pregather_push", t["need_ids"][0].data_ptr(), n_ptr,
                  self.home.data_ptr(), self.rank, self.S, self.local_row.data_ptr(), self.ptr,
                  self.row_bytes, self.stamp.data_ptr(), self.stage_row.data_ptr(),
                  self.stage_cap, self.boxes.data_ptr(), self.mbox, o[0], o[1], o[2], o[3], o[4],
                  uniq_row_ptr, it_dev_ptr, self.S, total_ptr, self.seq.data_ptr(),
                  self.err.data_ptr(), stream)
        if runner.desc.row_handle:
            _lib.call("hg_resolve_rows", t["need_ids"][0].data_ptr(), n_ptr, self.home.data_ptr(),
                      self.rank, self.local_row.data_ptr(), self.stage_row.data_ptr(),
                      runner.desc.row_handle, stream)

    def pregather_group(self, runners, uniq_table_ptr: int, total_ptr: int, stream,
                        it_dev_ptr: int) -> None:
        """Push pre-gather of a run-ahead group (DistGroupLoop): the reference
        ledger is charged per iteration (row *it_dev + 1 + j for runner j, own
        dedup per iteration, featstore.py:226-279), while the rows move in ONE
        deduplicated push with one request/completion handshake; then every
        runner's row handles are resolved against the shared staging map."""
        G = len(runners)
        o = self.mb_off
        ids = (C.c_void_p * G)(*[r.builder.tensors["need_ids"][0].data_ptr() for r in runners])
        ns = (C.c_void_p * G)(*[r.builder.tensors["totals"].data_ptr() for r in runners])
        # per-iteration ledger rows (one account + clear launch per iteration: the
        # one-launch group variant hg_remote_account_group measured 3-4 % slower in
        # the replayed loop -- its wide grid crowds the training branch)
        for j in range(G):
            _lib.call("hg_remote_account_at", ids[j], ns[j], self.home.data_ptr(), self.rank,
                      self.bitmap.data_ptr(), uniq_table_ptr, it_dev_ptr, 1 + j, self.S,
                      total_ptr, stream)
            _lib.call("hg_remote_clear", ids[j], ns[j], 0, self.bitmap.data_ptr(), stream)
        _lib.call("hg_pregather_push_multi", ids, ns, G, self.home.data_ptr(), self.rank, self.S,
                  self.local_row.data_ptr(), self.ptr, self.row_bytes, self.stamp.data_ptr(),
                  self.stage_row.data_ptr(), self.stage_cap, self.boxes.data_ptr(), self.mbox,
                  o[0], o[1], o[2], o[3], o[4], self.seq.data_ptr(), self.err.data_ptr(), stream)
        if all(r.desc.row_handle for r in runners):
            outs = (C.c_void_p * G)(*[r.desc.row_handle for r in runners])
            _lib.call("hg_resolve_rows_group", ids, ns, G, self.home.data_ptr(), self.rank,
                      self.local_row.data_ptr(), self.stage_row.data_ptr(), outs, stream)

    def check(self) -> None:
        """Raise if a push pre-gather gave up waiting on a peer or dropped an
        overflowing staging slot (device flag set by k_pg_wait / k_stage_mark)."""
        err = getattr(self, "err", None)
        if err is None:
            return
        code = int(err.item())
        if code:
            err.zero_()
            _lib.flag_status(code, "hg_pregather_push (peer wait timed out or staging overflow)")

    def close(self):
        for p in self.opened:
            _lib.call("hg_ipc_close", p)
        self.opened = []


# ---------------------------------------------------------------- graph loop



class DistGraphLoop:
    """CUDA-graph replay of the multi-GPU fast path (fused mode, initial trace
    table, NVLink push pre-gather) as a three-stage pipeline over three
    runners.  Replay x (iteration it, x = it % 3) runs three branches:

      build  : stage this rank's roots of it+2 from the device cursor
               (hg_iter_stage_ranged: variable count, at most `cap`) and
               build their micrographs (device root count) into runner x+2;
      gather : pre-gather the remote rows of it+1 (built by the previous
               replay) over NVLink into runner x+1's staging (ledger row from
               a second cursor) and run its layer-1 gather;
      train  : train runner x, copy the summed loss to a pinned slot, NCCL
               all-reduce + SGD (+ bf16 operand refresh).

    so sampling, the cross-GPU exchange and training of three consecutive
    iterations overlap.  Root count capacity `cap` pads with empty
    micrographs, which contribute nothing (zero loss rows and gradients)."""

    def __init__(self, tr: "MicrographTrainer", cap: int):
        self.tr, self.cap = tr, int(cap)
        dev = tr.device
        self.runners = tr.runners[:3]
        # training and the (cross-GPU latency-bound) pre-gather branch at high
        # stream priority, the SM-filling build branch at low priority
        from .engine import _streams
        self._cap_s, self.side_build = _streams(dev)
        self.side_gather = torch.cuda.Stream(dev, priority=-1)
        self.pin_loss = [torch.zeros(1, dtype=torch.float32).pin_memory() for _ in range(3)]
        self._dummy = torch.zeros(2, dtype=torch.int64, device=dev)
        m = tr.model
        total = tr.S * tr.B
        self.graphs = []
        cur = torch.cuda.current_stream(dev)
        before = _lib.launch_count()
        for x in range(3):
            run, nxt, nxt2 = (self.runners[(x + j) % 3] for j in range(3))
            g = torch.cuda.CUDAGraph()
            cap_s = self._cap_s
            cap_s.wait_stream(cur)
            with torch.cuda.graph(g, stream=cap_s):
                self.side_build.wait_stream(cap_s)
                self.side_gather.wait_stream(cap_s)
                with torch.cuda.stream(self.side_build):
                    self.build_ops(nxt2, self.side_build.cuda_stream)
                with torch.cuda.stream(self.side_gather):
                    self.gather_ops(nxt, self.side_gather.cuda_stream)
                cs = cap_s.cuda_stream
                run.desc.lowp_fresh = 1 if run.tc else 0
                _lib.call("hg_train_step", C.byref(run.desc), self.cap, cs)
                run.desc.lowp_fresh = 0
                self.pin_loss[x].copy_(run.loss[:self.cap].sum().reshape(1), non_blocking=True)
                if run.tc:  # SGD refreshes the bf16 operands: steps skip their transposes
                    tr._sync_update(run, cs, refresh=True)
                else:
                    tr._sync_update(None, cs, refresh=False)
                cap_s.wait_stream(self.side_build)
                cap_s.wait_stream(self.side_gather)
            cur.wait_stream(cap_s)
            self.graphs.append(g)
        self.launches = (_lib.launch_count() - before) // 3
        self.iters = tr.iters

    def build_ops(self, r: CellRunner, s) -> None:
        """Build cursor -> cursor + 1: stage and build that iteration into r."""
        tr = self.tr
        _lib.call("hg_iter_stage_ranged", tr._g_roots.data_ptr(), tr._g_ranges.data_ptr(),
                  tr._g_states.data_ptr(), tr.iters, tr._g_it.data_ptr(), self.cap, 1, 1,
                  r.roots.data_ptr(), r.n_dev.data_ptr(), r.keys.data_ptr(), s)
        r.builder.build(tr.graph, r.roots.data_ptr(), r.keys.data_ptr(), self.cap,
                        n_roots=self.cap, stream=s, n_dev=r.n_dev.data_ptr())

    def gather_ops(self, r: CellRunner, s) -> None:
        """Gather cursor -> cursor + 1: pre-gather (ledger row = that iteration)
        and the layer-1 gather of runner r, already built."""
        tr = self.tr
        # advance the gather cursor (cap 0: nothing staged)
        _lib.call("hg_iter_stage_ranged", tr._g_roots.data_ptr(), tr._g_ranges.data_ptr(),
                  tr._g_states.data_ptr(), tr.iters, tr._g_pg.data_ptr(), 0, 1, 1,
                  self._dummy.data_ptr(), self._dummy.data_ptr(),
                  self._dummy.data_ptr() + 8, s)
        tr.feats.pregather(r, tr._acct_rows.data_ptr(), tr._acct_total.data_ptr(), s,
                           it_dev_ptr=tr._g_pg.data_ptr())
        _lib.call("hg_step_prologue", C.byref(r.desc), self.cap, 1, s)

    def replay(self, x: int) -> None:
        self.graphs[x].replay()


class DistGroupLoop:
    """DistGraphLoop over groups of G iterations (the N > 1 counterpart of
    engine.GroupLoop).  Three sets of G runners rotate; replay x trains group
    g (set x: G train steps, each followed by the NCCL all-reduce + SGD),
    pre-gathers and layer-1-gathers group g+1 iteration by iteration (set
    x+1; the mailbox staging is reused per iteration, the ledger row follows
    the gather cursor) and stages + builds group g+2 in ONE launch (set x+2,
    hg_mg_build_group with per-batch device root counts, persistent grid
    beside the other branches).  Semantics are those of DistGraphLoop."""

    def __init__(self, tr: "MicrographTrainer", cap: int, G: int):
        from .engine import BUILD_CTAS_PER_SM, _streams
        from .sampler import GroupBuilder
        self.tr, self.cap, self.G = tr, int(cap), int(G)
        dev = tr.device
        mk = lambda: CellRunner(tr.graph, tr.runners[0].table, tr.model, tr.fanout,  # noqa: E731
                                tr.runners[0].max_roots, tr.labels)
        self.sets = [[mk() for _ in range(G)] for _ in range(3)]
        self.gb = [GroupBuilder([r.builder for r in st], per_batch=self.cap) for st in self.sets]
        self.descp = [(C.POINTER(_lib.StepDesc) * G)(*[C.pointer(r.desc) for r in st])
                      for st in self.sets]
        for st, gb in zip(self.sets, self.gb):
            for j, r in enumerate(st):
                tr.feats.bind_staged(r, tr._stage_cap)
                r.desc.roots = gb.roots_ptr(j)
                r.desc.agg1_ready = 1
        self.ctas_per_sm = BUILD_CTAS_PER_SM
        cap_s, self.side_build = _streams(dev)
        self.side_gather = torch.cuda.Stream(dev)
        self.pin_loss = [torch.zeros(1, dtype=torch.float32).pin_memory() for _ in range(3)]
        self._dummy = torch.zeros(2, dtype=torch.int64, device=dev)
        m = tr.model
        total = tr.S * tr.B
        self.graphs = []
        cur = torch.cuda.current_stream(dev)
        before = _lib.launch_count()
        for x in range(3):
            run, nxt, nxt2 = (self.sets[(x + j) % 3] for j in range(3))
            g = torch.cuda.CUDAGraph()
            cap_s.wait_stream(cur)
            with torch.cuda.graph(g, stream=cap_s):
                self.side_build.wait_stream(cap_s)
                self.side_gather.wait_stream(cap_s)
                with torch.cuda.stream(self.side_build):
                    self.build_ops((x + 2) % 3, self.side_build.cuda_stream)
                with torch.cuda.stream(self.side_gather):
                    self.gather_ops((x + 1) % 3, self.side_gather.cuda_stream)
                cs = cap_s.cuda_stream
                for r in run:
                    r.desc.lowp_fresh = 1 if r.tc else 0
                    _lib.call("hg_train_step", C.byref(r.desc), self.cap, cs)
                    r.desc.lowp_fresh = 0
                    if r.tc:
                        tr._sync_update(r, cs, refresh=True)
                    else:
                        tr._sync_update(None, cs, refresh=False)
                self.pin_loss[x].copy_(torch.stack([r.loss[:self.cap].sum() for r in run])
                                       .sum().reshape(1), non_blocking=True)
                cap_s.wait_stream(self.side_build)
                cap_s.wait_stream(self.side_gather)
            cur.wait_stream(cap_s)
            self.graphs.append(g)
        self.launches = (_lib.launch_count() - before) // 3
        self.iters = tr.iters

    def build_ops(self, k: int, s, ctas_per_sm: int = None) -> None:
        """Build cursor+1 .. cursor+G into set k; the cursor moves by G."""
        tr, gb, G = self.tr, self.gb[k], self.G
        for j in range(G):
            _lib.call("hg_iter_stage_ranged", tr._g_roots.data_ptr(), tr._g_ranges.data_ptr(),
                      tr._g_states.data_ptr(), tr.iters, tr._g_it.data_ptr(), self.cap, 1 + j,
                      G if j == G - 1 else 0, gb.roots_ptr(j), gb.n_dev.data_ptr() + 4 * j,
                      gb.keys.data_ptr() + 8 * j, s)
        gb.build(tr.graph, stream=s, n_dev=gb.n_dev.data_ptr(),
                 ctas_per_sm=self.ctas_per_sm if ctas_per_sm is None else ctas_per_sm)

    def gather_ops(self, k: int, s) -> None:
        """Pre-gather set k's G iterations in one push (ledger rows per
        iteration, cursor+1 .. cursor+G), advance the gather cursor by G, and
        run each iteration's layer-1 gather from the shared staging."""
        tr = self.tr
        tr.feats.pregather_group(self.sets[k], tr._acct_rows.data_ptr(),
                                 tr._acct_total.data_ptr(), s, tr._g_pg.data_ptr())
        _lib.call("hg_iter_stage_ranged", tr._g_roots.data_ptr(), tr._g_ranges.data_ptr(),
                  tr._g_states.data_ptr(), tr.iters, tr._g_pg.data_ptr(), 0, self.G, self.G,
                  self._dummy.data_ptr(), self._dummy.data_ptr(),
                  self._dummy.data_ptr() + 8, s)
        # the group's layer-1 gathers in ONE launch (per-batch row handles)
        _lib.call("hg_step_prologue_group", self.descp[k], self.G, 1, s)

    def replay(self, x: int) -> None:
        self.graphs[x].replay()

    def run_eager(self, it: int, s) -> None:
        """One replay's work for iterations it..it+G-1 launched eagerly on stream
        s, branch after branch (build the group, pre-gather + grouped layer-1
        gather, then the G train steps with all-reduce + SGD): the profiling
        pass of bench.py, where per-kernel CUDA-event sites need real launches.
        Collective: every rank runs it for the same `it`.  Leaves the loop
        unpositioned (the next step re-positions it)."""
        tr = self.tr
        tr._g_it.fill_(it - 1)
        tr._g_pg.fill_(it - 1)
        self.build_ops(0, s)
        self.gather_ops(0, s)
        m = tr.model
        total = tr.S * tr.B
        r0 = self.sets[0][0]
        if r0.tc:  # operands current before the first step (the replays leave them so)
            _lib.call("hg_sgd_refresh", C.byref(r0.desc), m.flat.data_ptr(), m.grad.data_ptr(),
                      m.flat.numel(), 0.0, 1.0, 0, s)
        for r in self.sets[0]:
            if r.tc:
                r.desc.lowp_fresh = 1
                _lib.call("hg_train_step", C.byref(r.desc), self.cap, s)
                r.desc.lowp_fresh = 0
                tr._sync_update(r, s, refresh=True)
            else:
                _lib.call("hg_train_step", C.byref(r.desc), self.cap, s)
                tr._sync_update(None, s, refresh=False)
        tr._gnext = None
        tr._gdone = None

    def check(self) -> None:
        for gb in self.gb:
            gb.check()


# ---------------------------------------------------------------- trainer

class MicrographTrainer:
    """One rank of the HopGNN micrograph strategy (+ pre-gathering)."""

    def __init__(self, graph: Graph, part: PartitionMap, model: ModelState, fanout, batch: int,
                 seed: int, lr: float = 0.1, dtype=torch.bfloat16, mode: str = "fused",
                 iterations: int = 0, group=None, use_tc: bool = True, pregather: bool = True,
                 strategy: str = "micrograph", graphs: bool = True, graph_group: int = 1,
                 allreduce: str = "p2p"):
        """strategy="micrograph": HopGNN feature-centric training (engine.py:562-623);
        "model-centric": the baseline it is measured against (engine.py:482-507) --
        GPU d trains all of batch d, fetching every remote row its micrographs
        need, no hops, same all-reduce.  pregather=True: iteration-scoped dedup staging over NCCL all-to-all (the
        paper's pre-gathering).  pregather=False: remote rows are read in place from
        the owner GPU over NVLink by the gather kernel (PeerFeatures); the ledger
        still charges the reference's deduplicated pre-gather bytes."""
        if mode not in ("fused", "faithful"):
            raise ValueError("mode must be 'fused' or 'faithful'")
        if strategy not in ("micrograph", "model-centric"):
            raise ValueError("strategy must be 'micrograph' or 'model-centric'")
        if allreduce not in ("p2p", "nccl"):
            raise ValueError("allreduce must be 'p2p' or 'nccl'")
        if strategy == "model-centric":
            mode = "fused"  # one cell per GPU, nothing to hop
        self.strategy = strategy
        self.pregather = pregather
        self.graphs = graphs
        self._dgl = None       # DistGraphLoop / DistGroupLoop
        # iterations per graph replay (DistGroupLoop when > 1)
        self.graph_group = max(1, min(int(graph_group), _lib.MAX_GROUP))
        self._gdone = None     # iterations < _gdone are already enqueued by a group replay
        self._gnext = None     # iteration the graph loop is positioned at
        self._eager_fast = 0   # eager fast-path steps taken (library warm-up before capture)
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
        if strategy == "model-centric":
            cap_roots = self.B
        staging = max(1, cap_roots * lay.cap_need[0] * (1 if mode == "fused" else self.S))
        staging = min(staging, part.n_vertices)
        n_runners = 1 if mode == "fused" else self.S
        if pregather:
            self.feats = ShardedFeatures(part, self.rank, model.D, seed, staging, dtype,
                                         self.device)
            table = self.feats.table
        else:
            self.feats = PeerFeatures(part, self.rank, model.D, seed, dtype, self.device, group)
            table = FeatureTable(1, model.D, dtype, self.device, model.Dp)  # shape carrier
        self.runners = [CellRunner(graph, table, model, self.fanout, cap_roots,
                                   self.labels, use_tc=use_tc) for _ in range(n_runners)]
        # load the loss-sum reduction kernel now (lazy module loading costs ~10 ms
        # on its first launch, which would otherwise land inside a timed step)
        self.runners[0].loss[:1].sum().item()
        if not pregather:
            for r in self.runners:
                self.feats.bind(r)
            # the push pre-gather's mailbox is set up collectively here; a group
            # push stages the distinct remote rows of graph_group iterations
            lay0 = self.runners[0].builder.layout
            self._stage_cap = min(self.runners[0].max_roots * lay0.cap_need[0]
                                  * self.graph_group, self.part.n_vertices)
            self.feats.alloc_mailbox(self._stage_cap)
        # device-side per-iteration pre-gather accounting (peer mode): [iter][home]
        self._acct_rows = None
        self._acct_total = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.table = TraceTable.initial(self.S)
        self.ledger = CommLedger()
        self.stats = FetchStats()
        self.traffic = Traffic()
        self.flat_bytes = model.flat.numel() * 4
        # pinned loss slots for the pipelined readback (allocated up front:
        # pinning costs ~10 ms, never inside a step)
        self._loss_pin = [torch.zeros(1, dtype=torch.float32).pin_memory() for _ in range(4)]
        self._loss_slot = 0
        self._loss_pending = []
        self._recv_p = torch.empty_like(model.flat) if mode == "faithful" else None
        self._recv_g = torch.empty_like(model.grad) if mode == "faithful" else None
        self._hop_err = torch.zeros(1, dtype=torch.int32, device=self.device)
        # our own NCCL communicator for the in-C all-reduce+SGD (and hops)
        self._comm = None
        self._comm_ok = True
        if self.S > 1:
            try:
                uid = (C.c_char * 128)()
                if self.rank == 0:
                    _lib.call("hg_nccl_unique_id", uid)
                obj = [bytes(uid)]
                dist.broadcast_object_list(obj, src=0, group=group)
                buf = (C.c_char * 128).from_buffer_copy(obj[0])
                comm = C.c_void_p()
                _lib.call("hg_nccl_init", buf, self.S, self.rank, C.byref(comm))
                self._comm = comm.value
            except RuntimeError:
                self._comm_ok = False  # fall back to torch.distributed collectives
        # gradient all-reduce of the fast paths: NVLink peer memory (default) or NCCL
        self._ar = None
        if self.S > 1 and allreduce == "p2p" and self._comm_ok and self._comm is not None:
            self._setup_p2p_allreduce()

    # ------------------------------------------------------------ epoch
    def begin_epoch(self, epoch: int) -> int:
        n = self.graph.n_vertices
        perm = epoch_permutation(self.seed, epoch, n, self.device)
        self.perm = perm.cpu().numpy()
        self.epoch = epoch
        self.iters = iterations_per_epoch(n, self.S, self.B, self.iter_cap)
        self._plan_epoch()
        if self._graph_eligible():
            self._graph_epoch_plan()
        return self.iters

    # ------------------------------------------------------------ graph loop
    def _graph_eligible(self) -> bool:
        return (self.graphs and self.S > 1 and self.mode == "fused" and not self.pregather
                and self._comm_ok and self._comm is not None)

    def _graph_epoch_plan(self) -> None:
        """Device copies of this epoch's root ranges / stream states for the graph
        loop's cursor, at fixed addresses (captured once)."""
        S, B, it_n = self.S, self.B, self.iters
        its = np.arange(it_n, dtype=np.int64)
        if self.strategy == "model-centric":
            roots = self.perm
            lo = (its * S + self.rank) * B
            ranges = np.stack([lo, lo + B], axis=1)
            cap = B
        else:
            roots = self._my_roots
            b = np.asarray(self._my_bounds, dtype=np.int64)
            ranges = np.stack([b[:-1], b[1:]], axis=1)
            cap = int((ranges[:, 1] - ranges[:, 0]).max()) if it_n else 1
            cap = min(-(-max(cap, 1) // 64) * 64, self.runners[0].max_roots)
        states = hash_vec(chain(self.sampler_seed, self.epoch), its).view(np.int64)
        dev = self.device
        fresh = (not hasattr(self, "_g_roots") or self._g_roots.numel() != len(roots)
                 or self._g_ranges.shape[0] != it_n)
        if fresh:
            self._g_roots = torch.empty(len(roots), dtype=torch.int64, device=dev)
            self._g_ranges = torch.empty((it_n, 2), dtype=torch.int64, device=dev)
            self._g_states = torch.empty(it_n, dtype=torch.int64, device=dev)
            self._g_it = torch.zeros(1, dtype=torch.int64, device=dev)
            self._g_pg = torch.zeros(1, dtype=torch.int64, device=dev)
            self._dgl = None
        self._g_roots.copy_(torch.from_numpy(np.ascontiguousarray(roots)))
        self._g_ranges.copy_(torch.from_numpy(np.ascontiguousarray(ranges)))
        self._g_states.copy_(torch.from_numpy(np.ascontiguousarray(states)))
        if self._dgl is not None and (self._dgl.cap < cap or self._dgl.iters != it_n):
            self._dgl = None
        self._g_cap = cap if self._dgl is None else self._dgl.cap
        self._acct_row_ptr(it_n - 1)
        self._gnext = None
        self._gdone = None

    def _graph_loop(self):
        if self._dgl is None:
            if self._eager_fast < 2 or not hasattr(self, "_ra"):
                return None
            self._drain_run_ahead()
            while len(self.runners) < 3:  # a third runner for the three-stage pipeline
                self.runners.append(CellRunner(self.graph, self.runners[0].table, self.model,
                                               self.fanout, self.runners[0].max_roots,
                                               self.labels))
            for r in self.runners[:3]:
                r.desc.roots = r.roots.data_ptr()
                r.desc.agg1_ready = 1
                self.feats.bind_staged(r, self._stage_cap)
            if self.graph_group > 1:
                self._dgl = DistGroupLoop(self, self._g_cap, self.graph_group)
            else:
                self._dgl = DistGraphLoop(self, self._g_cap)
        return self._dgl

    def _drain_run_ahead(self) -> None:
        if hasattr(self, "_ra"):
            self._ra.side.wait_stream(torch.cuda.current_stream(self.device))
            self._ra.reset()

    def _step_graph(self, gl: DistGraphLoop, it: int, want_loss: bool):
        x = it % 3
        if self._gnext != it:
            # position the pipeline: `it` built + pre-gathered + layer-1 gathered
            # into runner x, it+1 built into runner x+1 (eagerly, on this stream)
            self._drain_run_ahead()
            for r in gl.runners:  # the general cell path may have rebound these
                r.desc.roots = r.roots.data_ptr()
                r.desc.agg1_ready = 1
                self.feats.bind_staged(r, self._stage_cap)
            # an eager run-ahead build of `it` may already have charged its ledger row
            self._acct_rows[it].zero_()
            cs = torch.cuda.current_stream(self.device).cuda_stream
            self._g_it.fill_(it - 1)
            self._g_pg.fill_(it - 1)
            gl.build_ops(gl.runners[x], cs)
            gl.gather_ops(gl.runners[x], cs)
            gl.build_ops(gl.runners[(x + 1) % 3], cs)
            if gl.runners[x].tc:  # replays start from bf16 operands matching the parameters
                m = self.model
                _lib.call("hg_sgd_refresh", C.byref(gl.runners[x].desc), m.flat.data_ptr(),
                          m.grad.data_ptr(), m.flat.numel(), 0.0, 1.0, 0, cs)
            self._acct_iters = getattr(self, "_acct_iters", set())
            self._acct_iters.add(it)
        prev = None
        # pin slot x was written by the replay three steps back: read it before reuse
        while self._loss_pending and any(b is gl.pin_loss[x] for _, b in self._loss_pending):
            prev = self._drain_loss()
        gl.replay(x)  # trains `it`, pre-gathers it+1, builds it+2, all-reduce + SGD
        ev = torch.cuda.Event()
        ev.record()
        self._loss_pending.append((ev, gl.pin_loss[x]))
        if want_loss and prev is None and len(self._loss_pending) > 2:
            prev = self._drain_loss()
        if not want_loss:
            prev = None
        self._acct_iters = getattr(self, "_acct_iters", set())
        self._acct_iters.add(it + 1)
        self._fast_iters = getattr(self, "_fast_iters", 0) + 1
        self.traffic.allreduce_bytes += 2.0 * (self.S - 1) / self.S * self.flat_bytes
        self._gnext = it + 1
        return prev

    def _step_group(self, gl: "DistGroupLoop", it: int, want_loss: bool):
        """Group replay: trains it..it+G-1, gathers the next group, builds the
        one after (see DistGroupLoop)."""
        G = gl.G
        if self._gnext != it:
            # position: group it built + pre-gathered + gathered into set 0,
            # group it+G built into set 1 (eagerly, on this stream)
            self._drain_run_ahead()
            for st, gb in zip(gl.sets, gl.gb):
                for j, r in enumerate(st):
                    r.desc.roots = gb.roots_ptr(j)
                    r.desc.agg1_ready = 1
                    self.feats.bind_staged(r, self._stage_cap)
            for j in range(it, min(it + G, self.iters)):
                self._acct_rows[j].zero_()  # an eager run-ahead may have charged these
            cs = torch.cuda.current_stream(self.device).cuda_stream
            self._g_it.fill_(it - 1)
            self._g_pg.fill_(it - 1)
            gl.build_ops(0, cs, ctas_per_sm=0)
            gl.gather_ops(0, cs)
            gl.build_ops(1, cs, ctas_per_sm=0)
            r0 = gl.sets[0][0]
            if r0.tc:  # replays start from bf16 operands matching the parameters
                m = self.model
                _lib.call("hg_sgd_refresh", C.byref(r0.desc), m.flat.data_ptr(),
                          m.grad.data_ptr(), m.flat.numel(), 0.0, 1.0, 0, cs)
            self._acct_iters = getattr(self, "_acct_iters", set())
            self._acct_iters.update(range(it, min(it + G, self.iters)))
            self._gx = 0
        x = self._gx
        prev = None
        while self._loss_pending and any(b is gl.pin_loss[x] for _, b in self._loss_pending):
            prev = self._drain_loss()
        gl.replay(x)  # trains it..it+G-1, gathers the next group, builds the one after
        ev = torch.cuda.Event()
        ev.record()
        self._loss_pending.append((ev, gl.pin_loss[x]))
        if want_loss and prev is None and len(self._loss_pending) > 2:
            prev = self._drain_loss()
        if not want_loss:
            prev = None
        self._acct_iters = getattr(self, "_acct_iters", set())
        self._acct_iters.update(range(it + G, min(it + 2 * G, self.iters)))
        self._fast_iters = getattr(self, "_fast_iters", 0) + G
        self.traffic.allreduce_bytes += G * 2.0 * (self.S - 1) / self.S * self.flat_bytes
        self._gx = (x + 1) % 3
        self._gnext = self._gdone = it + G
        return prev

    def batches(self, it: int):
        n = len(self.perm)
        out = []
        for d in range(self.S):
            lo = min((it * self.S + d) * self.B, n)
            out.append(self.perm[lo:min(lo + self.B, n)])
        return out

    def _stage(self, runner: CellRunner, roots: np.ndarray, it: int) -> int:
        """Roots + iteration key into the runner's device buffers through a
        ring of pinned host buffers (asynchronous H2D, no stream sync)."""
        if not hasattr(self, "_pin"):
            cap = max(r.max_roots for r in self.runners) + 1
            self._pin = [torch.empty(cap, dtype=torch.int64).pin_memory() for _ in range(8)]
            self._pin_ev = [None] * 8
            self._pin_i = 0
        i = self._pin_i
        self._pin_i = (i + 1) % 8
        if self._pin_ev[i] is not None:
            self._pin_ev[i].synchronize()
        buf = self._pin[i]
        n = len(roots)
        buf[0] = int(np.uint64(chain(self.sampler_seed, self.epoch, it)).view(np.int64))
        if n:
            buf[1:n + 1].numpy()[:] = roots
        runner.keys[:1].copy_(buf[:1], non_blocking=True)
        if n:
            runner.roots[:n].copy_(buf[1:n + 1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._pin_ev[i] = ev
        runner.n_roots, runner.roots_per_state = n, max(n, 1)
        # general (host-planned) path: roots live in the runner, layer 1 is
        # gathered by the step itself, remote rows are read in place
        runner.desc.roots = runner.roots.data_ptr()
        runner.desc.agg1_ready = 0
        if not self.pregather:
            self.feats.bind(runner)
        return n

    # ------------------------------------------------------------ fast path
    def _plan_epoch(self) -> None:
        """Per-epoch host plan for the initial trace table: with cells[d][t] =
        groups[d][(d+t)%S] every root homed at this server is trained here, so
        iteration it's roots are a contiguous slice of perm[home[perm]==rank]."""
        S, B = self.S, self.B
        home_perm = self.part.home[self.perm]
        pos = np.flatnonzero(home_perm == self.rank)
        self._my_roots = np.ascontiguousarray(self.perm[pos])
        self._my_bounds = np.searchsorted(pos, np.arange(self.iters + 1, dtype=np.int64) * S * B)

    def _stage_ring(self, roots: np.ndarray, it: int):
        """One async H2D of [iteration key, roots...] through a pinned/device
        buffer ring; returns (roots_ptr, keys_ptr) on the device."""
        if not hasattr(self, "_ring_h"):
            cap = max(r.max_roots for r in self.runners) + 1
            self._ring_h = torch.empty((8, cap), dtype=torch.int64).pin_memory()
            self._ring_d = torch.empty((8, cap), dtype=torch.int64, device=self.device)
            self._ring_ev = [None] * 8
            self._ring_i = 0
        i = self._ring_i
        self._ring_i = (i + 1) % 8
        if self._ring_ev[i] is not None:
            self._ring_ev[i].synchronize()
        h = self._ring_h[i].numpy()
        n = len(roots)
        h[0] = np.uint64(chain(self.sampler_seed, self.epoch, it)).view(np.int64)
        h[1:n + 1] = roots
        self._ring_d[i, :n + 1].copy_(self._ring_h[i, :n + 1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._ring_ev[i] = ev
        base = self._ring_d[i].data_ptr()
        return base + 8, base

    def _iter_roots(self, it: int) -> np.ndarray:
        """Roots this GPU trains in iteration `it` under the initial table."""
        if self.strategy == "model-centric":
            lo = (it * self.S + self.rank) * self.B
            return self.perm[lo:lo + self.B]
        return self._my_roots[self._my_bounds[it]:self._my_bounds[it + 1]]

    def _fast_build(self, it: int):
        roots = self._iter_roots(it)
        n = len(roots)

        def launch(r, s):
            r.n_roots = n
            if not n:
                if not self.pregather:
                    # the push pre-gather is collective: take part with no requests
                    self.feats.pregather(r, self._acct_rows[it].data_ptr(),
                                         self._acct_total.data_ptr(), s, empty=True)
                return
            rp, kp = self._stage_ring(roots, it)
            r.builder.build(self.graph, rp, kp, n, n_roots=n, stream=s)
            r.desc.roots = rp
            if not self.pregather:
                self.feats.bind_staged(r, self._stage_cap)
                # device pre-gather of the remote rows (NVLink bulk copies) and the
                # parameter-independent layer-1 gather, both ahead of training
                self._acct_row_ptr(it)
                self.feats.pregather(r, self._acct_rows[it].data_ptr(),
                                     self._acct_total.data_ptr(), s)
                _lib.call("hg_step_prologue", C.byref(r.desc), n, 1, s)
                r.desc.agg1_ready = 1
                self._acct_iters = getattr(self, "_acct_iters", set())
                self._acct_iters.add(it)
        return launch

    def _acct_row_ptr(self, it: int) -> None:
        if self._acct_rows is None or self._acct_rows.shape[0] <= it:
            rows = max(it + 1, getattr(self, "iters", 1))
            t = torch.zeros((rows, self.S), dtype=torch.int64, device=self.device)
            if self._acct_rows is not None:
                t[:self._acct_rows.shape[0]] = self._acct_rows
            self._acct_rows = t

    def _step_fast(self, it: int, want_loss: bool):
        """Fused micrograph iteration without host synchronisation: build (+
        pre-gather accounting) of it+1 runs ahead on a side stream, training
        of it reads remote rows over NVLink, then all-reduce + SGD in C."""
        S = self.S
        s = torch.cuda.current_stream(self.device).cuda_stream
        self._eager_fast += 1
        if self._gnext is not None:
            if self._gnext == it and isinstance(self._dgl, DistGraphLoop):
                # the graph loop already built `it` into runner it%3: train it here
                return self._train_built(self._dgl.runners[it % 3], it, want_loss)
            self._drain_run_ahead()
            self._gnext = None
        if self.pregather:  # staging exchange needs host-known sizes: no run-ahead
            r = self.runners[0]
            self._fast_build(it)(r, s)
            # collective: a rank with no roots this iteration still takes part
            self._exchange([r] if r.n_roots else [], [r.n_roots], it)
        else:
            if not hasattr(self, "_ra"):
                from .engine import RunAhead
                self.runners.append(CellRunner(self.graph, self.runners[0].table, self.model,
                                               self.fanout, self.runners[0].max_roots,
                                               self.labels))
                self._ra = RunAhead(self.runners[:2], self.device)
            r = self._ra.acquire(it, self._fast_build(it))
        n = r.n_roots
        prev = None
        if n:
            _lib.call("hg_train_step", C.byref(r.desc), n, s)
            if want_loss:  # pipelined readback: this step's loss arrives next call
                self._loss_slot = (self._loss_slot + 1) % 4
                self._loss_pin[self._loss_slot].copy_(r.loss[:n].sum().reshape(1),
                                                      non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
                # values are read two steps late so the host never stalls the queue
                if len(self._loss_pending) >= 2:
                    prev = self._drain_loss()
                self._loss_pending.append((ev, self._loss_pin[self._loss_slot]))
        self._fast_iters = getattr(self, "_fast_iters", 0) + 1
        self._sync_update(None, s, refresh=False)
        if not self.pregather:
            self._ra.release(it)
            if it + 1 < self.iters:
                self._ra.prefetch(it + 1, self._fast_build(it + 1))
        if S > 1:
            self.traffic.allreduce_bytes += 2.0 * (S - 1) / S * self.flat_bytes
        return prev

    def _train_built(self, r: CellRunner, it: int, want_loss: bool):
        """Eagerly train a runner the graph loop built (the epoch's last iteration)."""
        self._gnext = None
        self._drain_run_ahead()
        s = torch.cuda.current_stream(self.device).cuda_stream
        cap = self._dgl.cap
        _lib.call("hg_train_step", C.byref(r.desc), cap, s)
        prev = None
        if want_loss:
            self._loss_slot = (self._loss_slot + 1) % 4
            self._loss_pin[self._loss_slot].copy_(r.loss[:cap].sum().reshape(1), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            if len(self._loss_pending) >= 2:
                prev = self._drain_loss()
            self._loss_pending.append((ev, self._loss_pin[self._loss_slot]))
        self._sync_update(None, s, refresh=False)
        self._fast_iters = getattr(self, "_fast_iters", 0) + 1
        self.traffic.allreduce_bytes += 2.0 * (self.S - 1) / self.S * self.flat_bytes
        return prev

    def _drain_loss(self):
        pend = getattr(self, "_loss_pending", None)
        if not pend:
            return None
        ev, buf = pend.pop(0)
        ev.synchronize()
        return float(buf.item())

    def last_loss(self):
        """Drain every pending step loss; returns the most recent (host sync)."""
        v = None
        while getattr(self, "_loss_pending", None):
            v = self._drain_loss()
        return v

    # ------------------------------------------------------------ iteration
    def step(self, it: int, want_loss: bool = True):
        """One iteration (engine.py:569-622).  Returns this rank's summed loss
        (a host sync) or None when want_loss is False."""
        if (self.mode == "fused" and (not self.table.removed or self.strategy == "model-centric")
                and self._comm_ok and len(self.perm) >= (it + 1) * self.S * self.B):
            G = self.graph_group
            if G > 1:
                if self._gdone is not None and self._gdone - G <= it < self._gdone:
                    return None  # enqueued by the last group replay
                if (self._graph_eligible() and hasattr(self, "_g_roots")
                        and it + 2 * G <= self.iters):
                    gl = self._graph_loop()
                    if gl is not None:
                        return self._step_group(gl, it, want_loss)
                if self._gnext == it and isinstance(self._dgl, DistGroupLoop):
                    # leaving the group loop: the last replay already pre-gathered
                    # (and charged) iterations it..it+G-1 into set _gx: train them
                    gl, x, out = self._dgl, self._gx, None
                    for j in range(G):
                        if it + j < self.iters:
                            out = self._train_built(gl.sets[x][j], it + j, want_loss)
                    self._gdone = it + G
                    return out
                self._gdone = None
            elif (self._graph_eligible() and hasattr(self, "_g_roots")
                    and it + 1 < self.iters):
                gl = self._graph_loop()
                if gl is not None:
                    return self._step_graph(gl, it, want_loss)
            return self._step_fast(it, want_loss)
        S, rank = self.S, self.rank
        batches = self.batches(it)
        if self.strategy == "model-centric":
            return self._step_model_centric(it, batches, want_loss)
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
            self._exchange([r] if n else [], [n], it)
            if n:
                _lib.call("hg_train_step", C.byref(r.desc), n, s)
                if want_loss:
                    loss = float(r.loss[:n].sum().item())
        else:
            active = []
            for (j, d, roots), r in zip(mine, self.runners):
                n = self._stage(r, roots, it)
                if n:
                    r.builder.build(self.graph, r.roots, r.keys, n, n_roots=n, stream=s)
                active.append(n)
            self._exchange([r for r, n in zip(self.runners, active) if n],
                           [n for n in active if n], it)
            for idx, ((j, d, roots), r) in enumerate(zip(mine, self.runners)):
                n = active[idx]
                if n:
                    _lib.call("hg_train_step", C.byref(r.desc), n, s)
                    if want_loss:
                        loss += float(r.loss[:n].sum().item())
                if j + 1 < cols:
                    self._hop(int(tt.server_of[0, j + 1] - tt.server_of[0, j]) % S)
        self._account_hops_and_sync()
        # synchronous update: all-reduce the accumulators, then SGD (model.py:299-324)
        if S > 1:
            dist.all_reduce(self.model.grad, group=self.group)
            self.traffic.allreduce_bytes += 2.0 * (S - 1) / S * self.flat_bytes
        self.model.sgd(self.lr, sum(len(b) for b in batches), stream=s)
        return loss if want_loss else None

    def _step_model_centric(self, it: int, batches, want_loss: bool):
        """Slow-path model-centric iteration (ragged last batch / no own comm)."""
        s = torch.cuda.current_stream(self.device).cuda_stream
        r = self.runners[0]
        n = self._stage(r, batches[self.rank], it)
        if n:
            r.builder.build(self.graph, r.roots, r.keys, n, n_roots=n, stream=s)
        self._exchange([r] if n else [], [n], it)
        loss = 0.0
        if n:
            _lib.call("hg_train_step", C.byref(r.desc), n, s)
            if want_loss:
                loss = float(r.loss[:n].sum().item())
        self._account_hops_and_sync()
        if self.S > 1:
            dist.all_reduce(self.model.grad, group=self.group)
            self.traffic.allreduce_bytes += 2.0 * (self.S - 1) / self.S * self.flat_bytes
        self.model.sgd(self.lr, sum(len(b) for b in batches), stream=s)
        return loss if want_loss else None

    def _exchange(self, runners, counts, it: int):
        if not self.pregather:
            self._account_remote(runners, it)
            return
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

    def _account_remote(self, runners, it: int):
        """Peer mode: rows are read in place, but the reference pre-gather plan
        (dedup remote rows per home per iteration) is still charged -- counted on
        the device into row `it` of an [iterations x S] table, no host sync."""
        if self.S == 1:
            return
        if self._acct_rows is None or self._acct_rows.shape[0] <= it:
            rows = max(it + 1, getattr(self, "iters", 1))
            t = torch.zeros((rows, self.S), dtype=torch.int64, device=self.device)
            if self._acct_rows is not None:
                t[:self._acct_rows.shape[0]] = self._acct_rows
            self._acct_rows = t
        s = torch.cuda.current_stream(self.device).cuda_stream
        row = self._acct_rows[it]
        # one plan per server-iteration: mark all runners' ids in one bitmap pass
        for r in runners:
            _lib.call("hg_remote_account", r.builder.tensors["need_ids"][0].data_ptr(),
                      r.builder.tensors["totals"].data_ptr(), 0, self.feats.home.data_ptr(),
                      self.rank, self.feats.bitmap.data_ptr(), row.data_ptr(),
                      self._acct_total.data_ptr(), s)
        for r in runners:
            _lib.call("hg_remote_clear", r.builder.tensors["need_ids"][0].data_ptr(),
                      r.builder.tensors["totals"].data_ptr(), 0, self.feats.bitmap.data_ptr(), s)
        self._acct_iters = getattr(self, "_acct_iters", set())
        self._acct_iters.add(it)

    def flush_accounting(self) -> None:
        """Move device-side pre-gather counts into the ledger (reference messages:
        one per (home -> server) per iteration with rows, featstore.py:271-274)
        and the fast path's per-iteration hop / all-reduce entries."""
        self.check()
        fast = getattr(self, "_fast_iters", 0)
        if fast:
            self._account_hops_and_sync(fast)
            self._fast_iters = 0
        if self.pregather or self._acct_rows is None:
            return
        rows = self._acct_rows.cpu().numpy()
        total_occ = int(self._acct_total.item())
        D = self.model.D
        row_bytes = self.feats.ld * (2 if self.feats.dtype == torch.bfloat16 else 4)
        for it in sorted(getattr(self, "_acct_iters", ())):
            for h, c in enumerate(rows[it].tolist()):
                if c:
                    self.ledger.add(h, self.rank, FEATURE, c * D * BYTES_PER_ELEM, 1)
                    self.stats.transferred += c
        # staged mode copies each distinct remote row once per iteration; the
        # peer-read gather loads every occurrence over NVLink
        moved = (int(sum(rows[it].sum() for it in getattr(self, "_acct_iters", ())))
                 if hasattr(self, "_ra") else total_occ)
        self.traffic.feature_rows += moved
        self.traffic.feature_bytes += moved * row_bytes
        self._acct_rows.zero_()
        self._acct_total.zero_()
        self._acct_iters = set()

    def _hop(self, delta: int):
        """Shift of (parameters, accumulator) by `delta` servers (engine.py:610-618):
        every trace-table column is a uniform shift, so each hop is a ring
        permutation over NVSwitch."""
        S, rank = self.S, self.rank
        m = self.model
        if self._comm is not None:
            # one grouped NCCL send/recv (hg_shift) and a device-side replica check:
            # no host synchronisation per hop; the flag is read by check()
            s = torch.cuda.current_stream(self.device).cuda_stream
            _lib.call("hg_shift", self._comm, rank, S, int(delta), m.flat.data_ptr(),
                      m.grad.data_ptr(), self._recv_p.data_ptr(), self._recv_g.data_ptr(),
                      m.flat.numel(), s)
            _lib.call("hg_flag_if_differ", self._recv_p.data_ptr(), m.flat.data_ptr(),
                      m.flat.numel(), self._hop_err.data_ptr(), s)
            m.grad.copy_(self._recv_g)
            self.traffic.hop_bytes += 2 * self.flat_bytes
            return
        nxt, prv = (rank + delta) % S, (rank - delta) % S
        ops = [dist.P2POp(dist.isend, m.flat, nxt, self.group),
               dist.P2POp(dist.isend, m.grad, nxt, self.group),
               dist.P2POp(dist.irecv, self._recv_p, prv, self.group),
               dist.P2POp(dist.irecv, self._recv_g, prv, self.group)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        if not torch.equal(self._recv_p, m.flat):
            raise InvariantViolation("replicas diverged during migration")
        m.grad.copy_(self._recv_g)
        self.traffic.hop_bytes += 2 * self.flat_bytes

    def _account_hops_and_sync(self, mult: int = 1):
        """Reference ledger entries this rank owns for `mult` iterations:
        MODEL+GRADIENT per hop arriving here (engine.py:610-618) and the ring
        all-reduce link leaving here (model.py:325-328)."""
        tt, S, rank = self.table, self.S, self.rank
        pb = self.model.param_bytes
        hops = 0 if self.strategy == "model-centric" else tt.n_columns - 1
        for j in range(hops):
            for d in range(tt.n_models):
                if int(tt.server_of[d, j + 1]) == rank:
                    src = int(tt.server_of[d, j])
                    self.ledger.add(src, rank, MODEL, pb * mult, mult)
                    self.ledger.add(src, rank, GRADIENT, pb * mult, mult)
        if S > 1:
            self.ledger.add(rank, (rank + 1) % S, GRADIENT, 2.0 * (S - 1) / S * pb * mult,
                            2 * (S - 1) * mult)

    def _setup_p2p_allreduce(self) -> None:
        """Exchange regions of the NVLink all-reduce (hg_p2p_allreduce):
        collective, at trainer setup."""
        n = self.model.flat.numel()
        nbytes = C.c_int64(0)
        _lib.call("hg_p2p_region_bytes", self.S, n, C.byref(nbytes))
        ptr = C.c_void_p()
        _lib.call("hg_alloc", nbytes.value, C.byref(ptr))
        handle = (C.c_char * 64)()
        _lib.call("hg_ipc_handle", ptr.value, handle)
        handles = [None] * self.S
        dist.all_gather_object(handles, bytes(handle), group=self.group)
        regions = []
        self._ar_opened = []
        for h, hb in enumerate(handles):
            if h == self.rank:
                regions.append(ptr.value)
                continue
            q = C.c_void_p()
            _lib.call("hg_ipc_open", (C.c_char * 64).from_buffer_copy(hb), C.byref(q))
            self._ar_opened.append(q.value)
            regions.append(q.value)
        dev = self.device
        self._ar = {"mine": ptr.value,
                    "regions": torch.tensor(regions, dtype=torch.int64, device=dev),
                    "seq": torch.zeros(1, dtype=torch.int64, device=dev),
                    "ctr": torch.zeros(1, dtype=torch.int32, device=dev),
                    "err": torch.zeros(1, dtype=torch.int32, device=dev)}

    def _sync_update(self, runner, stream, refresh: bool) -> None:
        """The synchronous update (model.py:299-324): all-reduce of the summed
        accumulators, theta -= lr * g / (S * B), gradient reset; refresh=True also
        rewrites the bf16 operand copies (hg_sgd_refresh).  All-reduce over NVLink
        peer memory (hg_p2p_allreduce) by default, NCCL when allreduce="nccl"."""
        m = self.model
        n = m.flat.numel()
        inv = 1.0 / (self.S * self.B)
        if self._ar is None:
            if refresh:
                _lib.call("hg_allreduce_sgd_refresh", self._comm, C.byref(runner.desc),
                          m.flat.data_ptr(), m.grad.data_ptr(), n, float(self.lr), inv, stream)
            else:
                _lib.call("hg_allreduce_sgd", self._comm, m.flat.data_ptr(), m.grad.data_ptr(),
                          n, float(self.lr), inv, stream)
            return
        a = self._ar
        _lib.call("hg_p2p_allreduce", m.grad.data_ptr(), n, a["regions"].data_ptr(), self.rank,
                  self.S, a["seq"].data_ptr(), a["ctr"].data_ptr(), a["err"].data_ptr(), stream)
        if refresh:
            _lib.call("hg_sgd_refresh", C.byref(runner.desc), m.flat.data_ptr(),
                      m.grad.data_ptr(), n, float(self.lr), inv, 1, stream)
        else:
            _lib.call("hg_sgd_update", m.flat.data_ptr(), m.grad.data_ptr(), None, n,
                      float(self.lr), inv, stream)

    def check(self) -> None:
        """Synchronise and raise on any device error flag: build errors (root
        out of range), push pre-gather timeouts / staging overflow."""
        for r in self.runners:
            r.check()
        if self._dgl is not None and hasattr(self._dgl, "check"):
            self._dgl.check()
        if hasattr(self.feats, "check"):
            self.feats.check()
        code = int(self._hop_err.item())
        if code:
            self._hop_err.zero_()
            _lib.flag_status(code, "model hop (replicas diverged during migration)")
        if self._ar is not None:
            code = int(self._ar["err"].item())
            if code:
                self._ar["err"].zero_()
                _lib.flag_status(code, "hg_p2p_allreduce (a peer never published its gradients)")

    def close(self) -> None:
        """Release peer mappings (CUDA IPC) held by this trainer."""
        if hasattr(self.feats, "close"):
            self.feats.close()
        for p in getattr(self, "_ar_opened", []):
            _lib.call("hg_ipc_close", p)
        self._ar_opened = []

    def global_ledger(self) -> CommLedger:
        """Merge every rank's ledger (collective)."""
        self.flush_accounting()
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


# ---------------------------------------------------------------- merging controller

@dataclass
class MergeEvent:
    """One controller decision (engine.py:764-770)."""
    epoch_start: int
    epochs: int
    columns: int
    avg_seconds: float
    action: str  # baseline | accepted | rejected | settled


def run_epoch(trainer: MicrographTrainer, epoch: int) -> float:
    """Train one epoch on the trainer's current trace table; returns its
    device-timed duration in seconds, max over ranks (identical on every
    rank, so controller decisions agree without further exchange)."""
    iters = trainer.begin_epoch(epoch)
    dev = trainer.device
    if dist.is_initialized() and trainer.S > 1:
        dist.barrier(group=trainer.group)
    torch.cuda.synchronize(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for it in range(iters):
        trainer.step(it, want_loss=False)
    t1.record()
    torch.cuda.synchronize(dev)
    trainer.flush_accounting()  # fast-path entries belong to this epoch's table
    sec = torch.tensor([t0.elapsed_time(t1) / 1e3], dtype=torch.float64, device=dev)
    if dist.is_initialized() and trainer.S > 1:
        dist.all_reduce(sec, op=dist.ReduceOp.MAX, group=trainer.group)
    return float(sec.item())


def counts_for_next_epoch(trainer: MicrographTrainer, tt: TraceTable, epoch: int) -> np.ndarray:
    """Cell root counts of `epoch`'s first iteration under `tt`
    (engine.py:836-842): the controller decides before running it."""
    S, B = trainer.S, trainer.B
    perm = epoch_permutation(trainer.seed, epoch, trainer.graph.n_vertices,
                             trainer.device).cpu().numpy()
    home = trainer.part.home
    batches = [perm[min(d * B, len(perm)):min((d + 1) * B, len(perm))] for d in range(S)]
    groups = [tuple(b[home[b] == s] for s in range(S)) for b in batches]
    cells = assign_cell_roots(tt, groups, chain(trainer.seed, SEED_MERGE, epoch, 0))
    return cell_counts(cells)


def merge_controller(trainer: MicrographTrainer, epochs: int, merge_k: int, cost=None):
    """Greedy column removal (engine.py:773-833): run K epochs, tentatively drop
    the column with the fewest roots, keep the drop only if the average epoch
    cost strictly shrinks, else revert and settle.  The cost is the measured
    epoch time (max over ranks) unless ``cost(table, seconds)`` overrides it
    (the reference uses its simulated clock).  Merged tables run through the
    general cell path; every rank reaches identical decisions.
    Returns (final table, [MergeEvent], per-epoch seconds)."""
    if trainer.strategy != "micrograph":
        raise ValueError("merging applies to the micrograph strategy")
    cost = cost or (lambda table, seconds: seconds)
    K = int(merge_k)
    tt = TraceTable.initial(trainer.S)
    history, times = [], []
    epoch = 0

    def run_block(table: TraceTable, count: int) -> float:
        nonlocal epoch
        vals = []
        for _ in range(count):
            trainer.table = table
            sec = run_epoch(trainer, epoch)
            times.append(sec)
            vals.append(float(cost(table, sec)))
            epoch += 1
        return float(np.mean(vals)) if vals else 0.0

    baseline = min(K, epochs)
    old = run_block(tt, baseline)
    history.append(MergeEvent(0, baseline, tt.n_columns, old, "baseline"))
    settled = False
    while not settled and epoch + K <= epochs and tt.n_columns >= 2:
        probe = tt.copy()
        probe.root_counts = counts_for_next_epoch(trainer, tt, epoch)
        target = find_fewest_column(probe)
        if target is None:
            break
        tentative = delete_column_and_redistribute(probe, target)
        tentative.validate()
        start = epoch
        new = run_block(tentative, K)
        if new < old:
            tt, old = tentative, new
            history.append(MergeEvent(start, K, tt.n_columns, new, "accepted"))
        else:
            history.append(MergeEvent(start, K, tentative.n_columns, new, "rejected"))
            settled = True
    if epoch < epochs:
        start = epoch
        avg = run_block(tt, epochs - epoch)
        history.append(MergeEvent(start, epochs - start, tt.n_columns, avg, "settled"))
    trainer.table = tt
    return tt, history, times
