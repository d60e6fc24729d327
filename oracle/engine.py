"""Scheduling + byte accounting of the micrograph strategy (restates ``engine.py``
and the ledger parts of ``featstore.py``).

Only what the hot path needs: the epoch permutation and batches
(engine.py:268-287), the trace table and per-cell root assignment with merge
replay (engine.py:103-205), pre-gather planning (featstore.py:226-239), the
byte ledger (featstore.py:32-87) and a full micrograph / model-centric
iteration driver (engine.py:485-507, 562-623) that yields ledger bytes and
post-update parameters for the multi-GPU parity tests.
"""
from __future__ import annotations

from collections import defaultdict

import numpy as np

from . import model as M
from .rng import chain, keyed, keyed_shuffle
from .sampler import sample_micrograph, stream_key

SEED_FEATURES, SEED_LABELS, SEED_BATCHES = 0x03, 0x04, 0x05
SEED_SAMPLER, SEED_MODEL, SEED_MERGE = 0x06, 0x07, 0x08
FEATURE, MODEL, GRADIENT = "feature", "model", "gradient"


def epoch_permutation(seed: int, epoch: int, n: int) -> np.ndarray:
    """Stable argsort of keyed hashes (engine.py:273-275)."""
    keys = keyed(chain(seed, SEED_BATCHES, epoch), np.arange(n, dtype=np.int64))
    return np.argsort(keys, kind="stable").astype(np.int64)


def epoch_batches(seed: int, epoch: int, n: int, n_servers: int, batch: int,
                  iterations: int = 0):
    """[iteration][model] root chunks of the permutation (engine.py:268-287)."""
    perm = epoch_permutation(seed, epoch, n)
    iters = max(1, n // (n_servers * batch))
    if iterations:
        iters = min(iters, iterations)
    out = []
    for it in range(iters):
        row = []
        for d in range(n_servers):
            lo = min((it * n_servers + d) * batch, n)
            row.append(perm[lo:min(lo + batch, n)])
        out.append(row)
    return out


# ---------------------------------------------------------------- trace table

def initial_table(n: int) -> np.ndarray:
    """server_of[d, t] = (d + t) mod n (engine.py:117-121)."""
    d = np.arange(n)[:, None]
    return (d + np.arange(n)[None, :]) % n


def even_split(count: int, parts: int) -> list:
    base, rem = divmod(count, parts)
    return [base + (i < rem) for i in range(parts)]


def delete_column(server_of: np.ndarray, counts: np.ndarray, col: int):
    """Drop a column, spreading its counts evenly (engine.py:162-178)."""
    keep = [j for j in range(server_of.shape[1]) if j != col]
    out = counts[:, keep].copy()
    for d in range(server_of.shape[0]):
        for i, extra in enumerate(even_split(int(counts[d, col]), len(keep))):
            out[d, i] += extra
    return server_of[:, keep].copy(), out


def fewest_column(counts: np.ndarray):
    """argmin column sum, ties low (engine.py:148-153)."""
    if counts.shape[1] < 2:
        return None
    return int(np.argmin(counts.sum(axis=0)))


def assign_cells(groups, removed, key: int):
    """cells[d][t] with merge-history replay (engine.py:181-205)."""
    n = len(groups)
    cells = [[groups[d][(d + t) % n] for t in range(n)] for d in range(n)]
    for ordinal, pos in enumerate(removed):
        for d in range(n):
            row = cells[d]
            moved = keyed_shuffle(chain(key, ordinal, d), row.pop(pos))
            start = 0
            for i, size in enumerate(even_split(len(moved), len(row))):
                if size:
                    row[i] = np.concatenate([row[i], moved[start:start + size]])
                start += size
    return cells


def model_at(server_of: np.ndarray, s: int, col: int) -> int:
    return int(np.flatnonzero(server_of[:, col] == s)[0])


# ---------------------------------------------------------------- ledger

class Ledger:
    """(src, dst, category) -> [bytes, messages] (featstore.py:32-87)."""

    def __init__(self):
        self.cells = defaultdict(lambda: [0.0, 0])

    def add(self, src, dst, cat, nbytes, msgs=1):
        if src == dst:
            raise RuntimeError("self-link")
        c = self.cells[(int(src), int(dst), cat)]
        c[0] += nbytes
        c[1] += msgs

    def by_category(self):
        out = {}
        for (_, _, cat), (b, _) in self.cells.items():
            out[cat] = out.get(cat, 0.0) + b
        return out

    def link(self, src, dst, cat):
        b, m = self.cells.get((src, dst, cat), (0.0, 0))
        return b, m


def pregather_plan(at: int, vertex_sets, home: np.ndarray):
    """Deduplicated remote ids grouped by home (featstore.py:226-239)."""
    if vertex_sets:
        need = np.unique(np.concatenate(vertex_sets))
    else:
        need = np.empty(0, dtype=np.int64)
    remote = need[home[need] != at]
    rh = home[remote]
    return [(int(s), remote[rh == s]) for s in np.unique(rh)]


# ---------------------------------------------------------------- drivers

class World:
    """Inputs of one simulated run (the reference SimWorld, engine.py:216-258)."""

    def __init__(self, offsets, targets, home, n_servers, seed, arch, dim, hidden,
                 n_classes, fanout, batch, lr=0.1, iterations=0, feat_rows=None):
        from .kernels import feature_rows
        self.offsets, self.targets = np.asarray(offsets), np.asarray(targets)
        self.home = np.asarray(home, dtype=np.int64)
        self.S, self.seed = n_servers, seed
        self.arch, self.dim, self.hidden, self.C = arch, dim, hidden, n_classes
        self.fanout, self.B, self.lr, self.iterations = tuple(fanout), batch, lr, iterations
        self.n = len(self.offsets) - 1
        fstate = chain(chain(seed, SEED_FEATURES), 0xFE)
        self.rows = feat_rows or (lambda ids: feature_rows(ids, dim, fstate))
        self.label_seed = chain(seed, SEED_LABELS)
        self.sampler_seed = chain(seed, SEED_SAMPLER)

    def fresh_params(self):
        return M.init_params(self.arch, self.dim, self.hidden, len(self.fanout), self.C,
                             chain(self.seed, SEED_MODEL))

    def micro(self, root, epoch, it):
        return sample_micrograph(self.offsets, self.targets, int(root), self.fanout,
                                 stream_key(self.sampler_seed, epoch, it, int(root)))


def _train_cell(world, P, micros, acc, loss_acc):
    if not micros:
        return
    need = np.unique(np.concatenate([m.vertices for m in micros]))
    rows = world.rows(need)
    labs = M.labels([m.root for m in micros], world.C, world.label_seed)
    for m, lab in zip(micros, labs):
        st = M.forward(m, rows[np.searchsorted(need, m.vertices)], P)
        loss, g = M.loss_and_grads(st, int(lab), P)
        M.add_into(acc, g)
        loss_acc.append(loss)


def micrograph_iteration(world, P, epoch, it, batches, server_of, removed=(),
                         pregather=True, ledger=None):
    """One iteration of _micrograph_epoch (engine.py:569-622); updates P in place.

    Returns (ledger, losses).  Ledger bytes follow the reference exactly:
    feature rows per (home -> server) per pre-gather message (or per cell
    without pre-gathering), MODEL+GRADIENT param_bytes per hop, ring
    all-reduce bytes at sync.
    """
    S = world.S
    ledger = ledger if ledger is not None else Ledger()
    groups = [tuple(np.asarray(b)[world.home[np.asarray(b)] == s] for s in range(S))
              for b in batches]
    cells = assign_cells(groups, removed, chain(world.seed, SEED_MERGE, epoch, it))
    roots = np.concatenate(batches)
    micros = {int(r): world.micro(r, epoch, it) for r in roots}
    pb = P.nbytes_ref
    cols = server_of.shape[1]
    if pregather:
        for s in range(S):
            sets = []
            for j in range(cols):
                d = model_at(server_of, s, j)
                sets += [micros[int(r)].vertices for r in cells[d][j]]
            for src, ids in pregather_plan(s, sets, world.home):
                ledger.add(src, s, FEATURE, len(ids) * world.dim * 4, 1)
    accs = [P.zeros() for _ in range(S)]
    losses = []
    for j in range(cols):
        for s in range(S):
            d = model_at(server_of, s, j)
            ms = [micros[int(r)] for r in cells[d][j]]
            if not pregather and ms:
                need = np.unique(np.concatenate([m.vertices for m in ms]))
                hs = world.home[need]
                for h in np.unique(hs):
                    if h != s:
                        ledger.add(h, s, FEATURE, int((hs == h).sum()) * world.dim * 4, 1)
            _train_cell(world, P, ms, accs[d], losses)
        if j + 1 < cols:
            for d in range(S):
                ledger.add(server_of[d, j], server_of[d, j + 1], MODEL, pb, 1)
                ledger.add(server_of[d, j], server_of[d, j + 1], GRADIENT, pb, 1)
    total = P.zeros()
    for a in accs:
        M.add_into(total, a)
    M.sgd_step(P, total, sum(len(b) for b in batches), world.lr)
    if S > 1:
        per = M.ring_allreduce_bytes(S, pb)
        for s in range(S):
            ledger.add(s, (s + 1) % S, GRADIENT, per, 2 * (S - 1))
    return ledger, losses


def model_centric_iteration(world, P, epoch, it, batches, ledger=None):
    """One iteration of _model_centric_epoch (engine.py:490-506)."""
    S = world.S
    ledger = ledger if ledger is not None else Ledger()
    accs = [P.zeros() for _ in range(S)]
    losses = []
    for d, b in enumerate(batches):
        ms = [world.micro(r, epoch, it) for r in b]
        if ms:
            need = np.unique(np.concatenate([m.vertices for m in ms]))
            hs = world.home[need]
            for h in np.unique(hs):
                if h != d:
                    ledger.add(h, d, FEATURE, int((hs == h).sum()) * world.dim * 4, 1)
        _train_cell(world, P, ms, accs[d], losses)
    total = P.zeros()
    for a in accs:
        M.add_into(total, a)
    M.sgd_step(P, total, sum(len(b) for b in batches), world.lr)
    if S > 1:
        per = M.ring_allreduce_bytes(S, P.nbytes_ref)
        for s in range(S):
            ledger.add(s, (s + 1) % S, GRADIENT, per, 2 * (S - 1))
    return ledger, losses
