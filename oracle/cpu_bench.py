"""CPU baseline of the micrograph training step (oracle port of the reference path).

TEST/BENCH INFRASTRUCTURE ONLY: executed by bench.py's ``cpu_baseline`` leg
and ``--impl reference`` arm, never by the product.

What is timed is the reference's per-iteration work for each root
(engine.py:290-295 + 434-445, model.py:213-329): sample the micrograph
(numba port of the frontier draw, _kernels_nb.py:55-86), gather its feature
rows, float64 forward, softmax-CE backward, gradient accumulation, then the
synchronous SGD update.  The synthetic graph is the row-local generator of
oracle/graphgen.py materialised lazily; rows and feature rows the sample
touches are materialised in an untimed warm-up pass, exactly like the
reference holds its CSR and FeatureStore in memory before training.
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import kernels as OK
from . import model as OM
from .graphgen import GraphSpec, LazyRows, build_tables
from .rng import chain, mix64


class LazyGraphSampler:
    """sample_micrograph (sampler.py:84-106) over lazily materialised rows."""

    def __init__(self, spec: GraphSpec):
        self.spec = spec
        self.rows = LazyRows(build_tables(spec))

    def frontier(self, frontier, fanout: int, state: int):
        counts = np.zeros(len(frontier), dtype=np.int64)
        parts = []
        for i, v in enumerate(frontier.tolist()):
            row = self.rows(v)
            sl = OK.draw_slots(state, v, len(row), fanout)
            counts[i] = len(sl)
            parts.append(row[sl])
        flat = np.concatenate(parts) if parts else np.empty(0, np.int64)
        return counts, flat

    def expanded_vertices(self, roots, fanout, keys) -> np.ndarray:
        """Sorted ids of every vertex the roots' micrographs expand (layers 1..L),
        hop by hop, materialising each hop's frontier rows in one vectorised
        pass (rows_csr)."""
        L = len(fanout)
        front = [np.array([int(r)], dtype=np.int64) for r in roots]
        seen = [np.concatenate(front)] if front else []
        for hop in range(1, L):
            self.rows.prefetch(np.concatenate(front))
            nxt = []
            for i, f in enumerate(front):
                _, flat = self.frontier(f, fanout[hop - 1], chain(int(keys[i]), hop))
                nxt.append(np.unique(flat))
            front = nxt
            seen.extend(front)
        out = np.unique(np.concatenate(seen)) if seen else np.empty(0, np.int64)
        self.rows.prefetch(out)
        return out

    def micrographs(self, roots, fanout, keys):
        """micrograph() for many roots (rows prefetched hop by hop)."""
        self.expanded_vertices(roots, fanout, keys)
        return [self.micrograph(int(r), fanout, int(k)) for r, k in zip(roots, keys)]

    def micrograph(self, root: int, fanout, key: int):
        from .sampler import Micro
        L = len(fanout)
        layers, pairs = [None] * (L + 1), [None] * L
        layers[L] = np.array([root], dtype=np.int64)
        for k in range(L - 1, -1, -1):
            hop = L - k
            front = layers[k + 1]
            counts, flat = self.frontier(front, fanout[hop - 1], chain(key, hop))
            layers[k] = np.unique(flat)
            pairs[k] = (np.repeat(np.arange(len(front)), counts),
                        np.searchsorted(layers[k], flat))
        return Micro(root, tuple(layers), tuple(pairs), np.unique(np.concatenate(layers)))


class CpuStep:
    """One process's share of the reference iteration on a bounded root sample."""

    def __init__(self, spec: GraphSpec, arch, fanout, dim, hidden, classes, seed, lr=0.1):
        self.g = LazyGraphSampler(spec)
        self.fanout = tuple(fanout)
        self.dim, self.C, self.lr = dim, classes, lr
        self.P = OM.init_params(arch, dim, hidden, len(fanout), classes, chain(seed, 0x07))
        self.sseed = chain(seed, 0x06)
        self.lseed = chain(seed, 0x04)
        self.fstate = chain(chain(seed, 0x03), 0xFE)
        self.feat = {}

    def _rows(self, ids):
        miss = [int(v) for v in ids if int(v) not in self.feat]
        if miss:
            block = OK.feature_rows(np.array(miss), self.dim, self.fstate)
            for v, r in zip(miss, block):
                self.feat[v] = r
        return np.stack([self.feat[int(v)] for v in ids])

    def warm(self, roots, epoch, it):
        for r in roots:
            m = self.g.micrograph(int(r), self.fanout, chain(self.sseed, epoch, it, int(r)))
            self._rows(m.vertices)

    def grads(self, roots, epoch, it):
        G = self.P.zeros()
        loss = 0.0
        labs = OM.labels(roots, self.C, self.lseed)
        for r, lab in zip(roots, labs):
            m = self.g.micrograph(int(r), self.fanout, chain(self.sseed, epoch, it, int(r)))
            st = OM.forward(m, self._rows(m.vertices), self.P)
            lo, g = OM.loss_and_grads(st, int(lab), self.P)
            OM.add_into(G, g)
            loss += lo
        return G, loss


def sample_roots(n: int, count: int, seed: int, step: int) -> np.ndarray:
    """Bounded sample of the epoch: roots as the keyed permutation would draw them
    (hash order of random ids), one disjoint slice per step."""
    h = np.array([mix64(chain(seed, 0x5A, step) ^ i) for i in range(count)], dtype=np.uint64)
    return (h % np.uint64(n)).astype(np.int64)


def run_single(spec, model_kw, seed, roots_per_step, steps, budget_s=20.0):
    """Single-core port timing.  Returns (seeds/s, roots timed)."""
    cs = CpuStep(spec, seed=seed, **model_kw)
    batches = [sample_roots(spec.n, roots_per_step, seed, s) for s in range(steps)]
    for i, b in enumerate(batches):
        cs.warm(b, 0, i)
    t0 = time.perf_counter()
    done = 0
    for i, b in enumerate(batches):
        G, _ = cs.grads(b, 0, i)
        OM.sgd_step(cs.P, G, len(b), cs.lr)
        done += len(b)
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return done / dt, done


# ---------------------------------------------------------------- multi-process arm

def _proc_main(conn, spec, model_kw, seed):
    cs = CpuStep(spec, seed=seed, **model_kw)
    while True:
        msg = conn.recv()
        if msg[0] == "warm":
            for roots, it in msg[1]:
                cs.warm(roots, 0, it)
            conn.send(None)
        elif msg[0] == "grads":
            _, roots, it, params = msg
            for a, b in zip(cs.P.arrays(), params):
                a[...] = b
            G, loss = cs.grads(roots, 0, it)
            conn.send(([a for a in G.arrays()], loss))
        else:
            break


def run_pool(spec, model_kw, seed, roots_per_step, steps, warmup, procs=None):
    """All host cores: every step's bounded root sample is split across worker
    processes (worker w always gets part w, so its warm row cache is the one it
    uses); gradients are summed and one SGD update is applied per step.
    Returns (seeds/s over the timed steps, procs, per-step seconds)."""
    import multiprocessing as mp
    procs = procs or os.cpu_count() or 1
    ctx = mp.get_context("fork")
    cs = CpuStep(spec, seed=seed, **model_kw)
    total = warmup + steps
    batches = [sample_roots(spec.n, roots_per_step, seed, s) for s in range(total)]
    parts = [np.array_split(b, procs) for b in batches]
    pipes, workers = [], []
    for w in range(procs):
        a, b = ctx.Pipe()
        p = ctx.Process(target=_proc_main, args=(b, spec, model_kw, seed), daemon=True)
        p.start()
        pipes.append(a)
        workers.append(p)
    try:
        for w, c in enumerate(pipes):   # untimed: materialise rows + feature rows
            c.send(("warm", [(parts[i][w], i) for i in range(total)]))
        for c in pipes:
            c.recv()
        times = []
        for i in range(total):
            t0 = time.perf_counter()
            params = [a.copy() for a in cs.P.arrays()]
            for w, c in enumerate(pipes):
                c.send(("grads", parts[i][w], i, params))
            G = cs.P.zeros()
            for c in pipes:
                arrs, _ = c.recv()
                for a, b in zip(G.arrays(), arrs):
                    a += b
            OM.sgd_step(cs.P, G, len(batches[i]), cs.lr)
            times.append(time.perf_counter() - t0)
    finally:
        for c in pipes:
            try:
                c.send(("stop",))
            except Exception:
                pass
        for p in workers:
            p.join(timeout=5)
    timed = times[warmup:]
    return roots_per_step * len(timed) / sum(timed), procs, timed
