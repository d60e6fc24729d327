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
from .sampler import GroupBuilder
from .trainer import CellRunner

SEED_GRAPH, SEED_PARTITION, SEED_FEATURES, SEED_LABELS = 0x01, 0x02, 0x03, 0x04
SEED_BATCHES, SEED_SAMPLER, SEED_MODEL, SEED_MERGE = 0x05, 0x06, 0x07, 0x08


# Stream priorities of the graph loops: the training chain (latency-bound,
# small grids) at high priority, the build / gather branch (throughput-bound,
# fills every SM) at low priority, so freed SM slots go to training first.
_TRAIN_PRIO = 1
# Resident build CTAs per SM on the graph loop's build branch (GroupLoop):
# 3 x 256 threads x 48 registers leaves a GEMM / gather CTA room on every SM,
# so the training branch is not starved while a group is being built.
BUILD_CTAS_PER_SM = 3


def _streams(dev):
    """(capture stream for the training branch, side stream for the build branch)."""
    if _TRAIN_PRIO:
        return torch.cuda.Stream(dev, priority=-_TRAIN_PRIO), torch.cuda.Stream(dev, priority=0)
    return torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def _u64_as_i64(vals) -> np.ndarray:
    return np.asarray([int(v) & ((1 << 64) - 1) for v in vals], dtype=np.uint64).view(np.int64)


class RunAhead:
    """Sampling run-ahead: micrograph construction does not
    depend on the parameters, so iteration it+1's build runs on a side stream
    while iteration it trains.  Two runners alternate; events order the
    build after the previous use of the same runner and the train after the
    build."""

    def __init__(self, runners, device):
        self.runners = runners
        self.side = torch.cuda.Stream(device)
        self.main = torch.cuda.current_stream(device)
        self.built = {}
        self.free = [None] * len(runners)

    def prefetch(self, it: int, build) -> None:
        if it in self.built:
            return
        i = it % len(self.runners)
        with torch.cuda.stream(self.side):
            if self.free[i] is not None:
                self.side.wait_event(self.free[i])
            build(self.runners[i], self.side.cuda_stream)
            ev = torch.cuda.Event()
            ev.record(self.side)
        self.built[it] = (i, ev)

    def acquire(self, it: int, build):
        self.prefetch(it, build)
        i, ev = self.built.pop(it)
        self.main.wait_event(ev)
        return self.runners[i]

    def release(self, it: int) -> None:
        ev = torch.cuda.Event()
        ev.record(self.main)
        self.free[it % len(self.runners)] = ev

    def reset(self) -> None:
        self.built.clear()


class GraphLoop:
    """CUDA-graph replay of the run-ahead loop (S = 1).  Two graphs alternate:
    graph x trains runner x (built by the previous replay) + SGD, and on a
    forked branch stages, builds and pre-gathers the next iteration into
    runner 1-x.  The iteration comes from a device cursor (hg_iter_stage), so
    every replay has identical launch arguments: one host call per step
    instead of ~30 launches, and the build branch overlaps the training branch
    inside the graph.  Optional per-graph extras: H2D of the next roots from a
    pinned slot (public end-to-end API) and D2H of the summed loss."""

    def __init__(self, tr: "Trainer", runners, e2e: bool = False):
        self.tr, self.runners, self.e2e = tr, runners, e2e
        dev = tr.device
        B = tr.B
        self._cap, self.side = _streams(dev)
        if e2e:
            self.pin_roots = [torch.empty(B, dtype=torch.int64).pin_memory() for _ in range(2)]
            self.pin_loss = [torch.zeros(1, dtype=torch.float32).pin_memory() for _ in range(2)]
        self.graphs = []
        self.launches = 0
        cur = torch.cuda.current_stream(dev)
        for x in range(2):
            run, nxt = runners[x], runners[1 - x]
            for r in (run, nxt):
                r.desc.roots = r.roots.data_ptr()
                r.desc.agg1_ready = 1
                r.n_roots = B
            g = torch.cuda.CUDAGraph()
            cap = self._cap
            cap.wait_stream(cur)
            before = _lib.launch_count()
            with torch.cuda.graph(g, stream=cap):
                self.side.wait_stream(cap)
                ss = self.side.cuda_stream
                with torch.cuda.stream(self.side):
                    if e2e:  # roots of the next step, written by the host into a pinned slot
                        nxt.roots.copy_(self.pin_roots[1 - x], non_blocking=True)
                    _lib.call("hg_iter_stage", tr._perm_buf.data_ptr(), tr._states_buf.data_ptr(),
                              tr.iters, tr._it_dev.data_ptr(), B, 1, 1,
                              None if e2e else nxt.roots.data_ptr(), nxt.keys.data_ptr(), ss)
                    nxt.builder.build(tr.graph, nxt.roots.data_ptr(), nxt.keys.data_ptr(), B,
                                      n_roots=B, stream=ss)
                    _lib.call("hg_step_prologue", C.byref(nxt.desc), B, 1, ss)
                cs = cap.cuda_stream
                m = tr.model
                if run.tc:  # SGD refreshes the bf16 operands: the step skips its transposes
                    run.desc.lowp_fresh = 1
                    _lib.call("hg_train_step_sgd", C.byref(run.desc), B, m.flat.data_ptr(),
                              m.grad.data_ptr(), m.flat.numel(), float(tr.lr), 1.0 / B, 1, cs)
                    run.desc.lowp_fresh = 0
                else:
                    _lib.call("hg_train_step", C.byref(run.desc), B, cs)
                    m.sgd(tr.lr, B, stream=cs)
                if e2e:
                    self.pin_loss[x].copy_(run.loss[:B].sum().reshape(1), non_blocking=True)
                cap.wait_stream(self.side)
            self.launches = _lib.launch_count() - before
            cur.wait_stream(cap)
            self.graphs.append(g)
        self.iters = tr.iters

    def replay(self, x: int) -> None:
        self.graphs[x].replay()


class GroupLoop:
    """CUDA-graph replay of the run-ahead loop over groups of G iterations
    (S = 1).  Two sets of G runners alternate: graph x trains set x's G
    iterations in order (train step + fused SGD/refresh each) while a forked
    branch stages the next G iterations from the device cursor, builds all
    their micrographs in ONE launch (hg_mg_build_group) and gathers their
    layer-1 features in ONE launch (hg_step_prologue_group) into set 1-x.
    Training semantics are those of the one-iteration loop (sampling never
    reads the parameters); what changes is launch shape: a 1024-root build is
    ~1.4 waves of build CTAs and a 100K-row gather is too short to reach HBM
    bandwidth, a G-iteration group keeps every SM busy through both tails.
    Optional e2e extras: the next group's roots arrive through a pinned host
    slot, and the group's per-iteration summed losses go back to pinned host
    memory."""

    def __init__(self, tr: "Trainer", sets, e2e: bool = False):
        self.tr, self.sets, self.e2e = tr, sets, e2e
        self.G = G = len(sets[0])
        dev, B = tr.device, tr.B
        self.gb = [GroupBuilder([r.builder for r in st]) for st in sets]
        for x in range(2):
            for b, r in enumerate(sets[x]):
                r.desc.roots = self.gb[x].roots_ptr(b)
                r.desc.agg1_ready = 1
                r.n_roots = B
        self.descp = [(C.POINTER(_lib.StepDesc) * G)(*[C.pointer(r.desc) for r in st])
                      for st in sets]
        self._cap, self.side = _streams(dev)
        if e2e:
            self.pin_roots = [torch.empty(G * B, dtype=torch.int64).pin_memory() for _ in range(2)]
            self.pin_loss = [torch.zeros(G, dtype=torch.float32).pin_memory() for _ in range(2)]
        self.graphs = []
        self.launches = 0
        self.x = 0
        cur = torch.cuda.current_stream(dev)
        m = tr.model
        for x in range(2):
            nxt = self.gb[1 - x]
            g = torch.cuda.CUDAGraph()
            cap = self._cap
            cap.wait_stream(cur)
            before = _lib.launch_count()
            with torch.cuda.graph(g, stream=cap):
                self.side.wait_stream(cap)
                ss = self.side.cuda_stream
                with torch.cuda.stream(self.side):
                    if e2e:  # roots of the next group, written by the host into a pinned slot
                        nxt.roots.copy_(self.pin_roots[1 - x], non_blocking=True)
                    _lib.call("hg_iter_stage_group", tr._perm_buf.data_ptr(),
                              tr._states_buf.data_ptr(), tr.iters, tr._it_dev.data_ptr(), B, G,
                              G, G, None if e2e else nxt.roots.data_ptr(), nxt.keys.data_ptr(), ss)
                    nxt.build(tr.graph, stream=ss, ctas_per_sm=BUILD_CTAS_PER_SM)
                    _lib.call("hg_step_prologue_group", self.descp[1 - x], G, 1, ss)
                cs = cap.cuda_stream
                for r in sets[x]:
                    if r.tc:  # SGD refreshes the bf16 operands: steps skip their transposes
                        r.desc.lowp_fresh = 1
                        _lib.call("hg_train_step_sgd", C.byref(r.desc), B, m.flat.data_ptr(),
                                  m.grad.data_ptr(), m.flat.numel(), float(tr.lr), 1.0 / B, 1, cs)
                        r.desc.lowp_fresh = 0
                    else:
                        _lib.call("hg_train_step", C.byref(r.desc), B, cs)
                        m.sgd(tr.lr, B, stream=cs)
                if e2e:
                    self.pin_loss[x].copy_(torch.stack([r.loss[:B].sum() for r in sets[x]]),
                                           non_blocking=True)
                cap.wait_stream(self.side)
            self.launches = _lib.launch_count() - before
            cur.wait_stream(cap)
            self.graphs.append(g)
        self.iters = tr.iters

    def restart(self, it: int, roots=None) -> None:
        """Position the loop at iteration `it` (it + G <= iters): build the
        group [it, it+G) into set 0 on the current stream, point the device
        cursor at it.  roots: device int64[G*B] (e2e), else the epoch plan."""
        tr = self.tr
        tr._drain_run_ahead()
        cur = torch.cuda.current_stream(tr.device)
        cur.wait_stream(self.side)
        s = cur.cuda_stream
        gb = self.gb[0]
        tr._it_dev.fill_(it)
        _lib.call("hg_iter_stage_group", tr._perm_buf.data_ptr(), tr._states_buf.data_ptr(),
                  tr.iters, tr._it_dev.data_ptr(), tr.B, self.G, 0, 0,
                  None if roots is not None else gb.roots.data_ptr(), gb.keys.data_ptr(), s)
        if roots is not None:
            gb.roots.copy_(roots, non_blocking=True)
        gb.build(tr.graph, stream=s)
        _lib.call("hg_step_prologue_group", self.descp[0], self.G, 1, s)
        r = self.sets[0][0]
        if r.tc:  # the replays' steps use the bf16 operands as the previous SGD left them
            m = tr.model
            _lib.call("hg_sgd_refresh", C.byref(r.desc), m.flat.data_ptr(), m.grad.data_ptr(),
                      m.flat.numel(), 0.0, 1.0, 0, s)
        self.x = 0

    def run_eager(self, it: int) -> None:
        """The body of one replay for iterations it..it+G-1 launched eagerly on
        the current stream, with the replay's configuration (build grid capped
        at BUILD_CTAS_PER_SM, grouped gather, steps on the bf16 operands the
        fused SGD + refresh keeps current): the profiling pass, where per-kernel
        CUDA-event sites need real launches.  The branches run one after the
        other here (in the replay the build overlaps training).  Leaves the
        loop unpositioned."""
        tr = self.tr
        cur = torch.cuda.current_stream(tr.device)
        cur.wait_stream(self.side)
        s = cur.cuda_stream
        gb = self.gb[0]
        B, G = tr.B, self.G
        gb.roots.copy_(tr.perm[it * B:(it + G) * B])
        gb.keys.copy_(tr.states[it:it + G])
        gb.build(tr.graph, stream=s, ctas_per_sm=BUILD_CTAS_PER_SM)
        _lib.call("hg_step_prologue_group", self.descp[0], G, 1, s)
        m = tr.model
        r0 = self.sets[0][0]
        if r0.tc:  # operands current before the first step (the replays leave them so)
            _lib.call("hg_sgd_refresh", C.byref(r0.desc), m.flat.data_ptr(), m.grad.data_ptr(),
                      m.flat.numel(), 0.0, 1.0, 0, s)
        for r in self.sets[0]:
            if r.tc:
                r.desc.lowp_fresh = 1
                _lib.call("hg_train_step_sgd", C.byref(r.desc), B, m.flat.data_ptr(),
                          m.grad.data_ptr(), m.flat.numel(), float(tr.lr), 1.0 / B, 1, s)
                r.desc.lowp_fresh = 0
            else:
                _lib.call("hg_train_step", C.byref(r.desc), B, s)
                m.sgd(tr.lr, B, stream=s)

    def replay(self) -> int:
        """Train the positioned group; returns the parity replayed."""
        x = self.x
        self.graphs[x].replay()
        self.x ^= 1
        return x

    def check(self) -> None:
        for gb in self.gb:
            gb.check()


class Trainer:
    """One model on one GPU (S = 1): the reference's micrograph and
    model-centric strategies coincide here (engine.py:485-507 with N = 1).
    ``graphs=True`` replays the steady-state loop as CUDA graphs (GraphLoop)."""

    def __init__(self, graph: Graph, table: FeatureTable, model: ModelState, fanout,
                 batch: int, seed: int, lr: float = 0.1, iterations: int = 0,
                 run_ahead: bool = True, graphs: bool = True, group: int = 1):
        self.graph, self.table, self.model = graph, table, model
        self.fanout = tuple(fanout)
        self.B, self.seed, self.lr, self.iter_cap = int(batch), int(seed), float(lr), iterations
        self.labels = LabelOracle(model.C, chain(seed, SEED_LABELS))
        self.sampler_seed = chain(seed, SEED_SAMPLER)
        self.runner = CellRunner(graph, table, model, self.fanout, self.B, self.labels)
        self.device = model.device
        self.epoch = None
        self.stream = torch.cuda.current_stream(self.device)
        self.run_ahead = run_ahead
        if run_ahead:
            self.ra = RunAhead([self.runner, CellRunner(graph, table, model, self.fanout, self.B,
                                                        self.labels)], self.device)
        self.last_runner = self.runner
        self.graphs = graphs and run_ahead
        self._gl = None       # GraphLoop for step()
        self._gl_e2e = None   # GraphLoop for train_step()
        self._gnext = None    # iteration the graph loop is positioned at
        self._eager_steps = 0
        # run-ahead group size of the graph loop (GroupLoop when > 1)
        if not 1 <= int(group) <= _lib.MAX_GROUP:
            raise ValueError(f"group must be 1..{_lib.MAX_GROUP}")
        self.G = int(group)
        self._gg = None       # GroupLoop for step()
        self._gg_e2e = None   # GroupLoop for train_group()
        self._gdone = None    # iterations < _gdone are already enqueued by a group replay

    # ------------------------------------------------------------ epoch plan
    def begin_epoch(self, epoch: int) -> int:
        """Permutation + per-iteration key states for `epoch`; returns #iterations."""
        n = self.graph.n_vertices
        self.perm = epoch_permutation(self.seed, epoch, n, self.device)
        self.iters = iterations_per_epoch(n, 1, self.B, self.iter_cap)
        states = [chain(self.sampler_seed, epoch, it) for it in range(self.iters)]
        self.states = torch.from_numpy(_u64_as_i64(states)).to(self.device)
        self.epoch = epoch
        if self.graphs:
            # graph-visible copies at fixed addresses (captured once per trainer)
            if not hasattr(self, "_perm_buf"):
                self._perm_buf = torch.empty_like(self.perm)
                self._states_buf = torch.empty_like(self.states)
                self._it_dev = torch.zeros(1, dtype=torch.int64, device=self.device)
            self._perm_buf.copy_(self.perm)
            self._states_buf.copy_(self.states)
            self._gnext = None
            self._gdone = None
        # run-ahead builds read perm/states from side streams: order them after
        # this epoch's permutation (written on the current stream)
        cur = torch.cuda.current_stream(self.device)
        for ra in (getattr(self, "ra", None), getattr(self, "_e2e_ra", None)):
            if ra is not None:
                ra.side.wait_stream(cur)
        return self.iters

    # ------------------------------------------------------------ graph loop
    def _graph_ready(self, attr: str, e2e: bool):
        gl = getattr(self, attr)
        if gl is not None and gl.iters != self.iters:
            gl = None
        if gl is None:
            if self._eager_steps < 2:  # library state (attributes, tensor maps) warmed eagerly
                return None
            self._drain_run_ahead()
            gl = GraphLoop(self, self.ra.runners if not e2e else self._e2e_ra.runners, e2e)
            setattr(self, attr, gl)
        return gl

    def _group_ready(self, attr: str, e2e: bool):
        gl = getattr(self, attr)
        if gl is not None and gl.iters != self.iters:
            gl = None
        if gl is None:
            if self._eager_steps < 2:  # library state (attributes, tensor maps) warmed eagerly
                return None
            self._drain_run_ahead()
            mk = lambda: CellRunner(self.graph, self.table, self.model, self.fanout, self.B,
                                    self.labels)
            sets = [[mk() for _ in range(self.G)] for _ in range(2)]
            gl = GroupLoop(self, sets, e2e)
            setattr(self, attr, gl)
        return gl

    def _drain_run_ahead(self) -> None:
        cur = torch.cuda.current_stream(self.device)
        for ra in (self.ra, getattr(self, "_e2e_ra", None)):
            if ra is not None:
                cur.wait_stream(ra.side)
                ra.reset()

    def _graph_restart(self, gl: GraphLoop, it: int, roots=None) -> None:
        """Position the graph loop at `it`: build it eagerly into runner it%2
        on the current stream, point the device cursor at it."""
        self._drain_run_ahead()
        if gl.e2e:
            cur = torch.cuda.current_stream(self.device)
            cur.wait_stream(gl.side)
        r = gl.runners[it % 2]
        s = torch.cuda.current_stream(self.device).cuda_stream
        if roots is None:
            roots = self.roots_of(it)
        n = roots.numel()
        r.roots[:n].copy_(roots, non_blocking=True)
        r.keys[:1].copy_(self.states[it:it + 1])
        r.builder.build(self.graph, r.roots.data_ptr(), r.keys.data_ptr(), n, n_roots=n, stream=s)
        r.desc.roots = r.roots.data_ptr()
        r.n_roots = n
        _lib.call("hg_step_prologue", C.byref(r.desc), n, 1, s)
        r.desc.agg1_ready = 1
        if r.tc:  # the replays' steps use the bf16 operands as the previous SGD left them
            m = self.model
            _lib.call("hg_sgd_refresh", C.byref(r.desc), m.flat.data_ptr(), m.grad.data_ptr(),
                      m.flat.numel(), 0.0, 1.0, 0, s)
        self._it_dev.fill_(it)

    def roots_of(self, it: int) -> torch.Tensor:
        lo = min(it * self.B, self.perm.numel())
        return self.perm[lo:min(lo + self.B, self.perm.numel())]

    # ------------------------------------------------------------ steps
    def _build(self, it: int):
        roots = self.roots_of(it)
        n = roots.numel()

        def launch(r, s):
            r.builder.build(self.graph, roots.data_ptr(), self.states.data_ptr() + 8 * it, n,
                            n_roots=n, stream=s)
            r.desc.roots = roots.data_ptr()
            r.n_roots = n
            if self.run_ahead:  # the layer-1 gather is parameter independent too
                _lib.call("hg_step_prologue", C.byref(r.desc), n, 1, s)
                r.desc.agg1_ready = 1
        return launch

    def step(self, it: int, stop: int = None) -> None:
        """One iteration with inputs already resident in HBM (no host sync).
        With run-ahead, iteration it+1's micrographs are built on a side
        stream while this iteration trains.  With group G > 1 a call at a
        group start enqueues iterations it..it+G-1 (one graph replay) when
        all of them are below `stop` (default: the epoch end); the calls for
        it+1..it+G-1 then return at once.  Other iterations run eagerly."""
        s = self.stream.cuda_stream
        if self.G > 1 and self.graphs:
            if self._gdone is not None and it < self._gdone and it >= self._gdone - self.G:
                return  # enqueued by the last group replay
            lim = self.iters if stop is None else min(int(stop), self.iters)
            gg = self._group_ready("_gg", False) if it + self.G <= lim else None
            if gg is not None:
                if self._gnext != it:
                    gg.restart(it)
                x = gg.replay()
                self._gnext = self._gdone = it + self.G
                self.last_runner = gg.sets[x][-1]
                self.last_group = (it, gg.sets[x])
                return
            self._gnext = self._gdone = None
        gl = self._graph_ready("_gl", False) if self.graphs and self.G == 1 else None
        if gl is not None and (it + 1 < self.iters or self._gnext == it):
            if self._gnext != it:
                self._graph_restart(gl, it)
            r = gl.runners[it % 2]
            if it + 1 < self.iters:
                gl.replay(it % 2)  # trains `it`, builds it+1 into the other runner
            else:  # last iteration of the epoch: nothing to build ahead
                _lib.call("hg_train_step", C.byref(r.desc), r.n_roots, s)
                self.model.sgd(self.lr, r.n_roots, stream=s)
            self._gnext = it + 1
            self.last_runner = r
            return
        if self._gnext is not None:
            # leaving the graph loop: its last replay may still be building into a
            # run-ahead runner -- order the side stream after it
            self.ra.side.wait_stream(torch.cuda.current_stream(self.device))
            self.ra.reset()
        self._gnext = None
        self._eager_steps += 1
        if not self.run_ahead:
            r = self.runner
            self._build(it)(r, s)
        else:
            r = self.ra.acquire(it, self._build(it))
        n = r.n_roots
        _lib.call("hg_train_step", C.byref(r.desc), n, s)
        self.model.sgd(self.lr, n, stream=s)
        self.last_runner = r
        if self.run_ahead:
            self.ra.release(it)
            if it + 1 < self.iters:
                self.ra.prefetch(it + 1, self._build(it + 1))

    def train_step(self, roots_host: torch.Tensor, it: int, next_roots_host=None):
        """Public end-to-end step (engine.py:434-445 semantics): this step's roots
        come from pinned host memory (`next_roots_host`, when the data loader
        already knows the next batch, lets its micrographs be built ahead), and
        every step's summed loss is copied back to the host.  The readback is
        pipelined one step: the call returns the PREVIOUS step's loss (None on
        the first call); ``last_loss()`` drains the final one."""
        if not hasattr(self, "_e2e"):
            cap = self.B
            self._e2e = {"dev": [torch.empty(cap, dtype=torch.int64, device=self.device)
                                 for _ in range(2)],
                         "loss": [torch.zeros(1, dtype=torch.float32).pin_memory()
                                  for _ in range(2)],
                         "slot": 0, "pending": None}
            self._e2e_ra = RunAhead([self.runner, CellRunner(
                self.graph, self.table, self.model, self.fanout, self.B, self.labels)],
                self.device) if self.run_ahead else None
        e = self._e2e
        if roots_host.numel() > self.B or (next_roots_host is not None
                                           and next_roots_host.numel() > self.B):
            raise ValueError(f"train_step takes at most B = {self.B} roots per step")
        # the captured graph stages and trains exactly B roots: a short batch
        # (the epoch tail) takes the eager path
        if (self.graphs and self.G == 1 and next_roots_host is not None
                and roots_host.numel() == self.B and next_roots_host.numel() == self.B):
            gl = self._graph_ready("_gl_e2e", True)
            if gl is not None:
                return self._train_step_graph(gl, roots_host, it, next_roots_host)
        if e.get("gnext") is not None and self._e2e_ra is not None:
            self._e2e_ra.side.wait_stream(torch.cuda.current_stream(self.device))
            self._e2e_ra.reset()
        e["gnext"] = None
        self._eager_steps += 1

        def build_for(j, roots_h):
            dev = e["dev"][j % 2]
            n = roots_h.numel()

            def launch(r, s):
                dev[:n].copy_(roots_h, non_blocking=True)
                r.builder.build(self.graph, dev.data_ptr(), self.states.data_ptr() + 8 * j, n,
                                n_roots=n, stream=s)
                r.desc.roots = dev.data_ptr()
                r.n_roots = n
                if self.run_ahead:
                    _lib.call("hg_step_prologue", C.byref(r.desc), n, 1, s)
                    r.desc.agg1_ready = 1
                else:
                    r.desc.agg1_ready = 0
            return launch

        s = self.stream.cuda_stream
        if self._e2e_ra is not None:
            r = self._e2e_ra.acquire(it, build_for(it, roots_host))
        else:
            r = self.runner
            build_for(it, roots_host)(r, s)
        n = r.n_roots
        _lib.call("hg_train_step", C.byref(r.desc), n, s)
        self.model.sgd(self.lr, n, stream=s)
        e["slot"] ^= 1
        e["loss"][e["slot"]].copy_(r.loss[:n].sum().reshape(1), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        if self._e2e_ra is not None:
            self._e2e_ra.release(it)
            if next_roots_host is not None:
                self._e2e_ra.prefetch(it + 1, build_for(it + 1, next_roots_host))
        prev = self._drain_loss()  # the previous step's loss, read once this one is queued
        e["pending"] = (ev, e["slot"])
        return prev

    def _train_step_graph(self, gl: GraphLoop, roots_host, it: int, next_roots_host):
        """train_step through the e2e GraphLoop: the host copies the next
        step's roots into a pinned slot and launches one graph; the graph's
        H2D / D2H copies move the roots in and the summed loss out."""
        e = self._e2e
        x = it % 2
        prev = None
        if e.get("gnext") != it:
            prev = self._drain_loss()  # an eager step's pending loss
            dev = e["dev"][x]
            n = roots_host.numel()
            dev[:n].copy_(roots_host, non_blocking=True)
            self._graph_restart(gl, it, dev[:n])
            e["gev"] = [None, None]
        # pinned roots slot 1-x was last read by replay(it-2) (same parity as this one)
        if e["gev"][x] is not None:
            e["gev"][x].synchronize()
        gl.pin_roots[1 - x].numpy()[:next_roots_host.numel()] = next_roots_host.numpy()
        gl.replay(x)
        ev = torch.cuda.Event()
        ev.record()
        e["gev"][x] = ev
        e["gnext"] = it + 1
        self.last_runner = gl.runners[x]
        # the previous step's loss: wait for replay(it-1) while replay(it) is queued
        ev_prev = e["gev"][1 - x]
        if ev_prev is not None:
            ev_prev.synchronize()
            prev = float(gl.pin_loss[1 - x].item())
        e["pending_graph"] = (ev, gl, x)
        return prev

    def train_group(self, roots_host: torch.Tensor, it: int, next_roots_host=None):
        """Public end-to-end API over a group of G iterations (the data loader
        hands out G batches at a time): roots_host = pinned int64[G*B], the
        roots of iterations it..it+G-1; next_roots_host = the next group's
        (lets its micrographs be built ahead).  Every group's per-iteration
        summed losses come back to the host; the readback is pipelined one
        group: the call returns the PREVIOUS group's G losses (None on the
        first call) and ``last_group_loss()`` drains the final one."""
        G, B = self.G, self.B
        if roots_host.numel() != G * B:
            raise ValueError(f"train_group takes G*B = {G * B} roots")
        if not hasattr(self, "_e2g"):
            self._e2g = {"dev": torch.empty(G * B, dtype=torch.int64, device=self.device),
                         "gnext": None, "gev": [None, None], "pending": None}
        e = self._e2g
        gl = None
        if G > 1 and self.graphs and next_roots_host is not None and it + 2 * G <= self.iters:
            gl = self._group_ready("_gg_e2e", True)
        if gl is None:  # eager: G public steps, losses held until the next call
            prev = self._drain_group()
            e["gnext"] = None
            out = []
            for b in range(G):
                nxt = (roots_host[(b + 1) * B:(b + 2) * B] if b + 1 < G else
                       (next_roots_host[:B] if next_roots_host is not None else None))
                r = self.train_step(roots_host[b * B:(b + 1) * B], it + b, nxt)
                if b > 0:
                    out.append(r)
            out.append(self.last_loss())
            e["pending"] = ("held", out)
            return prev
        x = gl.x
        prev = None
        if e["gnext"] != it:
            prev = self._drain_group()
            self._drain_loss()
            e["dev"].copy_(roots_host, non_blocking=True)
            gl.restart(it, e["dev"])
            e["gev"] = [None, None]
        # pinned roots slot 1-x was last read by the replay of parity x
        if e["gev"][x] is not None:
            e["gev"][x].synchronize()
        gl.pin_roots[1 - x].numpy()[:] = next_roots_host.numpy()
        gl.replay()
        ev = torch.cuda.Event()
        ev.record()
        e["gev"][x] = ev
        e["gnext"] = it + G
        self.last_runner = gl.sets[x][-1]
        ev_prev = e["gev"][1 - x]
        if ev_prev is not None and prev is None:
            ev_prev.synchronize()
            prev = gl.pin_loss[1 - x].tolist()
        e["pending"] = ("graph", ev, gl, x)
        return prev

    def _drain_group(self):
        e = getattr(self, "_e2g", None)
        if not e or e["pending"] is None:
            return None
        p, e["pending"] = e["pending"], None
        if p[0] == "held":
            return p[1]
        _, ev, gl, x = p
        ev.synchronize()
        return gl.pin_loss[x].tolist()

    def last_group_loss(self):
        """The G losses of the most recent train_group (host sync)."""
        return self._drain_group()

    def _drain_loss(self):
        e = getattr(self, "_e2e", None)
        if e and e.get("pending_graph") is not None:
            ev, gl, x = e["pending_graph"]
            ev.synchronize()
            e["pending_graph"] = None
            return float(gl.pin_loss[x].item())
        if not e or e["pending"] is None:
            return None
        ev, slot = e["pending"]
        ev.synchronize()
        e["pending"] = None
        return float(e["loss"][slot].item())

    def last_loss(self):
        """Loss of the most recent train_step (host sync)."""
        return self._drain_loss()

    def check(self) -> None:
        for gg in (self._gg, self._gg_e2e):
            if gg is not None:
                gg.check()
        self.runner.check()
        if self.run_ahead:
            for r in self.ra.runners:
                r.check()

    def batch_sizes(self):
        """(N_k, P_k) of the last built batch (synchronises)."""
        tot = self.runner.builder.tensors["totals"].cpu().numpy()
        L = len(self.fanout)
        return tot[:L + 1].tolist(), tot[L + 1:2 * L + 1].tolist()
