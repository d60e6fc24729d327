"""Trainer-level drop-in: ``run_strategy(RunConfig) -> [EpochMetrics]`` on one GPU.

Mirrors the reference's single-process trainer API (gnnsim ``engine.py``):
``run_strategy`` (849-863), ``run_model_centric`` (478-507),
``run_micrograph`` (547-623, with pre-gathering and the merge controller
779-833) and ``run_locality_optimized`` (510-544), taking the reference's
``RunConfig`` (config.py:32-99) and returning its ``EpochMetrics``
(engine.py:302-321) -- the same ledger, miss rate, alpha, imbalance,
trained compositions, column counts and simulated time (CostModel,
engine.py:46-90) -- so a gnnsim user switches by changing the import.

Like the reference, the S servers are simulated in one process (one GPU);
the multi-process, one-GPU-per-server trainer is
``distributed.MicrographTrainer``.  Per iteration every root of every model
is sampled, gathered and trained in ONE device step (``CellRunner``:
hg_mg_build + hg_train_step, then the synchronous SGD): models are
replicated and unchanged inside an iteration and the update is
sum(accumulators) / batch_total (model.py:315-324), so the per-cell split
only matters to the byte ledger, which is charged per cell from the
device-built micrographs' vertex sets exactly as ``run_cell`` /
``FeatureStore.fetch`` / ``execute_pregather`` charge it
(engine.py:428-463, featstore.py:141-158, 268-279).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from .distributed import (TraceTable, assign_cell_roots, cell_counts,
                          delete_column_and_redistribute, find_fewest_column)
from .errors import ConfigError, InvariantViolation
from .featstore import (BYTES_PER_ELEM, FEATURE, GRADIENT, MODEL, TOPOLOGY, CommLedger,
                        FeatureTable, FetchStats, plan_pregather)
from .graph import (Graph, PartitionMap, load_csr, load_edge_list, load_partition,
                    partition_greedy_locality, partition_hash, generate_sbm, SbmSpec)
from .model import LabelOracle, init_model
from .rng import chain
from .sampler import load_imbalance, redistribute_roots
from .trainer import CellRunner

STRATEGIES = ("model-centric", "naive", "locality-optimized", "micrograph", "micrograph+pg",
              "micrograph+pg+merge")
SEED_GRAPH, SEED_PARTITION, SEED_FEATURES, SEED_LABELS = 0x01, 0x02, 0x03, 0x04
SEED_BATCHES, SEED_SAMPLER, SEED_MODEL, SEED_MERGE = 0x05, 0x06, 0x07, 0x08


# ---------------------------------------------------------------- configuration

@dataclass
class RunConfig:
    """Same fields, defaults and validation as the reference (config.py:32-99)."""

    graph: str = "sbm"
    blocks: tuple = (100, 100)
    p_in: float = 0.2
    p_out: float = 0.01
    servers: int = 2
    partitioner: str = "greedy"
    partition_file: str = ""
    slack: float = 0.0
    layers: int = 2
    fanout: tuple = (3,)
    mode: str = "node-wise"
    dim: int = 8
    hidden: int = 8
    classes: int = 4
    arch: str = "gcn"
    lr: float = 0.1
    batch: int = 32
    epochs: int = 1
    iterations: int = 0
    strategy: str = "micrograph"
    merge_k: int = 1
    bandwidth: float = math.inf
    latency: float = 0.0
    sync_overhead: float = 0.0
    kernel_launch: float = 0.0
    compute_rate: float = 0.0
    seed: int = 0
    parallel: bool = False
    dump_batches: str = ""

    def __post_init__(self):
        self.validate()

    def validate(self) -> None:
        if self.servers < 1:
            raise ConfigError("servers must be >= 1")
        if self.layers < 1:
            raise ConfigError("layers must be >= 1")
        fo = self.fanout if isinstance(self.fanout, tuple) else (
            tuple(self.fanout) if isinstance(self.fanout, list) else (self.fanout,))
        if len(fo) == 1:
            fo = fo * self.layers
        if len(fo) != self.layers or any(f < 1 for f in fo):
            raise ConfigError("fanout must give one value, or one per layer, all >= 1")
        self.fanout = fo
        if self.mode not in ("node-wise", "layer-wise"):
            raise ConfigError(f"unknown sampling mode {self.mode!r}")
        if self.partitioner not in ("hash", "greedy", "file"):
            raise ConfigError(f"unknown partitioner {self.partitioner!r}")
        if self.partitioner == "file" and not self.partition_file:
            raise ConfigError("partitioner=file needs partition_file=")
        if self.strategy not in STRATEGIES:
            raise ConfigError(f"unknown strategy {self.strategy!r}; choose from "
                              + ", ".join(STRATEGIES))
        if self.arch not in ("gcn", "sage-mean"):
            raise ConfigError(f"unknown arch {self.arch!r}")
        if self.dim < 1 or self.hidden < 1 or self.classes < 2:
            raise ConfigError("need dim >= 1, hidden >= 1, classes >= 2")
        if self.batch < 1 or self.epochs < 1 or self.merge_k < 1:
            raise ConfigError("batch, epochs and merge_k must be >= 1")
        if self.iterations < 0:
            raise ConfigError("iterations must be >= 0")
        for name in ("bandwidth", "latency", "sync_overhead", "kernel_launch", "compute_rate",
                     "slack"):
            if getattr(self, name) < 0:
                raise ConfigError(f"{name} must be >= 0")
        if self.graph == "sbm" and (not self.blocks or any(b < 1 for b in self.blocks)):
            raise ConfigError("blocks must all be >= 1")

    def with_strategy(self, strategy: str) -> "RunConfig":
        return replace(self, strategy=strategy)


def as_run_config(cfg) -> RunConfig:
    """Accept the reference's RunConfig (or any object with its fields)."""
    if isinstance(cfg, RunConfig):
        return cfg
    names = RunConfig.__dataclass_fields__.keys()
    return RunConfig(**{k: getattr(cfg, k) for k in names if hasattr(cfg, k)})


# ---------------------------------------------------------------- simulated cost

@dataclass(frozen=True)
class CostModel:
    """Simulated time per step (engine.py:46-62); the merge controller decides on it."""

    bandwidth: float = math.inf
    latency: float = 0.0
    sync_overhead: float = 0.0
    kernel_launch: float = 0.0
    compute_rate: float = 0.0

    def __post_init__(self):
        for name in ("latency", "sync_overhead", "kernel_launch", "compute_rate"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")
        if self.bandwidth <= 0:
            raise ValueError("bandwidth must be > 0 (use inf for free links)")


@dataclass
class ServerWork:
    """One server's aggregates for one time step, comm charged at the receiver
    (engine.py:65-83)."""

    messages: int = 0
    bytes: float = 0.0
    launches: int = 0
    work_units: float = 0.0

    def add_comm(self, nbytes: float, messages: int) -> None:
        self.bytes += nbytes
        self.messages += messages

    def seconds(self, cm: CostModel) -> float:
        compute = cm.kernel_launch * self.launches + cm.compute_rate * self.work_units
        return compute + self.messages * cm.latency + self.bytes / cm.bandwidth


def simulated_step_time(works, cm: CostModel) -> float:
    """max over servers of (compute + comm) + sync overhead (engine.py:86-89)."""
    return max((w.seconds(cm) for w in works), default=0.0) + cm.sync_overhead


# ---------------------------------------------------------------- metrics

@dataclass
class EpochMetrics:
    """engine.py:302-321, plus ``device_seconds`` (measured, CUDA events)."""

    epoch: int
    strategy: str
    sim_seconds: float
    steps: int
    iterations: int
    bytes_by_category: dict
    miss_rate: float
    alpha: float
    imbalance: float
    busy_seconds: np.ndarray
    staged_bytes: float
    ledger: CommLedger
    trained: list
    composition_diverged: bool
    n_columns: int
    device_seconds: float = 0.0

    def total_bytes(self) -> float:
        return sum(self.bytes_by_category.values())


def alpha_ratio(metrics: EpochMetrics, param_bytes: int) -> float:
    """Remote training-data bytes per iteration over parameter bytes (engine.py:324-329)."""
    if param_bytes <= 0:
        raise ValueError("model must have parameters")
    data = metrics.bytes_by_category[FEATURE] + metrics.bytes_by_category[TOPOLOGY]
    return data / metrics.iterations / param_bytes


# ---------------------------------------------------------------- world

@dataclass
class World:
    """SimWorld (engine.py:212-258) with the numerics on the GPU: device CSR,
    fp32 feature table, device model, one CellRunner sized for an iteration."""

    cfg: RunConfig
    graph: Graph
    partition: PartitionMap
    table: FeatureTable
    labels: LabelOracle
    sampler_seed: int
    cm: CostModel
    model: object
    runner: CellRunner = field(default=None, repr=False)

    @property
    def n_servers(self) -> int:
        return self.cfg.servers

    @property
    def n_vertices(self) -> int:
        return self.graph.n_vertices


def build_world(cfg, device="cuda", modes_ok: bool = False) -> World:
    """engine.py:235-258 on the GPU.  Graph: "sbm" (generate_sbm, CUDA pair pass),
    a CSR1 file (*.csr) or an edge list; partitioner hash / greedy / file.
    The batched trainer samples node-wise; layer-wise worlds (modes_ok) serve
    the locality report (sampler.sample_micrograph, layer-wise hops)."""
    cfg = as_run_config(cfg)
    if cfg.mode != "node-wise" and not modes_ok:
        raise ConfigError("the batched trainer samples node-wise; layer-wise micrographs come "
                          "from sampler.sample_micrograph (kernels.pick_k_smallest)")
    if cfg.graph == "sbm":
        graph = generate_sbm(SbmSpec(tuple(cfg.blocks), cfg.p_in, cfg.p_out,
                                     chain(cfg.seed, SEED_GRAPH)), device)
    elif cfg.graph.endswith(".csr"):
        graph = load_csr(cfg.graph, device)
    else:
        graph = load_edge_list(cfg.graph, device=device)
    if cfg.partitioner == "hash":
        part = partition_hash(graph, cfg.servers, chain(cfg.seed, SEED_PARTITION))
    elif cfg.partitioner == "greedy":
        part = partition_greedy_locality(graph, cfg.servers, cfg.slack,
                                         chain(cfg.seed, SEED_PARTITION))
    else:
        part = load_partition(cfg.partition_file, cfg.servers)
        if part.n_vertices != graph.n_vertices:
            raise ConfigError("partition file does not cover the graph")
    table = FeatureTable.generated(graph.n_vertices, cfg.dim, cfg.seed, torch.float32, device)
    hidden = -(-cfg.hidden // 8) * 8
    if hidden != cfg.hidden:
        raise ConfigError("hidden must be a multiple of 8 on the device")
    model = init_model(cfg.arch, cfg.dim, cfg.hidden, cfg.layers, cfg.classes,
                       chain(cfg.seed, SEED_MODEL), device)
    labels = LabelOracle(cfg.classes, chain(cfg.seed, SEED_LABELS))
    cm = CostModel(cfg.bandwidth, cfg.latency, cfg.sync_overhead, cfg.kernel_launch,
                   cfg.compute_rate)
    w = World(cfg, graph, part, table, labels, chain(cfg.seed, SEED_SAMPLER), cm, model)
    cap = max(1, min(cfg.servers * cfg.batch, graph.n_vertices))
    w.runner = CellRunner(graph, table, model, cfg.fanout, cap, labels)
    return w


def epoch_batches(world: World, epoch: int) -> list:
    """[iteration][model] root chunks of the keyed permutation (engine.py:268-287)."""
    from .batching import epoch_permutation
    n, N, B = world.n_vertices, world.n_servers, world.cfg.batch
    perm = epoch_permutation(world.cfg.seed, epoch, n, world.graph.device).cpu().numpy()
    iters = max(1, n // (N * B))
    if world.cfg.iterations:
        iters = min(iters, world.cfg.iterations)
    out = []
    for it in range(iters):
        row = []
        for d in range(N):
            lo = min((it * N + d) * B, n)
            row.append(perm[lo:min(lo + B, n)])
        out.append(row)
    return out


class _Iteration:
    """One iteration's roots built + trained in one device step; per-root
    vertex sets (= need[0], Micrograph.vertices) for the ledger."""

    def __init__(self, world: World, roots: np.ndarray, epoch: int, it: int, batch_total: int):
        r = world.runner
        st = np.uint64(chain(world.sampler_seed, epoch, it)).view(np.int64)
        n = len(roots)
        self.vertices = {}
        if n:
            r.stage_roots(roots, [st], n)
            batch = r.launch()
            ids = batch.need_ids[0]
            off = batch.need_off[0][:n + 1].cpu().numpy()
            host = ids[:int(off[-1])].cpu().numpy().astype(np.int64)
            for i, v in enumerate(roots.tolist()):
                self.vertices[int(v)] = host[off[i]:off[i + 1]]
        # synchronous update over all models' accumulators (model.py:315-324)
        world.model.sgd(world.cfg.lr, batch_total)


class _Collector:
    """_EpochCollector (engine.py:332-410)."""

    def __init__(self, world: World, epoch: int, strategy: str):
        self.world, self.epoch, self.strategy = world, epoch, strategy
        self.ledger = CommLedger()
        self.stats = FetchStats()
        self.sim_seconds = 0.0
        self.steps = 0
        self.busy = np.zeros(world.n_servers, dtype=np.float64)
        self.imbalances = []
        self.staged_bytes = 0.0
        self.trained = []
        self.n_columns = world.n_servers
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        self.ev[0].record()

    def step(self, works) -> None:
        cm = self.world.cm
        self.sim_seconds += simulated_step_time(works, cm)
        for s, w in enumerate(works):
            self.busy[s] += w.seconds(cm)
        self.steps += 1

    def merge_cell(self, delta: CommLedger, stats: FetchStats) -> None:
        self.ledger.merge(delta)
        self.stats.merge(stats)

    def final_sync(self, param_bytes: int) -> None:
        """Ledger + simulated time of sync_and_update (model.py:325-328, engine.py:358-367)."""
        n = self.world.n_servers
        if n > 1:
            per_link = 2.0 * (n - 1) / n * param_bytes
            for s in range(n):
                self.ledger.add(s, (s + 1) % n, GRADIENT, per_link, 2 * (n - 1))
            t = self.world.cm.latency * 2 * (n - 1) + per_link / self.world.cm.bandwidth
            self.sim_seconds += t
            self.busy += t

    def finish(self, batches_per_iter, param_bytes: int) -> EpochMetrics:
        self.ev[1].record()
        torch.cuda.synchronize()
        diverged = False
        for trained, batches in zip(self.trained, batches_per_iter):
            for got, want in zip(trained, batches):
                if not np.array_equal(got, np.sort(np.asarray(want))):
                    diverged = True
        m = EpochMetrics(epoch=self.epoch, strategy=self.strategy, sim_seconds=self.sim_seconds,
                         steps=self.steps, iterations=len(batches_per_iter),
                         bytes_by_category=self.ledger.bytes_by_category(),
                         miss_rate=self.stats.miss_rate, alpha=0.0,
                         imbalance=float(np.mean(self.imbalances)) if self.imbalances else 0.0,
                         busy_seconds=self.busy, staged_bytes=self.staged_bytes,
                         ledger=self.ledger, trained=self.trained,
                         composition_diverged=diverged, n_columns=self.n_columns,
                         device_seconds=self.ev[0].elapsed_time(self.ev[1]) / 1000.0)
        m.alpha = alpha_ratio(m, param_bytes)
        return m


def _cell(world: World, server: int, roots, vertices, staged) -> tuple:
    """run_cell's accounting for one (server, cell) (engine.py:428-448, 451-463)."""
    ledger, stats, work = CommLedger(), FetchStats(), ServerWork()
    if len(roots):
        sets = [vertices[int(r)] for r in roots]
        needs = np.unique(np.concatenate(sets))
        homes = world.partition.home[needs]
        if staged is None:  # FeatureStore.fetch (featstore.py:141-158)
            stats.requested += len(needs)
            for s in np.unique(homes).tolist():
                count = int(np.count_nonzero(homes == s))
                if s == server:
                    stats.local += count
                    continue
                ledger.add(s, server, FEATURE, count * world.cfg.dim * BYTES_PER_ELEM, 1)
                stats.transferred += count
        else:  # _rows_via_staging (engine.py:451-463)
            local = int(np.count_nonzero(homes == server))
            stats.requested += len(needs)
            stats.local += local
            stats.staged += len(needs) - local
        work.launches += 1
        work.work_units += sum(len(v) for v in sets) * world.cfg.dim
        for (_, _, _), (b, msgs) in ledger.counters.items():
            work.add_comm(b, msgs)
    return ledger, stats, work


def _model_centric_epoch(world: World, epoch: int) -> EpochMetrics:
    """engine.py:485-507."""
    col = _Collector(world, epoch, "model-centric")
    col.n_columns = 1
    pb = world.model.param_bytes
    batches_per_iter = epoch_batches(world, epoch)
    for it, batches in enumerate(batches_per_iter):
        plan = redistribute_roots(batches, world.partition)
        col.imbalances.append(load_imbalance(plan))
        roots = np.concatenate(batches) if batches else np.empty(0, np.int64)
        itr = _Iteration(world, roots, epoch, it, sum(len(b) for b in batches))
        works = []
        for d in range(world.n_servers):
            ledger, stats, work = _cell(world, d, batches[d], itr.vertices, None)
            col.merge_cell(ledger, stats)
            works.append(work)
        col.step(works)
        col.trained.append([np.sort(np.asarray(b)) for b in batches])
        col.final_sync(pb)
    return col.finish(batches_per_iter, pb)


def _locality_epoch(world: World, epoch: int) -> EpochMetrics:
    """engine.py:510-544: redistributed roots trained where they live."""
    col = _Collector(world, epoch, "locality-optimized")
    col.n_columns = 1
    pb = world.model.param_bytes
    batches_per_iter = epoch_batches(world, epoch)
    S = world.n_servers
    for it, batches in enumerate(batches_per_iter):
        plan = redistribute_roots(batches, world.partition)
        col.imbalances.append(load_imbalance(plan))
        roots = np.concatenate(batches) if batches else np.empty(0, np.int64)
        itr = _Iteration(world, roots, epoch, it, sum(len(b) for b in batches))
        local = [np.concatenate([plan.groups[d][s] for d in range(S)]) for s in range(S)]
        works = []
        for s in range(S):
            ledger, stats, work = _cell(world, s, local[s], itr.vertices, None)
            col.merge_cell(ledger, stats)
            works.append(work)
        col.step(works)
        col.trained.append([np.sort(r) for r in local])
        col.final_sync(pb)
    return col.finish(batches_per_iter, pb)


def _micrograph_epoch(world: World, tt: TraceTable, epoch: int, pregather: bool,
                      name: str) -> EpochMetrics:
    """engine.py:562-623."""
    col = _Collector(world, epoch, name)
    col.n_columns = tt.n_columns
    pb = world.model.param_bytes
    D = world.cfg.dim
    batches_per_iter = epoch_batches(world, epoch)
    S = world.n_servers
    home = world.partition.home
    for it, batches in enumerate(batches_per_iter):
        plan = redistribute_roots(batches, world.partition)
        col.imbalances.append(load_imbalance(plan))
        roots = np.concatenate(batches) if batches else np.empty(0, np.int64)
        itr = _Iteration(world, roots, epoch, it, sum(len(b) for b in batches))
        cells = assign_cell_roots(tt, plan.groups, chain(world.cfg.seed, SEED_MERGE, epoch, it))
        tt.root_counts = cell_counts(cells)
        tt.validate()
        pending = [(0.0, 0) for _ in range(S)]
        staged = [None] * S
        if pregather:  # plan_pregather + execute_pregather per server (featstore.py:226-279)
            for s in range(S):
                sets = [itr.vertices[int(r)] for j in range(tt.n_columns)
                        for r in cells[tt.model_at(s, j)][j]]
                pg = plan_pregather(s, sets, home)
                delta, st = CommLedger(), FetchStats()
                for src, ids in pg.by_source:
                    delta.add(src, s, FEATURE, len(ids) * D * BYTES_PER_ELEM, 1)
                    st.transferred += len(ids)
                staged[s] = pg
                col.merge_cell(delta, st)
                col.staged_bytes += pg.total_rows * D * BYTES_PER_ELEM
                b, msgs = delta.total_bytes(), sum(m for _, m in delta.counters.values())
                pending[s] = (pending[s][0] + b, pending[s][1] + msgs)
        for j in range(tt.n_columns):
            works = []
            for s in range(S):
                d = tt.model_at(s, j)
                ledger, stats, work = _cell(world, s, cells[d][j], itr.vertices, staged[s])
                col.merge_cell(ledger, stats)
                work.add_comm(*pending[s])
                works.append(work)
            col.step(works)
            pending = [(0.0, 0) for _ in range(S)]
            if j + 1 < tt.n_columns:  # every model migrates with params + accumulator
                for d in range(tt.n_models):
                    src, dst = int(tt.server_of[d, j]), int(tt.server_of[d, j + 1])
                    col.ledger.add(src, dst, MODEL, pb, 1)
                    col.ledger.add(src, dst, GRADIENT, pb, 1)
                    pending[dst] = (pending[dst][0] + 2 * pb, pending[dst][1] + 2)
        col.trained.append([np.sort(np.concatenate(cells[d])) if cells[d] else
                            np.empty(0, dtype=np.int64) for d in range(tt.n_models)])
        col.final_sync(pb)
    return col.finish(batches_per_iter, pb)


@dataclass
class MergeEvent:
    """engine.py:770-777."""

    start_epoch: int
    epochs: int
    columns: int
    avg_seconds: float
    action: str


def _counts_for_next_epoch(world: World, tt: TraceTable, epoch: int) -> np.ndarray:
    """engine.py:836-842 (sampling-free: root counts only)."""
    batches = epoch_batches(world, epoch)[0]
    plan = redistribute_roots(batches, world.partition)
    cells = assign_cell_roots(tt, plan.groups, chain(world.cfg.seed, SEED_MERGE, epoch, 0))
    return cell_counts(cells)


def merge_controller(cfg, world: World = None, pregather: bool = True,
                     name: str = "micrograph+pg+merge"):
    """Greedy column removal on simulated epoch time (engine.py:779-833)."""
    cfg = as_run_config(cfg)
    K = cfg.merge_k
    world = world or build_world(cfg)
    tt = TraceTable.initial(world.n_servers)
    metrics, history = [], []
    epoch = 0

    def run_block(table, count):
        nonlocal epoch
        times = []
        for _ in range(count):
            m = _micrograph_epoch(world, table, epoch, pregather, name)
            metrics.append(m)
            times.append(m.sim_seconds)
            epoch += 1
        return float(np.mean(times)) if times else 0.0

    baseline = min(K, cfg.epochs)
    old = run_block(tt, baseline)
    history.append(MergeEvent(0, baseline, tt.n_columns, old, "baseline"))
    settled = False
    while not settled and epoch + K <= cfg.epochs and tt.n_columns >= 2:
        probe = tt.copy()
        probe.root_counts = _counts_for_next_epoch(world, tt, epoch)
        target = find_fewest_column(probe)
        if target is None:
            break
        tent = delete_column_and_redistribute(tt, target)
        tent.validate()
        start = epoch
        new = run_block(tent, K)
        if new < old:
            tt, old = tent, new
            history.append(MergeEvent(start, K, tt.n_columns, new, "accepted"))
        else:
            history.append(MergeEvent(start, K, tent.n_columns, new, "rejected"))
            settled = True
    if epoch < cfg.epochs:
        start = epoch
        avg = run_block(tt, cfg.epochs - epoch)
        history.append(MergeEvent(start, cfg.epochs - start, tt.n_columns, avg, "settled"))
    return metrics, tt, history


# ---------------------------------------------------------------- entry points

def run_model_centric(cfg, world: World = None) -> list:
    cfg = as_run_config(cfg)
    world = world or build_world(cfg)
    return [_model_centric_epoch(world, e) for e in range(cfg.epochs)]


def run_locality_optimized(cfg, world: World = None) -> list:
    cfg = as_run_config(cfg)
    world = world or build_world(cfg)
    return [_locality_epoch(world, e) for e in range(cfg.epochs)]


def run_micrograph(cfg, pregather: bool = False, merge: bool = False,
                   world: World = None) -> list:
    cfg = as_run_config(cfg)
    name = "micrograph" + ("+pg" if pregather else "") + ("+merge" if merge else "")
    world = world or build_world(cfg)
    if not merge:
        tt = TraceTable.initial(world.n_servers)
        return [_micrograph_epoch(world, tt, e, pregather, name) for e in range(cfg.epochs)]
    metrics, _, _ = merge_controller(cfg, world=world, pregather=pregather, name=name)
    return metrics


def run_strategy(cfg, world: World = None) -> list:
    """engine.py:849-863.  ``world`` (build_world(cfg)) may be passed to keep
    access to the trained device model."""
    cfg = as_run_config(cfg)
    s = cfg.strategy
    if s == "model-centric":
        return run_model_centric(cfg, world)
    if s == "locality-optimized":
        return run_locality_optimized(cfg, world)
    if s == "micrograph":
        return run_micrograph(cfg, pregather=False, merge=False, world=world)
    if s == "micrograph+pg":
        return run_micrograph(cfg, pregather=True, merge=False, world=world)
    if s == "micrograph+pg+merge":
        return run_micrograph(cfg, pregather=True, merge=True, world=world)
    if s == "naive":
        raise ConfigError("the naive whole-subgraph strategy (engine.py:626-763) is outside "
                          "the B200 hot path (SURVEY 8(f)4)")
    raise ConfigError(f"unknown strategy {s!r}")
