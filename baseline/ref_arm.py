"""Reference arm of bench.py: the UNMODIFIED reference timed on the host cores.

What runs is gnnsim itself (installed into baseline/_ref by
baseline/install_ref.sh), through its own public functions, per root exactly
as its engine does for one micrograph (engine.py:290-295, 434-445):

    sample_micrograph (sampler.py:84-106, numba sample_frontier)
      -> feature rows of m.vertices (FeatureStore.rows: searchsorted + take,
         featstore.py:127-136)
      -> forward (model.py:213-247) -> loss_and_backward (model.py:250-287)
      -> accumulate (model.py:161-164)

and per step one ``sync_and_update`` (model.py:299-329) over the per-worker
accumulators (the reference's all-reduce + SGD on every replica).

Scale.  gnnsim's in-memory ``Graph`` / ``FeatureStore`` cannot hold the
papers100M shape (7 GB CSR, 57 GB of fp32 features), so the bounded sample
is prepared untimed, like the reference holds its world in memory before
training: the gnnsim ``Graph`` is a full-size CSR (n + 1 offsets) whose rows
are materialised (oracle/graphgen.py rows_csr, the data generator) only for
the vertices the sampled micrographs expand -- every other row is empty and
never read -- and each worker holds the feature rows (gnnsim
``kernels.feature_rows``, the values the FeatureStore is filled with,
featstore.py:161-184) of every sampled micrograph's vertices, looked up
with ``searchsorted`` + ``take`` like ``FeatureStore.rows``.

Parallelism (all host cores, no per-step IPC of parameters or gradients):
the workers pull the step's roots in chunks of 4 from a shared counter (a
hub micrograph costs 10-100x a typical one, so static slices leave cores
idle); parameters and the per-worker gradient accumulators live in shared
memory; two barriers per step; the parent runs gnnsim's ``sync_and_update``
on the shared buffers.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def load_gnnsim():
    """gnnsim from baseline/_ref (None if not installed)."""
    if not os.path.isdir(os.path.join(REF, "gnnsim")):
        return None
    if REF not in sys.path:
        sys.path.insert(0, REF)
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "gnnsim_numba_cache"))
    import gnnsim  # noqa: F401
    from gnnsim import kernels, model, sampler, graph  # noqa: F401
    return sys.modules["gnnsim"]


def sample_roots(n: int, count: int, seed: int, step: int) -> np.ndarray:
    """The step's bounded root sample (hash order of random ids)."""
    from oracle.rng import chain, keyed
    h = keyed(chain(seed, 0x5A, step), np.arange(count, dtype=np.int64))
    return (h % np.uint64(n)).astype(np.int64)


class Workload:
    """Untimed preparation of the bounded sample of one bench config."""

    def __init__(self, cfg: dict, roots_per_step: int, steps: int):
        import gnnsim.graph as gg
        from gnnsim.rng import chain
        from gnnsim.sampler import SamplerConfig, stream_key
        from oracle.cpu_bench import LazyGraphSampler
        from oracle.graphgen import GraphSpec, rows_csr
        self.cfg = cfg
        spec = GraphSpec(**{k: cfg[k] for k in ("n", "avg_deg", "beta", "p_in", "n_blocks",
                                                 "d_cap", "seed")})
        self.n, self.B, self.steps = spec.n, int(roots_per_step), int(steps)
        seed = cfg["seed"]
        self.fanout = tuple(cfg["fanout"])
        self.scfg = SamplerConfig(len(self.fanout), self.fanout, seed=chain(seed, 0x06))
        self.roots = [sample_roots(spec.n, self.B, seed, s) for s in range(self.steps)]
        self.keys = [[stream_key(self.scfg.seed, 0, s, int(r)) for r in rs]
                     for s, rs in enumerate(self.roots)]
        # rows the micrographs expand: every layer but the last-drawn one
        lazy = LazyGraphSampler(spec)
        L = len(self.fanout)
        vs = np.unique(np.concatenate([
            lazy.expanded_vertices(self.roots[s], self.fanout, self.keys[s])
            for s in range(self.steps)]))
        off_s, tgt = rows_csr(lazy.rows.t, vs)
        deg = np.zeros(spec.n, dtype=np.int64)
        deg[vs] = np.diff(off_s)
        offsets = np.zeros(spec.n + 1, dtype=np.int64)
        np.cumsum(deg, out=offsets[1:])
        del deg
        self.graph = gg.Graph(spec.n, offsets, tgt, directed=True)
        self.rows_materialised = int(len(vs))
        self.L = L


class Shared:
    """Parameters and per-worker gradient accumulators in shared memory, viewed
    as gnnsim ModelState / GradAccumulator arrays."""

    def __init__(self, template, workers: int):
        shapes = [a.shape for a in template.params()]
        self.sizes = [int(np.prod(s)) for s in shapes]
        self.shapes = shapes
        total = sum(self.sizes)
        ctx = mp.get_context("fork")
        self.p_buf = ctx.RawArray("d", total)
        self.g_buf = ctx.RawArray("d", total * workers)
        self.total, self.workers = total, workers
        flat = np.frombuffer(self.p_buf, dtype=np.float64)
        o = 0
        for a, n in zip(template.params(), self.sizes):
            flat[o:o + n] = a.ravel()
            o += n

    def _views(self, buf, base):
        flat = np.frombuffer(buf, dtype=np.float64)
        out, o = [], base
        for s, n in zip(self.shapes, self.sizes):
            out.append(flat[o:o + n].reshape(s))
            o += n
        return out

    def model(self, arch):
        from gnnsim.model import ModelState
        v = self._views(self.p_buf, 0)
        L = (len(v) - 1) // 2
        return ModelState(arch, v[:L], v[L:2 * L], v[2 * L])

    def acc(self, w):
        from gnnsim.model import GradAccumulator, Gradients
        v = self._views(self.g_buf, w * self.total)
        L = (len(v) - 1) // 2
        return GradAccumulator(w, Gradients(v[:L], v[L:2 * L], v[2 * L]))


CHUNK = 4  # roots a worker takes per grab of the step's shared counter


def _worker(w, wl, shared, bar, ctr, arch, classes, lseed, fid, ftab):
    # one core per worker: numpy's BLAS would otherwise spawn a thread per
    # core in every worker and oversubscribe the host
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from gnnsim.model import LabelOracle, accumulate, forward, loss_and_backward
    from gnnsim.sampler import sample_micrograph
    model = shared.model(arch)
    acc = shared.acc(w)
    labels = LabelOracle(classes, lseed)
    bar.wait()  # ready
    for s in range(wl.steps):
        bar.wait()  # step s starts
        acc.reset()
        while True:  # dynamic schedule: hub micrographs cost 10-100x a typical one
            with ctr.get_lock():
                i0 = ctr.value
                ctr.value = i0 + CHUNK
            if i0 >= wl.B:
                break
            # engine.py:290-295 (sample the micrographs), then run_cell
            # (engine.py:428-445): one fetch of the unique needs, per micrograph
            # searchsorted + forward + label + backward + accumulate
            micros = [sample_micrograph(wl.graph, int(wl.roots[s][i]), wl.scfg, wl.keys[s][i])
                      for i in range(i0, min(i0 + CHUNK, wl.B))]
            needs = np.unique(np.concatenate([m.vertices for m in micros]))
            rows = ftab[np.searchsorted(fid, needs)]
            for m in micros:
                st = forward(m, rows[np.searchsorted(needs, m.vertices)], model)
                _, g = loss_and_backward(st, labels.label(m.root), model)
                accumulate(acc, g)
        bar.wait()  # step s gradients ready
        bar.wait()  # parent applied sync_and_update


def run(cfg: dict, roots_per_step: int, steps: int, warmup: int, procs: int = None):
    """Time `steps` steps after `warmup` untimed ones; returns (seeds/s, procs,
    per-step seconds, info)."""
    gs = load_gnnsim()
    if gs is None:
        raise RuntimeError("gnnsim not installed in baseline/_ref (run baseline/install_ref.sh)")
    from gnnsim.model import init_model, sync_and_update
    from gnnsim.rng import chain
    procs = procs or len(os.sched_getaffinity(0)) or 1
    t0 = time.perf_counter()
    wl = Workload(cfg, roots_per_step, warmup + steps)
    arch, dim, hidden, classes = cfg["arch"], cfg["dim"], cfg["hidden"], cfg["classes"]
    seed = cfg["seed"]
    template = init_model(arch, dim, hidden, len(wl.fanout), classes, chain(seed, 0x07))
    shared = Shared(template, procs)
    lseed = chain(seed, 0x04)
    # untimed, before the fork (shared copy-on-write by the workers): the
    # FeatureStore's rows of every vertex the sampled micrographs touch
    # (gnnsim kernels.feature_rows, the values init_features fills it with)
    import gnnsim.kernels as K
    from gnnsim.sampler import sample_micrograph
    ids = [sample_micrograph(wl.graph, int(r), wl.scfg, k).vertices
           for s in range(wl.steps) for r, k in zip(wl.roots[s], wl.keys[s])]
    fid = np.unique(np.concatenate(ids))
    del ids
    ftab = K.feature_rows(fid, dim, chain(chain(seed, 0x03), 0xFE))
    ctx = mp.get_context("fork")
    bar = ctx.Barrier(procs + 1)
    ctr = ctx.Value("q", 0)
    ps = [ctx.Process(target=_worker, args=(w, wl, shared, bar, ctr, arch, classes, lseed, fid,
                                            ftab), daemon=True) for w in range(procs)]
    for p in ps:
        p.start()
    model = shared.model(arch)
    accs = [shared.acc(w) for w in range(procs)]
    bar.wait()
    setup_s = time.perf_counter() - t0
    times = []
    try:
        for s in range(wl.steps):
            a = time.perf_counter()
            ctr.value = 0
            bar.wait()
            bar.wait()
            sync_and_update([model], accs, wl.B, 0.1)
            times.append(time.perf_counter() - a)
            bar.wait()
    finally:
        for p in ps:
            p.join(timeout=10)
    timed = times[warmup:]
    info = {"rows_materialised": wl.rows_materialised, "setup_s": round(setup_s, 1),
            "gnnsim_backend": gs.kernels.BACKEND}
    return wl.B * len(timed) / sum(timed), procs, timed, info
