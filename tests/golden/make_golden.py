"""Generate golden vectors by running the REFERENCE implementation (gnnsim).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb \
        python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  Inputs come from this repo's own synthetic
generator (oracle/graphgen.py) so the same CSR can be rebuilt anywhere; all
outputs are computed by ``gnnsim`` itself.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.environ.get("GNNSIM_SRC", "/root/reference/pkg/src"))

import gnnsim.engine as E  # noqa: E402
from gnnsim import kernels  # noqa: E402
from gnnsim.config import RunConfig  # noqa: E402
from gnnsim.engine import CostModel, SimWorld, TraceTable  # noqa: E402
from gnnsim.featstore import init_features  # noqa: E402
from gnnsim.graph import Graph, PartitionMap, from_pairs, partition_hash  # noqa: E402
from gnnsim.model import (LabelOracle, build_plan, forward, init_model,  # noqa: E402
                          loss_and_backward)
from gnnsim.rng import chain, hash_vec, mix64, uniform01_f64_vec  # noqa: E402
from gnnsim.sampler import SamplerConfig, sample_micrograph, stream_key  # noqa: E402

from oracle.graphgen import GraphSpec, build_csr, build_tables  # noqa: E402

OUT = HERE


def small_graph(n=3000, seed=11, beta=0.7, avg=12.0, cap=600):
    t = build_tables(GraphSpec(n=n, avg_deg=avg, beta=beta, p_in=0.9, n_blocks=4,
                               d_cap=cap, seed=seed))
    return build_csr(t)


def flat_micro(m):
    """Pack a Micrograph as flat arrays + offsets."""
    lay = list(m.layers)
    lay_off = np.cumsum([0] + [len(x) for x in lay])
    pd = [p[0] for p in m.pairs]
    ps = [p[1] for p in m.pairs]
    p_off = np.cumsum([0] + [len(x) for x in pd])
    return (np.concatenate(lay), lay_off, np.concatenate(pd) if pd else np.empty(0, np.int64),
            np.concatenate(ps) if ps else np.empty(0, np.int64), p_off, m.vertices)


def gen_rng():
    xs = np.array([0, 1, 2, 12345, 2**63, 2**64 - 1, 0xDEADBEEF], dtype=np.uint64)
    mixes = np.array([mix64(int(x)) for x in xs], dtype=np.uint64)
    chains = np.array([chain(1, 2), chain(0, 6), chain(7, 0, 0, 0), chain(3, 0xFE),
                       chain(chain(0, 3), 0xFE), chain(9, 5, 4, 3, 2, 1)], dtype=np.uint64)
    hv = hash_vec(chain(42, 7), np.arange(64))
    u = uniform01_f64_vec(hv)
    perm = np.argsort(hash_vec(chain(5, 0x05, 0), np.arange(1000)), kind="stable")
    np.savez(os.path.join(OUT, "rng.npz"), xs=xs, mixes=mixes, chains=chains, hv=hv, u=u,
             perm=perm)


def gen_kernels():
    offsets, targets = small_graph()
    deg = np.diff(offsets)
    frontier = np.concatenate([np.argsort(-deg)[:8], np.arange(0, 3000, 97)]).astype(np.int64)
    res = {"offsets": offsets, "targets": targets, "frontier": frontier}
    for f in (1, 3, 10, 15, 25):
        for si, st in enumerate((chain(1, 2), chain(99, 1), 0)):
            c, fl = kernels.sample_frontier(offsets, targets, frontier, f, st)
            res[f"counts_f{f}_s{si}"] = c
            res[f"flat_f{f}_s{si}"] = fl
    res["states"] = np.array([chain(1, 2), chain(99, 1), 0], dtype=np.uint64)
    ids = np.array([0, 1, 2, 3, 999, 123456, 110_999_999], dtype=np.int64)
    res["feat_ids"] = ids
    res["feat_state"] = np.array([chain(chain(0, 3), 0xFE)], dtype=np.uint64)
    res["feat_rows_128"] = kernels.feature_rows(ids, 128, chain(chain(0, 3), 0xFE))
    res["feat_rows_17"] = kernels.feature_rows(ids, 17, chain(11, 0xFE))
    pk_ids = np.sort(np.random.default_rng(3).choice(100000, 500, replace=False)).astype(np.int64)
    res["pk_ids"] = pk_ids
    for k in (1, 7, 100, 499, 500, 600):
        res[f"pk_{k}"] = kernels.pick_k_smallest(pk_ids, k, chain(5))
    # the star of SURVEY appendix A
    star = from_pairs(41, np.zeros(40, dtype=np.int64), np.arange(1, 41))
    res["star_offsets"], res["star_targets"] = star.offsets, star.targets
    c, fl = kernels.sample_frontier(star.offsets, star.targets, np.array([0]), 5, chain(7, 1))
    res["star_flat"] = fl
    np.savez(os.path.join(OUT, "kernels.npz"), **res)


def gen_micrographs():
    offsets, targets = small_graph()
    g = Graph(len(offsets) - 1, offsets, targets)
    res = {"offsets": offsets, "targets": targets}
    fanouts = {"f1": (7,), "f2": (15, 10), "f3": (10, 10, 10), "f4": (10, 10, 5, 5),
               "f2s": (10, 5)}
    roots = np.array([0, 1, 5, 17, 123, 2999, 1500, 777, 42, 2048], dtype=np.int64)
    deg = np.diff(offsets)
    roots = np.concatenate([roots, np.argsort(-deg)[:3]]).astype(np.int64)
    res["roots"] = roots
    seed = chain(3, 0x06)
    res["seed"] = np.array([seed], dtype=np.uint64)
    for name, fo in fanouts.items():
        cfg = SamplerConfig(len(fo), fo, seed=seed)
        for r in roots.tolist():
            m = sample_micrograph(g, r, cfg, stream_key(seed, 1, 2, r))
            lay, lay_off, pd, ps, p_off, verts = flat_micro(m)
            pre = f"{name}_r{r}_"
            res[pre + "layers"], res[pre + "lay_off"] = lay, lay_off
            res[pre + "pd"], res[pre + "ps"], res[pre + "p_off"] = pd, ps, p_off
            res[pre + "verts"] = verts
            plan = build_plan(m)
            for k, (sp, dp, spp, dg) in enumerate(plan.layers, start=1):
                res[pre + f"self{k}"], res[pre + f"dpos{k}"] = sp, dp
                res[pre + f"spos{k}"], res[pre + f"deg{k}"] = spp, dg
            for k, nd in enumerate(plan.need):
                res[pre + f"need{k}"] = nd
    np.savez_compressed(os.path.join(OUT, "micrographs.npz"), **res)


def gen_model():
    offsets, targets = small_graph()
    g = Graph(len(offsets) - 1, offsets, targets)
    res = {}
    seed = chain(4, 0x06)
    fstate = chain(chain(4, 0x03), 0xFE)
    for arch, fo, dim, hid, C in (("sage-mean", (15, 10), 24, 16, 7),
                                  ("gcn", (10, 10, 10), 20, 12, 5),
                                  ("sage-mean", (10, 10, 5, 5), 16, 8, 4)):
        cfg = SamplerConfig(len(fo), fo, seed=seed)
        model = init_model(arch, dim, hid, len(fo), C, chain(4, 0x07))
        lo = LabelOracle(C, chain(4, 0x04))
        tag = f"{arch}_{len(fo)}"
        for i, p in enumerate(model.params()):
            res[f"{tag}_init{i}"] = p
        for r in (3, 100, 2222):
            m = sample_micrograph(g, r, cfg, stream_key(seed, 0, 0, r))
            x = kernels.feature_rows(m.vertices, dim, fstate)
            st = forward(m, x, model)
            loss, gr = loss_and_backward(st, lo.label(r), model)
            res[f"{tag}_r{r}_logits"] = st.logits
            res[f"{tag}_r{r}_loss"] = np.array([loss])
            res[f"{tag}_r{r}_label"] = np.array([lo.label(r)])
            for i, a in enumerate(gr.arrays()):
                res[f"{tag}_r{r}_g{i}"] = a
    res["labels_C172"] = LabelOracle(172, chain(4, 0x04)).labels(np.arange(1000))
    np.savez_compressed(os.path.join(OUT, "model.npz"), **res)


def _world(S, arch, fo, dim, hid, C, batch, seed, iters, part="hash", n=3000):
    offsets, targets = small_graph(n=n)
    g = Graph(len(offsets) - 1, offsets, targets)
    if part == "hash":
        p = partition_hash(g, S, chain(seed, 0x02))
    else:  # planted blocks (4 blocks in small_graph) -> S servers
        blocks = (np.arange(g.n_vertices) * 4) // g.n_vertices
        p = PartitionMap((blocks * S) // 4, S)
    cfg = RunConfig(graph="x.csr", servers=S, partitioner="file", partition_file="x",
                    layers=len(fo), fanout=fo, dim=dim, hidden=hid, classes=C, arch=arch,
                    batch=batch, epochs=1, iterations=iters, seed=seed)
    fs = init_features(p, dim, seed=chain(seed, 0x03))
    lab = LabelOracle(C, chain(seed, 0x04))
    scfg = SamplerConfig(len(fo), fo, "node-wise", chain(seed, 0x06))
    return SimWorld(cfg, g, p, fs, lab, scfg, CostModel()), p.home


def gen_engine():
    res = {}
    cases = [("mg2", 2, "sage-mean", (15, 10), 16, 8, 5, 64, 1, 2, "hash"),
             ("mg4", 4, "sage-mean", (10, 5), 12, 8, 4, 32, 2, 2, "blocks"),
             ("mg4g", 4, "gcn", (5, 5, 5), 8, 8, 3, 16, 3, 1, "blocks"),
             ("mg1", 1, "sage-mean", (15, 10), 16, 8, 5, 128, 4, 2, "hash")]
    for tag, S, arch, fo, dim, hid, C, B, seed, iters, part in cases:
        for strat in ("model-centric", "micrograph", "micrograph+pg"):
            world, home = _world(S, arch, fo, dim, hid, C, B, seed, iters, part)
            models = E.fresh_models(world)
            if strat == "model-centric":
                m = E._model_centric_epoch(world, models, 0)
            else:
                m = E._micrograph_epoch(world, models, TraceTable.initial(S), 0,
                                        strat.endswith("pg"), strat)
            key = f"{tag}_{strat}"
            cats = sorted(m.bytes_by_category)
            res[key + "_cats"] = np.array(cats)
            res[key + "_bytes"] = np.array([m.bytes_by_category[c] for c in cats])
            links = sorted(m.ledger.counters.items())
            res[key + "_links"] = np.array([[s, d] for (s, d, _), _ in links], dtype=np.int64).reshape(-1, 2)
            res[key + "_linkcat"] = np.array([c for (_, _, c), _ in links])
            res[key + "_linkbytes"] = np.array([v[0] for _, v in links], dtype=np.float64)
            res[key + "_linkmsgs"] = np.array([v[1] for _, v in links], dtype=np.int64)
            res[key + "_miss"] = np.array([m.miss_rate])
            for i, p in enumerate(models[0].params()):
                res[key + f"_p{i}"] = p
        res[tag + "_home"] = home
        res[tag + "_cfg"] = np.array([S, len(fo), *fo, dim, hid, C, B, seed, iters])
        res[tag + "_arch"] = np.array([arch])
        batches = E.epoch_batches(world, 0)
        res[tag + "_batches"] = np.array([np.concatenate(b) for b in batches])
    # epoch permutation + merge replay
    part = PartitionMap(np.arange(40, dtype=np.int64) % 4, 4)
    from gnnsim.sampler import redistribute_roots
    batches = [np.arange(d * 10, (d + 1) * 10, dtype=np.int64) for d in range(4)]
    plan = redistribute_roots(batches, part)
    tt = TraceTable.initial(4)
    cells = E.assign_cell_roots(tt, plan, key=7)
    tt.root_counts = E.cell_counts(cells)
    tt2 = E.delete_column_and_redistribute(tt, 2)
    tt3 = E.delete_column_and_redistribute(tt2, 0)
    for name, t in (("tt2", tt2), ("tt3", tt3)):
        cl = E.assign_cell_roots(t, plan, key=7)
        res[name + "_removed"] = np.array(t.removed)
        res[name + "_flat"] = np.concatenate([np.concatenate([c, [-1]]) for row in cl for c in row])
        res[name + "_counts"] = t.root_counts
    np.savez(os.path.join(OUT, "engine.npz"), **res)


def gen_fixture_world():
    """The 8-vertex walkthrough (test_engine.py:24-49) ledger numbers."""
    cfg = RunConfig(servers=2, layers=2, fanout=(2,), dim=4, hidden=4, classes=2, batch=2, epochs=1)
    graph = from_pairs(8, np.array([5, 6, 1, 0, 2, 3]), np.array([6, 7, 5, 1, 3, 4]))
    part = PartitionMap(np.array([1, 1, 1, 1, 0, 0, 0, 0]), 2)
    world = SimWorld(cfg, graph, part, init_features(part, 4, seed=1), LabelOracle(2, 2),
                     SamplerConfig(2, (2, 2), "node-wise", 3), CostModel())
    E.epoch_batches = lambda w, e: [[np.array([6, 3]), np.array([5, 0])]]
    out = {"offsets": graph.offsets, "targets": graph.targets, "home": part.home}
    mc = E._model_centric_epoch(world, E.fresh_models(world), 0)
    mg = E._micrograph_epoch(world, E.fresh_models(world), TraceTable.initial(2), 0, False, "mg")
    pg = E._micrograph_epoch(world, E.fresh_models(world), TraceTable.initial(2), 0, True, "pg")
    for k, m in (("mc", mc), ("mg", mg), ("pg", pg)):
        out[k + "_rows_1_0"] = np.array([m.ledger.link(1, 0, "feature")[0] / 16])
        out[k + "_rows_0_1"] = np.array([m.ledger.link(0, 1, "feature")[0] / 16])
    np.savez(os.path.join(OUT, "fixture_world.npz"), **out)


if __name__ == "__main__":
    gen_rng()
    gen_kernels()
    gen_micrographs()
    gen_model()
    gen_engine()
    gen_fixture_world()
    print("golden vectors written to", OUT)
