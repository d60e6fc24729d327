"""Bit-exact parity of the CUDA sampling / graph / RNG path with the oracle
(which tests/test_oracle_golden.py pins to the reference's own outputs)."""
import numpy as np
import pytest
import torch

from oracle import engine as OE
from oracle import kernels as OK
from oracle import model as OM
from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables
from oracle.rng import chain, mix64
from oracle.sampler import sample_micrograph as o_sample, stream_key

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2409_00657_b200 as P
    from paper_2409_00657_b200 import graph, kernels, sampler  # noqa: F401
    return P


SPECS = [dict(n=3000, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4, d_cap=600, seed=11),
         dict(n=20000, avg_deg=20.0, beta=0.8, p_in=0.8, n_blocks=8, d_cap=5000, seed=5),
         dict(n=500, avg_deg=3.0, beta=0.5, p_in=1.0, n_blocks=1, d_cap=40, seed=1)]


@pytest.mark.parametrize("kw", SPECS, ids=["small", "hubs", "oneblock"])
def test_generator_matches_oracle(P, kw):
    from paper_2409_00657_b200.graph import GraphSpec, generate
    g = generate(GraphSpec(**kw))
    off, tgt = g.to_host()
    o_off, o_tgt = build_csr(build_tables(OSpec(**kw)))
    assert np.array_equal(off, o_off)
    assert np.array_equal(tgt, o_tgt)


def test_generator_chunked_sort_matches(P):
    from paper_2409_00657_b200.graph import GraphSpec, generate
    kw = SPECS[1]
    a = generate(GraphSpec(**kw))
    b = generate(GraphSpec(**kw), chunk_slots=1000)
    assert torch.equal(a.offsets, b.offsets) and torch.equal(a.targets, b.targets)


def test_sample_frontier_golden(P, golden):
    from paper_2409_00657_b200 import kernels
    g = golden("kernels")
    for f in (1, 3, 10, 15, 25):
        for si, st in enumerate(g["states"].tolist()):
            c, fl = kernels.sample_frontier(g["offsets"], g["targets"], g["frontier"], f, st)
            assert np.array_equal(c, g[f"counts_f{f}_s{si}"])
            assert np.array_equal(fl, g[f"flat_f{f}_s{si}"])
    c, fl = kernels.sample_frontier(g["star_offsets"], g["star_targets"], np.array([0]), 5,
                                    chain(7, 1))
    assert fl.tolist() == [6, 14, 29, 30, 32]


def test_sample_frontier_hubs_vs_oracle(P):
    from paper_2409_00657_b200 import kernels
    from paper_2409_00657_b200.graph import GraphSpec, generate
    kw = SPECS[1]
    g = generate(GraphSpec(**kw))
    off, tgt = g.to_host()
    deg = np.diff(off)
    frontier = np.concatenate([np.argsort(-deg)[:40], np.arange(0, kw["n"], 331)])
    for fo in (1, 2, 5, 15, 40):
        st = chain(3, fo)
        c, fl = kernels.sample_frontier(g.offsets, g.targets, frontier, fo, st)
        oc, ofl = OK.sample_frontier(off, tgt, frontier, fo, st)
        assert np.array_equal(c, oc) and np.array_equal(fl, ofl)


def test_feature_rows_golden(P, golden):
    from paper_2409_00657_b200 import kernels
    g = golden("kernels")
    st = int(g["feat_state"][0])
    assert np.array_equal(kernels.feature_rows(g["feat_ids"], 128, st), g["feat_rows_128"])
    assert np.array_equal(kernels.feature_rows(g["feat_ids"], 17, chain(11, 0xFE)),
                          g["feat_rows_17"])


FANOUTS = {"f1": (7,), "f2": (15, 10), "f3": (10, 10, 10), "f4": (10, 10, 5, 5), "f2s": (10, 5)}


@pytest.mark.parametrize("name", sorted(FANOUTS))
def test_micrographs_and_plans_golden(P, golden, name):
    from paper_2409_00657_b200.graph import Graph
    from paper_2409_00657_b200.sampler import (MicrographBuilder, SamplerConfig,
                                               sample_micrograph)
    g = golden("micrographs")
    G = Graph.from_host(g["offsets"], g["targets"])
    seed = int(g["seed"][0])
    fo = FANOUTS[name]
    roots = g["roots"]
    # single-root drop-in
    m0 = sample_micrograph(G, int(roots[0]), SamplerConfig(len(fo), fo, seed=seed),
                           stream_key(seed, 1, 2, int(roots[0])))
    assert np.array_equal(m0.vertices, g[f"{name}_r{int(roots[0])}_verts"])
    # batched builder with device-folded keys
    b = MicrographBuilder(fo, len(roots))
    st = torch.tensor([np.uint64(chain(seed, 1, 2)).view(np.int64)], device="cuda")
    batch = b.build(G, torch.from_numpy(roots).cuda(), st, len(roots))
    torch.cuda.synchronize()
    b.check()
    ms = batch.micrographs(roots)
    for i, r in enumerate(roots.tolist()):
        m = ms[i]
        pre = f"{name}_r{r}_"
        assert np.array_equal(np.concatenate(m.layers), g[pre + "layers"])
        assert np.array_equal(np.cumsum([0] + [len(x) for x in m.layers]), g[pre + "lay_off"])
        assert np.array_equal(np.concatenate([p[0] for p in m.pairs]), g[pre + "pd"])
        assert np.array_equal(np.concatenate([p[1] for p in m.pairs]), g[pre + "ps"])
        assert np.array_equal(m.vertices, g[pre + "verts"])
        need, steps = batch.plans(i)
        for k, nd in enumerate(need):
            assert np.array_equal(nd, g[pre + f"need{k}"])
        for k, (sp, dp, spp, dg) in enumerate(steps, start=1):
            assert np.array_equal(sp, g[pre + f"self{k}"])
            assert np.array_equal(dp, g[pre + f"dpos{k}"])
            assert np.array_equal(spp, g[pre + f"spos{k}"])
            assert np.array_equal(dg, g[pre + f"deg{k}"])


@pytest.mark.parametrize("fo", [(15, 10), (10, 10, 5, 5), (25, 3)])
def test_batch_vs_oracle_on_hub_graph(P, fo):
    from paper_2409_00657_b200.graph import GraphSpec, generate
    from paper_2409_00657_b200.sampler import MicrographBuilder
    kw = SPECS[1]
    G = generate(GraphSpec(**kw))
    off, tgt = G.to_host()
    deg = np.diff(off)
    rng = np.random.default_rng(0)
    roots = np.concatenate([np.argsort(-deg)[:16], rng.integers(0, kw["n"], 240)]).astype(np.int64)
    seed = chain(9, 0x06)
    b = MicrographBuilder(fo, len(roots))
    st = torch.tensor([np.uint64(chain(seed, 0, 7)).view(np.int64)], device="cuda")
    batch = b.build(G, torch.from_numpy(roots).cuda(), st, len(roots))
    torch.cuda.synchronize()
    b.check()
    got = batch.micrographs(roots)
    for r, m in zip(roots.tolist(), got):
        want = o_sample(off, tgt, r, fo, stream_key(seed, 0, 7, r), draw=OK.sample_frontier_nb)
        for a, w in zip(m.layers, want.layers):
            assert np.array_equal(a, w)
        for (d1, s1), (d2, s2) in zip(m.pairs, want.pairs):
            assert np.array_equal(d1, d2) and np.array_equal(s1, s2)
        assert np.array_equal(m.vertices, want.vertices)


def test_isolated_root_and_range_error(P):
    from paper_2409_00657_b200.graph import Graph
    from paper_2409_00657_b200.sampler import SamplerConfig, sample_micrograph
    G = Graph.from_host(np.array([0, 0, 1, 2]), np.array([2, 1]))
    m = sample_micrograph(G, 0, SamplerConfig(2, (2, 2)), stream_key(0, 0, 0, 0))
    assert m.vertex_count == 1 and all(len(d) == 0 for d, _ in m.pairs)
    with pytest.raises(ValueError, match="out of range"):
        sample_micrograph(G, 3, SamplerConfig(1, (2,)), 0)


def test_epoch_permutation_matches_oracle(P):
    from paper_2409_00657_b200.batching import epoch_permutation
    for n in (1, 1000, 100_003):
        perm = epoch_permutation(5, 0, n)
        assert np.array_equal(perm.cpu().numpy(), OE.epoch_permutation(5, 0, n))


def test_glorot_matches_oracle(P):
    from paper_2409_00657_b200.model import glorot_device
    for rows, cols, st in ((256, 256, chain(3, 0x11, 0)), (7, 5, 99)):
        w = glorot_device(rows, cols, st, torch.float64).cpu().numpy()
        assert np.array_equal(w, OM.glorot(rows, cols, st))


# ---------------------------------------------------------------- build kernels
# Two-layer micrographs with f1 <= 31 and f1*f2 <= 256 are built warp-per-root
# (k_mg_build_w2); hg_mg_build_mode(1) forces the CTA-per-root kernel.  Both
# must agree with each other and with the oracle, including hub rows above the
# warp draw limit (1024), self-loops (root inside its own layer 1), isolated
# roots, device root counts (empty micrographs) and the persistent grid.

def _build_both(G, fo, roots, state, n_dev=None, ctas_per_sm=0):
    from paper_2409_00657_b200 import _lib
    from paper_2409_00657_b200.sampler import GroupBuilder, MicrographBatch, MicrographBuilder
    out = []
    for mode in (0, 1):
        _lib.call("hg_mg_build_mode", mode)
        try:
            R = len(roots) // 2
            bs = [MicrographBuilder(fo, R) for _ in range(2)]
            gb = GroupBuilder(bs)
            gb.roots.copy_(torch.from_numpy(roots).cuda())
            gb.keys.copy_(torch.tensor(np.array([state, chain(state, 1)], dtype=np.uint64)
                                       .view(np.int64), device="cuda"))
            if n_dev is not None:
                gb.n_dev.copy_(torch.tensor(n_dev, dtype=torch.int32))
            gb.build(G, n_dev=gb.n_dev.data_ptr() if n_dev is not None else None,
                     ctas_per_sm=ctas_per_sm)
            torch.cuda.synchronize()
            gb.check()
            out.append([(b.tensors, MicrographBatch(len(fo), R, b.tensors)) for b in bs])
        finally:
            _lib.call("hg_mg_build_mode", 0)
    return out


@pytest.mark.parametrize("fo", [(15, 10), (10, 5), (25, 10), (31, 8), (1, 200), (3, 1)])
@pytest.mark.parametrize("cps", [0, 3])
def test_warp_build_matches_cta_build_and_oracle(P, fo, cps):
    from paper_2409_00657_b200.graph import GraphSpec, generate
    kw = SPECS[1]  # rows up to 5000: hop-1 and hop-2 hubs above the warp limit
    G = generate(GraphSpec(**kw))
    off, tgt = G.to_host()
    deg = np.diff(off)
    rng = np.random.default_rng(3)
    roots = np.concatenate([np.argsort(-deg)[:24], rng.integers(0, kw["n"], 176)]).astype(np.int64)
    rng.shuffle(roots)
    state = chain(chain(5, 0x06), 0, 9)
    fast, legacy = _build_both(G, fo, roots, state, ctas_per_sm=cps)
    R = len(roots) // 2
    for b in range(2):
        (tf, bf), (tl, bl) = fast[b], legacy[b]
        assert torch.equal(tf["totals"], tl["totals"])
        hf, hl = bf.to_host(), bl.to_host()
        for name in ("need_off", "pair_off"):
            for k in range(len(fo) + 1):
                if hf[name][k] is not None:
                    assert np.array_equal(hf[name][k], hl[name][k]), (name, k)
        tot = tf["totals"].cpu().numpy()
        L = len(fo)
        for k in range(L + 1):
            n = int(tot[k])
            assert np.array_equal(hf["need_ids"][k][:n], hl["need_ids"][k][:n]), ("need", k)
            assert np.array_equal(hf["in_layer"][k][:n], hl["in_layer"][k][:n]), ("inl", k)
            if k:
                p = int(tot[L + k])
                assert np.array_equal(hf["self_pos"][k][:n], hl["self_pos"][k][:n])
                assert np.array_equal(hf["nbr_off"][k][:n + 1], hl["nbr_off"][k][:n + 1])
                assert np.array_equal(hf["nbr_idx"][k][:p], hl["nbr_idx"][k][:p])
        st = state if b == 0 else chain(state, 1)
        rb = roots[b * R:(b + 1) * R]
        for r, m in zip(rb.tolist(), bf.micrographs(rb, hf)):
            want = o_sample(off, tgt, r, fo, mix64(st ^ r), draw=OK.sample_frontier_nb)
            assert all(np.array_equal(a, w) for a, w in zip(m.layers, want.layers))
            assert all(np.array_equal(d1, d2) and np.array_equal(s1, s2)
                       for (d1, s1), (d2, s2) in zip(m.pairs, want.pairs))
            assert np.array_equal(m.vertices, want.vertices)


def test_warp_build_self_loops_isolated_and_device_counts(P):
    """Self-loops put the root into its own layer 1 (need[1] == layer 1),
    isolated roots give |V| = 1, and batch slots past the device root count
    come out as empty micrographs -- the same in both kernels."""
    from paper_2409_00657_b200.graph import Graph
    rng = np.random.default_rng(11)
    n = 300
    rows = []
    for v in range(n):
        if v % 17 == 0:
            rows.append(np.empty(0, np.int64))           # isolated
            continue
        d = int(rng.integers(1, 60 if v % 5 else 1500))
        r = np.unique(rng.integers(0, n, d))
        if v % 3 == 0:
            r = np.union1d(r, [v])                        # self-loop
        rows.append(r)
    off = np.zeros(n + 1, np.int64)
    np.cumsum([len(r) for r in rows], out=off[1:])
    tgt = np.concatenate(rows)
    G = Graph.from_host(off, tgt)
    roots = rng.integers(0, n, 128).astype(np.int64)
    roots[:8] = np.arange(0, 8 * 17, 17)                  # isolated roots
    fo = (15, 10)
    state = chain(3, 4)
    fast, legacy = _build_both(G, fo, roots, state, n_dev=[64, 37])
    for b, cnt in ((0, 64), (1, 37)):
        tf, tl = fast[b][0], legacy[b][0]
        assert torch.equal(tf["totals"], tl["totals"])
        for name in ("need_ids", "in_layer", "self_pos", "nbr_idx"):
            for k in range(3):
                x, y = tf[name][k], tl[name][k]
                if x is None:
                    continue
                n_ = int(tf["totals"][k]) if name != "nbr_idx" else int(tf["totals"][2 + k])
                assert torch.equal(x[:n_], y[:n_]), (b, name, k)
        bf = fast[b][1]
        rb = roots[b * 64:b * 64 + cnt]
        got = bf.micrographs(rb)
        for r, m in zip(rb.tolist(), got):
            want = o_sample(off, tgt, r, fo, mix64((state if b == 0 else chain(state, 1)) ^ r))
            assert all(np.array_equal(a, w) for a, w in zip(m.layers, want.layers))
            assert np.array_equal(m.vertices, want.vertices)
        # slots past the device count: empty micrographs
        no = tf["need_off"][0].cpu().numpy()
        assert no[cnt] == no[64]


@pytest.mark.parametrize("fo", [(15, 10), (10, 10, 5, 5)])
@pytest.mark.parametrize("kind,S", [("blocks", 2), ("blocks", 8), ("hash", 3)])
def test_sharded_csr_build_matches_replicated(P, fo, kind, S):
    """Partitioned topology (graph.ShardedGraph): rows addressed per home shard
    (contiguous ranges or home/local-row arrays) build exactly what the
    replicated CSR builds -- both kernels, single and grouped builds."""
    from paper_2409_00657_b200.graph import (GraphSpec, PartitionMap, ShardedGraph, generate,
                                             partition_hash)
    from paper_2409_00657_b200.sampler import GroupBuilder, MicrographBuilder
    kw = SPECS[1]
    G = generate(GraphSpec(**kw))
    n = kw["n"]
    part = (PartitionMap((np.arange(n) * S) // n, S) if kind == "blocks"
            else partition_hash(n, S, 5))
    SG = ShardedGraph.split_local(G, part)
    assert SG.contiguous == (kind == "blocks")
    deg = np.diff(G.to_host()[0])
    roots = np.concatenate([np.argsort(-deg)[:16],
                            np.random.default_rng(S).integers(0, n, 112)]).astype(np.int64)
    st = torch.tensor([np.uint64(chain(7, S)).view(np.int64), np.uint64(chain(8, S)).view(np.int64)],
                      device="cuda")
    outs = []
    for g in (G, SG):
        bs = [MicrographBuilder(fo, 64) for _ in range(2)]
        gb = GroupBuilder(bs)
        gb.roots.copy_(torch.from_numpy(roots).cuda())
        gb.keys.copy_(st)
        gb.build(g, ctas_per_sm=2)
        single = MicrographBuilder(fo, 64)
        single.build(g, torch.from_numpy(roots[:64]).cuda(), st[:1], 64)
        torch.cuda.synchronize()
        gb.check()
        single.check()
        outs.append([b.tensors for b in bs] + [single.tensors])
    for a, b in zip(*outs):
        assert torch.equal(a["totals"], b["totals"])
        L = len(fo)
        for k in range(L + 1):
            nk = int(a["totals"][k])
            assert torch.equal(a["need_ids"][k][:nk], b["need_ids"][k][:nk])
            if k:
                p = int(a["totals"][L + k])
                assert torch.equal(a["nbr_idx"][k][:p], b["nbr_idx"][k][:p])
                assert torch.equal(a["nbr_off"][k][:nk + 1], b["nbr_off"][k][:nk + 1])
