"""Pin the CPU oracle to golden vectors produced by the reference (gnnsim).

The golden files were made by tests/golden/make_golden.py running the
reference itself; this file runs anywhere (no reference, no GPU).
"""
import numpy as np
import pytest

from oracle import engine as OE
from oracle import kernels as OK
from oracle import model as OM
from oracle.graphgen import GraphSpec, build_csr, build_tables
from oracle.rng import chain, keyed, mix64, unit_f64
from oracle.sampler import sample_micrograph, stream_key


def test_rng_golden(golden):
    g = golden("rng")
    assert [mix64(int(x)) for x in g["xs"]] == g["mixes"].tolist()
    want = [chain(1, 2), chain(0, 6), chain(7, 0, 0, 0), chain(3, 0xFE),
            chain(chain(0, 3), 0xFE), chain(9, 5, 4, 3, 2, 1)]
    assert want == g["chains"].tolist()
    hv = keyed(chain(42, 7), np.arange(64))
    assert np.array_equal(hv, g["hv"])
    assert np.array_equal(unit_f64(hv), g["u"])
    perm = OE.epoch_permutation(5, 0, 1000)
    assert np.array_equal(perm, g["perm"])
    # SURVEY appendix A constants
    assert mix64(0) == 0xE220A8397B1DCDAF
    assert chain(1, 2) == 0xBCD9DBB49673066B


def test_small_graph_rebuilds_identically(golden):
    g = golden("kernels")
    t = build_tables(GraphSpec(n=3000, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4,
                               d_cap=600, seed=11))
    off, tgt = build_csr(t)
    assert np.array_equal(off, g["offsets"]) and np.array_equal(tgt, g["targets"])


def test_sample_frontier_golden(golden):
    g = golden("kernels")
    for f in (1, 3, 10, 15, 25):
        for si, st in enumerate(g["states"].tolist()):
            c, fl = OK.sample_frontier(g["offsets"], g["targets"], g["frontier"], f, st)
            assert np.array_equal(c, g[f"counts_f{f}_s{si}"])
            assert np.array_equal(fl, g[f"flat_f{f}_s{si}"])
            if OK.HAVE_NUMBA:
                c2, fl2 = OK.sample_frontier_nb(g["offsets"], g["targets"], g["frontier"], f, st)
                assert np.array_equal(c2, c) and np.array_equal(fl2, fl)
    c, fl = OK.sample_frontier(g["star_offsets"], g["star_targets"], np.array([0]), 5, chain(7, 1))
    assert fl.tolist() == [6, 14, 29, 30, 32] == g["star_flat"].tolist()


def test_feature_rows_and_pick_golden(golden):
    g = golden("kernels")
    st = int(g["feat_state"][0])
    assert np.array_equal(OK.feature_rows(g["feat_ids"], 128, st), g["feat_rows_128"])
    assert np.array_equal(OK.feature_rows(g["feat_ids"], 17, chain(11, 0xFE)), g["feat_rows_17"])
    for k in (1, 7, 100, 499, 500, 600):
        assert np.array_equal(OK.pick_k_smallest(g["pk_ids"], k, chain(5)), g[f"pk_{k}"])


FANOUTS = {"f1": (7,), "f2": (15, 10), "f3": (10, 10, 10), "f4": (10, 10, 5, 5), "f2s": (10, 5)}


@pytest.mark.parametrize("name", sorted(FANOUTS))
def test_micrographs_and_plans_golden(golden, name):
    g = golden("micrographs")
    seed = int(g["seed"][0])
    fo = FANOUTS[name]
    for r in g["roots"].tolist():
        m = sample_micrograph(g["offsets"], g["targets"], r, fo, stream_key(seed, 1, 2, r))
        pre = f"{name}_r{r}_"
        assert np.array_equal(np.concatenate(m.layers), g[pre + "layers"])
        assert np.array_equal(np.cumsum([0] + [len(x) for x in m.layers]), g[pre + "lay_off"])
        assert np.array_equal(np.concatenate([p[0] for p in m.pairs]), g[pre + "pd"])
        assert np.array_equal(np.concatenate([p[1] for p in m.pairs]), g[pre + "ps"])
        assert np.array_equal(m.vertices, g[pre + "verts"])
        need, steps = OM.build_plan(m)
        for k, nd in enumerate(need):
            assert np.array_equal(nd, g[pre + f"need{k}"])
        for k, (sp, dp, spp, dg) in enumerate(steps, start=1):
            assert np.array_equal(sp, g[pre + f"self{k}"])
            assert np.array_equal(dp, g[pre + f"dpos{k}"])
            assert np.array_equal(spp, g[pre + f"spos{k}"])
            assert np.array_equal(dg, g[pre + f"deg{k}"])


MODEL_CASES = (("sage-mean", (15, 10), 24, 16, 7), ("gcn", (10, 10, 10), 20, 12, 5),
               ("sage-mean", (10, 10, 5, 5), 16, 8, 4))


@pytest.mark.parametrize("case", MODEL_CASES, ids=lambda c: f"{c[0]}-{len(c[1])}")
def test_model_forward_backward_golden(golden, case):
    arch, fo, dim, hid, C = case
    g = golden("model")
    kg = golden("kernels")
    tag = f"{arch}_{len(fo)}"
    P = OM.init_params(arch, dim, hid, len(fo), C, chain(4, 0x07))
    for i, a in enumerate(P.arrays()):
        assert np.array_equal(a, g[f"{tag}_init{i}"])
    seed = chain(4, 0x06)
    fstate = chain(chain(4, 0x03), 0xFE)
    for r in (3, 100, 2222):
        m = sample_micrograph(kg["offsets"], kg["targets"], r, fo, stream_key(seed, 0, 0, r))
        x = OK.feature_rows(m.vertices, dim, fstate)
        st = OM.forward(m, x, P)
        lab = int(OM.labels([r], C, chain(4, 0x04))[0])
        assert lab == int(g[f"{tag}_r{r}_label"][0])
        loss, G = OM.loss_and_grads(st, lab, P)
        np.testing.assert_allclose(st["logits"], g[f"{tag}_r{r}_logits"], rtol=1e-12, atol=1e-14)
        assert abs(loss - g[f"{tag}_r{r}_loss"][0]) <= 1e-12 * max(1.0, abs(loss))
        for i, a in enumerate(G.arrays()):
            np.testing.assert_allclose(a, g[f"{tag}_r{r}_g{i}"], rtol=1e-10, atol=1e-13)
    assert np.array_equal(OM.labels(np.arange(1000), 172, chain(4, 0x04)), g["labels_C172"])


def _golden_world(g, tag):
    from golden_world import world_from_golden
    return world_from_golden(g, tag)


@pytest.mark.parametrize("tag", ["mg2", "mg4", "mg4g", "mg1"])
@pytest.mark.parametrize("strat", ["model-centric", "micrograph", "micrograph+pg"])
def test_engine_ledger_and_params_golden(golden, tag, strat):
    g = golden("engine")
    world, iters = _golden_world(g, tag)
    P = world.fresh_params()
    led = OE.Ledger()
    for it, batches in enumerate(OE.epoch_batches(world.seed, 0, world.n, world.S, world.B, iters)):
        if strat == "model-centric":
            OE.model_centric_iteration(world, P, 0, it, batches, led)
        else:
            OE.micrograph_iteration(world, P, 0, it, batches, OE.initial_table(world.S), (),
                                    strat.endswith("pg"), led)
    key = f"{tag}_{strat}"
    got = led.by_category()
    for c, b in zip(g[key + "_cats"].tolist(), g[key + "_bytes"].tolist()):
        assert got.get(c, 0.0) == pytest.approx(b, rel=1e-12, abs=0)
    for (s, d), c, b, m in zip(g[key + "_links"].tolist(), g[key + "_linkcat"].tolist(),
                               g[key + "_linkbytes"].tolist(), g[key + "_linkmsgs"].tolist()):
        gb, gm = led.link(s, d, c)
        assert gb == pytest.approx(b, rel=1e-12) and gm == m
    for i, a in enumerate(P.arrays()):
        np.testing.assert_allclose(a, g[key + f"_p{i}"], rtol=1e-9, atol=1e-13)


def test_merge_replay_golden(golden):
    g = golden("engine")
    home = np.arange(40, dtype=np.int64) % 4
    batches = [np.arange(d * 10, (d + 1) * 10, dtype=np.int64) for d in range(4)]
    groups = [tuple(b[home[b] == s] for s in range(4)) for b in batches]
    for name in ("tt2", "tt3"):
        cells = OE.assign_cells(groups, tuple(g[name + "_removed"].tolist()), 7)
        flat = np.concatenate([np.concatenate([c, [-1]]) for row in cells for c in row])
        assert np.array_equal(flat, g[name + "_flat"])
    sv = OE.initial_table(4)
    counts = np.array([[len(c) for c in row] for row in OE.assign_cells(groups, (), 7)])
    sv2, c2 = OE.delete_column(sv, counts, 2)
    sv3, c3 = OE.delete_column(sv2, c2, 0)
    assert np.array_equal(c2, g["tt2_counts"]) and np.array_equal(c3, g["tt3_counts"])


def test_fixture_world_rows(golden):
    """The 8-vertex walkthrough: mc 3+3 rows, mg 5, pg 2 on link 1->0 (test_engine.py:169-212)."""
    g = golden("fixture_world")
    assert g["mc_rows_1_0"][0] == 3 and g["mc_rows_0_1"][0] == 3
    assert g["mg_rows_1_0"][0] + g["mg_rows_0_1"][0] == 5
    assert g["pg_rows_1_0"][0] == 2
    world = OE.World(g["offsets"], g["targets"], g["home"], 2, 0, "gcn", 4, 4, 2, (2, 2), 2)
    world.sampler_seed = 3
    P = world.fresh_params()
    batches = [np.array([6, 3]), np.array([5, 0])]
    for strat, key in (("mc", "mc"), ("mg", "mg"), ("pg", "pg")):
        led = OE.Ledger()
        if strat == "mc":
            OE.model_centric_iteration(world, P.copy(), 0, 0, batches, led)
        else:
            OE.micrograph_iteration(world, P.copy(), 0, 0, batches, OE.initial_table(2), (),
                                    strat == "pg", led)
        assert led.link(1, 0, "feature")[0] / 16 == g[key + "_rows_1_0"][0]
        assert led.link(0, 1, "feature")[0] / 16 == g[key + "_rows_0_1"][0]
