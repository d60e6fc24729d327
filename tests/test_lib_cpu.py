"""CPU-side checks of the C-ABI library: it builds, loads, exports every
symbol include/hopgnn.h declares, and its host-only entry points agree with
the oracle.  No kernel launches (no GPU here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2409_00657_b200 import build
    build.build()
    from paper_2409_00657_b200 import _lib
    return _lib


def header_symbols():
    text = open(os.path.join(REPO, "include", "hopgnn.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(hg_\w+)\(", text, re.M)))


def test_all_header_symbols_exported(lib):
    h = C.CDLL(lib.LIB_PATH)
    names = header_symbols()
    assert len(names) >= 10
    missing = [n for n in names if not hasattr(h, n)]
    assert not missing, missing


def test_signature_table_covers_header(lib):
    names = set(header_symbols()) - {"hg_last_error"}
    assert names <= set(lib.SIGNATURES), sorted(names - set(lib.SIGNATURES))


def test_layout_capacities(lib):
    from paper_2409_00657_b200.sampler import plan_layout
    lay = plan_layout((15, 10))
    assert lay.n_layers == 2
    assert list(lay.cap_lay)[:3] == [150, 15, 1]
    assert list(lay.cap_need)[:3] == [166, 16, 1]
    lay4 = plan_layout((10, 10, 5, 5))
    assert list(lay4.cap_need)[:5] == [3111, 611, 111, 11, 1]
    assert lay4.smem_bytes <= 227 * 1024


def test_layout_rejects_bad_config(lib):
    from paper_2409_00657_b200.errors import ConfigError
    from paper_2409_00657_b200.sampler import plan_layout
    with pytest.raises(ConfigError):
        plan_layout((0, 3))
    with pytest.raises(ConfigError):
        plan_layout((100, 100, 100))


def test_graph_tables_match_oracle(lib):
    from oracle.graphgen import GraphSpec as OSpec, build_tables
    from paper_2409_00657_b200.graph import GraphSpec, graph_tables
    for kw in (dict(n=3000, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4, d_cap=600, seed=11),
               dict(n=2_400_000, avg_deg=26.0, beta=0.6, p_in=0.9, n_blocks=8, d_cap=1 << 14, seed=2),
               dict(n=1000, avg_deg=5.0, beta=1.0, p_in=1.0, n_blocks=1, d_cap=50, seed=3)):
        t = graph_tables(GraphSpec(**kw))
        o = build_tables(OSpec(**kw))
        E = o.n_levels
        assert t.n_levels == E
        assert list(t.cum)[:E] == o.cum.tolist()
        assert list(t.lvl_size)[:E] == o.lvl_size.tolist()
        assert list(t.deg_lo)[:E] == o.deg_lo.tolist()
        assert list(t.deg_span)[:E] == o.deg_span.tolist()
        nb = kw["n_blocks"]
        assert list(t.block_start)[:nb + 1] == o.block_start.tolist()
        assert list(t.a)[:nb] == o.a.tolist() and list(t.a_inv)[:nb] == o.a_inv.tolist()
        assert list(t.c)[:nb] == o.c.tolist()
        if o.thr_in <= 0xFFFFFFFF:
            assert t.in_always == 0 and t.thr_in == o.thr_in
        else:
            assert t.in_always == 1


def test_product_rng_matches_oracle():
    from oracle import rng as orng
    from paper_2409_00657_b200 import rng
    for w in ((1, 2), (0, 6), (7, 0, 0, 0), (2**64 - 1, 5)):
        assert rng.chain(*w) == orng.chain(*w)
    assert np.array_equal(rng.hash_vec(123, np.arange(50)), orng.keyed(123, np.arange(50)))


def test_product_does_not_import_oracle():
    pkg = os.path.join(REPO, "paper_2409_00657_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
