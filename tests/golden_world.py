"""Rebuild the small engine worlds of tests/golden/engine.npz for the oracle."""
import numpy as np

from oracle import engine as OE
from oracle.graphgen import GraphSpec, build_csr, build_tables
from oracle.rng import chain


def small_csr(n=3000):
    t = build_tables(GraphSpec(n=n, avg_deg=12.0, beta=0.7, p_in=0.9, n_blocks=4,
                               d_cap=600, seed=11))
    return build_csr(t)


def world_from_golden(g, tag):
    cfg = g[tag + "_cfg"].tolist()
    S, L = cfg[0], cfg[1]
    fo = tuple(cfg[2:2 + L])
    dim, hid, C, B, seed, iters = cfg[2 + L:]
    arch = str(g[tag + "_arch"][0])
    off, tgt = small_csr()
    w = OE.World(off, tgt, g[tag + "_home"], S, seed, arch, dim, hid, C, fo, B)
    return w, iters


__all__ = ["small_csr", "world_from_golden", "chain", "np"]
