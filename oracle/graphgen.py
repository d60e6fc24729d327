"""Numpy twin of the device graph generator (``csrc/hg_graphgen.cu``).

The reference only ships a dense O(n^2) SBM generator (graph.py:173-209), which
cannot produce the 111M-vertex / 1.6B-entry papers100M-shaped inputs the
benchmark configs name.  Both sides therefore use this *row-local* planted
partition power-law generator: row v (its in-neighbour list, i.e. the CSR
range the sampler draws from) is a pure integer function of (spec, v).  That
lets the GPU build the whole CSR in one pass and lets the CPU oracle
materialise only the rows a bounded sample touches.

Spec (``GraphSpec``), all decisions integer after the host-side level table:

* blocks: ``block(v) = floor(nb * v / n)`` (contiguous planted blocks);
* popularity: inside block b of size nbk, local index i has rank
  ``r = (a_b * i + c_b) mod nbk`` (an affine bijection keyed on the seed);
* ranks are grouped in levels ``e = floor(log2(r+1))``; a level is drawn
  with probability proportional to sum of (r+1)^-beta over its ranks
  (``cum`` table, 2^32 scale), the rank inside the level uniformly;
* row length of v: uniform integer in ``[lo_e, hi_e]`` of v's level, so
  popular vertices also have long rows (power-law degree ~ popularity);
* slot t of row v: hA = chain(gkey, v, 2t), hB = chain(gkey, v, 2t+1);
  target block = own block iff ``hi32(hB) < thr_in`` else one of the other
  blocks (``lo32(hB) mod (nb-1)``), target rank from hA, target vertex via
  the inverse affine map; the row is then sorted, de-duplicated and
  self-loops dropped (canonical CSR form, graph.py:25-48).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .rng import U64, chain, mix64, mix64_array

MASK32 = (1 << 32) - 1


@dataclass(frozen=True)
class GraphSpec:
    n: int
    avg_deg: float
    beta: float = 0.6
    p_in: float = 0.9
    n_blocks: int = 8
    d_cap: int = 1 << 15
    seed: int = 0

    @property
    def key(self) -> int:
        return chain(self.seed, 0x01, 0xC5)


@dataclass
class GraphTables:
    """Host-side integer tables shared verbatim by the CPU twin and the GPU."""

    spec: GraphSpec
    block_start: np.ndarray   # int64 [nb+1]
    a: np.ndarray             # uint64 [nb]
    c: np.ndarray             # uint64 [nb]
    a_inv: np.ndarray         # uint64 [nb]
    n_levels: int
    cum: np.ndarray           # uint64 [n_levels]  (2^32 scale, last == 2^32)
    lvl_size: np.ndarray      # int64 [n_levels]   ranks per level (min block)
    deg_lo: np.ndarray        # int64 [n_levels]
    deg_span: np.ndarray      # int64 [n_levels]   hi - lo + 1
    thr_in: int               # uint32 threshold on hi32(hB)


def _coprime_multiplier(nbk: int, h: int) -> int:
    if nbk <= 2:
        return 1
    a = (h % (nbk - 1)) + 1
    while math.gcd(a, nbk) != 1:
        a = a % (nbk - 1) + 1
    return a


def build_tables(spec: GraphSpec) -> GraphTables:
    n, nb = spec.n, max(1, spec.n_blocks)
    if n < nb:
        raise ValueError("need at least one vertex per block")
    bs = np.array([(b * n + nb - 1) // nb for b in range(nb + 1)], dtype=np.int64)
    sizes = np.diff(bs)
    a = np.zeros(nb, dtype=np.uint64)
    c = np.zeros(nb, dtype=np.uint64)
    ai = np.zeros(nb, dtype=np.uint64)
    for b in range(nb):
        nbk = int(sizes[b])
        av = _coprime_multiplier(nbk, chain(spec.key, 0xAF, b))
        a[b] = av
        c[b] = chain(spec.key, 0xC0, b) % nbk
        ai[b] = pow(av, -1, nbk) if nbk > 1 else 0
    nmin = int(sizes.min())
    E = nmin.bit_length()  # levels 0..E-1 cover ranks [0, nmin)
    starts = np.array([(1 << e) - 1 for e in range(E)], dtype=np.int64)
    ends = np.minimum(np.array([(1 << (e + 1)) - 1 for e in range(E)], dtype=np.int64), nmin)
    lvl_size = ends - starts
    keep = lvl_size > 0
    starts, ends, lvl_size = starts[keep], ends[keep], lvl_size[keep]
    E = len(lvl_size)
    beta = spec.beta
    lo_x = starts.astype(np.float64) + 0.5
    hi_x = ends.astype(np.float64) + 0.5
    if abs(beta - 1.0) < 1e-12:
        W = np.log(hi_x) - np.log(lo_x)
    else:
        W = (hi_x ** (1.0 - beta) - lo_x ** (1.0 - beta)) / (1.0 - beta)
    cum = np.floor(np.cumsum(W) / W.sum() * 2.0 ** 32).astype(np.uint64)
    cum[-1] = np.uint64(1 << 32)
    # row length per level, calibrated so the mean raw length ~= avg_deg
    per_rank = W / lvl_size
    scale = spec.avg_deg / (per_rank @ lvl_size / lvl_size.sum())
    lo = hi = None
    for _ in range(30):
        mid = per_rank * scale
        lo = np.maximum(1, np.floor(0.5 * mid)).astype(np.int64)
        hi = np.maximum(lo, np.minimum(spec.d_cap, np.floor(1.5 * mid))).astype(np.int64)
        got = float(((lo + hi) / 2.0) @ lvl_size / lvl_size.sum())
        if abs(got - spec.avg_deg) < 1e-3 * spec.avg_deg:
            break
        scale *= spec.avg_deg / max(got, 1e-9)
    thr = 0 if spec.p_in <= 0 else (MASK32 + 1 if spec.p_in >= 1 else int(spec.p_in * 2.0 ** 32))
    if nb == 1:
        thr = MASK32 + 1
    return GraphTables(spec, bs, a, c, ai, E, cum, lvl_size, lo, hi - lo + 1, thr)


def _level(r: np.ndarray) -> np.ndarray:
    """floor(log2(r + 1)) for int64 r >= 0."""
    x = (r + 1).astype(np.uint64)
    e = np.zeros(x.shape, dtype=np.int64)
    for sh in (32, 16, 8, 4, 2, 1):
        big = x >= (U64(1) << U64(sh))
        e += big * sh
        x = np.where(big, x >> U64(sh), x)
    return e


def block_of(t: GraphTables, v: np.ndarray) -> np.ndarray:
    nb = t.spec.n_blocks
    return (np.asarray(v, dtype=np.int64) * nb) // t.spec.n


def rank_of(t: GraphTables, v: np.ndarray) -> np.ndarray:
    v = np.asarray(v, dtype=np.int64)
    b = block_of(t, v)
    nbk = (t.block_start[b + 1] - t.block_start[b]).astype(np.uint64)
    i = (v - t.block_start[b]).astype(np.uint64)
    return ((t.a[b] * i + t.c[b]) % nbk).astype(np.int64)


def raw_degree(t: GraphTables, v: np.ndarray) -> np.ndarray:
    """Pre-dedup row length of v (number of slots drawn)."""
    v = np.asarray(v, dtype=np.int64)
    e = np.minimum(_level(rank_of(t, v)), t.n_levels - 1)
    u = mix64_array(v.astype(np.uint64) ^ U64(chain(t.spec.key, 0xDE))) >> U64(32)
    span = t.deg_span[e].astype(np.uint64)
    return t.deg_lo[e] + ((u * span) >> U64(32)).astype(np.int64)


def raw_row(t: GraphTables, v: int) -> np.ndarray:
    """Slot draws of row v before sort/dedup (int64)."""
    v = int(v)
    d = int(raw_degree(t, np.array([v]))[0])
    rk = U64(mix64(t.spec.key ^ v))
    slots = np.arange(d, dtype=np.uint64)
    hA = mix64_array((U64(2) * slots) ^ rk)
    hB = mix64_array((U64(2) * slots + U64(1)) ^ rk)
    nb = t.spec.n_blocks
    own = int(block_of(t, np.array([v]))[0])
    inb = (hB >> U64(32)) < U64(t.thr_in) if t.thr_in <= MASK32 else np.ones(d, bool)
    if nb > 1:
        other = (own + 1 + ((hB & U64(MASK32)) % U64(nb - 1)).astype(np.int64)) % nb
        tb = np.where(inb, own, other)
    else:
        tb = np.full(d, own, dtype=np.int64)
    u = hA >> U64(32)
    e = np.searchsorted(t.cum, u, side="right")  # first level with u < cum[e]
    off = (((hA & U64(MASK32)) * t.lvl_size[e].astype(np.uint64)) >> U64(32)).astype(np.int64)
    r = ((U64(1) << e.astype(np.uint64)) - U64(1)).astype(np.int64) + off
    nbk = (t.block_start[tb + 1] - t.block_start[tb]).astype(np.uint64)
    rr = r.astype(np.uint64)
    # (r - c) mod nbk without underflow, then * a_inv mod nbk
    diff = (rr + nbk - (t.c[tb] % nbk)) % nbk
    i = (diff * t.a_inv[tb]) % nbk
    return t.block_start[tb] + i.astype(np.int64)


def row(t: GraphTables, v: int) -> np.ndarray:
    """Canonical CSR row of v: sorted, unique, no self-loop."""
    r = np.unique(raw_row(t, v))
    return r[r != v]


def build_csr(t: GraphTables):
    """Full CSR (small graphs only: tests and the cfg-1 CPU trainer)."""
    n = t.spec.n
    rows = [row(t, v) for v in range(n)]
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum([len(r) for r in rows], out=offsets[1:])
    targets = np.concatenate(rows) if n else np.empty(0, np.int64)
    return offsets, targets.astype(np.int64)


def rows_csr(t: GraphTables, vs) -> tuple:
    """Canonical rows of many vertices at once (vectorised ``row``): returns a
    sub-CSR (offsets int64[len(vs)+1], targets int64) whose row i is row(t, vs[i])."""
    vs = np.asarray(vs, dtype=np.int64)
    if len(vs) == 0:
        return np.zeros(1, np.int64), np.empty(0, np.int64)
    d = raw_degree(t, vs)
    owner = np.repeat(np.arange(len(vs), dtype=np.int64), d)
    start = np.zeros(len(vs) + 1, dtype=np.int64)
    np.cumsum(d, out=start[1:])
    slots = (np.arange(int(start[-1]), dtype=np.int64) - start[owner]).astype(np.uint64)
    v = vs[owner]
    rk = mix64_array(v.astype(np.uint64) ^ U64(t.spec.key))
    hA = mix64_array((U64(2) * slots) ^ rk)
    hB = mix64_array((U64(2) * slots + U64(1)) ^ rk)
    nb = t.spec.n_blocks
    own = block_of(t, v)
    inb = (hB >> U64(32)) < U64(t.thr_in) if t.thr_in <= MASK32 else np.ones(len(v), bool)
    if nb > 1:
        other = (own + 1 + ((hB & U64(MASK32)) % U64(nb - 1)).astype(np.int64)) % nb
        tb = np.where(inb, own, other)
    else:
        tb = own
    u = hA >> U64(32)
    e = np.searchsorted(t.cum, u, side="right")
    off = (((hA & U64(MASK32)) * t.lvl_size[e].astype(np.uint64)) >> U64(32)).astype(np.int64)
    r = ((U64(1) << e.astype(np.uint64)) - U64(1)).astype(np.int64) + off
    nbk = (t.block_start[tb + 1] - t.block_start[tb]).astype(np.uint64)
    diff = (r.astype(np.uint64) + nbk - (t.c[tb] % nbk)) % nbk
    tgt = t.block_start[tb] + ((diff * t.a_inv[tb]) % nbk).astype(np.int64)
    # per row: sort, unique, drop the self-loop (one lexsort over (owner, target))
    order = np.lexsort((tgt, owner))
    o, x = owner[order], tgt[order]
    keep = np.ones(len(x), dtype=bool)
    keep[1:] = (o[1:] != o[:-1]) | (x[1:] != x[:-1])
    keep &= x != vs[o]
    o, x = o[keep], x[keep]
    offsets = np.zeros(len(vs) + 1, dtype=np.int64)
    np.cumsum(np.bincount(o, minlength=len(vs)), out=offsets[1:])
    return offsets, x


class LazyRows:
    """CSR facade materialising rows on demand (CPU baseline on huge specs)."""

    def __init__(self, t: GraphTables):
        self.t = t
        self.cache: dict[int, np.ndarray] = {}

    def __call__(self, v: int) -> np.ndarray:
        r = self.cache.get(v)
        if r is None:
            r = row(self.t, v)
            self.cache[v] = r
        return r

    def prefetch(self, vs) -> None:
        """Materialise many rows in one vectorised pass (rows_csr)."""
        vs = np.unique(np.asarray(vs, dtype=np.int64))
        vs = np.array([v for v in vs.tolist() if v not in self.cache], dtype=np.int64)
        if not len(vs):
            return
        # chunks of <= ~4M raw slots (bounded temporaries on high-degree graphs)
        cum = np.cumsum(raw_degree(self.t, vs))
        cuts = np.searchsorted(cum, np.arange(1, int(cum[-1]) // (1 << 22) + 1) * (1 << 22))
        for part in np.split(vs, np.unique(cuts[(cuts > 0) & (cuts < len(vs))])):
            off, tgt = rows_csr(self.t, part)
            for i, v in enumerate(part.tolist()):
                self.cache[v] = tgt[off[i]:off[i + 1]]
