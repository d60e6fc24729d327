"""Device-resident CSR graphs, partitions and the synthetic generator.

Mirrors the reference ``gnnsim.graph`` objects used on the hot path:
``Graph`` (graph.py:25-74, canonical CSR: offsets int64[n+1], targets sorted
unique per row) and ``PartitionMap`` (graph.py:212-236), plus CSR1 file I/O
(graph.py:153-170) and ``partition_hash`` (graph.py:265-270).

The generator is the row-local planted-partition power-law model described
in ``oracle/graphgen.py`` (the CPU twin used only by tests); here the tables
are built on the host and the CSR on the GPU (``csrc/hg_graphgen.cu``).
"""
from __future__ import annotations

import ctypes as C
import math
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .rng import chain, hash_vec

_CSR_MAGIC = b"CSR1"
MASK32 = (1 << 32) - 1


# ---------------------------------------------------------------- spec

@dataclass(frozen=True)
class GraphSpec:
    """Synthetic graph: n vertices, mean raw row length, Zipf exponent beta,
    intra-block probability p_in over n_blocks contiguous planted blocks,
    row-length cap d_cap, seed."""

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

    def block_of(self, v):
        return (np.asarray(v, dtype=np.int64) * self.n_blocks) // self.n


def _coprime(nbk: int, h: int) -> int:
    if nbk <= 2:
        return 1
    a = h % (nbk - 1) + 1
    while math.gcd(a, nbk) != 1:
        a = a % (nbk - 1) + 1
    return a


def graph_tables(spec: GraphSpec) -> _lib.GraphTables:
    """Integer tables of the generator (shared verbatim with the CPU twin)."""
    n, nb = spec.n, spec.n_blocks
    if nb < 1 or nb > 64 or n < nb:
        raise ValueError("need 1 <= n_blocks <= 64 and n >= n_blocks")
    t = _lib.GraphTables()
    t.n, t.n_blocks, t.key = n, nb, spec.key
    t.deg_key = chain(spec.key, 0xDE)
    starts = [(b * n + nb - 1) // nb for b in range(nb + 1)]
    for b, s in enumerate(starts):
        t.block_start[b] = s
    sizes = [starts[b + 1] - starts[b] for b in range(nb)]
    for b in range(nb):
        nbk = sizes[b]
        a = _coprime(nbk, chain(spec.key, 0xAF, b))
        t.a[b] = a
        t.c[b] = chain(spec.key, 0xC0, b) % nbk
        t.a_inv[b] = pow(a, -1, nbk) if nbk > 1 else 0
    nmin = min(sizes)
    E = nmin.bit_length()
    st = np.array([(1 << e) - 1 for e in range(E)], dtype=np.int64)
    en = np.minimum(np.array([(1 << (e + 1)) - 1 for e in range(E)], dtype=np.int64), nmin)
    size = en - st
    lo_x, hi_x = st + 0.5, en + 0.5
    if abs(spec.beta - 1.0) < 1e-12:
        W = np.log(hi_x) - np.log(lo_x)
    else:
        W = (hi_x ** (1.0 - spec.beta) - lo_x ** (1.0 - spec.beta)) / (1.0 - spec.beta)
    cum = np.floor(np.cumsum(W) / W.sum() * 2.0 ** 32).astype(np.uint64)
    cum[-1] = np.uint64(1 << 32)
    per_rank = W / size
    scale = spec.avg_deg / (per_rank @ size / size.sum())
    lo = hi = None
    for _ in range(30):
        mid = per_rank * scale
        lo = np.maximum(1, np.floor(0.5 * mid)).astype(np.int64)
        hi = np.maximum(lo, np.minimum(spec.d_cap, np.floor(1.5 * mid))).astype(np.int64)
        got = float(((lo + hi) / 2.0) @ size / size.sum())
        if abs(got - spec.avg_deg) < 1e-3 * spec.avg_deg:
            break
        scale *= spec.avg_deg / max(got, 1e-9)
    t.n_levels = E
    for e in range(E):
        t.cum[e] = int(cum[e])
        t.lvl_size[e] = int(size[e])
        t.deg_lo[e] = int(lo[e])
        t.deg_span[e] = int(hi[e] - lo[e] + 1)
    if nb == 1 or spec.p_in >= 1.0:
        t.in_always, t.thr_in = 1, 0
    else:
        t.in_always = 0
        t.thr_in = 0 if spec.p_in <= 0 else min(int(spec.p_in * 2.0 ** 32), MASK32)
    return t


# ---------------------------------------------------------------- graph

class Graph:
    """Immutable canonical CSR held in HBM (targets int32, offsets int64)."""

    def __init__(self, n_vertices: int, offsets: torch.Tensor, targets: torch.Tensor,
                 directed: bool = True):
        if offsets.dtype != torch.int64 or targets.dtype != torch.int32:
            raise ValueError("offsets must be int64 and targets int32")
        if offsets.numel() != n_vertices + 1:
            raise ValueError("inconsistent CSR offsets")
        self.n_vertices = int(n_vertices)
        self.offsets = offsets.contiguous()
        self.targets = targets.contiguous()
        self.directed = directed

    @property
    def n_targets(self) -> int:
        return int(self.targets.numel())

    @property
    def device(self):
        return self.offsets.device

    def degrees(self) -> torch.Tensor:
        return self.offsets[1:] - self.offsets[:-1]

    def to_host(self):
        return self.offsets.cpu().numpy(), self.targets.cpu().numpy().astype(np.int64)

    @classmethod
    def from_host(cls, offsets, targets, device="cuda") -> "Graph":
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        targets = np.ascontiguousarray(targets)
        n = len(offsets) - 1
        if offsets[0] != 0 or offsets[-1] != len(targets):
            raise ValueError("inconsistent CSR offsets")
        if len(targets) and (targets.min() < 0 or targets.max() >= n):
            raise ValueError("target id out of range")
        if n >= 2 ** 31:
            raise ValueError("vertex ids must fit int32 on the device")
        return cls(n, torch.from_numpy(offsets).to(device),
                   torch.from_numpy(targets.astype(np.int32)).to(device))


def generate(spec: GraphSpec, device="cuda", chunk_slots: int = 1 << 30) -> Graph:
    """Build the CSR of `spec` on the GPU (4 passes, see csrc/hg_graphgen.cu)."""
    dev = torch.device(device)
    t = graph_tables(spec)
    n = spec.n
    stream = torch.cuda.current_stream(dev).cuda_stream
    raw_deg = torch.empty(n, dtype=torch.int64, device=dev)
    _lib.call("hg_graph_raw_degrees", C.byref(t), raw_deg.data_ptr(), stream)
    raw_off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(raw_deg, 0, out=raw_off[1:])
    del raw_deg
    total = int(raw_off[-1].item())
    raw = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    _lib.call("hg_graph_fill", C.byref(t), 0, n, raw_off.data_ptr(), raw.data_ptr(), stream)
    row_len = torch.empty(n, dtype=torch.int64, device=dev)
    # chunk boundaries keep every segmented sort below 2^31 slots
    marks = torch.tensor(list(range(chunk_slots, total, chunk_slots)), dtype=torch.int64,
                         device=dev)
    cuts = (torch.searchsorted(raw_off, marks, right=True).sub_(1).clamp_(0, n).cpu().tolist()
            if marks.numel() else [])
    bounds = sorted(set([0] + cuts + [n]))
    ws = None
    for v0, v1 in zip(bounds[:-1], bounds[1:]):
        if v1 <= v0:
            continue
        base = int(raw_off[v0].item())
        need = C.c_size_t(0)
        _lib.call("hg_graph_canonicalize", v0, v1, raw_off.data_ptr(), raw.data_ptr() + 4 * base,
                  row_len.data_ptr() + 8 * v0, None, C.byref(need), stream)
        if ws is None or ws.numel() < need.value:
            ws = torch.empty(need.value, dtype=torch.uint8, device=dev)
        _lib.call("hg_graph_canonicalize", v0, v1, raw_off.data_ptr(), raw.data_ptr() + 4 * base,
                  row_len.data_ptr() + 8 * v0, ws.data_ptr(), C.byref(C.c_size_t(ws.numel())),
                  stream)
    del ws
    offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(row_len, 0, out=offsets[1:])
    del row_len
    m = int(offsets[-1].item())
    targets = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    _lib.call("hg_graph_compact", 0, n, raw_off.data_ptr(), raw.data_ptr(), offsets.data_ptr(),
              targets.data_ptr(), stream)
    del raw, raw_off
    return Graph(n, offsets, targets[:m] if m else targets[:0])


# ---------------------------------------------------------------- partitions

class PartitionMap:
    """vertex id -> home server in [0, n_servers) (graph.py:212-236)."""

    def __init__(self, home, n_servers: int, device="cuda"):
        home = np.ascontiguousarray(home, dtype=np.int64)
        if n_servers < 1:
            raise ValueError("n_servers must be >= 1")
        if len(home) and (home.min() < 0 or home.max() >= n_servers):
            raise ValueError("home id out of range")
        self.home = home
        self.n_servers = int(n_servers)
        self._dev = {}
        self._device = device

    @property
    def n_vertices(self) -> int:
        return len(self.home)

    def home_device(self, device=None) -> torch.Tensor:
        dev = torch.device(device or self._device)
        key = str(dev)
        if key not in self._dev:
            self._dev[key] = torch.from_numpy(self.home.astype(np.int32)).to(dev)
        return self._dev[key]

    def part_sizes(self) -> np.ndarray:
        return np.bincount(self.home, minlength=self.n_servers)


def partition_hash(n_vertices: int, n_servers: int, seed: int) -> PartitionMap:
    """home(v) = chain(seed, 0xA7, v) mod S (graph.py:265-270)."""
    h = hash_vec(chain(seed, 0xA7), np.arange(n_vertices, dtype=np.int64))
    return PartitionMap((h % np.uint64(n_servers)).astype(np.int64), n_servers)


def partition_planted(spec: GraphSpec, n_servers: int) -> PartitionMap:
    """home(v) = floor(block(v) * S / n_blocks): planted blocks map to GPUs."""
    blocks = spec.block_of(np.arange(spec.n, dtype=np.int64))
    return PartitionMap((blocks * n_servers) // spec.n_blocks, n_servers)


def save_csr(g: Graph, path) -> None:
    """CSR1: magic, u64 n, u64 m, u64 offsets, u64 targets (graph.py:153-159)."""
    off, tgt = g.to_host()
    with open(path, "wb") as f:
        f.write(_CSR_MAGIC)
        f.write(struct.pack("<QQ", g.n_vertices, len(tgt)))
        f.write(off.astype("<u8").tobytes())
        f.write(tgt.astype("<u8").tobytes())


def load_csr(path, device="cuda") -> Graph:
    with open(path, "rb") as f:
        if f.read(4) != _CSR_MAGIC:
            raise ValueError("bad magic, expected b'CSR1'")
        n, m = struct.unpack("<QQ", f.read(16))
        off = np.frombuffer(f.read(8 * (n + 1)), dtype="<u8").astype(np.int64)
        tgt = np.frombuffer(f.read(8 * m), dtype="<u8").astype(np.int64)
    return Graph.from_host(off, tgt, device)
