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
from .errors import EdgeListError
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


class ShardedGraph:
    """CSR topology partitioned by home server (north_star): this GPU holds
    only the rows of the vertices homed on it; every peer's shard is mapped
    over NVLink (CUDA IPC), and the micrograph builds read a remote row in
    place from its owner (hg_mg_build_group_sharded).  Contiguous partitions
    (planted blocks) address rows by vertex ranges; arbitrary ones through
    per-vertex home / local-row arrays.  Collective construction: every rank
    of the group calls it together."""

    def __init__(self, n_vertices: int, part: "PartitionMap", rank: int,
                 local_offsets: torch.Tensor, local_targets: torch.Tensor, group=None):
        import torch.distributed as dist
        self.n_vertices = int(n_vertices)
        self.part, self.rank, self.S = part, int(rank), part.n_servers
        if self.S > _lib.MAX_SHARDS:
            raise ValueError(f"at most {_lib.MAX_SHARDS} shards")
        dev = local_offsets.device
        self.device = dev
        # the local shard in raw (IPC-exportable) allocations
        self._mine, self._opened = [], []
        ptrs = []
        for t in (local_offsets.contiguous(), local_targets.contiguous()):
            p = C.c_void_p()
            nbytes = max(t.numel() * t.element_size(), 16)
            _lib.call("hg_alloc", nbytes, C.byref(p))
            _lib.call("hg_memcpy_d2d", p.value, t.data_ptr(), t.numel() * t.element_size(),
                      torch.cuda.current_stream(dev).cuda_stream)
            self._mine.append(p.value)
            ptrs.append(p.value)
        torch.cuda.synchronize(dev)
        self.n_targets_local = int(local_targets.numel())
        handles = []
        for p in ptrs:
            h = (C.c_char * 64)()
            _lib.call("hg_ipc_handle", p, h)
            handles.append(bytes(h))
        every = [None] * self.S
        if dist.is_initialized() and self.S > 1:
            dist.all_gather_object(every, handles, group=group)
        else:
            every = [handles]
        sh = _lib.CsrShards()
        sh.n_shards = self.S
        for h, hs in enumerate(every):
            for j, hb in enumerate(hs):
                if h == self.rank:
                    ptr = ptrs[j]
                else:
                    q = C.c_void_p()
                    _lib.call("hg_ipc_open", (C.c_char * 64).from_buffer_copy(hb), C.byref(q))
                    self._opened.append(q.value)
                    ptr = q.value
                (sh.offsets if j == 0 else sh.targets)[h] = ptr
        self._address(sh)

    @staticmethod
    def _rows_of(g: "Graph", part: "PartitionMap", h: int):
        dev = g.device
        mine = torch.from_numpy(np.flatnonzero(part.home == h)).to(dev)
        lo, hi = g.offsets[mine], g.offsets[mine + 1]
        ln = hi - lo
        off = torch.zeros(mine.numel() + 1, dtype=torch.int64, device=dev)
        torch.cumsum(ln, 0, out=off[1:])
        m = int(off[-1].item())
        idx = (torch.repeat_interleave(lo - off[:-1], ln) +
               torch.arange(m, device=dev)) if m else torch.zeros(0, dtype=torch.int64, device=dev)
        tgt = g.targets[idx] if m else torch.zeros(1, dtype=torch.int32, device=dev)
        return off, tgt

    @classmethod
    def split_local(cls, g: "Graph", part: "PartitionMap") -> "ShardedGraph":
        """All S shards of g on ONE device (no IPC): the sharded addressing of
        the builds on a single GPU (tests)."""
        obj = cls.__new__(cls)
        obj.n_vertices, obj.part, obj.rank, obj.S = g.n_vertices, part, 0, part.n_servers
        obj.device, obj._mine, obj._opened = g.device, [], []
        obj._keep = [cls._rows_of(g, part, h) for h in range(obj.S)]
        sh = _lib.CsrShards()
        sh.n_shards = obj.S
        for h, (off, tgt) in enumerate(obj._keep):
            sh.offsets[h], sh.targets[h] = off.data_ptr(), tgt.data_ptr()
        obj._address(sh)
        return obj

    def _address(self, sh) -> None:
        home = self.part.home
        contiguous = bool(np.all(np.diff(home) >= 0)) if len(home) else True
        if contiguous:
            starts = np.searchsorted(home, np.arange(self.S)) if len(home) else np.zeros(self.S)
            for h in range(self.S):
                sh.vstart[h] = int(starts[h])
            sh.vstart[self.S] = self.n_vertices
            self.home_of = self.row_of = None
        else:
            row_of = np.empty(len(home), dtype=np.int32)
            for h in range(self.S):
                idx = np.flatnonzero(home == h)
                row_of[idx] = np.arange(len(idx), dtype=np.int32)
            self.home_of = self.part.home_device(self.device)
            self.row_of = torch.from_numpy(row_of).to(self.device)
            sh.home_of = self.home_of.data_ptr()
            sh.row_of = self.row_of.data_ptr()
        self.contiguous = contiguous
        self.shards = sh

    @classmethod
    def from_graph(cls, g: "Graph", part: "PartitionMap", rank: int, group=None):
        """This rank's rows of a full CSR (the full graph may be freed afterwards)."""
        off, tgt = cls._rows_of(g, part, rank)
        return cls(g.n_vertices, part, rank, off, tgt, group)

    def close(self) -> None:
        """Unmap the peers' shards and free this rank's (after a barrier: peers
        may still read it)."""
        for p in self._opened:
            _lib.call("hg_ipc_close", p)
        self._opened = []
        for p in self._mine:
            _lib.call("hg_free", p)
        self._mine = []


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


def partition_hash(g, n_servers: int, seed: int) -> PartitionMap:
    """home(v) = chain(seed, 0xA7, v) mod S (graph.py:265-270).  g: a Graph (the
    reference signature) or a vertex count."""
    if n_servers < 1:
        raise ValueError("n_servers must be >= 1")
    n = g.n_vertices if hasattr(g, "n_vertices") else int(g)
    h = hash_vec(chain(seed, 0xA7), np.arange(n, dtype=np.int64))
    return PartitionMap((h % np.uint64(n_servers)).astype(np.int64), n_servers)


def partition_greedy_locality(g: "Graph", n_servers: int, slack: float = 0.0,
                              seed: int = 0) -> PartitionMap:
    """BFS region growing into size-capped parts (graph.py:273-327) on the GPU
    (csrc/hg_partition.cu): seeds by degree descending / id ascending, cap
    ceil((1 + slack) n / S); identical homes to the reference.  The seed
    argument is unused, as in the reference."""
    if n_servers < 1:
        raise ValueError("n_servers must be >= 1")
    if slack < 0:
        raise ValueError("slack must be >= 0")
    n = g.n_vertices
    cap = max(1, int(np.ceil((1.0 + slack) * n / n_servers)))
    dev = g.device
    home = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    if n:
        # degree-descending, id-ascending seed order (graph.py:300): stable sort of -deg
        order = torch.argsort(-g.degrees(), stable=True)
        queue = torch.empty(n, dtype=torch.int32, device=dev)
        s = torch.cuda.current_stream(dev).cuda_stream
        _lib.call("hg_partition_greedy", g.offsets.data_ptr(), g.targets.data_ptr(), n,
                  n_servers, cap, order.data_ptr(), home.data_ptr(), queue.data_ptr(), s)
        left = home[:n] == -1
        if bool(left.any()):
            rank = torch.cumsum(left.to(torch.int64), 0) - 1
            _lib.call("hg_partition_leftovers", home.data_ptr(), n, n_servers, rank.data_ptr(), s)
    return PartitionMap(home[:n].cpu().numpy().astype(np.int64), n_servers, dev)


def save_partition(p: PartitionMap, path) -> None:
    """ASCII lines "vertex_id server_id" (graph.py:239-244)."""
    with open(path, "w", encoding="ascii") as f:
        f.write("".join(f"{v} {s}\n" for v, s in enumerate(p.home.tolist())))


def load_partition(path, n_servers: int = None) -> PartitionMap:
    """Inverse of save_partition (graph.py:247-262): '#' comments and blank lines
    skipped, every vertex 0..n-1 exactly once."""
    pairs = {}
    with open(path, "r", encoding="ascii") as f:
        for lineno, raw in enumerate(f, start=1):
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            if len(parts) != 2:
                raise EdgeListError(f"line {lineno}: expected 'vertex server'")
            pairs[int(parts[0])] = int(parts[1])
    n = max(pairs) + 1 if pairs else 0
    if len(pairs) != n:
        raise ValueError("partition file must cover vertices 0..n-1 exactly")
    home = np.array([pairs[v] for v in range(n)], dtype=np.int64)
    servers = n_servers if n_servers is not None else (int(home.max()) + 1 if n else 1)
    return PartitionMap(home, servers)


def from_pairs(n_vertices: int, us, vs, symmetrize: bool = True, drop_self_loops: bool = True,
               device="cuda") -> "Graph":
    """Canonical CSR from edge endpoints (graph.py:77-99), built on the device:
    duplicates collapse, self-loops dropped unless kept, both directions when
    symmetrize."""
    dev = torch.device(device)
    u = torch.as_tensor(np.asarray(us, dtype=np.int64), device=dev)
    v = torch.as_tensor(np.asarray(vs, dtype=np.int64), device=dev)
    if drop_self_loops:
        keep = u != v
        u, v = u[keep], v[keep]
    if symmetrize:
        u, v = torch.cat([u, v]), torch.cat([v, u])
    n = int(n_vertices)
    if u.numel():
        code = torch.unique(u * n + v)  # sorted: row-major, targets ascending per row
        u, v = code // n, code % n
    counts = torch.bincount(u, minlength=n) if n else torch.zeros(0, dtype=torch.int64,
                                                                  device=dev)
    offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=offsets[1:])
    if n >= 2 ** 31:
        raise ValueError("vertex ids must fit int32 on the device")
    return Graph(n, offsets, v.to(torch.int32), directed=not symmetrize)


def load_edge_list(source, n_vertices: int = None, device="cuda") -> "Graph":
    """"u v" lines -> undirected canonical CSR (graph.py:110-143), same errors."""
    if not hasattr(source, "read"):
        with open(source, "r", encoding="ascii") as f:
            return load_edge_list(f, n_vertices, device)
    us, vs, max_id = [], [], -1
    for lineno, raw in enumerate(source, start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        if len(parts) != 2:
            raise EdgeListError(f"line {lineno}: expected 'u v', got {line!r}")
        try:
            u, v = int(parts[0]), int(parts[1])
        except ValueError:
            raise EdgeListError(f"line {lineno}: non-integer vertex id in {line!r}") from None
        if u < 0 or v < 0:
            raise EdgeListError(f"line {lineno}: negative vertex id in {line!r}")
        if n_vertices is not None and (u >= n_vertices or v >= n_vertices):
            raise EdgeListError(f"line {lineno}: vertex id >= declared {n_vertices}")
        max_id = max(max_id, u, v)
        us.append(u)
        vs.append(v)
    n = n_vertices if n_vertices is not None else max_id + 1
    return from_pairs(max(n, 0), np.array(us, dtype=np.int64), np.array(vs, dtype=np.int64),
                      device=device)


@dataclass(frozen=True)
class SbmSpec:
    """Stochastic block model (graph.py:173-191): blocks of consecutive ids."""

    block_sizes: tuple
    p_in: float
    p_out: float
    seed: int

    def __post_init__(self):
        object.__setattr__(self, "block_sizes", tuple(int(b) for b in self.block_sizes))
        if any(b < 1 for b in self.block_sizes):
            raise ValueError("block sizes must be >= 1")
        if not (0.0 <= self.p_out <= self.p_in <= 1.0):
            raise ValueError("need 0 <= p_out <= p_in <= 1")

    @property
    def n_vertices(self) -> int:
        return sum(self.block_sizes)


def generate_sbm(spec: SbmSpec, device="cuda") -> "Graph":
    """Every unordered pair sampled once (graph.py:194-209): the pair pass is the
    CUDA sbm_edges (kernels.sbm_edges), the CSR is built by from_pairs."""
    from .kernels import probability_threshold, sbm_edges
    if not spec.block_sizes:
        raise ValueError("empty SBM spec: no blocks")
    block_of = np.repeat(np.arange(len(spec.block_sizes), dtype=np.int64),
                         np.array(spec.block_sizes, dtype=np.int64))
    mi, ti = probability_threshold(spec.p_in)
    mo, to = probability_threshold(spec.p_out)
    us, vs = sbm_edges(torch.as_tensor(block_of, device=device), mi, ti, mo, to,
                       chain(spec.seed, 0x5B))
    return from_pairs(spec.n_vertices, us, vs, device=device)


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
