"""Feature tables in HBM, byte-exact communication ledger, pre-gather plans.

Mirrors reference ``gnnsim.featstore``: ``CommLedger`` (featstore.py:32-87),
``FetchStats`` (featstore.py:90-107), feature generation (featstore.py:161-184,
row v = feature_rows(v)) and ``plan_pregather`` (featstore.py:226-239).
The ledger keeps the reference's 4-byte-per-element accounting so bytes are
directly comparable; ``actual`` counters record the bytes this implementation
really moved (bf16 rows, real hop payloads).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InvariantViolation
from .rng import chain

BYTES_PER_ELEM = 4
FEATURE = "feature"
MODEL = "model"
GRADIENT = "gradient"
INTERMEDIATE = "intermediate"
TOPOLOGY = "topology"
CATEGORIES = (FEATURE, MODEL, GRADIENT, INTERMEDIATE, TOPOLOGY)

SEED_FEATURES = 0x03


def feature_state(seed: int) -> int:
    """State of generated features: chain(chain(seed, 0x03), 0xFE) (featstore.py:167-168)."""
    return chain(chain(seed, SEED_FEATURES), 0xFE)


class CommLedger:
    """Per-directed-link byte/message counters, categorised (featstore.py:32-87)."""

    def __init__(self):
        self.counters: dict = {}
        self.events: list = []

    def add(self, src: int, dst: int, category: str, nbytes: float, messages: int = 1) -> None:
        if src == dst:
            raise InvariantViolation(f"self-link {src}->{dst} in ledger")
        if category not in CATEGORIES:
            raise ValueError(f"unknown category {category!r}")
        if nbytes < 0 or messages < 0:
            raise ValueError("ledger counters only grow")
        cell = self.counters.setdefault((int(src), int(dst), category), [0.0, 0])
        cell[0] += nbytes
        cell[1] += messages
        self.events.append((int(src), int(dst), category, nbytes, messages))

    def merge(self, other: "CommLedger") -> None:
        for k, (b, m) in other.counters.items():
            cell = self.counters.setdefault(k, [0.0, 0])
            cell[0] += b
            cell[1] += m
        self.events.extend(other.events)

    def bytes_by_category(self) -> dict:
        out = {c: 0.0 for c in CATEGORIES}
        for (_, _, cat), (b, _) in self.counters.items():
            out[cat] += b
        return out

    def messages_by_category(self) -> dict:
        out = {c: 0 for c in CATEGORIES}
        for (_, _, cat), (_, m) in self.counters.items():
            out[cat] += m
        return out

    def total_bytes(self) -> float:
        return sum(b for b, _ in self.counters.values())

    def link(self, src: int, dst: int, category: str):
        b, m = self.counters.get((src, dst, category), (0.0, 0))
        return b, m


@dataclass
class FetchStats:
    requested: int = 0
    local: int = 0
    staged: int = 0
    transferred: int = 0

    @property
    def miss_rate(self) -> float:
        return self.transferred / self.requested if self.requested else 0.0

    def merge(self, other: "FetchStats") -> None:
        self.requested += other.requested
        self.local += other.local
        self.staged += other.staged
        self.transferred += other.transferred


_FEAT_MAGIC = b"FEAT"


def write_feature_file(matrix, path) -> None:
    """magic "FEAT", little-endian u64 n and dim, n*dim f32 row-major
    (featstore.py:187-193)."""
    matrix = np.ascontiguousarray(matrix, dtype="<f4")
    with open(path, "wb") as f:
        f.write(_FEAT_MAGIC)
        f.write(struct.pack("<QQ", matrix.shape[0], matrix.shape[1]))
        f.write(matrix.tobytes())


def read_feature_file(path) -> np.ndarray:
    """Inverse of write_feature_file (featstore.py:196-205), same errors."""
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != _FEAT_MAGIC:
            raise ValueError(f"bad magic {magic!r}, expected {_FEAT_MAGIC!r}")
        n, dim = struct.unpack("<QQ", f.read(16))
        data = np.frombuffer(f.read(4 * n * dim), dtype="<f4")
        if len(data) != n * dim:
            raise ValueError("feature file truncated")
    return data.reshape(n, dim).astype(np.float32)


class FeatureTable:
    """Rows of the feature matrix resident in HBM.

    ``table[row]`` holds feature_rows(vertex) padded to ``ld`` columns;
    ``row_of`` (int32[n_vertices] or None = identity) maps vertex -> row, so
    a GPU can hold its own shard plus staged remote rows in one table.
    """

    def __init__(self, n_rows: int, dim: int, dtype=torch.bfloat16, device="cuda", ld=None):
        self.dim = int(dim)
        self.ld = int(ld or (dim + 7) // 8 * 8)
        self.dtype = dtype
        self.device = torch.device(device)
        self.table = torch.zeros((max(n_rows, 1), self.ld), dtype=dtype, device=self.device)
        self.row_of = None

    @property
    def act_dtype(self) -> int:
        return 1 if self.dtype == torch.bfloat16 else 0

    def fill_generated(self, first_vertex: int, count: int, state: int, row0: int = 0,
                       ids: torch.Tensor = None) -> None:
        """Rows row0.. = feature_rows(first_vertex..first_vertex+count), or of the
        int64 device `ids` (bit-exact f32; bf16 tables hold the RNE cast)."""
        code = 1 if self.dtype == torch.bfloat16 else 0
        ptr = self.table.data_ptr() + row0 * self.ld * self.table.element_size()
        _lib.call("hg_feature_table", ids.data_ptr() if ids is not None else None,
                  int(first_vertex), int(count), self.dim, self.ld,
                  int(state) & ((1 << 64) - 1), code, ptr,
                  torch.cuda.current_stream(self.device).cuda_stream)

    @classmethod
    def generated(cls, n_vertices: int, dim: int, seed: int, dtype=torch.bfloat16,
                  device="cuda", ld=None) -> "FeatureTable":
        """Whole matrix on one device (single-GPU / replicated layout)."""
        t = cls(n_vertices, dim, dtype, device, ld)
        t.fill_generated(0, n_vertices, feature_state(seed))
        return t

    @classmethod
    def from_matrix(cls, matrix, dtype=torch.float32, device="cuda", ld=None) -> "FeatureTable":
        """A loaded feature matrix (read_feature_file; featstore.py:161-184
        source="file") uploaded to HBM, rows padded to ld."""
        m = torch.as_tensor(np.ascontiguousarray(matrix, dtype=np.float32))
        t = cls(m.shape[0], m.shape[1], dtype, device, ld)
        t.table[:, :t.dim].copy_(m.to(device=t.device, dtype=dtype))
        return t

    @classmethod
    def from_file(cls, path, dtype=torch.float32, device="cuda", ld=None) -> "FeatureTable":
        return cls.from_matrix(read_feature_file(path), dtype, device, ld)

    def rows(self, ids) -> np.ndarray:
        ids = torch.as_tensor(np.asarray(ids, dtype=np.int64), device=self.device)
        r = ids if self.row_of is None else self.row_of[ids].long()
        return self.table[r, :self.dim].float().cpu().numpy()


@dataclass(frozen=True)
class PregatherPlan:
    """Deduplicated remote rows one server needs for an iteration (featstore.py:208-223)."""

    server: int
    by_source: tuple

    @property
    def total_rows(self) -> int:
        return sum(len(ids) for _, ids in self.by_source)

    @property
    def all_ids(self) -> np.ndarray:
        if not self.by_source:
            return np.empty(0, dtype=np.int64)
        return np.concatenate([ids for _, ids in self.by_source])


def plan_pregather(at: int, vertex_sets, home: np.ndarray) -> PregatherPlan:
    """Union the needs of every micrograph trained at `at`, minus local, by home."""
    sets = [np.asarray(v) for v in vertex_sets]
    need = np.unique(np.concatenate(sets)) if sets else np.empty(0, dtype=np.int64)
    remote = need[home[need] != at] if len(need) else need
    rh = home[remote] if len(remote) else np.empty(0, dtype=np.int64)
    return PregatherPlan(at, tuple((int(s), remote[rh == s]) for s in np.unique(rh)))
