"""Drop-in for the reference operator layer ``gnnsim.kernels`` (kernels.py:1-48).

Same function names and argument meaning; the implementation is the CUDA
library (no backend switch, no CPU fallback).  Inputs may be numpy arrays
(uploaded per call, the reference's calling convention) or CUDA tensors
(used in place).  Outputs are numpy arrays like the reference.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

BACKEND = "cuda"


def _dev(x, dtype, device="cuda"):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device=device)


def sample_frontier(offsets, targets, frontier, fanout: int, state: int):
    """(counts, flat) for one frontier (_kernels_nb.py:55-90)."""
    off = _dev(offsets, torch.int64)
    tgt = _dev(targets, torch.int32)
    fr = _dev(frontier, torch.int64)
    n = off.numel() - 1
    f = fr.numel()
    counts = torch.empty(max(f, 1), dtype=torch.int64, device=off.device)
    cap = max(f * int(fanout), 1)
    flat = torch.empty(cap, dtype=torch.int64, device=off.device)
    got = C.c_int64(0)
    stream = torch.cuda.current_stream(off.device).cuda_stream
    _lib.call("hg_sample_frontier", off.data_ptr(), tgt.data_ptr(), n, fr.data_ptr(), f,
              int(fanout), int(state) & ((1 << 64) - 1), counts.data_ptr(), flat.data_ptr(), cap,
              C.byref(got), stream)
    return counts[:f].cpu().numpy(), flat[:got.value].cpu().numpy()


def feature_rows(ids, dim: int, state: int) -> np.ndarray:
    """Deterministic float32 rows in [-0.5, 0.5) (_kernels_nb.py:109-122)."""
    idt = _dev(ids, torch.int64)
    out = torch.empty((idt.numel(), int(dim)), dtype=torch.float32, device=idt.device)
    stream = torch.cuda.current_stream(idt.device).cuda_stream
    _lib.call("hg_feature_rows", idt.data_ptr(), idt.numel(), int(dim),
              int(state) & ((1 << 64) - 1), out.data_ptr(), stream)
    return out.cpu().numpy()


def probability_threshold(p: float):
    """(mode, threshold) encoding of an acceptance probability (kernels.py:37-48)."""
    if p <= 0.0:
        return 0, 0
    if p >= 1.0:
        return 2, 0
    return 1, min(int(p * 2.0 ** 64), (1 << 64) - 1)
