"""Epoch root order and per-model batches (reference engine.py:268-287).

The permutation is a stable radix argsort of chain(seed, 0x05, epoch, v) on
the GPU (hg_epoch_permutation); batches are views into it.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .rng import chain

SEED_BATCHES = 0x05


def epoch_permutation(seed: int, epoch: int, n: int, device="cuda") -> torch.Tensor:
    """int64[n] permutation == np.argsort(keys, kind="stable") (engine.py:273-275)."""
    dev = torch.device(device)
    out = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    state = chain(seed, SEED_BATCHES, epoch)
    need = C.c_size_t(0)
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.call("hg_epoch_permutation", n, state, out.data_ptr(), None, C.byref(need), stream)
    ws = torch.empty(max(need.value, 1), dtype=torch.uint8, device=dev)
    _lib.call("hg_epoch_permutation", n, state, out.data_ptr(), ws.data_ptr(), C.byref(need),
              stream)
    return out[:n]


def iterations_per_epoch(n: int, n_models: int, batch: int, cap: int = 0) -> int:
    """max(1, n // (N*B)), optionally capped (engine.py:276-278)."""
    iters = max(1, n // (n_models * batch))
    return min(iters, cap) if cap else iters


def batch_slice(perm: torch.Tensor, it: int, d: int, n_models: int, batch: int) -> torch.Tensor:
    """Roots of model d at iteration it (engine.py:282-285)."""
    n = perm.numel()
    lo = min((it * n_models + d) * batch, n)
    return perm[lo:min(lo + batch, n)]
