"""GNN parameters and math on the device (drop-in for reference gnnsim.model)."""
from __future__ import annotations

import torch

from . import _lib


def glorot_device(rows: int, cols: int, state: int, dtype=torch.float64, device="cuda"):
    """Keyed Glorot uniform, bit-identical to model.py:87-90 (f64) ."""
    out = torch.empty((rows, cols), dtype=dtype, device=device)
    code = 0 if dtype == torch.float64 else 1
    _lib.call("hg_glorot", rows, cols, state & ((1 << 64) - 1), code, out.data_ptr(),
              torch.cuda.current_stream(out.device).cuda_stream)
    return out
