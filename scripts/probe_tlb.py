"""Diagnostic: random 256-byte row gather vs table footprint (TLB reach probe).

Times torch.index_select (a plain gather) of 105K random rows of 128 bf16
from tables of growing size, random vs sorted ids.  Used to decide whether
the layer-1 feature gather on the papers-shaped table (28 GB) is bound by
address translation rather than DRAM bandwidth.
"""
import torch

dev = torch.device("cuda")
rows = 105_000
D = 128
for gb in (0.25, 1, 4, 8, 16, 28):
    n = int(gb * 2**30 / (D * 2))
    t = torch.empty((n, D), dtype=torch.bfloat16, device=dev)
    t.view(torch.int16).random_()  # touch
    out = torch.empty((rows, D), dtype=torch.bfloat16, device=dev)
    flush = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
    for mode in ("random", "sorted"):
        ts = []
        for it in range(20):
            idx = torch.randint(0, n, (rows,), device=dev)
            if mode == "sorted":
                idx, _ = idx.sort()
            flush.zero_()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            torch.index_select(t, 0, idx, out=out)
            e1.record()
            torch.cuda.synchronize()
            if it >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        us = ts[len(ts) // 2]
        print(f"{gb:6.2f} GB {mode:6s} {us:7.2f} us  {rows*D*2*2/us/1e3:7.1f} GB/s (read+write)")
    del t, out, flush
    torch.cuda.empty_cache()
