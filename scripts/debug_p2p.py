"""Time the NVLink pre-gather copy (k_stage_copy) on synthetic remote row sets:
random over the whole remote shard vs a small window vs sequential rows.
torchrun --nproc-per-node 2 scripts/debug_p2p.py"""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_00657_b200 import _lib
from paper_2409_00657_b200.distributed import PeerFeatures
from paper_2409_00657_b200.graph import PartitionMap

rank, S = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", rank)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
n = 111_000_000
home = ((np.arange(n, dtype=np.int64) * 8 // n) * S // 8).astype(np.int64)
part = PartitionMap(home, S, dev)
pf = PeerFeatures(part, rank, 128, 0, torch.bfloat16, dev, None)


class _R:
    pass


r = _R()
r.desc = _lib.StepDesc()
pf.bind_staged(r, 200_000)
acct = torch.zeros(S, dtype=torch.int64, device=dev)
tot = torch.zeros(1, dtype=torch.int64, device=dev)
other = np.flatnonzero(home == (rank + 1) % S)
rng = np.random.default_rng(rank)
rows = 9000
sets = {"random/all": rng.choice(other, rows, replace=False),
        "random/64MB": other[rng.choice(250_000, rows, replace=False)],
        "sequential": other[:rows],
        "random/all x4": rng.choice(other, 4 * rows, replace=False)}
s = torch.cuda.current_stream().cuda_stream
for name, ids in sets.items():
    ids_d = torch.from_numpy(np.sort(ids).astype(np.int32)).to(dev)
    nd = torch.tensor([len(ids)], dtype=torch.int32, device=dev)
    _lib.prof_enable(True)
    for _ in range(20):
        _lib.call("hg_pregather_peer_at", ids_d.data_ptr(), nd.data_ptr(), pf.home.data_ptr(),
                  rank, pf.local_row.data_ptr(), pf.peers.data_ptr(), 256, pf.bitmap.data_ptr(),
                  pf.stage_list.data_ptr(), pf.stage_row.data_ptr(), pf.stage_count.data_ptr(),
                  pf.stage_cap, pf.staging.data_ptr(), acct.data_ptr(), None, S, tot.data_ptr(),
                  pf.err.data_ptr(), s)
    torch.cuda.synchronize()
    t, c = _lib.prof_read(_lib.PROF_PG_COPY)
    m, _ = _lib.prof_read(_lib.PROF_PG_MARK)
    _lib.prof_enable(False)
    us = t / c * 1000
    if rank == 0:
        print(f"{name:14s} rows={len(ids):6d} copy {us:8.1f} us  {len(ids)*256/us/1e3:7.1f} GB/s  mark {m/c*1000:.1f} us", flush=True)
dist.barrier()
pf.close()
dist.destroy_process_group()
