"""Where does the N>1 end-to-end time go?  torchrun --nproc-per-node 2."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import bench
from paper_2409_00657_b200.distributed import MicrographTrainer
from paper_2409_00657_b200.graph import GraphSpec, PartitionMap, generate
from paper_2409_00657_b200.model import init_model
from paper_2409_00657_b200.rng import chain

cfg = bench.CONFIGS[os.environ.get("CFG", "papers")]
rank, local, S = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", local)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
spec = GraphSpec(n=cfg["n"], avg_deg=cfg["avg_deg"], beta=cfg["beta"], p_in=cfg["p_in"],
                 n_blocks=cfg["n_blocks"], d_cap=cfg["d_cap"], seed=cfg["seed"])
g = generate(spec, dev)
blocks = (np.arange(spec.n, dtype=np.int64) * spec.n_blocks) // spec.n
part = PartitionMap((blocks * S) // spec.n_blocks, S, dev)
model = init_model(cfg["arch"], cfg["dim"], cfg["hidden"], len(cfg["fanout"]), cfg["classes"],
                   chain(cfg["seed"], 0x07), dev)
tr = MicrographTrainer(g, part, model, cfg["fanout"], cfg["batch"], cfg["seed"], pregather=False)
tr.begin_epoch(0)
it = 0
def loop(K, want):
    global it
    dist.barrier(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    hs = []
    for _ in range(K):
        h = time.perf_counter()
        tr.step(it, want_loss=want); it += 1
        hs.append(time.perf_counter() - h)
    h1 = time.perf_counter()
    if want:
        tr.last_loss()
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    return t / K * 1e3, float(np.median(hs)) * 1e3, float(np.max(hs)) * 1e3, (h1 - t0) / K * 1e3
loop(10, False)
res = {}
res["noloss"] = [round(x, 4) for x in loop(30, False)]
tr.flush_accounting()
tr.global_ledger()
res["loss_after_ledger"] = [round(x, 4) for x in loop(30, True)]
res["loss2"] = [round(x, 4) for x in loop(30, True)]
print(rank, json.dumps(res), flush=True)
dist.barrier()
dist.destroy_process_group()
