"""Micrograph-merging study on BASELINE configs[2] (cfg3: GCN-3, fanout
(10, 10, 10), Reddit-shaped graph, 602-d features), one process per GPU:

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/merge_study.py [--epochs 5]

Runs the merge controller (engine.py:779-833, PAPER Algorithm 1) on measured
epoch time (max over ranks): K = 1 epoch per decision, greedy removal of the
column with the fewest roots, kept only if the epoch gets faster.  Prints one
JSON line (rank 0): the decisions, per-epoch seconds, trace-table columns and
the reference-ledger bytes per epoch by category.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from bench import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=5)
    ap.add_argument("--iterations", type=int, default=40)
    ap.add_argument("--config", default="reddit")
    args = ap.parse_args()
    from paper_2409_00657_b200.distributed import MicrographTrainer, merge_controller
    from paper_2409_00657_b200.graph import GraphSpec, PartitionMap, ShardedGraph, generate
    from paper_2409_00657_b200.model import init_model
    from paper_2409_00657_b200.rng import chain
    rank, local = int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    S = dist.get_world_size()
    cfg = CONFIGS[args.config]
    spec = GraphSpec(**{k: cfg[k] for k in ("n", "avg_deg", "beta", "p_in", "n_blocks", "d_cap",
                                            "seed")})
    g = generate(spec, dev)
    blocks = (np.arange(spec.n, dtype=np.int64) * spec.n_blocks) // spec.n
    part = PartitionMap((blocks * S) // spec.n_blocks, S, dev)
    g = ShardedGraph.from_graph(g, part, rank)
    torch.cuda.empty_cache()
    model = init_model(cfg["arch"], cfg["dim"], cfg["hidden"], len(cfg["fanout"]),
                       cfg["classes"], chain(cfg["seed"], 0x07), dev)
    tr = MicrographTrainer(g, part, model, cfg["fanout"], cfg["batch"], cfg["seed"],
                           iterations=args.iterations)
    # one untimed epoch first: graph capture and library warm-up would otherwise
    # land in the controller's baseline epoch and bias it toward accepting a drop
    from paper_2409_00657_b200.distributed import run_epoch
    run_epoch(tr, 0)
    tr.ledger = type(tr.ledger)()
    tt, hist, times = merge_controller(tr, epochs=args.epochs, merge_k=1)
    led = tr.global_ledger()
    if rank == 0:
        print(json.dumps({
            "study": "merge controller on measured epoch time",
            "workload": cfg["workload"], "gpus": S, "epochs": args.epochs,
            "iterations_per_epoch": args.iterations, "batch_per_model": cfg["batch"],
            "events": [{"start_epoch": h.epoch_start, "epochs": h.epochs, "columns": h.columns,
                        "avg_seconds": round(h.avg_seconds, 5), "action": h.action}
                       for h in hist],
            "epoch_seconds": [round(t, 5) for t in times],
            "final_columns": tt.n_columns, "removed_columns": list(tt.removed),
            "ledger_bytes_total_by_category": {k: round(v, 1) for k, v in
                                               led.bytes_by_category().items()},
        }), flush=True)
    dist.barrier()
    tr.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
