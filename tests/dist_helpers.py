"""Worker bodies for multi-process tests (importable by torch.multiprocessing.spawn)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


class _Table:
    def __init__(self, table, row_of):
        self.table, self.row_of = table, row_of
        self.ld = table.shape[1]
        self.dtype = table.dtype


class FakeShard:
    """CPU stand-in for ShardedFeatures: same attributes pregather() uses."""

    def __init__(self, home, rank, S, dim, fstate, staging):
        from oracle.kernels import feature_rows
        local = np.flatnonzero(home == rank)
        self.n_local = len(local)
        table = torch.zeros((self.n_local + staging, dim), dtype=torch.float32)
        if self.n_local:
            table[:self.n_local] = torch.from_numpy(feature_rows(local, dim, fstate))
        row_of = torch.full((len(home),), -1, dtype=torch.int32)
        row_of[torch.from_numpy(local)] = torch.arange(self.n_local, dtype=torch.int32)
        self.table = _Table(table, row_of)
        self.staging_cap = staging
        self.home = torch.from_numpy(home.astype(np.int32))
        self.rank, self.S, self.device = rank, S, torch.device("cpu")


def pregather_worker(rank, world, init_file, result_file):
    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank,
                            world_size=world)
    from oracle.featstore_ref import pregather_expect
    from paper_2409_00657_b200.distributed import pregather
    n, dim, fstate = 500, 12, 77
    rng = np.random.default_rng(5)
    home = rng.integers(0, world, n)
    feats = FakeShard(home, rank, world, dim, fstate, staging=n)
    need = [torch.from_numpy(rng.integers(0, n, 40 + 13 * r).astype(np.int32))
            for r in range(rank + 2)]
    per_home, n_req, nbytes, req_bytes = pregather(feats, need)
    want_counts, want_ids, want_rows = pregather_expect(
        rank, [x.numpy() for x in need], home, world, dim, fstate)
    ok = np.array_equal(per_home, want_counts) and n_req == len(want_ids)
    got_rows = feats.table.table[feats.table.row_of[torch.from_numpy(want_ids)].long()].numpy()
    ok = ok and np.array_equal(got_rows, want_rows)
    ok = ok and nbytes == n_req * dim * 4 and req_bytes == n_req * 8
    with open(f"{result_file}.{rank}", "w") as f:
        f.write("ok" if ok else f"bad counts={per_home} want={want_counts}")
    dist.destroy_process_group()


def micrograph_worker(rank, world, init_file, result_file, mode, dtype_name, feat_mode="pg",
                      strategy="micrograph", iters=3, graph_group=1, csr="replicated",
                      allreduce="p2p"):
    """Full multi-GPU micrograph (or model-centric) iterations vs the oracle
    engine (ledger exact, parameters within tolerance)."""
    import json
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"file://{init_file}", rank=rank,
                            world_size=world)
    from oracle import engine as OE
    from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables
    from oracle.rng import chain, keyed
    from paper_2409_00657_b200.distributed import MicrographTrainer
    from paper_2409_00657_b200.graph import Graph, PartitionMap
    from paper_2409_00657_b200.model import init_model
    seed, arch, fo, D, H, C, B = 3, "sage-mean", (15, 10), 16, 64, 5, 64
    off, tgt = build_csr(build_tables(OSpec(n=3000, avg_deg=12.0, beta=0.7, p_in=0.9,
                                            n_blocks=4, d_cap=600, seed=11)))
    home = (keyed(chain(seed, 0x02, 0xA7), np.arange(3000)) % np.uint64(world)).astype(np.int64)
    dtype = torch.float32 if dtype_name == "f32" else torch.bfloat16
    if csr == "sharded-blocks":  # contiguous homes: planted-block style partition
        home = (np.arange(3000) * world) // 3000
    G = Graph.from_host(off, tgt, f"cuda:{rank}")
    part = PartitionMap(home, world, f"cuda:{rank}")
    if csr != "replicated":  # this rank keeps only its rows; peers' shards over NVLink
        from paper_2409_00657_b200.graph import ShardedGraph
        G = ShardedGraph.from_graph(G, part, rank)
    model = init_model(arch, D, H, len(fo), C, chain(seed, 0x07), f"cuda:{rank}")
    tr = MicrographTrainer(G, part, model, fo, B, seed, lr=0.1, dtype=dtype, mode=mode,
                           iterations=iters, pregather=(feat_mode == "pg"), strategy=strategy,
                           graph_group=graph_group, allreduce=allreduce)
    tr.begin_epoch(0)
    losses = [tr.step(it) for it in range(tr.iters)]
    torch.cuda.synchronize()
    graph_used = tr._dgl is not None
    led = tr.global_ledger()
    params = [p.tolist() for p in model.params()]
    out = {"ok": True, "msg": ""}
    if rank == 0:
        w = OE.World(off, tgt, home, world, seed, arch, D, H, C, fo, B, iterations=iters)
        P = w.fresh_params()
        oled = OE.Ledger()
        for it, batches in enumerate(OE.epoch_batches(seed, 0, 3000, world, B, iters)):
            if strategy == "model-centric":
                OE.model_centric_iteration(w, P, 0, it, batches, oled)
            else:
                OE.micrograph_iteration(w, P, 0, it, batches, OE.initial_table(world), (), True,
                                        oled)
        out = _compare(led, oled, model, P, dtype_name)
        out["losses"] = losses
        out["graph_used"] = graph_used
    with open(f"{result_file}.{rank}", "w") as f:
        json.dump(out, f)
    dist.barrier()
    dist.destroy_process_group()


def _compare(led, oled, model, P, dtype_name):
    out = {"ok": True, "msg": ""}
    got = {k: v for k, v in led.counters.items()}
    want = {k: tuple(v) for k, v in oled.cells.items()}
    for k in set(got) | set(want):
        gb, gm = got.get(k, (0.0, 0))
        wb, wm = want.get(k, (0.0, 0))
        if abs(gb - wb) > 1e-9 * max(1.0, abs(wb)) or gm != wm:
            out = {"ok": False, "msg": f"ledger {k}: got {gb},{gm} want {wb},{wm}"}
            break
    # bf16: numerics are pinned by test_step_gpu against a bf16-emulating oracle;
    # here only gross agreement with the exact float64 oracle is required
    tol = 1e-3 if dtype_name == "f32" else 1e-1
    for i, (a, b) in enumerate(zip(model.params(), P.arrays())):
        err = float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))
        if out["ok"] and err > tol:
            out = {"ok": False, "msg": f"param {i} rel err {err}"}
    return out


def merge_worker(rank, world, init_file, result_file, feat_mode):
    """Merging controller over 3 epochs (forced acceptance of the first drop)
    vs the oracle replaying the same decision: tables, ledger, parameters."""
    import json
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"file://{init_file}", rank=rank,
                            world_size=world)
    from oracle import engine as OE
    from oracle.graphgen import GraphSpec as OSpec, build_csr, build_tables
    from oracle.rng import chain, keyed
    from paper_2409_00657_b200.distributed import MicrographTrainer, merge_controller
    from paper_2409_00657_b200.graph import Graph, PartitionMap
    from paper_2409_00657_b200.model import init_model
    seed, arch, fo, D, H, C, B, iters, n = 4, "sage-mean", (10, 5), 16, 64, 5, 48, 2, 2500
    off, tgt = build_csr(build_tables(OSpec(n=n, avg_deg=10.0, beta=0.7, p_in=0.9,
                                            n_blocks=4, d_cap=500, seed=12)))
    home = (keyed(chain(seed, 0x02, 0xA7), np.arange(n)) % np.uint64(world)).astype(np.int64)
    G = Graph.from_host(off, tgt, f"cuda:{rank}")
    part = PartitionMap(home, world, f"cuda:{rank}")
    model = init_model(arch, D, H, len(fo), C, chain(seed, 0x07), f"cuda:{rank}")
    tr = MicrographTrainer(G, part, model, fo, B, seed, lr=0.1, dtype=torch.float32,
                           mode="fused", iterations=iters, pregather=(feat_mode == "pg"))
    tt, hist, times = merge_controller(tr, epochs=3, merge_k=1,
                                       cost=lambda table, sec: float(table.n_columns))
    torch.cuda.synchronize()
    led = tr.global_ledger()
    out = {"ok": True, "msg": ""}
    if rank == 0:
        acts = [(h.action, h.columns) for h in hist]
        want_acts = [("baseline", world), ("accepted", world - 1)]
        want_acts += [("accepted", world - 2)] if world > 2 else [("settled", 1)]
        w = OE.World(off, tgt, home, world, seed, arch, D, H, C, fo, B, iterations=iters)
        P = w.fresh_params()
        oled = OE.Ledger()
        server_of, removed = OE.initial_table(world), ()
        for epoch in range(3):
            if epoch > 0 and server_of.shape[1] >= 2:
                first = OE.epoch_batches(seed, epoch, n, world, B, iters)[0]
                groups = [tuple(b[home[b] == s] for s in range(world)) for b in first]
                cells = OE.assign_cells(groups, removed, chain(seed, 0x08, epoch, 0))
                counts = np.array([[len(c) for c in row] for row in cells])
                col = OE.fewest_column(counts)
                server_of, _ = OE.delete_column(server_of, counts, col)
                removed = removed + (col,)
            for it, batches in enumerate(OE.epoch_batches(seed, epoch, n, world, B, iters)):
                OE.micrograph_iteration(w, P, epoch, it, batches, server_of, removed, True, oled)
        if acts != want_acts:
            out = {"ok": False, "msg": f"events {acts} want {want_acts}"}
        elif tuple(tt.removed) != tuple(removed) or not np.array_equal(tt.server_of, server_of):
            out = {"ok": False, "msg": f"table {tt.removed} want {removed}"}
        else:
            out = _compare(led, oled, model, P, "f32")
        out["times"] = times
    with open(f"{result_file}.{rank}", "w") as f:
        json.dump(out, f)
    dist.barrier()
    dist.destroy_process_group()
