"""Scratch: locate the bench-shape sampling mismatch (generator vs sampler)."""
import sys, os, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from bench import CONFIGS
from oracle.graphgen import GraphSpec as OSpec, rows_csr, build_tables, row, raw_degree
from oracle.cpu_bench import LazyGraphSampler
from oracle.rng import chain
from paper_2409_00657_b200.graph import GraphSpec, generate
from test_parity_bench_gpu import _device_rows, _spec_kw

out = {}
for name in ("reddit", "papers"):
    cfg = CONFIGS[name]
    kw = _spec_kw(cfg)
    g = generate(GraphSpec(**kw))
    t = build_tables(OSpec(**kw))
    rng = np.random.default_rng(0)
    vs = np.unique(rng.integers(0, kw["n"], 3000))
    od, td = _device_rows(g, vs)
    oo, to = rows_csr(t, vs)
    dd, do = np.diff(od), np.diff(oo)
    bad = np.flatnonzero((dd != do) | np.array([not np.array_equal(td[od[i]:od[i+1]], to[oo[i]:oo[i+1]]) for i in range(len(vs))]))
    info = {"rows": len(vs), "bad_rows": int(len(bad))}
    if len(bad):
        i = bad[0]
        v = int(vs[i])
        info["first"] = {"v": v, "dev_deg": int(dd[i]), "cpu_deg": int(do[i]),
                         "raw_deg": int(raw_degree(t, np.array([v]))[0]),
                         "dev": td[od[i]:od[i+1]][:12].tolist(), "cpu": to[oo[i]:oo[i+1]][:12].tolist(),
                         "row()": row(t, v)[:12].tolist()}
        info["bad_frac_deg"] = float(np.mean(dd[bad] != do[bad]))
    out[name] = info
    print(name, json.dumps(info), flush=True)
    del g
    torch.cuda.empty_cache()
json.dump(out, open("gpurun_out/debug_parity.json", "w"), indent=1)
