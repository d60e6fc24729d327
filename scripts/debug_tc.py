import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2409_00657_b200 import _lib
from paper_2409_00657_b200.graph import GraphSpec, generate
from paper_2409_00657_b200.featstore import FeatureTable
from paper_2409_00657_b200.model import init_model, LabelOracle
from paper_2409_00657_b200.trainer import CellRunner
g = generate(GraphSpec(n=100000, avg_deg=15, beta=0.6, seed=1))
t = FeatureTable.generated(g.n_vertices, 128, 0, torch.bfloat16)
m = init_model("sage-mean", 128, 256, 2, 172, 3)
r = CellRunner(g, t, m, (15, 10), 1024, LabelOracle(172, 5))
print("use_tc", r.desc.use_tc, "act", r.desc.act_dtype, "H", r.desc.hidden, "sizeof", _lib.C.sizeof(_lib.StepDesc) if hasattr(_lib,'C') else None)
import ctypes
print("sizeof desc", ctypes.sizeof(_lib.StepDesc), "offset use_tc", _lib.StepDesc.use_tc.offset, "features", _lib.StepDesc.features.offset)
r.stage_roots(np.arange(1024), [np.int64(5)], 1024)
_lib.launch_count(reset=True)
r.launch(); torch.cuda.synchronize()
print("launches", _lib.launch_count())
