import sys, torch
sys.path.insert(0, '.')
from paper_2409_00657_b200 import _lib
from paper_2409_00657_b200.engine import Trainer
from paper_2409_00657_b200.featstore import FeatureTable
from paper_2409_00657_b200.graph import GraphSpec, generate
from paper_2409_00657_b200.model import init_model
g = generate(GraphSpec(n=1_000_000, avg_deg=15, beta=0.6, seed=1))
t = FeatureTable.generated(g.n_vertices, 128, 0, torch.bfloat16)
m = init_model("sage-mean", 128, 256, 2, 172, 3)
tr = Trainer(g, t, m, (15, 10), 1024, 0)
tr.begin_epoch(0)
print("use_tc", tr.runner.desc.use_tc, tr.runner.desc.act_dtype, tr.runner.desc.hidden)
for i in range(3):
    _lib.launch_count(reset=True)
    tr.step(i); torch.cuda.synchronize()
    print("launches", _lib.launch_count())
_lib.prof_enable(True)
for i in range(3, 8): tr.step(i)
torch.cuda.synchronize()
for s in range(7): print(s, _lib.prof_read(s))
