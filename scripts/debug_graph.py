"""Stream launches vs CUDA-graph replay of one hg_train_step (papers-like shape,
1M-vertex graph).  Shows how much of the step is launch gaps."""
import ctypes as C
import sys
import torch
sys.path.insert(0, '.')
from paper_2409_00657_b200 import _lib
from paper_2409_00657_b200.engine import Trainer
from paper_2409_00657_b200.featstore import FeatureTable
from paper_2409_00657_b200.graph import GraphSpec, generate
from paper_2409_00657_b200.model import init_model
g = generate(GraphSpec(n=2_000_000, avg_deg=15, beta=0.6, seed=1))
t = FeatureTable.generated(g.n_vertices, 128, 0, torch.bfloat16)
m = init_model("sage-mean", 128, 256, 2, 172, 3)
tr = Trainer(g, t, m, (15, 10), 1024, 0, run_ahead=False)
tr.begin_epoch(0)
tr.step(0)
torch.cuda.synchronize()
r = tr.runner
n = r.n_roots
print("n_roots", n)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) * 1000 / reps


def step():
    _lib.call("hg_train_step", C.byref(r.desc), n, torch.cuda.current_stream().cuda_stream)


print("stream launches  us/step", round(timeit(step), 1))
gr = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    step()
    torch.cuda.synchronize()
    with torch.cuda.graph(gr, stream=s):
        step()
print("graph replay     us/step", round(timeit(gr.replay), 1))
_lib.launch_count(reset=True)
step()
print("launches per step", _lib.launch_count())
