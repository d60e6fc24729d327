"""Time hg_gemm_bf16 on the train-step shapes (papers SAGE-2, B=1024).
    python scripts/bench_gemm.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_00657_b200 import _lib

dev = torch.device("cuda")
# (name, M, N, K, a_mn, b_mn, epi, split)
SHAPES = [("fwd1 agg1.W1 bias-relu", 11328, 256, 256, 0, 0, 1, 1),
          ("fwd2 agg2.W2 bias-relu", 1024, 256, 512, 0, 0, 1, 1),
          ("head h2.WcT", 1024, 172, 256, 0, 0, 0, 1),
          ("dz2 dl.Wcp", 1024, 256, 192, 0, 0, 0, 1),
          ("gWc h2T.dl", 256, 172, 1024, 1, 1, 2, 4),
          ("gW2 agg2T.dz2", 512, 256, 1024, 1, 1, 2, 8),
          ("dagg2 dz2.W2b", 1024, 512, 256, 0, 0, 0, 1),
          ("gW1 agg1T.dz1", 256, 256, 11328, 1, 1, 2, 37)]


def run(M, N, K, a_mn, b_mn, epi, split, reps=200):
    ldb = N if b_mn else K
    Np = (N + 63) // 64 * 64
    A = (torch.randn(K, M) if a_mn else torch.randn(M, K)).to(dev, torch.bfloat16)
    B = (torch.randn(K, Np) if b_mn else torch.randn(Np, K)).to(dev, torch.bfloat16)
    ldb = Np if b_mn else K
    Cm = torch.zeros(M, N, device=dev, dtype=torch.bfloat16 if epi == 1 else torch.float32)
    bias = torch.randn(N, device=dev)
    lda = M if a_mn else K

    def once():
        s = torch.cuda.current_stream().cuda_stream
        _lib.call("hg_gemm_bf16", A.data_ptr(), lda, a_mn, B.data_ptr(), ldb, b_mn, Cm.data_ptr(),
                  N, M, N, K, epi, bias.data_ptr(), split, s)
    for _ in range(10):
        once()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps // 20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / reps
    # check vs torch
    Af = A.float().t() if a_mn else A.float()
    Bf = B.float()[:, :N] if b_mn else B.float()[:N].t()
    ref = Af @ Bf
    if epi == 1:
        ref = torch.relu(ref + bias)
    got = Cm.float()
    if epi == 2:
        Cm.zero_(); once(); torch.cuda.synchronize(); got = Cm.float()
    err = float((got - ref).abs().max() / ref.abs().max())
    # cuBLAS (torch bf16 matmul) on the same shape, same graph-replay timing
    At = A.t() if a_mn else A
    Bt = B[:, :N] if b_mn else B[:N].t()
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    for _ in range(10):
        torch.matmul(At, Bt, out=out)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        for _ in range(20):
            torch.matmul(At, Bt, out=out)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps // 20):
        g2.replay()
    e1.record()
    torch.cuda.synchronize()
    cub = e0.elapsed_time(e1) * 1000 / reps
    return us, err, cub


tot = 0.0
for name, *shape in SHAPES:
    us, err, cub = run(*shape)
    tot += us
    M, N, K = shape[:3]
    print(f"{name:28s} M={M:6d} N={N:4d} K={K:6d}  {us:7.2f} us  "
          f"{2*M*N*K/us/1e6:8.1f} TF/s  err={err:.1e}  cuBLAS {cub:7.2f} us")
print(f"total {tot:.1f} us")
