"""tcgen05 bf16 GEMM (csrc/hg_umma.cu) against a torch fp32 reference of the
same op on the same bf16 inputs.  Tolerance: fp32 accumulation of bf16
products -> 1e-3 relative to max|ref| (plus 1 bf16 ulp on bf16 outputs)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def run(A, lda, a_mn, B, ldb, b_mn, C, ldc, M, N, K, epi, bias=None, split=1):
    from paper_2409_00657_b200 import _lib
    _lib.call("hg_gemm_bf16", A.data_ptr(), lda, int(a_mn), B.data_ptr(), ldb, int(b_mn),
              C.data_ptr(), ldc, M, N, K, epi, bias.data_ptr() if bias is not None else None,
              split, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 256, 256), (11357, 256, 256),
                                   (1000, 128, 512), (77, 64, 200), (1024, 192, 512)])
def test_kmajor_bias_relu_and_store(M, N, K):
    torch.manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = torch.randn(K, N, device="cuda") * 0.1
    Wt = W.t().contiguous().to(torch.bfloat16)          # [N x K] K-major B
    bias = torch.randn(N, device="cuda")
    ref = A.float() @ Wt.float().t()
    C = torch.zeros(M, N, device="cuda")
    run(A, K, False, Wt, K, False, C, N, M, N, K, 0)
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-3, err
    H = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    run(A, K, False, Wt, K, False, H, N, M, N, K, 1, bias)
    want = torch.relu(ref + bias)
    err = (H.float() - want).abs().max().item() / want.abs().max().item()
    assert err < 8e-3, err


@pytest.mark.parametrize("rows,I,N,split", [(64, 128, 256, 1), (11357, 256, 256, 16),
                                            (1024, 512, 256, 4), (5000, 128, 64, 7),
                                            (200, 256, 128, 3)])
def test_mnmajor_split_accumulate(rows, I, N, split):
    """dW = aggᵀ dz: both operands MN-major, reduction over graph rows, split-K
    partials added atomically into an existing accumulator."""
    torch.manual_seed(rows)
    agg = torch.randn(rows, I, device="cuda").to(torch.bfloat16)
    dz = torch.randn(rows, N, device="cuda").to(torch.bfloat16)
    ref = agg.float().t() @ dz.float()
    acc = torch.ones(I, N, device="cuda")
    run(agg, I, True, dz, N, True, acc, N, I, N, rows, 2, None, split)
    err = (acc - 1.0 - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-3, err
    C = torch.zeros(I, N, device="cuda")
    run(agg, I, True, dz, N, True, C, N, I, N, rows, 0)
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-3, err
