"""Kernel-level parity of the tcgen05 GEMM (K2) against a plain torch fp32
reference of the same op, through the C ABI entry point rlb_gemm."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_19225_b200 import _lib
    _lib.lib()
    return 0


def _rand(shape, scale=1.0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (scale * torch.randn(shape, generator=g, device="cuda")).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K,bn,sp", [(128, 128, 64, 128, 1), (512, 2048, 1536, 128, 1),
                                         (512, 2048, 1536, 128, 4), (200, 1536, 1536, 128, 6),
                                         (37, 4096, 256, 256, 1), (1000, 4608, 3584, 128, 2),
                                         (1, 128, 128, 128, 2), (300, 512, 256, 128, 1)])
def test_gemm_bf16_bias(dev, M, N, K, bn, sp):
    from paper_2510_19225_b200.instance import gemm
    A, B, bias = _rand((M, K), 1.0, 1), _rand((N, K), 0.05, 2), _rand((N,), 0.1, 3)
    out = gemm(dev, A, B, bias=bias, epilogue=0, block_n=bn, splits=sp)
    ref = A.float() @ B.float().T + bias.float()
    torch.testing.assert_close(out.float(), ref, rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("M,N,K,bn,sp", [(512, 1536, 8960, 128, 5), (130, 256, 1024, 128, 1),
                                         (64, 1536, 1536, 128, 6), (700, 3584, 18944, 128, 2)])
def test_gemm_residual_add(dev, M, N, K, bn, sp):
    from paper_2510_19225_b200.instance import gemm
    A, B = _rand((M, K), 1.0, 4), _rand((N, K), 0.02, 5)
    h = torch.randn(M, N, device="cuda")
    ref = h + A.float() @ B.float().T
    out = gemm(dev, A, B, out=h.clone(), epilogue=1, block_n=bn, splits=sp)
    # fp32 accumulation over K up to 18944 in a different order than cuBLAS
    torch.testing.assert_close(out, ref, rtol=2e-4, atol=5e-4)


@pytest.mark.parametrize("M,F,K,bn", [(512, 8960, 1536, 256), (77, 1024, 256, 128), (300, 1024, 256, 256)])
def test_gemm_swiglu_interleaved(dev, M, F, K, bn):
    from paper_2510_19225_b200.instance import gemm
    A = _rand((M, K), 1.0, 6)
    gate, up = _rand((F, K), 0.05, 7), _rand((F, K), 0.05, 8)
    # engine layout: 64-row gate block, 64-row up block, alternating
    wgu = torch.stack([gate.view(F // 64, 64, K), up.view(F // 64, 64, K)], 1).reshape(2 * F, K)
    out = gemm(dev, A, wgu.contiguous(), epilogue=2, block_n=bn)
    g, u = A.float() @ gate.float().T, A.float() @ up.float().T
    ref = torch.nn.functional.silu(g) * u
    torch.testing.assert_close(out.float(), ref, rtol=2e-2, atol=2e-2)


def test_gemm_fp32_logits_tail(dev):
    from paper_2510_19225_b200.instance import gemm
    M, N, K = 96, 151936, 1536
    A, B = _rand((M, K), 1.0, 9), _rand((N, K), 0.01, 10)
    out = gemm(dev, A, B, epilogue=3, block_n=256)
    ref = A.float() @ B.float().T
    torch.testing.assert_close(out, ref, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("sp", [1, 4])
def test_gemm_rows_batch_invariant(dev, sp):
    """A row's output is bit-identical whatever else is in the batch and
    wherever the row sits in it (the property migration resume relies on),
    with and without split-K."""
    from paper_2510_19225_b200.instance import gemm
    K, N = 1536, 2048
    B, bias = _rand((N, K), 0.05, 11), _rand((N,), 0.1, 12)
    rows = _rand((40, K), 1.0, 13)
    small = gemm(dev, rows.contiguous(), B, bias=bias, epilogue=0, block_n=128, splits=sp)
    big = _rand((3000, K), 1.0, 14)
    idx = torch.randperm(3000, generator=torch.Generator().manual_seed(0))[:40].cuda()
    big[idx] = rows
    out = gemm(dev, big, B, bias=bias, epilogue=0, block_n=128, splits=sp)
    assert torch.equal(out[idx], small)
