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


@pytest.mark.parametrize("M,N,K,bn,sp,bm", [(128, 128, 64, 128, 1, 256), (512, 2048, 1536, 128, 1, 256),
                                            (512, 2048, 1536, 128, 4, 256), (200, 1536, 1536, 128, 6, 256),
                                            (37, 4096, 256, 256, 1, 256), (1000, 4608, 3584, 128, 2, 256),
                                            (1, 128, 128, 128, 2, 256), (300, 512, 256, 128, 1, 256),
                                            (512, 2048, 1536, 128, 1, 128), (300, 4096, 256, 256, 1, 128),
                                            (77, 1536, 1536, 128, 3, 128)])
def test_gemm_bf16_bias(dev, M, N, K, bn, sp, bm):
    from paper_2510_19225_b200.instance import gemm
    A, B, bias = _rand((M, K), 1.0, 1), _rand((N, K), 0.05, 2), _rand((N,), 0.1, 3)
    out = gemm(dev, A, B, bias=bias, epilogue=0, block_n=bn, splits=sp, block_m=bm)
    ref = A.float() @ B.float().T + bias.float()
    torch.testing.assert_close(out.float(), ref, rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("M,N,K,bn,sp,bm", [(512, 1536, 8960, 128, 5, 256), (130, 256, 1024, 128, 1, 256),
                                            (64, 1536, 1536, 128, 6, 256), (700, 3584, 18944, 128, 2, 256),
                                            (512, 1536, 1536, 128, 1, 128), (300, 1536, 8960, 128, 4, 128),
                                            (1, 1536, 8960, 128, 7, 128), (200, 512, 1024, 256, 1, 256),
                                            (512, 1536, 8960, 128, 6, 256), (300, 1536, 8960, 128, 8, 256)])
def test_gemm_residual_add(dev, M, N, K, bn, sp, bm):
    """fp32 h += A.B^T; split-K (block_n 128) reduces its splits in a cluster."""
    from paper_2510_19225_b200.instance import gemm
    A, B = _rand((M, K), 1.0, 4), _rand((N, K), 0.02, 5)
    h = torch.randn(M, N, device="cuda")
    ref = h + A.float() @ B.float().T
    out = gemm(dev, A, B, out=h.clone(), epilogue=1, block_n=bn, splits=sp, block_m=bm)
    # fp32 accumulation over K up to 18944 in a different order than cuBLAS
    torch.testing.assert_close(out, ref, rtol=2e-4, atol=5e-4)


@pytest.mark.parametrize("M,F,K,bn,bm", [(512, 8960, 1536, 256, 256), (77, 1024, 256, 128, 256),
                                         (300, 1024, 256, 256, 256), (300, 1024, 256, 256, 128)])
def test_gemm_swiglu_interleaved(dev, M, F, K, bn, bm):
    from paper_2510_19225_b200.instance import gemm
    A = _rand((M, K), 1.0, 6)
    gate, up = _rand((F, K), 0.05, 7), _rand((F, K), 0.05, 8)
    # engine layout: 64-row gate block, 64-row up block, alternating
    wgu = torch.stack([gate.view(F // 64, 64, K), up.view(F // 64, 64, K)], 1).reshape(2 * F, K)
    out = gemm(dev, A, wgu.contiguous(), epilogue=2, block_n=bn, block_m=bm)
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


@pytest.mark.parametrize("sp,bm", [(1, 256), (4, 256), (1, 128)])
def test_gemm_rows_batch_invariant(dev, sp, bm):
    """A row's output is bit-identical whatever else is in the batch and
    wherever the row sits in it (the property migration resume relies on),
    with and without split-K."""
    from paper_2510_19225_b200.instance import gemm
    K, N = 1536, 2048
    B, bias = _rand((N, K), 0.05, 11), _rand((N,), 0.1, 12)
    rows = _rand((40, K), 1.0, 13)
    small = gemm(dev, rows.contiguous(), B, bias=bias, epilogue=0, block_n=128, splits=sp, block_m=bm)
    big = _rand((3000, K), 1.0, 14)
    idx = torch.randperm(3000, generator=torch.Generator().manual_seed(0))[:40].cuda()
    big[idx] = rows
    out = gemm(dev, big, B, bias=bias, epilogue=0, block_n=128, splits=sp, block_m=bm)
    assert torch.equal(out[idx], small)


@pytest.mark.parametrize("sp,bm", [(5, 256), (7, 128)])
def test_resadd_cluster_batch_invariant(dev, sp, bm):
    """The cluster split-K reduction sums a row's splits in the same order
    whatever the batch: bit-identical rows."""
    from paper_2510_19225_b200.instance import gemm
    K, N = 8960, 1536
    B = _rand((N, K), 0.02, 15)
    rows, h_rows = _rand((40, K), 1.0, 16), torch.randn(40, N, device="cuda")
    small = gemm(dev, rows.contiguous(), B, out=h_rows.clone(), epilogue=1, block_n=128, splits=sp,
                 block_m=bm)
    big, h = _rand((700, K), 1.0, 17), torch.randn(700, N, device="cuda")
    idx = torch.randperm(700, generator=torch.Generator().manual_seed(1))[:40].cuda()
    big[idx], h[idx] = rows, h_rows
    out = gemm(dev, big, B, out=h, epilogue=1, block_n=128, splits=sp, block_m=bm)
    assert torch.equal(out[idx], small)


@pytest.mark.parametrize("M", [512, 300, 4096, 77])
def test_gemm_swiglu_pair_tiles(dev, monkeypatch, M):
    """Persistent 2-SM pair tiles (cta_group::2, 256 x 256 tiles with
    double-buffered TMEM): same bits as the single-SM kernel."""
    from paper_2510_19225_b200.instance import gemm
    F, K = 8960, 1536
    A = _rand((M, K), 1.0, 23)
    wgu = _rand((2 * F, K), 0.05, 24)
    ref = gemm(dev, A, wgu, epilogue=2, block_n=256)
    monkeypatch.setenv("RLB_GEMM_PAIR", "2")
    out = gemm(dev, A, wgu, epilogue=2, block_n=256)
    assert torch.equal(out, ref)


@pytest.mark.parametrize("M,N,K,sp", [(512, 1536, 8960, 5), (300, 1536, 8960, 6), (2048, 1536, 8960, 5),
                                      (77, 1536, 1536, 3), (1000, 3584, 18944, 4), (512, 1536, 1536, 7)])
def test_gemm_splitk_partials_pair_tiles(dev, monkeypatch, M, N, K, sp):
    """Persistent 2-SM tiles writing split-K fp32 partials (the down / O
    projections above the small-batch plans): every split covers the same K
    blocks as the single-SM kernel, so the reduced result has the same bits."""
    from paper_2510_19225_b200.instance import gemm
    A, B = _rand((M, K), 1.0, 31), _rand((N, K), 0.02, 32)
    ref = gemm(dev, A, B, epilogue=3, block_n=128, splits=sp)
    monkeypatch.setenv("RLB_GEMM_PAIR", "2")
    out = gemm(dev, A, B, epilogue=3, block_n=128, splits=sp)
    assert torch.equal(out, ref)
    torch.testing.assert_close(out, A.float() @ B.float().T, rtol=2e-4, atol=5e-4)
