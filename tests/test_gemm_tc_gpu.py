"""tcgen05 tensor-core GEMM (ramp-head classifier) vs a torch fp32 matmul of
the same bf16 operands. bf16 x bf16 products are exact in fp32, so only the
fp32 accumulation order differs: tolerance 1e-3 relative to the output scale."""

from __future__ import annotations

import pytest
import torch

from oracle import heads_ref as H
from paper_2312_05385_b200.heads import LargeRampHead, linear_tc, pool_bf16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k,splits", [
    (256, 1000, 2048, 0),   # ResNet-50 last-stage ramp head, auto split-K
    (256, 1000, 2048, 1),   # no split
    (128, 128, 64, 1),      # one tile, one k-tile
    (100, 10, 64, 0),       # partial M tile, N < 64 (BN = 64 path)
    (33, 130, 200, 3),      # K not a multiple of 64, partial N tile
    (512, 256, 512, 2),
])
def test_gemm_matches_torch(cuda, m, n, k, splits):
    g = torch.Generator().manual_seed(m * 7 + n + k)
    a = torch.randn(m, k, generator=g).to(torch.bfloat16)
    b = torch.randn(n, k, generator=g).to(torch.bfloat16)
    bias = torch.randn(n, generator=g)
    ref = a.float() @ b.float().t() + bias
    got = linear_tc(a.cuda(), b.cuda(), bias.cuda(), splits=splits).cpu()
    scale = ref.abs().max().item()
    assert torch.allclose(got, ref, rtol=1e-3, atol=1e-3 * scale), (got - ref).abs().max()


def test_gemm_deterministic_across_runs(cuda):
    g = torch.Generator().manual_seed(5)
    a = torch.randn(256, 2048, generator=g).to(torch.bfloat16).cuda()
    b = torch.randn(1000, 2048, generator=g).to(torch.bfloat16).cuda()
    r1 = linear_tc(a, b, splits=8)
    r2 = linear_tc(a, b, splits=8)
    assert torch.equal(r1, r2)


def test_large_ramp_head_end_to_end(cuda):
    g = torch.Generator().manual_seed(9)
    feat = torch.randn(64, 512, 7, 7, generator=g)
    w = torch.randn(1000, 512, generator=g) * 0.05
    head = LargeRampHead(w.cuda(), None, conf="entropy", site=15)
    pooled = pool_bf16(feat.cuda())
    assert torch.allclose(pooled.float().cpu(), feat.mean(dim=(2, 3)), rtol=1e-2, atol=1e-2)
    res = head(feat.cuda(), 0.9, want_logits=True)
    ref = H.ramp_head(pooled.float().cpu(), w.to(torch.bfloat16).float())
    assert torch.allclose(res.logits.cpu(), ref, rtol=1e-3, atol=1e-3 * ref.abs().max().item())
    err_ref, _ = H.confidence(res.logits.cpu(), "entropy")
    assert torch.allclose(res.err.cpu().double(), err_ref, atol=2e-5, rtol=0)


@pytest.mark.parametrize("b,c,h,w,dtype", [(256, 256, 56, 56, torch.bfloat16), (3, 2048, 7, 7, torch.bfloat16),
                                           (5, 68, 9, 11, torch.float32), (2, 1024, 14, 14, torch.float32)])
def test_pool_channels_last_matches_nchw(cuda, b, c, h, w, dtype):
    """channels_last maps are pooled in place (k_pool_nhwc, no NCHW copy): each
    mean within one bf16 rounding of the fp64 mean; the NCHW path agrees the same way."""
    g = torch.Generator(device="cuda").manual_seed(b + c + h)
    x = torch.randn(b, c, h, w, generator=g, device="cuda").to(dtype)
    xl = x.contiguous(memory_format=torch.channels_last)
    assert not xl.is_contiguous()
    ref = x.double().mean(dim=(2, 3))
    for got in (pool_bf16(xl), pool_bf16(x)):
        tol = ref.abs().to(torch.float64) * 2.0 ** -8 + 1e-6  # one bf16 ulp (8-bit mantissa)
        assert ((got.double() - ref).abs() <= tol).all(), (got.double() - ref).abs().max()


@pytest.mark.parametrize("m,n,k", [(32, 3072, 1024), (32, 50257, 1024), (160, 4096, 1024),
                                   (1000, 700, 136), (8192, 2304, 768), (8192, 768, 3072)])
def test_gemm_bf16_out_and_backbone_shapes(cuda, m, n, k):
    """Backbone / decode shapes (GPT-2-medium decode at batch 32 and 160, BERT
    encoder tiles), fp32 and bf16 outputs, against cuBLAS fp32 on the same
    bf16 operands."""
    torch = cuda
    from paper_2312_05385_b200.heads import linear_tc

    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    x = torch.randn(m, k, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    bias = torch.randn(n, generator=g, device="cuda")
    ref = torch.nn.functional.linear(x.float(), w.float(), bias)
    scale = ref.abs().max().item()
    got = linear_tc(x, w, bias)
    assert torch.allclose(got, ref, rtol=1e-3, atol=1e-3 * scale), (got - ref).abs().max()
    gb = linear_tc(x, w, bias, out_bf16=True)
    assert gb.dtype == torch.bfloat16
    assert torch.allclose(gb.float(), ref, rtol=1e-2, atol=1e-2 * scale)


# ---------------------------------------------------------------- csrc/gemm.cu paths
def _ref_act(y, act):
    F = torch.nn.functional
    if act == "gelu":
        return F.gelu(y)
    if act == "gelu_tanh":
        return F.gelu(y, approximate="tanh")
    if act == "relu":
        return F.relu(y)
    return y


# (path, m, n, k): 1 = swap-AB split-K (any m: z tiles of 128 rows), 2 / 4 / 3 =
# persistent CTA pair with 256 x 256 / 192 / 128 tiles. Ragged m, n, k at every
# tile edge; k spans one to many k-tiles; several persistent tiles per pair.
PATH_CASES = [
    (1, 1, 64, 64), (1, 32, 3072, 1024), (1, 33, 130, 200), (1, 100, 1000, 2048),
    (1, 300, 777, 520), (1, 256, 50257, 256), (1, 160, 3072, 1024), (1, 200, 1024, 4096),
    (2, 257, 256, 64), (2, 1000, 700, 136), (2, 8192, 2304, 768), (2, 2048, 4096, 4096),
    (4, 600, 776, 1000), (4, 8192, 768, 3072),
    (3, 777, 136, 72), (3, 4096, 1024, 512),
    (5, 5000, 64, 576), (5, 300, 40, 128), (5, 1000, 200, 64),  # 64-wide tiles (one-chunk epilogue)
]


# the pair kernel's TMA store needs 16-byte output rows (path 1 takes any shape)
PATH_CASES_DT = [(p, m, n, k, bf) for bf in (False, True) for (p, m, n, k) in PATH_CASES
                 if p == 1 or (n * (2 if bf else 4)) % 16 == 0]


@pytest.mark.parametrize("path,m,n,k,out_bf16", PATH_CASES_DT)
def test_gemm3_paths_match_torch(cuda, path, m, n, k, out_bf16):
    """Every kernel path against torch fp32 on the same bf16 operands: fp32 out
    within 1e-3 of the output scale (accumulation order only), bf16 out within
    one bf16 rounding (2^-8 relative) on top of that."""
    from paper_2312_05385_b200.heads import gemm

    g = torch.Generator(device="cuda").manual_seed(m * 31 + n * 7 + k + path)
    x = torch.randn(m, k, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, generator=g, device="cuda") / k ** 0.5).to(torch.bfloat16)
    bias = torch.randn(n, generator=g, device="cuda") * 0.1
    ref = torch.nn.functional.linear(x.float(), w.float(), bias)
    scale = ref.abs().max().item()
    got = gemm(x, w, bias, out_bf16=out_bf16, path=path)
    assert got.dtype == (torch.bfloat16 if out_bf16 else torch.float32)
    tol = 1e-3 * scale + (ref.abs() * 2.0 ** -8 if out_bf16 else 0)
    assert ((got.float() - ref).abs() <= tol).all(), (got.float() - ref).abs().max()


@pytest.mark.parametrize("act", ["gelu", "gelu_tanh", "relu"])
@pytest.mark.parametrize("path,m,n,k", [(1, 32, 4096, 1024), (2, 1024, 3072, 768), (3, 512, 512, 256)])
def test_gemm3_fused_activation(cuda, act, path, m, n, k):
    """bias + activation in the epilogue (fp32) == torch's activation of the fp32
    product, bf16 output within one rounding."""
    from paper_2312_05385_b200.heads import gemm

    g = torch.Generator(device="cuda").manual_seed(n + k)
    x = torch.randn(m, k, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, generator=g, device="cuda") / k ** 0.5).to(torch.bfloat16)
    bias = torch.randn(n, generator=g, device="cuda") * 0.1
    ref = _ref_act(torch.nn.functional.linear(x.float(), w.float(), bias), act)
    got = gemm(x, w, bias, act=act, path=path).float()
    tol = 1e-3 * ref.abs().max().item() + ref.abs() * 2.0 ** -8
    assert ((got - ref).abs() <= tol).all(), (got - ref).abs().max()


@pytest.mark.parametrize("path,m,n,k,splits", [(1, 64, 1024, 4096, 8), (1, 200, 3072, 1024, 0),
                                                 (2, 4096, 2304, 768, 0), (4, 8192, 768, 3072, 0)])
def test_gemm3_deterministic(cuda, path, m, n, k, splits):
    """Bit-identical across runs: split-K partials are reduced in rank order,
    the pair kernel has no cross-CTA reduction."""
    from paper_2312_05385_b200.heads import gemm

    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(m, k, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, generator=g, device="cuda") / k ** 0.5).to(torch.bfloat16)
    r1 = gemm(x, w, None, path=path, splits=splits, out_bf16=False)
    r2 = gemm(x, w, None, path=path, splits=splits, out_bf16=False)
    assert torch.equal(r1, r2)


def test_gemm3_leading_dims_and_errors(cuda):
    from paper_2312_05385_b200.errors import ParameterError
    from paper_2312_05385_b200.heads import gemm

    x = torch.randn(4, 16, 256, device="cuda").to(torch.bfloat16)
    w = torch.randn(512, 256, device="cuda").to(torch.bfloat16)
    y = gemm(x, w)
    assert y.shape == (4, 16, 512)
    ref = torch.nn.functional.linear(x.float(), w.float())
    assert torch.allclose(y.float(), ref, rtol=1e-2, atol=1e-2 * ref.abs().max().item())
    with pytest.raises(ParameterError):
        gemm(x, w[:, :128])
    with pytest.raises(ParameterError):
        gemm(x.float(), w)
    with pytest.raises(ParameterError):
        gemm(x, w, act="swish")


@pytest.mark.parametrize("path,m,n,k,splits", [(0, 4000, 256, 64, 0), (3, 1000, 512, 128, 0),
                                               (1, 100, 256, 512, 4), (1, 60, 1024, 256, 1)])
@pytest.mark.parametrize("act", [None, "relu"])
def test_gemm3_residual_epilogue(cuda, path, m, n, k, splits, act):
    """act(A W^T + bias + R): a bottleneck's conv3 + shortcut + ReLU in one
    kernel, on the pair kernel (TMA-store epilogue) and on the swap kernel
    (unsplit stores and the split-K reduction)."""
    from paper_2312_05385_b200.heads import gemm

    g = torch.Generator().manual_seed(m + n + k)
    a = torch.randn(m, k, generator=g).to(torch.bfloat16)
    w = torch.randn(n, k, generator=g).to(torch.bfloat16) * 0.1
    bias = torch.randn(n, generator=g)
    r = torch.randn(m, n, generator=g).to(torch.bfloat16)
    ref = a.float() @ w.float().t() + bias + r.float()
    ref = torch.relu(ref) if act == "relu" else ref
    got = gemm(a.cuda(), w.cuda(), bias.cuda(), act=act, path=path, splits=splits, res=r.cuda()).float().cpu()
    scale = ref.abs().max().item()
    assert (got - ref).abs().max().item() <= 8e-3 * scale
