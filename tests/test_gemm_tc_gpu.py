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
