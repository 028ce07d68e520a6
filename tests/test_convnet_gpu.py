"""ResNet blocks on the repo's kernels (convnet.py, A14): every routed
convolution against a torch fp32 convolution of the same bf16 operands, and
whole routed backbones against the library path and an fp32 model.

Tolerances (bf16 serving form): a routed convolution's output rounds once to
bf16 from an fp32 accumulation, so it must match the fp32 reference within
bf16 resolution (rel 1e-2 of the output scale); whole backbones accumulate one
bf16 rounding per layer, so the routed and the library bf16 networks must each
stay within 5e-2 (relative to the logit scale) of the fp32 network and agree
on the argmax wherever the fp32 top-2 margin exceeds that bound."""

from __future__ import annotations

import copy

import pytest
import torch
import torch.nn.functional as F

from paper_2312_05385_b200 import convnet, ee_infer

pytestmark = pytest.mark.gpu
CL = torch.channels_last


def _bf(x):
    return x.to(torch.bfloat16).contiguous(memory_format=CL)


def _ref_conv(x, conv, act, res):
    y = F.conv2d(x.float(), conv.weight.float(), conv.bias.float(), conv.stride, conv.padding)
    if res is not None:
        y = y + res.float()
    return torch.relu(y) if act == "relu" else y


@pytest.mark.parametrize("k,stride,cin,cout,hw,b", [
    (1, 1, 64, 256, 56, 8),     # bottleneck conv3 shape (GEMM, pair kernel)
    (1, 1, 256, 64, 56, 8),     # bottleneck conv1
    (1, 2, 256, 512, 56, 4),    # strided downsample (gathered pixels + GEMM)
    (1, 1, 2048, 512, 7, 2),    # M = 98 <= 256: the swap-AB kernel
    (3, 1, 64, 64, 32, 8),      # spatial: implicit GEMM (TMA im2col), ResNet-18 CIFAR
    (3, 2, 128, 128, 28, 4),    # strided spatial
    (3, 1, 256, 256, 14, 3),    # ragged M (3 x 14 x 14 = 588 rows)
    (3, 1, 512, 512, 7, 5),     # layer4: 7x7 maps, tiles straddle images
    (3, 2, 64, 128, 32, 2),     # CIFAR downsampling block
    (1, 2, 64, 128, 32, 2),     # its strided 1x1 shortcut (implicit GEMM, traversal stride 2)
    (3, 1, 512, 512, 4, 32),    # CIFAR layer4 at B=32: 8 tiles over K=4608 -> split-K + epilogue pass
    (3, 1, 256, 256, 8, 32),    # CIFAR layer3: split-K
    (3, 2, 256, 512, 8, 3),     # tiny M, strided, split-K with a ragged last tile
    (7, 2, 3, 64, 224, 2),      # the ImageNet stem: explicit im2col (K 147 -> 192) + GEMM
    (3, 1, 3, 64, 32, 4),       # the CIFAR stem
    (3, 1, 24, 40, 15, 3),      # odd channels: im2col K 216 -> 256, ragged M
])
@pytest.mark.parametrize("act,with_res", [(None, False), ("relu", False), ("relu", True)])
def test_routed_conv_matches_fp32(cuda, k, stride, cin, cout, hw, b, act, with_res):
    g = torch.Generator(device="cuda").manual_seed(k * 100 + stride * 10 + cin % 7)
    conv = torch.nn.Conv2d(cin, cout, k, stride, k // 2, bias=True).cuda()
    with torch.no_grad():
        conv.weight.normal_(0, (2.0 / (cin * k * k)) ** 0.5, generator=g)
        conv.bias.normal_(0, 0.1, generator=g)
    conv = conv.to(torch.bfloat16).to(memory_format=CL)
    x = _bf(torch.randn(b, cin, hw, hw, generator=g, device="cuda"))
    ho = (hw + 2 * (k // 2) - k) // stride + 1
    res = _bf(torch.randn(b, cout, ho, ho, generator=g, device="cuda")) if with_res else None
    y = convnet.Conv(conv)(x, act=act, res=res)
    assert y.shape == (b, cout, ho, ho) and y.is_contiguous(memory_format=CL)
    ref = _ref_conv(x, conv, act, res)
    scale = ref.abs().max().item()
    err = (y.float() - ref).abs().max().item()
    assert err <= 1e-2 * scale, (err, scale)


@pytest.mark.parametrize("b,c,hw,k,stride,pad", [(2, 64, 112, 3, 2, 1), (3, 24, 17, 3, 2, 1), (1, 8, 9, 2, 2, 0),
                                               (2, 16, 10, 3, 1, 1), (1, 8, 7, 3, 2, 0)])
def test_maxpool_nhwc_matches_torch(cuda, b, c, hw, k, stride, pad):
    g = torch.Generator(device="cuda").manual_seed(c + hw)
    x = _bf(torch.randn(b, c, hw, hw, generator=g, device="cuda"))
    y = convnet.maxpool(x, k, stride, pad)
    assert torch.equal(y, F.max_pool2d(x, k, stride, pad))  # maxima of bf16 values: exact


def test_bias_act_one_pass(cuda):
    g = torch.Generator(device="cuda").manual_seed(1)
    x = _bf(torch.randn(4, 64, 9, 9, generator=g, device="cuda"))
    r = _bf(torch.randn(4, 64, 9, 9, generator=g, device="cuda"))
    bias = torch.randn(64, generator=g, device="cuda")
    y = convnet.bias_act(x, bias, "relu", r)
    ref = torch.relu(x.float() + bias.view(1, -1, 1, 1) + r.float())
    assert torch.allclose(y.float(), ref, rtol=8e-3, atol=1e-2)
    y0 = convnet.bias_act(x, None, None, None)
    assert torch.equal(y0, x)


@pytest.mark.parametrize("which", ["resnet50", "resnet18"])
def test_routed_backbone_vs_library_and_fp32(cuda, which):
    torch.backends.cudnn.allow_tf32 = False
    if which == "resnet50":
        pipe, m = ee_infer.resnet50_imagenet()
        shape, b = (3, 224, 224), 16
    else:
        pipe, m = ee_infer.resnet18_cifar()
        shape, b = (3, 32, 32), 64
    m32 = copy.deepcopy(m).eval()
    lib = copy.deepcopy(m)
    ee_infer.prepare_bf16(lib, channels_last=True, route=False)
    ee_infer.prepare_bf16(m, channels_last=True)  # routed: the pipeline's own modules
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(b, *shape, generator=g, device="cuda")
    with torch.no_grad():
        ref = m32(x).float()
        routed = pipe.stages[-1](_run_stages(pipe, _bf(x))).float()
        library = lib(_bf(x)).float()
    scale = ref.abs().max().item()
    for name, y in (("routed", routed), ("library", library)):
        err = (y - ref).abs().max().item()
        assert err <= 5e-2 * scale, (name, err, scale)
    top2 = ref.topk(2, dim=1).values
    clear = (top2[:, 0] - top2[:, 1]) > 0.1 * scale
    assert torch.equal(routed.argmax(1)[clear], ref.argmax(1)[clear])


def _run_stages(pipe, x):
    h = x
    for st in pipe.stages[:-1]:
        h = st(h)
    return h
