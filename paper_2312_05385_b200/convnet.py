"""ResNet blocks on the repo's own kernels (north star (1)).

Serving form: bf16, channels_last (NHWC), BatchNorm folded into the
convolutions (ee_infer.fold_batchnorm). An NHWC activation [B, C, H, W] is a
row-major [B*H*W, C] matrix, so

  * a 1x1 stride-1 convolution IS a GEMM against the [C_out, C_in] weight: it
    runs on the tcgen05 kernels of csrc/gemm.cu with the folded BN bias, the
    ReLU and, for a bottleneck's last convolution, the shortcut add fused into
    the epilogue (ee_gemm_bf16_res) — one kernel where the library path runs a
    convolution, a broadcast bias add, a clamp and an add;
  * a spatial convolution (3x3, any stride) and a strided 1x1 shortcut run as
    an implicit GEMM on the same tcgen05 pair kernel (ee_conv_bf16): the A
    operand is never materialised, every k-tile is one TMA im2col load of 128
    consecutive output pixels x 64 input channels for one filter tap (zero
    padding done by the TMA unit), with the same fused epilogue;
  * a convolution whose input channels are not a multiple of 64 (the
    3-channel stem) gets its A operand written out once (ee_im2col_bf16, K
    padded to a multiple of 8) and runs on the same GEMM with the same
    epilogue; the stem's max pool is one NHWC pass (ee_maxpool_nhwc_bf16);
  * anything else (output channels not a multiple of 8) stays on cuDNN without
    a bias and takes bias / ReLU / shortcut in ONE fused NHWC pass
    (ee_bias_act_bf16);
  * the classifier (global average pool + fc): for up to 256 classes ONE
    kernel, the fused ramp head (k_exit_fused: pool in fp32, fp32 FC over the
    bf16 weight) asked for its logits only; wider heads pool with
    k_pool_nhwc and run the fc on the tcgen05 GEMM. Logits are fp32.

route_resnet() rebinds the forward of every block of a prepared torchvision
ResNet in place, so an EEPipeline built on the model's modules picks it up.
Numerics: bf16 operands, fp32 accumulation and epilogue, one bf16 rounding per
convolution output (the library path rounds after the conv, after the bias and
after the add).
"""

from __future__ import annotations

from paper_2312_05385_b200 import _native as nat
from paper_2312_05385_b200.errors import ParameterError
from paper_2312_05385_b200.heads import ExitController, gemm, pool_bf16

ACT = {None: 0, "relu": 3}
_CONV_WORK: dict = {}  # conv shape -> ee_conv_workspace_size


def _rows(x):
    """NHWC view [B*H*W, C] of a channels_last [B, C, H, W] tensor (no copy)."""
    import torch

    if not x.is_contiguous(memory_format=torch.channels_last):
        x = x.contiguous(memory_format=torch.channels_last)
    b, c, h, w = x.shape
    return x.permute(0, 2, 3, 1).reshape(b * h * w, c), (b, c, h, w)


def _unrows(y, b, h, w):
    """[B*H*W, C] rows back to a channels_last [B, C, H, W] view."""
    return y.view(b, h, w, y.shape[1]).permute(0, 3, 1, 2)


def bias_act(x, bias, act=None, res=None, out=None):
    """act(x + bias (+ res)) over a channels_last bf16 map in one pass."""
    torch = nat.torch_cuda()
    xr, (b, c, h, w) = _rows(x)
    rr = _rows(res)[0] if res is not None else None
    y = torch.empty_like(xr) if out is None else out
    nat.check(nat.load_library().ee_bias_act_bf16(
        xr.data_ptr(), nat.ptr(bias), nat.ptr(rr), ACT[act], xr.shape[0], c, y.data_ptr(),
        nat.stream_handle(torch)))
    return _unrows(y, b, h, w)


class Conv:
    """One folded convolution (weight bf16, bias fp32) with its epilogue."""

    def __init__(self, conv):
        import torch

        if conv.groups != 1 or conv.dilation != (1, 1):
            raise ParameterError("grouped / dilated convolutions are not routed")
        self.conv = conv
        w = conv.weight.detach()
        self.k = w.shape[2:]
        self.stride = conv.stride
        self.padding = conv.padding
        self.bias = (conv.bias.detach().float().contiguous() if conv.bias is not None
                     else torch.zeros(w.shape[0], dtype=torch.float32, device=w.device))
        self.pointwise = tuple(self.k) == (1, 1) and tuple(self.padding) == (0, 0)
        self.w2d = w.reshape(w.shape[0], -1).contiguous() if self.pointwise else None
        self.w = w.contiguous(memory_format=torch.channels_last)

    def __call__(self, x, act=None, res=None, out=None):
        """`out`: optional channels_last bf16 [B, C_out, H_out, W_out] the result is
        written into (the GEMM paths; e.g. a compacted batch's next input buffer)."""
        import torch
        import torch.nn.functional as F

        cin, cout = x.shape[1], self.w.shape[0]
        if cin % 64 == 0 and cout % 8 == 0 and not (self.pointwise and self.stride == (1, 1)):
            return self._implicit_gemm(x, act, res, out)
        if out is None and cout % 8 == 0 and not self.pointwise and (x.shape[3] * cin) % 8 == 0:
            return self._explicit_im2col(x, act, res)
        if self.pointwise and x.shape[1] % 8 == 0:
            if self.stride != (1, 1):
                x = x[:, :, :: self.stride[0], :: self.stride[1]].contiguous(
                    memory_format=torch.channels_last)
            a, (b, _, h, w) = _rows(x)
            r = _rows(res)[0] if res is not None else None
            o = None
            if out is not None:
                if not out.is_contiguous(memory_format=torch.channels_last):
                    raise ParameterError("out must be channels_last")
                o = out.permute(0, 2, 3, 1).reshape(b * h * w, cout)  # a view: dense NHWC rows
            y = gemm(a, self.w2d, self.bias, act=act, res=r, out=o)
            return _unrows(y, b, h, w)
        if out is not None:
            raise ParameterError("this convolution has no direct-output path")
        y = F.conv2d(x, self.w, None, self.stride, self.padding)
        if y.shape[1] % 8:
            y = y + self.bias.to(y.dtype).view(1, -1, 1, 1)
            if res is not None:
                y = y + res
            return torch.relu(y) if act == "relu" else y
        return bias_act(y, self.bias, act, res, out=None)


    def _implicit_gemm(self, x, act, res, out=None):
        torch = nat.torch_cuda()
        if not x.is_contiguous(memory_format=torch.channels_last):
            x = x.contiguous(memory_format=torch.channels_last)
        b, c, h, w = x.shape
        kh, kw = self.k
        (sh, sw), (ph, pw) = self.stride, self.padding
        if sh != sw or ph != pw:
            raise ParameterError("square strides and paddings only")
        ho, wo = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
        cout = self.w.shape[0]
        if out is not None:
            if tuple(out.shape) != (b, cout, ho, wo) or not out.is_contiguous(memory_format=torch.channels_last):
                raise ParameterError("out must be a channels_last [B, C_out, H_out, W_out] map")
            y = out.permute(0, 2, 3, 1)
        else:
            y = torch.empty((b, ho, wo, cout), dtype=torch.bfloat16, device=x.device)
        r = None
        if res is not None:
            r = res if res.is_contiguous(memory_format=torch.channels_last) else \
                res.contiguous(memory_format=torch.channels_last)
        lib = nat.load_library()
        key = (b, h, w, c, cout, kh, kw, sh, ph)
        wb = _CONV_WORK.get(key)
        if wb is None:
            wb = int(lib.ee_conv_workspace_size(*key))
            nat.check(min(wb, 0))
            _CONV_WORK[key] = wb
        # split-K partials in torch's stream-ordered (CUDA-graph-aware) allocator
        work = torch.empty(wb, dtype=torch.uint8, device=x.device) if wb else None
        nat.check(lib.ee_conv_bf16(
            nat.workspace(), x.data_ptr(), b, h, w, c, self.w.data_ptr(), cout, kh, kw, sh, ph,
            self.bias.data_ptr(), nat.ptr(r), ACT[act], y.data_ptr(), nat.ptr(work), wb,
            nat.stream_handle(torch)))
        return y.permute(0, 3, 1, 2)


    def _explicit_im2col(self, x, act, res):
        torch = nat.torch_cuda()
        if not x.is_contiguous(memory_format=torch.channels_last):
            x = x.contiguous(memory_format=torch.channels_last)
        b, c, h, w = x.shape
        kh, kw = self.k
        (sh, sw), (ph, pw) = self.stride, self.padding
        if sh != sw or ph != pw:
            raise ParameterError("square strides and paddings only")
        seg = (kw * c + 7) // 8 * 8  # filter row r owns columns [r seg, r seg + kw c)
        kp = kh * seg  # a multiple of 8: the GEMM's last k-tile is zero-filled by TMA
        if getattr(self, "w_cols", None) is None or self.w_cols.shape[1] != kp:
            cout = self.w.shape[0]
            wc = torch.zeros((cout, kh, seg), dtype=torch.bfloat16, device=x.device)
            wc[:, :, : kw * c] = self.w.permute(0, 2, 3, 1).reshape(cout, kh, kw * c)
            self.w_cols = torch.nn.functional.pad(wc.reshape(cout, kh * seg), (0, kp - kh * seg)).contiguous()
        ho, wo = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
        a = torch.empty((b * ho * wo, kp), dtype=torch.bfloat16, device=x.device)
        nat.check(nat.load_library().ee_im2col_bf16(
            x.data_ptr(), b, h, w, c, kh, kw, sh, ph, kp, a.data_ptr(), nat.stream_handle(torch)))
        r = _rows(res)[0] if res is not None else None
        return _unrows(gemm(a, self.w_cols, self.bias, act=act, res=r), b, ho, wo)


def maxpool(x, k: int, stride: int, pad: int):
    """k x k max pooling of a channels_last bf16 map in one NHWC pass."""
    torch = nat.torch_cuda()
    if not x.is_contiguous(memory_format=torch.channels_last):
        x = x.contiguous(memory_format=torch.channels_last)
    b, c, h, w = x.shape
    ho, wo = (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1
    y = torch.empty((b, ho, wo, c), dtype=x.dtype, device=x.device)
    nat.check(nat.load_library().ee_maxpool_nhwc_bf16(
        x.data_ptr(), b, h, w, c, k, stride, pad, y.data_ptr(), nat.stream_handle(torch)))
    return y.permute(0, 3, 1, 2)


class BottleneckTC:
    """torchvision Bottleneck (BN folded): 1x1 -> 3x3 -> 1x1 + shortcut, ReLUs."""

    def __init__(self, blk):
        self.c1, self.c2, self.c3 = Conv(blk.conv1), Conv(blk.conv2), Conv(blk.conv3)
        self.ds = Conv(blk.downsample[0]) if blk.downsample is not None else None

    def __call__(self, x, out=None):
        y = self.c1(x, act="relu")
        y = self.c2(y, act="relu")
        idt = self.ds(x) if self.ds is not None else x
        return self.c3(y, act="relu", res=idt, out=out)


class BasicBlockTC:
    """torchvision BasicBlock (BN folded): 3x3 -> 3x3 + shortcut, ReLUs."""

    def __init__(self, blk):
        self.c1, self.c2 = Conv(blk.conv1), Conv(blk.conv2)
        self.ds = Conv(blk.downsample[0]) if blk.downsample is not None else None

    def __call__(self, x, out=None):
        y = self.c1(x, act="relu")
        idt = self.ds(x) if self.ds is not None else x
        return self.c2(y, act="relu", res=idt, out=out)


def run_into(stage, x, out):
    """stage(x) with its result written into `out` when the stage ends in a
    routed residual block (else None: the caller falls back to a copy)."""
    import torch

    if isinstance(stage, torch.nn.Sequential) and len(stage):
        last = stage[len(stage) - 1]
        if not isinstance(getattr(last, "forward", None), (BottleneckTC, BasicBlockTC)):
            return None
        for j in range(len(stage) - 1):
            x = stage[j](x)
        stage = last
    fwd = getattr(stage, "forward", None)
    if not isinstance(fwd, (BottleneckTC, BasicBlockTC)):
        return None
    return fwd(x, out=out)


def can_run_into(stage) -> bool:
    import torch

    if isinstance(stage, torch.nn.Sequential) and len(stage):
        stage = stage[len(stage) - 1]
    return isinstance(getattr(stage, "forward", None), (BottleneckTC, BasicBlockTC))


def route_resnet(model):
    """Rebind the forward of every residual block and the stem convolution of a
    folded bf16 channels_last torchvision ResNet to the repo's kernels (in
    place). The stem's ReLU moves into the convolution's epilogue."""
    import torch
    import torchvision

    for layer in (model.layer1, model.layer2, model.layer3, model.layer4):
        for blk in layer:
            if isinstance(blk, torchvision.models.resnet.Bottleneck):
                blk.forward = BottleneckTC(blk)
            else:
                blk.forward = BasicBlockTC(blk)
    route_classifier(model)
    stem = Conv(model.conv1)
    model.conv1.forward = lambda x: stem(x, act="relu")
    model.relu.forward = lambda x: x  # applied by the stem's epilogue (blocks use their own)
    mp = model.maxpool
    if isinstance(mp, torch.nn.MaxPool2d) and not mp.ceil_mode and mp.dilation in (1, (1, 1)):
        k = mp.kernel_size if isinstance(mp.kernel_size, int) else mp.kernel_size[0]
        st = mp.stride if isinstance(mp.stride, int) else mp.stride[0]
        pd = mp.padding if isinstance(mp.padding, int) else mp.padding[0]
        mp.forward = lambda x: maxpool(x, k, st, pd) if x.dtype == torch.bfloat16 and x.shape[1] % 8 == 0 \
            else torch.nn.functional.max_pool2d(x, k, st, pd)
    return model


class ClassifierTC:
    """avgpool + flatten + fc of a ResNet on the repo's kernels (bound to the
    avgpool module; the fc module becomes the identity). A map that is not
    channels_last bf16 keeps the library path."""

    def __init__(self, model):
        import torch

        fc = model.fc
        self.fc = fc
        self.w = fc.weight.detach().to(torch.bfloat16).contiguous()
        self.b = None if fc.bias is None else fc.bias.detach().float().contiguous()
        self.fused = ExitController(self.w, self.b) if fc.out_features <= 256 else None
        self.pool = model.avgpool.__class__.forward.__get__(model.avgpool)

    def __call__(self, x):
        import torch

        if not (x.dim() == 4 and x.dtype == torch.bfloat16 and x.shape[1] % 8 == 0
                and x.is_contiguous(memory_format=torch.channels_last)):
            return self.fc.__class__.forward(self.fc, torch.flatten(self.pool(x), 1))
        if self.fused is not None:  # pool + FC in one kernel; nobody "exits" (err < -1 never holds)
            return self.fused(x, -1.0, want_logits=True, compact=False).logits
        return gemm(pool_bf16(x), self.w, self.b, out_bf16=False)


def route_classifier(model):
    """Rebind a ResNet's avgpool to ClassifierTC (returns logits [B, classes]) and
    its fc to the identity: both the model's own forward (avgpool -> flatten ->
    fc) and an EEPipeline's final Sequential(avgpool, Flatten, fc) then run it."""
    if model.fc.in_features == model.fc.out_features:
        return None  # the fc could not tell logits from features: keep the library path
    head = ClassifierTC(model)
    model.avgpool.forward = head
    model.fc.forward = lambda x: x if x.dim() == 2 and x.shape[1] == head.fc.out_features \
        else head.fc.__class__.forward(head.fc, x)
    return head
