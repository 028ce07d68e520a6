"""Ramp heads and the fused exit controller.

There is no reference code for these rows: eesim abstracts a ramp to an
(err, label) signal per input. The paper defines a ramp as
"a final fc layer, prepended with a lightweight pooling" and
an input exits at the first active ramp whose error score is strictly below
that ramp's threshold (engine.py:189-220). Here one launch does the pooling,
the FC, the softmax confidence (1 - max p, or normalised entropy), the
threshold compare, a stable compaction of the surviving rows and the scatter
of exiting rows' results to their request slots (ee_exit_controller). Large
heads (e.g. 1000 ImageNet classes) take their logits from a GEMM and run the
same epilogue (ee_exit_from_logits).

The parity oracle is a plain torch fp32 restatement (oracle/heads_ref.py).
"""

from __future__ import annotations

from dataclasses import dataclass

from paper_2312_05385_b200 import _native as nat
from paper_2312_05385_b200.errors import ParameterError

CONF = {"maxprob": 0, "entropy": 1}


@dataclass
class ExitResult:
    err: "object"     # f32 [B]
    label: "object"   # i32 [B]
    exits: "object"   # u8  [B]
    keep: "object"    # i32 [B], first n_keep entries are the surviving rows (ascending)
    n_keep: "object"  # i32 [1] (device)
    logits: "object" = None

    def survivors(self):
        return self.keep[: int(self.n_keep.item())]


@dataclass
class SlotTable:
    """Per-request results of exited rows, filled by the scatter."""

    label: "object"  # i32 [slots]
    err: "object"    # f32 [slots]
    site: "object"   # i32 [slots]; -1 = not released yet

    @classmethod
    def empty(cls, slots: int):
        torch = nat.torch_cuda()
        return cls(torch.full((slots,), -1, dtype=torch.int32, device="cuda"),
                   torch.full((slots,), float("nan"), dtype=torch.float32, device="cuda"),
                   torch.full((slots,), -1, dtype=torch.int32, device="cuda"))

    @classmethod
    def uninitialized(cls, slots: int):
        """For a caller that releases every slot exactly once (a feedback-mode
        batch: each row exits at a ramp or at the final model): no fill kernels."""
        torch = nat.torch_cuda()
        buf = torch.empty((3, slots), dtype=torch.int32, device="cuda")
        return cls(buf[0], buf[1].view(torch.float32), buf[2])


def _outputs(torch, b, k, want_logits, out_err=None, out_label=None, out_exits=None, compact=True):
    dev = "cuda"
    return (out_err if out_err is not None else torch.empty(b, dtype=torch.float32, device=dev),
            out_label if out_label is not None else torch.empty(b, dtype=torch.int32, device=dev),
            out_exits if out_exits is not None else torch.empty(b, dtype=torch.uint8, device=dev),
            torch.empty((b, k), dtype=torch.float32, device=dev) if want_logits else None,
            torch.empty(b, dtype=torch.int32, device=dev) if compact else None,
            torch.empty(1, dtype=torch.int32, device=dev) if compact else None)


def _check_aux(torch, b, alive, slot):
    if alive is not None and (alive.dtype != torch.uint8 or alive.numel() != b or not alive.is_cuda):
        raise ParameterError("alive must be a CUDA uint8 tensor with one byte per row")
    if slot is not None and (slot.dtype != torch.int32 or slot.numel() != b or not slot.is_cuda):
        raise ParameterError("slot must be a CUDA int32 tensor with one entry per row")


class ExitController:
    """One ramp: fused pool -> FC -> confidence -> compare -> compact -> scatter."""

    def __init__(self, weight, bias=None, *, conf: str = "maxprob", site: int = 0):
        torch = nat.torch_cuda()
        if conf not in CONF:
            raise ParameterError(f"conf must be one of {sorted(CONF)}")
        if weight.dim() != 2:
            raise ParameterError("weight must be [K, C]")
        if weight.dtype not in (torch.float32, torch.bfloat16):
            raise ParameterError("weight must be fp32 or bf16")
        self.weight = weight.detach().contiguous().cuda()
        self.bias = None if bias is None else bias.detach().float().contiguous().cuda()
        self.k, self.c = self.weight.shape
        self.conf = conf
        self.site = site

    def __call__(self, feat, threshold, *, alive=None, slot=None,
                 slots: SlotTable | None = None, want_logits: bool = False,
                 out_err=None, out_label=None, compact: bool = True) -> ExitResult:
        """feat: [B, C, H, W] / [B, C] (NCHW) or channels-last memory format; fp32 or bf16.
        `threshold` is a float or a one-element CUDA f64 tensor (graph-capture friendly);
        out_err / out_label let the caller supply the per-row output buffers.
        compact=False: no survivor list (feedback mode keeps every row)."""
        torch = nat.torch_cuda()
        if feat.dtype not in (torch.float32, torch.bfloat16) or not feat.is_cuda:
            raise ParameterError("feat must be a CUDA fp32 or bf16 tensor")
        b = feat.shape[0]
        if feat.dim() == 2:
            c, hw, nhwc = feat.shape[1], 1, 0
            feat = feat.contiguous()
        elif feat.dim() == 4:
            c, hw = feat.shape[1], feat.shape[2] * feat.shape[3]
            if feat.is_contiguous(memory_format=torch.channels_last) and not feat.is_contiguous():
                nhwc = 1
            else:
                feat, nhwc = feat.contiguous(), 0
        else:
            raise ParameterError("feat must be [B, C] or [B, C, H, W]")
        if c != self.c:
            raise ParameterError(f"feat has {c} channels, head expects {self.c}")
        _check_aux(torch, b, alive, slot)
        err, label, exits, logits, keep, n_keep = _outputs(torch, b, self.k, want_logits,
                                                           out_err, out_label, compact=compact)
        th_val, th_ptr = _threshold_args(torch, threshold)
        nat.check(nat.load_library().ee_exit_controller(
            nat.workspace(), feat.data_ptr(), int(feat.dtype == torch.bfloat16), b, c, hw, nhwc,
            self.weight.data_ptr(), int(self.weight.dtype == torch.bfloat16), nat.ptr(self.bias),
            self.k, CONF[self.conf], th_val, th_ptr, nat.ptr(alive), nat.ptr(slot), self.site,
            err.data_ptr(), label.data_ptr(), exits.data_ptr(), nat.ptr(logits),
            nat.ptr(keep), nat.ptr(n_keep),
            nat.ptr(slots.label if slots else None), nat.ptr(slots.err if slots else None),
            nat.ptr(slots.site if slots else None), nat.stream_handle(torch)))
        return ExitResult(err, label, exits, keep, n_keep, logits)


def _threshold_args(torch, threshold):
    """(scalar, device pointer): a CUDA f64 tensor is read by the kernel at run time."""
    if hasattr(threshold, "data_ptr"):
        if threshold.dtype != torch.float64 or not threshold.is_cuda or threshold.numel() != 1:
            raise ParameterError("device threshold must be a one-element CUDA float64 tensor")
        return 0.0, threshold.data_ptr()
    return float(threshold), None


def exit_from_logits(logits, threshold, *, conf: str = "maxprob", site: int = 0,
                     alive=None, slot=None, slots: SlotTable | None = None,
                     out_err=None, out_label=None, out_exits=None,
                     compact: bool = True) -> ExitResult:
    """Confidence + compare + compaction + scatter over precomputed fp32 logits [B, K]."""
    torch = nat.torch_cuda()
    if logits.dtype != torch.float32 or logits.dim() != 2 or not logits.is_cuda:
        raise ParameterError("logits must be a CUDA fp32 [B, K] tensor")
    logits = logits.contiguous()
    b, k = logits.shape
    _check_aux(torch, b, alive, slot)
    err, label, exits, _, keep, n_keep = _outputs(torch, b, k, False, out_err, out_label, out_exits,
                                                  compact=compact)
    th_val, th_ptr = _threshold_args(torch, threshold)
    nat.check(nat.load_library().ee_exit_from_logits(
        nat.workspace(), logits.data_ptr(), b, k, CONF[conf], th_val, th_ptr, nat.ptr(alive),
        nat.ptr(slot), site, err.data_ptr(), label.data_ptr(), exits.data_ptr(),
        nat.ptr(keep), nat.ptr(n_keep),
        nat.ptr(slots.label if slots else None), nat.ptr(slots.err if slots else None),
        nat.ptr(slots.site if slots else None), nat.stream_handle(torch)))
    return ExitResult(err, label, exits, keep, n_keep, None)


def _rows_dense(t) -> bool:
    """Each row t[i] is one contiguous block at stride numel / B (contiguous,
    or channels_last: the batch dimension is outermost in both)."""
    import torch

    return t.is_contiguous() or (t.dim() == 4 and t.is_contiguous(memory_format=torch.channels_last))


def compact_rows(src, keep, n_keep, out=None):
    """Gather the surviving rows of `src` ([B, ...], contiguous or channels_last)
    into a dense buffer of the same memory format (compaction mode: downstream
    blocks run only on these rows). Returns the full-capacity output (or `out`,
    whose capacity may exceed B); its first n_keep rows are valid."""
    torch = nat.torch_cuda()
    if not _rows_dense(src):
        src = src.contiguous()
    b = src.shape[0]
    row_bytes = src.numel() // max(b, 1) * src.element_size()
    if row_bytes % 16:
        raise ParameterError("row size must be a multiple of 16 bytes")
    if out is None:
        out = torch.empty_like(src)  # preserves channels_last
    elif (not _rows_dense(out) or out.dtype != src.dtype or out.shape[0] < b
          or out.numel() // max(out.shape[0], 1) * out.element_size() != row_bytes):
        raise ParameterError("out must be a dense row buffer of the same row size and dtype")
    nat.check(nat.load_library().ee_compact_rows(
        src.data_ptr(), row_bytes, keep.data_ptr(), n_keep.data_ptr(), b, out.data_ptr(),
        nat.stream_handle(torch)))
    return out


def compact_meta(keep, n_keep, rows_in, cap: int, dummy: int, rows_out, alive_out, n_out=None):
    """Bookkeeping of the next compacted stage, on the device: rows_out[i] =
    rows_in[keep[i]] for i < n_keep (dummy after), alive_out[i] = i < n_keep,
    n_out = n_keep (ee_compact_meta)."""
    torch = nat.torch_cuda()
    nat.check(nat.load_library().ee_compact_meta(
        keep.data_ptr(), n_keep.data_ptr(), nat.ptr(rows_in), int(cap), int(dummy),
        rows_out.data_ptr(), alive_out.data_ptr(), nat.ptr(n_out), nat.stream_handle(torch)))


def scatter_signals(err, label, rows, err_table, label_table):
    """err_table[rows[i]] = err[i], label_table[rows[i]] = label[i] (one launch:
    ee_scatter_signals; rows int32 request slots)."""
    torch = nat.torch_cuda()
    n = rows.numel()
    if err.dtype != torch.float32 or label.dtype != torch.int32 or rows.dtype != torch.int32:
        raise ParameterError("scatter_signals takes fp32 err, int32 label and int32 rows")
    if err.numel() < n or label.numel() < n:
        raise ParameterError("fewer signals than rows")
    nat.check(nat.load_library().ee_scatter_signals(
        err.data_ptr(), label.data_ptr(), rows.data_ptr(), n, err_table.data_ptr(), label_table.data_ptr(),
        nat.stream_handle(torch)))


def compact_fill(buf, keep, n_keep, rows: int, rows_in, dummy: int, rows_out, alive_out, n_out=None):
    """In-place compaction of buf's first `rows` rows ([B, ...], contiguous or
    channels_last) to the survivors `keep` lists: survivors below n_keep stay,
    the ones above move into the exited rows' places (ee_compact_fill), and
    rows_out / alive_out / n_out describe the new order like compact_meta."""
    torch = nat.torch_cuda()
    if not _rows_dense(buf):
        raise ParameterError("compact_fill needs a dense row layout")
    row_bytes = buf.numel() // max(buf.shape[0], 1) * buf.element_size()
    if rows_in is not None and rows_in.data_ptr() == rows_out.data_ptr():
        raise ParameterError("rows_out must not alias rows_in")
    nat.check(nat.load_library().ee_compact_fill(
        buf.data_ptr(), row_bytes, keep.data_ptr(), n_keep.data_ptr(), int(rows), nat.ptr(rows_in),
        int(dummy), rows_out.data_ptr(), alive_out.data_ptr(), nat.ptr(n_out), nat.stream_handle(torch)))


def linear_tc(x, weight, bias=None, *, splits: int = 0, out_bf16: bool = False):
    """[M, N] = x bf16 [M, K] @ weight bf16 [N, K]^T + bias, fp32 out by default
    (ramp-head logits): `gemm` with no activation."""
    return gemm(x, weight, bias, out_bf16=out_bf16, splits=splits)


ACTS = {None: 0, "none": 0, "gelu": 1, "gelu_tanh": 2, "relu": 3}


def gemm(x, weight, bias=None, *, act=None, out_bf16: bool = True, path: int = 0,
         splits: int = 0, out=None, res=None):
    """act(x bf16 [M, K] @ weight bf16 [N, K]^T + bias) on the tcgen05 kernels of
    csrc/gemm.cu (ee_gemm_bf16_ex): the persistent CTA-pair kernel for M > 256, the
    swap-AB weight-streaming kernel (cluster split-K) for M <= 256. `act` is fused
    into the epilogue ("gelu" = erf form, "gelu_tanh", "relu"), after adding the
    optional bf16 residual `res` ([M, N] like the output). x may have leading
    batch dimensions; they are flattened into M."""
    torch = nat.torch_cuda()
    if x.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise ParameterError("gemm takes bf16 operands")
    if act not in ACTS:
        raise ParameterError(f"unknown activation {act!r}")
    lead = x.shape[:-1]
    k = x.shape[-1]
    x2 = x.reshape(-1, k)
    if not x2.is_contiguous():
        x2 = x2.contiguous()
    weight = weight if weight.is_contiguous() else weight.contiguous()
    m, n = x2.shape[0], weight.shape[0]
    if weight.shape[1] != k:
        raise ParameterError("inner dimensions differ")
    if out is None:
        out = torch.empty((m, n), dtype=torch.bfloat16 if out_bf16 else torch.float32,
                          device=x.device)
    b = None
    if bias is not None:
        b = bias if bias.dtype == torch.float32 and bias.is_contiguous() else bias.float().contiguous()
    lib = nat.load_library()
    key = (m, n, k, splits, path, int(out_bf16))
    wb = _WORK_BYTES.get(key)
    if wb is None:
        wb = int(lib.ee_gemm_workspace_size(m, n, k, splits, path, int(out_bf16)))
        nat.check(min(wb, 0))
        _WORK_BYTES[key] = wb
    # split-K partials in torch's stream-ordered (and CUDA-graph-aware) allocator
    work = torch.empty(wb, dtype=torch.uint8, device=x.device) if wb else None
    r = None
    if res is not None:
        r = res.reshape(-1, n)
        if r.dtype != torch.bfloat16 or r.shape[0] != m or not r.is_contiguous():
            raise ParameterError("res must be a contiguous bf16 [M, N] tensor")
    nat.check(lib.ee_gemm_bf16_res(
        nat.workspace(), x2.data_ptr(), weight.data_ptr(), nat.ptr(b), nat.ptr(r), out.data_ptr(),
        int(out_bf16), ACTS[act], m, n, k, splits, path, nat.ptr(work), wb,
        nat.stream_handle(torch)))
    return out.view(*lead, n)


_WORK_BYTES: dict = {}


def pool_bf16(x):
    """Global average pool of an NCHW or channels_last fp32/bf16 map to a bf16 [B, C]
    GEMM operand."""
    torch = nat.torch_cuda()
    if x.dtype not in (torch.float32, torch.bfloat16) or x.dim() != 4:
        raise ParameterError("pool_bf16 takes an fp32 or bf16 [B, C, H, W] tensor")
    b, c, h, w = x.shape
    out = torch.empty((b, c), dtype=torch.bfloat16, device="cuda")
    if (x.is_contiguous(memory_format=torch.channels_last) and not x.is_contiguous()
            and c % 4 == 0 and b <= 65535):
        # channels_last map: pooled in place, no NCHW copy
        nat.check(nat.load_library().ee_pool_nhwc_bf16(
            x.data_ptr(), int(x.dtype == torch.bfloat16), b, c, h * w, out.data_ptr(),
            nat.stream_handle(torch)))
        return out
    x = x.contiguous()
    nat.check(nat.load_library().ee_pool_bf16(x.data_ptr(), int(x.dtype == torch.bfloat16), b, c,
                                              h * w, out.data_ptr(), nat.stream_handle(torch)))
    return out


class LargeRampHead:
    """Ramp with a wide classifier (e.g. 1000 ImageNet classes): pool -> bf16
    tensor-core GEMM -> fused confidence / compare / compaction / scatter."""

    def __init__(self, weight, bias=None, *, conf: str = "maxprob", site: int = 0):
        torch = nat.torch_cuda()
        self.weight = weight.detach().to(torch.bfloat16).contiguous().cuda()
        self.bias = None if bias is None else bias.detach().float().contiguous().cuda()
        self.conf = conf
        self.site = site

    def __call__(self, feat, threshold, *, alive=None, slot=None,
                 slots: SlotTable | None = None, want_logits: bool = False,
                 out_err=None, out_label=None, compact: bool = True) -> ExitResult:
        torch = nat.torch_cuda()
        x = pool_bf16(feat) if feat.dim() == 4 else feat.to(torch.bfloat16)
        logits = linear_tc(x, self.weight, self.bias)
        res = exit_from_logits(logits, threshold, conf=self.conf, site=self.site, alive=alive,
                               slot=slot, slots=slots, out_err=out_err, out_label=out_label,
                               compact=compact)
        if want_logits:
            res.logits = logits
        return res
