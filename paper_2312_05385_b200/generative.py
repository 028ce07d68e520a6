"""Token-level early exit for generative decoding on the GPU (BASELINE config 5,
SURVEY §8a row A15; north star: "GPT-2-medium-shape decoder token-level early
exit with KV-cache fill for skipped layers, batch 32 decode, time-per-token").

The reference models this as a latency timeline (pkg/src/eesim/generative.py,
_SequenceSim at 170-273). Here the same schedule runs for real on a
GPT-2-medium-shape decoder (random init, bf16):

  * every decode step runs the prefix layers [0, L) for all B sequences, then
    the ramp: the model's own final LayerNorm + LM head on the layer-L hidden
    state ("GPT-2: final LN + LM head") as a 5th-gen
    tensor-core GEMM (ee_gemm_bf16_tn) followed by the fused confidence +
    strict-compare epilogue (ee_exit_from_logits; engine.py:207's rule);
  * a token that exits releases the ramp's argmax at once; its suffix layers
    [L, N) are deferred: its layer-L hidden state is parked per sequence
    (generative.py:217-218);
  * the next token of that sequence that does not exit carries every deferred
    suffix with it (generative.py:230-259): one suffix pass over the chunk
    [deferred..., current] fills the KV cache of the skipped layers for the
    deferred positions and computes the current token's output;
  * a sequence that parks flush_cap suffixes flushes them at once ("cap",
    generative.py:219-220), and the end of decoding flushes the rest ("end").

So the KV cache of every layer ends up exactly as full decoding would leave it
(inputs always run to completion), and every token — exited or
not — also gets the original model's output, which is the feedback the
reference's tuner consumes (token_feedback, generative.py:284-306).

Both passes run at fixed shapes (B x 1 prefix tokens, B x (flush_cap + 1)
suffix chunk slots with masks) and are captured as CUDA graphs; decode at
batch 32 is weight-bandwidth bound, so the padded suffix slots cost little.
The schedule itself (who parks, who carries, cap flushes, the next input
token) runs on the device between the two passes (ee_defer_plan /
ee_defer_finish), so the host enqueues every step without waiting on the GPU
and reads the token / flush histories once at the end (use_graphs=False keeps
the host-driven loop, eager, as the cross-check). Per-token release latency
(time-per-token) is measured with CUDA events: ramp release for exits, suffix
+ head for the rest.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from paper_2312_05385_b200 import _native as nat
from paper_2312_05385_b200.errors import ParameterError
from paper_2312_05385_b200.heads import exit_from_logits, gemm, linear_tc


@dataclass(frozen=True)
class GPT2Spec:
    n_layer: int = 24   # GPT-2-medium
    d_model: int = 1024
    n_head: int = 16
    vocab: int = 50257
    n_pos: int = 1024

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_head


class GPT2Decoder:
    """GPT-2-shape decoder weights (random init, GPT-2 init scheme) and a static
    KV cache [layer][B, H, T + 1, Dh] (slot T is a write sink for padding)."""

    def __init__(self, spec: GPT2Spec = GPT2Spec(), *, batch: int, max_tokens: int, seed: int = 0):
        torch = nat.torch_cuda()
        self.torch = torch
        self.spec = spec
        self.B = batch
        self.T = max_tokens
        if max_tokens > spec.n_pos:
            raise ParameterError(f"max_tokens {max_tokens} exceeds n_pos {spec.n_pos}")
        g = torch.Generator(device="cuda").manual_seed(seed)
        d, bf = spec.d_model, torch.bfloat16

        def normal(*shape, std=0.02):
            return (torch.randn(*shape, generator=g, device="cuda") * std).to(bf)

        self.wte = normal(spec.vocab, d)
        self.wpe = normal(spec.n_pos, d, std=0.01)
        proj_std = 0.02 / math.sqrt(2 * spec.n_layer)
        self.layers = []
        for _ in range(spec.n_layer):
            self.layers.append({
                "ln1_w": torch.ones(d, device="cuda", dtype=bf), "ln1_b": torch.zeros(d, device="cuda", dtype=bf),
                "qkv_w": normal(3 * d, d), "qkv_b": torch.zeros(3 * d, device="cuda", dtype=bf),
                "o_w": normal(d, d, std=proj_std), "o_b": torch.zeros(d, device="cuda", dtype=bf),
                "ln2_w": torch.ones(d, device="cuda", dtype=bf), "ln2_b": torch.zeros(d, device="cuda", dtype=bf),
                "fc_w": normal(4 * d, d), "fc_b": torch.zeros(4 * d, device="cuda", dtype=bf),
                "pr_w": normal(d, 4 * d, std=proj_std), "pr_b": torch.zeros(d, device="cuda", dtype=bf),
            })
        for w in self.layers:  # fp32 bias copies: the GEMM epilogues add them in fp32
            for k in ("qkv", "o", "fc", "pr"):
                w[k + "_b32"] = w[k + "_b"].float()
        self.lnf_w = torch.ones(d, device="cuda", dtype=bf)
        self.lnf_b = torch.zeros(d, device="cuda", dtype=bf)
        H, Dh = spec.n_head, spec.head_dim
        # K and V of a layer in one tensor [2, B, H, T+1, Dh]: one scatter writes both
        self.kv_cache = [torch.zeros(2, batch, H, max_tokens + 1, Dh, device="cuda", dtype=bf)
                         for _ in range(spec.n_layer)]
        self.k_cache = [kv[0] for kv in self.kv_cache]
        self.v_cache = [kv[1] for kv in self.kv_cache]
        self.rows = torch.arange(batch, device="cuda")
        self.key_idx = torch.arange(max_tokens + 1, device="cuda")

    # ---- one pass over layers [l0, l1) for a [B, q, d] chunk at absolute positions
    def layers_forward(self, h, pos, l0: int, l1: int):
        """h bf16 [B, q, d]; pos i64 [B, q] (-1 = padding: no KV write, output unused).
        Appends K/V at `pos` in layers [l0, l1) and attends causally over the cache."""
        torch = self.torch
        F = torch.nn.functional
        B, q, d = h.shape
        H, Dh, T = self.spec.n_head, self.spec.head_dim, self.T
        valid = pos >= 0
        wpos = torch.where(valid, pos, torch.full_like(pos, T))  # padding -> sink slot T
        # every layer appends K/V of token (b, i) at slot wpos[b, i] (ee_kv_append_bf16)
        wpos = wpos.to(torch.int64).contiguous()
        lib = nat.load_library()
        st = nat.stream_handle(torch)
        # key j visible to query (b, i) iff j <= pos[b, i]; padding queries see key 0 only
        qpos = torch.where(valid, pos, torch.zeros_like(pos))
        # short passes (decode, flushes: q <= 8 tokens) attend with the length-aware
        # kernel (ee_decode_attention_bf16), which reads only keys 0 .. qpos; longer
        # chunks use SDPA with an additive bf16 mask built once per pass
        short = q <= 8 and Dh == 64 and q * (T + 1) <= 51200
        qpos_c = qpos.to(torch.int64).contiguous()
        if not short:
            vis = (self.key_idx[None, None, :] <= qpos[:, :, None]) & (self.key_idx[None, None, :] < T)
            mask = torch.zeros(vis.shape, dtype=h.dtype, device=h.device).masked_fill_(
                ~vis, float("-inf"))[:, None, :, :]
        if l1 <= l0:
            return h
        # the residual stream is owned here and updated in place by the fused
        # add + LayerNorm kernel (ee_add_layernorm_bf16): h += y; x = LN(h)
        h = h.contiguous().clone()
        x = torch.empty_like(h)

        def add_ln(y, gamma, beta):
            nat.check(lib.ee_add_layernorm_bf16(h.data_ptr(), None if y is None else y.data_ptr(),
                                                gamma.data_ptr(), beta.data_ptr(), 1e-5, B * q, d,
                                                x.data_ptr(), st))

        add_ln(None, self.layers[l0]["ln1_w"], self.layers[l0]["ln1_b"])
        for l in range(l0, l1):
            w = self.layers[l]
            # projections: tcgen05 GEMMs (csrc/gemm.cu): the swap-AB weight-streaming
            # kernel for decode / flush passes, the CTA-pair kernel for prompts
            qkv = gemm(x, w["qkv_w"], w["qkv_b32"])  # [B, q, 3d] contiguous
            # K and V rows straight from the projection into their cache slots (one kernel)
            nat.check(lib.ee_kv_append_bf16(qkv.data_ptr(), wpos.data_ptr(), B, q, H, Dh, T + 1,
                                            self.kv_cache[l].data_ptr(), st))
            if short:  # decode / flush passes: length-aware kernel, output already [B, q, d]
                att = torch.empty(B, q, d, dtype=h.dtype, device=h.device)
                nat.check(lib.ee_decode_attention_bf16(qkv.data_ptr(), self.kv_cache[l].data_ptr(),
                                                       qpos_c.data_ptr(), B, q, H, Dh, T + 1,
                                                       att.data_ptr(), st))
            else:
                qh = qkv.view(B, q, 3, H, Dh)[:, :, 0].transpose(1, 2)
                att = F.scaled_dot_product_attention(qh, self.k_cache[l], self.v_cache[l],
                                                     attn_mask=mask).transpose(1, 2).reshape(B, q, d)
            add_ln(gemm(att, w["o_w"], w["o_b32"]), w["ln2_w"], w["ln2_b"])
            # bias + tanh-GELU in the GEMM epilogue, then the projection
            t = gemm(x, w["fc_w"], w["fc_b32"], act="gelu_tanh")
            y = gemm(t, w["pr_w"], w["pr_b32"])
            if l + 1 < l1:
                add_ln(y, self.layers[l + 1]["ln1_w"], self.layers[l + 1]["ln1_b"])
            else:
                h += y
        return h

    def embed(self, tokens, pos):
        return self.wte[tokens] + self.wpe[pos.clamp(min=0)]

    def head_logits(self, h2d):
        """Final LN + tied LM head on [M, d] -> fp32 [M, V] (tcgen05 GEMM)."""
        F = self.torch.nn.functional
        x = F.layer_norm(h2d, (self.spec.d_model,), self.lnf_w, self.lnf_b, eps=1e-5)
        return linear_tc(x.to(self.torch.bfloat16).contiguous(), self.wte)

    def reset(self):
        for kv in self.kv_cache:
            kv.zero_()

    def full_forward(self, tokens):
        """Teacher-forced causal forward of [B, T'] tokens through every layer
        (fresh cache, one chunk): the reference for KV-fill correctness."""
        torch = self.torch
        B, Tn = tokens.shape
        pos = torch.arange(Tn, device="cuda")[None, :].expand(B, Tn).contiguous()
        self.reset()
        h = self.layers_forward(self.embed(tokens, pos), pos, 0, self.spec.n_layer)
        F = torch.nn.functional
        return F.layer_norm(h, (self.spec.d_model,), self.lnf_w, self.lnf_b, eps=1e-5)


@dataclass
class TokenLog:
    """One generated token of one sequence (host)."""
    seq: int
    index: int        # 0 = first generated token
    err: float        # ramp error score
    ramp_label: int   # ramp argmax
    exited: bool
    released: int     # the token emitted (ramp label if exited, else the model's)
    final: int = -1   # the original model's token (filled when its suffix runs)
    tpt_ms: float = float("nan")


@dataclass
class DecodeReport:
    tokens: list[TokenLog]
    flushes: list[tuple[int, int, int, str]]  # (seq, step, count, kind)
    step_ms: list[float]
    final_hidden: dict = field(default_factory=dict)  # (seq, position) -> fp32 [d] (optional)


class TokenEEDecoder:
    """Batch decoding with one ramp after layer `ramp_layer` (max_ramps = 1,
    generative.py:78) and the reference's deferral schedule."""

    def __init__(self, model: GPT2Decoder, ramp_layer: int, threshold: float, *,
                 flush_cap: int = 4, conf: str = "maxprob", use_graphs: bool = True):
        if not 1 <= ramp_layer < model.spec.n_layer:
            raise ParameterError("ramp_layer must be inside the decoder")
        if flush_cap < 1:
            raise ParameterError("flush_cap must be >= 1")
        self.m = model
        self.L = ramp_layer
        self.cap = flush_cap
        self.conf = conf
        self.use_graphs = use_graphs
        torch = model.torch
        B, d, C = model.B, model.spec.d_model, flush_cap + 1
        self.threshold = torch.full((1,), float(threshold), dtype=torch.float64, device="cuda")
        # static buffers (CUDA-graph inputs / outputs)
        self.cur = torch.zeros(B, dtype=torch.long, device="cuda")
        self.ppos = torch.zeros(B, 1, dtype=torch.long, device="cuda")
        self.h_ramp = torch.zeros(B, d, dtype=torch.bfloat16, device="cuda")
        self.err = torch.zeros(B, dtype=torch.float32, device="cuda")
        self.label = torch.zeros(B, dtype=torch.int32, device="cuda")
        self.exits = torch.zeros(B, dtype=torch.uint8, device="cuda")
        self.chunk = torch.zeros(B, C, d, dtype=torch.bfloat16, device="cuda")
        self.spos = torch.full((B, C), -1, dtype=torch.long, device="cuda")
        self.final_label = torch.zeros(B * C, dtype=torch.int32, device="cuda")
        self.final_err = torch.zeros(B * C, dtype=torch.float32, device="cuda")
        self.final_h = torch.zeros(B, C, d, dtype=torch.float32, device="cuda")
        self.never = torch.full((1,), -1.0, dtype=torch.float64, device="cuda")  # argmax only
        self._dev = None  # device-scheduled decoding state (_device_state)

    # ---- the two fixed-shape passes
    def _prefix(self):
        m = self.m
        h = m.layers_forward(m.embed(self.cur[:, None], self.ppos), self.ppos, 0, self.L)
        self.h_ramp.copy_(h[:, 0])
        logits = m.head_logits(self.h_ramp)
        exit_from_logits(logits, self.threshold, conf=self.conf, site=0,
                         out_err=self.err, out_label=self.label, out_exits=self.exits)

    def _suffix(self):
        m = self.m
        B, C, d = self.chunk.shape
        h = m.layers_forward(self.chunk, self.spos, self.L, m.spec.n_layer)
        F = m.torch.nn.functional
        self.final_h.copy_(F.layer_norm(h, (d,), m.lnf_w, m.lnf_b, eps=1e-5).float())
        logits = linear_tc(self.final_h.view(B * C, d).to(m.torch.bfloat16).contiguous(), m.wte)
        exit_from_logits(logits, self.never, conf=self.conf, site=1,
                         out_err=self.final_err, out_label=self.final_label)

    def run_prefix(self):
        self._prefix()

    def run_suffix(self):
        self._suffix()

    # ---- the deferral schedule on the device (ee_defer_plan / ee_defer_finish)
    def _device_state(self):
        """Persistent device buffers of the on-device schedule (capacity: the
        model's max_tokens decode steps) and the ee_defer_state that points at them."""
        if self._dev is not None:
            return self._dev
        import ctypes

        torch = self.m.torch
        B, C, N = self.m.B, self.cap + 1, self.m.T
        z = lambda *shape, dt: torch.zeros(*shape, dtype=dt, device="cuda")  # noqa: E731
        t = {"step": z(1, dt=torch.int32), "n_def": z(B, dt=torch.int32), "qpos": z(B, dt=torch.int64),
             "def_step": z(B, C, dt=torch.int32), "mem_cnt": z(B, dt=torch.int32),
             "h_exit": z(N + 1, B, dt=torch.uint8), "h_err": z(N + 1, B, dt=torch.float32),
             "h_lab": z(N + 1, B, dt=torch.int32), "h_final": z(N + 1, B, dt=torch.int32),
             "h_cnt": z(N + 1, B, dt=torch.int32), "h_kind": z(N + 1, B, dt=torch.uint8),
             "h_qbase": z(N + 1, B, dt=torch.int64), "fixed": z(N, B, dt=torch.uint8)}

        class State(ctypes.Structure):
            _fields_ = [(k, ctypes.c_void_p) for k in ("step", "n_def", "qpos", "def_step", "mem_cnt",
                                                        "spos", "h_exit", "h_err", "h_lab", "h_final",
                                                        "h_cnt", "h_kind", "h_qbase")] + \
                       [("n_max", ctypes.c_int32), ("pad_", ctypes.c_int32)]

        st = State(**{k: (self.spos if k == "spos" else t[k]).data_ptr() for k, _ in State._fields_[:13]},
                   n_max=N, pad_=0)
        self._dev = {"t": t, "st": st, "hidden": None, "graphs": {}}
        return self._dev

    def _plan(self, end_mode: bool, use_fixed: bool):
        dev = self._dev
        m, torch = self.m, self.m.torch
        B, C, d = self.chunk.shape
        import ctypes

        nat.check(nat.load_library().ee_defer_plan(
            ctypes.byref(dev["st"]), B, C, d, self.cap, self.h_ramp.data_ptr(), self.chunk.data_ptr(),
            self.exits.data_ptr(), dev["t"]["fixed"].data_ptr() if use_fixed else None,
            self.err.data_ptr(), self.label.data_ptr(), int(end_mode), nat.stream_handle(torch)))

    def _finish(self, end_mode: bool):
        dev = self._dev
        torch = self.m.torch
        B, C, d = self.chunk.shape
        import ctypes

        hid = dev["hidden"]
        nat.check(nat.load_library().ee_defer_finish(
            ctypes.byref(dev["st"]), B, C, d, self.final_label.data_ptr(), self.label.data_ptr(),
            self.cur.data_ptr(), self.ppos.data_ptr(), self.final_h.data_ptr(),
            hid.data_ptr() if hid is not None else None, int(end_mode), nat.stream_handle(torch)))

    def _step_graphs(self, use_fixed: bool, keep_hidden: bool):
        """(A, B): A = prefix layers + ramp + plan, B = suffix + finish, captured once
        per (fixed exits, hidden history) variant."""
        dev = self._device_state()
        key = (use_fixed, keep_hidden)
        if key in dev["graphs"]:
            return dev["graphs"][key]
        torch = self.m.torch
        t = dev["t"]
        saved = {k: v.clone() for k, v in t.items()}
        saved_io = (self.cur.clone(), self.ppos.clone(), self.chunk.clone(), self.spos.clone())
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm-up (allocations), then restore the state
            self._prefix()
            self._plan(False, use_fixed)
            self._suffix()
            self._finish(False)
        torch.cuda.current_stream().wait_stream(s)
        for k, v in saved.items():
            t[k].copy_(v)
        for dst, src in zip((self.cur, self.ppos, self.chunk, self.spos), saved_io):
            dst.copy_(src)
        ga, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(ga):
            self._prefix()
            self._plan(False, use_fixed)
        with torch.cuda.graph(gb):
            self._suffix()
            self._finish(False)
        dev["graphs"][key] = (ga, gb)
        return ga, gb

    def _generate_device(self, prompt, n_new: int, keep_hidden: bool, fixed_exits) -> "DecodeReport":
        """The whole decode enqueued without a host round trip per step: the
        schedule lives in ee_defer_state, the host reads the histories once at
        the end. Same tokens, flushes and feedback as the host-driven loop."""
        torch = self.m.torch
        m = self.m
        B, C, d = self.chunk.shape
        dev = self._device_state()
        t = dev["t"]
        use_fixed = fixed_exits is not None
        if keep_hidden and dev["hidden"] is None:
            dev["hidden"] = torch.zeros(m.T + 1, B, C, d, dtype=torch.float32, device="cuda")
        ga, gb = self._step_graphs(use_fixed, keep_hidden)
        first, P = self.prefill(prompt)
        if P + n_new > m.T:
            raise ParameterError("prompt + new tokens exceed the KV cache")
        for v in t.values():
            v.zero_()
        t["qpos"].fill_(P)
        self.ppos.fill_(P)
        self.spos.fill_(-1)
        self.cur.copy_(first)
        if use_fixed:
            t["fixed"][:n_new].copy_(torch.as_tensor(np.asarray(fixed_exits, dtype=np.uint8)[:n_new]))
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_new)]
        for k in range(n_new):
            ev[k][0].record()
            ga.replay()
            ev[k][1].record()
            gb.replay()
            ev[k][2].record()
        # end of decoding: flush what is still parked
        self._plan(True, use_fixed)
        self._suffix()
        self._finish(True)
        torch.cuda.synchronize()
        h = {k: v.cpu().numpy() for k, v in t.items() if k.startswith("h_")}
        step_ms, t_ramp = [], []
        for k in range(n_new):
            t_ramp.append(ev[k][0].elapsed_time(ev[k][1]))
            step_ms.append(ev[k][0].elapsed_time(ev[k][2]))
        logs = []
        for k in range(n_new):
            for s_ in range(B):
                ex = bool(h["h_exit"][k, s_])
                lab = int(h["h_lab"][k, s_])
                fin = int(h["h_final"][k, s_])
                logs.append(TokenLog(s_, k, float(h["h_err"][k, s_]), lab, ex, lab if ex else fin, fin,
                                     t_ramp[k] if ex else step_ms[k]))
        names = {1: "carry", 2: "cap", 3: "end"}
        flushes = []
        hidden = {}
        hid = dev["hidden"].cpu() if keep_hidden else None
        for k in range(n_new + 1):
            row = m.T if k == n_new else k
            for s_ in range(B):
                cnt, kind = int(h["h_cnt"][row, s_]), int(h["h_kind"][row, s_])
                if kind in names:
                    flushes.append((s_, k, cnt - 1 if kind == 1 else cnt, names[kind]))
                if keep_hidden and cnt > 0:
                    q0 = int(h["h_qbase"][row, s_])
                    for i in range(cnt):
                        hidden[(s_, q0 + i)] = hid[row, s_, i].cuda()
        return DecodeReport(logs, flushes, step_ms, hidden)

    # ---- decoding
    def prefill(self, prompt):
        """Full forward over the prompt [B, P] (no early exit); returns the first
        generated token per sequence."""
        torch = self.m.torch
        m = self.m
        B, P = prompt.shape
        pos = torch.arange(P, device="cuda")[None, :].expand(B, P).contiguous()
        m.reset()
        h = m.layers_forward(m.embed(prompt, pos), pos, 0, m.spec.n_layer)
        logits = m.head_logits(h[:, -1].contiguous())
        res = exit_from_logits(logits, self.never, conf=self.conf)
        return res.label.long(), P

    def generate(self, prompt, n_new: int, *, keep_hidden: bool = False, timed: bool = True,
                 fixed_exits=None) -> DecodeReport:
        """Decode n_new tokens per sequence after `prompt` [B, P]. fixed_exits (bool
        [n_new, B], optional) forces the exit decisions (tests)."""
        torch = self.m.torch
        m = self.m
        B, C = m.B, self.cap + 1
        if prompt.shape[0] != B:
            raise ParameterError("prompt batch must equal the decoder batch")
        if self.use_graphs:  # the schedule on the device: no host round trip per step
            return self._generate_device(prompt, n_new, keep_hidden, fixed_exits)
        first, P = self.prefill(prompt)
        if P + n_new > m.T:
            raise ParameterError("prompt + new tokens exceed the KV cache")
        self.cur.copy_(first)
        p = np.full(B, P, dtype=np.int64)       # next position in the prefix layers
        q = np.full(B, P, dtype=np.int64)       # next position in the suffix layers
        deferred: list[list[TokenLog]] = [[] for _ in range(B)]
        logs: list[TokenLog] = []
        flushes: list[tuple[int, int, int, str]] = []
        step_ms: list[float] = []
        hidden: dict = {}
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]

        rows_t = torch.arange(B, device="cuda")

        def run_chunk(members: dict[int, list[TokenLog]], kinds: dict[int, str], step: int):
            """Suffix pass for {seq: [tokens...]} (deferred first, current last)."""
            sp = np.full((B, C), -1, dtype=np.int64)
            for s, toks in members.items():
                sp[s, :len(toks)] = np.arange(q[s], q[s] + len(toks))
            self.spos.copy_(torch.from_numpy(sp))
            self.run_suffix()
            fl = self.final_label.view(B, C).cpu().numpy()
            for s, toks in members.items():
                for i, t in enumerate(toks):
                    t.final = int(fl[s, i])
                    if keep_hidden:
                        hidden[(s, int(q[s]) + i)] = self.final_h[s, i].clone()
                q[s] += len(toks)
                if kinds.get(s):
                    flushes.append((s, step, sum(1 for t in toks if t.exited), kinds[s]))

        for step in range(n_new):
            self.ppos.copy_(torch.from_numpy(p[:, None]))
            ev[0].record()
            self.run_prefix()
            ev[1].record()
            exits = self.exits.cpu().numpy().astype(bool)
            if fixed_exits is not None:
                exits = np.asarray(fixed_exits[step], dtype=bool)
            err = self.err.cpu().numpy()
            lab = self.label.cpu().numpy()
            # park this step's layer-L hidden states behind each sequence's deferred ones
            slot = np.array([len(deferred[s]) for s in range(B)], dtype=np.int64)
            self.chunk[rows_t, torch.from_numpy(slot).cuda()] = self.h_ramp
            members, kinds = {}, {}
            for s in range(B):
                t = TokenLog(s, step, float(err[s]), int(lab[s]), bool(exits[s]), int(lab[s]))
                logs.append(t)
                deferred[s].append(t)
                if not exits[s]:  # carries every parked suffix with it
                    members[s] = deferred[s]
                    if len(deferred[s]) > 1:
                        kinds[s] = "carry"
                    deferred[s] = []
                elif len(deferred[s]) >= self.cap:
                    members[s] = deferred[s]
                    kinds[s] = "cap"
                    deferred[s] = []
                p[s] += 1
            if members:
                run_chunk(members, kinds, step)
            ev[2].record()
            ev[2].synchronize()
            t_ramp = ev[0].elapsed_time(ev[1])
            t_full = ev[0].elapsed_time(ev[2])
            step_ms.append(t_full)
            nxt = np.empty(B, dtype=np.int64)
            for s in range(B):
                t = logs[-B + s]
                t.tpt_ms = t_ramp if t.exited else t_full
                if not t.exited:
                    t.released = t.final
                nxt[s] = t.released
            self.cur.copy_(torch.from_numpy(nxt))
        # end of decoding: flush what is still parked
        members = {s: deferred[s] for s in range(B) if deferred[s]}
        if members:
            run_chunk(members, {s: "end" for s in members}, n_new)
        return DecodeReport(logs, flushes, step_ms, hidden)


def vanilla_step_ms(model: GPT2Decoder, prompt, n_new: int) -> list[float]:
    """Reference decode (no ramp): every token runs all layers + head, batch B,
    one CUDA graph per step shape. Returns per-step milliseconds."""
    torch = model.torch
    B, P = prompt.shape
    dec = TokenEEDecoder(model, ramp_layer=model.spec.n_layer - 1, threshold=0.0, use_graphs=False)
    first, _ = dec.prefill(prompt)
    cur = torch.zeros(B, dtype=torch.long, device="cuda")
    pos = torch.zeros(B, 1, dtype=torch.long, device="cuda")
    never = torch.full((1,), -1.0, dtype=torch.float64, device="cuda")
    lab = torch.zeros(B, dtype=torch.int32, device="cuda")
    errb = torch.zeros(B, dtype=torch.float32, device="cuda")

    def step():
        h = model.layers_forward(model.embed(cur[:, None], pos), pos, 0, model.spec.n_layer)
        logits = model.head_logits(h[:, 0].contiguous())
        exit_from_logits(logits, never, out_err=errb, out_label=lab)

    cur.copy_(first)
    pos.fill_(P)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    out = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(n_new):
        pos.fill_(P + i)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
        cur.copy_(lab.long())
    return out
