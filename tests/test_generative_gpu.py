"""Config 5: the GPU token-level early-exit decoder against
(1) the reference's timeline schedule, restated in oracle/generative_ref.py and
pinned to the reference in test_generative_oracle.py — which tokens exit, and
every cap / carry / end flush — and (2) a teacher-forced full forward: the KV
cache of the skipped layers is filled for real, so every token's final hidden
state must match a plain causal forward over the same token sequence."""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import make_chain
from oracle.generative_ref import sequence_timeline
from paper_2312_05385_b200.engine import EEConfig
from paper_2312_05385_b200.graph import find_feasible_sites
from paper_2312_05385_b200.trace import RampSignal

pytestmark = pytest.mark.gpu

SPEC_LAYERS = 24
RAMP = 12


def _decoder(torch, batch, max_tokens, threshold, cap=4, graphs=True):
    from paper_2312_05385_b200.generative import GPT2Decoder, GPT2Spec, TokenEEDecoder

    model = GPT2Decoder(GPT2Spec(), batch=batch, max_tokens=max_tokens, seed=0)
    return model, TokenEEDecoder(model, RAMP, threshold, flush_cap=cap, use_graphs=graphs)


def _oracle_check(rep, B, cap, threshold):
    prof = make_chain(SPEC_LAYERS, layer_ms=1.0, ramp_ms=0.1, name="gpt2m")
    site = find_feasible_sites(prof)[RAMP - 1]  # after layers 0..RAMP-1
    config = EEConfig(((site, float(threshold)),))
    for s in range(B):
        toks = [t for t in rep.tokens if t.seq == s]
        recs = [SimpleNamespace(ramp_signals={site.position: RampSignal(t.err, t.ramp_label)},
                                final_token=t.final) for t in toks]
        stats, flushes, _ = sequence_timeline(recs, prof, config, flush_cap=cap)
        assert [st.exit_site is not None for st in stats] == [t.exited for t in toks]
        assert [st.correct for st in stats] == [(t.ramp_label == t.final) if t.exited else True
                                                for t in toks]
        ours = [(c, k) for (sq, _, c, k) in rep.flushes if sq == s]
        assert ours == [(f.tokens, f.kind) for f in flushes]
        assert all(t.final >= 0 for t in toks)  # every token's suffix ran (feedback)


def _kv_check(torch, model, rep, prompt, first_inputs, n_new, tol=5e-2):
    """bf16 model, 24 layers: the decode passes and the teacher-forced forward run
    the same math at different GEMM tilings (decode chunks vs one long chunk:
    other split-K / z-tile plans, other fp32 accumulation orders), so final
    hidden states agree to bf16 noise (measured worst 2-4 % of the row's max);
    a missing or misplaced KV entry shows up as an O(1) error."""
    B, P = prompt.shape
    inputs = np.zeros((B, n_new), dtype=np.int64)
    for t in rep.tokens:
        if t.index + 1 < n_new:
            inputs[t.seq, t.index + 1] = t.released
    inputs[:, 0] = first_inputs
    full = torch.cat([prompt, torch.from_numpy(inputs).cuda()], dim=1)
    ref = model.full_forward(full).float()
    worst = 0.0
    for (s, pos), h in rep.final_hidden.items():
        r = ref[s, pos]
        worst = max(worst, float((h - r).abs().max() / r.abs().max()))
    assert len(rep.final_hidden) == B * n_new
    assert worst < tol, worst


def test_schedule_and_kv_fill_with_measured_exits(cuda):
    torch = cuda
    B, P, n_new = 4, 8, 24
    model, dec = _decoder(torch, B, P + n_new + 1, threshold=0.0)
    g = torch.Generator(device="cuda").manual_seed(1)
    prompt = torch.randint(0, 50257, (B, P), generator=g, device="cuda")
    probe = dec.generate(prompt, 6, timed=False)  # threshold 0: nothing exits
    errs = np.array([t.err for t in probe.tokens])
    assert not any(t.exited for t in probe.tokens)
    thr = float(np.median(errs))
    dec.threshold.fill_(thr)
    first, _ = dec.prefill(prompt)
    rep = dec.generate(prompt, n_new, keep_hidden=True)
    ex = np.mean([t.exited for t in rep.tokens])
    assert 0.05 < ex < 0.95, ex
    _oracle_check(rep, B, dec.cap, thr)
    _kv_check(torch, model, rep, prompt, first.cpu().numpy(), n_new)


def test_forced_cap_carry_end_flushes(cuda):
    """Seq 0 always exits (cap flushes), seq 1 alternates (carries), seq 2 never
    exits, seq 3 exits only at the end (end flush); eager and graph paths."""
    torch = cuda
    B, P, n_new, cap = 4, 5, 14, 3
    for graphs in (False, True):
        model, dec = _decoder(torch, B, P + n_new + 1, threshold=0.5, cap=cap, graphs=graphs)
        prompt = torch.randint(0, 50257, (B, P), generator=torch.Generator(device="cuda").manual_seed(2),
                               device="cuda")
        fixed = np.zeros((n_new, B), dtype=bool)
        fixed[:, 0] = True
        fixed[::2, 1] = True
        fixed[-2:, 3] = True
        first, _ = dec.prefill(prompt)
        rep = dec.generate(prompt, n_new, keep_hidden=True, fixed_exits=fixed)
        kinds = {s: [(c, k) for (sq, _, c, k) in rep.flushes if sq == s] for s in range(B)}
        assert kinds[0] == [(cap, "cap")] * (n_new // cap) + ([(n_new % cap, "end")] if n_new % cap else [])
        assert kinds[1] == [(1, "carry")] * (n_new // 2)
        assert kinds[2] == []
        assert kinds[3] == [(2, "end")]
        _kv_check(torch, model, rep, prompt, first.cpu().numpy(), n_new)


def test_kv_append_matches_scatter(cuda):
    """ee_kv_append_bf16 writes exactly the K/V rows a scatter into the cache
    would (padding rows to the sink slot), and nothing else."""
    import torch

    from paper_2312_05385_b200 import _native as nat

    B, q, H, Dh, T1 = 5, 3, 4, 64, 11
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = torch.randn(B, q, 3, H, Dh, generator=g, device="cuda").to(torch.bfloat16)
    pos = torch.tensor([[0, 1, 2], [4, 5, 10], [7, 10, 8], [3, 2, 1], [9, 8, 6]], device="cuda")
    kv = torch.randn(2, B, H, T1, Dh, generator=g, device="cuda").to(torch.bfloat16)
    ref = kv.clone()
    for b in range(B):
        for i in range(q):
            ref[0, b, :, pos[b, i]] = qkv[b, i, 1]
            ref[1, b, :, pos[b, i]] = qkv[b, i, 2]
    nat.check(nat.load_library().ee_kv_append_bf16(qkv.data_ptr(), pos.data_ptr(), B, q, H, Dh, T1,
                                                    kv.data_ptr(), nat.stream_handle(torch)))
    assert torch.equal(kv, ref)


def test_add_layernorm_matches_torch(cuda):
    """ee_add_layernorm_bf16: h += y rounded exactly like torch's bf16 add; x
    within bf16 rounding of torch's LayerNorm of that h."""
    import torch

    from paper_2312_05385_b200 import _native as nat

    g = torch.Generator(device="cuda").manual_seed(4)
    # rows >= 64 and d <= 2048 take the warp-per-row kernel (BERT 8192 x 768)
    for rows, d in ((32, 1024), (7, 64), (160, 1024), (8192, 768), (100, 2048), (70, 24), (65, 4096),
                    (64, 520), (96, 776)):
        h = torch.randn(rows, d, generator=g, device="cuda").to(torch.bfloat16)
        y = torch.randn(rows, d, generator=g, device="cuda").to(torch.bfloat16)
        gamma = (1 + 0.1 * torch.randn(d, generator=g, device="cuda")).to(torch.bfloat16)
        beta = (0.1 * torch.randn(d, generator=g, device="cuda")).to(torch.bfloat16)
        h_ref = h + y
        x_ref = torch.nn.functional.layer_norm(h_ref.float(), (d,), gamma.float(), beta.float(), eps=1e-5)
        x = torch.empty_like(h)
        nat.check(nat.load_library().ee_add_layernorm_bf16(
            h.data_ptr(), y.data_ptr(), gamma.data_ptr(), beta.data_ptr(), 1e-5, rows, d,
            x.data_ptr(), nat.stream_handle(torch)))
        assert torch.equal(h, h_ref)
        assert torch.allclose(x.float(), x_ref, rtol=2 ** -7, atol=2 ** -7)
        # LayerNorm only (no residual): h untouched
        h0 = h.clone()
        nat.check(nat.load_library().ee_add_layernorm_bf16(
            h.data_ptr(), None, gamma.data_ptr(), beta.data_ptr(), 1e-5, rows, d,
            x.data_ptr(), nat.stream_handle(torch)))
        assert torch.equal(h, h0)
        x_ref = torch.nn.functional.layer_norm(h0.float(), (d,), gamma.float(), beta.float(), eps=1e-5)
        assert torch.allclose(x.float(), x_ref, rtol=2 ** -7, atol=2 ** -7)


def test_decode_attention_matches_sdpa(cuda):
    """ee_decode_attention_bf16 (length-aware, q <= 8 queries per sequence)
    against torch SDPA with the equivalent mask, fp32 reference on the same
    bf16 operands; padding queries (qpos 0) see key 0 only."""
    import torch

    from paper_2312_05385_b200 import _native as nat

    g = torch.Generator(device="cuda").manual_seed(5)
    B, H, Dh, T1 = 6, 4, 64, 197
    for q in (1, 3, 8):
        qkv = torch.randn(B, q, 3, H, Dh, generator=g, device="cuda").to(torch.bfloat16)
        kv = torch.randn(2, B, H, T1, Dh, generator=g, device="cuda").to(torch.bfloat16)
        qpos = torch.randint(0, T1 - 1, (B, q), generator=g, device="cuda")
        qpos[0, -1] = 0
        qpos[1, 0] = T1 - 2
        out = torch.empty(B, q, H * Dh, dtype=torch.bfloat16, device="cuda")
        nat.check(nat.load_library().ee_decode_attention_bf16(
            qkv.data_ptr(), kv.data_ptr(), qpos.data_ptr(), B, q, H, Dh, T1, out.data_ptr(),
            nat.stream_handle(torch)))
        qh = qkv[:, :, 0].transpose(1, 2).float()
        keys = torch.arange(T1, device="cuda")
        vis = (keys[None, None, :] <= qpos[:, :, None]) & (keys[None, None, :] < T1 - 1)
        ref = torch.nn.functional.scaled_dot_product_attention(
            qh, kv[0].float(), kv[1].float(), attn_mask=vis[:, None])
        ref = ref.transpose(1, 2).reshape(B, q, H * Dh)
        assert torch.allclose(out.float(), ref, rtol=2e-2, atol=2e-2), (out.float() - ref).abs().max()
