"""BASELINE config 5: GPT-2-medium-shape decode, batch 32, token-level early exit
with one ramp (final LN + LM head after layer 12), deferred suffixes with real KV
fill. Time-per-token (per-token release latency, CUDA events) p50 with early exit
vs vanilla decoding of the same model; thresholds = err quantile of a probe run.
Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2312_05385_b200.generative import GPT2Decoder, GPT2Spec, TokenEEDecoder, vanilla_step_ms


def pct(x, q):
    return float(np.percentile(np.asarray(x), q))  # linear, as manifest.py:100-107


def main():
    B, P, N = int(os.environ.get("B", 32)), int(os.environ.get("P", 128)), int(os.environ.get("N", 128))
    ramp, cap = int(os.environ.get("RAMP", 12)), int(os.environ.get("CAP", 4))
    q = float(os.environ.get("Q", 0.5))
    model = GPT2Decoder(GPT2Spec(), batch=B, max_tokens=P + N + 1, seed=0)
    prompt = torch.randint(0, 50257, (B, P), generator=torch.Generator(device="cuda").manual_seed(0),
                           device="cuda")
    van = vanilla_step_ms(model, prompt, N)
    dec = TokenEEDecoder(model, ramp, 0.0, flush_cap=cap)
    probe = dec.generate(prompt, 16)
    thr = float(np.quantile([t.err for t in probe.tokens], q))
    dec.threshold.fill_(thr)
    dec.generate(prompt, 8)  # warm
    rep = dec.generate(prompt, N)
    tpt = [t.tpt_ms for t in rep.tokens]
    ex = [t for t in rep.tokens if t.exited]
    out = {
        "config": "config5: GPT-2-medium-shape decode (24 x 1024, 16 heads, vocab 50257, random init, bf16), "
                  f"batch {B}, prompt {P}, {N} new tokens, ramp after layer {ramp} (ln_f + LM head), "
                  f"flush_cap {cap}, threshold = q{q} of probe err",
        "tpt_p50_ms": pct(tpt, 50), "tpt_p90_ms": pct(tpt, 90),
        "vanilla_tpt_p50_ms": pct(van, 50),
        "tpt_p50_vs_vanilla": pct(tpt, 50) / pct(van, 50),
        "exit_rate": len(ex) / len(rep.tokens),
        "exit_tpt_p50_ms": pct([t.tpt_ms for t in ex], 50) if ex else None,
        "step_ms_mean": float(np.mean(rep.step_ms)), "vanilla_step_ms_mean": float(np.mean(van)),
        "tokens_per_s": B * N / (sum(rep.step_ms) / 1e3),
        "vanilla_tokens_per_s": B * N / (sum(van) / 1e3),
        "flushes": {k: sum(1 for f in rep.flushes if f[3] == k) for k in ("cap", "carry", "end")},
        "ramp_agrees_with_model": float(np.mean([t.ramp_label == t.final for t in ex])) if ex else None,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
