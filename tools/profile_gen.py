"""One vanilla decode step (24 layers at B x 1) and one EE step (12 prefix
layers + ramp + plan, then the 12-layer suffix over B x (cap + 1) chunk slots +
head + finish) of the config-5 model, each inside an NVTX range, for ncu launch
lists (not a benchmark)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05385_b200.generative import GPT2Decoder, GPT2Spec, TokenEEDecoder
B, P = 32, 128
model = GPT2Decoder(GPT2Spec(), batch=B, max_tokens=P + 64 + 1, seed=0)
prompt = torch.randint(0, 50257, (B, P), device="cuda")
dec = TokenEEDecoder(model, 12, 0.5)
dec.generate(prompt, 4)  # captures the step graphs
first, _ = dec.prefill(prompt)
pos = torch.full((B, 1), P, dtype=torch.long, device="cuda")
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("vanilla")
h = model.layers_forward(model.embed(first[:, None], pos), pos, 0, model.spec.n_layer)
logits = model.head_logits(h[:, 0].contiguous())
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
ga, gb = dec._step_graphs(False, False)
torch.cuda.nvtx.range_push("ee")
ga.replay()
gb.replay()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
