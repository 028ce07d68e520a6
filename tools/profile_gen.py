"""A few eager decode steps of the config-5 model for an ncu kernel list (not a benchmark)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05385_b200.generative import GPT2Decoder, GPT2Spec, TokenEEDecoder
B, P = 32, 128
model = GPT2Decoder(GPT2Spec(), batch=B, max_tokens=P + 64 + 1, seed=0)
prompt = torch.randint(0, 50257, (B, P), device="cuda")
dec = TokenEEDecoder(model, 12, 0.0, use_graphs=False)
first, _ = dec.prefill(prompt)
pos = torch.full((B, 1), P, dtype=torch.long, device="cuda")
torch.cuda.synchronize()
for _ in range(3):
    h = model.layers_forward(model.embed(first[:, None], pos), pos, 0, model.spec.n_layer)
torch.cuda.synchronize()
print("done")
