"""CPU baselines for BASELINE configs 1, 2, 3 and 5 (BASELINE.md "Configs 2, 3,
5": a PyTorch CPU fp32 restatement timed on all host cores, plus the reference
`eesim` exit decision on its signals).

For C1-C3 one step is one feedback-mode EE batch on the CPU: the fp32 backbone
(same architecture and shapes as ee_infer's builders, random init), every ramp
head (global-average-pool + FC + softmax confidence) and the reference's exit
rule per record (eesim.engine.evaluate_record from baseline/_ref, engine.py:189-220;
the package's host mirror when the reference is not installed). Each config
runs a bounded sample of its batch (scaled to samples/s) so the whole script
stays within a few minutes. C5 times GPT-2-medium-shape decode steps (HF GPT2,
fp32, KV cache) at batch 32 after a 128-token prompt. One JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def decider():
    """(decide(errs [R, B], labels [R, B], finals [B], thresholds) -> None, source)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "eesim")):
        sys.path.insert(0, ref)
        from eesim.engine import EEConfig, evaluate_record
        from eesim.graph import ModelProfile, find_feasible_sites
        from eesim.trace import RampSignal, RequestRecord
        src = "eesim.engine.evaluate_record (baseline/_ref)"
    else:
        from paper_2312_05385_b200.engine import EEConfig, evaluate_record
        from paper_2312_05385_b200.graph import ModelProfile, find_feasible_sites
        from paper_2312_05385_b200.trace import RampSignal, RequestRecord
        src = "host mirror of evaluate_record"

    def decide(err, lab, fin, th):
        r = err.shape[0]
        names = [f"s{j}" for j in range(r)]
        nodes = names + ["out"]
        prof = ModelProfile(nodes, list(zip(nodes, nodes[1:])), {x: {1: 1.0} for x in nodes},
                            {x: {1: 0.01} for x in names}, "out")
        sites = find_feasible_sites(prof)
        cfg = EEConfig(tuple(zip(sites, th)))
        for i in range(err.shape[1]):
            sig = {n: RampSignal(float(err[j, i]), int(lab[j, i])) for j, n in enumerate(names)}
            evaluate_record(RequestRecord(i, 0.0, sig, int(fin[i])), cfg, prof)
    return decide, src


def ramp(h, w):
    x = h.mean(dim=(2, 3)) if h.dim() == 4 else h
    p = torch.softmax(x @ w.t(), dim=1)
    return 1.0 - p.max(dim=1).values, p.argmax(dim=1)


def time_ee(stage_fn, heads, x, decide, reps=2):
    """Feedback-mode EE batch on the CPU: (seconds per batch, forward share)."""
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        with torch.no_grad():
            errs, labs, final = stage_fn(x, heads)
        t1 = time.perf_counter()
        e, l = np.stack(errs), np.stack(labs)
        th = [float(np.quantile(e[j], 0.1)) for j in range(e.shape[0])]
        decide(e, l, final, th)
        t2 = time.perf_counter()
        if best is None or t2 - t0 < best[0]:
            best = (t2 - t0, t1 - t0, t2 - t1)
    return best


def resnet_stages(m, blocks, final):
    def run(x, heads):
        errs, labs = [], []
        h = x
        for j, blk in enumerate(blocks):
            h = blk(h)
            if j in heads:
                e, l = ramp(h, heads[j])
                errs.append(e.numpy())
                labs.append(l.numpy())
        fin = final(h).argmax(dim=1).numpy()
        return errs, labs, fin
    return run


def main():
    torch.manual_seed(0)
    threads = torch.get_num_threads()
    decide, dsrc = decider()
    out = {"threads": threads, "cpu_model": cpu_model(), "dtype": "fp32", "decision": dsrc}

    only = set(os.environ.get("EEB200_CPU_CONFIGS", "c1,c2,c3,c5").split(","))
    # C1: ResNet-18 CIFAR, 6 ramps, B=32 (the full batch)
    if "c1" in only:
        c1(out, decide)
    if "c2" in only:
        c2(out, decide)
    if "c3" in only:
        c3(out, decide)
    if "c5" in only:
        c5(out)
    print(json.dumps(out))


def c1(out, decide):
    import torchvision

    m = torchvision.models.resnet18(num_classes=10)
    m.conv1 = torch.nn.Conv2d(3, 64, 3, 1, 1, bias=False)
    m.maxpool = torch.nn.Identity()
    m.eval()
    stem = torch.nn.Sequential(m.conv1, m.bn1, m.relu)
    blocks = [stem, m.layer1[0], m.layer1[1], m.layer2[0], m.layer2[1], m.layer3[0], m.layer3[1],
              m.layer4[0], m.layer4[1]]
    chans = [64, 64, 64, 128, 128, 256, 256, 512, 512]
    heads = {s: torch.randn(10, chans[s]) / chans[s] ** 0.5 for s in (0, 2, 3, 5, 6, 8)}
    final = torch.nn.Sequential(m.avgpool, torch.nn.Flatten(), m.fc)
    b = 32
    t, tf, td = time_ee(resnet_stages(m, blocks, final), heads, torch.randn(b, 3, 32, 32), decide)
    out["c1"] = {"config": "resnet18_cifar_6ramps", "batch": b, "sample": b,
                 "samples_per_s": b / t, "p50_batch_ms": t * 1e3, "forward_ms": tf * 1e3,
                 "decide_ms": td * 1e3}



def c2(out, decide):
    """BERT-base, 12 ramps (token 0 -> 2 classes, entropy), seq 128; sample 16 of 64."""
    from transformers import BertConfig, BertModel

    cfg = BertConfig(attn_implementation="sdpa")
    bert = BertModel(cfg, add_pooling_layer=False).eval()
    hw = {j: torch.randn(2, 768) / 768 ** 0.5 for j in range(12)}
    fw = torch.randn(2, 768) / 768 ** 0.5

    def bert_run(ids, heads):
        errs, labs = [], []
        h = bert.embeddings(input_ids=ids)
        for j, layer in enumerate(bert.encoder.layer):
            o = layer(h)
            h = o[0] if isinstance(o, tuple) else o
            p = torch.softmax(h[:, 0] @ heads[j].t(), dim=1)
            ent = -(p * torch.log(p.clamp_min(1e-30))).sum(dim=1) / np.log(2.0)
            errs.append(ent.numpy())
            labs.append(p.argmax(dim=1).numpy())
        return errs, labs, (h[:, 0] @ fw.t()).argmax(dim=1).numpy()

    s2 = 16
    t, tf, td = time_ee(bert_run, hw, torch.randint(0, 30522, (s2, 128)), decide)
    out["c2"] = {"config": "bert_base_12ramps_seq128_entropy", "batch": 64, "sample": s2,
                 "samples_per_s": s2 / t, "p50_batch_ms": t * 1e3 * 64 / s2,
                 "forward_ms_per_sample": tf * 1e3 / s2, "decide_ms_per_sample": td * 1e3 / s2}



def c3(out, decide):
    """ResNet-50 224x224, 16 ramps (1000 classes); sample 16 of 256."""
    import torchvision

    m = torchvision.models.resnet50().eval()
    stem = torch.nn.Sequential(m.conv1, m.bn1, m.relu, m.maxpool)
    blocks, chans = [], []
    for layer, c in ((m.layer1, 256), (m.layer2, 512), (m.layer3, 1024), (m.layer4, 2048)):
        for blk in layer:
            blocks.append(blk)
            chans.append(c)
    blocks[0] = torch.nn.Sequential(stem, blocks[0])
    heads = {s: torch.randn(1000, c) * (16.0 / c ** 0.5) for s, c in enumerate(chans)}
    final = torch.nn.Sequential(m.avgpool, torch.nn.Flatten(), m.fc)
    s3 = 16
    t, tf, td = time_ee(resnet_stages(m, blocks, final), heads, torch.randn(s3, 3, 224, 224), decide,
                        reps=1)
    out["c3"] = {"config": "resnet50_imagenet_16ramps", "batch": 256, "sample": s3,
                 "samples_per_s": s3 / t, "p50_batch_ms": t * 1e3 * 256 / s3,
                 "forward_ms_per_sample": tf * 1e3 / s3, "decide_ms_per_sample": td * 1e3 / s3}



def c5(out):
    """GPT-2-medium-shape decode, batch 32, prompt 128 (KV cache), fp32."""
    from transformers import GPT2Config, GPT2LMHeadModel

    gpt = GPT2LMHeadModel(GPT2Config(n_embd=1024, n_layer=24, n_head=16)).eval()
    ids = torch.randint(0, 50257, (32, 128))
    with torch.no_grad():
        o = gpt(ids, use_cache=True)
        past = o.past_key_values
        nxt = o.logits[:, -1].argmax(dim=1, keepdim=True)
        steps = []
        for _ in range(4):
            t0 = time.perf_counter()
            o = gpt(nxt, past_key_values=past, use_cache=True)
            past = o.past_key_values
            p = torch.softmax(o.logits[:, -1], dim=1)
            nxt = p.argmax(dim=1, keepdim=True)
            steps.append(time.perf_counter() - t0)
    tpt = float(np.median(steps))
    out["c5"] = {"config": "gpt2_medium_decode_b32", "batch": 32, "tpt_p50_ms": tpt * 1e3,
                 "tokens_per_s": 32 / tpt, "sample": "4 decode steps after a 128-token prompt, "
                 "full depth (the CPU arm exits nothing; vanilla decode)"}


if __name__ == "__main__":
    main()
