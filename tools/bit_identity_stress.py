"""Stress the bit-identity claims on random shapes (V incl. unaligned, lengths, micro-batch
sizes, advantage kinds): (a) the same iteration twice, (b) the fused actor loss+backward
pass vs the two passes, (c) a CUDA-graph replay vs eager.   python tools/bit_identity_stress.py [iters]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_11143_b200 import orl, synth  # noqa: E402
from paper_2405_11143_b200.pipeline import Buffers, GraphStep, PathConfig, run_iteration  # noqa: E402

DEV = torch.device("cuda:0")
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ctx = orl.Context(0)
KEYS = ("logp_old", "logp_ref", "kl", "shaped", "adv", "adv_lo", "ret", "logp_new", "entropy", "lse", "dlogp", "dv",
        "flags")
fails = 0
for it in range(iters):
    rng = np.random.default_rng(it)
    V = int(rng.choice([4096, 8192, 50257, 32000, 1001, 128256 // 8]))
    kind = str(rng.choice(["gae", "rpp", "grpo", "rpp_baseline"]))
    G = 2 if kind in ("grpo", "rpp_baseline") else 1
    B = int(rng.integers(1, 5)) * G
    T = int(rng.choice([16, 64, 200]))
    mb = int(rng.integers(1, B + 1))
    c2 = float(rng.choice([0.0, 0.01]))  # c2 = 0: the backward instantiations without the entropy term
    c = dict(synth.CONFIGS["llama8b"], V=V, adv_kind=kind, group_size=G, c2=c2)
    if kind == "grpo":
        c.update(kl_mode="loss", beta_loss=0.01, whiten=False, eps_v=0.0, c1=0.0)
    cfg = PathConfig.from_synth(c)
    L = synth.lengths_for(B, T, it, "mixed")
    tok = synth.tokens_for(B, T, V, it).to(DEV)
    lg = tuple(torch.empty(B, T, V, dtype=torch.bfloat16, device=DEV) for _ in range(3))
    synth.fill_logits_(lg, tok, it, 0, "stress")
    R = synth.rewards_for(B, it, "group_bernoulli" if G > 1 else "normal", G)
    vo, vn = synth.values_for(B, T, it)
    g = dict(tokens=tok, lengths=L.to(DEV), seq_reward=R.to(DEV), values_old=vo.to(DEV), values_new=vn.to(DEV))
    src = lambda role, s, e: lg[("old", "ref", "new").index(role)][s:e]  # noqa: E731
    res = {}
    for name, fused in (("a", True), ("b", True), ("two_pass", False)):
        dl = torch.full((B, T, V), 7.0, dtype=torch.bfloat16, device=DEV)
        bufs = Buffers(B, T, DEV, G)
        status, st = run_iteration(ctx, g, cfg, bufs, src, mb, grad_sink=lambda s, e: dl[s:e], fused_grad=fused)
        torch.cuda.synchronize()
        res[name] = (st, {k: getattr(bufs, k).clone() for k in KEYS if getattr(bufs, k) is not None}, dl)
    gb = Buffers(B, T, DEV, G)
    step = GraphStep(ctx, g, cfg, gb, src, mb)
    step.replay()
    torch.cuda.synchronize()
    eager = Buffers(B, T, DEV, G)
    st_e = run_iteration(ctx, g, cfg, eager, src, mb)
    msgs = []
    for other in ("b", "two_pass"):
        if res[other][0] != res["a"][0]:
            msgs.append(f"stats a vs {other}")
        for k, v in res["a"][1].items():
            if not torch.equal(v, res[other][1][k]):
                msgs.append(f"{k} a vs {other}")
        if not torch.equal(res["a"][2], res[other][2]):
            msgs.append(f"dlogits a vs {other}")
    if step.result() != st_e:
        msgs.append("graph stats")
    for k in KEYS:
        if k == "dv" and not cfg.critic:
            continue
        if getattr(eager, k) is not None and not torch.equal(getattr(gb, k), getattr(eager, k)):
            msgs.append(f"graph {k}")
    if msgs:
        fails += 1
        print(it, dict(V=V, kind=kind, B=B, T=T, mb=mb), msgs, flush=True)
print("fails", fails, "of", iters)
