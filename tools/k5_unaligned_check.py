"""Stress check: K5 on unaligned rows (TMA interior + scalar head/tail) vs the generic K5,
bit for bit, over many random inputs.  python tools/k5_unaligned_check.py [iters]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_11143_b200 import orl, synth  # noqa: E402

DEV = torch.device("cuda:0")
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
ctx = orl.Context(0)
fails = 0
for it in range(iters):
    for dtype, V, pad in (("f32", 1001, 1), ("bf16", 50257, 0), ("bf16", 4096, 5)):
        B, T = 3, 20
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        g = torch.Generator(device=DEV).manual_seed(1000 * it + V)
        x = (torch.randn(B, T, V + pad, device=DEV, generator=g) * 2).to(tdt)[..., :V]
        tok = synth.tokens_for(B, T, V, it).to(DEV)
        tok[0, :3] = torch.tensor([0, 1, V - 1], dtype=torch.int32, device=DEV)
        L = torch.tensor([T, 11, 0], dtype=torch.int32, device=DEV)
        z = lambda: torch.zeros(B, T, device=DEV)  # noqa: E731
        lse, ent = z(), z()
        w = torch.randn(B, T, device=DEV, generator=g) * 1e-3
        orl.orl_begin_iteration(ctx)
        orl.orl_logprobs(ctx, tok, L, x, z(), entropy=ent, lse=lse)
        adv = z()
        orl.orl_advantages(ctx, L, adv, kind="rpp", shaped_reward=z())
        orl.orl_whiten_stats(ctx, False)
        cfg = orl.PPOConfig(c2=0.01 if it % 2 else 0.0)  # both backward instantiations
        outs = {}
        for mode in ("tma", "generic", "tma2"):
            if mode == "generic":
                os.environ["ORL_K1_NO_UNALIGNED_TMA"] = "1"
            else:
                os.environ.pop("ORL_K1_NO_UNALIGNED_TMA", None)
            dl = torch.full((B, T, V + pad), 3.0, dtype=tdt, device=DEV)[..., :V]
            orl.orl_logits_grad(ctx, tok, L, x, cfg, lse, ent, w, dl, zero_masked=True)
            torch.cuda.synchronize()
            outs[mode] = dl.float().cpu().numpy()
        for a, b in (("tma", "generic"), ("tma", "tma2")):
            bad = np.argwhere(outs[a] != outs[b])
            if bad.size:
                fails += 1
                print(it, dtype, V, pad, a, b, len(bad), bad[:6].tolist(),
                      [(float(outs[a][tuple(i)]), float(outs[b][tuple(i)])) for i in bad[:3]], flush=True)
print("fails", fails)
