"""K1-only microbenchmark: GB/s of orl_logprobs / orl_ppo_loss on resident bf16 logits.

    python tools/k1_bench.py [--V 128256] [--rows 8192] [--iters 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_11143_b200 import orl, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--V", type=int, default=128256)
ap.add_argument("--T", type=int, default=1024)
ap.add_argument("--mb", type=int, default=8)
ap.add_argument("--nbuf", type=int, default=6)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--kinds", default="logp,logp+H,loss,sum,copy")
a = ap.parse_args()
dev = torch.device("cuda:0")
B, T, V = a.mb * a.nbuf, a.T, a.V
x = torch.randn(B, T, V, device=dev, dtype=torch.bfloat16)
tok = synth.tokens_for(B, T, V, 0).to(dev)
L = torch.full((B,), T, dtype=torch.int32, device=dev)
z = lambda: torch.zeros(B, T, device=dev)  # noqa: E731
lp, ent, lo, adv, lpn, dl = z(), z(), z(), z(), z(), z()
ctx = orl.Context(0)
orl.orl_begin_iteration(ctx)
orl.orl_advantages(ctx, L, adv, kind="rpp", shaped_reward=z())
orl.orl_whiten_stats(ctx, True)
cfg = orl.PPOConfig()


def run(kind, i):
    s = (i % a.nbuf) * a.mb
    xv = x[s:s + a.mb]
    if kind == "sum":            # torch reference: read-only streaming reduction
        return xv.sum(dtype=torch.float32)
    if kind == "copy":           # torch reference: the MEASURED_PEAKS copy (read + write bytes)
        return y.copy_(xv)
    if kind == "logp":
        orl.orl_logprobs(ctx, tok, L, xv, lp, seq_offset=s)
    elif kind == "logp+H":
        orl.orl_logprobs(ctx, tok, L, xv, lp, entropy=ent, seq_offset=s)
    else:
        orl.orl_ppo_loss(ctx, tok, L, xv, cfg, lo, adv, lpn, seq_offset=s, entropy=ent, dloss_dlogp=dl)


y = torch.empty_like(x[: a.mb])
for kind in a.kinds.split(","):
    for i in range(5):
        run(kind, i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.iters):
        run(kind, i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    gb = a.mb * T * V * 2 / 1e9 * (2 if kind == "copy" else 1)
    print(f"{kind:8s} V={V} rows={a.mb * T}: {ms * 1e3:8.1f} us/launch  {gb / ms * 1e3:8.1f} GB/s")
