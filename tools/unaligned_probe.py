"""Aligned vs misaligned rows of the same V and pitch through K1 (the unaligned-row TMA mode).
    python tools/unaligned_probe.py [--ncu]   (--ncu: one launch of each, for ncu -k regex:k1_tma)"""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2405_11143_b200 import orl, synth  # noqa: E402

dev = torch.device("cuda:0")
B, T, V = 8, 1024, 50264
x = torch.randn(4 * B, T, V + 8, device=dev).to(torch.bfloat16)
tok = synth.tokens_for(B, T, V, 0).to(dev)
L = torch.full((B,), T, dtype=torch.int32, device=dev)
lp = torch.zeros(B, T, device=dev)
ctx = orl.Context(0)
ncu = "--ncu" in sys.argv


def run(view, n=30):
    for i in range(1 if ncu else 3):
        orl.orl_logprobs(ctx, tok, L, view(i % 4), lp)
    torch.cuda.synchronize()
    if ncu:
        return 0.0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        orl.orl_logprobs(ctx, tok, L, view(i % 4), lp)
    b.record()
    torch.cuda.synchronize()
    return B * T * V * 2 / (a.elapsed_time(b) / n) / 1e6


orl.orl_begin_iteration(ctx)
for rep in range(1 if ncu else 2):
    print("aligned, pitch V+8            GB/s", run(lambda k: x[k * B:(k + 1) * B, :, :V]))
    print("misaligned by 4 B (offset 2)  GB/s", run(lambda k: x[k * B:(k + 1) * B, :, 2:V + 2]))
