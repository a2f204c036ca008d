"""NEXT-4 K6 A/B of two liborl builds (each its own binding instance), interleaved with the
unfused cuBLAS GEMM + K1, cool and after a warm-up; NVML SM clock per block.
    python tools/k6_lib_ab.py old.so new.so [--blocks 10] [--reps 10]"""
import argparse
import importlib.util
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_11143_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs=2)
ap.add_argument("--R", type=int, default=8192)
ap.add_argument("--T", type=int, default=1024)
ap.add_argument("--d", type=int, default=4096)
ap.add_argument("--V", type=int, default=128256)
ap.add_argument("--blocks", type=int, default=10)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--warm-seconds", type=float, default=20.0)
a = ap.parse_args()
mods = []
for i, path in enumerate(a.libs):
    os.environ["ORL_LIB_PATH"] = os.path.abspath(path)
    spec = importlib.util.spec_from_file_location(f"orl_k6ab_{i}", os.path.join(ROOT, "paper_2405_11143_b200", "orl.py"))
    m = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = m
    spec.loader.exec_module(m)
    mods.append((os.path.basename(path), m))
dev = torch.device("cuda:0")
B, T = a.R // a.T, a.T
b = synth.make_lmhead_batch(1, B, T, a.d, a.V, lengths="full", device=dev)
tok, L = b["tokens"].to(dev), b["lengths"].to(dev)
h, W = b["hidden_old"], b["weight"]
flops = 2.0 * a.R * a.d * a.V
logits = torch.empty(a.R, a.V, dtype=torch.bfloat16, device=dev)
arms, outs = {}, {}
for name, m in mods:
    ctx = m.Context(0)
    m.orl_begin_iteration(ctx)
    o = (torch.zeros(B, T, device=dev), torch.zeros(B, T, device=dev))
    outs[name] = o
    arms[name] = (lambda m=m, ctx=ctx, o=o: m.orl_lmhead_logprobs(ctx, tok, L, h, W, o[0], entropy=o[1]))
m0, ctx0 = mods[0][1], None
ctxu = m0.Context(0)
m0.orl_begin_iteration(ctxu)
ku = (torch.zeros(B, T, device=dev), torch.zeros(B, T, device=dev))
arms["cublas+K1"] = lambda: (torch.matmul(h, W.t(), out=logits),
                             m0.orl_logprobs(ctxu, tok, L, logits.view(B, T, a.V), ku[0], entropy=ku[1]))
for f in arms.values():
    f()
torch.cuda.synchronize()
import pynvml  # noqa: E402
pynvml.nvmlInit()
nv = pynvml.nvmlDeviceGetHandleByIndex(0)


def block(f, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM)


n0, n1 = mods[0][0], mods[1][0]
res = {"libs": [n0, n1], "outputs_identical": all(torch.equal(outs[n0][i], outs[n1][i]) for i in range(2))}
for state, warm in (("cool", 0.0), ("hot", a.warm_seconds)):
    t0 = time.time()
    while time.time() - t0 < warm:
        for f in arms.values():
            block(f, 3)
    per = {k: [] for k in arms}
    keys = list(arms)
    for rep in range(a.blocks if state == "hot" else 3):
        for k in keys[rep % len(keys):] + keys[:rep % len(keys)]:  # rotated: no first-position bias
            f = arms[k]
            per[k].append(block(f, a.reps if state == "hot" else 3))
    for k, v in per.items():
        res[f"{state}_{k}_ms"] = round(statistics.median(x[0] for x in v), 4)
        res[f"{state}_{k}_mhz"] = statistics.median(x[1] for x in v)
    for n in (n0, n1):
        res[f"{state}_{n}_vs_unfused"] = round(res[f"{state}_cublas+K1_ms"] / res[f"{state}_{n}_ms"], 4)
print(json.dumps(res))
