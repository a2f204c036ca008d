"""NEXT-4 K6 schedule sweep in one process (k6_plan re-reads its env knobs per call):
ORL_K6_MGROUP (row-block group), ORL_K6_TPS (vocab tiles per split), ORL_K6_POLA/POLB
(L2 policies of h / W).  Prints one JSON line per setting.  Under ncu, run with
--reps 1 --warm 0 so each setting is exactly one k6 launch.
    python tools/k6_sched.py [--R 8192] [--d 4096] [--V 128256] [--reps 20]"""
import argparse
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_11143_b200 import orl, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--R", type=int, default=8192)
ap.add_argument("--T", type=int, default=1024)
ap.add_argument("--d", type=int, default=4096)
ap.add_argument("--V", type=int, default=128256)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--warm", type=int, default=3)
ap.add_argument("--mgroup", default="32,16,8,4")
ap.add_argument("--tps", default="4,8")
ap.add_argument("--pola", default="1,0")
ap.add_argument("--polb", default="0")
a = ap.parse_args()
dev = torch.device("cuda:0")
B, T = a.R // a.T, a.T
b = synth.make_lmhead_batch(1, B, T, a.d, a.V, lengths="full", device=dev)
ctx = orl.Context(0)
tok, L = b["tokens"].to(dev), b["lengths"].to(dev)
h, W = b["hidden_old"], b["weight"]
logp = torch.zeros(B, T, device=dev)
H = torch.zeros(B, T, device=dev)
flops = 2.0 * a.R * a.d * a.V
orl.orl_begin_iteration(ctx)
ref = None
for mg, tps, pa, pb in itertools.product(a.mgroup.split(","), a.tps.split(","), a.pola.split(","),
                                         a.polb.split(",")):
    os.environ.update(ORL_K6_MGROUP=mg, ORL_K6_TPS=tps, ORL_K6_POLA=pa, ORL_K6_POLB=pb)
    fn = lambda: orl.orl_lmhead_logprobs(ctx, tok, L, h, W, logp, entropy=H)  # noqa: E731
    for _ in range(a.warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    same = None
    if ref is None:
        ref = logp.clone()
    else:
        same = bool(torch.equal(ref, logp))
    print(json.dumps({"mgroup": int(mg), "tps": int(tps), "pol_a": int(pa), "pol_b": int(pb), "ms": round(ms, 4),
                      "tflops": round(flops / ms / 1e9, 1), "bit_identical_to_first": same}), flush=True)
