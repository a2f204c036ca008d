"""NEXT-4 timing: orl_lmhead_logprobs (K6 tcgen05 GEMM + online LSE, then the merge)
vs the unfused baseline cuBLAS bf16 GEMM (torch.matmul, logits written to HBM) + K1.
    python tools/k6_bench.py [--R 8192] [--d 4096] [--V 128256] [--reps 20]"""
import argparse
import json
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2405_11143_b200 import orl, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--R", type=int, default=8192)
ap.add_argument("--T", type=int, default=1024)
ap.add_argument("--d", type=int, default=4096)
ap.add_argument("--V", type=int, default=128256)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--no-baseline", action="store_true")
ap.add_argument("--warm", type=int, default=3)
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


CLK = {}


def timeit(fn, reps, tag="x"):
    """CUDA-event time per call after warm-up; SM clock (NVML) sampled during the region."""
    import threading
    try:
        import pynvml
        pynvml.nvmlInit()
        hnd = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    except Exception:  # pragma: no cover
        hnd = None
    for _ in range(a.warm):
        fn()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def sampler():
        while hnd is not None and not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(hnd) / 1000.0))
            stop.wait(0.02)
    th = threading.Thread(target=sampler)
    th.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    if samples:
        cl = sorted(x[0] for x in samples)
        pw = sorted(x[1] for x in samples)
        CLK[tag] = {"sm_mhz_median": cl[len(cl) // 2], "power_w_median": pw[len(pw) // 2], "n": len(cl)}
    return ev[0].elapsed_time(ev[1]) / reps


def fused():
    orl.orl_lmhead_logprobs(ctx, tok, L, h, W, logp, entropy=H)


res = {"R": a.R, "d": a.d, "V": a.V, "gflop": flops / 1e9}
orl.orl_begin_iteration(ctx)
ms = timeit(fused, a.reps, "fused")
res["fused_ms"] = ms
res["fused_tflops"] = flops / ms / 1e9
if not a.no_baseline:
    logits = torch.empty(a.R, a.V, dtype=torch.bfloat16, device=dev)
    gemm = lambda: torch.matmul(h, W.t(), out=logits)  # noqa: E731
    res["cublas_ms"] = timeit(gemm, a.reps, "cublas")
    res["cublas_tflops"] = flops / res["cublas_ms"] / 1e9
    lg3 = logits.view(B, T, a.V)
    k1 = lambda: orl.orl_logprobs(ctx, tok, L, lg3, logp, entropy=H)  # noqa: E731
    res["k1_ms"] = timeit(k1, a.reps, "k1")
    res["unfused_ms"] = res["cublas_ms"] + res["k1_ms"]
    res["speedup_vs_unfused"] = res["unfused_ms"] / ms
res["clocks"] = CLK
for k in ("fused", "cublas"):
    if k in CLK and f"{k}_tflops" in res:  # FLOP per SM cycle at the sampled clock (peak 8192 bf16 dense)
        res[f"{k}_flop_per_sm_clk"] = res[f"{k}_tflops"] * 1e12 / (148 * CLK[k]["sm_mhz_median"] * 1e6)
print(json.dumps(res))
