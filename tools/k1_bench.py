"""K1-only microbenchmark: GB/s of orl_logprobs / orl_ppo_loss on resident bf16 logits.

    python tools/k1_bench.py [--V 128256] [--iters 30] [--warm-seconds 0] [--repeat 1]
    python tools/k1_bench.py --libs a.so,b.so ...   # interleave several liborl builds

With --warm-seconds the GPU first runs the loss kernel back to back for that
long (reaching its power/thermal steady state), then every (lib, kind) pair is
timed `--repeat` times, interleaved, and the median is reported with the SM
clock sampled during the run.
"""
import argparse
import ctypes
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--V", type=int, default=128256)
ap.add_argument("--T", type=int, default=1024)
ap.add_argument("--mb", type=int, default=8)
ap.add_argument("--nbuf", type=int, default=6)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--kinds", default="logp,logp+H,loss,sum,copy")
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--warm-seconds", type=float, default=0.0)
ap.add_argument("--libs", default="")
ap.add_argument("--c2", type=float, default=0.01, help="entropy coefficient of the loss (0: no entropy term)")
ap.add_argument("--l2-persist-mb", type=float, default=-1.0,
                help="experiment: cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize) before the run")
a = ap.parse_args()
if a.l2_persist_mb >= 0:
    import ctypes
    import nvidia.cuda_runtime as _cr
    _rt = ctypes.CDLL(os.path.join(list(_cr.__path__)[0], "lib", "libcudart.so.12"))
    torch.cuda.init()
    _v = ctypes.c_int(0)
    _rt.cudaDeviceGetAttribute(ctypes.byref(_v), 108, 0)  # cudaDevAttrMaxPersistingL2CacheSize
    _err = _rt.cudaDeviceSetLimit(0x06, ctypes.c_size_t(int(a.l2_persist_mb * 2**20)))  # cudaLimitPersistingL2CacheSize
    _got = ctypes.c_size_t(0)
    _rt.cudaDeviceGetLimit(ctypes.byref(_got), 0x06)
    print(f"persisting L2 limit: max {_v.value / 2**20:.1f} MB, set err {_err}, now {_got.value / 2**20:.1f} MB")

libs = a.libs.split(",") if a.libs else [os.environ.get("ORL_LIB_PATH", "")]
mods = []
import importlib.util  # noqa: E402

_ORL_PY = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2405_11143_b200", "orl.py")
for i, path in enumerate(libs):
    # each build gets its own binding module instance (own ctypes handle); importlib.reload
    # would mutate one shared module so that every "lib" ran the last build loaded
    if path:
        os.environ["ORL_LIB_PATH"] = os.path.abspath(path)
    spec = importlib.util.spec_from_file_location(f"orl_build_{i}", _ORL_PY)
    orl_mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = orl_mod
    spec.loader.exec_module(orl_mod)
    assert os.path.abspath(orl_mod.LIB_PATH) == os.path.abspath(path or orl_mod.LIB_PATH)
    mods.append((os.path.basename(path) or "liborl.so", orl_mod))

from paper_2405_11143_b200 import synth  # noqa: E402

dev = torch.device("cuda:0")
B, T, V = a.mb * a.nbuf, a.T, a.V
x = torch.randn(B, T, V, device=dev, dtype=torch.bfloat16)
tok = synth.tokens_for(B, T, V, 0).to(dev)
L = torch.full((B,), T, dtype=torch.int32, device=dev)
z = lambda: torch.zeros(B, T, device=dev)  # noqa: E731
lp, ent, lo, adv, lpn, dl, lse = z(), z(), z(), z(), z(), z(), z()
y = torch.empty_like(x[: a.mb])
dlog = torch.empty_like(x[: a.mb])
ctxs = {}
for name, orl in mods:
    ctx = orl.Context(0)
    orl.orl_begin_iteration(ctx)
    orl.orl_advantages(ctx, L, adv, kind="rpp", shaped_reward=z())
    orl.orl_whiten_stats(ctx, True)
    cfg = orl.PPOConfig(c2=a.c2)
    orl.orl_ppo_loss(ctx, tok, L, x[: a.mb], cfg, lo, adv, lpn, entropy=ent, lse=lse, dloss_dlogp=dl)
    ctxs[name] = (orl, ctx, cfg)


def run(name, kind, i):
    orl, ctx, cfg = ctxs[name]
    s = (i % a.nbuf) * a.mb
    xv = x[s:s + a.mb]
    if kind == "sum":            # torch reference: read-only streaming reduction
        return xv.sum(dtype=torch.float32)
    if kind == "copy":           # torch reference: the MEASURED_PEAKS copy (read + write bytes)
        return y.copy_(xv)
    if kind == "grad":           # NEXT-1 backward: read logits + write dlogits
        return orl.orl_logits_grad(ctx, tok, L, xv, cfg, lse, ent, dl, dlog, seq_offset=s)
    if kind == "lossgrad":       # fused actor forward + backward: read once (+ L2 re-read), write dlogits
        return orl.orl_ppo_loss_and_grad(ctx, tok, L, xv, cfg, lo, adv, lpn, seq_offset=s, entropy=ent, lse=lse,
                                         dloss_dlogp=dl, dlogits=dlog)
    if kind == "logp":
        orl.orl_logprobs(ctx, tok, L, xv, lp, seq_offset=s)
    elif kind == "logp+H":
        orl.orl_logprobs(ctx, tok, L, xv, lp, entropy=ent, seq_offset=s)
    else:
        orl.orl_ppo_loss(ctx, tok, L, xv, cfg, lo, adv, lpn, seq_offset=s, entropy=ent, dloss_dlogp=dl)


def timed(name, kind):
    for i in range(3):
        run(name, kind, i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.iters):
        run(name, kind, i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.iters


smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu", "--format=csv,noheader,nounits",
                        "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
if a.warm_seconds > 0:
    t0 = time.time()
    first = next(iter(ctxs))
    while time.time() - t0 < a.warm_seconds:
        timed(first, "loss")
try:  # per-block SM clock / power (NVML, sampled right after each timed block)
    import pynvml
    pynvml.nvmlInit()
    _nv = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    def _clk():
        return (pynvml.nvmlDeviceGetClockInfo(_nv, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(_nv) / 1e3)
except Exception:  # pragma: no cover
    _clk = None
res, rclk = {}, {}
names = list(ctxs)
for r in range(a.repeat):
    # rotate the build order every repeat: the first build of a cycle runs at a higher clock
    # under the power cap (measured ~8 %), so a fixed order biases interleaved A/Bs
    for name in names[r % len(names):] + names[:r % len(names)]:
        for kind in a.kinds.split(","):
            res.setdefault((name, kind), []).append(timed(name, kind))
            if _clk:
                rclk.setdefault((name, kind), []).append(_clk())
smi.terminate()
out, _ = smi.communicate()
clk = [float(l.split(",")[0]) for l in out.strip().splitlines() if l.strip()]
pw = [float(l.split(",")[1]) for l in out.strip().splitlines() if l.strip()]
for (name, kind), v in res.items():
    ms = statistics.median(v)
    gb = a.mb * T * V * 2 / 1e9 * (2 if kind in ("copy", "grad", "lossgrad") else 1)
    ck = rclk.get((name, kind))
    cks = (f"  [{statistics.median(c for c, _ in ck):.0f} MHz {statistics.median(w for _, w in ck):.0f} W]"
           if ck else "")
    print(f"{name:28s} {kind:7s} V={V}: {ms * 1e3:8.1f} us/launch  {gb / ms * 1e3:8.1f} GB/s  "
          f"(min {min(v) * 1e3:.1f} max {max(v) * 1e3:.1f}){cks}")
if clk:
    print(f"SM clock median {statistics.median(clk):.0f} MHz (min {min(clk):.0f}), power median {statistics.median(pw):.0f} W")
