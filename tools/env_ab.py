"""A/B of one liborl build under environment-variable switches (read by the library per call),
interleaved in one process, cool and after a warm-up.  Used for the round-2 K7 re-check:
    python tools/env_ab.py build_var/libk7era.so "K7:" "K1fused:ORL_FUSED_K1=1"
"""
import os
import statistics
import subprocess
import sys
import time
import importlib.util

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

os.environ["ORL_LIB_PATH"] = os.path.abspath(sys.argv[1])
spec = importlib.util.spec_from_file_location("orl_env_ab", os.environ.get("ORL_BINDING") or os.path.join(ROOT, "paper_2405_11143_b200", "orl.py"))
orl = importlib.util.module_from_spec(spec)
sys.modules[spec.name] = orl
spec.loader.exec_module(orl)
from paper_2405_11143_b200 import synth  # noqa: E402

arms = []
for a in sys.argv[2:]:
    name, _, env = a.partition(":")
    arms.append((name, dict(kv.split("=", 1) for kv in env.split(",") if kv)))
dev = torch.device("cuda:0")
nb, mb, T, V = 6, 8, 1024, 128256
x = torch.randn(nb * mb, T, V, device=dev, dtype=torch.bfloat16)
tok = synth.tokens_for(nb * mb, T, V, 0).to(dev)
L = torch.full((nb * mb,), T, dtype=torch.int32, device=dev)
z = lambda: torch.zeros(nb * mb, T, device=dev)  # noqa: E731
lo, adv, lpn, dl, lse, ent = z(), z(), z(), z(), z(), z()
dlog = torch.empty_like(x[:mb])
ctx = orl.Context(0)
orl.orl_begin_iteration(ctx)
orl.orl_advantages(ctx, L, adv, kind="rpp", shaped_reward=z())
orl.orl_whiten_stats(ctx, True)
cfg = orl.PPOConfig(c2=0.01)


def set_env(env):
    for _, e in arms:
        for k in e:
            os.environ.pop(k, None)
    os.environ.update(env)


def timed(env, iters=30):
    set_env(env)
    for i in range(3):
        orl.orl_ppo_loss_and_grad(ctx, tok, L, x[(i % nb) * mb:(i % nb + 1) * mb], cfg, lo, adv, lpn, seq_offset=(i % nb) * mb,
                                  entropy=ent, lse=lse, dloss_dlogp=dl, dlogits=dlog)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        s = (i % nb) * mb
        orl.orl_ppo_loss_and_grad(ctx, tok, L, x[s:s + mb], cfg, lo, adv, lpn, seq_offset=s, entropy=ent, lse=lse,
                                  dloss_dlogp=dl, dlogits=dlog)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


for state, warm in (("cool", 0.0), ("hot", 20.0)):
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms",
                            "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    t0 = time.time()
    while time.time() - t0 < warm:
        timed(arms[0][1], 50)
    res = {n: [] for n, _ in arms}
    for r in range(8):
        for n, e in arms:
            res[n].append(timed(e))
    smi.terminate()
    out, _ = smi.communicate()
    clk = [float(l.split(",")[0]) for l in out.strip().splitlines() if l.strip()]
    for n, v in res.items():
        print(f"{state} {n:10s} fused pass {statistics.median(v):7.1f} us (min {min(v):.1f} max {max(v):.1f})")
    if clk:
        print(f"{state} SM clock median {statistics.median(clk):.0f} MHz")
