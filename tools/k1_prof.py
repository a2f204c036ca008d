"""Latency probes of the fused actor pass (builds with -DORL_K1_PROF): epilogue latency from
the row's partial states being complete to the backward constants being published, and
the consumers' wait for those constants, in SM cycles per row.  Cool, then after a warm-up.
    python tools/k1_prof.py build_var/libprof3.so [...]"""
import ctypes
import importlib.util
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2405_11143_b200 import synth  # noqa: E402

dev = torch.device("cuda:0")
B, T, V = 8, 1024, 128256
x = torch.randn(B, T, V, device=dev, dtype=torch.bfloat16)
tok = synth.tokens_for(B, T, V, 0).to(dev)
L = torch.full((B,), T, dtype=torch.int32, device=dev)
z = lambda: torch.zeros(B, T, device=dev)  # noqa: E731
lo, adv, lpn, dl, lse, ent = z(), z(), z(), z(), z(), z()
dlog = torch.empty_like(x)
for i, path in enumerate(sys.argv[1:]):
    os.environ["ORL_LIB_PATH"] = os.path.abspath(path)
    spec = importlib.util.spec_from_file_location(f"orl_p{i}", os.path.join(ROOT, "paper_2405_11143_b200", "orl.py"))
    orl = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = orl
    spec.loader.exec_module(orl)
    ctx = orl.Context(0)
    orl.orl_begin_iteration(ctx)
    orl.orl_advantages(ctx, L, adv, kind="rpp", shaped_reward=z())
    orl.orl_whiten_stats(ctx, True)
    cfg = orl.PPOConfig(c2=0.01)
    buf = (ctypes.c_ulonglong * 8)()

    def run(n):
        for _ in range(n):
            orl.orl_ppo_loss_and_grad(ctx, tok, L, x, cfg, lo, adv, lpn, entropy=ent, lse=lse, dloss_dlogp=dl,
                                      dlogits=dlog)
        torch.cuda.synchronize()

    for state, warm in (("cool", 0.0), ("hot", 15.0)):
        t0 = time.time()
        while time.time() - t0 < warm:
            run(50)
        run(2)
        orl._lib.orl_debug_k1_prof(buf)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(20)
        e1.record()
        torch.cuda.synchronize()
        orl._lib.orl_debug_k1_prof(buf)
        v = list(buf)
        us = e0.elapsed_time(e1) / 20 * 1e3
        print(f"{os.path.basename(path):14s} {state}: {us:6.1f} us/launch  epilogue full->publish {v[0] / max(v[2], 1):7.0f} cyc "
              f"(merge {v[1] / max(v[2], 1):5.0f})  consumer wait for constants {v[3] / max(v[4], 1):6.0f} cyc/row  "
              f"consumer publish {v[5] / max(v[6], 1):5.0f} cyc/row")
