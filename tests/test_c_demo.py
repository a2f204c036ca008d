"""The C ABI used from plain C (examples/orl_demo.c: C99 + the CUDA runtime, no Python,
no PyTorch in the process): the header compiles as C99 with -Wall -Wextra -Werror and the
program links against liborl.so (CPU test); on the GPU the C program's iteration gives
statistics and per-token outputs bit-identical to the same iteration through the Python
binding (same kernels, same launches), and within the oracle's tolerances."""
from __future__ import annotations

import json
import os
import subprocess

import numpy as np
import pytest
import torch

from paper_2405_11143_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2405_11143_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    from paper_2405_11143_b200 import build
    build.build()
    exe = str(tmp_path / "orl_demo")
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-O2", os.path.join(ROOT, "examples", "orl_demo.c"),
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"), "-L", PKG, "-l:liborl.so",
           "-L", os.path.join(CUDA, "lib64"), "-lcudart", f"-Wl,-rpath,{PKG}", "-o", exe]
    subprocess.run(cmd, check=True)
    return exe


def test_c_demo_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)
    nm = subprocess.run(["nm", "-u", exe], capture_output=True, text=True).stdout
    for sym in ("orl_create", "orl_logprobs", "orl_advantages", "orl_whiten_stats", "orl_ppo_loss", "orl_finalize"):
        assert sym in nm
    assert "torch" not in nm and "Py" not in nm


@pytest.mark.gpu
def test_c_demo_matches_python_binding(tmp_path):
    from paper_2405_11143_b200 import orl
    from paper_2405_11143_b200.pipeline import Buffers, PathConfig, run_iteration
    exe = _build(tmp_path)
    B, T, V = 5, 64, 4096
    dev = torch.device("cuda:0")
    L = synth.lengths_for(B, T, 61, "mixed")
    tok = synth.tokens_for(B, T, V, 61)
    lg = tuple(torch.empty(B, T, V, dtype=torch.bfloat16, device=dev) for _ in range(3))
    synth.fill_logits_(lg, tok.to(dev), 61, 0, "stress")
    R = synth.rewards_for(B, 61, "normal", 1)
    v_old, v_new = synth.values_for(B, T, 61)
    d = tmp_path
    for name, x in (("logits_old", lg[0]), ("logits_ref", lg[1]), ("logits_new", lg[2])):
        x.cpu().view(torch.int16).numpy().tofile(d / f"{name}.bin")
    tok.numpy().astype(np.int32).tofile(d / "tokens.bin")
    L.numpy().astype(np.int32).tofile(d / "lengths.bin")
    R.numpy().astype(np.float32).tofile(d / "seq_reward.bin")
    v_old.numpy().astype(np.float32).tofile(d / "values_old.bin")
    v_new.numpy().astype(np.float32).tofile(d / "values_new.bin")
    out = subprocess.run([exe, str(d), str(B), str(T), str(V)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    c_st = json.loads(out.stdout.strip().splitlines()[-1])
    assert c_st["status"] == 0
    # the same iteration through the Python binding
    cfg = PathConfig(adv_kind="gae", gamma=1.0, lam=0.95, whiten=True, kl_est_reward="k1", beta_reward=0.01,
                     ppo=orl.PPOConfig(eps_low=0.2, eps_high=0.2, eps_value=0.2, c1=0.5, kl_loss_est="k1"))
    batch = dict(tokens=tok.to(dev), lengths=L.to(dev), seq_reward=R.to(dev), values_old=v_old.to(dev),
                 values_new=v_new.to(dev))
    ctx = orl.Context(0)
    bufs = Buffers(B, T, dev)
    status, st = run_iteration(ctx, batch, cfg, bufs, lambda role, s, e: lg[("old", "ref", "new").index(role)][s:e],
                               mb=2)
    torch.cuda.synchronize()
    ctx.close()
    assert status == "ORL_OK"
    for k, v in st.items():
        if k in c_st and isinstance(v, float):
            assert c_st[k] == v, (k, c_st[k], v)                 # bit-identical (%.17g round-trips)
    c_logp = np.fromfile(d / "c_logp_new.bin", dtype=np.float32).reshape(B, T)
    c_adv = np.fromfile(d / "c_adv.bin", dtype=np.float32).reshape(B, T)
    assert np.array_equal(c_logp, bufs.logp_new.cpu().numpy())
    assert np.array_equal(c_adv, bufs.adv.cpu().numpy())
