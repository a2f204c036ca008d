"""A whole iteration captured as one CUDA graph (pipeline.GraphStep: every liborl launch
of run_iteration, orl_finalize_async instead of the synchronising orl_finalize) must
give bit-identical per-token outputs and statistics to the eager calls, on the inputs
present at replay time (the graph reads the resident logits in place)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2405_11143_b200 import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2405_11143_b200 import orl
    from paper_2405_11143_b200.pipeline import Buffers, GraphStep, PathConfig, run_iteration

DEV = torch.device("cuda:0")
KEYS = ("logp_old", "logp_ref", "kl", "shaped", "adv", "ret", "logp_new", "entropy", "lse", "dlogp", "dv")


def _batch(seed, B, T, V, kind):
    from tests.test_gpu_parity import _gpu_batch
    return _gpu_batch(seed, B, T, V, "mixed", "group_bernoulli" if kind == "grpo" else "normal",
                      2 if kind == "grpo" else 1)


def _cfg(kind):
    c = dict(synth.CONFIGS["llama8b"], adv_kind=kind, group_size=2 if kind == "grpo" else 1)
    if kind == "grpo":
        c.update(kl_mode="loss", beta_loss=0.01, whiten=False, eps_v=0.0, c1=0.0)
    return PathConfig.from_synth(c)


@pytest.mark.parametrize("kind", ["gae", "grpo"])
def test_graph_replay_bit_identical_to_eager(kind):
    B, T, V = 6, 96, 4096
    cfg = _cfg(kind)
    g = _batch(51, B, T, V, kind)
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    ctx = orl.Context(0)
    eager = Buffers(B, T, DEV, cfg.group_size)
    st_e = run_iteration(ctx, g, cfg, eager, src, mb=4)
    torch.cuda.synchronize()
    gb = Buffers(B, T, DEV, cfg.group_size)
    step = GraphStep(ctx, g, cfg, gb, src, mb=4)
    assert step.kernels > 0
    keys = [k for k in KEYS if cfg.critic or k != "dv"]  # no critic: dL/dV is not an output
    for _ in range(2):  # replays are idempotent
        for k in keys:
            getattr(gb, k).fill_(7.0)
        step.replay()
        torch.cuda.synchronize()
        assert step.result() == st_e
        for k in keys:
            assert torch.equal(getattr(gb, k), getattr(eager, k)), k
    # new logits written into the same resident buffers: the replay sees them
    fresh = _batch(52, B, T, V, kind)
    for r in ("old", "ref", "new"):
        g[f"logits_{r}"].copy_(fresh[f"logits_{r}"])
    st_e2 = run_iteration(ctx, g, cfg, eager, src, mb=4)
    step.replay()
    torch.cuda.synchronize()
    assert step.result() == st_e2
    assert st_e2 != st_e
    for k in keys:
        assert torch.equal(getattr(gb, k), getattr(eager, k)), k
    ctx.close()


def test_finalize_async_decode_matches_finalize():
    B, T, V = 4, 64, 2048
    cfg = _cfg("gae")
    g = _batch(53, B, T, V, "gae")
    g["tokens"][1, 3] = V + 5  # a data error: same status both ways
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    ctx = orl.Context(0)
    b1 = Buffers(B, T, DEV)
    st1 = run_iteration(ctx, g, cfg, b1, src, mb=2)
    b2 = Buffers(B, T, DEV)
    assert run_iteration(ctx, g, cfg, b2, src, mb=2, finalize="async") is None
    st2 = orl.orl_stats_decode(b2.final_dev.cpu().numpy(), cfg.ppo)
    assert st1[0] == "ORL_E_TOKEN_RANGE" and st2[0] == st1[0]
    for k, v in st1[1].items():  # NaN-aware: the bad token poisons the means
        assert (v != v and st2[1][k] != st2[1][k]) or st2[1][k] == v, k
    assert np.array_equal(b2.final_dev[:orl.STATS_N].cpu().numpy(), b1.stats_dev.cpu().numpy(), equal_nan=True)
    with pytest.raises(ValueError):
        orl.orl_finalize_async(ctx, cfg.ppo, torch.zeros(4, dtype=torch.float64, device=DEV))
    ctx.close()


def test_reserve_then_strict_capture_without_warmup():
    """orl_reserve pre-sizes every workspace, so an iteration can be captured in CUDA's
    strict (global) capture mode with no eager warm-up; the replay equals eager."""
    B, T, V = 5, 80, 3000
    cfg = _cfg("gae")
    g = _batch(54, B, T, V, "gae")
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    ctx = orl.Context(0)
    orl.orl_reserve(ctx, B)
    gb = Buffers(B, T, DEV, cfg.group_size)
    graph = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph):          # capture_error_mode="global"
        run_iteration(ctx, g, cfg, gb, src, mb=2, stream=torch.cuda.current_stream(), finalize="async")
    graph.replay()
    torch.cuda.synchronize()
    got = orl.orl_stats_decode(gb.final_dev.cpu().numpy(), cfg.ppo)
    eager = Buffers(B, T, DEV, cfg.group_size)
    want = run_iteration(ctx, g, cfg, eager, src, mb=2)
    assert got == want
    for k in KEYS:
        assert torch.equal(getattr(gb, k), getattr(eager, k)), k
    with pytest.raises(orl.OrlError):
        orl.orl_reserve(ctx, -1)
    ctx.close()
