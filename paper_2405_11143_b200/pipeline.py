"""Host orchestration of one PPO/RLVR iteration on one rank through liborl.

Call order follows PAPER.md App. C: old-policy log-probs
 -> reference log-probs + KL-shaped reward -> advantages
 -> global normalisation (collective C1) -> actor pass with the
PPO loss -> statistics (collective C2).  Only launches and buffer
bookkeeping live here; the arithmetic is in liborl.so.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, NamedTuple, Optional, Union

import torch

from . import orl as _orl


@dataclass
class PathConfig:
    adv_kind: str = "gae"
    gamma: float = 1.0
    lam: float = 0.95
    group_size: int = 1
    whiten: bool = True
    kl_mode: str = "reward"          # "reward": beta k(old,ref) shapes r'; "loss": beta k(new,ref) in the loss
    kl_est_reward: str = "k1"
    beta_reward: float = 0.01
    inv_temp: float = 1.0
    use_ref: bool = True
    ppo: _orl.PPOConfig = field(default_factory=_orl.PPOConfig)

    @classmethod
    def from_synth(cls, c: dict) -> "PathConfig":
        kl_mode = c.get("kl_mode", "reward")
        return cls(adv_kind=c["adv_kind"], gamma=c["gamma"], lam=c["lam"], group_size=c.get("group_size", 1),
                   whiten=c["whiten"], kl_mode=kl_mode, kl_est_reward=c.get("kl_est_reward", "k1"),
                   beta_reward=c.get("beta_reward", 0.0) if kl_mode == "reward" else 0.0,
                   ppo=_orl.PPOConfig(eps_low=c["eps_low"], eps_high=c["eps_high"], eps_value=c["eps_v"],
                                      c1=c["c1"], c2=c["c2"], beta_loss=c.get("beta_loss", 0.0),
                                      kl_loss_est=c.get("kl_est_loss", "k2"), kl_in_loss=kl_mode == "loss",
                                      loss_agg=c.get("loss_agg", "token_mean")))

    @property
    def critic(self) -> bool:
        return self.adv_kind == "gae"


class Buffers:
    """Per-token [B,T] fp32 outputs of the rank-local batch (device)."""

    def __init__(self, B: int, T: int, device, group_size: int = 1, grads: bool = True):
        f = lambda: torch.zeros(B, T, dtype=torch.float32, device=device)  # noqa: E731
        self.logp_old, self.logp_ref, self.kl, self.shaped = f(), f(), f(), f()
        self.adv, self.ret, self.logp_new, self.entropy = f(), f(), f(), f()
        self.adv_lo = f()  # A - (float)A: the actor pass whitens adv + adv_lo (fp64-exact, Z33)
        self.lse = f()
        self.dlogp = f() if grads else None
        self.dv = f() if grads else None
        # per-token decisions of the actor pass: bit 0 clipped, 1 value-clipped, 2 guard, 3 non-finite
        self.flags = torch.zeros(B, T, dtype=torch.uint8, device=device)
        self.keep = torch.zeros(max(1, B // max(1, group_size)), dtype=torch.uint8, device=device)
        self.stats_dev = torch.zeros(_orl.STATS_N, dtype=torch.float64, device=device)
        self.final_dev = torch.zeros(_orl.FINAL_N, dtype=torch.float64, device=device)  # orl_finalize_async


class LmHeadRows(NamedTuple):
    """NEXT-4 source: a micro-batch's final hidden states [R, d] (row b*T + t, or packed
    by `cu_seqlens`) and the policy's LM-head weight [V, d], both bf16."""
    hidden: torch.Tensor
    weight: torch.Tensor
    cu_seqlens: Optional[torch.Tensor] = None


# (role, seq_start, seq_end) -> [e-s, T, V] logits, or LmHeadRows (NEXT-4)
LogitsSource = Callable[[str, int, int], Union[torch.Tensor, LmHeadRows]]


def microbatches(B: int, mb: int):
    return [(s, min(B, s + mb)) for s in range(0, B, mb)]


def run_iteration(ctx: _orl.Context, batch: dict, cfg: PathConfig, bufs: Buffers, logits: LogitsSource,
                  mb: int, stream: Optional[torch.cuda.Stream] = None, finalize: bool = True,
                  on_k1: Optional[Callable[[str], object]] = None,
                  grad_sink: Optional[Callable[[int, int], torch.Tensor]] = None, fused_grad: bool = True,
                  pdl_chain: Optional[bool] = None):
    """One iteration on this rank.  `batch` holds device tensors tokens [B,T] int32,
    lengths [B] int32, seq_reward [B] f32 and (critic) values_old / values_new [B,T].
    `on_k1(tag)` (optional) is called around every K1 launch for timing hooks.
    `grad_sink(s, e)` (optional, NEXT-1) returns the [e-s, T, V] dlogits view the
    backward pass (orl_logits_grad) writes for micro-batch [s, e).
    `pdl_chain` (optional) sets orl_set_pdl_chain for this iteration only: True is
    valid when the logits source launches no kernel that writes the logits with an
    early PDL trigger (resident tensors, slices, copies, plain torch kernels)."""
    if pdl_chain is None:
        return _run_iteration(ctx, batch, cfg, bufs, logits, mb, stream, finalize, on_k1, grad_sink, fused_grad)
    prev = ctx.pdl_chain
    ctx.pdl_chain = pdl_chain
    try:
        return _run_iteration(ctx, batch, cfg, bufs, logits, mb, stream, finalize, on_k1, grad_sink, fused_grad)
    finally:
        ctx.pdl_chain = prev


def _run_iteration(ctx, batch, cfg, bufs, logits, mb, stream, finalize, on_k1, grad_sink, fused_grad):
    tok, L = batch["tokens"], batch["lengths"]
    B, T = tok.shape
    mbs = microbatches(B, mb)
    hook = on_k1 or (lambda tag: None)
    nvtx = torch.cuda.nvtx.range                       # per-stage ranges for nsys / ncu --nvtx
    _orl.orl_begin_iteration(ctx, stream)

    def s1(src, s, e, out, **kw):
        if isinstance(src, LmHeadRows):               # NEXT-4: logits never materialised
            return _orl.orl_lmhead_logprobs(ctx, tok, L, src.hidden, src.weight, out, B=e - s, seq_offset=s,
                                            inv_temp=cfg.inv_temp, cu_seqlens=src.cu_seqlens, stream=stream,
                                            **kw)
        return _orl.orl_logprobs(ctx, tok, L, src, out, seq_offset=s, inv_temp=cfg.inv_temp, stream=stream,
                                 **kw)

    with nvtx("orl S1 old"):
        for s, e in mbs:                               # S1, old policy
            h = hook("old")
            s1(logits("old", s, e), s, e, bufs.logp_old)
            if h: h()
    if not cfg.use_ref:
        raise NotImplementedError("the paper's PPO loop always has a reference model (P:193)")
    with nvtx("orl S1-S3 ref"):
        for s, e in mbs:                               # S1+S2+S3, reference
            h = hook("ref")
            s1(logits("ref", s, e), s, e, bufs.logp_ref, partner_logp=bufs.logp_old, kl_est=cfg.kl_est_reward,
               beta_reward=cfg.beta_reward if cfg.kl_mode == "reward" else 0.0,
               seq_reward=batch["seq_reward"], kl=bufs.kl, shaped_reward=bufs.shaped)
            if h: h()
    with nvtx("orl S4-S6 advantages + C1"):
        _orl.orl_advantages(ctx, L, bufs.adv, kind=cfg.adv_kind, gamma=cfg.gamma, lam=cfg.lam,   # S4/S4'/S5
                            group_size=cfg.group_size, shaped_reward=bufs.shaped,
                            values=batch.get("values_old") if cfg.critic else None,
                            seq_reward=batch["seq_reward"], ret=bufs.ret,
                            group_keep=bufs.keep if cfg.adv_kind in ("grpo", "rpp_baseline") else None,
                            adv_lo=bufs.adv_lo, stream=stream)
        _orl.orl_whiten_stats(ctx, cfg.whiten and cfg.adv_kind != "grpo", stream)     # S6 + C1
    critic = cfg.critic and batch.get("values_new") is not None
    if grad_sink is not None and fused_grad:           # S1 + S7..S9 + NEXT-1 in one pass
        with nvtx("orl S1 S7-S9 actor + dL/dlogits"):
            _actor_fused(ctx, cfg, batch, bufs, logits, mbs, hook, grad_sink, critic, tok, L, stream)
        with nvtx("orl S10 + C2"):
            return _finish(ctx, cfg, bufs, stream, finalize)
    with nvtx("orl S1 S7-S9 actor"):
        _actor(ctx, cfg, batch, bufs, logits, mbs, hook, grad_sink, critic, tok, L, stream)
    with nvtx("orl S10 + C2"):
        return _finish(ctx, cfg, bufs, stream, finalize)                   # S10 + C2


def _no_lmhead(src):
    if isinstance(src, LmHeadRows):
        raise NotImplementedError("dL/dlogits needs materialised logits; the LM-head path (NEXT-4) is forward-only")
    return src


def _actor_fused(ctx, cfg, batch, bufs, logits, mbs, hook, grad_sink, critic, tok, L, stream):
    for s, e in mbs:
        h = hook("new+grad")
        _orl.orl_ppo_loss_and_grad(ctx, tok, L, _no_lmhead(logits("new", s, e)), cfg.ppo, bufs.logp_old, bufs.adv,
                                   bufs.logp_new, seq_offset=s, inv_temp=cfg.inv_temp, logp_ref=bufs.logp_ref,
                                   ret=bufs.ret if critic else None,
                                   v_new=batch["values_new"] if critic else None,
                                   v_old=batch["values_old"] if critic else None, entropy=bufs.entropy,
                                   lse=bufs.lse, dloss_dlogp=bufs.dlogp, dloss_dv=bufs.dv if critic else None,
                                   flags=bufs.flags, adv_lo=bufs.adv_lo, dlogits=grad_sink(s, e), stream=stream)
        if h: h()


def _actor(ctx, cfg, batch, bufs, logits, mbs, hook, grad_sink, critic, tok, L, stream):
    for s, e in mbs:                                   # S1 + S7..S9, actor
        h = hook("new")
        src = logits("new", s, e)
        kw = dict(seq_offset=s, inv_temp=cfg.inv_temp, logp_ref=bufs.logp_ref,
                  ret=bufs.ret if critic else None, v_new=batch["values_new"] if critic else None,
                  v_old=batch["values_old"] if critic else None, entropy=bufs.entropy,
                  lse=bufs.lse, dloss_dlogp=bufs.dlogp, dloss_dv=bufs.dv if critic else None, flags=bufs.flags,
                  adv_lo=bufs.adv_lo, stream=stream)
        if isinstance(src, LmHeadRows):
            if grad_sink is not None:
                _no_lmhead(src)
            _orl.orl_lmhead_ppo_loss(ctx, tok, L, src.hidden, src.weight, cfg.ppo, bufs.logp_old, bufs.adv,
                                     bufs.logp_new, B=e - s, cu_seqlens=src.cu_seqlens, **kw)
        else:
            _orl.orl_ppo_loss(ctx, tok, L, src, cfg.ppo, bufs.logp_old, bufs.adv, bufs.logp_new, **kw)
        if h: h()
    if grad_sink is not None:                          # NEXT-1: dL/dlogits
        for s, e in mbs:
            h = hook("grad")
            _orl.orl_logits_grad(ctx, tok, L, _no_lmhead(logits("new", s, e)), cfg.ppo, bufs.lse, bufs.entropy, bufs.dlogp,
                                 grad_sink(s, e), seq_offset=s, inv_temp=cfg.inv_temp, stream=stream)
            if h: h()


def _finish(ctx, cfg, bufs, stream, finalize):
    """finalize=True: orl_finalize (synchronises, returns (status, stats)); "async":
    orl_finalize_async into bufs.final_dev (no host sync, graph-capturable; decode later
    with orl_stats_decode); False: nothing."""
    if finalize == "async":
        _orl.orl_finalize_async(ctx, cfg.ppo, bufs.final_dev, stream=stream)
        return None
    if not finalize:
        return None
    return _orl.orl_finalize(ctx, cfg.ppo, dev_out=bufs.stats_dev, stream=stream)


class GraphStep:
    """A whole iteration (every launch of run_iteration, C1/C2 included) captured once
    into a CUDA graph and replayed with a single launch.  The logits source must return
    the same (resident) tensors every time; their contents may change between replays.
    The statistics land in bufs.final_dev; result() copies them to the host and decodes."""

    def __init__(self, ctx, batch: dict, cfg: PathConfig, bufs: Buffers, logits: LogitsSource, mb: int,
                 warmup: int = 1, pdl_chain: Optional[bool] = None):
        self.ctx, self.cfg, self.bufs = ctx, cfg, bufs
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):                   # eager warm-up sizes every workspace
            for _ in range(max(1, warmup)):
                run_iteration(ctx, batch, cfg, bufs, logits, mb, stream=side, finalize="async", pdl_chain=pdl_chain)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        l0 = ctx.launch_count
        with torch.cuda.graph(self.graph, capture_error_mode="relaxed"):
            run_iteration(ctx, batch, cfg, bufs, logits, mb, stream=torch.cuda.current_stream(),
                          finalize="async", pdl_chain=pdl_chain)
        self.kernels = ctx.launch_count - l0           # liborl kernels inside the graph

    def replay(self):
        self.graph.replay()

    def result(self):
        return _orl.orl_stats_decode(self.bufs.final_dev.cpu().numpy(), self.cfg.ppo)
