"""Seeded synthetic rollouts shaped like the paper's workloads.

Shared by the tests, ``bench.py`` and ``__graft_entry__.smoke()``: this module
produces INPUTS only.  It holds none of the method's arithmetic (no softmax,
KL, GAE, whitening or loss), imports neither ``oracle`` nor the CUDA binding,
and both the oracle and the CUDA path consume what it returns.

Recipe (after SURVEY.md 8(d)):
  * target token y ~ U[0, V)
  * logits: old = X, ref = X + 0.1 N(0,1), new = X + 0.2 N(0,1), with a target
    boost b shared by the three roles added at index y;
      realistic: X = 1.0 N(0,1), b ~ U(12,20) with prob 0.9 else 0
                 (CoT-like: mostly confident tokens, ~10% "fork" tokens)
      stress:    X = 2.0 N(0,1), b ~ U(0,12)  (exercises the clip branches)
    then cast to bf16 with round-to-nearest-even (or kept fp32 for the tiny
    config).
  * values: V_old ~ N(0,1), V_new = V_old + 0.3 N(0,1)
  * rewards: N(0,1) (RM-like), Bernoulli(0.5) (verifiable), or per-group
    p_g ~ U(0,1), R ~ Bernoulli(p_g) (GRPO; yields some constant groups)
Seeds: per micro-batch mb and role r in {old=0, ref=1, new=2} the generator
seed is seed*1_000_003 + 7*mb + r.
"""
from __future__ import annotations

import numpy as np
import torch

ROLES = ("old", "ref", "new")

# BASELINE.json "configs", in order.  lengths: "full" = every L_b = T.
CONFIGS = {
    "tiny": dict(B=4, T=16, V=32, dtype="f32", adv_kind="gae", gamma=1.0, lam=0.95,
                 kl_est_reward="k1", beta_reward=0.1, eps_low=0.2, eps_high=0.2, eps_v=0.2,
                 c1=0.5, c2=0.01, whiten=True, rewards="normal", group_size=1, mb=4),
    "llama8b": dict(B=128, T=1024, V=128256, dtype="bf16", adv_kind="gae", gamma=1.0, lam=0.95,
                    kl_est_reward="k1", beta_reward=0.01, eps_low=0.2, eps_high=0.2, eps_v=0.2,
                    c1=0.5, c2=0.0, whiten=True, rewards="normal", group_size=1, mb=8),
    "longcot": dict(B=32, T=8192, V=152064, dtype="bf16", adv_kind="gae", gamma=1.0, lam=1.0,
                    kl_est_reward="k3", beta_reward=0.01, eps_low=0.2, eps_high=0.28, eps_v=0.2,
                    c1=0.5, c2=0.0, whiten=True, rewards="bernoulli", group_size=1, mb=4),
    "grpo": dict(B=2048, T=4096, V=128256, dtype="bf16", adv_kind="grpo", gamma=1.0, lam=1.0,
                 kl_mode="loss", kl_est_loss="k2", beta_loss=0.001, kl_est_reward="k1",
                 beta_reward=0.0, eps_low=0.2, eps_high=0.2, eps_v=0.0, c1=0.0, c2=0.0,
                 whiten=False, rewards="group_bernoulli", group_size=8, mb=8),
    "rpp8": dict(B=1024, T=2048, V=128256, dtype="bf16", adv_kind="rpp", gamma=1.0, lam=1.0,
                 kl_est_reward="k1", beta_reward=0.01, eps_low=0.2, eps_high=0.2, eps_v=0.0,
                 c1=0.0, c2=0.0, whiten=True, rewards="bernoulli", group_size=1, mb=16),
    # not a BASELINE.json config: the north star's target shape (V = 128256, T = 8192
    # rollouts), long-CoT settings of "longcot" on the Llama vocabulary; a bench leg only
    "target": dict(B=16, T=8192, V=128256, dtype="bf16", adv_kind="gae", gamma=1.0, lam=1.0,
                   kl_est_reward="k3", beta_reward=0.01, eps_low=0.2, eps_high=0.28, eps_v=0.2,
                   c1=0.5, c2=0.0, whiten=True, rewards="bernoulli", group_size=1, mb=4),
}
# SURVEY 8(d) secondary (ragged) lengths per config, for lengths_for()
SECONDARY_LENGTHS = {"tiny": "tiny", "llama8b": "mixed", "longcot": "cot", "grpo": "mixed", "rpp8": "mixed",
                     "target": "cot"}


def role_seed(seed: int, mb: int, role: int) -> int:
    return int(seed) * 1_000_003 + 7 * int(mb) + int(role)


def lengths_for(B: int, T: int, seed: int, mode: str = "full") -> torch.Tensor:
    """int32 [B] response lengths.  full: all T.  mixed: U{T//16..T} (SURVEY 8(d)
    secondary lengths: llama8b U{64..1024}, grpo U{256..4096}, rpp8 U{128..2048}).
    cot: long-CoT mix, 40% at T and the rest U{T//8..T} (longcot: U{1024..8192}).
    tiny: the hand-picked {T, 11/16 T, 5/16 T, 1} pattern plus a 0-length response."""
    if mode == "full":
        return torch.full((B,), T, dtype=torch.int32)
    if mode == "cot":
        g = torch.Generator().manual_seed(role_seed(seed, 10_000, 5))
        L = torch.randint(max(1, T // 8), T + 1, (B,), generator=g, dtype=torch.int32)
        full = torch.rand(B, generator=g) < 0.4
        return torch.where(full, torch.full_like(L, T), L)
    if mode == "tiny":
        pat = [T, max(1, (11 * T) // 16), max(1, (5 * T) // 16), 1, 0, T, max(1, T // 2), 3 % (T + 1)]
        return torch.tensor([pat[i % len(pat)] for i in range(B)], dtype=torch.int32)
    g = torch.Generator().manual_seed(role_seed(seed, 10_000, 5))
    lo = max(1, T // 16)
    return torch.randint(lo, T + 1, (B,), generator=g, dtype=torch.int32)


def tokens_for(B: int, T: int, V: int, seed: int, device="cpu") -> torch.Tensor:
    g = torch.Generator(device=device).manual_seed(role_seed(seed, 10_000, 3))
    return torch.randint(0, V, (B, T), generator=g, device=device, dtype=torch.int32)


def rewards_for(B: int, seed: int, kind: str, group_size: int = 1) -> torch.Tensor:
    g = torch.Generator().manual_seed(role_seed(seed, 10_000, 4))
    if kind == "normal":
        return torch.randn(B, generator=g, dtype=torch.float32)
    if kind == "bernoulli":
        return torch.bernoulli(torch.full((B,), 0.5), generator=g).float()
    if kind == "group_bernoulli":
        G = max(1, group_size)
        p = torch.rand(B // G, generator=g).repeat_interleave(G)
        return torch.bernoulli(p, generator=g).float()
    raise ValueError(kind)


def values_for(B: int, T: int, seed: int):
    g = torch.Generator().manual_seed(role_seed(seed, 10_000, 6))
    v_old = torch.randn(B, T, generator=g)
    v_new = v_old + 0.3 * torch.randn(B, T, generator=g)
    return v_old, v_new


@torch.no_grad()
def fill_logits_(bufs, tokens, seed: int, mb: int, mode: str = "realistic", chunk_rows: int = 1024):
    """Fill the three role buffers ([b,T,V], same shape, bf16 or fp32, any device)
    in place for micro-batch ``mb``.  Works in row chunks so no fp32 copy of a
    whole buffer is ever materialised."""
    old, ref, new = bufs
    b, T, V = old.shape
    dev = old.device
    g = torch.Generator(device=dev).manual_seed(role_seed(seed, mb, 0))
    g1 = torch.Generator(device=dev).manual_seed(role_seed(seed, mb, 1))
    g2 = torch.Generator(device=dev).manual_seed(role_seed(seed, mb, 2))
    scale = 1.0 if mode == "realistic" else 2.0
    ro, rr, rn = old.view(-1, V), ref.view(-1, V), new.view(-1, V)
    tok = tokens.reshape(-1).to(dev, torch.int64)
    n = ro.shape[0]
    for s in range(0, n, chunk_rows):
        e = min(n, s + chunk_rows)
        X = torch.randn(e - s, V, generator=g, device=dev) * scale
        if mode == "realistic":
            boost = torch.rand(e - s, generator=g, device=dev) * 8 + 12
            boost = boost * (torch.rand(e - s, generator=g, device=dev) < 0.9)
        else:
            boost = torch.rand(e - s, generator=g, device=dev) * 12
        idx = tok[s:e].unsqueeze(1)
        X.scatter_add_(1, idx, boost.unsqueeze(1))
        ro[s:e] = X
        rr[s:e] = X + 0.1 * torch.randn(e - s, V, generator=g1, device=dev)
        rn[s:e] = X + 0.2 * torch.randn(e - s, V, generator=g2, device=dev)
    return bufs


def to_numpy_logits(t: torch.Tensor) -> np.ndarray:
    """bf16 -> uint16 bit patterns (what the oracle reads); fp32 -> float32."""
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def make_batch(seed: int, B: int, T: int, V: int, dtype="f32", mode="realistic",
               lengths="tiny", rewards="normal", group_size=1, device="cpu"):
    """A whole rank-local batch as torch tensors (one micro-batch, mb=0)."""
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    L = lengths_for(B, T, seed, lengths) if isinstance(lengths, str) else torch.as_tensor(lengths, dtype=torch.int32)
    tok = tokens_for(B, T, V, seed)
    bufs = tuple(torch.empty(B, T, V, dtype=tdt, device=device) for _ in ROLES)
    fill_logits_(bufs, tok, seed, 0, mode)
    R = rewards_for(B, seed, rewards, group_size)
    v_old, v_new = values_for(B, T, seed)
    return dict(logits_old=bufs[0], logits_ref=bufs[1], logits_new=bufs[2], tokens=tok,
                lengths=L, seq_reward=R, values_old=v_old, values_new=v_new)


def batch_to_numpy(batch) -> dict:
    out = {}
    for k, v in batch.items():
        if k.startswith("logits_"):
            out[k] = to_numpy_logits(v)
        elif isinstance(v, torch.Tensor):
            out[k] = v.detach().cpu().numpy()
        else:
            out[k] = v
    return out


def tiny_numpy(seed: int, B=4, T=16, V=32, mode="stress", rewards="normal", group_size=1):
    return batch_to_numpy(make_batch(seed, B, T, V, "f32", mode, "tiny", rewards, group_size))


def split_bounds(B: int, n: int, group_size: int = 1):
    """Contiguous, group-aligned sequence blocks for n ranks."""
    G = max(1, group_size)
    if B % G:
        raise ValueError("batch is not a whole number of groups")
    ng = B // G
    cuts = [(ng * r // n) * G for r in range(n + 1)]
    return [(cuts[r], cuts[r + 1]) for r in range(n)]


def split_bounds_tokens(lengths, n: int, group_size: int = 1):
    """Contiguous, group-aligned rank shards balanced by valid tokens (SPEC S:468:
    shards "weighted by token counts"): rank r takes the groups whose
    token prefix midpoint falls in [r/n, (r+1)/n) of the total.  Sequence order is
    kept, so concatenating the shards gives the batch back."""
    L = np.clip(np.asarray(lengths, dtype=np.int64), 0, None)
    G = max(1, group_size)
    B = L.size
    if B % G:
        raise ValueError("batch is not a whole number of groups")
    if n < 1:
        raise ValueError("n >= 1")
    gt = L.reshape(-1, G).sum(axis=1).astype(np.float64)
    total = gt.sum()
    if total <= 0:
        return split_bounds(B, n, group_size)
    mid = np.cumsum(gt) - 0.5 * gt                  # token midpoint of each group
    owner = np.minimum((mid * n / total).astype(np.int64), n - 1)
    cuts = [0] + [int(np.searchsorted(owner, r, side="left")) * G for r in range(1, n)] + [B]
    if B // G >= n:                                  # every rank gets at least one group
        for r in range(1, n):
            cuts[r] = min(max(cuts[r], cuts[r - 1] + G), B - (n - r) * G)
    return [(cuts[r], cuts[r + 1]) for r in range(n)]


def split_numpy(batch: dict, n: int, group_size: int = 1):
    B = len(batch["lengths"])
    out = []
    for s, e in split_bounds(B, n, group_size):
        out.append({k: v[s:e] for k, v in batch.items()})
    return out


@torch.no_grad()
def make_lmhead_batch(seed: int, B: int, T: int, d: int, V: int, lengths="mixed", rewards="normal",
                      group_size: int = 1, packed: bool = False, device="cpu", logit_std: float = 3.0):
    """NEXT-4 inputs: final hidden states of the three roles and
    one bf16 LM-head weight.  Rows: b*T + t (padded) or packed by cu_seqlens (valid
    tokens only).  hidden_old = s_r N(0, I) with a per-row scale s_r ~ U(0.5, 1.5)
    (entropy varies by row), hidden_ref = hidden_old + 0.05 N, hidden_new =
    hidden_old + 0.03 N; W ~ N(0, logit_std^2 / d) so logits have std ~ logit_std s_r."""
    L = lengths_for(B, T, seed, lengths) if isinstance(lengths, str) else torch.as_tensor(lengths, dtype=torch.int32)
    tok = tokens_for(B, T, V, seed)
    if packed:
        cu = torch.zeros(B + 1, dtype=torch.int32)
        cu[1:] = torch.cumsum(L.clamp(0, T), 0)
        R = int(cu[-1])
    else:
        cu = None
        R = B * T
    R = max(R, 1)
    g = torch.Generator(device=device).manual_seed(role_seed(seed, 20_000, 0))
    base = torch.randn(R, d, generator=g, device=device)
    base *= torch.rand(R, 1, generator=g, device=device) + 0.5
    hid = {"old": base.to(torch.bfloat16),
           "ref": (base + 0.05 * torch.randn(R, d, generator=g, device=device)).to(torch.bfloat16),
           "new": (base + 0.03 * torch.randn(R, d, generator=g, device=device)).to(torch.bfloat16)}
    del base
    W = torch.empty(V, d, dtype=torch.bfloat16, device=device)
    for s in range(0, V, 8192):  # chunked: no fp32 copy of the whole matrix
        e = min(V, s + 8192)
        W[s:e] = (torch.randn(e - s, d, generator=g, device=device) * (logit_std / d ** 0.5)).to(torch.bfloat16)
    R_ = rewards_for(B, seed, rewards, group_size)
    v_old, v_new = values_for(B, T, seed)
    return dict(hidden_old=hid["old"], hidden_ref=hid["ref"], hidden_new=hid["new"], weight=W, tokens=tok,
                lengths=L, cu_seqlens=cu, seq_reward=R_, values_old=v_old, values_new=v_new)
