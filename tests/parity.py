"""Parity helpers shared by the GPU tests and __graft_entry__.smoke().

Tolerances (BASELINE.json north star):
  * bit-exact: gathered raw logits, masks (exact zeros), clip decisions,
    error counters;
  * log-probs / entropy / lse from bf16 logits: |gpu - oracle| <= 2e-3 absolute,
    with a regression alarm at 1e-4 (the kernel's real error is ~1e-6);
  * fp32 KL, rewards, advantages, returns, losses, gradients, stats:
    |g - o| <= 1e-5 * max(|o|, s) with s the RMS of the oracle values over the
    valid tokens (for per-token arrays) or the mean |term| (for means).
"""
from __future__ import annotations

import numpy as np

LOGP_ABS = 2e-3
LOGP_ALARM = 1e-4
REL = 1e-5


def valid_mask(lengths, T):
    L = np.asarray(lengths)
    return np.arange(T)[None, :] < L[:, None]


def check_masked_zero(name, g, mask):
    bad = g[~mask]
    assert np.all(bad == 0.0), f"{name}: masked positions are not exactly 0 ({np.count_nonzero(bad)})"


def check_abs(name, g, o, mask, tol=LOGP_ABS, alarm=LOGP_ALARM):
    d = np.abs(g[mask].astype(np.float64) - o[mask])
    mx = float(d.max()) if d.size else 0.0
    assert mx <= tol, f"{name}: max |gpu-oracle| = {mx:.3e} > {tol}"
    assert mx <= alarm, f"{name}: max |gpu-oracle| = {mx:.3e} above the {alarm} regression alarm"
    check_masked_zero(name, g, mask)
    return mx


def check_rel(name, g, o, mask=None, rel=REL, floor=None):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    if mask is not None:
        check_masked_zero(name, g, mask)
        g, o = g[mask], o[mask]
    if o.size == 0:
        return 0.0
    s = floor if floor is not None else float(np.sqrt(np.mean(o * o)))
    lim = rel * np.maximum(np.abs(o), s)
    err = np.abs(g - o)
    worst = float(np.max(err / np.maximum(lim, 1e-300)))
    assert np.all(err <= lim), f"{name}: worst err/limit = {worst:.3f} (rel {rel}, floor {s:.3e})"
    return worst


def check_stats(gpu: dict, ora: dict, ora_sums=None, rel=REL):
    """Compare the GPU stats dict with the oracle's (pipeline()[1]['stats'])."""
    N = ora["n_tokens"]
    assert gpu["n_tokens"] == N, (gpu["n_tokens"], N)
    for k in ("policy_loss", "value_loss", "entropy", "kl", "approx_kl_old", "ratio_mean", "total_loss"):
        o, g = ora[k], gpu[k]
        scale = max(abs(o), 1e-6)
        if ora_sums is not None and k == "policy_loss":
            scale = max(abs(o), 1e-3)
        assert abs(g - o) <= rel * max(scale, 1.0 if k == "ratio_mean" else scale), (k, g, o)
    for k in ("clip_frac", "value_clip_frac"):
        assert abs(gpu[k] - ora[k]) <= 1.0 / max(N, 1) + 1e-12, (k, gpu[k], ora[k])
