"""End-to-end oracle: the stages of orl_oracle.c composed in the paper's order.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md App. C (lines 189-201) orders one PPO iteration as: rollout records
log pi_theta_old -> reference log-probs + reward -> KL-shaped
reward, TD residuals, GAE, returns -> advantage normalisation
-> clipped surrogate + critic loss + entropy.  The batch is a list of
rank-local shards (contiguous sequence blocks); global quantities
(whitening moments, token count N, loss sums) are formed over ALL shards in
shard order, exactly as if the shards were one batch.
"""
from __future__ import annotations

import numpy as np

from . import (broadcast_seq, discounted_returns, gae, group_advantages, group_mean_subtract,
               logprobs, ppo_loss, shape_rewards, stats, whiten, whiten_moments)

DEFAULTS = dict(inv_temp=1.0, kl_mode="reward", kl_est_reward="k1", beta_reward=0.01,
                adv_kind="gae", gamma=1.0, lam=0.95, group_size=1, whiten=True,
                eps_low=0.2, eps_high=0.2, eps_v=0.2, c1=0.5, c2=0.0, beta_loss=0.0,
                kl_est_loss="k2", ratio_guard=30.0, loss_agg="token_mean")


def _s1(shard, role, inv_temp):
    if f"logp_{role}" in shard:          # stage isolation: upstream supplied
        return dict(logp=np.asarray(shard[f"logp_{role}"], np.float64),
                    entropy=np.asarray(shard.get(f"entropy_{role}", 0.0), np.float64))
    return logprobs(shard[f"logits_{role}"], shard["tokens"], shard["lengths"], inv_temp)


def pipeline(shards, cfg=None):
    cfg = {**DEFAULTS, **(cfg or {})}
    kind = cfg["adv_kind"]
    G = int(cfg["group_size"])
    out = []
    # ---- experience: S1 old/ref, S2+S3 shaping, S4/S4'/S5 advantages -------------
    for sh in shards:
        L = np.asarray(sh["lengths"], np.int64)
        R = np.asarray(sh["seq_reward"], np.float64)
        o = {}
        s_old = _s1(sh, "old", cfg["inv_temp"])
        o["logp_old"] = s_old["logp"]
        has_ref = ("logits_ref" in sh) or ("logp_ref" in sh)
        o["logp_ref"] = _s1(sh, "ref", cfg["inv_temp"])["logp"] if has_ref else None
        beta_r = cfg["beta_reward"] if (cfg["kl_mode"] == "reward" and has_ref) else 0.0
        ref_for_kl = o["logp_ref"] if has_ref else o["logp_old"]
        R_shape = group_mean_subtract(R, G) if kind == "rpp_baseline" else R
        o["kl"], o["shaped_reward"] = shape_rewards(L, o["logp_old"], ref_for_kl,
                                                    cfg["kl_est_reward"], beta_r, R_shape)
        T = o["logp_old"].shape[1]
        if kind == "gae":
            o["adv"], o["ret"] = gae(L, o["shaped_reward"], sh["values_old"], cfg["gamma"], cfg["lam"])
        elif kind in ("rpp", "rpp_baseline"):
            o["adv"] = discounted_returns(L, o["shaped_reward"], cfg["gamma"])
            o["ret"] = o["adv"]
        elif kind == "grpo":
            a_seq, keep = group_advantages(R, G)
            o["adv"] = broadcast_seq(L, a_seq, T)
            o["ret"] = None
            o["group_keep"] = keep
        else:
            raise ValueError(kind)
        out.append(o)

    # ---- S6 global whitening over all shards' valid tokens (shard order) ----------
    valid = np.concatenate([o["adv"][b, : int(L_b)] for o, sh in zip(out, shards)
                            for b, L_b in enumerate(sh["lengths"])] or [np.zeros(0)])
    n_global = float(valid.size)
    n_seq = float(sum(int(np.count_nonzero(np.asarray(sh["lengths"]) > 0)) for sh in shards))
    seq_mean = cfg["loss_agg"] == "seq_mean_token_mean"
    do_whiten = bool(cfg["whiten"]) and kind != "grpo"
    mean, std, warn = whiten_moments(valid)
    glob = dict(n_global=n_global, n_seq=n_seq, adv_mean=mean, adv_std=std, whiten_warn=warn and do_whiten)
    for o, sh in zip(out, shards):
        if do_whiten and not warn:
            o["adv_w"] = whiten(o["adv"], sh["lengths"], mean, std)
        else:
            o["adv_w"] = o["adv"]

    # ---- S7-S9 loss per shard, S10 sums in shard order ---------------------------
    sums = np.zeros(15)
    for o, sh in zip(out, shards):
        s_new = _s1(sh, "new", cfg["inv_temp"])
        o["logp_new"], o["entropy"] = s_new["logp"], s_new["entropy"]
        critic = sh.get("values_new") is not None and kind == "gae"
        res = ppo_loss(sh["lengths"], o["logp_new"], o["logp_old"], o["adv_w"],
                       logp_ref=o["logp_ref"], ret=o["ret"] if critic else None,
                       v_new=sh.get("values_new") if critic else None,
                       v_old=sh.get("values_old") if critic else None,
                       entropy=o["entropy"], eps_low=cfg["eps_low"], eps_high=cfg["eps_high"],
                       eps_v=cfg["eps_v"], c1=cfg["c1"] if critic else 0.0,
                       beta_loss=cfg["beta_loss"], kl_est=cfg["kl_est_loss"],
                       kl_in_loss=cfg["kl_mode"] == "loss" and o["logp_ref"] is not None,
                       ratio_guard=cfg["ratio_guard"], n_global=n_global, seq_mean=seq_mean, n_seq=n_seq)
        o.update(obj=res["obj"], clipped=res["clipped"], flags=res["flags"], vl=res["vl"], dlogp=res["dlogp"],
                 dv=res["dv"], sums=res["sums"])
        sums = sums + res["sums"]
    kl_in_loss = cfg["kl_mode"] == "loss" and out and out[0]["logp_ref"] is not None
    st = stats(sums, c1=cfg["c1"], c2=cfg["c2"], beta_loss=cfg["beta_loss"], kl_in_loss=kl_in_loss,
               seq_mean=seq_mean, n_seq=n_seq)
    glob.update(sums=sums, stats=st)
    return out, glob
