"""GPU parity: liborl.so (through the C ABI) vs the fp64 oracle on the same
seeded synthetic inputs.  Every test here needs a B200.

Stage isolation: each downstream stage is compared with the
oracle stage fed the GPU's own fp32 upstream outputs; the whole chain from
logits is also compared end to end on the tiny fp32 config.
"""
from __future__ import annotations

import importlib
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2405_11143_b200 import synth
from tests import parity

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2405_11143_b200 import orl
    from paper_2405_11143_b200.pipeline import Buffers, PathConfig, run_iteration

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def ctx():
    c = orl.Context(0)
    yield c
    c.close()


def _to_dev(batch):
    return {k: (v.to(DEV) if isinstance(v, torch.Tensor) else v) for k, v in batch.items()}


def _run(ctx, batch_dev, cfg, mb, grads=True, pdl_chain=None):
    B, T = batch_dev["tokens"].shape
    bufs = Buffers(B, T, DEV, cfg.group_size, grads=grads)
    src = lambda role, s, e: batch_dev[f"logits_{role}"][s:e]  # noqa: E731
    status, st = run_iteration(ctx, batch_dev, cfg, bufs, src, mb=mb, pdl_chain=pdl_chain)
    torch.cuda.synchronize()
    return status, st, bufs


def _np(t):
    return t.detach().cpu().numpy()


def _isolated_oracle(npb, bufs, ocfg):
    """Oracle downstream of S1, fed the GPU's fp32 log-probs / entropy."""
    sh = dict(npb)
    sh["logp_old"] = _np(bufs.logp_old).astype(np.float64)
    sh["logp_ref"] = _np(bufs.logp_ref).astype(np.float64)
    sh["logp_new"] = _np(bufs.logp_new).astype(np.float64)
    sh["entropy_new"] = _np(bufs.entropy).astype(np.float64)
    out, glob = oracle.pipeline([sh], ocfg)
    glob["isolated_input"] = (sh, dict(importlib.import_module("oracle.pipeline").DEFAULTS, **ocfg))
    return out, glob


def _isolated_loss(bufs, sh, ocfg, mask):
    """The oracle's loss stage fed the GPU's own fp32 upstream (logp_new/old/ref, adv + adv_lo,
    ret, entropy), whitened with the oracle's moments over the GPU's advantages.  Returns the
    oracle.ppo_loss result, the whitened advantages and the moments (mu, sd) or None."""
    L = sh["lengths"]
    f64 = lambda t: _np(t).astype(np.float64)  # noqa: E731
    adv = f64(bufs.adv) + f64(bufs.adv_lo)            # the value the actor pass whitens (Z33)
    kind = ocfg["adv_kind"]
    whiten = bool(ocfg["whiten"]) and kind != "grpo"
    Aw, mom = adv, None
    if whiten:
        mu, sd, warn = oracle.whiten_moments(adv[mask])
        if not warn:
            Aw, mom = oracle.whiten(adv, L, mu, sd), (mu, sd)
    critic = kind == "gae" and sh.get("values_new") is not None
    res = oracle.ppo_loss(L, f64(bufs.logp_new), f64(bufs.logp_old), Aw, logp_ref=f64(bufs.logp_ref),
                          ret=f64(bufs.ret) if critic else None, v_new=sh["values_new"] if critic else None,
                          v_old=sh["values_old"] if critic else None, entropy=f64(bufs.entropy),
                          eps_low=ocfg["eps_low"], eps_high=ocfg["eps_high"], eps_v=ocfg["eps_v"],
                          c1=ocfg["c1"] if critic else 0.0, beta_loss=ocfg["beta_loss"], kl_est=ocfg["kl_est_loss"],
                          kl_in_loss=ocfg["kl_mode"] == "loss", ratio_guard=ocfg["ratio_guard"])
    return res, Aw, mom


def _check_flags(bufs, sh, ocfg, mask, name):
    """Per-token decisions bit-exact: the loss stage of the
    oracle fed the GPU's own fp32 upstream (logp_new/old/ref, adv, ret, entropy; the
    whitening moments taken by the oracle over the GPU's fp32 advantages) vs the actor
    pass's flags output.  bit 0 clipped (Z16), 1 value-clipped (Z13), 2 ratio guard
    (Z22), 3 non-finite.  Tie bands (excluded and counted): rho within 1e-9 of a clip
    edge (fp64 exp may differ by an ulp), |A'| < 1e-12, |dold| within 1e-9 of the guard."""
    f64 = lambda t: _np(t).astype(np.float64)  # noqa: E731
    res, Aw, _ = _isolated_loss(bufs, sh, ocfg, mask)
    g, o = _np(bufs.flags).astype(np.int64), res["flags"].astype(np.int64)
    assert np.all(g[~mask] == 0), f"{name}: flags at masked positions"
    dold = f64(bufs.logp_new) - f64(bufs.logp_old)
    rho = np.exp(dold)
    tie_rho = (np.abs(rho - (1 - ocfg["eps_low"])) < 1e-9) | (np.abs(rho - (1 + ocfg["eps_high"])) < 1e-9)
    # A' == 0 exactly (constant GRPO groups) is decided identically on both sides; only a
    # tiny nonzero A' could flip sign between one- and two-pass whitening moments
    tie_p = tie_rho | ((np.abs(Aw) < 1e-12) & (Aw != 0))
    tie_g = np.abs(np.abs(dold) - ocfg["ratio_guard"]) < 1e-9
    for bit, tie in ((0, tie_p), (1, np.zeros_like(mask)), (2, tie_g), (3, np.zeros_like(mask))):
        sel = mask & ~tie
        gb, ob = (g >> bit) & 1, (o >> bit) & 1
        assert np.array_equal(gb[sel], ob[sel]), f"{name}: flag bit {bit} differs on {np.count_nonzero(gb[sel] != ob[sel])} tokens"
    assert np.count_nonzero(tie_p & mask) <= max(2, mask.sum() // 10000), f"{name}: too many policy ties"
    assert np.count_nonzero(tie_g & mask) <= 1
    return int(np.count_nonzero(o[mask] & 1)), int(np.count_nonzero(o[mask] & 2))


def _check_downstream(bufs, o, glob, st, mask, cfg_name, ppo_tol=parity.REL, raw_shaped=None):
    parity.check_rel("kl", _np(bufs.kl), o["kl"], mask)
    # RPP-baseline: the GPU shapes with the raw R_b and K3 subtracts mu_g at t = L_b - 1
    # (orl.h orl_advantages); the oracle shapes R_b - mu_g.  Compare the raw shaping then.
    parity.check_rel("shaped_reward", _np(bufs.shaped), o["shaped_reward"] if raw_shaped is None else raw_shaped,
                     mask)
    if raw_shaped is None:
        parity.check_rel("adv", _np(bufs.adv), o["adv"], mask)
        if o.get("ret") is not None:
            parity.check_rel("ret", _np(bufs.ret), o["ret"], mask)
    else:
        # RPP-baseline, S4' in isolation: the oracle's returns of the GPU's own fp32 shaped
        # rewards with mu_g subtracted at t = L_b - 1.  (From the log-probs, the oracle shapes
        # R_b - mu_g - beta k in fp64, while the S3 output the GPU hands to K3 holds the fp32
        # R_b - beta k: in a group of equal rewards the advantage is the KL shaping alone,
        # ~1e-6, and that fp32 rounding (<= 2^-24 |R_b|) is its resolution -- Z40.)
        L, Tn = glob["isolated_input"][0]["lengths"], mask.shape[1]
        R = glob["isolated_input"][0]["seq_reward"].astype(np.float64)
        G = glob["isolated_input"][1]["group_size"]
        mu = R - oracle.group_mean_subtract(R, G)
        r = _np(bufs.shaped).astype(np.float64)
        for b_ in range(len(L)):
            if L[b_] > 0:
                r[b_, L[b_] - 1] -= mu[b_]
        a_iso = oracle.discounted_returns(L, r, glob["isolated_input"][1]["gamma"])
        parity.check_rel("adv", _np(bufs.adv), a_iso, mask)
        if bufs.ret is not None and o.get("ret") is not None:
            parity.check_rel("ret", _np(bufs.ret), a_iso, mask)
        # the loss stage then in isolation too (fed the GPU's advantages)
        sh_, ocfg_ = glob["isolated_input"]
        res_, _, mom_ = _isolated_loss(bufs, sh_, ocfg_, mask)
        o = dict(o, dlogp=res_["dlogp"], obj=res_["obj"], vl=res_["vl"])
        iso_st = oracle.stats(res_["sums"], c1=0.0, c2=ocfg_["c2"], beta_loss=ocfg_["beta_loss"],
                              kl_in_loss=ocfg_["kl_mode"] == "loss")
        glob = dict(glob, stats=iso_st)
        if mom_ is not None:
            glob["adv_mean"], glob["adv_std"] = mom_
    parity.check_rel("dloss_dlogp", _np(bufs.dlogp), o["dlogp"], mask)
    if bufs.dv is not None:
        parity.check_rel("dloss_dv", _np(bufs.dv), o["dv"], mask)
    # per-token decisions (clip, value clip, guard, non-finite) bit-exact, every config
    if "isolated_input" in glob:
        _check_flags(bufs, *glob["isolated_input"], mask, cfg_name)
    lp_n, lp_o = _np(bufs.logp_new).astype(np.float64), _np(bufs.logp_old).astype(np.float64)
    rho = np.exp(lp_n - lp_o)
    tie = (np.abs(rho - 0.8) < 1e-6) | (np.abs(rho - 1.2) < 1e-6) | (np.abs(rho - 1.28) < 1e-6)
    gs, os_ = st, glob["stats"]
    assert gs["n_tokens"] == os_["n_tokens"]
    ntie = np.count_nonzero(tie & mask)
    for k in ("clip_frac", "value_clip_frac"):
        assert abs(gs[k] - os_[k]) <= 1e-12 + ntie / max(1, mask.sum()), (k, gs[k], os_[k])
    # scale floors: the mean |per-token term| of each statistic
    mabs = lambda a: float(np.mean(np.abs(a[mask]))) if mask.any() else 0.0  # noqa: E731
    floors = dict(policy_loss=mabs(o["obj"]), value_loss=mabs(o["vl"]), entropy=mabs(o["entropy"]),
                  kl=1e-6, approx_kl_old=1e-6, ratio_mean=1.0)
    floors["total_loss"] = sum(floors[k] for k in ("policy_loss", "value_loss", "entropy"))
    for k, fl in floors.items():
        g_, o_ = gs[k], os_[k]
        assert abs(g_ - o_) <= ppo_tol * max(abs(o_), fl), (k, g_, o_, fl)
    if os_["n_tokens"] >= 2 and gs["adv_std"]:
        for g_, o_ in ((gs["adv_mean"], glob["adv_mean"]), (gs["adv_std"], glob["adv_std"])):
            assert abs(g_ - o_) <= 1e-6 * max(1.0, abs(o_)), (g_, o_)


# --------------------------------------------------------------------------- tiny, end to end
@pytest.mark.parametrize("kind", ["gae", "rpp", "rpp_baseline", "grpo"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tiny_end_to_end_and_isolated(ctx, kind, seed):
    c = dict(synth.CONFIGS["tiny"])
    B = 8
    c.update(adv_kind=kind, group_size=2 if kind in ("grpo", "rpp_baseline") else 1)
    if kind == "grpo":
        c.update(kl_mode="loss", kl_est_loss="k2", beta_loss=0.05, whiten=False, eps_v=0.0, c1=0.0)
    if kind.startswith("rpp"):
        c.update(eps_v=0.0, c1=0.0)
    batch = synth.make_batch(seed, B, c["T"], c["V"], "f32", "stress", "tiny", c["rewards"])
    cfg = PathConfig.from_synth(c)
    status, st, bufs = _run(ctx, _to_dev(batch), cfg, mb=3)
    assert status == "ORL_OK", status
    npb = synth.batch_to_numpy(batch)
    m = parity.valid_mask(npb["lengths"], c["T"])
    # end to end from the fp32 logits
    out, glob = oracle.pipeline([npb], c)
    o = out[0]
    parity.check_abs("logp_old", _np(bufs.logp_old), o["logp_old"], m)
    parity.check_abs("logp_ref", _np(bufs.logp_ref), o["logp_ref"], m)
    parity.check_abs("logp_new", _np(bufs.logp_new), o["logp_new"], m)
    parity.check_abs("entropy", _np(bufs.entropy), o["entropy"], m)
    parity.check_rel("adv(e2e)", _np(bufs.adv), o["adv"], m, rel=1e-4)
    # stage isolation at the 1e-5 bar
    out_i, glob_i = _isolated_oracle(npb, bufs, c)
    raw = None
    if kind == "rpp_baseline":
        raw = oracle.shape_rewards(npb["lengths"], _np(bufs.logp_old), _np(bufs.logp_ref), c["kl_est_reward"],
                                   c["beta_reward"], npb["seq_reward"])[1]
    _check_downstream(bufs, out_i[0], glob_i, st, m, f"tiny-{kind}", raw_shaped=raw)
    if kind in ("grpo", "rpp_baseline"):
        keep = oracle.group_advantages(npb["seq_reward"], 2)[1]
        assert np.array_equal(_np(bufs.keep)[: B // 2], keep)


def test_tiny_gathered_bit_exact_and_lse(ctx):
    c = synth.CONFIGS["tiny"]
    batch = synth.make_batch(5, 8, 16, 32, "f32", "stress", "tiny")
    g = _to_dev(batch)
    B, T = 8, 16
    logp, ent, lse, gat = (torch.full((B, T), 7.0, device=DEV) for _ in range(4))
    orl.orl_begin_iteration(ctx)
    orl.orl_logprobs(ctx, g["tokens"], g["lengths"], g["logits_old"], logp, entropy=ent, lse=lse,
                     gathered=gat, inv_temp=1 / 0.7)
    torch.cuda.synchronize()
    npb = synth.batch_to_numpy(batch)
    o = oracle.logprobs(npb["logits_old"], npb["tokens"], npb["lengths"], 1 / 0.7)
    m = parity.valid_mask(npb["lengths"], T)
    assert np.array_equal(_np(gat)[m], o["gathered"][m].astype(np.float32))
    parity.check_abs("lse", _np(lse), o["lse"], m)
    parity.check_abs("logp", _np(logp), o["logp"], m)
    parity.check_abs("entropy", _np(ent), o["entropy"], m)


# --------------------------------------------------------------------------- bf16 mid size
def _gpu_batch(seed, B, T, V, lengths="mixed", rewards="normal", group_size=1, mode="realistic"):
    L = synth.lengths_for(B, T, seed, lengths)
    tok = synth.tokens_for(B, T, V, seed)
    bufs = tuple(torch.empty(B, T, V, dtype=torch.bfloat16, device=DEV) for _ in range(3))
    synth.fill_logits_(bufs, tok, seed, 0, mode)
    R = synth.rewards_for(B, seed, rewards, group_size)
    v_old, v_new = synth.values_for(B, T, seed)
    return dict(logits_old=bufs[0], logits_ref=bufs[1], logits_new=bufs[2], tokens=tok.to(DEV),
                lengths=L.to(DEV), seq_reward=R.to(DEV), values_old=v_old.to(DEV), values_new=v_new.to(DEV))


@pytest.mark.parametrize("mode", ["realistic", "stress"])
def test_mid_bf16_llama_vocab(ctx, mode):
    c = dict(synth.CONFIGS["llama8b"])
    B, T, V = 4, 256, c["V"]
    g = _gpu_batch(11, B, T, V, "mixed", mode=mode)
    cfg = PathConfig.from_synth(c)
    status, st, bufs = _run(ctx, g, cfg, mb=3)
    assert status == "ORL_OK"
    npb = synth.batch_to_numpy({k: v for k, v in g.items()})
    m = parity.valid_mask(npb["lengths"], T)
    for role, buf in (("old", bufs.logp_old), ("ref", bufs.logp_ref), ("new", bufs.logp_new)):
        o = oracle.logprobs(npb[f"logits_{role}"], npb["tokens"], npb["lengths"])
        parity.check_abs(f"logp_{role}", _np(buf), o["logp"], m)
        if role == "new":
            parity.check_abs("entropy", _np(bufs.entropy), o["entropy"], m)
    out_i, glob_i = _isolated_oracle(npb, bufs, c)
    _check_downstream(bufs, out_i[0], glob_i, st, m, f"mid-{mode}")


# --------------------------------------------------------------------------- full sizes, sampled
def _sampled_rows_check(g, bufs, n_rows=48, seed=0):
    """S1 at the full V on rows sampled across the batch, one by one."""
    L = _np(g["lengths"])
    B, T = g["tokens"].shape
    rng = np.random.default_rng(seed)
    valid = [(b, t) for b in range(B) for t in [0, int(L[b]) - 1, int(rng.integers(0, max(1, L[b])))] if L[b] > 0]
    pick = [valid[i] for i in rng.choice(len(valid), size=min(n_rows, len(valid)), replace=False)]
    tok = _np(g["tokens"])
    for role, buf in (("old", bufs.logp_old), ("ref", bufs.logp_ref), ("new", bufs.logp_new)):
        rows = torch.stack([g[f"logits_{role}"][b, t] for b, t in pick]).unsqueeze(1)
        x = synth.to_numpy_logits(rows)
        o = oracle.logprobs(x, np.array([[tok[b, t]] for b, t in pick], np.int32), np.ones(len(pick), np.int32))
        gv = np.array([[_np(buf)[b, t]] for b, t in pick])
        parity.check_abs(f"logp_{role}@full", gv, o["logp"], np.ones_like(gv, bool))
        if role == "new":
            gh = np.array([[_np(bufs.entropy)[b, t]] for b, t in pick])
            parity.check_abs("entropy@full", gh, o["entropy"], np.ones_like(gh, bool))


@pytest.mark.parametrize("name,B", [("llama8b", 128), ("longcot", 8), ("grpo", 16), ("rpp8", 16)])
def test_full_size_sampled(ctx, name, B):
    """BASELINE.json configs at their full T and V (llama8b also at its full B), in the
    launch configuration bench.py times (same micro-batch size)."""
    c = dict(synth.CONFIGS[name])
    T, V = c["T"], c["V"]
    free = torch.cuda.mem_get_info()[0]
    need = 3 * B * T * V * 2 * 1.05
    if need > free:
        pytest.skip(f"needs {need / 1e9:.0f} GB")
    g = _gpu_batch(1234, B, T, V, "full" if name == "llama8b" else "mixed", c["rewards"], c["group_size"])
    cfg = PathConfig.from_synth(c)
    # bench.py's launch configuration: its micro-batch size and PDL chaining between the K1 launches
    status, st, bufs = _run(ctx, g, cfg, mb=min(c["mb"], B), pdl_chain=True)
    assert status == "ORL_OK", status
    _sampled_rows_check(g, bufs)
    # downstream stages on the whole batch, oracle fed the GPU's fp32 upstream
    npb = {k: (v.detach().cpu().numpy() if isinstance(v, torch.Tensor) and not k.startswith("logits_") else v)
           for k, v in g.items() if not k.startswith("logits_")}
    m = parity.valid_mask(npb["lengths"], T)
    out_i, glob_i = _isolated_oracle(npb, bufs, c)
    _check_downstream(bufs, out_i[0], glob_i, st, m, name)
    del g
    torch.cuda.empty_cache()


# --------------------------------------------------------------------------- edge cases / errors
@pytest.mark.parametrize("path", ["unaligned_tma", "generic"])
def test_generic_path_unaligned_vocab(ctx, path, monkeypatch):
    """V = 50257 bf16 rows are not 16-byte multiples: by default the TMA kernel streams
    each row's 16-byte aligned interior and loads the head/tail elements singly;
    ORL_K1_NO_UNALIGNED_TMA selects the generic (non-TMA) kernel."""
    if path == "generic":
        monkeypatch.setenv("ORL_K1_NO_UNALIGNED_TMA", "1")
    B, T, V = 3, 40, 50257
    g = _gpu_batch(3, B, T, V, "mixed")
    # targets in the rows' unaligned heads and tails too
    g["tokens"][0, :8] = torch.arange(8, device=DEV, dtype=torch.int32)
    g["tokens"][1, :8] = torch.arange(V - 8, V, device=DEV, dtype=torch.int32)
    cfg = PathConfig.from_synth(dict(synth.CONFIGS["llama8b"], V=V))
    status, st, bufs = _run(ctx, g, cfg, mb=2)
    assert status == "ORL_OK"
    npb = synth.batch_to_numpy(g)
    m = parity.valid_mask(npb["lengths"], T)
    o = oracle.logprobs(npb["logits_new"], npb["tokens"], npb["lengths"])
    parity.check_abs("logp_new", _np(bufs.logp_new), o["logp"], m)
    parity.check_abs("entropy", _np(bufs.entropy), o["entropy"], m)


@pytest.mark.parametrize("dtype,V,pad", [("bf16", 50257, 0), ("bf16", 32000, 3), ("f32", 50257, 0),
                                         ("f32", 1001, 1), ("bf16", 33, 0)])
def test_unaligned_tma_matches_generic_and_oracle(ctx, monkeypatch, dtype, V, pad):
    """Unaligned rows through the TMA kernel (aligned interior + scalar head/tail) vs the
    generic kernel and the oracle; gathered raw logits bit-exact; targets placed in
    heads and tails; a +80 spike in a head forces the scalar rescale."""
    B, T = 3, 24
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = torch.randn(B, T, V + pad, device=DEV) * 2
    x[0, 3, 1] = 80.0
    x = x.to(tdt)[..., :V]
    tok = synth.tokens_for(B, T, V, 5).to(DEV)
    tok[0, :4] = torch.tensor([0, 1, 2, 3], dtype=torch.int32, device=DEV)
    tok[1, :4] = torch.tensor([V - 1, V - 2, V - 3, V - 4], dtype=torch.int32, device=DEV) % V
    L = torch.tensor([T, T - 5, 7], dtype=torch.int32, device=DEV)
    outs = {}
    for mode in ("tma", "generic"):
        if mode == "generic":
            monkeypatch.setenv("ORL_K1_NO_UNALIGNED_TMA", "1")
        o = {k: torch.full((B, T), 7.0, device=DEV) for k in ("logp", "entropy", "lse", "gathered")}
        orl.orl_begin_iteration(ctx)
        orl.orl_logprobs(ctx, tok, L, x, o["logp"], entropy=o["entropy"], lse=o["lse"], gathered=o["gathered"],
                         inv_temp=1 / 0.7)
        torch.cuda.synchronize()
        outs[mode] = {k: _np(v) for k, v in o.items()}
    monkeypatch.delenv("ORL_K1_NO_UNALIGNED_TMA")
    xn = x.float().cpu().numpy() if dtype == "f32" else synth.to_numpy_logits(x)
    ora = oracle.logprobs(xn, _np(tok), _np(L), 1 / 0.7)
    m = parity.valid_mask(_np(L), T)
    for mode in ("tma", "generic"):
        for k in ("logp", "entropy", "lse"):
            parity.check_abs(f"{mode} {k}", outs[mode][k], ora[k], m)
        assert np.array_equal(outs[mode]["gathered"][m], ora["gathered"][m].astype(np.float32)), mode
    np.testing.assert_allclose(outs["tma"]["logp"][m], outs["generic"]["logp"][m], atol=2e-6)


def test_forced_generic_matches_tma(ctx, monkeypatch):
    B, T, V = 2, 64, 4096
    g = _gpu_batch(4, B, T, V, "mixed")
    cfg = PathConfig.from_synth(dict(synth.CONFIGS["llama8b"], V=V))
    _, st1, b1 = _run(ctx, g, cfg, mb=2)
    monkeypatch.setenv("ORL_FORCE_GENERIC", "1")
    _, st2, b2 = _run(ctx, g, cfg, mb=2)
    m = parity.valid_mask(_np(g["lengths"]), T)
    np.testing.assert_allclose(_np(b1.logp_new)[m], _np(b2.logp_new)[m], atol=2e-6)
    np.testing.assert_allclose(_np(b1.entropy)[m], _np(b2.entropy)[m], atol=2e-5)


def test_strided_response_aligned_view(ctx):
    """Logits of full sequences (prompt + response), sliced at prompt_len - 1 (Z1)."""
    B, P, T, V = 3, 5, 24, 1024
    full = torch.randn(B, P + T, V, device=DEV).to(torch.bfloat16)
    view = full[:, P - 1:P - 1 + T, :]
    tok = synth.tokens_for(B, T, V, 9).to(DEV)
    L = torch.tensor([24, 10, 1], dtype=torch.int32, device=DEV)
    logp = torch.zeros(B, T, device=DEV)
    orl.orl_begin_iteration(ctx)
    orl.orl_logprobs(ctx, tok, L, view, logp)
    torch.cuda.synchronize()
    o = oracle.logprobs(synth.to_numpy_logits(view), _np(tok), _np(L))
    parity.check_abs("logp(view)", _np(logp), o["logp"], parity.valid_mask(_np(L), T))


def test_neg_inf_entries_and_errors(ctx):
    B, T, V = 2, 8, 2048
    x = torch.randn(B, T, V, device=DEV) * 2
    x[0, 1, 100:700] = float("-inf")             # allowed (Z26)
    x[0, 2, :] = float("-inf")                   # whole row -inf: non-finite
    x[1, 3, 5] = float("nan")                    # NaN logit: non-finite
    xb = x.to(torch.bfloat16)
    tok = synth.tokens_for(B, T, V, 2).to(DEV)
    tok[0, 1] = 3                                # target not at a -inf entry
    tok[1, 5] = V + 7                            # out of vocabulary
    L = torch.tensor([8, 8], dtype=torch.int32, device=DEV)
    logp, ent = torch.zeros(B, T, device=DEV), torch.zeros(B, T, device=DEV)
    orl.orl_begin_iteration(ctx)
    orl.orl_logprobs(ctx, tok, L, xb, logp, entropy=ent)
    torch.cuda.synchronize()
    o = oracle.logprobs(synth.to_numpy_logits(xb), _np(tok), _np(L))
    lp, en = _np(logp), _np(ent)
    ok = np.ones((B, T), bool)
    ok[0, 2] = ok[1, 3] = ok[1, 5] = False
    parity.check_abs("logp", np.where(ok, lp, 0), np.where(ok, o["logp"], 0), ok)
    parity.check_abs("entropy", np.where(ok, en, 0), np.where(ok, o["entropy"], 0), ok)
    assert np.isnan(lp[0, 2]) and np.isnan(lp[1, 3]) and np.isnan(lp[1, 5])
    status, st = orl.orl_finalize(ctx, orl.PPOConfig())
    assert status == "ORL_E_TOKEN_RANGE"
    assert st["n_token_range"] == 1 and st["n_nonfinite"] == 2


@pytest.mark.parametrize("V", [128256, 50257])
def test_extreme_rows_overflow_redo_path(ctx, V):
    """Rows that force the fast path's exact redo (an element > the thread's seed max +
    64 log2 units, SURVEY 8(c) S1 pins): +60 / +1000 spikes at non-target and target
    positions (after each thread's first vector), a +1e4 spike, a uniform row, a row at
    -1e30 except the target, a very negative spike, wide +-50 noise; TMA (V = 128256)
    and generic (V = 50257) paths; inv_temp 1 and 1/0.7."""
    B, T = 2, 8
    x = torch.randn(B, T, V, device=DEV)
    tok = synth.tokens_for(B, T, V, 9).to(DEV)
    tgt = lambda b, t: int(tok[b, t])  # noqa: E731
    far = lambda b, t: (tgt(b, t) + V // 2) % V  # noqa: E731
    x[0, 0, far(0, 0)] = 60.0
    x[0, 1, far(0, 1)] = 1000.0
    x[0, 2, tgt(0, 2)] = 80.0
    x[0, 3, far(0, 3)] = 1.0e4
    x[0, 4, :] = 0.0
    x[0, 5, :] = -1.0e30
    x[0, 5, tgt(0, 5)] = 0.0
    x[0, 6, far(0, 6)] = -1.0e4
    x[0, 7] = (torch.rand(V, device=DEV) - 0.5) * 100.0
    x[1, 0, V - 1] = 200.0                            # spike in the last (tail) element
    x[1, 1, :64] = 90.0                               # spikes inside the first vectors
    xb = x.to(torch.bfloat16)
    L = torch.tensor([T, T], dtype=torch.int32, device=DEV)
    for inv_temp in (1.0, 1 / 0.7):
        logp, ent, lse = (torch.zeros(B, T, device=DEV) for _ in range(3))
        orl.orl_begin_iteration(ctx)
        orl.orl_logprobs(ctx, tok, L, xb, logp, entropy=ent, lse=lse, inv_temp=inv_temp)
        torch.cuda.synchronize()
        o = oracle.logprobs(synth.to_numpy_logits(xb), _np(tok), _np(L), inv_temp)
        m = np.ones((B, T), bool)
        for name, g in (("logp", logp), ("entropy", ent), ("lse", lse)):
            # the 2e-3 bar everywhere; the 1e-4 alarm scaled by the fp32 output format at these
            # magnitudes (|logp| up to 1.4e4 here, whose fp32 ulp is ~1e-3)
            parity.check_abs(f"{name} (inv_temp {inv_temp:.3f})", _np(g), o[name], m, alarm=parity.LOGP_ABS)
            err = np.abs(_np(g).astype(np.float64) - o[name])
            assert np.all(err <= np.maximum(parity.LOGP_ALARM, 4 * 2.0 ** -24 * np.abs(o[name]))), (name, err.max())
        status, st = orl.orl_finalize(ctx, orl.PPOConfig())
        assert st["n_nonfinite"] == 0 and st["n_token_range"] == 0, st


def test_logits_beyond_fp32_range_are_flagged(ctx):
    """Reading Z34: a finite bf16 logit whose scaled value x * inv_temp * log2(e) exceeds
    the fp32 range (|x| >~ 2.4e38 at inv_temp = 1) cannot be represented by the kernel:
    a large positive one makes the row NaN and counts as non-finite (never a silent wrong
    value); a large negative one is an exp of -inf, i.e. an ordinary zero-probability entry."""
    for V in (128256, 50257):
        B, T = 1, 4
        x = torch.randn(B, T, V, device=DEV)
        tok = synth.tokens_for(B, T, V, 3).to(DEV)
        x[0, 0, (int(tok[0, 0]) + 7) % V] = 3.0e38
        x[0, 1, int(tok[0, 1])] = 3.0e38
        x[0, 2, (int(tok[0, 2]) + 5) % V] = -3.0e38
        xb = x.to(torch.bfloat16)
        L = torch.tensor([T], dtype=torch.int32, device=DEV)
        logp, ent = torch.zeros(B, T, device=DEV), torch.zeros(B, T, device=DEV)
        orl.orl_begin_iteration(ctx)
        orl.orl_logprobs(ctx, tok, L, xb, logp, entropy=ent)
        torch.cuda.synchronize()
        lp = _np(logp)
        assert np.isnan(lp[0, 0]) and np.isnan(lp[0, 1])
        o = oracle.logprobs(synth.to_numpy_logits(xb), _np(tok), _np(L))
        ok = np.array([[False, False, True, True]])
        parity.check_abs("logp", np.where(ok, lp, 0), np.where(ok, o["logp"], 0), ok)
        status, st = orl.orl_finalize(ctx, orl.PPOConfig())
        assert status == "ORL_E_NONFINITE" and st["n_nonfinite"] == 2


def test_ratio_guard_and_empty_batch(ctx):
    B, T, V = 2, 4, 256
    x = torch.randn(B, T, V, device=DEV)
    tok = synth.tokens_for(B, T, V, 1).to(DEV)
    L = torch.tensor([4, 0], dtype=torch.int32, device=DEV)
    z = lambda: torch.zeros(B, T, device=DEV)  # noqa: E731
    lo, adv, lpn = z(), z(), z()
    lo[0, 2] = -60.0                              # |logp_new - logp_old| > 30
    orl.orl_begin_iteration(ctx)
    orl.orl_advantages(ctx, L, adv, kind="rpp", gamma=1.0, shaped_reward=z())
    orl.orl_whiten_stats(ctx, False)
    orl.orl_ppo_loss(ctx, tok, L, x, orl.PPOConfig(), lo, adv, lpn)
    status, st = orl.orl_finalize(ctx, orl.PPOConfig())
    assert status == "ORL_E_NUMERIC_GUARD" and st["n_guard"] == 1 and st["n_tokens"] == 4
    L0 = torch.zeros(B, dtype=torch.int32, device=DEV)
    orl.orl_begin_iteration(ctx)
    orl.orl_advantages(ctx, L0, adv, kind="rpp", gamma=1.0, shaped_reward=z())
    orl.orl_whiten_stats(ctx, True)
    orl.orl_ppo_loss(ctx, tok, L0, x, orl.PPOConfig(), lo, adv, lpn)
    status, st = orl.orl_finalize(ctx, orl.PPOConfig())
    assert status == "ORL_E_EMPTY_BATCH" and st["whiten_warn"] == 1
    assert torch.all(lpn == 0) and torch.all(adv == 0)


def test_host_argument_errors(ctx):
    B, T, V = 2, 4, 64
    x = torch.randn(B, T, V, device=DEV)
    tok = torch.zeros(B, T, dtype=torch.int32, device=DEV)
    L = torch.full((B,), T, dtype=torch.int32, device=DEV)
    lp = torch.zeros(B, T, device=DEV)
    with pytest.raises(orl.OrlError) as e:
        orl.orl_logprobs(ctx, tok, L, x, lp, inv_temp=0.0)
    assert e.value.name == "ORL_E_INVALID_ARG"
    with pytest.raises(orl.OrlError) as e:
        orl.orl_logprobs(ctx, tok, L, x, lp, kl=lp)
    assert e.value.name == "ORL_E_INVALID_ARG"
    with pytest.raises(orl.OrlError) as e:
        orl.orl_advantages(ctx, L, lp, kind="grpo", group_size=3, seq_reward=L.float())
    assert e.value.name == "ORL_E_GROUP_SPLIT"
    orl.orl_begin_iteration(ctx)
    with pytest.raises(orl.OrlError) as e:
        orl.orl_ppo_loss(ctx, tok, L, x, orl.PPOConfig(), lp, lp, lp)
    assert e.value.name == "ORL_E_STATE"
    with pytest.raises(TypeError):
        orl.orl_logprobs(ctx, tok, L, x.to(torch.float16), lp)

    # the C ABI itself: a per-token array 2 bytes off a 4-byte boundary (the binding only
    # hands over tensor pointers, so call liborl directly)
    import ctypes
    rows, lg = orl._rows(tok, L, tok.shape[0], tok.shape[1], 0), orl._logits(x)
    st = orl._lib.orl_logprobs(ctx.h, ctypes.byref(rows), ctypes.byref(lg), 1.0, ctypes.c_void_p(lp.data_ptr() + 2),
                               None, None, None, None, 1, 0.0, None, None, None, None)
    assert orl.STATUS[st] == "ORL_E_ALIGN"
    # a logits row of 2 GiB or more (V * element size >= 2^31) is rejected before any access:
    # the kernels keep row offsets in 32 bits (orl.h, orl_logits.V)
    for dtype, V_big in ((0, 1 << 30), (1, 1 << 29)):   # ORL_BF16, ORL_F32
        big = orl.Logits(x.data_ptr(), dtype, 0, V_big, V_big, V_big)
        st = orl._lib.orl_logprobs(ctx.h, ctypes.byref(rows), ctypes.byref(big), 1.0, ctypes.c_void_p(lp.data_ptr()),
                                   None, None, None, None, 1, 0.0, None, None, None, None)
        assert orl.STATUS[st] == "ORL_E_SHAPE", (dtype, orl.STATUS[st])


# --------------------------------------------------------------------------- determinism / DP
def test_run_to_run_bit_reproducible(ctx):
    c = dict(synth.CONFIGS["llama8b"])
    g = _gpu_batch(21, 6, 128, 8192, "mixed")
    cfg = PathConfig.from_synth(c)
    _, s1, b1 = _run(ctx, g, cfg, mb=4)
    _, s2, b2 = _run(ctx, g, cfg, mb=4)
    assert s1 == s2
    for k in ("logp_old", "logp_ref", "logp_new", "entropy", "adv", "ret", "dlogp"):
        assert torch.equal(getattr(b1, k), getattr(b2, k)), k


@pytest.mark.parametrize("kind,n", [("gae", 2), ("rpp", 4), ("grpo", 2), ("gae", 8), ("grpo", 4)])
def test_shard_emulation_matches_single_rank(kind, n):
    """n virtual ranks on one GPU, partials exchanged through the collective
    boundary hooks (the exact device merges NCCL feeds), vs one rank."""
    B, T, V = 8, 64, 2048
    c = dict(synth.CONFIGS["llama8b"], adv_kind=kind, group_size=2 if kind == "grpo" else 1)
    if kind == "grpo":
        c.update(kl_mode="loss", beta_loss=0.01, whiten=False, eps_v=0.0, c1=0.0)
    cfg = PathConfig.from_synth(c)
    g = _gpu_batch(31, B, T, V, "mixed", "group_bernoulli" if kind == "grpo" else "normal", 2)
    one = orl.Context(0)
    _, st1, b1 = _run(one, g, cfg, mb=3)
    bounds = synth.split_bounds(B, n, c["group_size"])
    ctxs = [orl.Context(0) for _ in bounds]
    shard_bufs = []
    for cx, (s, e) in zip(ctxs, bounds):
        gs = {k: v[s:e] for k, v in g.items()}
        bb = Buffers(e - s, T, DEV, c["group_size"])
        src = lambda role, a, z, gs=gs: gs[f"logits_{role}"][a:z]  # noqa: E731
        # experience half up to the advantages
        orl.orl_begin_iteration(cx)
        for a, z in [(a, min(e - s, a + 3)) for a in range(0, e - s, 3)]:
            orl.orl_logprobs(cx, gs["tokens"], gs["lengths"], src("old", a, z), bb.logp_old, seq_offset=a)
        for a, z in [(a, min(e - s, a + 3)) for a in range(0, e - s, 3)]:
            orl.orl_logprobs(cx, gs["tokens"], gs["lengths"], src("ref", a, z), bb.logp_ref, seq_offset=a,
                             partner_logp=bb.logp_old, kl_est=cfg.kl_est_reward,
                             beta_reward=cfg.beta_reward, seq_reward=gs["seq_reward"], kl=bb.kl,
                             shaped_reward=bb.shaped)
        orl.orl_advantages(cx, gs["lengths"], bb.adv, kind=kind, gamma=cfg.gamma, lam=cfg.lam,
                           group_size=cfg.group_size, shaped_reward=bb.shaped,
                           values=gs["values_old"] if cfg.critic else None, seq_reward=gs["seq_reward"],
                           ret=bb.ret, adv_lo=bb.adv_lo)
        shard_bufs.append((gs, bb, src))
    wparts = np.stack([orl.orl_export_partials(cx, 0) for cx in ctxs])
    for cx in ctxs:
        orl.orl_import_partials(cx, 0, wparts)
        orl.orl_whiten_stats(cx, cfg.whiten and kind != "grpo")
    for cx, (gs, bb, src) in zip(ctxs, shard_bufs):
        Bs = gs["tokens"].shape[0]
        for a, z in [(a, min(Bs, a + 3)) for a in range(0, Bs, 3)]:
            crit = cfg.critic
            orl.orl_ppo_loss(cx, gs["tokens"], gs["lengths"], src("new", a, z), cfg.ppo, bb.logp_old, bb.adv,
                             bb.logp_new, seq_offset=a, logp_ref=bb.logp_ref, ret=bb.ret if crit else None,
                             v_new=gs["values_new"] if crit else None, v_old=gs["values_old"] if crit else None,
                             entropy=bb.entropy, dloss_dlogp=bb.dlogp, adv_lo=bb.adv_lo)
    sparts = np.stack([orl.orl_export_partials(cx, 1) for cx in ctxs])
    res = []
    for cx in ctxs:
        orl.orl_import_partials(cx, 1, sparts)
        res.append(orl.orl_finalize(cx, cfg.ppo))
    for status, st in res:
        assert status == "ORL_OK"
        assert st == res[0][1]                      # every rank bit-identical
        for k, v in st1.items():
            if isinstance(v, float):
                assert abs(st[k] - v) <= 1e-12 * max(1.0, abs(v)), (k, st[k], v)
    for (s, e), (gs, bb, _) in zip(bounds, shard_bufs):
        assert torch.equal(bb.logp_new, b1.logp_new[s:e])
        assert torch.equal(bb.adv, b1.adv[s:e])
        torch.testing.assert_close(bb.dlogp, b1.dlogp[s:e], rtol=1e-6, atol=1e-12)
    for cx in ctxs + [one]:
        cx.close()


# --------------------------------------------------------------------------- NEXT-1
def _check_grad(g, o, mask_rows, rel, name, w, H, a, inv_temp):
    """|gpu - oracle| <= rel |o| + 1e-5 S_row, S_row = inv_temp (|w| + a (1 + H)) bounds the
    size of the two terms of dL/dz_v before they cancel (fp32 w, H, lse carry ~1e-7)."""
    for (b, t) in zip(*np.nonzero(mask_rows)):
        gr, orow = g[b, t].astype(np.float64), o[b, t]
        S = inv_temp * (abs(w[b, t]) + a * (1.0 + abs(H[b, t])))
        err = np.abs(gr - orow)
        lim = rel * np.abs(orow) + 1e-5 * S
        assert np.all(err <= lim), (name, b, t, float((err / lim).max()))
        assert abs(gr.sum()) <= (1e-4 if rel < 1e-3 else 1e-2) * np.abs(gr).sum() + 1e-6 * S  # shift invariance
    for (b, t) in zip(*np.nonzero(~mask_rows)):
        assert np.all(g[b, t] == 0), (name, "masked row not zero")


@pytest.mark.parametrize("dtype,V,inv_temp", [("f32", 32, 1.0), ("f32", 1000, 1 / 0.7), ("bf16", 4096, 1.0),
                                               ("bf16", 50257, 1.0)])
def test_next1_logits_grad_parity(ctx, dtype, V, inv_temp):
    """dL/dlogits from the GPU backward pass vs the oracle's, fed the GPU's own
    saved per-token quantities (dloss_dlogp) -- stage isolation."""
    B, T = 4, 24
    c = dict(synth.CONFIGS["llama8b"], c2=0.01, V=V, inv_temp=inv_temp)
    if dtype == "f32":
        batch = synth.make_batch(7, B, T, V, "f32", "stress", "tiny")
        g = _to_dev(batch)
    else:
        g = _gpu_batch(7, B, T, V, "mixed", mode="stress")
    cfg = PathConfig.from_synth(c)
    cfg.inv_temp = inv_temp
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    dl = torch.full((B, T, V), 3.0, dtype=tdt, device=DEV)
    bufs = Buffers(B, T, DEV)
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    status, st = run_iteration(ctx, g, cfg, bufs, src, mb=3, grad_sink=lambda s, e: dl[s:e])
    torch.cuda.synchronize()
    assert status == "ORL_OK"
    npb = synth.batch_to_numpy(g)
    m = parity.valid_mask(npb["lengths"], T)
    o = oracle.logits_grad(npb["logits_new"], npb["tokens"], npb["lengths"], _np(bufs.dlogp).astype(np.float64),
                           inv_temp, 0.01, float(m.sum()))
    gg = dl.float().cpu().numpy()
    H = oracle.logprobs(npb["logits_new"], npb["tokens"], npb["lengths"], inv_temp)["entropy"]
    _check_grad(gg, o, m, 2e-5 if dtype == "f32" else 8e-3, f"{dtype}-{V}", _np(bufs.dlogp), H,
                0.01 / float(m.sum()), inv_temp)


@pytest.mark.parametrize("c2", [0.01, 0.0])
@pytest.mark.parametrize("fused", [True, False])
def test_next1_masked_vocab_entries(ctx, fused, c2):
    """Vocabulary entries masked in the actor logits (Z39): a -inf logit has p = 0; with an
    entropy term (c2 != 0) the formula's p (ln p + H) is 0 * (-inf), so its gradient element
    is NaN on both sides (GPU and the fp64 oracle), without one (c2 = 0) it is -w p = 0 on
    both sides; a large finite negative logit (-1e30, the documented mask value) gets an
    exact zero gradient; every other element stays finite and matches the oracle."""
    B, T, V = 3, 16, 2176
    c = dict(synth.CONFIGS["llama8b"], c2=c2, V=V)
    g = _gpu_batch(17, B, T, V, "mixed", mode="realistic")
    x = g["logits_new"]
    tok = g["tokens"].long()
    gen = torch.Generator(device="cpu").manual_seed(5)
    masked = torch.rand(B, T, V, generator=gen) < 0.05
    kind = torch.rand(B, T, V, generator=gen) < 0.5          # half -inf, half -1e30
    masked.scatter_(2, tok.cpu().unsqueeze(-1), False)       # never the sampled token
    neg_inf = (masked & kind).to(DEV)
    neg_big = (masked & ~kind).to(DEV)
    x[neg_inf] = float("-inf")
    x[neg_big] = -1e30
    cfg = PathConfig.from_synth(c)
    dl = torch.full((B, T, V), 3.0, dtype=torch.bfloat16, device=DEV)
    bufs = Buffers(B, T, DEV)
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    status, st = run_iteration(ctx, g, cfg, bufs, src, mb=2, grad_sink=lambda s, e: dl[s:e], fused_grad=fused)
    torch.cuda.synchronize()
    assert status == "ORL_OK", status
    npb = synth.batch_to_numpy(g)
    m = parity.valid_mask(npb["lengths"], T)
    with np.errstate(invalid="ignore"):
        o = oracle.logits_grad(npb["logits_new"], npb["tokens"], npb["lengths"], _np(bufs.dlogp).astype(np.float64),
                               1.0, c2, float(m.sum()))
    gg = dl.float().cpu().numpy()
    vm = np.broadcast_to(m[..., None], gg.shape)
    ni, nb = neg_inf.cpu().numpy() & vm, neg_big.cpu().numpy() & vm
    assert ni.sum() > 0 and nb.sum() > 0
    if c2 != 0.0:
        assert np.isnan(gg[ni]).all() and np.isnan(o[ni]).all()
    else:
        assert (gg[ni] == 0).all() and (o[ni] == 0).all()
    assert (gg[nb] == 0).all() and (o[nb] == 0).all()
    rest = vm & ~ni & ~nb
    assert np.isfinite(gg[rest]).all()
    err = np.abs(gg[rest] - o[rest])
    assert (err <= 8e-3 * np.abs(o[rest]) + 1e-6).all(), float(err.max())


def _grad_bound(x_rows, tok, lse, H, w, a, inv_temp, o, out_bf16):
    """Derived per-element bound for dL/dx (NEXT-1) of one row, GPU vs the fp64 oracle.
    The GPU evaluates g_v = inv_temp (p_v (a (ln p_v + H) - w) + [v = y] w) in fp32 from
    its saved fp32 lse, H, w (stage isolation: the oracle uses the same w, its own fp64
    lse and H), p_v = 2^(x_v c - lse log2 e).  Error sources:
      * p_v: |d ln p| <= |dlse| + 2^-23 (|x c| + |lse log2 e|) ln 2 + 2^-22 (MUFU ex2),
        |dlse| <= 1e-6 (S1's measured 5.4e-7 bound at V = 128256);
      * the factor a (ln p + H) - w: |dH| <= 1e-6 plus fp32 rounding of each operand;
      * at v = y, the delta term: cancellation of p_y w against w, error |w| |d p_y|;
      * the final rounding to the output dtype: 1/2 ulp = 2^-8 |g| (bf16), 2^-24 (fp32);
      * below the smallest normal (2^-126) everything is absolute: + 2^-126.
    bound_v = r_out (|o_v| + e_v) + e_v with
    e_v = inv_temp (p_v (|w| + a (|ln p_v| + |H| + 1)) eps_p + p_v a 2e-6) + [v = y] inv_temp |w| p_y eps_p."""
    z = inv_temp * x_rows
    lp = z - lse
    p = np.exp(lp)
    c = inv_temp * 1.4426950408889634
    eps_p = 1e-6 + (2.0 ** -23) * (np.abs(x_rows * c) + abs(lse) * 1.4426950408889634) * np.log(2) + 2.0 ** -22
    e = inv_temp * (p * (abs(w) + a * (np.abs(lp) + abs(H) + 1.0)) * eps_p + p * a * 2e-6)
    e[tok] += inv_temp * abs(w) * p[tok] * eps_p[tok]
    # below the smallest normal fp32 / bf16 (2^-126) the GPU's exp2 and output rounding are
    # absolute, not relative: one absolute 2^-126 covers that range
    e += 2.0 ** -126
    r_out = 2.0 ** -8 if out_bf16 else 2.0 ** -24
    return r_out * (np.abs(o) + e) + e


@pytest.mark.parametrize("V", [128256, 152064])
@pytest.mark.parametrize("fused", [True, False])
def test_next1_full_vocab_derived_bound(ctx, V, fused):
    """NEXT-1 at the BASELINE vocabularies (Llama-3 128256, Qwen2.5 152064), bf16, in the
    bench's launch configuration (the fused loss + backward pass, orl_ppo_loss_and_grad,
    and the two-pass orl_ppo_loss + orl_logits_grad / K5): every element of every valid
    row within the derived bound of _grad_bound; masked rows exactly 0; each row's
    gradient sums to ~0 (softmax shift invariance)."""
    B, T = 3, 40
    c = dict(synth.CONFIGS["llama8b"], c2=0.01, V=V)
    g = _gpu_batch(29, B, T, V, "mixed", mode="stress")
    cfg = PathConfig.from_synth(c)
    dl = torch.full((B, T, V), 3.0, dtype=torch.bfloat16, device=DEV)
    bufs = Buffers(B, T, DEV)
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    status, st = run_iteration(ctx, g, cfg, bufs, src, mb=2, grad_sink=lambda s, e: dl[s:e], fused_grad=fused)
    torch.cuda.synchronize()
    assert status == "ORL_OK"
    npb = synth.batch_to_numpy({k: v for k, v in g.items() if k in ("logits_new", "tokens", "lengths")})
    m = parity.valid_mask(npb["lengths"], T)
    N = float(m.sum())
    a = 0.01 / N
    w = _np(bufs.dlogp).astype(np.float64)
    gg = dl.float().cpu().numpy()
    n_el, worst = 0, 0.0
    for b in range(B):
        for t in range(T):
            if not m[b, t]:
                assert np.all(gg[b, t] == 0)
                continue
            x = (npb["logits_new"][b, t].astype(np.uint32) << 16).view(np.float32).astype(np.float64)
            y = int(npb["tokens"][b, t])
            o = oracle.logits_grad_row(x, y, 1.0, w[b, t], a)
            lse, _, H = oracle.row_logsoftmax(x, y)
            bound = _grad_bound(x, y, lse, H, w[b, t], a, 1.0, o, True)
            err = np.abs(gg[b, t] - o)
            worst = max(worst, float((err / bound).max()))
            assert np.all(err <= bound), (b, t, float((err / bound).max()))
            assert abs(gg[b, t].sum()) <= 1e-2 * np.abs(gg[b, t]).sum() + 1e-12
            n_el += V
    assert n_el >= 40 * V and worst > 0


def test_mid_size_end_to_end_chain_grpo_and_gae(ctx):
    """the whole chain from the logits at mid size (B = 8, T = 512,
    V = 128256 bf16, stress logits so the clip branches are exercised) against the
    oracle run end to end from the same logits -- log-probs at the north star's 2e-3
    (with the 1e-4 alarm), advantages / returns / per-token gradients / statistics at
    1e-5, per-token decisions bit-exact outside a 1e-5 ratio tie band -- for GAE with
    global whitening (C2-like) and GRPO with the k2 KL loss (C4-like)."""
    B, T, V = 8, 512, 128256
    for name in ("llama8b", "grpo"):
        c = dict(synth.CONFIGS[name])
        G = c["group_size"]
        g = _gpu_batch(808, B, T, V, "mixed", c["rewards"], G, mode="stress")
        if name == "grpo":                                 # one group of 8: not a constant one
            g["seq_reward"] = torch.tensor([1, 0, 1, 1, 0, 0, 1, 0], dtype=torch.float32, device=DEV)
        cfg = PathConfig.from_synth(c)
        status, st, bufs = _run(ctx, g, cfg, mb=3)
        assert status == "ORL_OK", status
        npb = synth.batch_to_numpy(g)
        m = parity.valid_mask(npb["lengths"], T)
        out, glob = oracle.pipeline([npb], c)
        o = out[0]
        for k, buf in (("logp_old", bufs.logp_old), ("logp_ref", bufs.logp_ref), ("logp_new", bufs.logp_new),
                       ("entropy", bufs.entropy)):
            parity.check_abs(f"{name} {k}", _np(buf), o[k], m)
        parity.check_rel(f"{name} adv", _np(bufs.adv), o["adv"], m)
        if o.get("ret") is not None:
            parity.check_rel(f"{name} ret", _np(bufs.ret), o["ret"], m)
        parity.check_rel(f"{name} dloss_dlogp", _np(bufs.dlogp), o["dlogp"], m)
        if name == "llama8b":
            parity.check_rel(f"{name} dloss_dv", _np(bufs.dv), o["dv"], m)
        lp_n, lp_o = _np(bufs.logp_new).astype(np.float64), _np(bufs.logp_old).astype(np.float64)
        rho = np.exp(lp_n - lp_o)
        tie = (np.abs(rho - (1 - c["eps_low"])) < 1e-5) | (np.abs(rho - (1 + c["eps_high"])) < 1e-5)
        gf, of = _np(bufs.flags).astype(np.int64), o["flags"].astype(np.int64)
        sel = m & ~tie
        assert np.array_equal(gf[sel] & 1, of[sel] & 1), f"{name}: clip decisions differ"
        if name == "llama8b":
            vn, vo, R = npb["values_new"], npb["values_old"], o["ret"]
            e1 = vn - R
            e2 = vo + np.clip(vn - vo, -c["eps_v"], c["eps_v"]) - R
            vtie = np.abs(e1 * e1 - e2 * e2) < 1e-5 * (np.abs(e1) + np.abs(e2)) + 1e-12
            assert np.array_equal(gf[m & ~vtie] & 2, of[m & ~vtie] & 2), f"{name}: value-clip decisions differ"
        n_clip = int(np.count_nonzero(of[m] & 1))
        assert n_clip > 0.01 * m.sum(), f"{name}: stress logits should clip (got {n_clip})"
        mabs = lambda a: float(np.mean(np.abs(a[m])))  # noqa: E731
        floors = dict(policy_loss=mabs(o["obj"]), value_loss=mabs(o["vl"]) or 1e-6, entropy=mabs(o["entropy"]),
                      kl=1e-6, approx_kl_old=1e-6, ratio_mean=1.0)
        floors["total_loss"] = sum(floors[k] for k in ("policy_loss", "value_loss", "entropy"))
        for k, fl in floors.items():
            assert abs(st[k] - glob["stats"][k]) <= parity.REL * max(abs(glob["stats"][k]), fl), \
                (name, k, st[k], glob["stats"][k])
        assert abs(st["clip_frac"] - glob["stats"]["clip_frac"]) <= (np.count_nonzero(tie & m) + 1e-9) / m.sum()
        del g
        torch.cuda.empty_cache()


def test_binding_rejects_bad_arguments(ctx):
    """orl.py checks every pointer argument before the C call (dtype, device,
    contiguity, size): int64 token ids, short or CPU per-token arrays, a micro-batch
    outside the rank batch and a wrong flags dtype raise instead of reaching the kernels."""
    B, T, V = 2, 8, 64
    g = _gpu_batch(1, B, T, V, "mixed")
    logp = torch.zeros(B, T, device=DEV)
    with pytest.raises(TypeError):
        orl.orl_logprobs(ctx, g["tokens"].long(), g["lengths"], g["logits_old"], logp)
    with pytest.raises(ValueError):
        orl.orl_logprobs(ctx, g["tokens"], g["lengths"], g["logits_old"], torch.zeros(B, T - 1, device=DEV))
    with pytest.raises(ValueError):
        orl.orl_logprobs(ctx, g["tokens"], g["lengths"], g["logits_old"], logp.cpu())
    with pytest.raises(ValueError):
        orl.orl_logprobs(ctx, g["tokens"], g["lengths"], g["logits_old"], logp, seq_offset=1)
    with pytest.raises(ValueError):
        orl.orl_logprobs(ctx, g["tokens"], g["lengths"], g["logits_old"].cpu(), logp)
    with pytest.raises(TypeError):
        orl.orl_advantages(ctx, g["lengths"].long(), torch.zeros(B, T, device=DEV), kind="rpp",
                           shaped_reward=torch.zeros(B, T, device=DEV))
    orl.orl_begin_iteration(ctx)
    orl.orl_logprobs(ctx, g["tokens"], g["lengths"], g["logits_old"], logp)
    orl.orl_advantages(ctx, g["lengths"], torch.zeros(B, T, device=DEV), kind="rpp",
                       shaped_reward=torch.zeros(B, T, device=DEV))
    orl.orl_whiten_stats(ctx, True)
    z = torch.zeros(B, T, device=DEV)
    with pytest.raises(TypeError):
        orl.orl_ppo_loss(ctx, g["tokens"], g["lengths"], g["logits_new"], orl.PPOConfig(), z, z, z.clone(),
                         flags=torch.zeros(B, T, device=DEV))
    with pytest.raises(ValueError):
        orl.orl_ppo_loss(ctx, g["tokens"], g["lengths"], g["logits_new"], orl.PPOConfig(), z, z[:1], z.clone())


@pytest.mark.parametrize("dtype,V,pad", [("bf16", 50257, 0), ("bf16", 4096, 5), ("f32", 1001, 1)])
def test_next1_unaligned_tma_matches_generic(ctx, monkeypatch, dtype, V, pad):
    """K5 on unaligned rows (aligned interior by TMA, scalar head / tail, target in a
    head or tail, masked rows zero-filled) gives the same bits as the generic kernel."""
    B, T = 3, 20
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = (torch.randn(B, T, V + pad, device=DEV) * 2).to(tdt)[..., :V]
    tok = synth.tokens_for(B, T, V, 8).to(DEV)
    tok[0, :3] = torch.tensor([0, 1, V - 1], dtype=torch.int32, device=DEV)
    L = torch.tensor([T, 11, 0], dtype=torch.int32, device=DEV)
    z = lambda: torch.zeros(B, T, device=DEV)  # noqa: E731
    lse, ent, w = z(), z(), torch.randn(B, T, device=DEV) * 1e-3
    orl.orl_begin_iteration(ctx)
    orl.orl_logprobs(ctx, tok, L, x, z(), entropy=ent, lse=lse)
    adv = z()
    orl.orl_advantages(ctx, L, adv, kind="rpp", shaped_reward=z())
    orl.orl_whiten_stats(ctx, False)
    cfg = orl.PPOConfig(c2=0.01)
    outs = {}
    for mode in ("tma", "generic"):
        if mode == "generic":
            monkeypatch.setenv("ORL_K1_NO_UNALIGNED_TMA", "1")
        dl = torch.full((B, T, V + pad), 3.0, dtype=tdt, device=DEV)[..., :V]
        orl.orl_logits_grad(ctx, tok, L, x, cfg, lse, ent, w, dl, zero_masked=True)
        torch.cuda.synchronize()
        outs[mode] = dl.float().cpu().numpy()
    monkeypatch.delenv("ORL_K1_NO_UNALIGNED_TMA")
    bad = np.argwhere(outs["tma"] != outs["generic"])
    assert bad.size == 0, (len(bad), bad[:8].tolist(), [(outs["tma"][tuple(i)], outs["generic"][tuple(i)])
                                                        for i in bad[:4]], _np(tok)[0, :4].tolist())
    assert np.all(outs["tma"][1, 11:] == 0) and np.all(outs["tma"][2] == 0)


@pytest.mark.parametrize("V", [256, 257])
def test_large_microbatch_global_prefix(ctx, V):
    """B > 1024 sequences in one call: the length prefix lives in global memory (aligned
    rows, and V = 257: unaligned rows through the TMA kernels)."""
    B, T = 1500, 3
    g = _gpu_batch(17, B, T, V, "mixed")
    g["lengths"] = torch.randint(0, T + 1, (B,), dtype=torch.int32, device=DEV)
    cfg = PathConfig.from_synth(dict(synth.CONFIGS["llama8b"], V=V, c2=0.01))
    dl = torch.full((B, T, V), 5.0, dtype=torch.bfloat16, device=DEV)
    bufs = Buffers(B, T, DEV)
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    status, st = run_iteration(ctx, g, cfg, bufs, src, mb=B, grad_sink=lambda s, e: dl[s:e])
    torch.cuda.synchronize()
    assert status == "ORL_OK"
    npb = synth.batch_to_numpy(g)
    m = parity.valid_mask(npb["lengths"], T)
    o = oracle.logprobs(npb["logits_new"], npb["tokens"], npb["lengths"])
    parity.check_abs("logp_new", _np(bufs.logp_new), o["logp"], m)
    parity.check_abs("entropy", _np(bufs.entropy), o["entropy"], m)
    out_i, glob_i = _isolated_oracle(npb, bufs, dict(synth.CONFIGS["llama8b"], V=V, c2=0.01))
    _check_downstream(bufs, out_i[0], glob_i, st, m, "largeB")
    assert torch.all(dl.float()[~torch.from_numpy(m).to(DEV)] == 0)


def test_nccl_one_rank_communicator_matches_local():
    """The NCCL all-gather path of C1/C2 (a 1-rank communicator) gives the same bits
    as the local merge."""
    B, T, V = 6, 64, 2048
    c = dict(synth.CONFIGS["llama8b"], V=V)
    cfg = PathConfig.from_synth(c)
    g = _gpu_batch(41, B, T, V, "mixed")
    a = orl.Context(0)
    n = orl.Context(0, 1, 0, orl.orl_get_unique_id())
    _, s1, b1 = _run(a, g, cfg, mb=4)
    _, s2, b2 = _run(n, g, cfg, mb=4)
    assert s1 == s2
    assert torch.equal(b1.dlogp, b2.dlogp) and torch.equal(b1.adv, b2.adv)
    a.close()
    n.close()


def test_next2_packed_varlen_matches_padded(ctx):
    """Packed varlen logits ([total, V] + cu_seqlens, NEXT-2) give bit-identical per-token
    outputs and dlogits to the padded [B, T, V] layout (rows are computed independently)."""
    B, T, V = 5, 40, 4096
    g = _gpu_batch(23, B, T, V, "mixed")
    L = g["lengths"].long()
    cu = torch.zeros(B + 1, dtype=torch.int32, device=DEV)
    cu[1:] = torch.cumsum(L, 0).int()
    packed = {r: torch.cat([g[f"logits_{r}"][b, : int(L[b])] for b in range(B)]) for r in ("old", "ref", "new")}
    cfg = PathConfig.from_synth(dict(synth.CONFIGS["llama8b"], V=V, c2=0.01))
    # padded reference run
    dl_pad = torch.zeros(B, T, V, dtype=torch.bfloat16, device=DEV)
    bp = Buffers(B, T, DEV)
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    status, st_pad = run_iteration(ctx, g, cfg, bp, src, mb=2, grad_sink=lambda s, e: dl_pad[s:e])
    assert status == "ORL_OK"
    # packed run through the same calls, micro-batches of 2 sequences
    bk = Buffers(B, T, DEV)
    tok = g["tokens"]
    dl_pk = torch.zeros_like(packed["new"])
    mbs = [(s, min(B, s + 2)) for s in range(0, B, 2)]
    view = lambda r, s: packed[r][int(cu[s]):]  # noqa: E731
    orl.orl_begin_iteration(ctx)
    for s, e in mbs:
        orl.orl_logprobs(ctx, tok, g["lengths"], view("old", s), bk.logp_old, seq_offset=s, cu_seqlens=cu, n_seq=e - s)
    for s, e in mbs:
        orl.orl_logprobs(ctx, tok, g["lengths"], view("ref", s), bk.logp_ref, seq_offset=s, cu_seqlens=cu,
                         n_seq=e - s, partner_logp=bk.logp_old, kl_est=cfg.kl_est_reward, beta_reward=cfg.beta_reward,
                         seq_reward=g["seq_reward"], kl=bk.kl, shaped_reward=bk.shaped)
    orl.orl_advantages(ctx, g["lengths"], bk.adv, kind="gae", gamma=cfg.gamma, lam=cfg.lam, shaped_reward=bk.shaped,
                       values=g["values_old"], seq_reward=g["seq_reward"], ret=bk.ret, adv_lo=bk.adv_lo)
    orl.orl_whiten_stats(ctx, True)
    for s, e in mbs:
        orl.orl_ppo_loss(ctx, tok, g["lengths"], view("new", s), cfg.ppo, bk.logp_old, bk.adv, bk.logp_new,
                         seq_offset=s, cu_seqlens=cu, n_seq=e - s, logp_ref=bk.logp_ref, ret=bk.ret,
                         v_new=g["values_new"], v_old=g["values_old"], entropy=bk.entropy, lse=bk.lse,
                         dloss_dlogp=bk.dlogp, dloss_dv=bk.dv, adv_lo=bk.adv_lo)
    for s, e in mbs:
        orl.orl_logits_grad(ctx, tok, g["lengths"], view("new", s), cfg.ppo, bk.lse, bk.entropy, bk.dlogp,
                            dl_pk[int(cu[s]):], seq_offset=s, cu_seqlens=cu, n_seq=e - s)
    status, st_pk = orl.orl_finalize(ctx, cfg.ppo)
    assert status == "ORL_OK" and st_pk == st_pad
    for k in ("logp_old", "logp_ref", "logp_new", "entropy", "adv", "ret", "dlogp", "dv", "lse"):
        assert torch.equal(getattr(bk, k), getattr(bp, k)), k
    for b in range(B):
        assert torch.equal(dl_pk[int(cu[b]):int(cu[b + 1])], dl_pad[b, : int(L[b])])


@pytest.mark.parametrize("kind", ["gae", "grpo"])
def test_next2_seq_mean_aggregation(ctx, kind):
    """Sequence-mean loss aggregation (NEXT-2, Z31): stats, per-token gradients and
    dL/dlogits against the oracle (stage isolation), tiny fp32 and mid bf16."""
    for dtype, V, B, T in (("f32", 32, 8, 16), ("bf16", 4096, 6, 48)):
        c = dict(synth.CONFIGS["tiny"], V=V, adv_kind=kind, loss_agg="seq_mean_token_mean", c2=0.02,
                 group_size=2 if kind == "grpo" else 1)
        if kind == "grpo":
            c.update(kl_mode="loss", kl_est_loss="k3", beta_loss=0.05, whiten=False, eps_v=0.0, c1=0.0)
        if dtype == "f32":
            g = _to_dev(synth.make_batch(3, B, T, V, "f32", "stress", "tiny", c["rewards"], c["group_size"]))
        else:
            g = _gpu_batch(3, B, T, V, "mixed", "group_bernoulli" if kind == "grpo" else "normal", 2, "stress")
        cfg = PathConfig.from_synth(c)
        tdt = torch.float32 if dtype == "f32" else torch.bfloat16
        dl = torch.zeros(B, T, V, dtype=tdt, device=DEV)
        bufs = Buffers(B, T, DEV, c["group_size"])
        src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
        status, st = run_iteration(ctx, g, cfg, bufs, src, mb=3, grad_sink=lambda s, e: dl[s:e])
        torch.cuda.synchronize()
        assert status == "ORL_OK"
        npb = synth.batch_to_numpy(g)
        m = parity.valid_mask(npb["lengths"], T)
        out_i, glob_i = _isolated_oracle(npb, bufs, c)
        _check_downstream(bufs, out_i[0], glob_i, st, m, f"seqmean-{kind}-{dtype}")
        n_seq = float(np.count_nonzero(npb["lengths"] > 0))
        o = oracle.logits_grad(npb["logits_new"], npb["tokens"], npb["lengths"], _np(bufs.dlogp).astype(np.float64),
                               1.0, 0.02, float(m.sum()), seq_mean=True, n_seq=n_seq)
        H = oracle.logprobs(npb["logits_new"], npb["tokens"], npb["lengths"])["entropy"]
        # per-row entropy weight a = c2 / (n_seq L_b): bound it by the largest (shortest row)
        a_max = 0.02 / (n_seq * max(1, int(npb["lengths"][npb["lengths"] > 0].min())))
        _check_grad(dl.float().cpu().numpy(), o, m, 2e-5 if dtype == "f32" else 8e-3, f"seqmean-{dtype}",
                    _np(bufs.dlogp), H, a_max, 1.0)


@pytest.mark.parametrize("agg", ["token_mean", "seq_mean_token_mean"])
@pytest.mark.parametrize("V,pad", [(8192, 0), (50257, 0), (8192, 3)])
def test_next1_fused_forward_backward_matches_two_passes(ctx, agg, V, pad):
    """orl_ppo_loss_and_grad (one pass, the row re-read from L2) gives the same bits as
    orl_ppo_loss followed by orl_logits_grad (K5); also for unaligned rows (V = 50257,
    padded pitches: the aligned interiors by TMA, heads / tails singly; targets in them)."""
    B, T = 6, 96
    g = _gpu_batch(29, B, T, V, "mixed", mode="stress")
    g["tokens"][0, :4] = torch.tensor([0, 1, V - 1, V - 2], dtype=torch.int32, device=DEV)
    if pad:
        for r in ("old", "ref", "new"):
            buf = torch.zeros(B, T, V + pad, dtype=torch.bfloat16, device=DEV)
            buf[..., :V] = g[f"logits_{r}"]
            g[f"logits_{r}"] = buf[..., :V]
    cfg = PathConfig.from_synth(dict(synth.CONFIGS["llama8b"], V=V, c2=0.01, loss_agg=agg))
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    out = {}
    for fused in (True, False):
        dl = torch.full((B, T, V + pad), 7.0, dtype=torch.bfloat16, device=DEV)[..., :V]
        bufs = Buffers(B, T, DEV)
        status, st = run_iteration(ctx, g, cfg, bufs, src, mb=4, grad_sink=lambda s, e: dl[s:e], fused_grad=fused)
        torch.cuda.synchronize()
        assert status == "ORL_OK"
        out[fused] = (st, dl, bufs)
    assert out[True][0] == out[False][0]
    assert torch.equal(out[True][1], out[False][1])
    for k in ("logp_new", "entropy", "lse", "dlogp", "dv"):
        assert torch.equal(getattr(out[True][2], k), getattr(out[False][2], k)), k


@pytest.mark.parametrize("dtype,V,B,T,agg", [("bf16", 128256, 3, 40, "token_mean"), ("bf16", 8192, 6, 96, "seq_mean_token_mean"),
                                             ("bf16", 152064, 2, 24, "token_mean"), ("f32", 4096, 5, 33, "token_mean"),
                                             ("bf16", 136, 7, 50, "token_mean")])
def test_next1_fused_pass_spikes_and_bound(ctx, dtype, V, B, T, agg):
    """The fused actor pass (orl_ppo_loss_and_grad) at the BASELINE vocabularies and odd
    shapes, with spikes far above the first-vector seed (the exact redo) in old, ref and
    actor logits: log-probs / entropy / lse against the oracle, the same outputs as the
    two-pass path (orl_ppo_loss + K5), decisions bit-exact, every dlogits element within
    the derived NEXT-1 bound of the fp64 oracle, masked rows exactly 0, run-to-run bit
    identical."""
    c = dict(synth.CONFIGS["llama8b"], V=V, c2=0.01, loss_agg=agg)
    if dtype == "f32":
        g = _to_dev(synth.make_batch(31, B, T, V, "f32", "stress", "tiny"))
    else:
        g = _gpu_batch(31, B, T, V, "mixed", mode="stress")
    g["tokens"][0, :4] = torch.tensor([0, 1, V - 1, V // 2], dtype=torch.int32, device=DEV)
    # spikes far above the first-vector seed (> 64 log2 units): the exact redo of a held half-row,
    # in the first and in the second half of a row
    for r in ("old", "ref", "new"):
        g[f"logits_{r}"][1, 0, 5] = 90.0
        g[f"logits_{r}"][1, 1, V - 3] = 70.0
    cfg = PathConfig.from_synth(c)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    out = {}
    for key, fused in (("fused", True), ("fused2", True), ("two", False)):
        dl = torch.full((B, T, V), 7.0, dtype=tdt, device=DEV)
        bufs = Buffers(B, T, DEV)
        status, st = run_iteration(ctx, g, cfg, bufs, src, mb=2, grad_sink=lambda s, e: dl[s:e], fused_grad=fused)
        torch.cuda.synchronize()
        assert status == "ORL_OK", status
        out[key] = (st, dl, bufs)
    assert out["fused"][0] == out["fused2"][0] and torch.equal(out["fused"][1], out["fused2"][1])  # run to run
    m = parity.valid_mask(_np(g["lengths"]), T)
    (st7, dl7, b7), (st2, dl2, b2) = out["fused"], out["two"]
    npb = synth.batch_to_numpy({k: g[k] for k in ("logits_new", "tokens", "lengths")})
    ora = oracle.logprobs(npb["logits_new"], npb["tokens"], npb["lengths"])
    for k in ("logp_new", "entropy", "lse"):
        parity.check_abs(f"fused {k}", _np(getattr(b7, k)), ora[k.replace("_new", "")], m)
        np.testing.assert_allclose(_np(getattr(b7, k))[m], _np(getattr(b2, k))[m], rtol=0, atol=5e-5, err_msg=k)
    parity.check_rel("dlogp", _np(b7.dlogp), _np(b2.dlogp).astype(np.float64), m, rel=1e-5)
    assert np.array_equal(_np(b7.flags), _np(b2.flags))
    for k in ("policy_loss", "entropy", "kl", "ratio_mean", "total_loss", "value_loss"):
        assert abs(st7[k] - st2[k]) <= 1e-5 * max(abs(st2[k]), 1e-3), (k, st7[k], st2[k])
    gg = dl7.float().cpu().numpy()
    assert np.all(gg[~m] == 0)
    w = _np(b7.dlogp).astype(np.float64)
    N = float(m.sum())
    L = npb["lengths"]
    for b in range(B):
        a = 0.01 / (float((L > 0).sum()) * float(L[b])) if agg != "token_mean" else 0.01 / N
        for t in range(int(L[b])):
            row = npb["logits_new"][b, t]
            x = (row.astype(np.uint32) << 16).view(np.float32).astype(np.float64) if dtype == "bf16" \
                else row.astype(np.float64)
            y = int(npb["tokens"][b, t])
            o = oracle.logits_grad_row(x, y, 1.0, w[b, t], a)
            lse, _, H = oracle.row_logsoftmax(x, y)
            bound = _grad_bound(x, y, lse, H, w[b, t], a, 1.0, o, dtype == "bf16")
            err = np.abs(gg[b, t] - o)
            assert np.all(err <= bound), (b, t, float((err / bound).max()))


@pytest.mark.parametrize("kind", ["rpp", "gae"])
def test_whitening_near_constant_advantages(ctx, kind):
    """Z33: global whitening of nearly constant advantages (|mu|/sigma ~ 1e7: gamma = 1, one
    reward per sequence, tiny KL shaping) is exact to fp64 because the actor pass whitens
    adv + adv_lo (orl_advantages' low part). Stage-isolated: the oracle's S4 is fed the GPU's
    own fp32 shaped rewards (at this conditioning the fp32 rounding of r' itself is of the
    order of sigma), then whitening and the loss stage; A + A_lo, A', dL/dlogp and the
    statistics at the 1e-5 bar, decisions bit-exact."""
    B, T, V = 3, 64, 512
    c = dict(synth.CONFIGS["llama8b"], V=V, adv_kind=kind, gamma=1.0, lam=1.0, beta_reward=1e-7, eps_v=0.2)
    g = _gpu_batch(41, B, T, V, "full")
    g["seq_reward"] = torch.full((B,), 5.0, device=DEV)
    if kind == "gae":
        g["values_old"] = torch.zeros(B, T, device=DEV)
    cfg = PathConfig.from_synth(c)
    status, st, bufs = _run(ctx, g, cfg, mb=2)
    assert status == "ORL_OK"
    L = _np(g["lengths"])
    m = parity.valid_mask(L, T)
    f64 = lambda t: _np(t).astype(np.float64)  # noqa: E731
    r = f64(bufs.shaped)                                   # the GPU's S3 output
    if kind == "gae":
        A, R = oracle.gae(L, r, f64(g["values_old"]), 1.0, 1.0)
    else:
        A = R = oracle.discounted_returns(L, r, 1.0)
    A_gpu = f64(bufs.adv) + f64(bufs.adv_lo)
    np.testing.assert_allclose(A_gpu[m], A[m], rtol=1e-13, atol=0)   # ~48-bit advantages
    mu, sd, warn = oracle.whiten_moments(A[m])
    assert not warn and abs(mu) / sd > 1e6, (mu, sd)
    assert abs(st["adv_mean"] - mu) <= 1e-12 * abs(mu) and abs(st["adv_std"] - sd) <= 1e-5 * sd
    Aw = oracle.whiten(A, L, mu, sd)
    crit = kind == "gae"
    res = oracle.ppo_loss(L, f64(bufs.logp_new), f64(bufs.logp_old), Aw, logp_ref=f64(bufs.logp_ref),
                          ret=R if crit else None, v_new=f64(g["values_new"]) if crit else None,
                          v_old=f64(g["values_old"]) if crit else None, entropy=f64(bufs.entropy),
                          eps_low=c["eps_low"], eps_high=c["eps_high"], eps_v=c["eps_v"], c1=c["c1"] if crit else 0.0)
    parity.check_rel("dloss_dlogp", _np(bufs.dlogp), res["dlogp"], m)
    rho = np.exp(f64(bufs.logp_new) - f64(bufs.logp_old))
    tie = (np.abs(rho - 0.8) < 1e-9) | (np.abs(rho - 1.2) < 1e-9)
    assert np.array_equal((_np(bufs.flags) & 1)[m & ~tie], (res["flags"] & 1)[m & ~tie])
    ost = oracle.stats(res["sums"], c1=c["c1"] if crit else 0.0)
    fl = float(np.mean(np.abs(res["obj"][m])))
    assert abs(st["policy_loss"] - ost["policy_loss"]) <= parity.REL * max(abs(ost["policy_loss"]), fl)
    # without the low part the fp32 advantages could not carry sigma / |mu| ~ 1e-7
    assert np.any(_np(bufs.adv_lo)[m] != 0)


def test_pdl_chain_is_bit_identical(ctx):
    """orl_set_pdl_chain only changes when a K1 launch may start reading (its producer does
    not wait for the previous grid): every output and statistic is bit-identical with and
    without it, for every pass of an iteration (logprob, reward, loss and fused modes)."""
    c = dict(synth.CONFIGS["llama8b"], c2=0.01)
    B, T, V = 12, 160, 8192
    g = _gpu_batch(55, B, T, V, "mixed", mode="stress")
    cfg = PathConfig.from_synth(dict(c, V=V))
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    out = {}
    for chain in (False, True):
        dl = torch.zeros(B, T, V, dtype=torch.bfloat16, device=DEV)
        bufs = Buffers(B, T, DEV)
        res = run_iteration(ctx, g, cfg, bufs, src, mb=3, pdl_chain=chain, grad_sink=lambda s, e: dl[s:e])
        torch.cuda.synchronize()
        out[chain] = (res, bufs, dl)
    assert out[False][0] == out[True][0]
    for k in ("logp_old", "logp_ref", "kl", "shaped", "adv", "adv_lo", "ret", "logp_new", "entropy", "lse", "dlogp",
              "dv", "flags"):
        assert torch.equal(getattr(out[False][1], k), getattr(out[True][1], k)), k
    assert torch.equal(out[False][2], out[True][2])
    assert ctx.pdl_chain is False                     # run_iteration restores the context setting


def test_lengths_from_attention_mask(ctx):
    """orl_lengths_from_mask (Z10): leading-ones count of right-padded masks, bit-exact
    against oracle.lengths_from_mask; a non-prefix mask is reported as ORL_E_MASK; an iteration on
    mask-derived lengths equals the one on the true lengths bit for bit."""
    rng = np.random.default_rng(7)
    B, T = 37, 300
    L = rng.integers(0, T + 1, size=B).astype(np.int32)
    L[0], L[1] = 0, T
    mask = (np.arange(T)[None, :] < L[:, None]).astype(np.uint8)
    got = torch.full((B,), -5, dtype=torch.int32, device=DEV)
    orl.orl_begin_iteration(ctx)
    orl.orl_lengths_from_mask(ctx, torch.from_numpy(mask).to(DEV), got)
    torch.cuda.synchronize()
    want, nbad = oracle.lengths_from_mask(mask)
    assert nbad == 0 and np.array_equal(_np(got), want) and np.array_equal(want, L)
    bad = mask.copy()
    bad[5, L[5] + 3 if L[5] + 3 < T else 0] = 1 if L[5] + 3 < T else 0
    bad[9, :] = 0
    bad[9, 7] = 1                                       # a hole-y row: leading prefix 0, error
    orl.orl_begin_iteration(ctx)
    orl.orl_lengths_from_mask(ctx, torch.from_numpy(bad).to(DEV).bool(), got)
    status, st = orl.orl_finalize(ctx, orl.PPOConfig())
    assert status == "ORL_E_MASK"
    lead, nbad = oracle.lengths_from_mask(bad)
    assert nbad >= 1 and np.array_equal(_np(got), lead)
    # whole iteration on mask-derived lengths == on the true lengths
    c = dict(synth.CONFIGS["llama8b"])
    g = _gpu_batch(71, 6, 96, 2048, "mixed")
    cfg = PathConfig.from_synth(c)
    _, st1, b1 = _run(ctx, g, cfg, mb=4)
    m6 = (torch.arange(96, device=DEV)[None, :] < g["lengths"][:, None]).to(torch.uint8)
    g2 = dict(g, lengths=torch.empty_like(g["lengths"]))
    orl.orl_begin_iteration(ctx)
    orl.orl_lengths_from_mask(ctx, m6, g2["lengths"])
    _, st2, b2 = _run(ctx, g2, cfg, mb=4)
    assert st1 == st2 and torch.equal(b1.adv, b2.adv) and torch.equal(b1.logp_new, b2.logp_new)
    with pytest.raises(TypeError):
        orl.orl_lengths_from_mask(ctx, m6.float(), g2["lengths"])


@pytest.mark.parametrize("n", [0, 1, 37, 1024, 5000])
def test_dapo_keep_compact(ctx, n):
    """orl_keep_compact (NEXT-2, DAPO dynamic sampling): the kept groups' indices in order
    and their count, bit-exact against oracle.keep_compact; also straight from
    orl_advantages' mask (itself bit-exact against oracle.group_advantages)."""
    rng = np.random.default_rng(n)
    keep = (rng.random(n) < 0.6).astype(np.uint8)
    if n > 2:
        keep[:2] = [1, 0]
    idx = torch.full((max(n, 1),), -7, dtype=torch.int32, device=DEV)
    cnt = torch.full((1,), -7, dtype=torch.int32, device=DEV)
    orl.orl_keep_compact(ctx, torch.from_numpy(keep).to(DEV), idx, cnt)
    torch.cuda.synchronize()
    want = oracle.keep_compact(keep)
    assert int(cnt.item()) == want.size
    assert np.array_equal(_np(idx)[: want.size], want)
    if n == 37:  # the mask GRPO writes for a batch with some constant-reward groups
        G, ng = 4, 16
        R = torch.tensor(rng.integers(0, 2, size=G * ng), dtype=torch.float32)
        R[:G] = 1.0                              # a constant group: dropped
        L = torch.full((G * ng,), 5, dtype=torch.int32, device=DEV)
        adv = torch.zeros(G * ng, 5, device=DEV)
        gk = torch.zeros(ng, dtype=torch.uint8, device=DEV)
        orl.orl_begin_iteration(ctx)
        orl.orl_advantages(ctx, L, adv, kind="grpo", group_size=G, seq_reward=R.to(DEV), group_keep=gk)
        gi = torch.zeros(ng, dtype=torch.int32, device=DEV)
        orl.orl_keep_compact(ctx, gk, gi, cnt)
        torch.cuda.synchronize()
        _, k_or = oracle.group_advantages(R.numpy().astype(np.float64), G)
        assert np.array_equal(_np(gk), k_or)                     # keep-mask bit-exact vs the oracle
        want = oracle.keep_compact(k_or)
        assert int(cnt.item()) == want.size and 0 not in _np(gi)[: int(cnt.item())].tolist()
        assert np.array_equal(_np(gi)[: int(cnt.item())], want)
