"""Pins for the oracle's STAGE COMPOSITION (oracle/pipeline.py), -m "not gpu".

Every GPU end-to-end and stage-isolated parity test compares against
``oracle.pipeline()``, so its wiring is pinned here by what the paper and the
mathematics fix, not by re-running the oracle's own stage functions:

  * W3 through the whole pipeline (hand-worked): KL sign and
    orientation d = logp_old - logp_ref (Z4), r' = [t = L-1] R - beta k
    (Z7), GAE on the experience-time values (Z9), and the
    on-policy loss identity rho = 1, obj = A (north star).
  * sum_t r'_t = R_b - beta sum_t k_t on random batches.
  * GRPO advantages are group-normalised only, never re-whitened (Z19):
    equal to the numpy population-std closed form for every token, whether
    whitening is requested or not; W4 values.
  * REINFORCE++-baseline (Z23): with gamma = 1 and beta = 0 the return is the
    closed form R_b - mean_g(R) at every valid token; in general it equals the
    plain REINFORCE++ pipeline run on the rewards R_b - mu_g.
  * KL-in-loss ("k2 as the loss function", P:197 gradient): the
    pipeline's per-token dlogp equals central differences of the pipeline's own
    total_loss with respect to logp_new; total = policy_loss + beta * kl
    (recomposition).
  * Z9: the critic values of the loss (values_new) never reach A or R; the
    experience-time values (values_old) do.
  * Global whitening (Z19): over all shards' valid tokens the whitened
    advantages have mean 0 and population std 1 (to the 1e-8 epsilon).

tools/mutate_oracle.py applies plausible wiring mistakes to a scratch copy of
the oracle and checks that each one fails at least one of these tests.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle.pipeline import pipeline

rng = np.random.default_rng(20240517)


def _shard(logp_old, logp_ref, L, R, values_old=None, values_new=None, logp_new=None, entropy=None):
    """A stage-isolated shard: the S1 outputs are supplied, the rest is computed."""
    logp_old = np.atleast_2d(np.asarray(logp_old, np.float64))
    B, T = logp_old.shape
    sh = dict(lengths=np.asarray(L, np.int32), seq_reward=np.asarray(R, np.float64),
              tokens=np.zeros((B, T), np.int32), logp_old=logp_old,
              logp_ref=np.atleast_2d(np.asarray(logp_ref, np.float64)),
              logp_new=logp_old.copy() if logp_new is None else np.atleast_2d(np.asarray(logp_new, np.float64)),
              entropy_new=np.zeros((B, T)) if entropy is None else entropy)
    if values_old is not None:
        sh["values_old"] = np.atleast_2d(np.asarray(values_old, np.float64))
    if values_new is not None:
        sh["values_new"] = np.atleast_2d(np.asarray(values_new, np.float64))
    return sh


def _random_shard(B, T, seed, with_values=True, group_reward=False, G=1):
    r = np.random.default_rng(seed)
    L = r.integers(1, T + 1, size=B).astype(np.int32)
    L[0] = T
    lo = r.normal(-1.5, 0.6, (B, T))
    lr = lo + r.normal(0, 0.3, (B, T))
    ln = lo + r.normal(0, 0.15, (B, T))
    if group_reward:
        p = np.repeat(r.random(B // G), G)
        R = (r.random(B) < p).astype(np.float64)
    else:
        R = r.normal(0, 1, B)
    vo = r.normal(0, 1, (B, T)) if with_values else None
    vn = vo + r.normal(0, 0.3, (B, T)) if with_values else None
    H = np.abs(r.normal(1.0, 0.5, (B, T)))
    return _shard(lo, lr, L, R, vo, vn, ln, H)


def _valid(sh):
    L = sh["lengths"]
    T = sh["logp_old"].shape[1]
    return np.arange(T)[None, :] < L[:, None]


# ----------------------------------------------------------------------------- W3
@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_pipeline_worked_example_w3(golden, case):
    """W3 end to end through pipeline(): shaping (sign, estimator orientation, reward
    placement), GAE on V_old (values_new deliberately different), returns, and the
    on-policy loss identity (logp_new = logp_old: rho = 1, obj = A, no clipping,
    dlogp = -A/N)."""
    g = golden("w3_shaping_gae_t3.json")
    c = g["cases"][case]
    V = np.array(g["V"])
    sh = _shard(g["logp_old"], g["logp_ref"], [3], [g["R"]], values_old=V,
                values_new=V + np.array([0.3, -0.2, 0.5]))
    cfg = dict(adv_kind="gae", gamma=c["gamma"], lam=c["lam"], beta_reward=g["beta"], kl_est_reward="k1",
               whiten=False, eps_v=0.0, c1=0.5)
    out, glob = pipeline([sh], cfg)
    o = out[0]
    np.testing.assert_allclose(o["kl"][0], g["kl_out"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(o["shaped_reward"][0], g["shaped"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(o["adv"][0], c["adv"], rtol=0, atol=1e-14)
    # R_t = A_t + V_old(s_t); case 0 prints R
    np.testing.assert_allclose(o["ret"][0], c.get("ret", np.array(c["adv"]) + V), rtol=0, atol=1e-14)
    # on-policy: rho = 1, nothing clipped, obj = A, policy_loss = -mean(A)   (north star)
    A = np.array(c["adv"])
    st = glob["stats"]
    assert st["clip_frac"] == 0.0 and st["ratio_mean"] == 1.0 and st["approx_kl_old"] == 0.0
    assert abs(st["policy_loss"] + A.mean()) < 1e-15
    np.testing.assert_allclose(o["dlogp"][0], -A / 3.0, rtol=0, atol=1e-16)
    # the value loss is the plain MSE of values_new against R (eps_v <= 0)
    vn = sh["values_new"][0]
    assert abs(st["value_loss"] - np.mean((vn - o["ret"][0]) ** 2)) < 1e-15


@pytest.mark.parametrize("kl", ["k1", "k2", "k3"])
def test_pipeline_shaping_sum_and_orientation(kl):
    """sum_t r'_t = R_b - beta sum_t k(logp_old - logp_ref) (Z4, Z7); the actor's
    logp_new never enters the shaping; kl_mode=loss shapes with R only."""
    sh = _random_shard(6, 9, 11)
    beta = 0.37
    out, _ = pipeline([sh], dict(adv_kind="rpp", gamma=1.0, beta_reward=beta, kl_est_reward=kl, whiten=False))
    o = out[0]
    m = _valid(sh)
    d = sh["logp_old"] - sh["logp_ref"]
    k = {"k1": d, "k2": 0.5 * d * d, "k3": np.exp(-d) - 1 + d}[kl]
    for b in range(6):
        Lb = sh["lengths"][b]
        assert abs(o["shaped_reward"][b, :Lb].sum() - (sh["seq_reward"][b] - beta * k[b, :Lb].sum())) < 1e-12
        # REINFORCE++ with gamma = 1: G_0 = sum_t r'_t (north star, Z23)
        assert abs(o["adv"][b, 0] - o["shaped_reward"][b, :Lb].sum()) < 1e-12
    # logp_new does not reach the experience side
    sh2 = dict(sh, logp_new=sh["logp_new"] + 0.5)
    out2, _ = pipeline([sh2], dict(adv_kind="rpp", gamma=1.0, beta_reward=beta, kl_est_reward=kl, whiten=False))
    assert np.array_equal(out2[0]["shaped_reward"], o["shaped_reward"]) and np.array_equal(out2[0]["adv"], o["adv"])
    # kl_mode = loss: r' = [t = L_b - 1] R_b exactly (no shaping, Z5)
    out3, _ = pipeline([sh], dict(adv_kind="rpp", gamma=1.0, kl_mode="loss", beta_reward=beta, beta_loss=0.1,
                                  whiten=False))
    want = np.zeros_like(o["shaped_reward"])
    for b in range(6):
        want[b, sh["lengths"][b] - 1] = sh["seq_reward"][b]
    assert np.array_equal(out3[0]["shaped_reward"], want)


# ----------------------------------------------------------------------------- GRPO (Z19)
@pytest.mark.parametrize("whiten", [True, False])
def test_pipeline_grpo_is_group_normalised_only(whiten):
    """GRPO (Z19, Z20): A' at every valid token is the group closed
    form (R_b - mean_g)/(pop std_g + 1e-8), 0 for a constant group -- with or without
    whitening requested, and across a rank split (whitening never touches GRPO)."""
    G, ng, T = 4, 6, 7
    sh = _random_shard(G * ng, T, 5, with_values=False, group_reward=True, G=G)
    R = sh["seq_reward"].copy()
    R[:G] = [1.0, 0.0, 0.0, 1.0]            # W4: +-0.99999998
    R[G:2 * G] = 1.0                        # constant group: exactly 0
    sh["seq_reward"] = R
    cfg = dict(adv_kind="grpo", group_size=G, kl_mode="loss", beta_loss=0.001, kl_est_loss="k2", whiten=whiten,
               eps_v=0.0, c1=0.0)
    out, glob = pipeline([sh], cfg)
    want = np.zeros(G * ng)
    for g in range(ng):
        x = R[g * G:(g + 1) * G]
        want[g * G:(g + 1) * G] = 0.0 if x.max() == x.min() else (x - x.mean()) / (x.std() + 1e-8)
    m = _valid(sh)
    A = np.where(m, want[:, None], 0.0)
    np.testing.assert_allclose(out[0]["adv_w"], A, rtol=0, atol=1e-14)
    np.testing.assert_allclose(out[0]["adv_w"][:G, 0], [0.99999998, -0.99999998, -0.99999998, 0.99999998],
                               rtol=0, atol=1e-15)
    assert np.all(out[0]["adv_w"][G:2 * G] == 0.0)
    # the stats see exactly these advantages: with logp_new = logp_old + delta the policy
    # objective is sum min(rho A, clip(rho) A) over them
    rho = np.exp(sh["logp_new"] - sh["logp_old"])
    obj = np.minimum(rho * A, np.clip(rho, 0.8, 1.2) * A)
    assert abs(glob["stats"]["policy_loss"] + obj[m].mean()) < 1e-13
    outs, _ = pipeline([{k: v[:G * 3] for k, v in sh.items()}, {k: v[G * 3:] for k, v in sh.items()}], cfg)
    np.testing.assert_allclose(np.concatenate([outs[0]["adv_w"], outs[1]["adv_w"]]), A, rtol=0, atol=1e-14)


# ----------------------------------------------------------------------------- REINFORCE++-baseline
def test_pipeline_rpp_baseline_subtracts_group_mean():
    """REINFORCE++-baseline (Z23): with gamma = 1 and no KL shaping the return at every
    valid token is R_b - mean_g(R) (closed form); with shaping it equals the plain
    REINFORCE++ pipeline on the rewards R_b - mu_g."""
    G, ng, T = 4, 5, 8
    sh = _random_shard(G * ng, T, 9, with_values=False, group_reward=True, G=G)
    R = sh["seq_reward"]
    mu = np.repeat(R.reshape(ng, G).mean(axis=1), G)
    m = _valid(sh)
    out, _ = pipeline([sh], dict(adv_kind="rpp_baseline", group_size=G, gamma=1.0, beta_reward=0.0, whiten=False))
    np.testing.assert_allclose(out[0]["adv"], np.where(m, (R - mu)[:, None], 0.0), rtol=0, atol=1e-15)
    cfg = dict(gamma=0.97, beta_reward=0.05, kl_est_reward="k3", whiten=True, group_size=G)
    out_b, gb = pipeline([sh], dict(cfg, adv_kind="rpp_baseline"))
    out_p, gp = pipeline([dict(sh, seq_reward=R - mu)], dict(cfg, adv_kind="rpp"))
    np.testing.assert_allclose(out_b[0]["adv"], out_p[0]["adv"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(out_b[0]["adv_w"], out_p[0]["adv_w"], rtol=0, atol=1e-12)
    assert abs(gb["stats"]["policy_loss"] - gp["stats"]["policy_loss"]) < 1e-13


# ----------------------------------------------------------------------------- KL in the loss
@pytest.mark.parametrize("kind,kl", [("grpo", "k2"), ("grpo", "k3"), ("gae", "k1"), ("rpp", "k2")])
def test_pipeline_dlogp_is_the_gradient_of_its_total(kind, kl):
    """dlogp of pipeline() = central differences of pipeline()'s own total_loss w.r.t.
    logp_new ("gradient computation"; P:94 k2 as the loss), with the KL-in-loss
    term, DAPO decoupled clip and the critic; total = policy + c1 value - c2 H + beta kl."""
    G = 2
    sh = _random_shard(4, 5, 21, with_values=(kind == "gae"), group_reward=(kind == "grpo"), G=G)
    beta = 0.3
    cfg = dict(adv_kind=kind, group_size=G, kl_mode="loss", beta_loss=beta, kl_est_loss=kl, eps_low=0.2,
               eps_high=0.28, eps_v=0.2, c1=0.5, c2=0.01, whiten=kind != "grpo", lam=0.9, gamma=0.99)
    out, glob = pipeline([sh], cfg)
    st = glob["stats"]
    assert abs(st["total_loss"] - (st["policy_loss"] + 0.5 * st["value_loss"] * (kind == "gae")
                                   - 0.01 * st["entropy"] + beta * st["kl"])) < 1e-14
    d = sh["logp_new"] - sh["logp_ref"]
    kk = {"k1": d, "k2": 0.5 * d * d, "k3": np.exp(-d) - 1 + d}[kl]
    m = _valid(sh)
    assert abs(st["kl"] - kk[m].mean()) < 1e-14
    dl = out[0]["dlogp"]
    h = 1e-6
    rho = np.exp(sh["logp_new"] - sh["logp_old"])
    n_checked = 0
    for b in range(4):
        for t in range(5):
            if not m[b, t]:
                assert dl[b, t] == 0.0
                continue
            if min(abs(rho[b, t] - 0.8), abs(rho[b, t] - 1.28)) < 1e-4:
                continue                                            # a kink (Z17)
            tot = []
            for s in (+h, -h):
                ln = sh["logp_new"].copy()
                ln[b, t] += s
                tot.append(pipeline([dict(sh, logp_new=ln)], cfg)[1]["stats"]["total_loss"])
            fd = (tot[0] - tot[1]) / (2 * h)
            assert abs(fd - dl[b, t]) < 1e-8, (b, t, fd, dl[b, t])
            n_checked += 1
    assert n_checked >= 10


# ----------------------------------------------------------------------------- Z9 critic values
def test_pipeline_gae_uses_experience_values_only():
    """Z9 (P:195 V(s_t) at experience time, P:197 critic loss): values_new never reaches
    A or R; values_old does; values_new is what the value loss compares to R."""
    sh = _random_shard(5, 6, 33)
    cfg = dict(adv_kind="gae", gamma=0.99, lam=0.95, whiten=True, eps_v=0.2, c1=0.5)
    out, glob = pipeline([sh], cfg)
    out2, glob2 = pipeline([dict(sh, values_new=sh["values_new"] + 0.25)], cfg)
    assert np.array_equal(out[0]["adv"], out2[0]["adv"]) and np.array_equal(out[0]["ret"], out2[0]["ret"])
    assert glob2["stats"]["value_loss"] != glob["stats"]["value_loss"]
    out3, _ = pipeline([dict(sh, values_old=sh["values_old"] + 0.25)], cfg)
    assert not np.array_equal(out[0]["adv"], out3[0]["adv"])
    # R_t - A_t = V_old(s_t) on valid tokens (P:195 R_t = A_t + V(s_t))
    m = _valid(sh)
    np.testing.assert_allclose((out[0]["ret"] - out[0]["adv"])[m], sh["values_old"][m], rtol=0, atol=1e-14)


# ----------------------------------------------------------------------------- global whitening
@pytest.mark.parametrize("kind", ["gae", "rpp"])
def test_pipeline_global_whitening_moments(kind):
    """P:201 advantage normalisation, global over all ranks (Z18, Z19): over the valid
    tokens of every shard the whitened advantages have mean 0 and std sigma/(sigma+1e-8)."""
    shards = [_random_shard(3, 7, 40 + i) for i in range(3)]
    out, glob = pipeline(shards, dict(adv_kind=kind, whiten=True, gamma=0.99, lam=0.9))
    a = np.concatenate([o["adv"][_valid(s)] for o, s in zip(out, shards)])
    aw = np.concatenate([o["adv_w"][_valid(s)] for o, s in zip(out, shards)])
    assert abs(aw.mean()) < 1e-14
    assert abs(aw.std() - a.std() / (a.std() + 1e-8)) < 1e-13
    assert abs(glob["adv_mean"] - a.mean()) < 1e-14 and abs(glob["adv_std"] - a.std()) < 1e-14


# ----------------------------------------------------------------------------- NEXT-2 helpers
def test_lengths_from_mask_pins():
    """Z10: leading-ones count of right-padded masks; a non-prefix row is counted and
    keeps its leading prefix (brute force on every 0/1 mask of T = 6)."""
    T = 6
    rows = np.array([[(i >> t) & 1 for t in range(T)] for i in range(1 << T)], np.uint8)
    L, bad = oracle.lengths_from_mask(rows)
    for r, Lr in zip(rows, L):
        lead = 0
        while lead < T and r[lead]:
            lead += 1
        assert Lr == lead
    prefix = [all(r[t] >= r[t + 1] for t in range(T - 1)) for r in rows]
    assert bad == (1 << T) - sum(prefix) and sum(prefix) == T + 1
    Ls = rng.integers(0, 50, size=40).astype(np.int32)
    m = (np.arange(49)[None, :] < Ls[:, None]).astype(np.uint8)
    L2, bad2 = oracle.lengths_from_mask(m)
    assert bad2 == 0 and np.array_equal(L2, np.minimum(Ls, 49))


def test_keep_compact_pins():
    """NEXT-2 (DAPO): kept groups in increasing order (library routine on
    random masks; the GRPO keep flags of a batch with constant groups)."""
    for n in (0, 1, 7, 300):
        k = (rng.random(n) < 0.5).astype(np.uint8)
        assert np.array_equal(oracle.keep_compact(k), np.flatnonzero(k))
    R = np.array([1, 1, 1, 1, 0, 1, 0, 0, 0, 0, 0, 0, 0.5, 0.5, 0.5, 0.25], float)
    _, keep = oracle.group_advantages(R, 4)
    assert list(oracle.keep_compact(keep)) == [1, 3]


def test_dapo_keep_threshold_boundary():
    """a group is dropped iff max - min < 1e-12, so a spread of exactly 1e-12 is kept."""
    R = np.array([0.0, 1e-12, 0.0, 0.99e-12, 5.0, 5.0, 0.0, 1.0])
    assert 1e-12 - 0.0 == 1e-12
    _, keep = oracle.group_advantages(R, 2)
    assert list(keep) == [1, 0, 0, 1]


@pytest.mark.parametrize("kind", ["gae", "rpp", "grpo"])
def test_pipeline_per_token_outputs_shard_invariant(kind):
    """every per-token output (A', dL/dlogp, dL/dV) is the same whether the
    batch is one rank or split into contiguous rank shards: N, mu, sigma are global."""
    G = 2
    full = _random_shard(12, 6, 77, with_values=kind == "gae", group_reward=kind == "grpo", G=G)
    cfg = dict(adv_kind=kind, group_size=G, kl_mode="loss" if kind == "grpo" else "reward", beta_loss=0.01,
               beta_reward=0.05, c2=0.01, eps_v=0.2, c1=0.5)
    o1, _ = pipeline([full], cfg)
    for cuts in ([0, 4, 12], [0, 2, 6, 12]):
        shards = [{k: v[s:e] for k, v in full.items()} for s, e in zip(cuts[:-1], cuts[1:])]
        on, _ = pipeline(shards, cfg)
        for key in ("adv_w", "dlogp", "dv"):
            np.testing.assert_allclose(np.concatenate([o[key] for o in on]), o1[0][key], rtol=1e-12, atol=1e-15,
                                       err_msg=key)
