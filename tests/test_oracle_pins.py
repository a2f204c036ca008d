"""Pins for the fp64 oracle (CPU only).

Each test checks the oracle against something other than itself: values the
spec/paper fix for a worked example (tests/golden/, each with its citation),
closed forms, 50-digit mpmath brute force, exact enumeration, independent
algorithms (backward recursions, numpy/scipy library routines), invariants and
finite differences.  A plausible slip anywhere in orl_oracle.c (dropped term,
wrong sign/index, transposed operand, population vs sample std, strict vs
non-strict clip test) fails at least one of them.
"""
import math

import mpmath as mp
import numpy as np
import pytest
import torch

import oracle

mp.mp.dps = 50
rng = np.random.default_rng(20240511)


# ----------------------------------------------------------------------------- S1
def _mp_row(x, y):
    xs = [mp.mpf(float(v)) for v in x]
    lse = mp.log(mp.fsum(mp.e ** v for v in xs))
    H = -mp.fsum(mp.e ** (v - lse) * (v - lse) for v in xs)
    return lse, xs[y] - lse, H


def test_s1_worked_example_w1(golden):
    g = golden("w1_logsoftmax_v4.json")
    lse, logp, H = oracle.row_logsoftmax(np.array(g["x"], float), g["y"])
    assert abs(lse - float(g["lse"])) < 1e-14
    assert abs(logp - float(g["logp"])) < 1e-14
    assert abs(H - float(g["entropy"])) < 1e-14


@pytest.mark.parametrize("V", [1, 2, 3, 7, 16, 32])
def test_s1_vs_mpmath_bruteforce(V):
    for trial in range(8):
        scale = [0.5, 3.0, 20.0][trial % 3]
        x = rng.normal(0, scale, V)
        y = int(rng.integers(V))
        lse, logp, H = oracle.row_logsoftmax(x, y)
        mlse, mlogp, mH = _mp_row(x, y)
        assert abs(lse - float(mlse)) <= 1e-13 * max(1.0, abs(float(mlse)))
        assert abs(logp - float(mlogp)) <= 1e-13 * max(1.0, abs(float(mlogp)))
        assert abs(H - float(mH)) <= 1e-12


@pytest.mark.parametrize("V", [128256, 152064, 32])
def test_s1_uniform_row(V):
    lse, logp, H = oracle.row_logsoftmax(np.full(V, 0.37), V // 3)
    assert abs(logp + math.log(V)) < 1e-12
    assert abs(H - math.log(V)) < 1e-10


def test_s1_v1_and_two_token_closed_form():
    lse, logp, H = oracle.row_logsoftmax(np.array([3.5]), 0)
    assert logp == 0.0 and H == 0.0
    for a, b in [(0.0, 0.0), (1.0, -2.0), (-5.0, 30.0)]:
        _, lp, _ = oracle.row_logsoftmax(np.array([a, b]), 0)
        softplus = math.log1p(math.exp(b - a)) if b - a < 30 else (b - a) + math.log1p(math.exp(a - b))
        assert abs(lp + softplus) < 1e-13


def test_s1_normalisation_and_shift_invariance():
    V = 1000
    x = rng.normal(0, 4, V)
    total = mp.fsum(mp.e ** mp.mpf(oracle.row_logsoftmax(x, y)[1]) for y in range(0, V))
    assert abs(float(total) - 1.0) < 1e-12
    a = oracle.row_logsoftmax(x, 17)
    b = oracle.row_logsoftmax(x + 123.25, 17)
    assert abs(a[1] - b[1]) < 1e-12 and abs(a[2] - b[2]) < 1e-11


def test_s1_spike_row_entropy_near_zero():
    V = 128256
    x = np.zeros(V)
    x[5] = 60.0
    lse, logp, H = oracle.row_logsoftmax(x, 5)
    bound = (V - 1) * math.exp(-60) * 61 + 1e-15      # H <= sum_{v != y} p_v (1 - ln p_v) ...
    assert 0.0 <= H <= bound
    assert abs(logp) < V * math.exp(-60) * 1.01


def test_s1_batch_layout_masks_bf16_and_errors():
    B, T, V = 3, 5, 33
    x32 = rng.normal(0, 2, (B, T, V)).astype(np.float32)
    bf = torch.from_numpy(x32).to(torch.bfloat16)
    bits = bf.view(torch.int16).numpy().view(np.uint16)
    x_exact = bf.to(torch.float64).numpy()                 # torch's bf16 -> f64 (independent)
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    lengths = np.array([5, 2, 0], np.int32)
    inv_temp = 1.0 / 0.7
    out = oracle.logprobs(bits, tokens, lengths, inv_temp)
    for b in range(B):
        for t in range(T):
            if t >= lengths[b]:
                for k in ("logp", "entropy", "lse", "gathered"):
                    assert out[k][b, t] == 0.0
                continue
            mlse, mlogp, mH = _mp_row(x_exact[b, t] * inv_temp, tokens[b, t])
            assert abs(out["logp"][b, t] - float(mlogp)) < 1e-12
            assert abs(out["entropy"][b, t] - float(mH)) < 1e-12
            assert out["gathered"][b, t] == x_exact[b, t, tokens[b, t]]
    # strided view (response-aligned slice of a longer sequence, Z1)
    full = rng.normal(0, 1, (2, 9, V)).astype(np.float32)
    view = full[:, 3:8, :]
    o2 = oracle.logprobs(view, tokens[:2], np.array([5, 5], np.int32))
    o3 = oracle.logprobs(np.ascontiguousarray(view), tokens[:2], np.array([5, 5], np.int32))
    assert np.array_equal(o2["logp"], o3["logp"])
    # out-of-vocabulary token and NaN row are input errors (Z26)
    tok_bad = tokens.copy()
    tok_bad[0, 1] = V
    x_nan = x32.copy()
    x_nan[0, 2, 4] = np.nan
    o4 = oracle.logprobs(x_nan, tok_bad, lengths)
    assert o4["n_token_range"] == 1 and o4["n_nonfinite"] == 1
    assert math.isnan(o4["logp"][0, 1]) and math.isnan(o4["logp"][0, 2])


def test_s1_neg_inf_entries_allowed():
    x = np.array([0.0, -np.inf, 1.0, -np.inf])
    lse, logp, H = oracle.row_logsoftmax(x, 2)
    assert abs(lse - math.log(1 + math.e)) < 1e-14
    p0 = 1 / (1 + math.e)
    assert abs(H - (-(p0 * math.log(p0)) - (1 - p0) * math.log(1 - p0))) < 1e-14


# ----------------------------------------------------------------------------- S2
def test_s2_spec_examples(golden):
    g = golden("spec_examples.json")
    for k in ("k1", "k2", "k3"):
        assert oracle.kl(0.0, k) == 0.0
    assert abs(oracle.kl(g["kl_d"], "k2") - float(g["k2"])) < 1e-16
    assert abs(oracle.kl(g["kl_d"], "k3") - float(g["k3"])) < 1e-15
    assert abs(oracle.kl(g["kl_d_neg"], "k3") - float(g["k3_neg"])) < 1e-15
    assert oracle.kl(0.2, "k1") == 0.2 and oracle.kl(-0.3, "k1") == -0.3


def test_s2_exact_enumeration_w2(golden):
    g = golden("w2_kl_enumeration.json")
    pi, pr = np.array(g["pi"]), np.array(g["pi_ref"])
    from scipy.special import rel_entr
    kl_scipy = float(rel_entr(pi, pr).sum())
    d = np.log(pi) - np.log(pr)
    e1 = sum(p * oracle.kl(di, "k1") for p, di in zip(pi, d))
    e2 = sum(p * oracle.kl(di, "k2") for p, di in zip(pi, d))
    e3 = sum(p * oracle.kl(di, "k3") for p, di in zip(pi, d))
    assert abs(e1 - float(g["kl"])) < 1e-12 and abs(e1 - kl_scipy) < 1e-12
    assert abs(e2 - float(g["e_k2"])) < 1e-12
    # k3 with d = logp - logp_ref, samples from pi: E[exp(-d)] = 1 -> E[k3] = E[k1]
    assert abs(e3 - float(g["kl"])) < 1e-12


def test_s2_nonnegativity_and_gradients():
    ds = np.concatenate([rng.normal(0, 3, 20000), [-30, -1e-9, 0, 1e-9, 30]])
    for d in ds:
        assert oracle.kl(d, "k2") >= 0.0
        assert oracle.kl(d, "k3") >= 0.0
    for d in rng.normal(0, 1, 50):
        for k in ("k1", "k2", "k3"):
            h = 1e-6
            fd = (oracle.kl(d + h, k) - oracle.kl(d - h, k)) / (2 * h)
            assert abs(fd - oracle.kl_grad(d, k)) < 1e-7


# ----------------------------------------------------------------------------- S3
def test_s3_worked_example_w3(golden):
    g = golden("w3_shaping_gae_t3.json")
    kl, r = oracle.shape_rewards([3], [g["logp_old"]], [g["logp_ref"]], g["kl"], g["beta"], [g["R"]])
    np.testing.assert_allclose(kl[0], g["kl_out"], atol=1e-15)
    np.testing.assert_allclose(r[0], g["shaped"], atol=1e-15)


def test_s3_special_cases_and_sum():
    B, T = 4, 9
    L = np.array([9, 4, 1, 0], np.int32)
    a, b = rng.normal(-1, 0.5, (B, T)), rng.normal(-1, 0.5, (B, T))
    R = rng.normal(0, 1, B)
    _, r0 = oracle.shape_rewards(L, a, b, "k3", 0.0, R)        # beta = 0 -> r' = r
    for i in range(B):
        expect = np.zeros(T)
        if L[i] > 0:
            expect[L[i] - 1] = R[i]
        assert np.array_equal(r0[i], expect)
    _, r1 = oracle.shape_rewards(L, a, b, "k1", 1.0, np.zeros(B))  # r' = -(logp - logp_ref)
    for i in range(B):
        np.testing.assert_allclose(r1[i, : L[i]], -(a[i, : L[i]] - b[i, : L[i]]), atol=1e-15)
        assert np.all(r1[i, L[i]:] == 0.0)
    kl, r2 = oracle.shape_rewards(L, a, b, "k2", 0.3, R)
    for i in range(B):
        if L[i]:
            assert abs(r2[i].sum() - (R[i] - 0.3 * kl[i].sum())) < 1e-12


# ----------------------------------------------------------------------------- S4
def _gae_backward(r, V, L, g, lam):
    """Independent algorithm: the standard backward recursion."""
    A = np.zeros_like(r)
    last = 0.0
    for t in reversed(range(L)):
        vn = V[t + 1] if t + 1 < L else 0.0
        last = r[t] + g * vn - V[t] + g * lam * last
        A[t] = last
    return A


def test_s4_worked_example_w3(golden):
    g = golden("w3_shaping_gae_t3.json")
    for c in g["cases"]:
        A, R = oracle.gae([3], [g["shaped"]], [g["V"]], c["gamma"], c["lam"])
        np.testing.assert_allclose(A[0], c["adv"], atol=1e-14)
        if "ret" in c:
            np.testing.assert_allclose(R[0], c["ret"], atol=1e-14)


def test_s4_recursion_vs_definition_1000_trajectories():
    # recursion == double-sum within 1e-10 for gamma,lambda in {0,.5,.95,1}^2
    grid = [0.0, 0.5, 0.95, 1.0]
    n = 0
    for g in grid:
        for lam in grid:
            for _ in range(63):
                T = int(rng.integers(1, 33))
                L = int(rng.integers(0, T + 1))
                r, V = rng.normal(0, 1, (1, T)), rng.normal(0, 1, (1, T))
                A, R = oracle.gae([L], r, V, g, lam)
                ref = _gae_backward(r[0], V[0], L, g, lam)
                assert np.max(np.abs(A[0] - ref)) < 1e-10
                np.testing.assert_allclose(R[0, :L], A[0, :L] + V[0, :L], atol=1e-15)
                assert np.all(A[0, L:] == 0) and np.all(R[0, L:] == 0)
                n += 1
    assert n >= 1000


def test_s4_closed_forms():
    T = 40
    r, V = rng.normal(0, 1, (1, T)), rng.normal(0, 1, (1, T))
    # lambda = 0 -> A = delta exactly
    A, _ = oracle.gae([T], r, V, 0.9, 0.0)
    delta = r[0] + 0.9 * np.append(V[0, 1:], 0.0) - V[0]
    np.testing.assert_allclose(A[0], delta, atol=1e-15)
    # lambda = 1 -> A = discounted return - V (north star); computed with numpy powers
    for g in (1.0, 0.9):
        A, _ = oracle.gae([T], r, V, g, 1.0)
        disc = np.array([sum(g ** (s - t) * r[0, s] for s in range(t, T)) for t in range(T)])
        np.testing.assert_allclose(A[0], disc - V[0], atol=1e-12)
    # gamma = lambda = 1, V = 0 -> reward-to-go, reversed cumsum
    A, _ = oracle.gae([T], r, np.zeros((1, T)), 1.0, 1.0)
    np.testing.assert_allclose(A[0], np.cumsum(r[0][::-1])[::-1], atol=1e-12)


def test_s4p_reinforce_returns():
    T = 30
    r = rng.normal(0, 1, (2, T))
    L = np.array([30, 11], np.int32)
    G1 = oracle.discounted_returns(L, r, 1.0)
    for i in range(2):
        np.testing.assert_allclose(G1[i, : L[i]], np.cumsum(r[i, : L[i]][::-1])[::-1], atol=1e-12)
        assert np.all(G1[i, L[i]:] == 0)
    ones = np.ones((1, T))
    G = oracle.discounted_returns([T], ones, 0.9)
    n = T - np.arange(T)
    np.testing.assert_allclose(G[0], (1 - 0.9 ** n) / (1 - 0.9), atol=1e-12)


# ----------------------------------------------------------------------------- S5
def test_s5_grpo_examples(golden):
    g = golden("spec_examples.json")
    for case in g["grpo"]:
        adv, keep = oracle.group_advantages(case["R"], len(case["R"]))
        np.testing.assert_allclose(adv, case["adv"], atol=1e-12)
        assert keep[0] == (0 if len(set(case["R"])) == 1 else 1)
    adv, _ = oracle.group_advantages([0.9, 0.9, 0.9], 3)
    assert np.all(adv == 0.0)


def test_s5_grpo_vs_numpy_and_group_sums():
    R = rng.random(64)
    R[8:16] = 0.25                       # a constant group
    adv, keep = oracle.group_advantages(R, 8)
    for gi in range(8):
        Rg = R[gi * 8:(gi + 1) * 8]
        if gi == 1:
            assert np.all(adv[8:16] == 0.0) and keep[1] == 0
            continue
        expect = (Rg - Rg.mean()) / (np.std(Rg, ddof=0) + 1e-8)   # population std
        np.testing.assert_allclose(adv[gi * 8:(gi + 1) * 8], expect, rtol=1e-12)
        assert abs(adv[gi * 8:(gi + 1) * 8].sum()) < 1e-9 and keep[gi] == 1
    with pytest.raises(ValueError):
        oracle.group_advantages(R[:10], 8)
    base = oracle.group_mean_subtract(R, 8)
    for gi in range(8):
        np.testing.assert_allclose(base[gi * 8:(gi + 1) * 8], R[gi * 8:(gi + 1) * 8] - R[gi * 8:(gi + 1) * 8].mean(), atol=1e-15)


def test_s5_dynamic_sampling_keep_brute_force():
    R = rng.integers(0, 2, 40).astype(float)
    _, keep = oracle.group_advantages(R, 4)
    for gi in range(10):
        assert keep[gi] == (1 if len(set(R[gi * 4:(gi + 1) * 4])) > 1 else 0)


# ----------------------------------------------------------------------------- S6
def test_s6_whitening(golden):
    g = golden("spec_examples.json")
    a = np.array(g["whiten"][0]["a"], float)
    m, s, w = oracle.whiten_moments(a)
    assert not w
    np.testing.assert_allclose([oracle.whiten_value(v, m, s) for v in a], g["whiten"][0]["out"], atol=1e-15)
    m, s, _ = oracle.whiten_moments(np.full(17, 3.25))
    assert m == 3.25 and s == 0.0 and oracle.whiten_value(3.25, m, s) == 0.0
    x = rng.normal(5, 3, 10001)
    m, s, _ = oracle.whiten_moments(x)
    assert abs(m - np.mean(x)) < 1e-12 and abs(s - np.std(x, ddof=0)) < 1e-12
    y = np.array([oracle.whiten_value(v, m, s) for v in x])
    assert abs(y.mean()) < 1e-9 and abs(y.std() - 1) < 1e-6
    assert oracle.whiten_moments(np.array([2.0]))[2] is True       # < 2 tokens: warn, no-op


# ----------------------------------------------------------------------------- S7-S10
def test_s7_worked_example_w5(golden):
    g = golden("w5_ppo_loss.json")
    lo = [-1.0, -1.0 - math.log(1.5), -2.0 + math.log(2.0), -0.3]
    res = oracle.ppo_loss([4], [g["logp_new"]], [lo], [g["adv"]], eps_low=g["eps_low"],
                          eps_high=g["eps_high"])
    np.testing.assert_allclose(res["obj"][0], g["obj"], atol=1e-14)
    assert list(res["clipped"][0]) == g["clipped"]
    st = oracle.stats(res["sums"])
    assert abs(st["policy_loss"] - g["policy_loss"]) < 1e-14
    assert st["clip_frac"] == g["clip_frac"]
    np.testing.assert_allclose(st["ratio_mean"], np.mean(g["rho"]), atol=1e-14)
    vc = g["value_case"]
    res = oracle.ppo_loss([1], [[-1.0]], [[-1.0]], [[1.0]], ret=[[vc["ret"]]], v_new=[[vc["v_new"]]],
                          v_old=[[vc["v_old"]]], eps_v=vc["eps_v"], c1=1.0)
    assert abs(res["vl"][0, 0] - vc["vl"]) < 1e-14 and res["dv"][0, 0] == vc["dvl"]
    # per-token decision bits: W5's value case takes the clipped branch (0.64 > 0.25),
    # the policy term is on-policy (rho = 1, never clipped, Z16)
    assert res["flags"][0, 0] == 2
    # ratio guard (Z22) and a non-finite loss term set bits 2 and 3
    r2 = oracle.ppo_loss([2], [[0.0, -40.0]], [[0.0, -5.0]], [[1.0, float("nan")]])
    assert list(r2["flags"][0]) == [0, 4 | 8]


def test_s7_spec_examples(golden):
    for case in golden("spec_examples.json")["ratio_examples"]:
        res = oracle.ppo_loss([1], [[math.log(case["rho"])]], [[0.0]], [[case["A"]]],
                              eps_low=case["eps_low"], eps_high=case["eps_high"])
        assert abs(res["obj"][0, 0] - case["obj"]) < 1e-12 and res["clipped"][0, 0] == 1
    # on-policy identity (north star): ratio 1, loss -1, zero clip fraction
    lp = rng.normal(-1, 0.3, (3, 7))
    res = oracle.ppo_loss([7, 7, 7], lp, lp, np.ones((3, 7)))
    st = oracle.stats(res["sums"])
    assert st["policy_loss"] == -1.0 and st["clip_frac"] == 0.0 and st["ratio_mean"] == 1.0
    assert st["approx_kl_old"] == 0.0
    np.testing.assert_allclose(res["dlogp"], -1.0 / 21, atol=1e-16)


def _loss_fn(lp_new, kw):
    res = oracle.ppo_loss(kw["L"], lp_new, kw["lo"], kw["A"], logp_ref=kw["lr"], ret=kw["R"],
                          v_new=kw["vn"], v_old=kw["vo"], eps_low=0.2, eps_high=0.28, eps_v=0.2,
                          c1=0.5, beta_loss=0.05, kl_est=kw["k"], kl_in_loss=True)
    st = oracle.stats(res["sums"], c1=0.5, beta_loss=0.05, kl_in_loss=True)
    return st["total_loss"], res


@pytest.mark.parametrize("k", ["k1", "k2", "k3"])
def test_s7_gradient_finite_differences(k):
    """d total / d logp_new and d total / d V_new by central differences."""
    B, T = 2, 6
    L = np.array([6, 4], np.int32)
    kw = dict(L=L, lo=rng.normal(-1, 0.2, (B, T)), A=rng.normal(0, 1, (B, T)), lr=rng.normal(-1, 0.2, (B, T)),
              R=rng.normal(0, 1, (B, T)), vo=rng.normal(0, 1, (B, T)), k=k)
    kw["vn"] = kw["vo"] + rng.normal(0, 0.3, (B, T))
    lp = kw["lo"] + rng.normal(0, 0.25, (B, T))
    _, res = _loss_fn(lp, kw)
    h = 1e-6
    n_clip = 0
    for b in range(B):
        for t in range(L[b]):
            p, m = lp.copy(), lp.copy()
            p[b, t] += h
            m[b, t] -= h
            fd = (_loss_fn(p, kw)[0] - _loss_fn(m, kw)[0]) / (2 * h)
            assert abs(fd - res["dlogp"][b, t]) < 1e-7
            if res["clipped"][b, t]:
                n_clip += 1
                # clip branch: only the KL term remains
                d = lp[b, t] - kw["lr"][b, t]
                assert abs(res["dlogp"][b, t] - 0.05 * oracle.kl_grad(d, k) / L.sum()) < 1e-15
            vp, vm = dict(kw), dict(kw)
            vp["vn"], vm["vn"] = kw["vn"].copy(), kw["vn"].copy()
            vp["vn"][b, t] += h
            vm["vn"][b, t] -= h
            fdv = (_loss_fn(lp, vp)[0] - _loss_fn(lp, vm)[0]) / (2 * h)
            assert abs(fdv - res["dv"][b, t]) < 1e-7
    assert n_clip > 0


def test_s7_symmetric_relabel_and_masking_and_recomposition():
    B, T = 3, 8
    L = np.array([8, 3, 0], np.int32)
    lo = rng.normal(-1, 0.2, (B, T))
    ln = lo + rng.normal(0, 0.3, (B, T))
    A = rng.normal(0, 1, (B, T))
    r1 = oracle.ppo_loss(L, ln, lo, A, eps_low=0.25, eps_high=0.25)
    assert r1["sums"][5] > 0
    # masked tokens: editing any input there leaves every output bit-identical
    ln2, lo2, A2 = ln.copy(), lo.copy(), A.copy()
    for b in range(B):
        ln2[b, L[b]:] = 99.0
        lo2[b, L[b]:] = -7.0
        A2[b, L[b]:] = np.nan
    r2 = oracle.ppo_loss(L, ln2, lo2, A2, eps_low=0.25, eps_high=0.25)
    for k in ("obj", "dlogp", "sums"):
        assert np.array_equal(r1[k], r2[k])
    # total recomposition within 1e-12
    kw = dict(logp_ref=lo + 0.05, ret=A * 0.5, v_new=A * 0.4, v_old=A * 0.45, entropy=np.abs(A),
              eps_v=0.1, c1=0.7, beta_loss=0.3, kl_est="k3", kl_in_loss=True)
    r3 = oracle.ppo_loss(L, ln, lo, A, **kw)
    st = oracle.stats(r3["sums"], c1=0.7, c2=0.01, beta_loss=0.3, kl_in_loss=True)
    total = st["policy_loss"] + 0.7 * st["value_loss"] - 0.01 * st["entropy"] + 0.3 * st["kl"]
    assert abs(total - st["total_loss"]) < 1e-12
    assert st["n_tokens"] == 11
    # each statistic against its definition written with numpy on the valid tokens
    m = np.zeros((B, T), bool)
    for b in range(B):
        m[b, :L[b]] = True
    rho = np.exp(ln[m] - lo[m])
    assert abs(st["approx_kl_old"] - np.mean(rho - 1 - np.log(rho))) < 1e-14   # k3(old vs new), Z27
    dref = ln[m] - kw["logp_ref"][m]
    assert abs(st["kl"] - np.mean(np.exp(-dref) - 1 + dref)) < 1e-14
    assert abs(st["entropy"] - np.mean(np.abs(A[m]))) < 1e-14
    assert abs(st["ratio_mean"] - np.mean(rho)) < 1e-14
    vn, vo, R = kw["v_new"][m], kw["v_old"][m], kw["ret"][m]
    vc = vo + np.clip(vn - vo, -0.1, 0.1)
    assert abs(st["value_loss"] - np.mean(np.maximum((vn - R) ** 2, (vc - R) ** 2))) < 1e-14
    assert st["value_clip_frac"] == np.mean((vc - R) ** 2 > (vn - R) ** 2)
    Am = A[m]
    cl = np.clip(rho, 0.8, 1.2) * Am < rho * Am
    assert st["clip_frac"] == np.mean(cl)
    assert abs(st["policy_loss"] + np.mean(np.minimum(rho * Am, np.clip(rho, 0.8, 1.2) * Am))) < 1e-14
    # an unclipped value loss equals plain MSE when eps_v <= 0
    r4 = oracle.ppo_loss(L, ln, lo, A, ret=A * 0.5, v_new=A * 0.4, v_old=A * 0.45, eps_v=0.0, c1=1.0)
    mse = sum(((A[b, :L[b]] * 0.4 - A[b, :L[b]] * 0.5) ** 2).sum() for b in range(B))
    assert abs(r4["sums"][2] - mse) < 1e-13


def test_s7_ratio_guard_and_empty():
    res = oracle.ppo_loss([2], [[0.0, -40.0]], [[0.0, -5.0]], [[1.0, 1.0]])
    assert res["sums"][9] == 1
    st = oracle.stats(np.zeros(11))
    assert st["empty"]


# ----------------------------------------------------------------------------- pipeline
def _tiny_batch(seed, B=4, T=16, V=32, bf16=False):
    from paper_2405_11143_b200 import synth
    return synth.tiny_numpy(seed, B=B, T=T, V=V)


@pytest.mark.parametrize("kind", ["gae", "rpp", "rpp_baseline", "grpo"])
def test_pipeline_shard_invariance(kind):
    """Result is invariant to how the batch is split into rank shards."""
    from paper_2405_11143_b200 import synth
    full = synth.tiny_numpy(1, B=8, T=16, V=32)
    cfg = dict(adv_kind=kind, group_size=2, kl_mode="loss" if kind == "grpo" else "reward",
               beta_loss=0.001, kl_est_loss="k2", c2=0.01)
    _, g1 = oracle.pipeline([full], cfg)
    for n in (2, 4):
        shards = synth.split_numpy(full, n)
        _, gn = oracle.pipeline(shards, cfg)
        for k, v in g1["stats"].items():
            if isinstance(v, float):
                assert abs(v - gn["stats"][k]) <= 1e-12 * max(1.0, abs(v)), (k, v, gn["stats"][k])


# ----------------------------------------------------------------------------- NEXT-1
@pytest.mark.parametrize("k", ["k1", "k2", "k3"])
def test_next1_logits_grad_finite_differences(k):
    """dL/dlogits of the whole oracle chain (logprobs -> ppo_loss -> stats total)
    by central differences in fp64, against oracle.logits_grad (NEXT-1)."""
    B, T, V = 2, 3, 6
    L = np.array([3, 2], np.int32)
    x = rng.normal(0, 1.5, (B, T, V))
    tok = rng.integers(0, V, (B, T)).astype(np.int32)
    lo = rng.normal(-1.5, 0.3, (B, T))
    lr = lo + rng.normal(0, 0.2, (B, T))
    A = rng.normal(0, 1, (B, T))
    inv_temp, c2, beta = 1 / 0.8, 0.05, 0.1

    def total(xn):
        o = oracle.logprobs(xn, tok, L, inv_temp)
        res = oracle.ppo_loss(L, o["logp"], lo, A, logp_ref=lr, entropy=o["entropy"], eps_low=0.2,
                              eps_high=0.28, beta_loss=beta, kl_est=k, kl_in_loss=True)
        st = oracle.stats(res["sums"], c2=c2, beta_loss=beta, kl_in_loss=True)
        return st["total_loss"], res

    _, res = total(x)
    g = oracle.logits_grad(x, tok, L, res["dlogp"], inv_temp, c2, float(L.sum()))
    h = 1e-6
    for b in range(B):
        for t in range(T):
            for v in range(V):
                xp, xm = x.copy(), x.copy()
                xp[b, t, v] += h
                xm[b, t, v] -= h
                fd = (total(xp)[0] - total(xm)[0]) / (2 * h)
                assert abs(fd - g[b, t, v]) < 2e-8, (b, t, v, fd, g[b, t, v])
                if t >= L[b]:
                    assert g[b, t, v] == 0.0
    # each valid row's gradient sums to 0 (softmax shift invariance)
    for b in range(B):
        for t in range(L[b]):
            assert abs(g[b, t].sum()) < 1e-13


@pytest.mark.parametrize("c2", [0.0, 0.05])
def test_next1_masked_entries_equal_reduced_vocabulary(c2):
    """Z39: a -inf logit leaves the softmax as if its entry did not exist, so on the finite
    entries the gradient equals that of the row with the entry removed (a plain
    re-evaluation on the reduced vocabulary).  At the -inf entry itself p = 0: with c2 = 0
    the loss has no entropy term and the gradient is -w p = 0 exactly; with c2 != 0 the
    formula's p (ln p + H) is 0 * (-inf) = NaN."""
    V, y, inv_temp, w, n = 9, 4, 1.3, -0.7, 5.0
    x = rng.normal(0, 2.0, V)
    masked = np.array([1, 6])
    xm = x.copy()
    xm[masked] = -np.inf
    with np.errstate(invalid="ignore"):
        g = oracle.logits_grad(xm.reshape(1, 1, V), np.array([[y]], np.int32), np.array([1], np.int32),
                               np.array([[w]]), inv_temp, c2, n)[0, 0]
    keep = np.setdiff1d(np.arange(V), masked)
    gr = oracle.logits_grad(x[keep].reshape(1, 1, -1), np.array([[int(np.searchsorted(keep, y))]], np.int32),
                            np.array([1], np.int32), np.array([[w]]), inv_temp, c2, n)[0, 0]
    assert np.allclose(g[keep], gr, rtol=1e-14, atol=1e-16)
    if c2 == 0.0:
        assert (g[masked] == 0.0).all()
        # and the plain definition: inv_temp w (delta_vy - p_v)
        z = inv_temp * x[keep]
        p = np.exp(z - z.max()) / np.exp(z - z.max()).sum()
        ref = inv_temp * w * ((keep == y).astype(float) - p)
        assert np.allclose(g[keep], ref, rtol=1e-13, atol=1e-16)
    else:
        assert np.isnan(g[masked]).all()


# ----------------------------------------------------------------------------- NEXT-3
def test_next3_kl_controller_spec_examples(golden):
    for c in golden("spec_examples.json")["kl_controller"]:
        b, stop = oracle.kl_controller_step(c["beta"], c["target"], c["horizon"], c["observed"], c["max_kl"])
        assert abs(b - c["beta_out"]) < 1e-15 and stop == c["early_stop"]
    # the proportional error is clipped to +-0.5: far-off observations move beta by 1 +- 0.5/horizon
    assert oracle.kl_controller_step(1.0, 0.01, 2.0, 1e6, 1e9)[0] == 1.25
    assert oracle.kl_controller_step(1.0, 0.01, 2.0, 0.0, 1e9)[0] == 0.75


# ----------------------------------------------------------------------------- NEXT-2 seq-mean
def test_next2_seq_mean_aggregation_definition_and_gradients():
    """Sequence-mean loss aggregation (Z31): against its numpy definition, equal to the
    token mean when every response has the same length, and its per-token
    derivatives by central differences."""
    B, T = 4, 6
    L = np.array([6, 2, 0, 3], np.int32)
    lo = rng.normal(-1, 0.2, (B, T))
    ln = lo + rng.normal(0, 0.3, (B, T))
    A, R = rng.normal(0, 1, (B, T)), rng.normal(0, 1, (B, T))
    vo = rng.normal(0, 1, (B, T))
    vn = vo + rng.normal(0, 0.3, (B, T))
    lr, H = lo + 0.05, np.abs(rng.normal(1, 0.5, (B, T)))
    kw = dict(logp_ref=lr, ret=R, v_new=vn, v_old=vo, entropy=H, eps_v=0.2, c1=0.5, beta_loss=0.1,
              kl_est="k2", kl_in_loss=True, eps_low=0.2, eps_high=0.28)
    res = oracle.ppo_loss(L, ln, lo, A, seq_mean=True, **kw)
    st = oracle.stats(res["sums"], c1=0.5, c2=0.01, beta_loss=0.1, kl_in_loss=True, seq_mean=True, n_seq=3.0)
    seqs = [b for b in range(B) if L[b] > 0]
    per = lambda a: np.mean([a[b, :L[b]].mean() for b in seqs])  # noqa: E731
    assert abs(st["policy_loss"] + per(res["obj"])) < 1e-14
    assert abs(st["value_loss"] - per(res["vl"])) < 1e-14
    assert abs(st["entropy"] - per(H)) < 1e-14
    d = ln - lr
    assert abs(st["kl"] - per(0.5 * d * d)) < 1e-14
    # token-mean shares are unchanged by the aggregation mode
    st_tok = oracle.stats(res["sums"], c1=0.5, c2=0.01, beta_loss=0.1, kl_in_loss=True)
    for k in ("clip_frac", "value_clip_frac", "ratio_mean", "approx_kl_old", "n_tokens"):
        assert st[k] == st_tok[k]
    # equal lengths: seq-mean == token-mean
    Le = np.array([4, 4, 4, 4], np.int32)
    r1 = oracle.ppo_loss(Le, ln, lo, A, seq_mean=True, **kw)
    s1 = oracle.stats(r1["sums"], c1=0.5, c2=0.01, beta_loss=0.1, kl_in_loss=True, seq_mean=True, n_seq=4.0)
    s0 = oracle.stats(r1["sums"], c1=0.5, c2=0.01, beta_loss=0.1, kl_in_loss=True)
    for k in ("policy_loss", "value_loss", "entropy", "kl", "total_loss"):
        assert abs(s1[k] - s0[k]) < 1e-14
    r2 = oracle.ppo_loss(Le, ln, lo, A, **kw)
    np.testing.assert_allclose(r1["dlogp"], r2["dlogp"], rtol=1e-14, atol=1e-17)
    # derivatives of the seq-mean total by central differences
    def tot(lpn, vnn):
        r = oracle.ppo_loss(L, lpn, lo, A, seq_mean=True, **dict(kw, v_new=vnn))
        return oracle.stats(r["sums"], c1=0.5, c2=0.01, beta_loss=0.1, kl_in_loss=True, seq_mean=True,
                            n_seq=3.0)["total_loss"]
    h = 1e-6
    for b in seqs:
        for t in range(L[b]):
            p, m = ln.copy(), ln.copy()
            p[b, t] += h
            m[b, t] -= h
            assert abs((tot(p, vn) - tot(m, vn)) / (2 * h) - res["dlogp"][b, t]) < 1e-7
            p, m = vn.copy(), vn.copy()
            p[b, t] += h
            m[b, t] -= h
            assert abs((tot(ln, p) - tot(ln, m)) / (2 * h) - res["dv"][b, t]) < 1e-7


def test_next2_seq_mean_logits_grad_finite_differences():
    B, T, V = 2, 3, 5
    L = np.array([3, 1], np.int32)
    x = rng.normal(0, 1.5, (B, T, V))
    tok = rng.integers(0, V, (B, T)).astype(np.int32)
    lo = rng.normal(-1.5, 0.3, (B, T))
    A = rng.normal(0, 1, (B, T))

    def total(xn):
        o = oracle.logprobs(xn, tok, L)
        r = oracle.ppo_loss(L, o["logp"], lo, A, entropy=o["entropy"], seq_mean=True)
        return oracle.stats(r["sums"], c2=0.05, seq_mean=True, n_seq=2.0)["total_loss"], r

    _, r = total(x)
    g = oracle.logits_grad(x, tok, L, r["dlogp"], 1.0, 0.05, float(L.sum()), seq_mean=True, n_seq=2.0)
    h = 1e-6
    for b in range(B):
        for t in range(L[b]):
            for v in range(V):
                xp, xm = x.copy(), x.copy()
                xp[b, t, v] += h
                xm[b, t, v] -= h
                assert abs((total(xp)[0] - total(xm)[0]) / (2 * h) - g[b, t, v]) < 2e-8


# ----------------------------------------------------------------------------- NEXT-4
def _bf16_bits(a):
    """Round fp32 values to bf16 bit patterns (RNE) with torch (a library routine)."""
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


def _bf16_val(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def test_next4_lmhead_vs_library_bruteforce():
    """z = h W^T then log-softmax / logsumexp / entropy, all via numpy + scipy."""
    from scipy.special import log_softmax, logsumexp
    R, d, V = 9, 48, 37
    h = _bf16_bits(rng.normal(0, 1, (R, d)))
    W = _bf16_bits(rng.normal(0, 0.3, (V, d)))
    y = rng.integers(0, V, R).astype(np.int32)
    for inv_temp in (1.0, 1.0 / 0.7):
        o = oracle.lmhead_rows(h, W, y, inv_temp)
        z = _bf16_val(h) @ _bf16_val(W).T
        ls = log_softmax(inv_temp * z, axis=1)
        np.testing.assert_allclose(o["lse"], logsumexp(inv_temp * z, axis=1), rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(o["logp"], ls[np.arange(R), y], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(o["entropy"], -(np.exp(ls) * ls).sum(1), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(o["z_y"], z[np.arange(R), y], rtol=1e-14, atol=1e-14)


def test_next4_zero_head_is_uniform():
    """W = 0: every logit is 0 -> lse = ln V, H = ln V, logp = -ln V (closed form)."""
    R, d, V = 5, 16, 50
    h = _bf16_bits(rng.normal(0, 1, (R, d)))
    W = np.zeros((V, d), np.uint16)
    o = oracle.lmhead_rows(h, W, np.arange(R, dtype=np.int32), 1.3)
    np.testing.assert_allclose(o["lse"], math.log(V), rtol=1e-15)
    np.testing.assert_allclose(o["entropy"], math.log(V), rtol=1e-14)
    np.testing.assert_allclose(o["logp"], -math.log(V), rtol=1e-15)


def test_next4_common_row_shift_invariance():
    """W_v -> W_v + w0 for every v adds h.w0 to every logit of the row: logp and
    H are unchanged, lse moves by inv_temp h.w0.  Small-integer bf16 values keep
    every sum exact."""
    R, d, V = 6, 12, 21
    h = _bf16_bits(rng.integers(-3, 4, (R, d)).astype(np.float32))
    W0 = rng.integers(-2, 3, (V, d)).astype(np.float32)
    w0 = rng.integers(-2, 3, d).astype(np.float32)
    y = rng.integers(0, V, R).astype(np.int32)
    a = oracle.lmhead_rows(h, _bf16_bits(W0), y, 0.5)
    b = oracle.lmhead_rows(h, _bf16_bits(W0 + w0), y, 0.5)
    shift = 0.5 * (_bf16_val(h) @ w0.astype(np.float64))
    np.testing.assert_allclose(b["logp"], a["logp"], atol=1e-12)
    np.testing.assert_allclose(b["entropy"], a["entropy"], atol=1e-12)
    np.testing.assert_allclose(b["lse"] - a["lse"], shift, atol=1e-12)


def test_next4_identity_head_reduces_to_s1():
    """W = c I (V = d): z_{r,v} = c h_{r,v}, so NEXT-4 equals S1 on those logits
    and gathered z_y = c h_{r,y}; masked rows (y < 0) are zeros, y >= V is NaN."""
    R, d = 7, 32
    c = 2.0
    hv = rng.normal(0, 2, (R, d)).astype(np.float32)
    h = _bf16_bits(hv)
    W = _bf16_bits(c * np.eye(d, dtype=np.float32))
    y = rng.integers(0, d, R).astype(np.int32)
    y[2] = -1
    y[5] = d
    o = oracle.lmhead_rows(h, W, y, 1.0)
    logits = (c * _bf16_val(h)).astype(np.float32).reshape(1, R, d)
    toks = np.where(y < 0, 0, np.minimum(y, d - 1)).reshape(1, R)
    s1 = oracle.logprobs(logits, toks, np.array([R], np.int32), 1.0)
    for r in range(R):
        if r == 2:
            assert o["logp"][r] == 0.0 and o["entropy"][r] == 0.0 and o["lse"][r] == 0.0
        elif r == 5:
            assert np.isnan(o["logp"][r]) and np.isnan(o["lse"][r])
        else:
            assert abs(o["logp"][r] - s1["logp"][0, r]) < 1e-12
            assert abs(o["entropy"][r] - s1["entropy"][0, r]) < 1e-12
            assert abs(o["z_y"][r] - c * _bf16_val(h)[r, y[r]]) == 0.0
