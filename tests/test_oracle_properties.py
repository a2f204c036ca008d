"""Property-based pins of the oracle (hypothesis, seeded and bounded): invariances and
identities the paper's definitions imply, on random small inputs.  Each would catch a
plausible slip the fixed examples of test_oracle_pins.py might not (an index or sign
error that happens to vanish on a worked example).

  S1  vocabulary permutation invariance; inv_temp t on x equals
                        inv_temp 1 on t*x; sum_v exp(logp_v) = 1; H in [0, ln V];
                        logp = x_y - lse exactly.
  S2    k1 antisymmetric, k2 symmetric and >= 0, k3 >= 0 (to ulp(1)) with
                        k3(d) - k3(-d) = e^-d - e^d + 2d.
  S4           with V = 0 GAE is linear in the rewards; lambda = 1 gives the
                        discounted return minus V for any V.
  S6           whitening is invariant to A -> a A + b (a > 0) up to the 1e-8
                        guard.
  S7           for A' > 0 the objective is non-decreasing in rho and capped at
                        (1 + eps_high) A'; for A' < 0 it is capped at (1 - eps_low) A'.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

hyp = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402

import oracle  # noqa: E402

SET = settings(max_examples=60, deadline=None, derandomize=True)
floats = st.floats(min_value=-30.0, max_value=30.0, allow_nan=False, allow_infinity=False)


@SET
@given(st.lists(floats, min_size=1, max_size=40), st.integers(0, 10 ** 6), st.integers(0, 10 ** 6))
def test_s1_permutation_invariance_and_normalisation(xs, yseed, pseed):
    x = np.array(xs)
    V = x.size
    y = yseed % V
    perm = np.random.default_rng(pseed).permutation(V)
    lse, logp, H = oracle.row_logsoftmax(x, y)
    lse2, logp2, H2 = oracle.row_logsoftmax(x[perm], int(np.flatnonzero(perm == y)[0]))
    assert abs(lse - lse2) <= 1e-12 * max(1.0, abs(lse))
    assert abs(logp - logp2) <= 1e-12 * max(1.0, abs(logp))
    assert abs(H - H2) <= 1e-12 * max(1.0, H)
    assert logp == pytest.approx(x[y] - lse, abs=1e-12 * max(1.0, abs(lse)))
    tot = sum(math.exp(oracle.row_logsoftmax(x, v)[1]) for v in range(V))
    assert abs(tot - 1.0) <= 1e-12
    assert -1e-12 <= H <= math.log(V) + 1e-12


@SET
@given(st.lists(floats, min_size=2, max_size=24), st.floats(min_value=0.2, max_value=4.0), st.integers(0, 10 ** 6))
def test_s1_temperature_is_a_logit_scale(xs, inv_temp, yseed):
    x = np.array(xs, dtype=np.float32)[None, None, :]
    y = np.array([[yseed % x.shape[2]]], dtype=np.int32)
    L = np.array([1], dtype=np.int32)
    a = oracle.logprobs(x, y, L, inv_temp)
    b = oracle.logprobs((x.astype(np.float64) * inv_temp), y, L, 1.0)
    for k in ("logp", "entropy", "lse"):
        assert a[k][0, 0] == pytest.approx(b[k][0, 0], rel=1e-12, abs=1e-12)


@SET
@given(st.floats(min_value=-20.0, max_value=20.0, allow_nan=False))
def test_s2_estimator_identities(d):
    assert oracle.kl(d, "k1") == -oracle.kl(-d, "k1")
    assert oracle.kl(d, "k2") == oracle.kl(-d, "k2") >= 0.0
    k3p, k3m = oracle.kl(d, "k3"), oracle.kl(-d, "k3")
    # k3 = e^-d - 1 + d >= 0 mathematically; the fp64 formula cancels to within ulp(1)
    assert k3p >= -2.3e-16 and k3m >= -2.3e-16
    assert k3p - k3m == pytest.approx(math.exp(-d) - math.exp(d) + 2 * d, rel=1e-9, abs=1e-12)


@SET
@given(st.integers(1, 12), st.floats(min_value=0.0, max_value=1.0), st.floats(min_value=0.0, max_value=1.0),
       st.integers(0, 10 ** 6))
def test_s4_gae_linearity_and_lambda_one(T, gamma, lam, seed):
    rng = np.random.default_rng(seed)
    L = np.array([T, max(0, T - 3)], dtype=np.int32)
    r1, r2 = rng.normal(size=(2, T)), rng.normal(size=(2, T))
    Z = np.zeros((2, T))
    a1, _ = oracle.gae(L, r1, Z, gamma, lam)
    a2, _ = oracle.gae(L, r2, Z, gamma, lam)
    a12, _ = oracle.gae(L, r1 + r2, Z, gamma, lam)
    assert np.allclose(a12, a1 + a2, rtol=1e-12, atol=1e-12)
    V = rng.normal(size=(2, T))
    a, ret = oracle.gae(L, r1, V, gamma, 1.0)
    G = oracle.discounted_returns(L, r1, gamma)
    for b in range(2):
        n = int(L[b])
        assert np.allclose(a[b, :n], G[b, :n] - V[b, :n], rtol=1e-12, atol=1e-12)
        assert np.allclose(ret[b, :n], G[b, :n], rtol=1e-12, atol=1e-12)


@SET
@given(st.lists(st.floats(min_value=-5.0, max_value=5.0), min_size=3, max_size=30),
       st.floats(min_value=0.5, max_value=20.0), st.floats(min_value=-10.0, max_value=10.0))
def test_s6_whitening_affine_invariance(xs, a, b):
    x = np.array(xs)
    m1, s1, _ = oracle.whiten_moments(x)
    if s1 < 1e-3:
        return
    m2, s2, _ = oracle.whiten_moments(a * x + b)
    for v in x:
        w1 = oracle.whiten_value(v, m1, s1)
        w2 = oracle.whiten_value(a * v + b, m2, s2)
        assert w1 == pytest.approx(w2, rel=1e-6, abs=1e-6)   # the 1e-8 guard scales by 1/a


@SET
@given(st.floats(min_value=-3.0, max_value=3.0), st.floats(min_value=0.01, max_value=5.0),
       st.floats(min_value=0.05, max_value=0.5), st.floats(min_value=0.05, max_value=0.5))
def test_s7_objective_monotone_and_capped(logratio, advmag, eps_low, eps_high):
    lo = np.zeros((1, 2))
    for sign in (1.0, -1.0):
        A = np.full((1, 2), sign * advmag)
        ln = np.array([[logratio, logratio + 0.1]])
        res = oracle.ppo_loss(np.array([2], dtype=np.int32), ln, lo, A, eps_low=eps_low, eps_high=eps_high)
        obj = res["obj"][0]
        if sign > 0:
            assert obj[1] >= obj[0] - 1e-12
            assert obj.max() <= (1 + eps_high) * advmag + 1e-12
        else:
            assert np.all(obj <= (1 - eps_low) * (-advmag) + 1e-12)
            assert obj[1] <= obj[0] + 1e-12
