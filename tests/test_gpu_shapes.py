"""Seeded random shape sweep of the whole iteration (S1..S10) against the fp64 oracle:
tiny and odd vocabularies (V = 1, 2, 3, 7, ... 50257: the TMA path, the generic
unaligned path and their tails), B and T from 1, lengths with zeros and full rows,
padded row pitches (strided logits views), fp32 and bf16, inv_temp != 1, every
advantage kind.  S1 outputs are compared end to end from the logits (2e-3 absolute,
the north star's bound, with the 1e-4 regression alarm of tests/parity.py); every
downstream stage stage-isolated at the 1e-5 relative bar (test_gpu_parity helpers).
"""
from __future__ import annotations

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
VOCABS = [1, 2, 3, 7, 8, 9, 31, 100, 257, 1000, 4097, 8193, 50257]
KINDS = ["gae", "rpp", "rpp_baseline", "grpo"]


def _case(i):
    rng = np.random.default_rng(1000 + i)
    V = VOCABS[i % len(VOCABS)]
    kind = KINDS[i % len(KINDS)]
    G = 2 if kind in ("grpo", "rpp_baseline") else 1
    B = int(rng.integers(1, 5)) * G
    T = int(rng.choice([1, 2, 5, 16, 33, 70]))
    L = rng.integers(0, T + 1, size=B)
    if i % 3 == 0:
        L[0] = T                       # a full row
    if L.sum() == 0:
        L[-1] = max(1, T // 2)
    dtype = "bf16" if i % 2 else "f32"
    pad = int(rng.choice([0, 0, 1, 3, 8]))
    inv_temp = float(rng.choice([1.0, 1.0, 1 / 0.7, 2.0]))
    mb = int(rng.integers(1, B + 1))
    return dict(V=V, kind=kind, G=G, B=B, T=T, L=L.astype(np.int32), dtype=dtype, pad=pad, inv_temp=inv_temp, mb=mb)


@pytest.mark.parametrize("i", range(int(os.environ.get("ORL_SHAPE_SWEEP", "26"))))  # extended runs: ORL_SHAPE_SWEEP=N
def test_random_shapes_end_to_end(i):
    from tests.test_gpu_parity import _check_downstream, _isolated_oracle, _np
    cs = _case(i)
    V, B, T, kind, G = cs["V"], cs["B"], cs["T"], cs["kind"], cs["G"]
    c = dict(synth.CONFIGS["tiny"], V=V, T=T, adv_kind=kind, group_size=G)
    if kind == "grpo":
        c.update(kl_mode="loss", kl_est_loss="k2", beta_loss=0.05, whiten=False, eps_v=0.0, c1=0.0)
    if kind.startswith("rpp"):
        c.update(eps_v=0.0, c1=0.0)
    batch = synth.make_batch(i, B, T, V, cs["dtype"], "stress", cs["L"], "group_bernoulli" if G > 1 else "normal",
                             G)
    cfg = PathConfig.from_synth(c)
    cfg.inv_temp = cs["inv_temp"]
    g = {k: (v.to(DEV) if isinstance(v, torch.Tensor) else v) for k, v in batch.items()}
    if cs["pad"]:                      # row pitch V + pad: strided [B, T, V] views
        for r in ("old", "ref", "new"):
            x = g[f"logits_{r}"]
            buf = torch.full((B, T, V + cs["pad"]), float("nan"), dtype=x.dtype, device=DEV)
            buf[..., :V] = x
            g[f"logits_{r}"] = buf[..., :V]
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    ctx = orl.Context(0)
    bufs = Buffers(B, T, DEV, G)
    status, st = run_iteration(ctx, g, cfg, bufs, src, mb=cs["mb"])
    torch.cuda.synchronize()
    ctx.close()
    assert status == "ORL_OK", (status, cs)
    npb = synth.batch_to_numpy(batch)
    m = parity.valid_mask(npb["lengths"], T)
    for role, buf in (("old", bufs.logp_old), ("ref", bufs.logp_ref), ("new", bufs.logp_new)):
        o = oracle.logprobs(npb[f"logits_{role}"], npb["tokens"], npb["lengths"], cs["inv_temp"])
        parity.check_abs(f"logp_{role}", _np(buf), o["logp"], m)
        if role == "new":
            parity.check_abs("entropy", _np(bufs.entropy), o["entropy"], m)
            if V == 1:                 # a one-word vocabulary: logp = 0 and H = 0, up to fp32 rounding
                assert np.all(np.abs(_np(buf)[m]) <= 1e-6) and np.all(np.abs(_np(bufs.entropy)[m]) <= 1e-6)
    ocfg = dict(c, kl_mode=c.get("kl_mode", "reward"))
    ocfg["inv_temp"] = cs["inv_temp"]
    out_i, glob_i = _isolated_oracle(npb, bufs, ocfg)
    # near-constant advantages (|mu|/sigma > 1e4) are compared like the rest: the actor pass
    # whitens adv + adv_lo, the fp64 scan value (Z33)
    raw = None
    if kind == "rpp_baseline":
        raw = oracle.shape_rewards(npb["lengths"], _np(bufs.logp_old), _np(bufs.logp_ref), c["kl_est_reward"],
                                   c["beta_reward"], npb["seq_reward"])[1]
    _check_downstream(bufs, out_i[0], glob_i, st, m, f"shape-{i}-{kind}-V{V}", raw_shaped=raw)
