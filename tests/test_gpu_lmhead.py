"""GPU parity of NEXT-4 (LM-head GEMM on tcgen05 fused with the online LSE)
against the fp64 oracle (oracle.lmhead_rows / lmhead_logprobs), through the
C ABI (orl_lmhead_logprobs, orl_lmhead_ppo_loss).

Tolerance (NEXT-4): the kernel multiplies bf16 inputs
exactly and accumulates in fp32, so |z_gpu - z| <= gamma_d sum_k |h_k W_vk|
with gamma_d ~ d 2^-24 (worst case, Higham); logp and lse move by at most
2 inv_temp max_v of that, entropy likewise.  Every test asserts the error
under min(that bound + 1e-5, 2e-3) -- 2e-3 being the north star's S1 bound.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2405_11143_b200 import synth
from tests import parity

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2405_11143_b200 import orl
    from paper_2405_11143_b200.pipeline import Buffers, LmHeadRows, PathConfig, run_iteration

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def ctx():
    c = orl.Context(0)
    yield c
    c.close()


def _bits(t):
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def _val(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32)


def _bound(h_bits, W_bits, inv_temp):
    """Per-row derived bound on |logp|, |lse|, |H| error (module docstring)."""
    d = h_bits.shape[1]
    s = np.abs(_val(h_bits)) @ np.abs(_val(W_bits)).T  # [R, V] sum_k |h W|
    return np.minimum(2.0 * inv_temp * d * 2.0 ** -24 * s.max(1) + 1e-5, parity.LOGP_ABS)


def _scatter_bound(bound_rows, B, T, lengths, cu):
    bs, ts, rs = oracle.lmhead_row_index(B, T, lengths, cu)
    out = np.zeros((B, T))
    out[bs, ts] = bound_rows[rs]
    return out


def _check(name, g, o, mask, bound):
    g = g.astype(np.float64)
    parity.check_masked_zero(name, g, mask)
    err = np.abs(g[mask] - o[mask])
    lim = bound[mask]
    worst = float(np.max(err / lim)) if err.size else 0.0
    assert np.all(err <= lim), f"{name}: worst err/bound = {worst:.3f}, max err {err.max():.3e}"
    return float(err.max()) if err.size else 0.0


def _run_logprobs(ctx, b, role="old", inv_temp=1.0):
    B, T = b["tokens"].shape
    tok, L = b["tokens"].to(DEV), b["lengths"].to(DEV)
    cu = b["cu_seqlens"].to(DEV) if b["cu_seqlens"] is not None else None
    outs = {k: torch.full((B, T), 7.0, device=DEV) for k in ("logp", "entropy", "lse", "gathered")}
    orl.orl_begin_iteration(ctx)
    orl.orl_lmhead_logprobs(ctx, tok, L, b[f"hidden_{role}"].to(DEV), b["weight"].to(DEV), outs["logp"],
                            inv_temp=inv_temp, entropy=outs["entropy"], lse=outs["lse"],
                            gathered=outs["gathered"], cu_seqlens=cu)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in outs.items()}


@pytest.mark.parametrize("packed", [False, True])
@pytest.mark.parametrize("inv_temp", [1.0, 1.0 / 0.7])
def test_lmhead_logprobs_parity_small(ctx, packed, inv_temp):
    """3 sequences, d = 192 (3 k-blocks), V = 1000 (last vocab tile 232 wide)."""
    B, T, d, V = 3, 40, 192, 1000
    b = synth.make_lmhead_batch(11, B, T, d, V, lengths=[40, 17, 1], packed=packed)
    g = _run_logprobs(ctx, b, inv_temp=inv_temp)
    hb, Wb = _bits(b["hidden_old"]), _bits(b["weight"])
    cu = None if b["cu_seqlens"] is None else b["cu_seqlens"].numpy()
    o = oracle.lmhead_logprobs(hb, Wb, b["tokens"].numpy(), b["lengths"].numpy(), inv_temp, cu)
    mask = parity.valid_mask(b["lengths"].numpy(), T)
    bound = _scatter_bound(_bound(hb, Wb, inv_temp), B, T, b["lengths"].numpy(), cu)
    for k in ("logp", "entropy", "lse"):
        _check(k, g[k], o[k], mask, bound)
    _check("gathered z_y", g["gathered"], o["z_y"], mask, bound / (2 * inv_temp))


def test_lmhead_many_tiles_and_splits(ctx, monkeypatch):
    """R = 800 rows (7 M-tiles, ragged), d = 320 (5 k-blocks), V = 5000 (20 vocab tiles):
    3 tiles per split -> 7 splits merged in order; also the default plan."""
    B, T, d, V = 4, 200, 320, 5000
    b = synth.make_lmhead_batch(12, B, T, d, V, lengths="mixed")
    hb, Wb = _bits(b["hidden_old"]), _bits(b["weight"])
    o = oracle.lmhead_logprobs(hb, Wb, b["tokens"].numpy(), b["lengths"].numpy(), 1.0)
    mask = parity.valid_mask(b["lengths"].numpy(), T)
    bound = _scatter_bound(_bound(hb, Wb, 1.0), B, T, b["lengths"].numpy(), None)
    res = []
    for tps in ("3", None):
        if tps:
            monkeypatch.setenv("ORL_K6_TPS", tps)
        else:
            monkeypatch.delenv("ORL_K6_TPS", raising=False)
        g = _run_logprobs(ctx, b)
        for k in ("logp", "entropy", "lse"):
            _check(k, g[k], o[k], mask, bound)
        res.append(g)
    # the split plan changes only the merge order of partials: results agree closely
    assert np.max(np.abs(res[0]["logp"] - res[1]["logp"])) < 1e-5


def test_lmhead_microbatch_offset_packed(ctx):
    """A micro-batch [2, 5) of a 6-sequence batch with packed hidden rows."""
    B, T, d, V = 6, 64, 128, 768
    b = synth.make_lmhead_batch(13, B, T, d, V, lengths="mixed", packed=True)
    cu = b["cu_seqlens"]
    s, e = 2, 5
    hid = b["hidden_old"][int(cu[s]):int(cu[e])]
    tok, L, cud = b["tokens"].to(DEV), b["lengths"].to(DEV), cu.to(DEV)
    logp = torch.full((B, T), 7.0, device=DEV)
    H = torch.full((B, T), 7.0, device=DEV)
    orl.orl_begin_iteration(ctx)
    orl.orl_lmhead_logprobs(ctx, tok, L, hid.to(DEV), b["weight"].to(DEV), logp, B=e - s, seq_offset=s,
                            entropy=H, cu_seqlens=cud)
    torch.cuda.synchronize()
    g, gH = logp.cpu().numpy(), H.cpu().numpy()
    hb, Wb = _bits(b["hidden_old"]), _bits(b["weight"])
    o = oracle.lmhead_logprobs(hb, Wb, b["tokens"].numpy(), b["lengths"].numpy(), 1.0, cu.numpy())
    mask = parity.valid_mask(b["lengths"].numpy(), T)
    mine = np.zeros_like(mask)
    mine[s:e] = mask[s:e]
    bound = _scatter_bound(_bound(hb, Wb, 1.0), B, T, b["lengths"].numpy(), cu.numpy())
    _check("logp", np.where(mine, g, 0.0), np.where(mine, o["logp"], 0.0), mine, bound)
    _check("entropy", np.where(mine, gH, 0.0), np.where(mine, o["entropy"], 0.0), mine, bound)
    assert np.all(g[s:e][~mask[s:e]] == 0.0)          # masked positions of the call: exact zeros
    assert np.all(g[:s] == 7.0) and np.all(g[e:] == 7.0)  # other micro-batches untouched


@pytest.mark.parametrize("kind", ["gae", "grpo"])
def test_lmhead_full_iteration_vs_oracle(ctx, kind):
    """run_iteration with LM-head sources for old/ref/new (S1..S10): the S1 outputs
    vs the LM-head oracle, then every downstream stage vs the oracle fed the GPU's
    own log-probs (stage isolation, as tests/test_gpu_parity.py)."""
    from tests.test_gpu_parity import _check_downstream
    B, T, d, V = 8, 48, 256, 1536
    G = 4 if kind == "grpo" else 1
    b = synth.make_lmhead_batch(14, B, T, d, V, lengths="mixed",
                                rewards="group_bernoulli" if kind == "grpo" else "normal", group_size=G)
    c = dict(synth.CONFIGS["tiny"], adv_kind=kind, group_size=G)
    if kind == "grpo":
        c.update(kl_mode="loss", beta_loss=0.01, kl_est_loss="k2", whiten=False, c1=0.0, eps_v=0.0)
    cfg = PathConfig.from_synth(c)
    batch = {k: (v.to(DEV) if isinstance(v, torch.Tensor) else v) for k, v in b.items()}
    bufs = Buffers(B, T, DEV, G, grads=True)
    src = lambda role, s, e: LmHeadRows(batch[f"hidden_{role}"][s * T:e * T], batch["weight"])  # noqa: E731
    status, st = run_iteration(ctx, batch, cfg, bufs, src, mb=3)
    torch.cuda.synchronize()
    assert status == "ORL_OK", status
    L = b["lengths"].numpy()
    mask = parity.valid_mask(L, T)
    hb = {r: _bits(b[f"hidden_{r}"]) for r in ("old", "ref", "new")}
    Wb = _bits(b["weight"])
    ora = {r: oracle.lmhead_logprobs(hb[r], Wb, b["tokens"].numpy(), L, cfg.inv_temp) for r in hb}
    for r, buf in (("old", bufs.logp_old), ("ref", bufs.logp_ref), ("new", bufs.logp_new)):
        bound = _scatter_bound(_bound(hb[r], Wb, cfg.inv_temp), B, T, L, None)
        _check(f"logp_{r}", buf.cpu().numpy(), ora[r]["logp"], mask, bound)
    bound = _scatter_bound(_bound(hb["new"], Wb, cfg.inv_temp), B, T, L, None)
    _check("entropy_new", bufs.entropy.cpu().numpy(), ora["new"]["entropy"], mask, bound)
    npb = {k: b[k].numpy() for k in ("tokens", "lengths", "seq_reward", "values_old", "values_new")}
    npb["logp_old"] = bufs.logp_old.cpu().numpy().astype(np.float64)
    npb["logp_ref"] = bufs.logp_ref.cpu().numpy().astype(np.float64)
    npb["logp_new"] = bufs.logp_new.cpu().numpy().astype(np.float64)
    npb["entropy_new"] = bufs.entropy.cpu().numpy().astype(np.float64)
    out, glob = oracle.pipeline([npb], c)
    _check_downstream(bufs, out[0], glob, st, mask, f"lmhead-{kind}")


def test_lmhead_full_size_sampled_rows(ctx):
    """BASELINE llama8b micro-batch shape: 8 x 1024 rows, d = 4096, V = 128256 (the
    launch configuration bench.py times); 24 sampled rows vs the oracle."""
    B, T, d, V = 8, 1024, 4096, 128256
    b = synth.make_lmhead_batch(15, B, T, d, V, lengths="full", device=DEV)
    g = _run_logprobs(ctx, b)
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(B * T, 24, replace=False))
    rows[:2] = [0, B * T - 1]
    hb = _bits(b["hidden_old"][torch.as_tensor(rows, device=DEV)])
    Wb = _bits(b["weight"])
    y = b["tokens"].reshape(-1).cpu().numpy()[rows]
    o = oracle.lmhead_rows(hb, Wb, y, 1.0)
    bound = _bound(hb, Wb, 1.0)
    for k, ok in (("logp", "logp"), ("entropy", "entropy"), ("lse", "lse")):
        gv = g[k].reshape(-1)[rows].astype(np.float64)
        err = np.abs(gv - o[ok])
        assert np.all(err <= bound), (k, float(err.max()), float(bound.min()))
    assert np.all(np.isfinite(g["logp"]))


def test_lmhead_qwen_shape_ragged_sampled_rows(ctx):
    """Qwen2.5-7B-shaped head (longcot config): d = 3584 (56 k-blocks), V = 152064
    (594 vocab tiles, 149 splits with a 2-tile tail split), two T = 8192 responses
    with a ragged second length (16,384 hidden rows, 64 CTA-pair row blocks); 16
    sampled valid rows vs the oracle, masked rows exact zeros."""
    B, T, d, V = 2, 8192, 3584, 152064
    b = synth.make_lmhead_batch(19, B, T, d, V, lengths=[8192, 5000], device=DEV)
    g = _run_logprobs(ctx, b)
    L = b["lengths"].cpu().numpy()
    mask = parity.valid_mask(L, T)
    assert np.all(g["logp"][~mask] == 0.0) and np.all(g["entropy"][~mask] == 0.0)
    rng = np.random.default_rng(1)
    valid = np.flatnonzero(mask.reshape(-1))
    rows = np.sort(rng.choice(valid, 16, replace=False))
    rows[0], rows[-1] = valid[0], valid[-1]
    hb = _bits(b["hidden_old"][torch.as_tensor(rows, device=DEV)])
    Wb = _bits(b["weight"])
    y = b["tokens"].reshape(-1).cpu().numpy()[rows]
    o = oracle.lmhead_rows(hb, Wb, y, 1.0)
    bound = _bound(hb, Wb, 1.0)
    for k in ("logp", "entropy", "lse"):
        err = np.abs(g[k].reshape(-1)[rows].astype(np.float64) - o[k])
        assert np.all(err <= bound), (k, float(err.max()), float(bound.min()))


def test_lmhead_token_range_and_mask_errors(ctx):
    B, T, d, V = 2, 16, 64, 300
    b = synth.make_lmhead_batch(16, B, T, d, V, lengths=[16, 9])
    b["tokens"][0, 3] = V
    b["tokens"][1, 2] = -5
    g = _run_logprobs(ctx, b)
    assert np.isnan(g["logp"][0, 3]) and np.isnan(g["logp"][1, 2])
    ok = parity.valid_mask(b["lengths"].numpy(), T)
    ok[0, 3] = ok[1, 2] = False
    assert np.all(np.isfinite(g["logp"][ok]))
    status, stats = orl.orl_finalize(ctx, orl.PPOConfig())
    assert stats["n_token_range"] == 2
    # hidden too short for the lengths: NaN outputs, no out-of-bounds read, its own status
    # (ORL_E_SHAPE, counted apart from invalid lengths / masks)
    b2 = synth.make_lmhead_batch(16, B, T, d, V, lengths=[16, 9])
    b2["hidden_old"] = b2["hidden_old"][:20]
    g2 = _run_logprobs(ctx, b2)
    assert np.all(np.isnan(g2["logp"][1, 4:9])) and np.all(np.isfinite(g2["logp"][1, :4]))
    status, stats = orl.orl_finalize(ctx, orl.PPOConfig())
    assert status == "ORL_E_SHAPE", status
    assert "5 valid token(s) map to LM-head rows" in orl.orl_last_error(ctx)


def test_lmhead_host_argument_errors(ctx):
    B, T, d, V = 2, 8, 64, 256
    b = synth.make_lmhead_batch(17, B, T, d, V, lengths="full")
    tok, L = b["tokens"].to(DEV), b["lengths"].to(DEV)
    h, W = b["hidden_old"].to(DEV), b["weight"].to(DEV)
    logp = torch.zeros(B, T, device=DEV)
    with pytest.raises(orl.OrlError) as e:  # hidden pitch 60 elements = 120 B: not 16-byte aligned
        hp = torch.zeros(B * T, 60, dtype=torch.bfloat16, device=DEV)
        Wp = torch.zeros(V, 60, dtype=torch.bfloat16, device=DEV)
        orl.orl_lmhead_logprobs(ctx, tok, L, hp, Wp, logp)
    assert e.value.status == 3
    with pytest.raises(ValueError):
        orl.orl_lmhead_logprobs(ctx, tok, L, h, W[:, :32], logp)
    with pytest.raises(TypeError):
        orl.orl_lmhead_logprobs(ctx, tok, L, h.float(), W, logp)


def test_lmhead_run_to_run_bit_identical(ctx):
    B, T, d, V = 4, 100, 256, 3000
    b = synth.make_lmhead_batch(18, B, T, d, V, lengths="mixed")
    g1 = _run_logprobs(ctx, b)
    g2 = _run_logprobs(ctx, b)
    for k in g1:
        assert np.array_equal(g1[k], g2[k], equal_nan=True), k


@pytest.mark.parametrize("i", range(16))
def test_lmhead_random_shapes(ctx, i):
    """Seeded random LM-head shapes around the tiling edges: R from 1 row to a few CTA-pair
    row blocks (ragged), d a multiple of 8 (16-byte rows) but often not of 64 (partial
    k-block), V from 2 to a few vocab tiles and splits (ragged last tile), packed or padded,
    inv_temp != 1; logp / entropy / lse vs the oracle within the derived bound."""
    rng = np.random.default_rng(500 + i)
    B = int(rng.integers(1, 4))
    T = int(rng.choice([1, 7, 64, 130]))
    d = int(rng.choice([8, 40, 64, 72, 136, 200, 264]))
    V = int(rng.choice([2, 17, 255, 256, 257, 700, 1500, 2600]))
    packed = bool(rng.integers(0, 2))
    inv_temp = float(rng.choice([1.0, 1 / 0.7]))
    L = rng.integers(0, T + 1, size=B)
    L[0] = max(int(L[0]), 1)
    b = synth.make_lmhead_batch(600 + i, B, T, d, V, lengths=L.tolist(), packed=packed)
    g = _run_logprobs(ctx, b, inv_temp=inv_temp)
    hb, Wb = _bits(b["hidden_old"]), _bits(b["weight"])
    cu = None if b["cu_seqlens"] is None else b["cu_seqlens"].numpy()
    o = oracle.lmhead_logprobs(hb, Wb, b["tokens"].numpy(), b["lengths"].numpy(), inv_temp, cu)
    mask = parity.valid_mask(b["lengths"].numpy(), T)
    bound = _scatter_bound(_bound(hb, Wb, inv_temp), B, T, b["lengths"].numpy(), cu)
    for k in ("logp", "entropy", "lse"):
        _check(k, g[k], o[k], mask, bound)
