"""fp64 CPU oracle for the OpenRLHF PPO/RLVR logits -> training-signal path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product (``paper_2405_11143_b200``) never imports it, and this
package imports nothing from the product.

The arithmetic lives in ``orl_oracle.c`` (plain fp64 loops, each function
citing PAPER.md / SPEC.md); this module only marshals numpy arrays through
ctypes and composes the stages in the paper's order (App. C,
lines 189-201: rollout log-probs -> reference log-probs and KL-shaped reward
-> GAE -> normalisation -> PPO loss).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "orl_oracle.c")
_LIB = os.path.join(_HERE, "liborl_oracle.so")
_lock = threading.Lock()
_lib = None

KL = {"k1": 1, "k2": 2, "k3": 3}


def build() -> str:
    """Compile liborl_oracle.so with gcc (plain C, -O2, no fast-math)."""
    cmd = ["gcc", "-O2", "-std=c11", "-fno-fast-math", "-Wall", "-shared", "-fPIC",
           "-o", _LIB, _SRC, "-lm"]
    subprocess.run(cmd, check=True)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if (not os.path.exists(_LIB)) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, f64, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_int
        lib.oracle_row_logsoftmax.argtypes = [P, i64, i64, P, P, P]
        lib.oracle_row_logsoftmax.restype = i32
        lib.oracle_logprobs.argtypes = [P, i32, i64, i64, i64, i64, i64, P, P, f64,
                                        P, P, P, P, P, P]
        lib.oracle_logprobs.restype = None
        lib.oracle_kl.argtypes = [f64, i32]
        lib.oracle_kl.restype = f64
        lib.oracle_kl_grad.argtypes = [f64, i32]
        lib.oracle_kl_grad.restype = f64
        lib.oracle_shape_rewards.argtypes = [i64, i64, P, P, P, i32, f64, P, P, P]
        lib.oracle_shape_rewards.restype = None
        lib.oracle_gae.argtypes = [i64, i64, P, P, P, f64, f64, P, P]
        lib.oracle_gae.restype = None
        lib.oracle_discounted_returns.argtypes = [i64, i64, P, P, f64, P]
        lib.oracle_discounted_returns.restype = None
        lib.oracle_group_advantages.argtypes = [i64, i64, P, P, P]
        lib.oracle_group_advantages.restype = i32
        lib.oracle_group_mean_subtract.argtypes = [i64, i64, P, P]
        lib.oracle_group_mean_subtract.restype = i32
        lib.oracle_broadcast_seq.argtypes = [i64, i64, P, P, P]
        lib.oracle_broadcast_seq.restype = None
        lib.oracle_whiten_moments.argtypes = [P, i64, P, P]
        lib.oracle_whiten_moments.restype = i32
        lib.oracle_whiten_value.argtypes = [f64, f64, f64]
        lib.oracle_whiten_value.restype = f64
        lib.oracle_ppo_loss.argtypes = [i64, i64, P, P, P, P, P, P, P, P, P,
                                        f64, f64, f64, f64, f64, i32, i32, f64, f64, i32, f64,
                                        P, P, P, P, P, P]
        lib.oracle_ppo_loss.restype = None
        lib.oracle_logits_grad_row.argtypes = [P, i64, i64, f64, f64, f64, P]
        lib.oracle_logits_grad_row.restype = None
        lib.oracle_kl_controller_step.argtypes = [P, f64, f64, f64, f64]
        lib.oracle_kl_controller_step.restype = i32
        lib.oracle_stats.argtypes = [P, f64, f64, f64, i32, i32, f64, P]
        lib.oracle_lmhead_rows.argtypes = [P, i64, P, i64, i64, i64, i64, P, f64, P, P, P, P]
        lib.oracle_lmhead_rows.restype = i64
        lib.oracle_stats.restype = i32
        lib.oracle_lengths_from_mask.argtypes = [i64, i64, P, P]
        lib.oracle_lengths_from_mask.restype = i64
        lib.oracle_keep_compact.argtypes = [i64, P, P]
        lib.oracle_keep_compact.restype = i64
        _lib = lib
        return lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


# --------------------------------------------------------------------------- S1
def row_logsoftmax(x, y):
    """(lse, logp, entropy) of one row x (fp64, already scaled by inv_temp)."""
    lib = _load()
    x = _f64(x)
    out = np.zeros(3)
    o = out.ctypes.data
    lib.oracle_row_logsoftmax(_p(x), x.size, int(y), o, o + 8, o + 16)
    return float(out[0]), float(out[1]), float(out[2])


def logprobs(logits, tokens, lengths, inv_temp=1.0, bf16=None):
    """S1 over a [B,T,V] batch (or any strided view with unit V stride).

    ``logits`` is either float32 or uint16 (bf16 bit patterns; pass
    ``bf16=True``).  Returns dict of [B,T] fp64 arrays: logp, entropy, lse,
    gathered, and the counters n_token_range / n_nonfinite.
    """
    lib = _load()
    if bf16 is None:
        bf16 = logits.dtype == np.uint16
    dt = 0 if bf16 else (2 if logits.dtype == np.float64 else 1)
    assert dt != 1 or logits.dtype == np.float32, logits.dtype
    item = logits.itemsize
    assert logits.strides[2] == item, "V must be unit stride"
    B, T, V = logits.shape
    sb, st = logits.strides[0] // item, logits.strides[1] // item
    tokens, lengths = _i32(tokens), _i32(lengths)
    outs = {k: np.zeros((B, T)) for k in ("logp", "entropy", "lse", "gathered")}
    cnt = np.zeros(2, dtype=np.int64)
    base = logits.__array_interface__["data"][0]
    lib.oracle_logprobs(ctypes.c_void_p(base), dt, B, T, V, sb, st,
                        _p(tokens), _p(lengths), float(inv_temp),
                        _p(outs["logp"]), _p(outs["entropy"]), _p(outs["lse"]),
                        _p(outs["gathered"]), cnt.ctypes.data, cnt.ctypes.data + 8)
    outs["n_token_range"] = int(cnt[0])
    outs["n_nonfinite"] = int(cnt[1])
    return outs


# --------------------------------------------------------------------------- S2/S3
def kl(d, kind):
    return _load().oracle_kl(float(d), KL.get(kind, kind))


def kl_grad(d, kind):
    return _load().oracle_kl_grad(float(d), KL.get(kind, kind))


def shape_rewards(lengths, logp_a, logp_b, kind, beta, seq_reward):
    lib = _load()
    logp_a, logp_b = _f64(logp_a), _f64(logp_b)
    B, T = logp_a.shape
    lengths, R = _i32(lengths), _f64(seq_reward)
    kl_out, r_out = np.zeros((B, T)), np.zeros((B, T))
    lib.oracle_shape_rewards(B, T, _p(lengths), _p(logp_a), _p(logp_b),
                             KL.get(kind, kind), float(beta), _p(R), _p(kl_out), _p(r_out))
    return kl_out, r_out


# --------------------------------------------------------------------------- S4/S5
def gae(lengths, rewards, values, gamma, lam):
    lib = _load()
    r, V = _f64(rewards), _f64(values)
    B, T = r.shape
    lengths = _i32(lengths)
    adv, ret = np.zeros((B, T)), np.zeros((B, T))
    lib.oracle_gae(B, T, _p(lengths), _p(r), _p(V), float(gamma), float(lam), _p(adv), _p(ret))
    return adv, ret


def discounted_returns(lengths, rewards, gamma):
    lib = _load()
    r = _f64(rewards)
    B, T = r.shape
    lengths = _i32(lengths)
    out = np.zeros((B, T))
    lib.oracle_discounted_returns(B, T, _p(lengths), _p(r), float(gamma), _p(out))
    return out


def group_advantages(seq_reward, group_size):
    lib = _load()
    R = _f64(seq_reward)
    B = R.size
    adv = np.zeros(B)
    keep = np.zeros(max(B // max(group_size, 1), 1), dtype=np.uint8)
    rc = lib.oracle_group_advantages(B, int(group_size), _p(R), _p(adv), _p(keep))
    if rc:
        raise ValueError("batch is not a whole number of groups")
    return adv, keep[: B // group_size]


def group_mean_subtract(seq_reward, group_size):
    lib = _load()
    R = _f64(seq_reward)
    out = np.zeros(R.size)
    if lib.oracle_group_mean_subtract(R.size, int(group_size), _p(R), _p(out)):
        raise ValueError("batch is not a whole number of groups")
    return out


def broadcast_seq(lengths, per_seq, T):
    lib = _load()
    per_seq = _f64(per_seq)
    B = per_seq.size
    lengths = _i32(lengths)
    out = np.zeros((B, T))
    lib.oracle_broadcast_seq(B, T, _p(lengths), _p(per_seq), _p(out))
    return out


# --------------------------------------------------------------------------- S6
def whiten_moments(values):
    lib = _load()
    a = _f64(np.ravel(values))
    out = np.zeros(2)
    warn = lib.oracle_whiten_moments(_p(a), a.size, out.ctypes.data, out.ctypes.data + 8)
    return float(out[0]), float(out[1]), bool(warn)


def whiten_value(a, mean, std):
    return _load().oracle_whiten_value(float(a), float(mean), float(std))


def whiten(adv, lengths, mean, std):
    """A' = (A - mean)/(std + 1e-8) on valid tokens, element by element."""
    lib = _load()
    out = np.zeros_like(_f64(adv))
    B, T = out.shape
    for b in range(B):
        for t in range(int(lengths[b])):
            out[b, t] = lib.oracle_whiten_value(float(adv[b, t]), mean, std)
    return out


# --------------------------------------------------------------------------- S7-S10
def ppo_loss(lengths, logp_new, logp_old, adv_w, *, logp_ref=None, ret=None, v_new=None,
             v_old=None, entropy=None, eps_low=0.2, eps_high=0.2, eps_v=0.0, c1=0.0,
             beta_loss=0.0, kl_est="k1", kl_in_loss=False, ratio_guard=30.0, n_global=None,
             seq_mean=False, n_seq=None):
    lib = _load()
    logp_new, logp_old, adv_w = _f64(logp_new), _f64(logp_old), _f64(adv_w)
    B, T = logp_new.shape
    lengths = _i32(lengths)
    if n_global is None:
        n_global = float(np.minimum(lengths, T).clip(min=0).sum())
    if n_seq is None:
        n_seq = float(np.count_nonzero(lengths > 0))
    sums = np.zeros(15)
    obj, vl, dlogp, dv = (np.zeros((B, T)) for _ in range(4))
    clipped = np.zeros((B, T), dtype=np.uint8)
    logp_ref, ret, v_new, v_old, entropy = map(_f64, (logp_ref, ret, v_new, v_old, entropy))
    lib.oracle_ppo_loss(B, T, _p(lengths), _p(logp_new), _p(logp_old), _p(logp_ref), _p(adv_w),
                        _p(ret), _p(v_new), _p(v_old), _p(entropy), float(eps_low),
                        float(eps_high), float(eps_v), float(c1), float(beta_loss),
                        KL.get(kl_est, kl_est), int(bool(kl_in_loss)), float(ratio_guard),
                        float(n_global), int(bool(seq_mean)), float(n_seq),
                        _p(sums), _p(obj), _p(clipped), _p(vl), _p(dlogp), _p(dv))
    # `flags`: bit 0 clipped (Z16), 1 value-clipped (Z13), 2 ratio guard (Z22), 3 non-finite
    return dict(sums=sums, obj=obj, clipped=clipped & 1, flags=clipped, vl=vl, dlogp=dlogp, dv=dv)


STAT_NAMES = ("n_tokens", "policy_loss", "value_loss", "entropy", "kl", "approx_kl_old",
              "clip_frac", "value_clip_frac", "ratio_mean", "total_loss")


def stats(sums, c1=0.0, c2=0.0, beta_loss=0.0, kl_in_loss=False, seq_mean=False, n_seq=0.0):
    lib = _load()
    sums = _f64(np.concatenate([np.ravel(sums), np.zeros(max(0, 15 - np.size(sums)))]))
    out = np.zeros(10)
    rc = lib.oracle_stats(_p(sums), float(c1), float(c2), float(beta_loss),
                          int(bool(kl_in_loss)), int(bool(seq_mean)), float(n_seq), _p(out))
    d = dict(zip(STAT_NAMES, map(float, out)))
    d["empty"] = bool(rc)
    d["n_guard"] = int(sums[9])
    d["n_nonfinite"] = int(sums[10])
    return d


# --------------------------------------------------------------------------- NEXT-1
def logits_grad_row(x, y, inv_temp, w, a):
    """dL/dx of one valid row (raw logits x, fp64): NEXT-1."""
    lib = _load()
    x = _f64(x)
    g = np.zeros(x.size)
    lib.oracle_logits_grad_row(_p(x), x.size, int(y), float(inv_temp), float(w), float(a), _p(g))
    return g


def lmhead_rows(h_bits, W_bits, y, inv_temp=1.0):
    """NEXT-4: S1 of the LM-head logits z = h W^T (fp64) per row.

    h_bits [R, d] and W_bits [V, d] are bf16 bit patterns (uint16); y [R]
    (int32; y < 0 = row not computed).  Returns dict logp, entropy, lse, z_y
    ([R] fp64) and n_nonfinite."""
    lib = _load()
    h = np.ascontiguousarray(h_bits, dtype=np.uint16)
    W = np.ascontiguousarray(W_bits, dtype=np.uint16)
    y = _i32(y)
    R, d = h.shape
    V = W.shape[0]
    assert W.shape[1] == d and y.shape == (R,)
    out = {k: np.zeros(R) for k in ("logp", "entropy", "lse", "z_y")}
    bad = lib.oracle_lmhead_rows(_p(h), d, _p(W), d, R, d, V, _p(y), float(inv_temp), _p(out["logp"]),
                                 _p(out["entropy"]), _p(out["lse"]), _p(out["z_y"]))
    out["n_nonfinite"] = int(bad)
    return out


def lmhead_row_index(B, T, lengths, cu_seqlens=None, seq_offset=0):
    """Hidden-row index of every valid (b,t) of a call (orl.h orl_lmhead):
    packed cu_seqlens[so+b] - cu_seqlens[so] + t, else b*T + t.  Returns
    (b, t, r) arrays in (b,t) order."""
    bs, ts, rs = [], [], []
    for b in range(B):
        for t in range(int(lengths[seq_offset + b])):
            r = (int(cu_seqlens[seq_offset + b]) - int(cu_seqlens[seq_offset]) + t) if cu_seqlens is not None \
                else b * T + t
            bs.append(b), ts.append(t), rs.append(r)
    return np.array(bs, dtype=np.int64), np.array(ts, dtype=np.int64), np.array(rs, dtype=np.int64)


def lmhead_logprobs(h_bits, W_bits, tokens, lengths, inv_temp=1.0, cu_seqlens=None):
    """NEXT-4 over a batch: [B,T] logp, entropy, lse (zeros at masked positions)
    from the hidden rows h_bits [R, d] (row index as in lmhead_row_index)."""
    B, T = tokens.shape
    bs, ts, rs = lmhead_row_index(B, T, lengths, cu_seqlens)
    R = h_bits.shape[0]
    y = np.full(R, -1, dtype=np.int32)
    y[rs] = tokens[bs, ts]
    o = lmhead_rows(h_bits, W_bits, y, inv_temp)
    res = {}
    for k in ("logp", "entropy", "lse", "z_y"):
        a = np.zeros((B, T))
        a[bs, ts] = o[k][rs]
        res[k] = a
    res["n_nonfinite"] = o["n_nonfinite"]
    return res


def logits_grad(logits, tokens, lengths, dlogp, inv_temp, c2, n_global, seq_mean=False, n_seq=0.0):
    """[B,T,V] dL/dlogits (zeros on masked rows); `logits` as for logprobs().
    The entropy weight per row is c2/N (token mean) or c2/(n_seq L_b) (NEXT-2 seq-mean)."""
    B, T, V = logits.shape
    out = np.zeros((B, T, V))
    for b in range(B):
        if int(lengths[b]) <= 0:
            continue
        a = c2 / (n_seq * float(lengths[b])) if seq_mean else c2 / n_global
        for t in range(int(lengths[b])):
            row = logits[b, t]
            x = (row.astype(np.uint32) << 16).view(np.float32).astype(np.float64) \
                if row.dtype == np.uint16 else row.astype(np.float64)
            out[b, t] = logits_grad_row(x, tokens[b, t], inv_temp, dlogp[b, t], a)
    return out


def kl_controller_step(beta, target, horizon, observed, max_kl):
    """NEXT-3: (new beta, early_stop)."""
    b = np.array([float(beta)])
    stop = _load().oracle_kl_controller_step(_p(b), float(target), float(horizon), float(observed), float(max_kl))
    return float(b[0]), bool(stop)


# --------------------------------------------------------------------------- NEXT-2 helpers
def lengths_from_mask(mask):
    """Z10: (lengths [B] int32, number of non-prefix rows) of a [B,T] attention mask."""
    m = np.ascontiguousarray(np.asarray(mask) != 0, dtype=np.uint8)
    B, T = m.shape
    L = np.zeros(B, dtype=np.int32)
    bad = _load().oracle_lengths_from_mask(B, T, _p(m), _p(L))
    return L, int(bad)


def keep_compact(keep):
    """NEXT-2 (DAPO): indices of the kept groups in increasing order."""
    k = np.ascontiguousarray(np.asarray(keep) != 0, dtype=np.uint8)
    idx = np.zeros(max(k.size, 1), dtype=np.int32)
    n = _load().oracle_keep_compact(k.size, _p(k), _p(idx))
    return idx[:n].copy()


from .pipeline import pipeline  # noqa: E402  (composition of the stages above)
