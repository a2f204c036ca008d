"""Thin ctypes binding of liborl.so (include/orl.h).

Argument marshalling only: every step of the path runs in the CUDA kernels of
liborl.so.  Functions carry the C names (orl_logprobs, orl_advantages, ...)
and take torch CUDA tensors (PyTorch is used for device memory and streams).
Importing this module fails loudly if liborl.so is missing: there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ORL_LIB_PATH") or os.path.join(_PKG, "liborl.so")   # override: tuning builds
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2405_11143_b200.build` "
                      "(or __graft_entry__.build()); there is no CPU fallback")
_lib = ctypes.CDLL(LIB_PATH)

UNIQUE_ID_BYTES = 128
STATS_N = 16
PEER_HANDLE_BYTES = 64
FINAL_N = 20
PARTIALS_N = 24
LOSS_AGG = {"token_mean": 0, "seq_mean_token_mean": 1}
MAX_SEQ_PER_CALL = 8192

STATUS = {0: "ORL_OK", 1: "ORL_E_INVALID_ARG", 2: "ORL_E_SHAPE", 3: "ORL_E_ALIGN", 4: "ORL_E_DTYPE",
          5: "ORL_E_TOKEN_RANGE", 6: "ORL_E_MASK", 7: "ORL_E_NONFINITE", 8: "ORL_E_NUMERIC_GUARD",
          9: "ORL_E_EMPTY_BATCH", 10: "ORL_E_GROUP_SPLIT", 11: "ORL_E_CUDA", 12: "ORL_E_NCCL",
          13: "ORL_E_STATE"}
ST = {v: k for k, v in STATUS.items()}
DTYPE = {torch.bfloat16: 0, torch.float32: 1}
KL = {"k1": 1, "k2": 2, "k3": 3}
ADV = {"gae": 0, "grpo": 1, "rpp": 2, "rpp_baseline": 3}


class Logits(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("V", ctypes.c_int64), ("stride_b", ctypes.c_int64), ("stride_t", ctypes.c_int64)]


class Rows(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int64), ("T", ctypes.c_int64), ("seq_offset", ctypes.c_int64),
                ("tokens", ctypes.c_void_p), ("lengths", ctypes.c_void_p), ("cu_seqlens", ctypes.c_void_p)]


class LmHead(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_void_p), ("weight", ctypes.c_void_p), ("R", ctypes.c_int64),
                ("d", ctypes.c_int64), ("V", ctypes.c_int64), ("ld_hidden", ctypes.c_int64),
                ("ld_weight", ctypes.c_int64)]


class PpoCfg(ctypes.Structure):
    _fields_ = [("eps_low", ctypes.c_double), ("eps_high", ctypes.c_double),
                ("eps_value", ctypes.c_double), ("c1", ctypes.c_double), ("c2", ctypes.c_double),
                ("beta_loss", ctypes.c_double), ("kl_loss_est", ctypes.c_int32),
                ("kl_in_loss", ctypes.c_int32), ("ratio_guard", ctypes.c_double),
                ("loss_agg", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in (
        "n_tokens", "policy_loss", "value_loss", "entropy", "kl", "approx_kl_old", "clip_frac",
        "value_clip_frac", "ratio_mean", "total_loss", "adv_mean", "adv_std")] + [
        ("n_guard", ctypes.c_int64), ("n_nonfinite", ctypes.c_int64), ("n_token_range", ctypes.c_int64),
        ("whiten_warn", ctypes.c_int32), ("pad_", ctypes.c_int32)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "pad_"}


_P, _I64, _I32, _F32, _F64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_double
_lib.orl_version.restype = ctypes.c_int
_lib.orl_get_unique_id.argtypes = [ctypes.c_char_p]
_lib.orl_create.argtypes = [_I32, _I32, _I32, ctypes.c_char_p, ctypes.POINTER(_P)]
_lib.orl_destroy.argtypes = [_P]
_lib.orl_last_error.argtypes = [_P]
_lib.orl_last_error.restype = ctypes.c_char_p
_lib.orl_launch_count.argtypes = [_P]
_lib.orl_launch_count.restype = ctypes.c_uint64
_lib.orl_begin_iteration.argtypes = [_P, _P]
_lib.orl_logprobs.argtypes = [_P, ctypes.POINTER(Rows), ctypes.POINTER(Logits), _F32, _P, _P, _P, _P,
                              _P, _I32, _F64, _P, _P, _P, _P]
_lib.orl_advantages.argtypes = [_P, _I64, _I64, _P, _I32, _F64, _F64, _I32, _P, _P, _P, _P, _P, _P, _P, _P]
_lib.orl_whiten_stats.argtypes = [_P, _I32, _P]
_lib.orl_ppo_loss.argtypes = [_P, ctypes.POINTER(Rows), ctypes.POINTER(Logits), _F32,
                              ctypes.POINTER(PpoCfg), _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]
_lib.orl_ppo_loss_and_grad.argtypes = [_P, ctypes.POINTER(Rows), ctypes.POINTER(Logits), _F32,
                                       ctypes.POINTER(PpoCfg), _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                       _P, _P, _I64, _I64, _I32, _P]
_lib.orl_logits_grad.argtypes = [_P, ctypes.POINTER(Rows), ctypes.POINTER(Logits), _F32, ctypes.POINTER(PpoCfg),
                                 _P, _P, _P, _P, _I64, _I64, _I32, _P]
_lib.orl_lmhead_logprobs.argtypes = [_P, ctypes.POINTER(Rows), ctypes.POINTER(LmHead), _F32, _P, _P, _P, _P,
                                     _P, _I32, _F64, _P, _P, _P, _P]
_lib.orl_lmhead_ppo_loss.argtypes = [_P, ctypes.POINTER(Rows), ctypes.POINTER(LmHead), _F32,
                                     ctypes.POINTER(PpoCfg), _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]
_lib.orl_set_pdl_chain.argtypes = [_P, _I32]
_lib.orl_get_pdl_chain.argtypes = [_P]
_lib.orl_get_pdl_chain.restype = ctypes.c_int
_lib.orl_finalize.argtypes = [_P, ctypes.POINTER(PpoCfg), ctypes.POINTER(Stats), _P, _P]
_lib.orl_export_partials.argtypes = [_P, _I32, _P, _P]
_lib.orl_import_partials.argtypes = [_P, _I32, _P, _I32, _P]
_lib.orl_reserve.argtypes = [_P, _I64, _I64, _I64]
_lib.orl_lengths_from_mask.argtypes = [_P, _I64, _I64, _P, _P, _P]
_lib.orl_keep_compact.argtypes = [_P, _I64, _P, _P, _P, _P]
_lib.orl_finalize_async.argtypes = [_P, ctypes.POINTER(PpoCfg), _P, _P]
_lib.orl_stats_decode.argtypes = [_P, _F64, ctypes.POINTER(Stats)]
_lib.orl_peer_handle.argtypes = [_P, ctypes.c_char_p]
_lib.orl_peer_open.argtypes = [_P, ctypes.c_char_p]
_lib.orl_set_collective.argtypes = [_P, _I32]
_lib.orl_get_collective.argtypes = [_P]
_lib.orl_get_collective.restype = ctypes.c_int
_lib.orl_kl_controller_step.argtypes = [ctypes.POINTER(_F64), _F64, _F64, _F64, _F64, ctypes.POINTER(ctypes.c_int)]
for _f in ("orl_set_pdl_chain", "orl_kl_controller_step", "orl_get_unique_id", "orl_create", "orl_destroy", "orl_begin_iteration", "orl_logprobs",
           "orl_advantages", "orl_whiten_stats", "orl_ppo_loss", "orl_finalize",
           "orl_export_partials", "orl_import_partials", "orl_logits_grad", "orl_ppo_loss_and_grad"):
    getattr(_lib, _f).restype = ctypes.c_int


class OrlError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


@dataclass
class PPOConfig:
    eps_low: float = 0.2
    eps_high: float = 0.2
    eps_value: float = 0.2
    c1: float = 0.5
    c2: float = 0.0
    beta_loss: float = 0.0
    kl_loss_est: str = "k2"
    kl_in_loss: bool = False
    ratio_guard: float = 30.0
    loss_agg: str = "token_mean"

    def c(self) -> PpoCfg:
        return PpoCfg(self.eps_low, self.eps_high, self.eps_value, self.c1, self.c2, self.beta_loss,
                      KL[self.kl_loss_est], int(bool(self.kl_in_loss)), self.ratio_guard,
                      LOSS_AGG[self.loss_agg], 0)


def version() -> int:
    return _lib.orl_version()


# C names for the context-level calls (the Context class wraps the same functions)
def orl_version() -> int:
    return _lib.orl_version()


def orl_create(device: int = 0, world: int = 1, rank: int = 0, unique_id: bytes | None = None) -> "Context":
    return Context(device, world, rank, unique_id)


def orl_destroy(ctx: "Context") -> None:
    ctx.close()


def orl_last_error(ctx: "Context | None" = None) -> str:
    return _lib.orl_last_error(ctx.h if ctx is not None else None).decode()


def orl_launch_count(ctx: "Context") -> int:
    return ctx.launch_count


def orl_set_collective(ctx: "Context", mode: str) -> None:
    ctx.set_collective(mode)


def orl_get_collective(ctx: "Context") -> str:
    return ctx.collective


def orl_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(UNIQUE_ID_BYTES)
    st = _lib.orl_get_unique_id(buf)
    if st:
        raise OrlError(st, _lib.orl_last_error(None).decode())
    return buf.raw


class Context:
    """Owns an orl_ctx (NCCL communicator, fp64 accumulators, error counters)."""

    def __init__(self, device: int = 0, world: int = 1, rank: int = 0, unique_id: bytes | None = None):
        h = ctypes.c_void_p()
        st = _lib.orl_create(int(device), int(world), int(rank), unique_id, ctypes.byref(h))
        if st:
            raise OrlError(st, _lib.orl_last_error(None).decode())
        self.h, self.device, self.world, self.rank = h, device, world, rank

    def close(self):
        if getattr(self, "h", None):
            _lib.orl_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, st: int, allow=()):
        if st and st not in allow:
            raise OrlError(st, _lib.orl_last_error(self.h).decode())
        return st

    @property
    def launch_count(self) -> int:
        return int(_lib.orl_launch_count(self.h))

    @property
    def collective(self) -> str:
        return {0: "nccl", 1: "peer"}.get(int(_lib.orl_get_collective(self.h)), "?")

    def enable_peer(self, group=None):
        """C1/C2 as peer-memory kernels: all-gather the exchange-buffer handles over
        torch.distributed (`group`), then map them (collective over the ranks)."""
        handles = exchange_peer_handles(orl_peer_handle(self), self.world, group)
        orl_peer_open(self, handles)

    def set_collective(self, mode: str):
        self.check(_lib.orl_set_collective(self.h, {"nccl": 0, "peer": 1}[mode]))

    @property
    def pdl_chain(self) -> bool:
        return int(_lib.orl_get_pdl_chain(self.h)) == 1

    @pdl_chain.setter
    def pdl_chain(self, enable: bool):
        """orl_set_pdl_chain: see orl.h for the precondition of enable=True."""
        self.check(_lib.orl_set_pdl_chain(self.h, int(bool(enable))))


def orl_set_pdl_chain(ctx: "Context", enable: bool) -> None:
    ctx.pdl_chain = enable


def orl_get_pdl_chain(ctx: "Context") -> bool:
    return ctx.pdl_chain


def orl_peer_handle(ctx: "Context") -> bytes:
    buf = ctypes.create_string_buffer(PEER_HANDLE_BYTES)
    ctx.check(_lib.orl_peer_handle(ctx.h, buf))
    return buf.raw


def orl_peer_open(ctx: "Context", handles) -> None:
    blob = b"".join(handles)
    if len(blob) != PEER_HANDLE_BYTES * ctx.world:
        raise ValueError(f"need {ctx.world} handles of {PEER_HANDLE_BYTES} bytes")
    ctx.check(_lib.orl_peer_open(ctx.h, blob))


def exchange_peer_handles(mine: bytes, world: int, group=None) -> list:
    """Rank-ordered list of every rank's handle (torch.distributed all_gather_object)."""
    import torch.distributed as dist

    out = [None] * world
    dist.all_gather_object(out, mine, group=group)
    if any(not isinstance(h, bytes) or len(h) != PEER_HANDLE_BYTES for h in out):
        raise ValueError("malformed peer handle")
    return out


# ----------------------------------------------------------------------------- argument checks
# Every pointer handed to liborl is checked here first (dtype, device, contiguity,
# size), so a wrong tensor raises TypeError / ValueError instead of an out-of-bounds
# device access or silently reinterpreted bits (e.g. int64 token ids read as int32).
def _on_ctx(ctx, name, t):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if not t.is_cuda or (t.device.index if t.device.index is not None else torch.cuda.current_device()) != ctx.device:
        raise ValueError(f"{name} must be a CUDA tensor on cuda:{ctx.device} (got {t.device})")


def _arr(ctx, name, t, dtype, numel, optional=True):
    """A contiguous device array of `dtype` with at least `numel` elements."""
    if t is None:
        if optional:
            return None
        raise ValueError(f"{name} is required")
    _on_ctx(ctx, name, t)
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype} (got {t.dtype})")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.numel() < numel:
        raise ValueError(f"{name} has {t.numel()} elements, needs >= {numel}")
    return t


def _tok(ctx, tokens, lengths, B, seq_offset, cu_seqlens=None):
    """tokens int32 [B_total, T], lengths int32 [B_total], the call's sequences inside."""
    _arr(ctx, "tokens", tokens, torch.int32, 0, optional=False)
    if tokens.dim() != 2:
        raise ValueError("tokens must be [B_total, T]")
    Bt, T = tokens.shape
    _arr(ctx, "lengths", lengths, torch.int32, Bt, optional=False)
    if seq_offset < 0 or B < 1 or seq_offset + B > Bt:
        raise ValueError(f"sequences [{seq_offset}, {seq_offset + B}) outside the rank batch of {Bt}")
    _arr(ctx, "cu_seqlens", cu_seqlens, torch.int32, Bt + 1)
    return Bt, T


def _tokarr(ctx, Bt, T, **arrays):
    """Per-token fp32 [B_total, T] arrays (None = not given)."""
    for name, t in arrays.items():
        _arr(ctx, name, t, torch.float32, Bt * T)


# ----------------------------------------------------------------------------- C-named calls
def _rows(tokens, lengths, B, T, seq_offset, cu_seqlens=None):
    return Rows(int(B), int(T), int(seq_offset), tokens.data_ptr(), lengths.data_ptr(),
                None if cu_seqlens is None else cu_seqlens.data_ptr())


def _packed(x, B):
    """A packed [total, V] logits tensor seen as the [B, 1, V]-shaped descriptor the C
    ABI wants (stride_b unused with cu_seqlens; stride_t = row pitch)."""
    if x.dtype not in DTYPE:
        raise TypeError(f"logits dtype {x.dtype} (bf16 or fp32 expected)")
    if x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("packed logits must be a [total, V] view with unit stride along V")
    return Logits(x.data_ptr(), DTYPE[x.dtype], 0, x.shape[-1], 0, x.stride(-2))


def _logits(x):
    if x.dtype not in DTYPE:
        raise TypeError(f"logits dtype {x.dtype} (bf16 or fp32 expected)")
    if x.dim() != 3 or x.stride(2) != 1:
        raise ValueError("logits must be a [B,T,V] view with unit stride along V")
    return Logits(x.data_ptr(), DTYPE[x.dtype], 0, x.shape[2], x.stride(0), x.stride(1))


def orl_reserve(ctx: Context, max_seqs: int, max_lm_rows: int = 0, max_vocab: int = 0):
    """Pre-size the workspaces so later calls within these sizes never allocate."""
    return ctx.check(_lib.orl_reserve(ctx.h, int(max_seqs), int(max_lm_rows), int(max_vocab)))


def orl_lengths_from_mask(ctx: Context, mask, lengths, stream=None):
    """lengths[b] = leading ones of the u8/bool [B, T] right-padded mask (non-prefix rows
    are counted as ORL_E_MASK at orl_finalize)."""
    if mask.dtype not in (torch.uint8, torch.bool) or mask.dim() != 2 or not mask.is_contiguous():
        raise TypeError("mask must be a contiguous [B, T] uint8/bool tensor")
    _on_ctx(ctx, "mask", mask)
    _arr(ctx, "lengths", lengths, torch.int32, mask.shape[0], optional=False)
    if lengths.dtype != torch.int32 or lengths.numel() < mask.shape[0]:
        raise TypeError("lengths must be int32 [B]")
    B, T = mask.shape
    return ctx.check(_lib.orl_lengths_from_mask(ctx.h, B, T, _ptr(mask), _ptr(lengths), _stream(stream)))


def orl_keep_compact(ctx: Context, group_keep, kept_groups, n_kept, stream=None):
    """Indices of the kept groups (DAPO dynamic sampling) in increasing order + their count."""
    if group_keep.dtype != torch.uint8 or kept_groups.dtype != torch.int32 or n_kept.dtype != torch.int32:
        raise TypeError("group_keep uint8, kept_groups / n_kept int32")
    n = group_keep.numel()
    for name, t in (("group_keep", group_keep), ("kept_groups", kept_groups), ("n_kept", n_kept)):
        _on_ctx(ctx, name, t)
    if kept_groups.numel() < n:
        raise ValueError("kept_groups must hold n_groups entries")
    return ctx.check(_lib.orl_keep_compact(ctx.h, n, _ptr(group_keep), _ptr(kept_groups), _ptr(n_kept),
                                           _stream(stream)))


def orl_begin_iteration(ctx: Context, stream=None):
    return ctx.check(_lib.orl_begin_iteration(ctx.h, _stream(stream)))


def _lg(ctx, logits, B, cu_seqlens):
    _on_ctx(ctx, "logits", logits)
    return _packed(logits, B) if cu_seqlens is not None else _logits(logits)


def _nseq(logits, cu_seqlens, n_seq):
    if cu_seqlens is None:
        return logits.shape[0]
    if n_seq is None:
        raise ValueError("packed logits (cu_seqlens) need n_seq, the sequences in the call")
    return int(n_seq)


def _flags(ctx, flags, Bt, T):
    return _arr(ctx, "flags", flags, torch.uint8, Bt * T)


def orl_logprobs(ctx: Context, tokens, lengths, logits, logp, *, seq_offset=0, inv_temp=1.0,
                 entropy=None, lse=None, gathered=None, partner_logp=None, kl_est="k1",
                 beta_reward=0.0, seq_reward=None, kl=None, shaped_reward=None, stream=None,
                 cu_seqlens=None, n_seq=None):
    """S1 (+S2/S3 with partner_logp) on the micro-batch logits[0:B] = sequences
    [seq_offset, seq_offset+B) of the rank batch; per-token arrays are [B_total, T].
    Packed varlen (NEXT-2): pass `cu_seqlens` and a [total, V] `logits` whose row 0 is
    token cu_seqlens[seq_offset], plus `n_seq` (the B of the call)."""
    B = _nseq(logits, cu_seqlens, n_seq)
    Bt, T = _tok(ctx, tokens, lengths, B, seq_offset, cu_seqlens)
    _arr(ctx, "logp", logp, torch.float32, Bt * T, optional=False)
    _tokarr(ctx, Bt, T, entropy=entropy, lse=lse, gathered=gathered, partner_logp=partner_logp, kl=kl,
            shaped_reward=shaped_reward)
    _arr(ctx, "seq_reward", seq_reward, torch.float32, Bt)
    rows = _rows(tokens, lengths, B, T, seq_offset, cu_seqlens)
    lg = _lg(ctx, logits, B, cu_seqlens)
    st = _lib.orl_logprobs(ctx.h, ctypes.byref(rows), ctypes.byref(lg), float(inv_temp), _ptr(logp),
                           _ptr(entropy), _ptr(lse), _ptr(gathered), _ptr(partner_logp),
                           KL.get(kl_est, kl_est), float(beta_reward), _ptr(seq_reward), _ptr(kl),
                           _ptr(shaped_reward), _stream(stream))
    return ctx.check(st)


def _lmhead(hidden, weight):
    if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
        raise TypeError("LM head hidden states and weight must be bf16")
    if hidden.dim() != 2 or weight.dim() != 2 or hidden.stride(1) != 1 or weight.stride(1) != 1:
        raise ValueError("hidden [R, d] and weight [V, d] must be 2-D with unit stride along d")
    if hidden.shape[1] != weight.shape[1]:
        raise ValueError(f"hidden size mismatch: {hidden.shape[1]} vs {weight.shape[1]}")
    return LmHead(hidden.data_ptr(), weight.data_ptr(), hidden.shape[0], hidden.shape[1], weight.shape[0],
                  hidden.stride(0), weight.stride(0))


def _head(ctx, hidden, weight):
    _on_ctx(ctx, "hidden", hidden)
    _on_ctx(ctx, "weight", weight)
    return _lmhead(hidden, weight)


def orl_lmhead_logprobs(ctx: Context, tokens, lengths, hidden, weight, logp, *, B=None, seq_offset=0,
                        inv_temp=1.0, entropy=None, lse=None, gathered=None, partner_logp=None, kl_est="k1",
                        beta_reward=0.0, seq_reward=None, kl=None, shaped_reward=None, stream=None,
                        cu_seqlens=None):
    """NEXT-4: orl_logprobs with logits = hidden @ weight.T computed on the tensor cores
    (never materialised).  hidden [R, d] holds the call's rows: packed by `cu_seqlens`
    or b*T + t; `B` = sequences in the call (default: all from seq_offset)."""
    if B is None:
        B = tokens.shape[0] - seq_offset
    Bt, T = _tok(ctx, tokens, lengths, B, seq_offset, cu_seqlens)
    _arr(ctx, "logp", logp, torch.float32, Bt * T, optional=False)
    _tokarr(ctx, Bt, T, entropy=entropy, lse=lse, gathered=gathered, partner_logp=partner_logp, kl=kl,
            shaped_reward=shaped_reward)
    _arr(ctx, "seq_reward", seq_reward, torch.float32, Bt)
    rows, hd = _rows(tokens, lengths, B, T, seq_offset, cu_seqlens), _head(ctx, hidden, weight)
    st = _lib.orl_lmhead_logprobs(ctx.h, ctypes.byref(rows), ctypes.byref(hd), float(inv_temp), _ptr(logp),
                                  _ptr(entropy), _ptr(lse), _ptr(gathered), _ptr(partner_logp),
                                  KL.get(kl_est, kl_est), float(beta_reward), _ptr(seq_reward), _ptr(kl),
                                  _ptr(shaped_reward), _stream(stream))
    return ctx.check(st)


def _loss_arrays(ctx, Bt, T, logp_old, adv, logp_new, logp_ref, ret, v_new, v_old, entropy, lse, dloss_dlogp,
                 dloss_dv, flags, adv_lo=None):
    for name, t in (("logp_old", logp_old), ("adv", adv), ("logp_new", logp_new)):
        _arr(ctx, name, t, torch.float32, Bt * T, optional=False)
    _tokarr(ctx, Bt, T, logp_ref=logp_ref, ret=ret, v_new=v_new, v_old=v_old, entropy=entropy, lse=lse,
            dloss_dlogp=dloss_dlogp, dloss_dv=dloss_dv, adv_lo=adv_lo)
    _flags(ctx, flags, Bt, T)


def orl_lmhead_ppo_loss(ctx: Context, tokens, lengths, hidden, weight, cfg, logp_old, adv, logp_new, *,
                        B=None, seq_offset=0, inv_temp=1.0, logp_ref=None, ret=None, v_new=None, v_old=None,
                        entropy=None, lse=None, dloss_dlogp=None, dloss_dv=None, flags=None, stream=None,
                        cu_seqlens=None, adv_lo=None):
    """NEXT-4: orl_ppo_loss with the actor logits computed from its LM head."""
    if B is None:
        B = tokens.shape[0] - seq_offset
    Bt, T = _tok(ctx, tokens, lengths, B, seq_offset, cu_seqlens)
    _loss_arrays(ctx, Bt, T, logp_old, adv, logp_new, logp_ref, ret, v_new, v_old, entropy, lse, dloss_dlogp,
                 dloss_dv, flags, adv_lo)
    rows, hd, c = _rows(tokens, lengths, B, T, seq_offset, cu_seqlens), _head(ctx, hidden, weight), cfg.c()
    st = _lib.orl_lmhead_ppo_loss(ctx.h, ctypes.byref(rows), ctypes.byref(hd), float(inv_temp), ctypes.byref(c),
                                  _ptr(logp_old), _ptr(logp_ref), _ptr(adv), _ptr(adv_lo), _ptr(ret), _ptr(v_new),
                                  _ptr(v_old), _ptr(logp_new), _ptr(entropy), _ptr(lse), _ptr(dloss_dlogp),
                                  _ptr(dloss_dv), _ptr(flags), _stream(stream))
    return ctx.check(st)


def orl_advantages(ctx: Context, lengths, adv, *, kind="gae", gamma=1.0, lam=0.95, group_size=1,
                   shaped_reward=None, values=None, seq_reward=None, ret=None, group_keep=None,
                   adv_lo=None, stream=None):
    """S4/S4'/S5; `adv_lo` (optional fp32 [B, T]) receives A - (float)A (pass it to the
    actor pass: fp64-exact whitening of nearly constant advantages, Z33)."""
    _arr(ctx, "adv", adv, torch.float32, 0, optional=False)
    if adv.dim() != 2:
        raise ValueError("adv must be [B, T]")
    B, T = adv.shape
    _arr(ctx, "lengths", lengths, torch.int32, B, optional=False)
    _tokarr(ctx, B, T, shaped_reward=shaped_reward, values=values, ret=ret, adv_lo=adv_lo)
    _arr(ctx, "seq_reward", seq_reward, torch.float32, B)
    _arr(ctx, "group_keep", group_keep, torch.uint8, B // max(1, int(group_size)))
    st = _lib.orl_advantages(ctx.h, B, T, _ptr(lengths), ADV.get(kind, kind), float(gamma), float(lam),
                             int(group_size), _ptr(shaped_reward), _ptr(values), _ptr(seq_reward),
                             _ptr(adv), _ptr(adv_lo), _ptr(ret), _ptr(group_keep), _stream(stream))
    return ctx.check(st)


def orl_whiten_stats(ctx: Context, whiten: bool, stream=None):
    return ctx.check(_lib.orl_whiten_stats(ctx.h, int(bool(whiten)), _stream(stream)))


def orl_ppo_loss(ctx: Context, tokens, lengths, logits, cfg: PPOConfig, logp_old, adv, logp_new, *,
                 seq_offset=0, inv_temp=1.0, logp_ref=None, ret=None, v_new=None, v_old=None,
                 entropy=None, lse=None, dloss_dlogp=None, dloss_dv=None, flags=None, stream=None,
                 cu_seqlens=None, n_seq=None, adv_lo=None):
    """S1 + S7..S9 on the actor logits; `flags` (optional uint8 [B_total, T]) receives the
    per-token decisions (bit 0 clipped, 1 value-clipped, 2 ratio guard, 3 non-finite);
    `adv_lo` (optional) is orl_advantages' low part (A = adv + adv_lo)."""
    B = _nseq(logits, cu_seqlens, n_seq)
    Bt, T = _tok(ctx, tokens, lengths, B, seq_offset, cu_seqlens)
    _loss_arrays(ctx, Bt, T, logp_old, adv, logp_new, logp_ref, ret, v_new, v_old, entropy, lse, dloss_dlogp,
                 dloss_dv, flags, adv_lo)
    rows, c = _rows(tokens, lengths, B, T, seq_offset, cu_seqlens), cfg.c()
    lg = _lg(ctx, logits, B, cu_seqlens)
    st = _lib.orl_ppo_loss(ctx.h, ctypes.byref(rows), ctypes.byref(lg), float(inv_temp), ctypes.byref(c),
                           _ptr(logp_old), _ptr(logp_ref), _ptr(adv), _ptr(adv_lo), _ptr(ret), _ptr(v_new),
                           _ptr(v_old), _ptr(logp_new), _ptr(entropy), _ptr(lse), _ptr(dloss_dlogp),
                           _ptr(dloss_dv), _ptr(flags), _stream(stream))
    return ctx.check(st)


def _dlogits(ctx, dlogits, logits):
    _on_ctx(ctx, "dlogits", dlogits)
    if dlogits.dtype != logits.dtype or dlogits.shape[-1] != logits.shape[-1] or dlogits.stride(-1) != 1:
        raise ValueError("dlogits must be a view with the logits dtype, V and unit V stride")
    if dlogits.dim() != logits.dim() or tuple(dlogits.shape[:-1]) != tuple(logits.shape[:-1]):
        raise ValueError(f"dlogits shape {tuple(dlogits.shape)} does not match the logits {tuple(logits.shape)}")


def orl_ppo_loss_and_grad(ctx: Context, tokens, lengths, logits, cfg: PPOConfig, logp_old, adv, logp_new, *,
                          entropy, lse, dloss_dlogp, dlogits, seq_offset=0, inv_temp=1.0, logp_ref=None,
                          ret=None, v_new=None, v_old=None, dloss_dv=None, flags=None, zero_masked=True,
                          stream=None, cu_seqlens=None, n_seq=None, adv_lo=None):
    """S1 + S7..S9 + NEXT-1 in one pass over the actor logits (the row is re-read from L2)."""
    B = _nseq(logits, cu_seqlens, n_seq)
    Bt, T = _tok(ctx, tokens, lengths, B, seq_offset, cu_seqlens)
    for name, t in (("entropy", entropy), ("lse", lse), ("dloss_dlogp", dloss_dlogp)):
        _arr(ctx, name, t, torch.float32, Bt * T, optional=False)
    _loss_arrays(ctx, Bt, T, logp_old, adv, logp_new, logp_ref, ret, v_new, v_old, entropy, lse, dloss_dlogp,
                 dloss_dv, flags, adv_lo)
    _dlogits(ctx, dlogits, logits)
    rows, c = _rows(tokens, lengths, B, T, seq_offset, cu_seqlens), cfg.c()
    lg = _lg(ctx, logits, B, cu_seqlens)
    sb = 0 if cu_seqlens is not None else dlogits.stride(0)
    st = _lib.orl_ppo_loss_and_grad(ctx.h, ctypes.byref(rows), ctypes.byref(lg), float(inv_temp), ctypes.byref(c),
                                    _ptr(logp_old), _ptr(logp_ref), _ptr(adv), _ptr(adv_lo), _ptr(ret), _ptr(v_new),
                                    _ptr(v_old), _ptr(logp_new), _ptr(entropy), _ptr(lse), _ptr(dloss_dlogp),
                                    _ptr(dloss_dv), _ptr(flags), _ptr(dlogits), sb, dlogits.stride(-2),
                                    int(bool(zero_masked)), _stream(stream))
    return ctx.check(st)


def orl_logits_grad(ctx: Context, tokens, lengths, logits, cfg: PPOConfig, lse, entropy, dloss_dlogp, dlogits, *,
                    seq_offset=0, inv_temp=1.0, zero_masked=True, stream=None, cu_seqlens=None, n_seq=None):
    """NEXT-1: dL/dlogits of the micro-batch logits[0:B] into dlogits[0:B] (same dtype/shape view;
    packed [total, V] tensors with cu_seqlens)."""
    B = _nseq(logits, cu_seqlens, n_seq)
    Bt, T = _tok(ctx, tokens, lengths, B, seq_offset, cu_seqlens)
    for name, t in (("lse", lse), ("entropy", entropy), ("dloss_dlogp", dloss_dlogp)):
        _arr(ctx, name, t, torch.float32, Bt * T, optional=False)
    _dlogits(ctx, dlogits, logits)
    rows, c = _rows(tokens, lengths, B, T, seq_offset, cu_seqlens), cfg.c()
    lg = _lg(ctx, logits, B, cu_seqlens)
    sb = 0 if cu_seqlens is not None else dlogits.stride(0)
    st = _lib.orl_logits_grad(ctx.h, ctypes.byref(rows), ctypes.byref(lg), float(inv_temp), ctypes.byref(c),
                              _ptr(lse), _ptr(entropy), _ptr(dloss_dlogp), _ptr(dlogits), sb,
                              dlogits.stride(-2), int(bool(zero_masked)), _stream(stream))
    return ctx.check(st)


# statuses orl_finalize / orl_stats_decode return for data found on the device (outputs are
# still written); ORL_E_SHAPE there = valid tokens mapped to LM-head rows beyond the hidden matrix
DATA_ERRORS = (ST["ORL_E_TOKEN_RANGE"], ST["ORL_E_MASK"], ST["ORL_E_SHAPE"], ST["ORL_E_NONFINITE"],
               ST["ORL_E_NUMERIC_GUARD"], ST["ORL_E_EMPTY_BATCH"])


def orl_finalize(ctx: Context, cfg: PPOConfig, dev_out=None, stream=None, raise_on_data_error=False):
    """Returns (status_name, stats dict).  Data errors are returned, not raised,
    unless raise_on_data_error."""
    out, c = Stats(), cfg.c()
    st = _lib.orl_finalize(ctx.h, ctypes.byref(c), ctypes.byref(out), _ptr(dev_out), _stream(stream))
    ctx.check(st, allow=() if raise_on_data_error else DATA_ERRORS)
    return STATUS[st], out.as_dict()


def orl_finalize_async(ctx: Context, cfg: PPOConfig, dev_out, stream=None):
    """S10 + C2 without a host sync (graph-capturable); dev_out: float64 [FINAL_N] on the device."""
    if dev_out.dtype != torch.float64 or dev_out.numel() < FINAL_N or not dev_out.is_cuda:
        raise ValueError(f"dev_out must be a float64 CUDA tensor of >= {FINAL_N} elements")
    c = cfg.c()
    ctx.check(_lib.orl_finalize_async(ctx.h, ctypes.byref(c), _ptr(dev_out), _stream(stream)))


def orl_stats_decode(final_vec, cfg: PPOConfig):
    """Host: (status_name, stats dict) from a host copy of orl_finalize_async's vector."""
    import numpy as np
    v = np.ascontiguousarray(np.asarray(final_vec, dtype=np.float64)[:FINAL_N])
    out = Stats()
    st = _lib.orl_stats_decode(v.ctypes.data_as(ctypes.c_void_p), float(cfg.ratio_guard), ctypes.byref(out))
    if st and st not in DATA_ERRORS:
        raise OrlError(st, _lib.orl_last_error(None).decode())
    return STATUS[st], out.as_dict()


def orl_export_partials(ctx: Context, which: int, stream=None):
    import numpy as np
    n = 4 if which == 0 else PARTIALS_N
    buf = np.zeros(n, dtype=np.float64)
    ctx.check(_lib.orl_export_partials(ctx.h, int(which), buf.ctypes.data_as(ctypes.c_void_p), _stream(stream)))
    return buf


def orl_import_partials(ctx: Context, which: int, host_all, stream=None):
    import numpy as np
    arr = np.ascontiguousarray(host_all, dtype=np.float64)
    world = arr.shape[0]
    ctx.check(_lib.orl_import_partials(ctx.h, int(which), arr.ctypes.data_as(ctypes.c_void_p), world,
                                       _stream(stream)))


def orl_kl_controller_step(beta: float, target: float, horizon: float, observed_kl: float, max_kl: float):
    """NEXT-3 (host only): returns (new beta, early_stop)."""
    b, stop = ctypes.c_double(beta), ctypes.c_int(0)
    st = _lib.orl_kl_controller_step(ctypes.byref(b), float(target), float(horizon), float(observed_kl),
                                     float(max_kl), ctypes.byref(stop))
    if st:
        raise OrlError(st, _lib.orl_last_error(None).decode())
    return b.value, bool(stop.value)
