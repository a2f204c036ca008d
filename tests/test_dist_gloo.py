"""CPU coverage of the N > 1 path (world_size 2 over gloo).

The GPU path shards the batch by contiguous, group-aligned sequence blocks and
exchanges exactly two things: C1, every rank's whitening
partial before the actor pass, and C2, every rank's loss/stat partial after
it, both merged in rank order.  Here each gloo rank runs the oracle on its
own shard and exchanges the same quantities with torch.distributed; the
result must equal the single-process oracle over the whole batch.  The
unique-id broadcast and the max-over-ranks timing of bench.py are exercised
with the same process group.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_11143_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, q, split="tokens"):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from oracle import pipeline as _p  # noqa: F401

        full = synth.tiny_numpy(7, B=8, T=16, V=32, rewards="group_bernoulli" if kind == "grpo" else "normal",
                                group_size=2)
        G = 2 if kind in ("grpo", "rpp_baseline") else 1
        cfg = dict(synth.CONFIGS["tiny"], adv_kind=kind, group_size=G)
        if kind == "grpo":
            cfg.update(kl_mode="loss", beta_loss=0.01, kl_est_loss="k2", whiten=False, c1=0.0, eps_v=0.0)
        # bench.py's shards: contiguous, group-aligned, balanced by valid tokens
        bounds = synth.split_bounds_tokens(full["lengths"], world, G) if split == "tokens" \
            else synth.split_bounds(8, world, G)
        s, e = bounds[rank]
        shard = {k: v[s:e] for k, v in full.items()}
        # unique-id broadcast as bench.py does it
        uid = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        assert uid[0] == bytes(range(128))
        # rank-local experience (S1..S5): the oracle on this shard alone
        out, _ = oracle.pipeline([shard], cfg)
        o = out[0]
        L = shard["lengths"]
        local_valid = np.concatenate([o["adv"][b, :L[b]] for b in range(len(L))] or [np.zeros(0)])
        # C1: gather every rank's advantages' moments input (here: the values) in rank order
        gathered = [None] * world
        dist.all_gather_object(gathered, local_valid)
        allv = np.concatenate(gathered)
        mean, std, warn = oracle.whiten_moments(allv)
        do_w = cfg["whiten"] and kind != "grpo" and not warn
        adv_w = oracle.whiten(o["adv"], L, mean, std) if do_w else o["adv"]
        res = oracle.ppo_loss(L, o["logp_new"], o["logp_old"], adv_w, logp_ref=o["logp_ref"],
                              ret=o["ret"] if kind == "gae" else None,
                              v_new=shard["values_new"] if kind == "gae" else None,
                              v_old=shard["values_old"] if kind == "gae" else None, entropy=o["entropy"],
                              eps_low=cfg["eps_low"], eps_high=cfg["eps_high"], eps_v=cfg["eps_v"],
                              c1=cfg["c1"] if kind == "gae" else 0.0, beta_loss=cfg.get("beta_loss", 0.0),
                              kl_est=cfg.get("kl_est_loss", "k2"), kl_in_loss=cfg.get("kl_mode") == "loss",
                              n_global=float(allv.size))
        # C2: gather the loss partials and sum them in rank order
        sums = [None] * world
        dist.all_gather_object(sums, res["sums"])
        tot = np.zeros(15)
        for r in range(world):
            tot = tot + sums[r]
        st = oracle.stats(tot, c1=cfg["c1"], c2=cfg["c2"], beta_loss=cfg.get("beta_loss", 0.0),
                          kl_in_loss=cfg.get("kl_mode") == "loss")
        # max-over-ranks timing reduction (bench.py)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == world
        if rank == 0:
            _, glob = oracle.pipeline([full], cfg)
            q.put(("ok", st, glob["stats"]))
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover
        import traceback
        q.put(("err", traceback.format_exc(), None))


@pytest.mark.parametrize("kind,split", [("gae", "tokens"), ("rpp", "tokens"), ("grpo", "tokens"),
                                        ("gae", "sequences")])
def test_two_rank_protocol_matches_single_process(kind, split):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q, split)) for r in range(2)]
    for p in procs:
        p.start()
    status, st, ref = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", st
    for k, v in ref.items():
        if isinstance(v, float):
            assert abs(st[k] - v) <= 1e-12 * max(1.0, abs(v)), (k, st[k], v)


def test_split_bounds_cover_and_align():
    for B, n, G in [(1024, 8, 1), (2048, 8, 8), (10, 3, 1), (16, 4, 4), (8, 8, 2)]:
        b = synth.split_bounds(B, n, G)
        assert b[0][0] == 0 and b[-1][1] == B
        assert all(b[i][1] == b[i + 1][0] for i in range(n - 1))
        assert all(s % G == 0 and e % G == 0 for s, e in b)
        sizes = [e - s for s, e in b]
        assert max(sizes) - min(sizes) <= G
    with pytest.raises(ValueError):
        synth.split_bounds(10, 2, 4)


def _peer_handle_worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2405_11143_b200 import orl
        mine = bytes([rank]) * orl.PEER_HANDLE_BYTES         # stands in for a cudaIpcMemHandle_t
        got = orl.exchange_peer_handles(mine, world)
        bad = None
        try:
            orl.exchange_peer_handles(b"short", world)         # every rank sends a malformed one
        except ValueError as ex:
            bad = str(ex)
        q.put((rank, got, bad))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc(), None))


def test_peer_handle_exchange_rank_ordered():
    """Host side of orl_peer_open's setup (orl.Context.enable_peer): the exchange-buffer
    handles are all-gathered over torch.distributed in rank order, malformed ones rejected."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_handle_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    from paper_2405_11143_b200 import orl
    for rank, got, bad in res:
        assert isinstance(got, list), got
        assert got == [bytes([r]) * orl.PEER_HANDLE_BYTES for r in range(world)]
        assert bad and "malformed" in bad
