"""GPU tests of C1 / C2 as single peer-memory kernels (orl_peer_handle / orl_peer_open,
include/orl.h), with REAL separate ranks: n processes (torch.multiprocessing, gloo for
the handle exchange) share the one GPU of this box, each with its own context and
exchange buffer mapped into the others through CUDA IPC.  The kernels' protocol is the
one an 8-GPU NVLink box runs (stores into every rank's slot, release/acquire epoch
flags, rank-ordered merge); only the link differs.

Checks: every rank's statistics are bit-identical, within
1e-12 of one rank over the whole batch, per-token outputs of each shard bit-identical
to the one-rank run's slice, across two iterations (both exchange-buffer parities);
a rank that never arrives makes the waits time out and orl_finalize report ORL_E_NCCL.
"""
from __future__ import annotations

import os
import socket
import traceback

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2405_11143_b200 import synth

pytestmark = pytest.mark.gpu

B, T, V = 8, 64, 2048


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _config(kind):
    c = dict(synth.CONFIGS["llama8b"], adv_kind=kind, group_size=2 if kind == "grpo" else 1)
    if kind == "grpo":
        c.update(kl_mode="loss", beta_loss=0.01, whiten=False, eps_v=0.0, c1=0.0)
    return c


def _batch(kind, dev):
    from tests.test_gpu_parity import _gpu_batch
    return _gpu_batch(41, B, T, V, "mixed", "group_bernoulli" if kind == "grpo" else "normal", 2)


def _iterate(ctx, g, cfg, mb=3):
    from paper_2405_11143_b200.pipeline import Buffers, run_iteration
    Bs = g["tokens"].shape[0]
    bufs = Buffers(Bs, T, torch.device("cuda", 0), cfg.group_size, grads=True)
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    status, st = run_iteration(ctx, g, cfg, bufs, src, mb=mb)
    torch.cuda.synchronize()
    return status, st, bufs


def _worker(rank, world, port, kind, mode, q):
    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        # bounded waits: ~1-2 s per wait before a timeout is reported, never a hang
        os.environ["ORL_PEER_SPIN_LIMIT"] = "20000" if mode == "timeout" else "4000000"
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2405_11143_b200 import orl
        from paper_2405_11143_b200.pipeline import PathConfig
        c = _config(kind)
        cfg = PathConfig.from_synth(c)
        ctx = orl.Context(0, world, rank, None)
        ctx.enable_peer()
        assert ctx.collective == "peer"
        g = _batch(kind, torch.device("cuda", 0))
        s, e = synth.split_bounds(B, world, c["group_size"])[rank]
        gs = {k: v[s:e] for k, v in g.items()}
        out = []
        if mode == "graph":  # the whole iteration, peer kernels included, as one CUDA graph per rank
            from paper_2405_11143_b200.pipeline import Buffers, GraphStep
            status, st, _ = _iterate(ctx, gs, cfg)
            gb = Buffers(e - s, T, torch.device("cuda", 0), cfg.group_size, grads=True)
            step = GraphStep(ctx, gs, cfg, gb, lambda role, a, z: gs[f"logits_{role}"][a:z], mb=3)
            for _ in range(3):  # epochs advance on the device across replays
                step.replay()
                torch.cuda.synchronize()
                out.append((status, st, step.result()))
            dist.barrier()
        elif mode == "timeout":
            if rank == 0:  # rank 1 never runs an iteration: both waits of rank 0 time out
                try:
                    status, st, _ = _iterate(ctx, gs, cfg)
                except orl.OrlError as err:
                    status, st = orl.STATUS[err.status], None
                out.append((status, st))
            dist.barrier()
        else:
            for _ in range(2):  # epochs 1 and 2: both parities of the exchange buffer
                status, st, bufs = _iterate(ctx, gs, cfg)
                out.append((status, st, bufs.adv.cpu().numpy(), bufs.logp_new.cpu().numpy(), bufs.dlogp.cpu().numpy()))
            dist.barrier()
        ctx.close()
        q.put((rank, "ok", out))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        q.put((rank, "error", traceback.format_exc()))


def _spawn(world, kind, mode):
    ctxmp = mp.get_context("spawn")
    q = ctxmp.Queue()
    port = _free_port()
    procs = [ctxmp.Process(target=_worker, args=(r, world, port, kind, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    res, deadline = {}, time.monotonic() + 300
    while len(res) < world and time.monotonic() < deadline:
        try:
            rank, tag, payload = q.get(timeout=2)
            res[rank] = (tag, payload)
        except queue.Empty:
            dead = [r for r, p in enumerate(procs) if p.exitcode not in (None, 0) and r not in res]
            if dead:  # a rank crashed without reporting (e.g. a signal)
                break
    for p in procs:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    for r, p in enumerate(procs):
        if r not in res:
            res[r] = ("error", f"rank {r} did not report (exitcode {p.exitcode})")
    errs = [p for t, p in res.values() if t == "error"]
    if errs and any("cudaIpcOpenMemHandle" in e or "exclusive" in e.lower() for e in errs):
        pytest.skip("CUDA IPC between processes on this GPU unavailable: " + errs[0].splitlines()[-1])
    assert not errs, errs[0]
    return res


@pytest.mark.parametrize("kind,world", [("gae", 2), ("rpp", 4), ("grpo", 2), ("gae", 8)])
def test_peer_collectives_real_ranks_match_single_rank(kind, world):
    from paper_2405_11143_b200 import orl
    from paper_2405_11143_b200.pipeline import PathConfig
    res = _spawn(world, kind, "run")
    c = _config(kind)
    cfg = PathConfig.from_synth(c)
    one = orl.Context(0)
    g = _batch(kind, torch.device("cuda", 0))
    status1, st1, b1 = _iterate(one, g, cfg)
    one.close()
    assert status1 == "ORL_OK"
    bounds = synth.split_bounds(B, world, c["group_size"])
    for it in range(2):
        first = res[0][1][it][1]
        for r in range(world):
            status, st, adv, logp_new, dlogp = res[r][1][it]
            assert status == "ORL_OK", status
            assert st == first                               # every rank bit-identical
            for k, v in st1.items():
                if isinstance(v, float):
                    assert abs(st[k] - v) <= 1e-12 * max(1.0, abs(v)), (k, st[k], v)
            s, e = bounds[r]
            assert np.array_equal(adv, b1.adv[s:e].cpu().numpy())
            assert np.array_equal(logp_new, b1.logp_new[s:e].cpu().numpy())
            np.testing.assert_allclose(dlogp, b1.dlogp[s:e].cpu().numpy(), rtol=1e-6, atol=1e-12)


def test_peer_collective_missing_rank_times_out():
    res = _spawn(2, "gae", "timeout")
    status, st = res[0][1][0]
    assert status == "ORL_E_NCCL", status


def test_peer_collectives_inside_cuda_graph_replays():
    res = _spawn(2, "gae", "graph")
    first = res[0][1][0][1]
    for r in range(2):
        for status, st, (gstatus, gst) in res[r][1]:
            assert status == "ORL_OK" and gstatus == "ORL_OK"
            assert st == first and gst == first      # eager == replay, bit for bit, on every rank
