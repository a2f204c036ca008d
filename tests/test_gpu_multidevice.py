"""GPU tests of the N > 1 path with one process per DEVICE (skipped unless the box has at
least 2 GPUs; this build's boxes have one, so these run on an 8-GPU node only).

Each rank owns cuda:rank, an NCCL process group (torch.distributed), and an orl context
with its own NCCL communicator created from a unique id broadcast by rank 0 (the same
plumbing bench.py uses under torchrun).  Per rank the batch shard is the token-balanced,
group-aligned contiguous block (synth.split_bounds_tokens).  Checks:
  * C1/C2 over NCCL all-gathers: every rank's statistics bit-identical, within 1e-12 of
    one context over the whole batch, per-token outputs bit-identical to its slices;
  * C1/C2 as the single peer-memory kernels over NVLink (cross-device CUDA IPC mappings,
    system-scope release/acquire): bit-identical to the NCCL path, two iterations (both
    exchange-buffer parities).
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

# ORL_TEST_WORLD=1 runs the same code with one rank (a 1-rank NCCL communicator; the peer
# transport then stays NCCL) to exercise the test itself on a one-GPU box
FORCED_WORLD = int(os.environ.get("ORL_TEST_WORLD", "0"))
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2 and not FORCED_WORLD,
                                 reason="needs >= 2 GPUs (one process per device)")]

B, T, V = 32, 96, 4096


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _config(kind):
    c = dict(synth.CONFIGS["llama8b"], adv_kind=kind, group_size=4 if kind == "grpo" else 1)
    if kind == "grpo":
        c.update(kl_mode="loss", beta_loss=0.01, whiten=False, eps_v=0.0, c1=0.0)
    return c


def _host_batch(kind):
    c = _config(kind)
    return synth.make_batch(77, B, T, V, "bf16", "stress", "mixed",
                            "group_bernoulli" if kind == "grpo" else "normal", c["group_size"])


def _iterate(ctx, g, cfg, dev, mb=3):
    from paper_2405_11143_b200.pipeline import Buffers, run_iteration
    bufs = Buffers(g["tokens"].shape[0], T, dev, cfg.group_size, grads=True)
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    status, st = run_iteration(ctx, g, cfg, bufs, src, mb=mb)
    torch.cuda.synchronize(dev)
    return status, st, {k: getattr(bufs, k).cpu().numpy() for k in ("adv", "logp_new", "dlogp")}


def _worker(rank, world, port, kind, q):
    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dev = torch.device("cuda", rank)
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        from paper_2405_11143_b200 import orl
        from paper_2405_11143_b200.pipeline import PathConfig
        c = _config(kind)
        cfg = PathConfig.from_synth(c)
        uid = [orl.orl_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = orl.Context(rank, world, rank, uid[0])
        assert ctx.collective == "nccl"
        hb = _host_batch(kind)
        bounds = synth.split_bounds_tokens(hb["lengths"].numpy(), world, c["group_size"])
        s, e = bounds[rank]
        g = {k: v[s:e].to(dev) for k, v in hb.items()}
        out = {"bounds": bounds, "nccl": [], "peer": []}
        for _ in range(2):
            out["nccl"].append(_iterate(ctx, g, cfg, dev))
        ctx.enable_peer()
        assert ctx.collective == ("peer" if world > 1 else "nccl")
        for _ in range(2):
            out["peer"].append(_iterate(ctx, g, cfg, dev))
        dist.barrier()
        ctx.close()
        q.put((rank, "ok", out))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        q.put((rank, "error", traceback.format_exc()))


def _spawn(world, kind):
    import queue
    import time
    ctxmp = mp.get_context("spawn")
    q = ctxmp.Queue()
    port = _free_port()
    procs = [ctxmp.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res, deadline = {}, time.monotonic() + 600
    while len(res) < world and time.monotonic() < deadline:
        try:
            rank, tag, payload = q.get(timeout=2)
            res[rank] = (tag, payload)
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for r, p in enumerate(procs) if r not in res):
                break
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    for r, p in enumerate(procs):
        res.setdefault(r, ("error", f"rank {r} did not report (exitcode {p.exitcode})"))
    errs = [p for t, p in res.values() if t == "error"]
    assert not errs, errs[0]
    return {r: p for r, (t, p) in res.items()}


@pytest.mark.parametrize("kind", ["gae", "grpo", "rpp"])
def test_one_process_per_device_nccl_and_peer(kind):
    from paper_2405_11143_b200 import orl
    from paper_2405_11143_b200.pipeline import PathConfig
    world = FORCED_WORLD or min(torch.cuda.device_count(), 8)
    res = _spawn(world, kind)
    c = _config(kind)
    cfg = PathConfig.from_synth(c)
    dev = torch.device("cuda", 0)
    one = orl.Context(0)
    hb = _host_batch(kind)
    status1, st1, o1 = _iterate(one, {k: v.to(dev) for k, v in hb.items()}, cfg, dev)
    one.close()
    assert status1 == "ORL_OK"
    first = res[0]["nccl"][0][1]
    for r in range(world):
        s, e = res[r]["bounds"][r]
        for path in ("nccl", "peer"):
            for status, st, o in res[r][path]:
                assert status == "ORL_OK", (r, path, status)
                assert st == first, (r, path)                       # every rank, both transports, bit-identical
                for k, v in st1.items():
                    if isinstance(v, float):
                        assert abs(st[k] - v) <= 1e-12 * max(1.0, abs(v)), (k, st[k], v)
                assert np.array_equal(o["adv"], o1["adv"][s:e])
                assert np.array_equal(o["logp_new"], o1["logp_new"][s:e])
                np.testing.assert_allclose(o["dlogp"], o1["dlogp"][s:e], rtol=1e-6, atol=1e-12)
