"""Diagnose the peer-memory collectives with real ranks sharing one GPU: each rank logs
every stage (flushed) to gpurun_out/peer_diag_r<rank>.log.
    timeout 120 python tools/peer_diag.py [world] [spin_limit]"""
import os
import socket
import sys
import time
import traceback

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, spin):
    log = open(os.path.join(ROOT, "gpurun_out", f"peer_diag_r{rank}.log"), "w")
    t0 = time.time()

    def say(*a):
        print(f"[{time.time() - t0:7.2f}s r{rank}]", *a, file=log, flush=True)
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), ORL_PEER_SPIN_LIMIT=str(spin))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        say("gloo up")
        torch.cuda.set_device(0)
        from paper_2405_11143_b200 import orl, synth
        from paper_2405_11143_b200.pipeline import Buffers, PathConfig, run_iteration
        ctx = orl.Context(0, world, rank, None)
        say("ctx")
        h = orl.orl_peer_handle(ctx)
        say("handle", h[:8].hex())
        hs = orl.exchange_peer_handles(h, world)
        say("exchanged")
        orl.orl_peer_open(ctx, hs)
        say("opened, collective =", ctx.collective)
        c = dict(synth.CONFIGS["tiny"])
        B, T, V = 4, 16, 32
        batch = synth.make_batch(0, B, T, V, "f32", "stress", "tiny", c["rewards"])
        s, e = synth.split_bounds(B, world, 1)[rank]
        g = {k: (v[s:e].cuda() if isinstance(v, torch.Tensor) and v.dim() > 0 else v) for k, v in batch.items()}
        cfg = PathConfig.from_synth(c)
        bufs = Buffers(e - s, T, torch.device("cuda", 0))
        dist.barrier()
        say("barrier before iteration")
        orl.orl_begin_iteration(ctx)
        for r in ("old",):
            orl.orl_logprobs(ctx, g["tokens"], g["lengths"], g[f"logits_{r}"], bufs.logp_old)
        orl.orl_logprobs(ctx, g["tokens"], g["lengths"], g["logits_ref"], bufs.logp_ref, partner_logp=bufs.logp_old,
                         seq_reward=g["seq_reward"], kl=bufs.kl, shaped_reward=bufs.shaped, beta_reward=0.1)
        orl.orl_advantages(ctx, g["lengths"], bufs.adv, shaped_reward=bufs.shaped, values=g["values_old"],
                           seq_reward=g["seq_reward"], ret=bufs.ret)
        torch.cuda.synchronize()
        say("advantages done")
        orl.orl_whiten_stats(ctx, True)
        say("whiten launched")
        torch.cuda.synchronize()
        say("whiten synced")
        orl.orl_ppo_loss(ctx, g["tokens"], g["lengths"], g["logits_new"], cfg.ppo, bufs.logp_old, bufs.adv,
                         bufs.logp_new, logp_ref=bufs.logp_ref, entropy=bufs.entropy)
        torch.cuda.synchronize()
        say("loss done")
        try:
            st = orl.orl_finalize(ctx, cfg.ppo)
            say("finalize", st[0], {k: st[1][k] for k in ("n_tokens", "policy_loss", "adv_mean")})
        except orl.OrlError as ex:
            say("finalize error", ex)
        dist.barrier()
        ctx.close()
        say("done")
    except Exception:
        say("EXC", traceback.format_exc())


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    spin = int(sys.argv[2]) if len(sys.argv) > 2 else 2_000_000
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(worker, args=(world, port, spin), nprocs=world, start_method="spawn", join=True)
