"""Stress the peer-memory C1/C2 kernels with real ranks sharing this GPU: `world` processes
run `iters` iterations on fresh random shards (ragged lengths, every advantage kind); every
rank's statistics must be bit-identical, and equal (1e-12) to rank 0's single-context run
over the whole batch.   python tools/peer_stress.py [world] [iters]"""
import os
import socket
import sys
import traceback

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, iters, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), ORL_PEER_SPIN_LIMIT="4000000")
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2405_11143_b200 import orl, synth
        from paper_2405_11143_b200.pipeline import Buffers, PathConfig, run_iteration
        dev = torch.device("cuda", 0)
        ctx = orl.Context(0, world, rank, None)
        ctx.enable_peer()
        one = orl.Context(0) if rank == 0 else None
        bad = 0
        for it in range(iters):
            kind = ["gae", "rpp", "grpo", "rpp_baseline"][it % 4]
            G = 2 if kind in ("grpo", "rpp_baseline") else 1
            B, T, V = 2 * world * G, 48, 2048
            c = dict(synth.CONFIGS["llama8b"], V=V, adv_kind=kind, group_size=G)
            if kind == "grpo":
                c.update(kl_mode="loss", beta_loss=0.01, whiten=False, eps_v=0.0, c1=0.0)
            cfg = PathConfig.from_synth(c)
            L = synth.lengths_for(B, T, it, "mixed")
            tok = synth.tokens_for(B, T, V, it).to(dev)
            lg = tuple(torch.empty(B, T, V, dtype=torch.bfloat16, device=dev) for _ in range(3))
            synth.fill_logits_(lg, tok, it, 0, "stress")
            R = synth.rewards_for(B, it, "group_bernoulli" if G > 1 else "normal", G)
            vo, vn = synth.values_for(B, T, it)
            g = dict(tokens=tok, lengths=L.to(dev), seq_reward=R.to(dev), values_old=vo.to(dev),
                     values_new=vn.to(dev))
            s, e = synth.split_bounds(B, world, G)[rank]
            gs = {k: v[s:e] for k, v in g.items()}
            src = lambda role, a, z: lg[("old", "ref", "new").index(role)][s + a:s + z]  # noqa: E731
            status, st = run_iteration(ctx, gs, cfg, Buffers(e - s, T, dev, G), src, mb=1 + it % 3)
            allst = [None] * world
            dist.all_gather_object(allst, st)
            if any(x != allst[0] for x in allst) or status != "ORL_OK":
                bad += 1
            if rank == 0:
                src1 = lambda role, a, z: lg[("old", "ref", "new").index(role)][a:z]  # noqa: E731
                _, st1 = run_iteration(one, g, cfg, Buffers(B, T, dev, G), src1, mb=2)
                for k, v in st1.items():
                    if isinstance(v, float) and abs(st[k] - v) > 1e-12 * max(1.0, abs(v)):
                        bad += 1
                        break
        q.put((rank, bad))
        dist.barrier()
    except Exception:
        q.put((rank, traceback.format_exc()))


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctxmp = mp.get_context("spawn")
    q = ctxmp.Queue()
    ps = [ctxmp.Process(target=worker, args=(r, world, port, iters, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=900) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    print("world", world, "iters", iters, "results (rank, bad iterations):", sorted(res, key=lambda x: x[0]))
