#!/usr/bin/env python
"""Benchmark of the logits -> PPO-loss path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama8b] [--impl ours|reference]

One step = one PPO iteration of the whole hot path on every rank (S1 old,
S1+S2+S3 ref, S4 advantages, S6 + collective C1, S1+S7..S9 actor, S10 +
collective C2) over a resident synthetic rollout of the named BASELINE.json
configuration (default configs[1], "llama8b": B=128, T=1024, V=128256 bf16).
N > 1 is launched by torchrun (one process per GPU); per-GPU work is fixed
(weak scaling: each rank holds its own B-sequence shard of a B*N batch).

Prints ONE JSON line on rank 0 (see DESIGN.md section 7 for every field).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "tokens/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except (OSError, ValueError, KeyError, TypeError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _bf16_peak(sustained: bool):
    """Dense bf16 tensor peak in TFLOP/s: MEASURED_PEAKS.json (cuBLAS, burst or the
    seconds-long power-capped loop), else the profiling guide's fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    key = "bf16_tflops_sustained" if sustained else "bf16_tflops"
    try:
        return float(json.load(open(p))[key]), f"measured (MEASURED_PEAKS.json {key}, cuBLAS)"
    except (OSError, ValueError, KeyError, TypeError):
        pass
    return (1400.0, "fallback sustained (B200_PROFILING.md ~1.4 PFLOP/s under the power cap)") if sustained else \
        (1590.0, "fallback burst (B200_PROFILING.md 1.59 PFLOP/s)")


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _workload_desc(name, c, B, world):
    return (f"{name}: B={B}/rank T={c['T']} V={c['V']} {c['dtype']} logits x3 models resident in HBM, "
            f"adv={c['adv_kind']} gamma={c['gamma']} lambda={c['lam']} whiten={c['whiten']} "
            f"eps=({c['eps_low']},{c['eps_high']}) eps_v={c['eps_v']} kl={c.get('kl_mode', 'reward')}, "
            f"micro-batch {c['mb']} seq, all L_b = T")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle (CPU) leg
def _oracle_sample(logits_fn, batch_np, c, n_seq, cores):
    """Time the fp64 oracle on the first n_seq sequences: S1 for the three models
    (rows split over `cores` threads; ctypes releases the GIL), then the rest of
    the pipeline.  Returns (tokens, seconds)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor

    sh = {k: v[:n_seq] for k, v in batch_np.items()}
    T = sh["tokens"].shape[1]
    t0 = time.perf_counter()
    for role in ("old", "ref", "new"):
        x = logits_fn(role, n_seq)                       # host [n_seq, T, V]
        flat = x.reshape(n_seq * T, 1, x.shape[-1])
        tok = sh["tokens"].reshape(-1, 1)
        ones = np.minimum(np.arange(T)[None, :] < sh["lengths"][:, None], 1).astype(np.int32).reshape(-1)
        parts = np.array_split(np.arange(n_seq * T), cores)

        def work(idx):
            if idx.size == 0:
                return idx, None
            return idx, oracle.logprobs(flat[idx[0]:idx[-1] + 1], tok[idx[0]:idx[-1] + 1], ones[idx[0]:idx[-1] + 1])

        lp = np.zeros(n_seq * T)
        ent = np.zeros(n_seq * T)
        with ThreadPoolExecutor(cores) as ex:
            for idx, o in ex.map(work, parts):
                if o is not None:
                    lp[idx] = o["logp"][:, 0]
                    ent[idx] = o["entropy"][:, 0]
        sh[f"logp_{role}"] = lp.reshape(n_seq, T)
        if role == "new":
            sh["entropy_new"] = ent.reshape(n_seq, T)
    oracle.pipeline([sh], c)
    dt = time.perf_counter() - t0
    return int(np.minimum(sh["lengths"], T).sum()), dt


def run_reference(args):
    """--impl reference: the fp64 oracle on the host cores, bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2405_11143_b200 import synth

    c = dict(synth.CONFIGS[args.config])
    T, V = c["T"], c["V"]
    G = max(1, c["group_size"])
    n_seq = max(G, (args.ref_seqs // G) * G)               # whole groups (GRPO)
    cap = min(T, -(-(args.ref_seqs * min(T, 1024)) // n_seq))  # ~ref_seqs x 1024 valid tokens per step
    cores = len(os.sched_getaffinity(0))
    dev = torch.device("cuda:0") if torch.cuda.is_available() else torch.device("cpu")
    # only the first `cap` positions of each response are in the sample: generate [n_seq, cap, V]
    batch = synth.make_batch(1234, n_seq, cap, V, c["dtype"], "realistic", "full", c["rewards"],
                             c["group_size"], device=dev)
    bnp = synth.batch_to_numpy(batch)
    fn = lambda role, n: bnp[f"logits_{role}"][:n]  # noqa: E731
    times, toks = [], 0
    for i in range(args.warmup + args.steps):
        toks, dt = _oracle_sample(fn, {k: v for k, v in bnp.items() if not k.startswith("logits_")}, c, n_seq, cores)
        if i >= args.warmup:
            times.append(dt)
    mean = sum(times) / len(times)
    val = toks / mean
    sample = (f"{n_seq} sequences of {args.config} with lengths capped at {cap} ({toks} tokens, 3 x {toks} "
              f"vocab rows of V={V}), per step")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload_desc(args.config, c, n_seq, 1) + " (oracle sample)",
                       "global_batch": n_seq, "seq_len": T, "parallelism": "host threads"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch.distributed as dist

    from paper_2405_11143_b200 import orl, synth
    from paper_2405_11143_b200.pipeline import Buffers, PathConfig, run_iteration

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # ORL_BENCH_SHARED_GPU=1 (functional test of the N > 1 code path on a one-GPU box; its
    # timings are not measurements): every rank on cuda:0, gloo process group, no NCCL
    # communicator (two ranks cannot share a GPU in NCCL), C1/C2 over the peer kernels.
    shared = os.environ.get("ORL_BENCH_SHARED_GPU") == "1" and world > 1
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # under torchrun (even with one rank) use the distributed plumbing: NCCL process
    # group, unique-id broadcast, liborl NCCL communicator, barriers, max over ranks
    dist_mode = "WORLD_SIZE" in os.environ
    if shared:
        dist.init_process_group("gloo")
        ctx = orl.Context(local, world, rank, None)
    elif dist_mode:
        dist.init_process_group("nccl", device_id=dev)
        uid = [orl.orl_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = orl.Context(local, world, rank, uid[0])
    else:
        ctx = orl.Context(local)

    c = dict(synth.CONFIGS[args.config])
    B, T, V, mb = c["B"], c["T"], c["V"], c["mb"]
    if args.batch:
        B = args.batch
    pool_mb = 0
    cfg = PathConfig.from_synth(c)
    seed = 1234 + rank
    tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    elt = 2 if tdt == torch.bfloat16 else 4

    # ---- resident synthetic rollout (generated up front; not timed) ----------
    L = synth.lengths_for(B, T, seed, "full").to(dev)
    tok = synth.tokens_for(B, T, V, seed).to(dev)
    R = synth.rewards_for(B, seed, c["rewards"], c["group_size"]).to(dev)
    v_old, v_new = (v.to(dev) for v in synth.values_for(B, T, seed))
    full_bytes = 3 * B * T * V * elt
    pooled = full_bytes > 0.80 * torch.cuda.mem_get_info()[0]
    if pooled:
        # The three models' logits of this config do not fit in HBM (e.g. longcot
        # 3 x 79.7 GB, grpo 3 x 2.15 TB): every micro-batch streams from a pool of
        # `pool_mb` micro-batch buffers per model (>= 8 GB each, >> L2), filled once.
        per_mb = mb * T * V * elt
        pool_mb = max(1, min(len(range(0, B, mb)), int(0.70 * torch.cuda.mem_get_info()[0] // (3 * per_mb))))
        pool = {r: torch.empty(pool_mb * mb, T, V, dtype=tdt, device=dev) for r in synth.ROLES}
        for k in range(pool_mb):
            sl = slice(k * mb, (k + 1) * mb)
            synth.fill_logits_(tuple(pool[r][sl] for r in synth.ROLES), tok[sl], seed, k, "realistic")
        logits = None

        def src(role, s, e):
            k = (s // mb) % pool_mb
            return pool[role][k * mb:k * mb + (e - s)]
    else:
        logits = {r: torch.empty(B, T, V, dtype=tdt, device=dev) for r in synth.ROLES}
        for s in range(0, B, mb):
            e = min(B, s + mb)
            synth.fill_logits_(tuple(logits[r][s:e] for r in synth.ROLES), tok[s:e], seed, s // mb, "realistic")
        src = lambda role, s, e: logits[role][s:e]  # noqa: E731
    batch = dict(tokens=tok, lengths=L, seq_reward=R, values_old=v_old, values_new=v_new)
    bufs = Buffers(B, T, dev, c["group_size"])
    stream = torch.cuda.current_stream()
    n_tok_rank = int(L.clamp(max=T).sum().item())
    n_mb = len(range(0, B, mb))

    # K1 timing on the launching stream: one event before the first launch of each
    # pass (old / ref / actor) and one after its last launch, so the interval is the
    # wall time of that pass's back-to-back K1 launches (PDL lets consecutive K1
    # launches overlap their tail/prologue, so per-launch intervals would overlap).
    events = []      # (tag, n_launches, start_event, end_event)
    cur = {}

    def hook(tag):
        if cur.get("tag") != tag:
            a = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            cur.update(tag=tag, start=a, n=0)

        def done():
            cur["n"] += 1
            if cur["n"] == n_mb:
                b = torch.cuda.Event(enable_timing=True)
                b.record(stream)
                events.append((tag, cur["n"], cur["start"], b))
                cur.clear()
        return done

    def step(timing):
        return run_iteration(ctx, batch, cfg, bufs, src, mb, stream=stream, on_k1=hook if timing else None)

    # C1/C2 transport at N > 1: the single-kernel peer-memory collectives (orl_peer_open)
    # when every rank can map the others' exchange buffers, checked against the NCCL
    # all-gather path on the first warm-up steps (statistics must be bit-identical).
    coll = "local" if world == 1 else "nccl"
    if shared:
        ctx.enable_peer()
        coll = "peer (shared-GPU functional test: no NCCL reference)"
    elif world > 1 and args.collective == "peer":
        why = ""
        try:
            ctx.enable_peer()
            ok = 1.0
        except Exception as exc:  # mapping failed on this rank
            ok, why = 0.0, str(exc)[:80]
        t = torch.tensor([ok], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if t.item() == 1.0:
            try:
                ctx.set_collective("nccl")
                _, st_nccl = step(False)
                ctx.set_collective("peer")
                _, st_peer = step(False)
                same = 1.0 if st_nccl == st_peer else 0.0
                why = "" if same else "peer stats differed from NCCL"
            except Exception as exc:
                same, why = 0.0, str(exc)[:80]
            t = torch.tensor([same], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if t.item() == 1.0:
            coll = "peer (single-kernel C1/C2 over peer memory; stats bit-identical to NCCL in warm-up)"
        else:
            ctx.set_collective("nccl")
            coll = f"nccl ({why or 'peer path unavailable on another rank'})"
    for _ in range(args.warmup):
        status, st = step(False)
    torch.cuda.synchronize()
    if dist_mode:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    l0 = ctx.launch_count
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    t0, t1 = evs[0], evs[-1]
    t0.record(stream)
    for i in range(args.steps):
        status, st = step(True)
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    if dist_mode:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = (ctx.launch_count - l0) // args.steps
    ms = t0.elapsed_time(t1) / args.steps
    if dist_mode:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    total_tokens = n_tok_rank * world
    value = total_tokens / (ms / 1e3)

    # ---- the same step captured once as a CUDA graph and replayed ---------------
    graph = None
    if args.graph:
        graph = run_graph(args, ctx, batch, cfg, bufs, src, mb, dev, stream, world, total_tokens, status, st)

    # ---- roofline of the dominant kernel (K1) --------------------------------
    side = {"old": 8, "ref": 8 + 12, "new": 8 + 24 + 16}   # side bytes per token (DESIGN 5.1)
    k1_ms = sum(a.elapsed_time(b) for _, _, a, b in events)
    stage = {}
    for tag, _, a, b in events:
        stage[tag] = stage.get(tag, 0.0) + a.elapsed_time(b) / args.steps
    stage_ms = {"S1_old": round(stage.get("old", 0.0), 4), "S1-S3_ref": round(stage.get("ref", 0.0), 4),
                "S1_S7-S9_actor": round(stage.get("new", 0.0), 4),
                "S4-S6_C1_S10_C2_and_gaps": round(ms - sum(stage.values()), 4)}
    k1_bytes = 0
    for tag, n, _, _ in events:
        k1_bytes += n * (mb * T) * (V * elt + side[tag])
    k1_bytes = k1_bytes * (n_tok_rank / (B * T))           # only valid rows are read
    n_k1 = sum(n for _, n, _, _ in events)
    achieved = k1_bytes / (k1_ms / 1e3) / 1e9
    peak, peak_src = _peaks()
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            for e in pj.get("configs", [pj]):   # one ncu capture per (V, T, micro-batch) shape
                if e.get("V") == V and e.get("T") == T and e.get("mb") == mb:
                    traffic = e["dram_bytes_per_launch"]
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "kernel": "k1_tma_kernel (S1 + epilogues)", "launches_per_step": n_k1 // args.steps,
            "algorithmic_bytes_per_launch": int(k1_bytes / max(n_k1, 1)), "k1_share_of_step": round(k1_ms / (ms * args.steps), 4),
            "peak_source": peak_src}

    # ---- NEXT-1: the backward pass dL/dlogits (separate leg, not in `value`) ----
    next1 = None
    if not args.no_next1 and world == 1 and not pooled:
        next1 = run_next1(args, ctx, c, cfg, batch, logits, bufs, mb, dev, stream, n_tok_rank)

    # ---- NEXT-4: the same iteration from final hidden states (LM head fused) ---
    next4 = None
    if args.next4 and world == 1 and not pooled:
        next4 = run_next4(args, ctx, c, cfg, batch, bufs, mb, dev, stream, n_tok_rank)

    # ---- e2e: host buffers, H2D/D2H inside the timed region --------------------
    e2e = None
    if not args.no_e2e and not pooled:
        e2e = run_e2e(args, ctx, c, cfg, batch, logits, bufs, mb, dev, world, total_tokens, rank)

    # ---- oracle on the host cores (rank 0, N = 1 only) ------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = len(os.sched_getaffinity(0))
        G = max(1, c["group_size"])

        def sample(n_want, tok_cap, ncores):
            """Whole groups of the first sequences, lengths capped so the sample holds
            about tok_cap valid tokens (the oracle's per-token cost is the 3 V-long rows)."""
            n = max(G, (n_want // G) * G)
            n = min(n, mb) if pooled else n
            n = max(G, (n // G) * G)
            bnp = {k: v[:n].detach().cpu().numpy() for k, v in batch.items()}
            cap = max(1, -(-tok_cap // n))
            bnp["lengths"] = np.minimum(bnp["lengths"], cap).astype(np.int32)
            hl = {r: synth.to_numpy_logits(src(r, 0, n)) for r in synth.ROLES}
            toks, dt = _oracle_sample(lambda role, k: hl[role][:k], bnp, c, n, ncores)
            desc = (f"first {n} sequences of the same rollout, lengths capped at {min(cap, T)} "
                    f"({toks} tokens, 3 x {toks} vocab rows), {dt:.1f} s wall")
            return toks / dt, desc

        v_all, d_all = sample(args.ref_seqs, args.ref_seqs * min(T, 1024), cores)
        cpu = {"value": v_all, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": d_all,
               "cpu_model": _cpu_model()}
        # the same oracle on one core (1-core and all-core)
        v_one, d_one = sample(1, 1024, 1)
        cpu["single_core"] = {"value": v_one, "unit": UNIT, "cores": 1, "sample": d_one}
        # the whole step's oracle time extrapolated from the sample, and the ratio
        cpu["extrapolated_step_s"] = round(total_tokens / v_all, 1)
        cpu["gpu_over_cpu"] = round(value / v_all, 1)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 4),
                "stage_ms_per_step": stage_ms, "ms_per_step_stats": {"mean": round(statistics.mean(per_step), 4),
                                      "median": round(statistics.median(per_step), 4),
                                      "min": round(min(per_step), 4), "max": round(max(per_step), 4),
                                      "rank": "rank 0 (value uses the max over ranks of the mean)"}, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": c["dtype"], "data": "synthetic",
                "config": {"workload": _workload_desc(args.config, c, B, world), "global_batch": B * world,
                           "seq_len": T, "vocab": V, "parallelism": f"dp{world}", "collective": coll,
                           "l2": "inputs larger than L2 (3 x %.1f GB logits per rank vs 126 MB L2)" % (B * T * V * elt / 1e9),
                           "logits": ("pool of %d micro-batch buffers per model reused across the %d micro-batches "
                                      "(full batch does not fit)" % (pool_mb, n_mb)) if pooled else "resident"},
                "status": status, "stats": {k: (round(v, 6) if isinstance(v, float) else v) for k, v in st.items()},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": int(launches),
                "next1_logits_grad": next1, "next4_lmhead": next4, "graph_replay": graph,
                "per_gpu_tokens_per_s": round(value / world, 1)}
        if shared:
            line["test_mode"] = "ORL_BENCH_SHARED_GPU: all ranks on one GPU (functional test, not a measurement)"
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist_mode:
        dist.destroy_process_group()


def run_graph(args, ctx, batch, cfg, bufs, src, mb, dev, stream, world, total_tokens, status_eager, st_eager):
    """The timed step (all S1..S10 launches, C1/C2 included) captured once into a CUDA
    graph (pipeline.GraphStep, orl_finalize_async) and replayed K times; the replayed
    statistics must equal the eager step's bit for bit."""
    import torch.distributed as dist

    from paper_2405_11143_b200.pipeline import GraphStep

    step = GraphStep(ctx, batch, cfg, bufs, src, mb)
    gs = torch.cuda.current_stream()
    for _ in range(2):
        step.replay()
    torch.cuda.synchronize()
    same = step.result() == (status_eager, st_eager)
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(gs)
    for _ in range(args.steps):
        step.replay()
    b.record(gs)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    if dist.is_initialized():
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    return {"tokens_per_s": round(total_tokens / (ms / 1e3), 1), "ms_per_step": round(ms, 4),
            "kernels_per_graph": int(step.kernels), "graph_launches_per_step": 1,
            "stats_bit_identical_to_eager": bool(same), "steps": args.steps}


def run_next1(args, ctx, c, cfg, batch, logits, bufs, mb, dev, stream, n_tok):
    """Time the NEXT-1 backward pass (orl_logits_grad) over every micro-batch of
    the actor logits: reads V*2 B and writes V*2 B per token.  Uses the per-token
    lse / entropy / dloss_dlogp the timed steps left in `bufs`."""
    from paper_2405_11143_b200 import orl

    B, T, V = batch["tokens"].shape[0], c["T"], c["V"]
    free = torch.cuda.mem_get_info()[0]
    need = B * T * V * 2
    if need > free - (4 << 30):
        return {"skipped": f"needs {need / 1e9:.1f} GB for dlogits"}
    dl = torch.empty(B, T, V, dtype=logits["new"].dtype, device=dev)
    tok, L = batch["tokens"], batch["lengths"]

    def once():
        for s in range(0, B, mb):
            e = min(B, s + mb)
            orl.orl_logits_grad(ctx, tok, L, logits["new"][s:e], cfg.ppo, bufs.lse, bufs.entropy, bufs.dlogp,
                                dl[s:e], seq_offset=s, inv_temp=cfg.inv_temp, stream=stream)

    def fused():
        critic = cfg.critic
        for s in range(0, B, mb):
            e = min(B, s + mb)
            orl.orl_ppo_loss_and_grad(ctx, tok, L, logits["new"][s:e], cfg.ppo, bufs.logp_old, bufs.adv,
                                      bufs.logp_new, seq_offset=s, inv_temp=cfg.inv_temp, logp_ref=bufs.logp_ref,
                                      ret=bufs.ret if critic else None,
                                      v_new=batch["values_new"] if critic else None,
                                      v_old=batch["values_old"] if critic else None, entropy=bufs.entropy,
                                      lse=bufs.lse, dloss_dlogp=bufs.dlogp, dloss_dv=bufs.dv if critic else None,
                                      dlogits=dl[s:e], stream=stream)

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    reps = max(3, args.steps // 4)
    ms = timed(once)
    byts = n_tok * V * 2 * 2
    peak, _ = _peaks()
    # fused actor pass (loss epilogue + backward, the row re-read from L2); its
    # bytes are those of the two-pass path minus the HBM re-read it avoids
    ms_f = timed(fused)
    del dl
    torch.cuda.empty_cache()
    return {"tokens_per_s": round(n_tok / (ms / 1e3), 1), "ms_per_pass": round(ms, 4),
            "roofline": {"bound": "hbm", "achieved": round(byts / (ms / 1e3) / 1e9, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(byts / (ms / 1e3) / 1e9 / peak, 4),
                         "bytes": "V*2 read + V*2 written per valid token"},
            "kernel": "k5_tma_kernel", "launches": len(range(0, B, mb)), "reps": reps,
            "fused_actor_pass": {"api": "orl_ppo_loss_and_grad", "tokens_per_s": round(n_tok / (ms_f / 1e3), 1),
                                 "ms": round(ms_f, 4),
                                 "algorithmic_GBps": round(byts / (ms_f / 1e3) / 1e9, 1)}}


def run_next4(args, ctx, c, cfg, batch, bufs, mb, dev, stream, n_tok):
    """NEXT-4 leg (not part of `value`): the whole iteration with every S1 pass computed
    from the model's final hidden states through its LM head, [R, d] x [V, d]^T on the
    tcgen05 tensor cores fused with the online log-sum-exp (K6, orl_lmhead_*), against
    the unfused baseline: cuBLAS bf16 GEMM (torch.matmul) writing each micro-batch's
    logits to HBM, then K1.  d = 4096 (Llama-3-8B hidden size)."""
    from paper_2405_11143_b200 import synth
    from paper_2405_11143_b200.pipeline import LmHeadRows, run_iteration

    B, T, V, d = batch["tokens"].shape[0], c["T"], c["V"], args.hidden
    R = B * T
    g = torch.Generator(device=dev).manual_seed(synth.role_seed(4321, 30_000, 0))
    # as synth.make_lmhead_batch: hidden_old = s_r N(0, I), ref = old + 0.05 N, new = old + 0.03 N
    hid = {r: torch.empty(R, d, dtype=torch.bfloat16, device=dev) for r in synth.ROLES}
    for s in range(0, R, 16384):
        e = min(R, s + 16384)
        base = torch.randn(e - s, d, generator=g, device=dev) * (torch.rand(e - s, 1, generator=g, device=dev) + 0.5)
        for r, sd in zip(synth.ROLES, (0.0, 0.05, 0.03)):
            hid[r][s:e] = (base + sd * torch.randn(e - s, d, generator=g, device=dev)).to(torch.bfloat16)
    W = torch.empty(V, d, dtype=torch.bfloat16, device=dev)
    for s in range(0, V, 8192):
        e = min(V, s + 8192)
        W[s:e] = (torch.randn(e - s, d, generator=g, device=dev) * (3.0 / d ** 0.5)).to(torch.bfloat16)
    fused_src = lambda role, s, e: LmHeadRows(hid[role][s * T:e * T], W)  # noqa: E731
    scratch = torch.empty(mb * T, V, dtype=torch.bfloat16, device=dev)

    def unfused_src(role, s, e):
        out = scratch[: (e - s) * T]
        torch.matmul(hid[role][s * T:e * T], W.t(), out=out)
        return out.view(e - s, T, V)

    def timed(src, reps):
        for _ in range(2):
            run_iteration(ctx, batch, cfg, bufs, src, mb, stream=stream)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            status, st = run_iteration(ctx, batch, cfg, bufs, src, mb, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps, status, st

    reps = max(2, args.steps // 5)
    l0 = ctx.launch_count
    ms_f, status, st = timed(fused_src, reps)
    launches = (ctx.launch_count - l0) // (reps + 2)
    ms_u, status_u, st_u = timed(unfused_src, reps)
    flops = 3 * 2.0 * R * d * V
    peak, peak_src = _bf16_peak(sustained=True)
    ach = flops / (ms_f / 1e3) / 1e12
    del scratch
    e2e = None if args.no_e2e else _next4_e2e(ctx, cfg, batch, bufs, mb, hid, W, T, n_tok, reps)
    del hid, W
    torch.cuda.empty_cache()
    return {"tokens_per_s": round(n_tok / (ms_f / 1e3), 1), "ms_per_step": round(ms_f, 3), "status": status,
            "hidden": d, "reps": reps, "gpu_launches": int(launches),
            "policy_loss": round(st["policy_loss"], 6), "entropy": round(st["entropy"], 6),
            "roofline": {"bound": "tensor", "achieved": round(ach, 1), "peak": peak, "unit": "TFLOP/s",
                         "frac": round(ach / peak, 4), "flops": "3 x 2 R d V per step (old, ref, actor heads)",
                         "peak_source": peak_src, "kernel": "k6_lmhead_2sm_kernel + k6_merge_kernel (whole step)"},
            "unfused_cublas_plus_k1": {"tokens_per_s": round(n_tok / (ms_u / 1e3), 1), "ms_per_step": round(ms_u, 3),
                                       "status": status_u, "policy_loss": round(st_u["policy_loss"], 6)},
            "speedup_vs_unfused": round(ms_u / ms_f, 4), "e2e_from_host_hidden_states": e2e}


def _next4_e2e(ctx, cfg, batch, bufs, mb, hid, W, T, n_tok, steps):
    """NEXT-4 end to end through the public API with the step's inputs in pinned HOST
    memory: every step copies the LM-head weight and each micro-batch's final hidden
    states of the three roles host -> device (double-buffered on a copy stream, the
    copies overlapping the tensor-core work) plus the per-token inputs, and
    orl_finalize reads the statistics back and synchronises (host clock)."""
    from paper_2405_11143_b200.pipeline import LmHeadRows, run_iteration

    B = batch["tokens"].shape[0]
    hh = {r: v.cpu().pin_memory() for r, v in hid.items()}
    hW = W.cpu().pin_memory()
    small = {k: v.cpu().pin_memory() for k, v in batch.items()}
    dW = torch.empty_like(W)
    stage = [torch.empty(mb * T, W.shape[1], dtype=W.dtype, device=W.device) for _ in range(2)]
    dbatch = {k: torch.empty_like(v) for k, v in batch.items()}
    comp, copy = torch.cuda.current_stream(), torch.cuda.Stream()
    order = [(r, s) for r in ("old", "ref", "new") for s in range(0, B, mb)]
    h2d = sum(v.numel() * v.element_size() for v in small.values()) + hW.numel() * hW.element_size()
    h2d += sum(v.numel() * v.element_size() for v in hh.values())

    def one_step():
        for k, v in small.items():
            dbatch[k].copy_(v, non_blocking=True)
        with torch.cuda.stream(copy):
            dW.copy_(hW, non_blocking=True)
            ew = torch.cuda.Event()
            ew.record(copy)
        slot_free, pending, counter = [None, None], {}, {"i": 0}

        def fetch(i):
            r, s = order[i]
            e = min(B, s + mb)
            with torch.cuda.stream(copy):
                if slot_free[i % 2] is not None:
                    copy.wait_event(slot_free[i % 2])
                stage[i % 2][: (e - s) * T].copy_(hh[r][s * T:e * T], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            pending[i] = ev

        def src(role, s, e):
            i = counter["i"]
            counter["i"] += 1
            if i == 0:
                comp.wait_event(ew)
            comp.wait_event(pending.pop(i))
            if i + 1 < len(order):
                fetch(i + 1)
            return LmHeadRows(stage[i % 2][: (e - s) * T], dW)

        def hook(tag):
            def after():
                ev = torch.cuda.Event()
                ev.record(comp)
                slot_free[(counter["i"] - 1) % 2] = ev
            return after

        fetch(0)
        return run_iteration(ctx, dbatch, cfg, bufs, src, mb, stream=comp, on_k1=hook)

    one_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        status, _ = one_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    del hh, hW, dW, stage
    return {"value": round(n_tok / dt, 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": 16 * 8 + 4 * 8, "steps": steps, "status": status,
            "note": "final hidden states (3 roles) + LM-head weight streamed from pinned host memory each step; "
                    "host clock"}


def run_e2e(args, ctx, c, cfg, batch, logits, bufs, mb, dev, world, total_tokens, rank):
    """Same iteration through the public API with the step's inputs in pinned
    HOST memory: every step copies each micro-batch's three logits blocks plus
    the per-token inputs host->device (double-buffered on a copy stream) and
    orl_finalize reads the stats back (D2H) and synchronises.  The pinned pool
    holds one micro-batch per role and is re-sent for every micro-batch, so the
    bytes moved per step are the full step's."""
    import torch.distributed as dist

    from paper_2405_11143_b200.pipeline import run_iteration

    B = batch["tokens"].shape[0]
    host = {r: logits[r][:mb].cpu().pin_memory() for r in logits}
    small = {k: v.cpu().pin_memory() for k, v in batch.items()}
    stage = [{r: torch.empty_like(logits[r][:mb]) for r in logits} for _ in range(2)]
    dbatch = {k: torch.empty_like(v) for k, v in batch.items()}
    comp, copy = torch.cuda.current_stream(), torch.cuda.Stream()
    order = [(r, s) for r in ("old", "ref", "new") for s in range(0, B, mb)]
    h2d = sum(v.numel() * v.element_size() for v in small.values())
    h2d += sum((min(B, s + mb) - s) * host[r][0].numel() * host[r].element_size() for r, s in order)
    d2h = 16 * 8 + 4 * 8

    def one_step():
        for k, v in small.items():
            dbatch[k].copy_(v, non_blocking=True)
        slot_free = [None, None]
        pending = {}
        counter = {"i": 0}

        def fetch(i):
            r, s = order[i]
            e = min(B, s + mb)
            with torch.cuda.stream(copy):
                if slot_free[i % 2] is not None:
                    copy.wait_event(slot_free[i % 2])
                stage[i % 2][r][: e - s].copy_(host[r][: e - s], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            pending[i] = ev

        def src(role, s, e):
            i = counter["i"]
            counter["i"] += 1
            comp.wait_event(pending.pop(i))
            if i + 1 < len(order):
                fetch(i + 1)
            return stage[i % 2][role][: e - s]

        def hook(tag):
            def after():
                i = counter["i"] - 1
                ev = torch.cuda.Event()
                ev.record(comp)
                slot_free[i % 2] = ev          # slot i%2 may be refilled after this K1
            return after

        fetch(0)
        return run_iteration(ctx, dbatch, cfg, bufs, src, mb, stream=comp, on_k1=hook)

    steps = max(2, args.steps // 5)
    one_step()
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    if dist.is_initialized():
        tt = torch.tensor([dt], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    del stage, host
    return {"value": round(total_tokens / dt, 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": d2h, "steps": steps,
            "note": "logits streamed from pinned host memory over PCIe each step (double-buffered); host clock"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=10,
                    help="untimed steps; default 10: the paper excludes the first 10 steps (P:94, S:535)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--batch", type=int, default=0, help="override B per rank (testing)")
    ap.add_argument("--ref-seqs", type=int, default=4, help="oracle sample size (sequences)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-next1", action="store_true")
    ap.add_argument("--next4", type=int, default=1, help="run the NEXT-4 LM-head leg (1/0)")
    ap.add_argument("--collective", default="peer", choices=["peer", "nccl"],
                    help="C1/C2 transport at N > 1 (peer: single peer-memory kernels, NCCL-checked)")
    ap.add_argument("--hidden", type=int, default=4096, help="NEXT-4 hidden size d")
    ap.add_argument("--graph", type=int, default=1, help="time the CUDA-graph replay of the step (1/0)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
